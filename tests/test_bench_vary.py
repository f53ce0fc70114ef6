"""The GPU scaling bench (scripts/bench_vary.py, reference bench.cpp / criterion 8):
CPU checks of the host logic; one small GPU run."""
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "scripts"))

import bench_vary  # noqa: E402
from paper_1709_09479_b200 import dcsc  # noqa: E402


def test_fit_r_squared_restatement():
    assert bench_vary.fit_r_squared([1, 2, 3, 4], [2, 4, 6, 8]) == pytest.approx(1.0)
    x = [1.0, 2.0, 3.0, 4.0]
    y = [1.0, 3.0, 2.0, 5.0]
    b, a = np.polyfit(x, y, 1)
    pred = a + b * np.array(x)
    ref = 1 - ((np.array(y) - pred) ** 2).sum() / ((np.array(y) - np.mean(y)) ** 2).sum()
    assert bench_vary.fit_r_squared(x, y) == pytest.approx(ref)


def test_bench_csv_format(tmp_path):
    rows = [{"varied_value": 4.0, "phase": "coding", "mean_ms_per_outer": 1.5, "std_ms": 0.1},
            {"varied_value": 4.0, "phase": "learning", "mean_ms_per_outer": 2.25, "std_ms": 0.0}]
    p = tmp_path / "b.csv"
    bench_vary.write_bench_csv(str(p), rows)
    assert p.read_text() == ("varied_value,phase,mean_ms_per_outer_iter,std_ms\n"
                             "4,coding,1.5,0.10000000000000001\n4,learning,2.25,0\n")


def test_bench_rejects_bad_grids():
    with pytest.raises(ValueError):
        bench_vary.run_bench("k", [], 1, (16, 16), (3, 3), 2, 1, 1, 0.5, 1, 64, 10, 10, 0)
    with pytest.raises(ValueError):
        bench_vary.run_bench("k", [1.0], 0, (16, 16), (3, 3), 2, 1, 1, 0.5, 1, 64, 10, 10, 0)


def test_synth_dataset_matches_reference_generator():
    from oracle import dcsc_np
    x = dcsc.synth_dataset(2, 1, (4, 5), 7)
    rng = dcsc_np._MT19937_64(7)
    want = np.array([(rng.next() >> 11) * 2.0 ** -53 for _ in range(40)]).reshape(2, 4, 5)
    assert np.array_equal(x, want)


@pytest.mark.gpu
def test_bench_vary_runs_on_gpu(tmp_path):
    out = tmp_path / "b.csv"
    r = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "bench_vary.py"), "--vary", "n", "--grid",
                        "1,2", "--size", "20x20", "--filter-size", "5x5", "--filters", "4", "--outer", "2",
                        "--precision", "64", "--max-admm", "20", "--cg-max", "20", "--out", str(out)],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    lines = out.read_text().splitlines()
    assert lines[0] == "varied_value,phase,mean_ms_per_outer_iter,std_ms" and len(lines) == 5
