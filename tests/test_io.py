"""CPU: the product's CSCT tensor and trace-CSV formats are byte-compatible
with the reference's tensor_io.cpp / trace_io.cpp (compiled into oracle/_ref)."""
import numpy as np
import pytest

from oracle import ref
from paper_1709_09479_b200 import dcsc

pytestmark = pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")


@pytest.mark.parametrize("shape", [(7,), (3, 1, 5, 5), (2, 16, 20)])
def test_tensor_bytes_match_reference(tmp_path, shape):
    v = np.random.default_rng(sum(shape)).standard_normal(shape)
    v.flat[0] = -0.0
    a, b = str(tmp_path / "ours.csct"), str(tmp_path / "ref.csct")
    dcsc.write_tensor(a, v)
    ref.write_tensor(b, v)
    assert open(a, "rb").read() == open(b, "rb").read()
    assert np.array_equal(dcsc.read_tensor(b), v)
    assert np.array_equal(ref.read_tensor(a, shape), v)


def test_tensor_reader_rejects_bad_files(tmp_path):
    p = tmp_path / "t.csct"
    dcsc.write_tensor(str(p), np.arange(6.0).reshape(2, 3))
    raw = p.read_bytes()
    (tmp_path / "magic.csct").write_bytes(b"XSCT" + raw[4:])
    (tmp_path / "short.csct").write_bytes(raw[:-3])
    (tmp_path / "trail.csct").write_bytes(raw + b"\0")
    for name in ("magic", "short", "trail"):
        with pytest.raises(dcsc.IoError):
            dcsc.read_tensor(str(tmp_path / f"{name}.csct"))


def test_trace_csv_bytes_match_reference(tmp_path):
    trace = [
        dict(outer_iter=1, phase=0, total=100.57070864605366, data_term=90.1, l1_term=10.47070864605366,
             admm_iters=1500, cg_iters=0, elapsed_ms=12.25),
        dict(outer_iter=1, phase=1, total=98.04522157273809, data_term=87.57451292668443, l1_term=10.47070864605366,
             admm_iters=0, cg_iters=631, elapsed_ms=3.0e-3),
    ]
    a, b = str(tmp_path / "ours.csv"), str(tmp_path / "ref.csv")
    dcsc.write_trace_csv(a, trace)
    ref.write_trace_csv(b, trace)
    assert open(a, "rb").read() == open(b, "rb").read()
    back = dcsc.read_trace_csv(b)
    assert [r["phase"] for r in back] == [0, 1]
    assert back[1]["cg_iters"] == 631 and back[0]["total"] == trace[0]["total"]


def test_trace_reader_rejects_bad_header(tmp_path):
    p = tmp_path / "bad.csv"
    p.write_text("outer,phase\n1,coding\n")
    with pytest.raises(dcsc.IoError):
        dcsc.read_trace_csv(str(p))
