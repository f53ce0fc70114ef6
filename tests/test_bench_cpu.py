"""bench.py's reference arm runs on CPU (the compiled reference solver on the
host cores): its JSON line carries the contract's keys, it never maps the CUDA
product library, under a multi-process launch only rank 0 prints, and
`--gpus N` outside torchrun spawns N ranks itself."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(extra_env=None, *args):
    env = dict(os.environ, **(extra_env or {}))
    env.pop("WORLD_SIZE", None) if not (extra_env and "WORLD_SIZE" in extra_env) else None
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                           "--warmup", "0", "--config", "c4", *args], capture_output=True, text=True, env=env,
                          timeout=900, cwd=ROOT)


def _check_line(d, n_gpus):
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference" and d["value"] > 0 and d["n_gpus"] == n_gpus
    assert d["config"]["workload"].startswith("C4")
    cb = d["cpu_baseline"]
    assert cb["kind"] == "reference" and cb["cores"] >= 1 and cb["sample"] and cb["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["timed_outer_iters"] == [1]


def test_reference_arm_json_line():
    r = _run()
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1
    _check_line(json.loads(lines[0]), 1)


def test_reference_arm_other_ranks_are_silent():
    r = _run({"RANK": "1", "WORLD_SIZE": "2", "LOCAL_RANK": "1"}, "--gpus", "2")
    assert r.returncode == 0, r.stderr[-2000:]
    assert r.stdout.strip() == ""


def test_gpus_flag_spawns_ranks():
    """`--gpus 2` outside torchrun re-launches under torch.distributed.run: two
    processes, rank 0 alone prints one line with n_gpus = 2."""
    r = _run(None, "--gpus", "2")
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1, r.stdout
    _check_line(json.loads(lines[0]), 2)
