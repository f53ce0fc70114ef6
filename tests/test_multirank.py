"""Multi-rank paths with world_size 2 over gloo (127.0.0.1).

CPU: the host all-reduce callback and the image sharding.
GPU: two ranks sharing one GPU (host-side gloo reductions only, no kernel
waits on another rank) reproduce a single-rank run_csc: the sharded learning
(correlation partials + CG scalars summed over ranks) gives the same trace.
"""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from paper_1709_09479_b200 import dcsc

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
WORKER = os.path.join(ROOT, "tests", "mr", "worker.py")


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def launch(world, mode, tmp_path, extra_env=None):
    port = free_port()
    procs, outs = [], []
    for r in range(world):
        out = str(tmp_path / f"rank{r}.npz")
        env = dict(os.environ, RANK=str(r), WORLD_SIZE=str(world), MASTER_ADDR="127.0.0.1",
                   MASTER_PORT=str(port), MR_OUT=out, MR_MODE=mode, **(extra_env or {}))
        procs.append(subprocess.Popen([sys.executable, WORKER], env=env, stdout=subprocess.PIPE,
                                      stderr=subprocess.STDOUT, text=True))
        outs.append(out)
    for p in procs:
        o, _ = p.communicate(timeout=600)
        assert p.returncode == 0, o[-3000:]
    return [np.load(o) for o in outs]


def test_shard_ranges_cover_all_images():
    for n in (1, 7, 10, 256, 2048):
        for w in (1, 2, 3, 8):
            rs = [dcsc.shard_range(n, w, r) for r in range(w)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
            assert max(b - a for a, b in rs) - min(b - a for a, b in rs) <= 1


def test_gloo_allreduce_callback_two_ranks(tmp_path):
    res = launch(2, "cpu", tmp_path)
    expect = (np.arange(5) + 1.0) * 3.0
    for r in res:
        assert int(r["rc"]) == 0
        assert np.array_equal(r["buf"], expect)
    assert list(res[0]["shard"]) == [0, 5] and list(res[1]["shard"]) == [5, 10]


@pytest.mark.gpu
def test_two_ranks_match_single_rank(tmp_path):
    res = launch(2, "gpu", tmp_path)
    N, grid, K, m = 4, (20, 20), 6, 5
    x, _ = dcsc.synth_generate(N, grid, K, m, 0.05, 0.01, 7, False)
    cfg = dcsc.SolverConfig(beta=0.2, max_outer=3, normalize=0, seed=11, tol=1e-300)
    one = dcsc.run_csc(x, K, (m, m), cfg, precision=64)
    keys = ["total", "data_term", "l1_term", "admm_iters", "cg_iters", "mu_iters", "l0"]
    single = np.array([[r[k] for k in keys] for r in one["trace"]], dtype=np.float64)
    for r in res:
        t = r["trace"]
        assert t.shape == single.shape
        assert np.all(np.abs(t[:, :3] - single[:, :3]) <= 1e-9 * np.abs(single[:, :3]))
        assert np.array_equal(t[:, 3], single[:, 3]) and np.array_equal(t[:, 5], single[:, 5])
        assert np.all(np.abs(t[:, 4] - single[:, 4]) <= 2)
        assert np.abs(r["dict"] - one["dict"]).max() <= 1e-8 * np.abs(one["dict"]).max()
    maps = np.concatenate([res[0]["maps"], res[1]["maps"]])
    assert np.abs(maps - one["maps"]).max() <= 1e-8 * np.abs(one["maps"]).max()


@pytest.mark.gpu
def test_two_ranks_match_single_rank_joint_channels(tmp_path):
    """Joint mode (J = 2): per-channel CG under the shared mu ascent, sharded over ranks."""
    sys.path.insert(0, os.path.join(ROOT, "tests", "mr"))
    import worker  # noqa: E402
    res = launch(2, "gpu_j", tmp_path)
    N, grid, K, m = 4, (20, 20), 6, 5
    x = worker.mr_signals(dcsc, N, grid, K, m, 2)
    cfg = dcsc.SolverConfig(beta=0.2, max_outer=3, normalize=0, seed=11, tol=1e-300)
    one = dcsc.run_csc(x, K, (m, m), cfg, precision=64)
    keys = ["total", "data_term", "l1_term", "admm_iters", "cg_iters", "mu_iters", "l0"]
    single = np.array([[r[k] for k in keys] for r in one["trace"]], dtype=np.float64)
    for r in res:
        t = r["trace"]
        assert t.shape == single.shape
        assert np.all(np.abs(t[:, :3] - single[:, :3]) <= 1e-9 * np.abs(single[:, :3]))
        assert np.array_equal(t[:, 3], single[:, 3]) and np.array_equal(t[:, 5], single[:, 5])
        assert np.abs(r["dict"] - one["dict"]).max() <= 1e-8 * np.abs(one["dict"]).max()


@pytest.mark.gpu
def test_nccl_reducer_one_rank_multi_paths_match_single_rank():
    """The NCCL reducer end to end on one GPU: a 1-rank communicator with
    DCSC_FORCE_MULTI=1 takes every multi-rank path (crop-then-all-reduce of the
    correlations, all-reduced CG scalars and trace sums) through ncclAllReduce;
    the run must equal the plain single-rank run (FP64)."""
    import subprocess
    import sys

    code = r'''
import json, os, sys
import numpy as np
sys.path.insert(0, os.getcwd())
from paper_1709_09479_b200 import dcsc
x, _ = dcsc.synth_generate(3, (20, 20), 5, 5, 0.05, 0.01, 17, False)
cfg = dcsc.SolverConfig(beta=0.2, max_outer=3, normalize=0, seed=4, tol=1e-300)
out = {}
for mode in ("plain", "nccl"):
    with dcsc.Context(3, (20, 20), 5, (5, 5), cfg, 64) as ctx:
        if mode == "nccl":
            ctx.set_comm_nccl(1, 0, dcsc.nccl_unique_id())
        ctx.set_signals(x)
        ctx.init_variables()
        rows, _ = ctx.run(3)
        out[mode] = ([r["total"] for r in rows], [r["cg_iters"] for r in rows], ctx.get_dictionary().tolist())
print(json.dumps(out))
'''
    env = dict(os.environ, DCSC_FORCE_MULTI="1")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, timeout=600,
                       cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert r.returncode == 0, r.stderr[-3000:]
    import json
    out = json.loads(r.stdout.strip().splitlines()[-1])
    (tp, cp, dp), (tn, cn, dn) = out["plain"], out["nccl"]
    assert cp == cn
    assert max(abs(a - b) / abs(b) for a, b in zip(tn, tp)) <= 1e-10
    assert np.abs(np.array(dn) - np.array(dp)).max() <= 1e-9


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3])
def test_frequency_sharded_learning_matches_single_rank(tmp_path, world):
    """Frequency-sharded learning (BASELINE.json north_star): ranks own
    contiguous bin ranges of every image's spectra after the z_hat / x_hat
    all-to-all (here through the gloo callback, ranks sharing one GPU; 3 ranks:
    uneven image and bin splits); the run equals the single-rank run (FP64)."""
    res = launch(world, "gpu_freq", tmp_path)
    N, grid, K, m = 4, (20, 20), 6, 5
    x, _ = dcsc.synth_generate(N, grid, K, m, 0.05, 0.01, 7, False)
    cfg = dcsc.SolverConfig(beta=0.2, max_outer=3, normalize=0, seed=11, tol=1e-300)
    one = dcsc.run_csc(x, K, (m, m), cfg, precision=64)
    keys = ["total", "data_term", "l1_term", "admm_iters", "cg_iters", "mu_iters", "l0"]
    single = np.array([[r[k] for k in keys] for r in one["trace"]], dtype=np.float64)
    for r in res:
        t = r["trace"]
        assert t.shape == single.shape
        assert np.all(np.abs(t[:, :3] - single[:, :3]) <= 1e-9 * np.abs(single[:, :3]))
        assert np.array_equal(t[:, 3], single[:, 3]) and np.array_equal(t[:, 5], single[:, 5])
        assert np.all(np.abs(t[:, 4] - single[:, 4]) <= 2)
        assert np.abs(r["dict"] - one["dict"]).max() <= 1e-8 * np.abs(one["dict"]).max()


@pytest.mark.gpu
def test_nccl_frequency_sharded_one_rank_matches_single_rank():
    """The NCCL all-to-all (grouped ncclSend / ncclRecv to itself) and the
    frequency-sharded learning code path on a forced 1-rank communicator."""
    code = r'''
import json, os, sys
import numpy as np
sys.path.insert(0, os.getcwd())
from paper_1709_09479_b200 import dcsc
x, _ = dcsc.synth_generate(3, (20, 20), 5, 5, 0.05, 0.01, 17, False)
cfg = dcsc.SolverConfig(beta=0.2, max_outer=3, normalize=0, seed=4, tol=1e-300)
out = {}
for mode in ("plain", "freq"):
    with dcsc.Context(3, (20, 20), 5, (5, 5), cfg, 64) as ctx:
        if mode == "freq":
            ctx.set_comm_nccl(1, 0, dcsc.nccl_unique_id())
            ctx.set_learning_layout("freq")
        ctx.set_signals(x)
        rows, _ = ctx.run(3)
        out[mode] = ([r["total"] for r in rows], [r["cg_iters"] for r in rows], ctx.get_dictionary().tolist())
print(json.dumps(out))
'''
    env = dict(os.environ, DCSC_FORCE_MULTI="1")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    import json
    out = json.loads(r.stdout.strip().splitlines()[-1])
    (tp, cp, dp), (tn, cn, dn) = out["plain"], out["freq"]
    assert cp == cn
    assert max(abs(a - b) / abs(b) for a, b in zip(tn, tp)) <= 1e-10
    assert np.abs(np.array(dn) - np.array(dp)).max() <= 1e-9


@pytest.mark.gpu
def test_two_ranks_tensor_core_coding_match_single_rank(tmp_path, monkeypatch):
    """Image-sharded coding on the tensor-core pass (each rank's images as two
    half-batches on two streams) + sharded learning reproduce a single-rank FP32
    run at the FP32 tolerance with equal ADMM iteration counts."""
    res = launch(2, "gpu_tc", tmp_path, {"DCSC_TC": "1"})
    monkeypatch.setenv("DCSC_TC", "1")
    N, grid, K, m = 4, (128, 128), 8, 11
    x, _ = dcsc.synth_generate(N, grid, K, m, 0.05, 0.01, 7, False)
    cfg = dcsc.SolverConfig(beta=0.5, max_outer=3, max_admm=60, normalize=0, seed=11, tol=1e-300)
    one = dcsc.run_csc(x, K, (m, m), cfg, precision=32)
    keys = ["total", "data_term", "l1_term", "admm_iters", "cg_iters", "mu_iters", "l0"]
    single = np.array([[r[k] for k in keys] for r in one["trace"]], dtype=np.float64)
    for r in res:
        t = r["trace"]
        assert t.shape == single.shape
        assert np.all(np.abs(t[:, :3] - single[:, :3]) <= 1e-4 * np.abs(single[:, :3]))
        assert np.array_equal(t[:, 3], single[:, 3])
        assert np.abs(r["dict"] - one["dict"]).max() <= 1e-4 * np.abs(one["dict"]).max()
