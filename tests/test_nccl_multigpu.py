"""Multi-GPU NCCL parity (runs whenever >= 2 GPUs are visible; skipped on a
one-GPU box): one process per GPU, our NCCL communicator (dlopen'ed
libnccl.so.2), both learning layouts (image-sharded crop all-reduce;
frequency-sharded with the grouped ncclSend/ncclRecv z_hat all-to-all); the
FP64 run equals the single-GPU run."""
import os
import subprocess
import sys

import numpy as np
import pytest

from paper_1709_09479_b200 import dcsc

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
WORKER = os.path.join(ROOT, "tests", "mr", "nccl_worker.py")


def n_gpus():
    try:
        out = subprocess.run(["nvidia-smi", "-L"], capture_output=True, text=True, timeout=60).stdout
        return sum(1 for ln in out.splitlines() if ln.startswith("GPU "))
    except Exception:
        return 0


@pytest.mark.parametrize("layout", ["image", "freq"])
def test_nccl_ranks_match_single_gpu(tmp_path, layout):
    world = min(n_gpus(), 4)
    if world < 2:
        pytest.skip("needs >= 2 GPUs")
    idf = str(tmp_path / "nccl.id")
    procs, outs = [], []
    for r in range(world):
        out = str(tmp_path / f"r{r}.npz")
        env = dict(os.environ, RANK=str(r), WORLD_SIZE=str(world), MR_OUT=out, MR_ID=idf, MR_LAYOUT=layout)
        procs.append(subprocess.Popen([sys.executable, WORKER], env=env, stdout=subprocess.PIPE,
                                      stderr=subprocess.STDOUT, text=True))
        outs.append(out)
    for p in procs:
        o, _ = p.communicate(timeout=600)
        assert p.returncode == 0, o[-3000:]
    N, grid, K, m = 6, (64, 64), 8, 7
    x, _ = dcsc.synth_generate(N, grid, K, m, 0.02, 0.01, 5, False)
    cfg = dcsc.SolverConfig(beta=0.3, max_outer=2, normalize=0, seed=3, tol=1e-300, max_admm=100)
    one = dcsc.run_csc(x, K, (m, m), cfg, precision=64)
    keys = ["total", "data_term", "l1_term", "admm_iters", "cg_iters", "mu_iters", "l0"]
    single = np.array([[r[k] for k in keys] for r in one["trace"]], dtype=np.float64)
    for o in outs:
        r = np.load(o)
        t = r["trace"]
        assert np.all(np.abs(t[:, :3] - single[:, :3]) <= 1e-9 * np.abs(single[:, :3]))
        assert np.array_equal(t[:, 3], single[:, 3]) and np.array_equal(t[:, 5], single[:, 5])
        assert np.abs(r["dict"] - one["dict"]).max() <= 1e-8 * np.abs(one["dict"]).max()
