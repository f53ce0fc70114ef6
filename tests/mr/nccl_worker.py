"""One rank of a real multi-GPU NCCL run (tests/test_nccl_multigpu.py): rank r
on GPU r, the NCCL unique id passed through a file. Env: RANK, WORLD_SIZE,
MR_OUT, MR_ID (id file), MR_LAYOUT (image|freq)."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)


def main():
    from paper_1709_09479_b200 import dcsc

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    idf = os.environ["MR_ID"]
    if rank == 0:
        with open(idf + ".tmp", "wb") as f:
            f.write(dcsc.nccl_unique_id())
        os.replace(idf + ".tmp", idf)
    t0 = time.time()
    while not os.path.exists(idf):
        if time.time() - t0 > 120:
            raise RuntimeError("no NCCL id")
        time.sleep(0.05)
    uid = open(idf, "rb").read()
    N, grid, K, m = 6, (64, 64), 8, 7
    x, _ = dcsc.synth_generate(N, grid, K, m, 0.02, 0.01, 5, False)
    n0, n1 = dcsc.shard_range(N, world, rank)
    cfg = dcsc.SolverConfig(beta=0.3, max_outer=2, normalize=0, seed=3, tol=1e-300, max_admm=100)
    with dcsc.Context(n1 - n0, grid, K, (m, m), cfg, 64, device=rank) as ctx:
        ctx.set_comm_nccl(world, rank, uid)
        ctx.set_learning_layout(os.environ.get("MR_LAYOUT", "image"))
        ctx.set_signals(x[n0:n1])
        trace, _ = ctx.run(cfg.max_outer)
        keys = ["total", "data_term", "l1_term", "admm_iters", "cg_iters", "mu_iters", "l0"]
        np.savez(os.environ["MR_OUT"], trace=np.array([[r[k] for k in keys] for r in trace], dtype=np.float64),
                 dict=ctx.get_dictionary())


if __name__ == "__main__":
    main()
