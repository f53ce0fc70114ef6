"""One rank of a multi-rank run_csc (tests/test_multirank.py). Env: RANK,
WORLD_SIZE, MASTER_ADDR, MASTER_PORT, MR_OUT (npz path), MR_MODE (gpu|gpu_j|cpu)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)


def mr_signals(dcsc, N, grid, K, m, J):
    """J = 1: the seeded generator; J > 1: channel j from seed 7 + j."""
    xs = [dcsc.synth_generate(N, grid, K, m, 0.05, 0.01, 7 + j, False)[0] for j in range(J)]
    return xs[0] if J == 1 else np.ascontiguousarray(np.stack(xs, axis=1))


def main():
    import torch.distributed as dist
    from paper_1709_09479_b200 import dcsc

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dist.init_process_group("gloo", rank=rank, world_size=world)
    out = os.environ["MR_OUT"]
    if os.environ.get("MR_MODE") == "cpu":
        # host logic only: the callback sums buffers across ranks
        fn = dcsc.gloo_allreduce_fn()
        buf = (np.arange(5, dtype=np.float64) + 1.0) * (rank + 1)
        rc = fn(buf.ctypes.data_as(dcsc.C.POINTER(dcsc.C.c_double)), buf.size, None)
        n0, n1 = dcsc.shard_range(10, world, rank)
        np.savez(out, buf=buf, rc=rc, shard=np.array([n0, n1]))
        dist.destroy_process_group()
        return
    N, grid, K, m = 4, (20, 20), 6, 5
    mode = os.environ.get("MR_MODE")
    J = 2 if mode == "gpu_j" else 1
    prec = 64
    if mode == "gpu_tc":  # FP32 128 x 128, 11 x 11: the tensor-core coding pass (forced by the test's DCSC_TC=1)
        N, grid, K, m, prec = 4, (128, 128), 8, 11, 32
    x = mr_signals(dcsc, N, grid, K, m, J)
    n0, n1 = dcsc.shard_range(N, world, rank)
    cfg = dcsc.SolverConfig(beta=0.2, max_outer=3, normalize=0, seed=11, tol=1e-300)
    if mode == "gpu_tc":
        cfg = dcsc.SolverConfig(beta=0.5, max_outer=3, max_admm=60, normalize=0, seed=11, tol=1e-300)
    with dcsc.Context(n1 - n0, grid, K, (m, m), cfg, prec, channels=J) as ctx:
        ctx.set_comm_callback(world, rank, dcsc.gloo_allreduce_fn())
        if mode == "gpu_freq":  # frequency-sharded learning (one z_hat all-to-all per outer iteration)
            ctx.set_learning_layout("freq")
        ctx.set_signals(x[n0:n1])
        trace, _ = ctx.run(cfg.max_outer)
        keys = ["total", "data_term", "l1_term", "admm_iters", "cg_iters", "mu_iters", "l0"]
        np.savez(out, trace=np.array([[r[k] for k in keys] for r in trace], dtype=np.float64),
                 dict=ctx.get_dictionary(), maps=ctx.get_maps())
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
