"""Per-kernel-family device time of one full outer iteration (run_step) at a
bench config (after `warm` warm-up outer iterations), per-launch CUDA events.

python scripts/family_times_run.py c3 3
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_1709_09479_b200 import dcsc  # noqa: E402

FAMS = ["coding pass", "lambda / band / split", "contract (z_hat streams)", "mask", "other (r2c / c2r / ...)"]
name = sys.argv[1] if len(sys.argv) > 1 else "c3"
warm = int(sys.argv[2]) if len(sys.argv) > 2 else 3
cfg = bench.CONFIGS[name]
x, _ = bench.make_data(cfg, 0, cfg["N"])
sc = dcsc.SolverConfig(beta=cfg["beta"], max_admm=cfg["max_admm"], normalize=0, seed=bench.SEED, tol=1e-300)
with dcsc.Context(cfg["N"], (cfg["H"], cfg["W"]), cfg["K"], (cfg["m"], cfg["m"]), sc, cfg["prec"]) as ctx:
    ctx.set_signals(x)
    ctx.run_begin()
    for _ in range(warm):
        ctx.run_step()
    ctx.set_profiling(1)
    t = time.time()
    rows = ctx.run_step()
    wall = (time.time() - t) * 1e3
    tot = 0.0
    for f, nm in enumerate(FAMS):
        ms, n = ctx.kernel_time(f)
        tot += ms
        print(f"{nm:28s} {ms:10.2f} ms  {n:7d} launches")
    print(f"{'sum':28s} {tot:10.2f} ms   wall {wall:.1f} ms  rows {rows}")
