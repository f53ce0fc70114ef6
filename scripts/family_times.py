"""Per-kernel-family device time of a coding-only run at a bench config's
shape (per-launch CUDA events, profiling mode 1).

python scripts/family_times.py c3 20      # config, ADMM iterations
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_1709_09479_b200 import dcsc  # noqa: E402

FAMS = ["coding pass", "lambda / band / split", "contract", "mask", "other (r2c / c2r / ...)"]

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
admm = int(sys.argv[2]) if len(sys.argv) > 2 else 20
cfg = bench.CONFIGS[name]
x, d = bench.make_data(cfg, 0, cfg["N"])
sc = dcsc.SolverConfig(beta=cfg["beta"], max_admm=admm, normalize=0, seed=bench.SEED, tol=1e-300)
with dcsc.Context(cfg["N"], (cfg["H"], cfg["W"]), cfg["K"], (cfg["m"], cfg["m"]), sc, cfg["prec"]) as ctx:
    ctx.set_signals(x)
    ctx.set_dictionary(d)
    ctx.coding()
    ctx.set_coding_state(None, None)
    ctx.set_profiling(1)
    t = time.time()
    st = ctx.coding()
    wall = (time.time() - t) * 1e3
    tot = 0.0
    for f, nm in enumerate(FAMS):
        ms, n = ctx.kernel_time(f)
        tot += ms
        print(f"{nm:28s} {ms:9.2f} ms  {n:6d} launches  {ms / max(admm, 1):7.3f} ms/iter")
    print(f"{'sum':28s} {tot:9.2f} ms   wall {wall:.1f} ms   iters {st[0]['admm_iters']}")
