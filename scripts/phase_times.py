#!/usr/bin/env python3
"""Wall time per run_csc half-step without per-launch profiling events (the
trace's elapsed_ms), for judging host-side overhead against run_trace.py's
per-kernel device times. usage: phase_times.py c2 [outer]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_1709_09479_b200 import dcsc  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
outer = int(sys.argv[2]) if len(sys.argv) > 2 else 2
cfg = bench.CONFIGS[name]
x, _ = bench.make_data(cfg, 0, cfg["N"])
sc = dcsc.SolverConfig(beta=cfg["beta"], max_admm=cfg["max_admm"], normalize=0, seed=bench.SEED, tol=1e-300)
ctx = dcsc.Context(cfg["N"], (cfg["H"], cfg["W"]), cfg["K"], (cfg["m"], cfg["m"]), sc, cfg["prec"])
ctx.set_signals(x)
trace, _ = ctx.run(outer)
print(json.dumps([{k: r[k] for k in ("outer_iter", "phase", "admm_iters", "cg_iters", "mu_iters", "elapsed_ms",
                                     "wall_ms")} for r in trace]))
