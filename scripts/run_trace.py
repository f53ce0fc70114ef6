#!/usr/bin/env python3
"""Run run_csc on a BASELINE config for a few outer iterations and print the
trace (per half-step objective, ADMM/CG/mu iterations, wall ms) plus the
per-kernel-family device time. usage: run_trace.py c2 [outer]"""
import json
import os
import sys
import time

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
ctx.set_profiling(True)
t0 = time.perf_counter()
trace, _ = ctx.run(outer)
wall = time.perf_counter() - t0
fams = ["coding_pass_admm", "lambda_update", "learning_contract", "learning_mask", "other"]
out = {"config": name, "outer": outer, "wall_s": wall,
       "kernel_ms": {f: round(ctx.kernel_time(i)[0], 2) for i, f in enumerate(fams)},
       "launches": {f: ctx.kernel_time(i)[1] for i, f in enumerate(fams)},
       "trace": [{k: (round(v, 6) if isinstance(v, float) else v) for k, v in r.items()} for r in trace]}
print(json.dumps(out, indent=1))
