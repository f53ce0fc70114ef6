#!/usr/bin/env python3
"""A/B timing of library variants on one box: alternates DCSC_LIB between the
given .so files (a fresh process per run) on one bench config and prints the
coding-pass ms per launch of each run. usage: ab.py CONFIG STEPS ROUNDS lib1 lib2 ..."""
import json
import os
import subprocess
import sys

cfg, steps, rounds = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
libs = sys.argv[4:]
res = {lib: [] for lib in libs}
for r in range(rounds):
    for lib in libs:
        env = dict(os.environ)
        if lib != "main":
            env["DCSC_LIB"] = lib
        out = subprocess.run([sys.executable, "bench.py", "--config", cfg, "--steps", str(steps), "--warmup", "5",
                              "--no-cpu-baseline"], capture_output=True, text=True, env=env, timeout=900)
        try:
            d = json.loads(out.stdout.strip().splitlines()[-1])
            res[lib].append(round(d["roofline"]["avg_launch_ms"], 4))
        except Exception:
            res[lib].append(None)
            sys.stderr.write(out.stderr[-2000:])
        print(lib, res[lib][-1], flush=True)
for lib in libs:
    v = [x for x in res[lib] if x]
    print("SUMMARY", lib, "min", min(v) if v else None, "runs", res[lib], flush=True)
