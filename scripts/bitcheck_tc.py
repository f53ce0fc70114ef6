#!/usr/bin/env python3
"""Bit-identity check of two library builds on the tensor-core coding pass: codes a few 256x256 FP32 images
(DCSC_TC=1) and writes / compares the raw maps and duals. usage: bitcheck_tc.py write|compare FILE"""
import os
import sys

import numpy as np

os.environ["DCSC_TC"] = "1"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1709_09479_b200 import dcsc  # noqa: E402

x, _ = dcsc.synth_generate(3, (256, 256), 16, 11, 0.02, 0.01, 11, True)
rng = np.random.default_rng(5)
d = rng.standard_normal((16, 11, 11))
d /= np.linalg.norm(d.reshape(16, -1), axis=1)[:, None, None]
cfg = dcsc.SolverConfig(beta=0.5, max_admm=25, normalize=0, tol=1e-300)
with dcsc.Context(3, (256, 256), 16, (11, 11), cfg, 32) as ctx:
    ctx.set_signals(x)
    ctx.set_dictionary(d)
    assert ctx.coding_path() == "tensor", ctx.coding_path()
    ctx.coding()
    th, z, lam = ctx.get_coding_state()
if sys.argv[1] == "write":
    np.savez(sys.argv[2], th=th, z=z, lam=lam)
    print("written", float(np.abs(z).max()))
else:
    o = np.load(sys.argv[2])
    same = all(np.array_equal(a, o[k]) and np.array_equal(np.signbit(a), np.signbit(o[k]))
               for k, a in (("th", th), ("z", z), ("lam", lam)))
    print("bit-identical" if same else "DIFFERENT", float(np.abs(z - o["z"]).max()))
    sys.exit(0 if same else 1)
