"""Tensor-core coding pass vs the FFT coding pass on the same inputs (GPU box).

python scripts/tc_check.py [N] [admm]
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1709_09479_b200 import dcsc  # noqa: E402


def run(tc, grid, K, N, admm, seed=3, m=11):
    os.environ["DCSC_TC"] = "1" if tc else "0"
    cfg = dcsc.SolverConfig(beta=0.5, rho=0.1, max_admm=admm, seed=seed)
    x, dtrue = dcsc.synth_generate(N, grid, K, m, 0.01, 0.01, seed, True)[:2]
    with dcsc.Context(N, grid, K, (m, m), cfg, precision=32) as ctx:
        ctx.set_signals(x)
        ctx.init_variables()
        ctx.coding()  # warm (and the first call's setup)
        ctx.init_variables()
        ctx.set_signals(x)
        t = time.time()
        st = ctx.coding()
        el = time.time() - t
        th, z, lam = ctx.get_coding_state()
    return st, th, z, lam, el


def main():
    N = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    admm = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    cases = (((256, 256), 128, 11), ((128, 128), 64, 11), ((100, 100), 100, 11), ((80, 80), 24, 11),
             ((64, 64), 32, 7), ((64, 64), 20, 7))
    only = os.environ.get("TC_ONLY")
    for grid, K, m in cases:
        if only and str(grid[0]) not in only.split(","):
            continue
        a = run(True, grid, K, N, admm, m=m)
        b = run(False, grid, K, N, admm, m=m)
        rel = lambda u, v: float(np.abs(u - v).max() / max(np.abs(v).max(), 1e-30))
        print(f"grid {grid} K={K} N={N} admm<={admm}: tc {a[4]*1e3:.1f} ms  fft {b[4]*1e3:.1f} ms")
        print("  iters tc ", [s["admm_iters"] for s in a[0]], " fft", [s["admm_iters"] for s in b[0]])
        for key in ("primal_residual", "z_change", "theta_change", "dual_objective"):
            va = np.array([s[key] for s in a[0]])
            vb = np.array([s[key] for s in b[0]])
            print(f"  {key}: max rel diff {np.abs(va - vb).max() / max(np.abs(vb).max(), 1e-30):.3e}")
        print(f"  theta rel {rel(a[1], b[1]):.3e}  z rel {rel(a[2], b[2]):.3e}  lambda rel {rel(a[3], b[3]):.3e}")
        sa, sb = np.abs(a[2]) > 0, np.abs(b[2]) > 0
        print(f"  support mismatches {int((sa != sb).sum())} of {sa.size} (nnz {int(sb.sum())})")


if __name__ == "__main__":
    main()
