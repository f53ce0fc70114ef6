#!/usr/bin/env python3
"""Generate the golden fixtures in tests/golden/ from the reference itself.

The reference solver (oracle/_ref/libdcsc_ref.so: the unmodified reference
translation units + FFTW3 shim, built by oracle/Makefile) is run on the seeded
BASELINE.json generator inputs. The GPU tests compare against these files, so
they need neither the reference sources nor its build on the GPU box.

usage: python tests/golden/make_golden.py [small|c1slice|tcsc|c0|all]
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import ref  # noqa: E402
from paper_1709_09479_b200 import dcsc  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
TRACE_KEYS = ["outer_iter", "phase", "total", "data_term", "l1_term", "residual_norm", "admm_iters", "cg_iters",
              "mu_iters", "l0"]


def trace_array(trace):
    return np.array([[row[k] for k in TRACE_KEYS] for row in trace], dtype=np.float64)


def run_case(name, N, grid, K, m, p, sigma, seed, fp32, cfg, threads=0):
    x, d_true = dcsc.synth_generate(N, grid, K, m, p, sigma, seed, fp32)
    ref.set_threads(threads)
    t0 = time.time()
    r = ref.run(x, K, (m, m), cfg)
    dt = time.time() - t0
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), x=x, trace=trace_array(r["trace"]),
                        trace_keys=np.array(TRACE_KEYS), dicts=r["dicts"],
                        maps_l0=np.array([(np.abs(r["maps"]) > 1e-12 * np.abs(r["maps"]).max()).sum()]),
                        maps_sum=np.abs(r["maps"]).sum(axis=(1, 2, 3)), maps_sq=(r["maps"] ** 2).sum(axis=(1, 2, 3)),
                        cfg=np.array([cfg.beta, cfg.rho, cfg.tol, cfg.max_outer, cfg.max_admm, cfg.max_mu_iters,
                                      cfg.cg_tol, cfg.cg_max, cfg.mu_floor, cfg.seed, cfg.normalize]),
                        shape=np.array([N, grid[0], grid[1], K, m]), gen=np.array([p, sigma, seed, fp32]),
                        seconds=np.array([dt]))
    print(f"{name}: {len(r['trace'])} rows in {dt:.1f}s")


def coding_case(name, N, grid, K, m, p, sigma, seed, fp32, beta, max_admm):
    x, d_true = dcsc.synth_generate(N, grid, K, m, p, sigma, seed, fp32)
    cfg = ref.Cfg(beta=beta, max_admm=max_admm, normalize=0)
    rows = []
    for n in range(N):
        z, (th, _, lam), st = ref.solve_coding(x[n], d_true, cfg)
        ob = ref.objective(x[n], d_true, z, beta)
        rows.append([st["admm_iters"], st["converged"], st["dual_objective"], ob[0], ob[1], ob[2],
                     (np.abs(z) > 1e-12 * np.abs(z).max()).sum(), np.abs(z).sum(), (z * z).sum(),
                     (lam * lam).sum()])
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), x=x, d=d_true, rows=np.array(rows),
                        cols=np.array(["admm_iters", "converged", "dual_objective", "data", "l1", "total", "l0",
                                       "z_abs_sum", "z_sq_sum", "lam_sq_sum"]),
                        gen=np.array([p, sigma, seed, fp32]), beta=np.array([beta]), max_admm=np.array([max_admm]))
    print(f"{name}: {N} images")


def tcsc_case(name, N, J, grid, K, m, p, sigma, seed, cfg):
    """Joint channel mode (J > 1, the reference's TCSC path): channel j of the
    signals is the generator's output for seed + j (as bench.py's J-channel data)."""
    x = np.stack([dcsc.synth_generate(N, grid, K, m, p, sigma, seed + j, False)[0] for j in range(J)], axis=1)
    ref.set_threads(0)
    t0 = time.time()
    r = ref.run_j(x, K, (m, m), cfg)
    dt = time.time() - t0
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), x=x, trace=trace_array(r["trace"]),
                        trace_keys=np.array(TRACE_KEYS), dicts=r["dicts"],
                        maps_l0=np.array([(np.abs(r["maps"]) > 1e-12 * np.abs(r["maps"]).max()).sum()]),
                        cfg=np.array([cfg.beta, cfg.rho, cfg.tol, cfg.max_outer, cfg.max_admm, cfg.max_mu_iters,
                                      cfg.cg_tol, cfg.cg_max, cfg.mu_floor, cfg.seed, cfg.normalize]),
                        shape=np.array([N, grid[0], grid[1], K, m, J]), gen=np.array([p, sigma, seed, 0]),
                        seconds=np.array([dt]))
    print(f"{name}: {len(r['trace'])} rows in {dt:.1f}s")


def main(which):
    if which in ("small", "all"):
        run_case("run_small_fp64", 3, (20, 20), 6, 5, 0.05, 0.01, 7, False,
                 ref.Cfg(beta=0.2, max_outer=4, normalize=0, seed=11, tol=1e-300))
        run_case("run_c2shape_fp32", 4, (100, 100), 12, 11, 0.02, 0.01, 5, True,
                 ref.Cfg(beta=0.5, max_outer=2, max_admm=200, normalize=0, seed=2, tol=1e-300))
    if which in ("c1slice", "all"):
        coding_case("coding_c1slice_fp32", 2, (128, 128), 64, 11, 0.01, 0.01, 20250917, True, 0.5, 50)
    if which in ("tcsc", "all"):
        tcsc_case("run_tcsc_j3_fp64", 3, 3, (20, 20), 6, 5, 0.05, 0.01, 7,
                  ref.Cfg(beta=0.2, max_outer=3, max_admm=200, normalize=1, seed=11, tol=1e-300))
    if which in ("c0", "all"):
        # BASELINE.json configs[0]: N=10 100x100 FP64, K=100 11x11, beta=1.0, 10 outer iterations
        run_case("run_c0_fp64", 10, (100, 100), 100, 11, 0.01, 0.01, 20250917, False,
                 ref.Cfg(beta=1.0, max_outer=10, normalize=0, seed=0, tol=1e-300))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "small")
