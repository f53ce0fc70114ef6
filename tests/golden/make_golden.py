#!/usr/bin/env python3
"""Generate the golden fixtures in tests/golden/ from the reference itself.

The reference solver (oracle/_ref/libdcsc_ref.so: the unmodified reference
translation units + FFTW3 shim, built by oracle/Makefile) is run on the seeded
BASELINE.json generator inputs. The GPU tests compare against these files, so
they need neither the reference sources nor its build on the GPU box.

usage: python tests/golden/make_golden.py [small|c1slice|tcsc|c0|c1|c2|c3|c4|all]

The BASELINE-config fixtures (c1, c2, c3, c4) store only checksums of the
inputs (the GPU tests regenerate them with the same seeded generator and check
the checksum) plus, per outer iteration, the trace row, the accepted
dictionary, the acceptance flags and the near-tie counts of the accepted maps.
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


def x_checksum(x):
    """Order-sensitive checksum of the generated inputs (float64 sums of x and i*x)."""
    flat = x.reshape(-1)
    return np.array([flat.sum(), (flat * np.arange(flat.size, dtype=np.float64)).sum(), float(flat.size)])


def run_full(name, N, grid, K, m, p, sigma, seed, fp32, cfg):
    """A BASELINE config through the instrumented run_csc replica (per-outer dictionaries,
    near-tie counts, acceptance flags); per-image objective passes run in parallel."""
    x, _ = ref.synth_generate(N, grid, K, m, p, sigma, seed, fp32)
    ref.set_threads(0)
    ref.set_parallel_objective(True)
    t0 = time.time()
    r = ref.run(x, K, (m, m), cfg, want_maps=False)
    dt = time.time() - t0
    ref.set_parallel_objective(False)
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), x_sum=x_checksum(x), trace=trace_array(r["trace"]),
                        trace_keys=np.array(TRACE_KEYS), dicts=r["dicts"], ties=r["ties"], accepts=r["accepts"],
                        cfg=np.array([cfg.beta, cfg.rho, cfg.tol, cfg.max_outer, cfg.max_admm, cfg.max_mu_iters,
                                      cfg.cg_tol, cfg.cg_max, cfg.mu_floor, cfg.seed, cfg.normalize]),
                        shape=np.array([N, grid[0], grid[1], K, m]), gen=np.array([p, sigma, seed, fp32]),
                        seconds=np.array([dt]), threads=np.array([os.cpu_count()]))
    print(f"{name}: {len(r['trace'])} rows in {dt:.1f}s", flush=True)


def coding_full(name, N, grid, K, m, p, sigma, seed, fp32, beta, max_admm):
    """C1: solve_coding of every image (cold start, ground-truth dictionary), one
    image per host thread; per-image stats, objective, l0, checksums and the
    near-tie counts of the soft-threshold argument u = theta - z/rho."""
    from concurrent.futures import ThreadPoolExecutor
    x, d_true = ref.synth_generate(N, grid, K, m, p, sigma, seed, fp32)
    cfg = ref.Cfg(beta=beta, max_admm=max_admm, normalize=0)
    ref.set_threads(1)
    bands = np.array([1e-7, 1e-6, 1e-5, 1e-4])

    def one(n):
        z, (th, zz, lam), st = ref.solve_coding(x[n], d_true, cfg)
        ob = ref.objective(x[n], d_true, z, beta)
        gap = np.abs(np.abs(th - zz / cfg.rho) - beta)
        ties = [(gap <= b * beta).sum() for b in bands]
        return [st["admm_iters"], st["converged"], st["dual_objective"], ob[0], ob[1], ob[2],
                (np.abs(z) > 1e-12 * np.abs(z).max()).sum(), np.abs(z).sum(), (z * z).sum(), (lam * lam).sum()] + ties

    t0 = time.time()
    with ThreadPoolExecutor(os.cpu_count()) as ex:
        rows = list(ex.map(one, range(N)))
    dt = time.time() - t0
    ref.set_threads(0)
    # the reference's own batched coding (OpenMP over images, pipeline.cpp:221) timed at full size
    t1 = time.time()
    ref.coding_batch(x, d_true, cfg)
    dt_batch = time.time() - t1
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), x_sum=x_checksum(x), d=d_true, rows=np.array(rows),
                        cols=np.array(["admm_iters", "converged", "dual_objective", "data", "l1", "total", "l0",
                                       "z_abs_sum", "z_sq_sum", "lam_sq_sum", "ties_1e-7", "ties_1e-6",
                                       "ties_1e-5", "ties_1e-4"]),
                        gen=np.array([p, sigma, seed, fp32]), beta=np.array([beta]), max_admm=np.array([max_admm]),
                        shape=np.array([N, grid[0], grid[1], K, m]), seconds=np.array([dt]),
                        coding_batch_seconds=np.array([dt_batch]), threads=np.array([os.cpu_count()]))
    print(f"{name}: {N} images in {dt:.1f}s (reference coding_batch at full size {dt_batch:.1f}s on "
          f"{os.cpu_count()} threads)", flush=True)


SEED = 20250917  # bench.py SEED


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


    # BASELINE.json configs at full (C1, C2) or subset (C3, C4) size, FP32 inputs
    if which in ("c4", "all"):  # configs[4] on an N/8 subset at full K, 64x64: 2 outer iterations
        run_full("run_c4sub_fp32", 256, (64, 64), 32, 7, 0.005, 0.05, SEED, True,
                 ref.Cfg(beta=0.5, max_outer=2, normalize=0, seed=SEED, tol=1e-300))
    if which in ("c1", "all"):  # configs[1] at full size: 256 images, 50 ADMM iterations
        coding_full("coding_c1_fp32", 256, (128, 128), 64, 11, 0.01, 0.01, SEED, True, 0.5, 50)
    if which in ("c2", "all"):  # configs[2] at full size: 2 of its 20 outer iterations
        run_full("run_c2_fp32", 100, (100, 100), 100, 11, 0.02, 0.01, SEED, True,
                 ref.Cfg(beta=0.5, max_outer=2, normalize=0, seed=SEED, tol=1e-300))
    if which in ("c3", "all"):  # configs[3] on an N/16 subset at full K, 256x256, ADMM capped at 50
        run_full("run_c3sub_fp32", 32, (256, 256), 128, 11, 0.01, 0.01, SEED, True,
                 ref.Cfg(beta=0.5, max_outer=1, max_admm=50, normalize=0, seed=SEED, tol=1e-300))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "small")
