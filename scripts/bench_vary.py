#!/usr/bin/env python3
"""GPU counterpart of the reference's scaling bench (`csc bench --vary k|n|beta`,
proj/src/bench.cpp:23-99, tools/csc_main.cpp run_bench_cmd) and of acceptance
criterion 8 (tests/acceptance_main.cpp:373-413): short run_csc runs over a
parameter grid on the reference's synthetic dataset (bench.cpp:9-21), timing
the coding and learning phases from the trace's elapsed_ms (solver calls only).

Writes the reference's CSV (`varied_value,phase,mean_ms_per_outer_iter,std_ms`,
bench.cpp:103-109) and prints one JSON line with the per-inner-iteration costs
and the R^2 of the linear fits the acceptance check uses.

usage: bench_vary.py --vary k --grid 4,8,16,32 [--repeats 2] [--size 64x64]
       [--filter-size 11x11] [--filters 8] [--images 2] [--channels 1]
       [--outer 3] [--precision 32] [--max-admm 500] [--out bench.csv]
"""
import argparse
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1709_09479_b200 import dcsc  # noqa: E402


def fit_r_squared(x, y):
    """Least-squares line fit R^2 (acceptance_main.cpp:66-85)."""
    n = float(len(x))
    sx, sy = sum(x), sum(y)
    sxx = sum(v * v for v in x)
    sxy = sum(a * b for a, b in zip(x, y))
    b = (n * sxy - sx * sy) / (n * sxx - sx * sx)
    a = (sy - b * sx) / n
    mean = sy / n
    ss_res = sum((yi - (a + b * xi)) ** 2 for xi, yi in zip(x, y))
    ss_tot = sum((yi - mean) ** 2 for yi in y)
    return 1.0 - ss_res / ss_tot if ss_tot > 0 else 1.0


def stats_of(v):
    mean = sum(v) / len(v)
    return mean, math.sqrt(sum((x - mean) ** 2 for x in v) / len(v))


def run_bench(vary, grid, repeats, dims, support, filters, images, channels, beta, outer, precision, max_admm,
              cg_max, seed):
    """bench.cpp:23-99 on the GPU path."""
    if not grid:
        raise ValueError("bench grid is empty")
    if repeats < 1:
        raise ValueError("bench repeats must be >= 1")
    rows = []
    for value in grid:
        K, N, b = filters, images, beta
        if vary == "k":
            K = int(value)
        elif vary == "n":
            N = int(value)
        else:
            b = value
        if K < 1 or N < 1:
            raise ValueError("bench grid holds a non-positive size")
        cfg = dcsc.SolverConfig(beta=b, max_outer=outer, tol=1e-300, max_admm=max_admm, cg_max=cg_max, seed=seed)
        coding_ms, learning_ms = [], []
        admm, cg, ctot, ltot = 0, 0, 0.0, 0.0
        for rep in range(repeats):
            x = dcsc.synth_dataset(N, channels, dims, seed + rep)
            with dcsc.Context(N, dims, K, support, cfg, precision, channels=channels) as ctx:
                ctx.set_signals(x)
                trace, _ = ctx.run(outer)
            for r in trace:
                if r["phase"] == 0:
                    coding_ms.append(r["elapsed_ms"])
                    ctot += r["elapsed_ms"]
                    admm += r["admm_iters"]
                else:
                    learning_ms.append(r["elapsed_ms"])
                    ltot += r["elapsed_ms"]
                    cg += r["cg_iters"]
        cm, cs = stats_of(coding_ms)
        lm, ls = stats_of(learning_ms)
        rows.append({"varied_value": value, "phase": "coding", "mean_ms_per_outer": cm, "std_ms": cs,
                     "mean_ms_per_admm_iter": ctot / admm if admm else 0.0, "mean_ms_per_cg_iter": 0.0})
        rows.append({"varied_value": value, "phase": "learning", "mean_ms_per_outer": lm, "std_ms": ls,
                     "mean_ms_per_admm_iter": 0.0, "mean_ms_per_cg_iter": ltot / cg if cg else 0.0})
    return rows


def fmt17(v):
    """std::ostream with precision(17) (default float format, %.17g)."""
    return "%.17g" % v


def write_bench_csv(path, rows):
    """bench.cpp:103-109."""
    with open(path, "w") as f:
        f.write("varied_value,phase,mean_ms_per_outer_iter,std_ms\n")
        for r in rows:
            f.write(f"{fmt17(r['varied_value'])},{r['phase']},{fmt17(r['mean_ms_per_outer'])},{fmt17(r['std_ms'])}\n")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--vary", choices=["k", "n", "beta"], default="k")
    ap.add_argument("--grid", default="4,8,16,32")
    ap.add_argument("--repeats", type=int, default=1)
    ap.add_argument("--size", default="64x64")
    ap.add_argument("--filter-size", default="11x11")
    ap.add_argument("--filters", type=int, default=8)
    ap.add_argument("--images", type=int, default=2)
    ap.add_argument("--channels", type=int, default=1)
    ap.add_argument("--beta", type=float, default=0.5)
    ap.add_argument("--outer", type=int, default=3)
    ap.add_argument("--precision", type=int, default=32)
    ap.add_argument("--max-admm", type=int, default=500)
    ap.add_argument("--cg-max", type=int, default=300)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    dims = tuple(int(v) for v in a.size.split("x"))
    support = tuple(int(v) for v in a.filter_size.split("x"))
    grid = [float(v) for v in a.grid.split(",") if v]
    rows = run_bench(a.vary, grid, a.repeats, dims, support, a.filters, a.images, a.channels, a.beta, a.outer,
                     a.precision, a.max_admm, a.cg_max, a.seed)
    if a.out:
        write_bench_csv(a.out, rows)
    cod = [r for r in rows if r["phase"] == "coding"]
    xs = [r["varied_value"] for r in cod]
    out = {"vary": a.vary, "grid": grid, "rows": rows}
    if len(xs) >= 2 and a.vary in ("k", "n"):
        key = "mean_ms_per_admm_iter" if a.vary == "k" else "mean_ms_per_outer"
        out["r2_coding_linear"] = fit_r_squared(xs, [r[key] for r in cod])
    print(json.dumps(out))


if __name__ == "__main__":
    main()
