#!/usr/bin/env python3
"""Where does the FP32 path depart from the FP64 reference? (diagnostic, GPU)

Prints, for C2-shaped problems, the relative dictionary error of the GPU FP32
learning step against the reference's FP64 learning on the SAME (FP32-rounded)
maps, the mu / CG iteration counts of both, and the same for the FP64 GPU path.
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import ref  # noqa: E402
from paper_1709_09479_b200 import dcsc  # noqa: E402


def rel(a, b):
    return float(np.abs(np.asarray(a) - np.asarray(b)).max() / max(np.abs(b).max(), 1e-300))


def learning_replay(N, grid, K, m, p, seed, beta, admm, **kw):
    x, dtrue = dcsc.synth_generate(N, grid, K, m, p, 0.01, seed, True)
    d0 = ref.init_dictionary(K, (m, m), grid, seed=3)
    ref.set_threads(0)
    _, maps = ref.coding_batch(x, d0, ref.Cfg(beta=beta, max_admm=admm, normalize=0), want_maps=True)
    maps = maps.astype(np.float32).astype(np.float64)
    out = {"N": N, "grid": grid, "K": K, **kw}
    d_r, st_r, s_r = ref.solve_learning(x, maps, (m, m), ref.Cfg(beta=beta, normalize=0, **kw))
    out["ref"] = {"mu_iters": s_r["mu_iters"], "cg_iters": s_r["cg_iters"]}
    for prec in (32, 64):
        d_g, st_g, s_g = dcsc.solve_learning(x, maps, (m, m), dcsc.SolverConfig(beta=beta, normalize=0, **kw),
                                             precision=prec)
        out[f"fp{prec}"] = {"d_rel": rel(d_g, d_r), "mu_rel": rel(st_g.mu, st_r[1]),
                            "mu_iters": s_g["mu_iters"], "cg_iters": s_g["cg_iters"]}
    return out


def main():
    res = []
    for kw in ({"max_mu_iters": 1}, {"max_mu_iters": 3}, {}):
        res.append(learning_replay(8, (100, 100), 24, 11, 0.02, 5, 0.5, 100, **kw))
        print(json.dumps(res[-1]), flush=True)
    res.append(learning_replay(16, (64, 64), 32, 7, 0.005, 8, 0.5, 100))
    print(json.dumps(res[-1]), flush=True)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "parity_probe.json"), "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__" and len(sys.argv) == 1:
    main()


def run_probe(N, grid, K, m, p, seed, outer, **kw):
    """Per-outer dictionaries and trace of a full FP32 GPU run against the reference run."""
    x, _ = dcsc.synth_generate(N, grid, K, m, p, 0.01, seed, True)
    cfg = dict(beta=0.5, max_outer=outer, normalize=0, seed=seed, tol=1e-300, **kw)
    ref.set_threads(0)
    r = ref.run(x, K, (m, m), ref.Cfg(**cfg))
    out = []
    for prec in (32, 64):
        with dcsc.Context(N, grid, K, (m, m), dcsc.SolverConfig(**cfg), prec) as ctx:
            ctx.set_signals(x)
            ctx.run_begin()
            for o in range(outer):
                rows, _ = ctx.run_step()
                d = ctx.get_dictionary()
                rr = r["trace"][2 * o: 2 * o + 2]
                out.append({"prec": prec, "outer": o + 1, "d_rel": rel(d, r["dicts"][o + 1]),
                            "total_rel": [abs(a["total"] - b["total"]) / abs(b["total"]) for a, b in zip(rows, rr)],
                            "l0": [rows[0]["l0"], rr[0]["l0"]],
                            "admm": [rows[0]["admm_iters"], rr[0]["admm_iters"]],
                            "mu": [rows[1]["mu_iters"], rr[1]["mu_iters"]],
                            "cg": [rows[1]["cg_iters"], rr[1]["cg_iters"]]})
                print(json.dumps(out[-1]), flush=True)
    return out


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "run":
    run_probe(4, (100, 100), 12, 11, 0.02, 5, 3, max_admm=200)
    run_probe(12, (100, 100), 24, 11, 0.02, 5, 3)
    run_probe(24, (64, 64), 16, 7, 0.005, 8, 3)
