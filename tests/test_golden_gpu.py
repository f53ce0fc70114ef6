"""GPU vs the committed golden fixtures (tests/golden/, produced by the reference
solver through tests/golden/make_golden.py). Needs no reference build on the box."""
import os

import numpy as np
import pytest

from paper_1709_09479_b200 import dcsc

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def load(name):
    path = os.path.join(GOLD, name + ".npz")
    if not os.path.exists(path):
        pytest.skip(f"fixture {name} not generated")
    return np.load(path)


def cfg_of(g):
    c = g["cfg"]
    return dcsc.SolverConfig(beta=float(c[0]), rho=float(c[1]), tol=float(c[2]), max_outer=int(c[3]),
                             max_admm=int(c[4]), max_mu_iters=int(c[5]), cg_tol=float(c[6]), cg_max=int(c[7]),
                             mu_floor=float(c[8]), seed=int(c[9]), normalize=int(c[10]))


def run_gpu(g, precision, dict_tol=None, channels=1):
    """run_csc one outer iteration at a time; with dict_tol every accepted
    dictionary (g["dicts"][o + 1], pipeline.cpp:272) is compared as the run goes."""
    shape = [int(v) for v in g["shape"]]
    N, H, W, K, m = shape[:5]
    if "gen" in g.files and channels == 1:
        x, _ = dcsc.synth_generate(N, (H, W), K, m, float(g["gen"][0]), float(g["gen"][1]), int(g["gen"][2]),
                                   bool(g["gen"][3]))
        assert np.array_equal(x, g["x"])
    x = g["x"]
    cfg = cfg_of(g)
    trace = []
    with dcsc.Context(N, (H, W), K, (m, m), cfg, precision, channels=channels) as ctx:
        ctx.set_signals(x)
        ctx.run_begin()
        for o in range(cfg.max_outer):
            rows, done = ctx.run_step()
            trace.extend(rows)
            if dict_tol is not None:
                dref = g["dicts"][o + 1]
                err = np.abs(ctx.get_dictionary() - dref).max() / np.abs(dref).max()
                assert err <= dict_tol, ("dictionary after outer", o + 1, err)
            if done:
                break
        return trace, ctx.get_dictionary(), ctx.get_maps()


def check_trace(trace, g, tol, exact_iters, l0_slack=0.0):
    keys = list(g["trace_keys"])
    gt = g["trace"]
    assert len(trace) == len(gt)
    for row, grow in zip(trace, gt):
        for k in ("total", "data_term", "l1_term"):
            ref_v = grow[keys.index(k)]
            assert abs(row[k] - ref_v) <= tol * abs(ref_v), (k, row[k], ref_v)
        if exact_iters:
            for k in ("admm_iters", "mu_iters"):
                assert row[k] == grow[keys.index(k)], (k, row, grow)
            if row["phase"] == 0:  # ||z||_0 of the accepted maps (objective.cpp:59-81)
                l0_ref = grow[keys.index("l0")]
                assert abs(row["l0"] - l0_ref) <= l0_slack * l0_ref, ("l0", row["l0"], l0_ref)


def test_golden_small_fp64():
    g = load("run_small_fp64")
    trace, d, maps = run_gpu(g, 64, dict_tol=1e-8)
    check_trace(trace, g, 1e-9, exact_iters=True)
    assert np.abs(d - g["dicts"][-1]).max() <= 1e-8 * np.abs(g["dicts"][-1]).max()
    l0 = (maps != 0).sum()
    assert abs(int(l0) - int(g["maps_l0"][0])) <= 0.001 * int(g["maps_l0"][0]) + 2


def test_golden_c2shape_fp32():
    g = load("run_c2shape_fp32")
    trace, d, _ = run_gpu(g, 32, dict_tol=1e-4)
    check_trace(trace, g, 1e-4, exact_iters=True, l0_slack=1e-4)  # FP32 vs the FP64 reference: l0 modulo near-ties


def test_golden_c1slice_coding_fp32():
    g = load("coding_c1slice_fp32")
    x, d = g["x"], g["d"]
    beta, max_admm = float(g["beta"][0]), int(g["max_admm"][0])
    cols = list(g["cols"])
    N = x.shape[0]
    with dcsc.Context(N, x.shape[1:], d.shape[0], d.shape[1:], dcsc.SolverConfig(beta=beta, max_admm=max_admm,
                                                                                 normalize=0), 32) as ctx:
        ctx.set_signals(x)
        ctx.set_dictionary(d)
        st = ctx.coding()
        _, z, lam = ctx.get_coding_state()
        ctx.set_maps(z)
        ob = ctx.objective()
    for n in range(N):
        row = g["rows"][n]
        assert st[n]["admm_iters"] == row[cols.index("admm_iters")]
        assert abs(ob[n][2] - row[cols.index("total")]) <= 1e-4 * abs(row[cols.index("total")])
        assert abs(st[n]["dual_objective"] - row[cols.index("dual_objective")]) <= 1e-4 * abs(row[cols.index("dual_objective")])
        l0 = (z[n] != 0).sum()
        assert abs(l0 - row[cols.index("l0")]) <= 0.01 * row[cols.index("l0")]


@pytest.mark.slow
def test_golden_c0_fp64():
    """BASELINE.json configs[0] at full size: 10 outer iterations, FP64, <= 1e-9."""
    g = load("run_c0_fp64")
    trace, d, _ = run_gpu(g, 64, dict_tol=1e-8)
    check_trace(trace, g, 1e-9, exact_iters=True)
    dref = g["dicts"][-1]
    assert np.abs(d - dref).max() <= 1e-8 * np.abs(dref).max()


def test_golden_tcsc_j3_fp64():
    """Joint channel mode (J = 3) against the reference TCSC run: <= 1e-8, same iteration counts."""
    g = load("run_tcsc_j3_fp64")
    J = int(g["shape"][5])
    trace, d, _ = run_gpu(g, 64, dict_tol=1e-7, channels=J)
    check_trace(trace, g, 1e-8, exact_iters=True)
    dref = g["dicts"][-1]
    assert np.abs(d - dref).max() <= 1e-7 * np.abs(dref).max()
