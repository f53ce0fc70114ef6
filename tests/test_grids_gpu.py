"""The added grid families against the reference (GPU): 32x32 (the reference's
acceptance dataset grid, tests/acceptance_main.cpp:140), 48x48, 80x80 (FP32)
and FP64 128x128 (a 4-CTA cluster family like FP32 256x256).

FP64: <= 1e-9 relative with identical iteration counts; FP32: <= 1e-4
(BASELINE.json north_star)."""
import numpy as np
import pytest

from oracle import ref
from paper_1709_09479_b200 import dcsc

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.abs(np.asarray(a) - np.asarray(b)).max() / max(np.abs(b).max(), 1e-300))


@pytest.mark.parametrize("H,W,prec", [(32, 32, 64), (32, 32, 32), (48, 48, 64), (48, 48, 32), (80, 80, 32),
                                      (128, 128, 64)])
def test_dft_matches_reference(H, W, prec):
    rng = np.random.default_rng(H + prec)
    x = rng.standard_normal((3, H, W))
    if prec == 32:
        x = x.astype(np.float32).astype(np.float64)
    g = dcsc.forward_dft2(x, prec)
    r = np.stack([ref.forward_dft(xi) for xi in x])[..., : W // 2 + 1]
    tol = 1e-13 if prec == 64 else 2e-6
    assert rel(g.view(np.float64), r.view(np.float64)) <= tol
    assert rel(dcsc.inverse_dft2(g, W, prec), x) <= tol


@pytest.mark.parametrize("H,K,m,prec", [(32, 6, 5, 64), (48, 5, 7, 64), (80, 4, 7, 32), (128, 5, 11, 64)])
def test_coding_matches_reference(H, K, m, prec):
    x, _ = dcsc.synth_generate(2, (H, H), K, m, 0.02, 0.01, 3, prec == 32)
    d = ref.init_dictionary(K, (m, m), (H, H), seed=4)
    cfg = dict(beta=0.3, max_admm=60, normalize=0)
    for n in range(2):
        z_r, st_r, s_r = ref.solve_coding(x[n], d, ref.Cfg(**cfg))
        z_g, st_g, s_g = dcsc.solve_coding(x[n], d, dcsc.SolverConfig(**cfg), precision=prec)
        if prec == 64:
            assert s_g["admm_iters"] == s_r["admm_iters"]
            assert rel(z_g, z_r) <= 1e-9
            assert abs(s_g["dual_objective"] - s_r["dual_objective"]) <= 1e-9 * abs(s_r["dual_objective"])
        else:
            og = dcsc.evaluate_objective(x[n], d, z_g, cfg["beta"], precision=32)
            orf = ref.objective(x[n], d, z_r, cfg["beta"])
            assert abs(og[2] - orf[2]) <= 1e-4 * abs(orf[2])


@pytest.mark.parametrize("H,K,m,prec", [(32, 4, 5, 64), (128, 3, 11, 64), (80, 4, 7, 32)])
def test_run_matches_reference(H, K, m, prec):
    x, _ = dcsc.synth_generate(2, (H, H), K, m, 0.03, 0.01, 8, prec == 32)
    kw = dict(beta=0.3, max_outer=2, normalize=0, seed=5, tol=1e-300, max_admm=80)
    r = ref.run(x, K, (m, m), ref.Cfg(**kw))
    g = dcsc.run_csc(x, K, (m, m), dcsc.SolverConfig(**kw), precision=prec)
    tol = 1e-8 if prec == 64 else 1e-4
    for a, b in zip(g["trace"], r["trace"]):
        for key in ("total", "data_term", "l1_term"):
            assert abs(a[key] - b[key]) <= tol * abs(b[key]), (key, a, b)
        if prec == 64:
            assert a["admm_iters"] == b["admm_iters"] and a["mu_iters"] == b["mu_iters"]
    assert rel(g["dict"], r["dicts"][-1]) <= (1e-7 if prec == 64 else 1e-4)


def test_acceptance_dataset_monotone_run_matches_reference():
    """The reference's acceptance run (acceptance_main.cpp:133-155): synthetic_dataset({32, 32},
    1, 4, 99) (bench.cpp:9-21), K=16 5x5, beta 0.5, rho 0.1, tol 1e-3, 8 outer iterations, 250
    ADMM iterations, seed 31, default Global normalisation; FP64 trace equal to the reference's
    run_csc and non-increasing (criterion: monotone trace)."""
    xs = dcsc.synth_dataset(4, 1, (32, 32), 99)
    kw = dict(beta=0.5, rho=0.1, tol=1e-3, max_outer=8, max_admm=250, seed=31, normalize=1)
    r = ref.run_csc(xs, 16, (5, 5), ref.Cfg(**kw))
    g = dcsc.run_csc(xs, 16, (5, 5), dcsc.SolverConfig(**kw), precision=64)
    assert len(g["trace"]) == len(r["trace"])
    for a, b in zip(g["trace"], r["trace"]):
        assert a["admm_iters"] == b["admm_iters"]
        assert abs(a["total"] - b["total"]) <= 1e-9 * abs(b["total"])
    totals = [row["total"] for row in g["trace"]]
    assert all(t1 <= t0 * (1 + 1e-12) for t0, t1 in zip(totals, totals[1:]))
    assert rel(g["dict"], r["dict"]) <= 1e-7
