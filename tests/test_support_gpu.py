"""Soft-threshold support and warm states against the reference (GPU).

Support, bit-exact away from ties (BASELINE.json north_star): from the same
warm ADMM state (theta, z) the reference and the GPU each run ONE coding
iteration (max_admm = 1, coding.cpp:223-284); z' = -rho soft(u, beta) with
u = t - z/rho, so the support is {|u| > beta}. The GPU's support (exact zeros
of its closed-form update) must equal the reference's (|z'| > 1e-12 max|z'|,
the reference's update leaves ~1e-17 residues) on every entry outside the tie
band ||u| - beta| <= TIE * eps * max(max|t|, max|z/rho|) (eps of the GPU's
storage precision; TIE = 64 covers the FFT round trip's normwise error).

Warm states that are not ADMM-consistent (theta != clamp(theta - z/rho): a
theta outside the box, z given without theta) follow the reference's first
iteration (w = theta + z/rho, theta_old = theta) exactly.
"""
import numpy as np
import pytest

from oracle import ref
from paper_1709_09479_b200 import dcsc

pytestmark = pytest.mark.gpu
TIE = 64.0


def problem(N, grid, K, m, seed, fp32):
    x, d_true = dcsc.synth_generate(N, grid, K, m, 0.02, 0.01, seed, fp32)
    return x, ref.init_dictionary(K, (m, m), grid, seed=seed + 1)


@pytest.mark.parametrize("grid,K,m,prec,warm_iters", [((128, 128), 16, 11, 32, 7), ((100, 100), 12, 11, 64, 9),
                                                      ((64, 64), 8, 7, 32, 15), ((256, 256), 6, 11, 32, 5)])
def test_support_one_iteration_replay(grid, K, m, prec, warm_iters):
    beta, rho = 0.5, 0.1
    x, d = problem(1, grid, K, m, 31, prec == 32)
    cfg_w = ref.Cfg(beta=beta, rho=rho, max_admm=warm_iters, normalize=0)
    _, (theta, z, lam), _ = ref.solve_coding(x[0], d, cfg_w)
    if prec == 32:  # the GPU stores the state in FP32: replay both sides from the rounded state
        u32 = (theta - z / rho).astype(np.float32).astype(np.float64)
        theta = np.clip(u32, -beta, beta)
        z = rho * (theta - u32)
    z_r, (th_r, _, _), _ = ref.solve_coding(x[0], d, ref.Cfg(beta=beta, rho=rho, max_admm=1, normalize=0),
                                            (theta, z, lam))
    with dcsc.Context(1, grid, K, (m, m), dcsc.SolverConfig(beta=beta, rho=rho, max_admm=1, normalize=0), prec) as ctx:
        ctx.set_signals(x)
        ctx.set_dictionary(d)
        ctx.set_coding_state(theta[None], z[None])
        ctx.coding()
        _, z_g, _ = ctx.get_coding_state()
    z_g = z_g[0]
    u_r = th_r - z_r / rho                      # the reference's soft-threshold argument
    t_r = u_r + z / rho
    eps = np.finfo(np.float32 if prec == 32 else np.float64).eps
    band = TIE * eps * max(np.abs(t_r).max(), np.abs(z / rho).max())
    away = np.abs(np.abs(u_r) - beta) > band
    sup_r = np.abs(z_r) > 1e-12 * np.abs(z_r).max()
    sup_g = z_g != 0
    mism = (sup_r != sup_g) & away
    assert away.mean() > 0.99
    assert sup_r.sum() > 0
    assert not mism.any(), (int(mism.sum()), int(away.size - away.sum()))


@pytest.mark.parametrize("kind", ["theta_zero_z_nonzero", "theta_outside_box", "theta_only"])
def test_inconsistent_warm_state_matches_reference(kind):
    """ADMM from a warm state the GPU's single u = theta - z/rho array cannot
    represent: the first iteration uses theta itself (CodingArgs::theta0)."""
    beta, rho = 0.3, 0.1
    x, d = problem(1, (20, 20), 4, 5, 5, False)
    rng = np.random.default_rng(3)
    K = 4
    if kind == "theta_zero_z_nonzero":
        theta = np.zeros((K, 20, 20))
        z = rng.standard_normal((K, 20, 20)) * 0.05
    elif kind == "theta_outside_box":
        theta = rng.standard_normal((K, 20, 20))
        z = rng.standard_normal((K, 20, 20)) * 0.01
    else:
        theta = rng.uniform(-beta, beta, (K, 20, 20))
        z = np.zeros((K, 20, 20))
    lam = np.zeros((20, 20))
    for iters in (1, 40):
        cfg = ref.Cfg(beta=beta, rho=rho, max_admm=iters, normalize=0)
        z_r, (th_r, _, lam_r), s_r = ref.solve_coding(x[0], d, cfg, (theta, z, lam))
        with dcsc.Context(1, (20, 20), K, (5, 5), dcsc.SolverConfig(beta=beta, rho=rho, max_admm=iters, normalize=0),
                          64) as ctx:
            ctx.set_signals(x)
            ctx.set_dictionary(d)
            ctx.set_coding_state(theta[None], z[None])
            th_back, z_back, _ = ctx.get_coding_state()
            assert np.abs(th_back[0] - theta).max() <= 1e-12 and np.abs(z_back[0] - z).max() <= 1e-12
            st = ctx.coding()
            th_g, z_g, lam_g = ctx.get_coding_state()
        assert st[0]["admm_iters"] == s_r["admm_iters"]
        for key in ("theta_change", "z_change", "primal_residual"):
            assert abs(st[0][key] - s_r[key]) <= 1e-9 * max(abs(s_r[key]), 1e-300), (iters, key)
        sc = max(np.abs(z_r).max(), 1e-300)
        assert np.abs(z_g[0] - z_r).max() <= 1e-9 * sc, iters
        assert np.abs(lam_g[0] - lam_r).max() <= 1e-9 * np.abs(lam_r).max(), iters
