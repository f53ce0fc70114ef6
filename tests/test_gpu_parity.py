"""GPU parity: the CUDA path (through the C-ABI) against the oracle.

The oracle is oracle/_ref/libdcsc_ref.so — the reference's own solver
translation units compiled here (oracle/Makefile) — on identical seeded inputs.
Tolerances (BASELINE.json north_star): FP64 <= 1e-9 relative, FP32 <= 1e-4.
"""
import numpy as np
import pytest

from oracle import ref
from paper_1709_09479_b200 import dcsc

pytestmark = pytest.mark.gpu

FP64_TOL = 1e-9
FP32_TOL = 1e-4


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def problem(N, grid, K, m, p=0.05, sigma=0.01, seed=7, fp32=False):
    x, _ = dcsc.synth_generate(N, grid, K, m, p, sigma, seed, fp32)
    d0 = ref.init_dictionary(K, (m, m), grid, seed=3)
    return x, d0


# ---------------------------------------------------------------- FFT
@pytest.mark.parametrize("H,W", [(16, 16), (16, 20), (20, 20), (64, 64), (100, 100)])
def test_dft_fp64_matches_reference(H, W):
    rng = np.random.default_rng(H * 1000 + W)
    x = rng.standard_normal((3, H, W))
    g = dcsc.forward_dft2(x, 64)
    r = np.stack([ref.forward_dft(xi) for xi in x])[..., : W // 2 + 1]
    assert rel(g.view(np.float64), r.view(np.float64)) <= 1e-13
    back = dcsc.inverse_dft2(g, W, 64)
    assert rel(back, x) <= 1e-13


@pytest.mark.parametrize("H,W", [(16, 16), (16, 20), (20, 20), (64, 64), (100, 100), (128, 128), (256, 256)])
def test_dft_fp32_matches_reference(H, W):
    rng = np.random.default_rng(H * 7 + W)
    x = rng.standard_normal((4, H, W)).astype(np.float32).astype(np.float64)
    g = dcsc.forward_dft2(x, 32)
    r = np.stack([ref.forward_dft(xi) for xi in x])[..., : W // 2 + 1]
    assert rel(g.view(np.float64), r.view(np.float64)) <= 2e-6
    back = dcsc.inverse_dft2(r, W, 32)
    assert rel(back, x) <= 2e-6


def test_dft_fp32_256_large_batch():
    # 300 planes on the persistent 256 x 256 cluster transforms (more planes than
    # resident clusters: every cluster walks several); numpy's FP64 FFT as the reference
    rng = np.random.default_rng(256)
    x = rng.standard_normal((300, 256, 256)).astype(np.float32).astype(np.float64)
    g = dcsc.forward_dft2(x, 32)
    r = np.fft.rfft2(x)
    assert rel(g.view(np.float64), r.view(np.float64)) <= 2e-6
    for i in (0, 32, 33, 299):
        assert rel(g[i].view(np.float64), r[i].view(np.float64)) <= 2e-6
    back = dcsc.inverse_dft2(r, 256, 32)
    assert rel(back, x) <= 2e-6
    assert rel(back[299], x[299]) <= 2e-6


def test_dft_known_answers():
    # test_spectral.cpp:15-32: impulse -> all ones; constant c -> (D c, 0, ...)
    x = np.zeros((1, 16, 20))
    x[0, 0, 0] = 1.0
    g = dcsc.forward_dft2(x, 64)
    assert np.abs(g - 1.0).max() <= 1e-14
    c = np.full((1, 16, 20), 0.75)
    g = dcsc.forward_dft2(c, 64)
    assert abs(g[0, 0, 0] - 0.75 * 320) <= 1e-12
    g[0, 0, 0] = 0
    assert np.abs(g).max() <= 1e-12


# ---------------------------------------------------------------- coding
@pytest.mark.parametrize("grid,K,m,beta", [((20, 20), 4, 5, 0.1), ((16, 20), 3, 3, 0.05),
                                           ((64, 64), 8, 7, 0.5)])
def test_coding_fp64_matches_reference(grid, K, m, beta):
    x, d = problem(1, grid, K, m)
    cfg = ref.Cfg(beta=beta, max_admm=300, normalize=0)
    z_r, st_r, s_r = ref.solve_coding(x[0], d, cfg)
    z_g, st_g, s_g = dcsc.solve_coding(x[0], d, dcsc.SolverConfig(beta=beta, max_admm=300, normalize=0), precision=64)
    assert s_g["admm_iters"] == s_r["admm_iters"]
    assert s_g["converged"] == s_r["converged"]
    assert rel(z_g, z_r) <= FP64_TOL
    assert rel(st_g.theta, st_r[0]) <= FP64_TOL
    assert rel(st_g.lam, st_r[2]) <= FP64_TOL
    for key in ("dual_objective", "primal_residual", "z_change", "theta_change"):
        assert abs(s_g[key] - s_r[key]) <= FP64_TOL * max(abs(s_r[key]), 1e-12) + 1e-13, key
    assert s_g["dual_rescaled"] == s_r["dual_rescaled"]
    # warm restart from the returned state (pipeline warm start, coding.hpp:15-25)
    z_r2, _, s_r2 = ref.solve_coding(x[0], d * 0.9, cfg, st_r)
    z_g2, _, s_g2 = dcsc.solve_coding(x[0], d * 0.9, dcsc.SolverConfig(beta=beta, max_admm=300, normalize=0),
                                      st_g, precision=64)
    assert s_g2["admm_iters"] == s_r2["admm_iters"]
    assert rel(z_g2, z_r2) <= FP64_TOL


def test_coding_degenerate_dictionary():
    x, d = problem(1, (20, 20), 4, 5)
    d = np.zeros_like(d)
    z, st, s = dcsc.solve_coding(x[0], d, dcsc.SolverConfig(normalize=0))
    assert s["degenerate_dictionary"] and s["converged"]
    assert np.all(z == 0)
    assert np.allclose(st.lam, -x[0])


def test_coding_fp32_matches_reference():
    x, d = problem(1, (100, 100), 16, 11, fp32=True)
    cfg = ref.Cfg(beta=0.5, max_admm=50, normalize=0)
    z_r, st_r, s_r = ref.solve_coding(x[0], d, cfg)
    z_g, st_g, s_g = dcsc.solve_coding(x[0], d, dcsc.SolverConfig(beta=0.5, max_admm=50, normalize=0), precision=32)
    assert s_g["admm_iters"] == s_r["admm_iters"]
    assert rel(z_g, z_r) <= FP32_TOL  # element-wise maps, relative to max|z|
    og = dcsc.evaluate_objective(x[0], d, z_g, 0.5, precision=64)
    orf = ref.objective(x[0], d, z_r, 0.5)
    assert abs(og[2] - orf[2]) <= FP32_TOL * abs(orf[2])


# ---------------------------------------------------------------- objective
def test_objective_fp64_matches_reference():
    x, d = problem(2, (20, 20), 4, 5)
    rng = np.random.default_rng(5)
    z = rng.standard_normal((2, 4, 20, 20)) * (rng.random((2, 4, 20, 20)) < 0.1)
    with dcsc.Context(2, (20, 20), 4, (5, 5), dcsc.SolverConfig(beta=0.3, normalize=0), 64) as ctx:
        ctx.set_signals(x)
        ctx.set_dictionary(d)
        ctx.set_maps(z)
        og = ctx.objective()
        ld = ctx.learning_data_term()
    for n in range(2):
        orf = ref.objective(x[n], d, z[n], 0.3)
        for a, b in zip(og[n], orf):
            assert abs(a - b) <= FP64_TOL * abs(b)
    assert abs(ld - (og[0][0] + og[1][0])) <= FP64_TOL * ld


# ---------------------------------------------------------------- learning
def coded_maps(x, d, beta, max_admm=200):
    cfg = ref.Cfg(beta=beta, max_admm=max_admm, normalize=0)
    return np.stack([ref.solve_coding(xi, d, cfg)[0] for xi in x])


def test_learning_apply_fp64_matches_reference():
    x, d = problem(3, (16, 20), 4, 5)
    maps = coded_maps(x, d, 0.1)
    mu = np.array([1.0, 0.3, 2e-7, 5.0])
    rng = np.random.default_rng(9)
    v = rng.standard_normal(x.shape)
    out_r = ref.learning_apply(maps, (5, 5), mu, 1e-6, v)
    with dcsc.Context(3, (16, 20), 4, (5, 5), dcsc.SolverConfig(normalize=0), 64) as ctx:
        ctx.set_signals(x)
        ctx.set_maps(maps)
        out_g = ctx.learning_apply(mu, v)
    assert rel(out_g, out_r) <= 1e-12


@pytest.mark.parametrize("grid,N,K,m", [((20, 20), 3, 4, 5), ((16, 20), 2, 3, 3)])
def test_learning_fp64_matches_reference(grid, N, K, m):
    x, d = problem(N, grid, K, m)
    maps = coded_maps(x, d, 0.1)
    cfg = ref.Cfg(beta=0.1, normalize=0)
    d_r, st_r, s_r = ref.solve_learning(x, maps, (m, m), cfg)
    d_g, st_g, s_g = dcsc.solve_learning(x, maps, (m, m), dcsc.SolverConfig(beta=0.1, normalize=0), precision=64)
    assert s_g["mu_iters"] == s_r["mu_iters"]
    assert abs(s_g["cg_iters"] - s_r["cg_iters"]) <= max(2, 0.02 * s_r["cg_iters"])
    assert rel(d_g, d_r) <= 1e-7
    assert rel(st_g.mu, st_r[1]) <= 1e-7
    # warm second solve
    d_r2, _, s_r2 = ref.solve_learning(x, maps * 1.1, (m, m), cfg, st_r)
    d_g2, _, s_g2 = dcsc.solve_learning(x, maps * 1.1, (m, m), dcsc.SolverConfig(beta=0.1, normalize=0), st_g,
                                        precision=64)
    assert rel(d_g2, d_r2) <= 1e-7


def test_learning_degenerate_zero_maps():
    x, d = problem(2, (20, 20), 4, 5)
    d_g, _, s = dcsc.solve_learning(x, np.zeros((2, 4, 20, 20)), (5, 5), dcsc.SolverConfig(normalize=0))
    assert s["degenerate"] and np.all(d_g == 0)


# ---------------------------------------------------------------- full run
def compare_runs(g, r, tol):
    tg, tr = g["trace"], r["trace"]
    assert len(tg) == len(tr)
    for a, b in zip(tg, tr):
        assert a["phase"] == b["phase"]
        for key in ("total", "data_term", "l1_term"):
            assert abs(a[key] - b[key]) <= tol * abs(b[key]) + 1e-300, (a, b, key)


def test_run_fp64_small_matches_reference():
    x, _ = problem(3, (20, 20), 6, 5, p=0.05)
    cfg = ref.Cfg(beta=0.2, max_outer=3, normalize=0, seed=11, tol=1e-300)
    r = ref.run(x, 6, (5, 5), cfg)
    g = dcsc.run_csc(x, 6, (5, 5), dcsc.SolverConfig(beta=0.2, max_outer=3, normalize=0, seed=11, tol=1e-300),
                     precision=64)
    compare_runs(g, r, 1e-8)
    for a, b in zip(g["trace"], r["trace"]):
        assert a["admm_iters"] == b["admm_iters"]
        assert a["mu_iters"] == b["mu_iters"]
    assert rel(g["dict"], r["dict"]) <= 1e-7


# ---------------------------------------------------------------- 256 x 256 (C3 planes: 4-CTA cluster FFT)
def test_cluster_plane_coding_fp32_matches_reference():
    x, d = problem(1, (256, 256), 4, 11, p=0.01, fp32=True)
    cfg = ref.Cfg(beta=0.5, max_admm=25, normalize=0)
    z_r, st_r, s_r = ref.solve_coding(x[0], d, cfg)
    z_g, st_g, s_g = dcsc.solve_coding(x[0], d, dcsc.SolverConfig(beta=0.5, max_admm=25, normalize=0), precision=32)
    assert s_g["admm_iters"] == s_r["admm_iters"]
    assert rel(z_g, z_r) <= FP32_TOL
    og = dcsc.evaluate_objective(x[0], d, z_g, 0.5, precision=32)
    orf = ref.objective(x[0], d, z_r, 0.5)
    assert abs(og[2] - orf[2]) <= FP32_TOL * abs(orf[2])
    assert abs(s_g["dual_objective"] - s_r["dual_objective"]) <= FP32_TOL * abs(s_r["dual_objective"])


def test_cluster_plane_learning_apply_fp32_matches_reference():
    rng = np.random.default_rng(21)
    maps = rng.standard_normal((2, 3, 256, 256)) * (rng.random((2, 3, 256, 256)) < 0.01)
    mu = np.array([1.0, 0.4, 2.0])
    v = rng.standard_normal((2, 256, 256))
    out_r = ref.learning_apply(maps, (11, 11), mu, 1e-6, v)
    with dcsc.Context(2, (256, 256), 3, (11, 11), dcsc.SolverConfig(normalize=0), 32) as ctx:
        ctx.set_signals(np.zeros((2, 256, 256)))
        ctx.set_maps(maps.astype(np.float32).astype(np.float64))
        out_g = ctx.learning_apply(mu, v)
    assert rel(out_g, out_r) <= 1e-5


def test_cluster_plane_learning_fp32_matches_reference():
    x, d = problem(2, (256, 256), 3, 11, p=0.01, fp32=True)
    maps = np.stack([ref.solve_coding(xi, d, ref.Cfg(beta=0.5, max_admm=10, normalize=0))[0] for xi in x])
    maps = maps.astype(np.float32).astype(np.float64)
    cfg = ref.Cfg(beta=0.5, normalize=0, max_mu_iters=2, cg_max=12)
    d_r, _, s_r = ref.solve_learning(x, maps, (11, 11), cfg)
    d_g, _, s_g = dcsc.solve_learning(x, maps, (11, 11), dcsc.SolverConfig(beta=0.5, normalize=0, max_mu_iters=2,
                                                                           cg_max=12), precision=32)
    assert s_g["mu_iters"] == s_r["mu_iters"]
    assert rel(d_g, d_r) <= FP32_TOL
    # the learning data term of both dictionaries agrees to the FP32 bar
    with dcsc.Context(2, (256, 256), 3, (11, 11), dcsc.SolverConfig(normalize=0), 64 if False else 32) as ctx:
        ctx.set_signals(x)
        ctx.set_maps(maps)
        a, b = ctx.learning_data_term(d_g), ctx.learning_data_term(d_r)
    assert abs(a - b) <= FP32_TOL * abs(b)


def test_cluster_plane_run_fp32_matches_reference():
    """run_csc on the 256x256 cluster family over 2 outer iterations: the
    learned dictionary re-enters coding through set_dictionary (rank-blocked
    d_hat copy rebuilt), so a stale copy would show in the second outer step."""
    x, _ = problem(2, (256, 256), 3, 11, p=0.01, fp32=True)
    kw = dict(beta=0.5, max_outer=2, normalize=0, seed=9, tol=1e-300, max_admm=20, max_mu_iters=3, cg_max=15)
    r = ref.run(x, 3, (11, 11), ref.Cfg(**kw))
    g = dcsc.run_csc(x, 3, (11, 11), dcsc.SolverConfig(**kw), precision=32)
    compare_runs(g, r, FP32_TOL)
    assert rel(g["dict"], r["dict"]) <= FP32_TOL


@pytest.mark.parametrize("mode", [1, 2])
def test_run_with_normalisation_matches_reference(mode):
    """normalize Global (1) / Local (2) (pipeline.cpp:78-121) inside run_csc."""
    rng = np.random.default_rng(40 + mode)
    x = rng.random((2, 20, 20)) * 3.0 + 1.0  # raw, un-normalised signals
    cfg = ref.Cfg(beta=0.3, max_outer=2, normalize=mode, seed=5, tol=1e-300, max_admm=120)
    r = ref.run(x, 4, (5, 5), cfg)
    g = dcsc.run_csc(x, 4, (5, 5), dcsc.SolverConfig(beta=0.3, max_outer=2, normalize=mode, seed=5, tol=1e-300,
                                                     max_admm=120), precision=64)
    compare_runs(g, r, 1e-9)
    assert rel(g["dict"], r["dict"]) <= 1e-7


# ---------------------------------------------------------------- edge cases
def test_single_filter_and_full_support_fp64():
    # K = 1 and a filter support equal to the grid (types.cpp:106-114 allows support == dims)
    x, _ = problem(1, (16, 16), 1, 16)
    d = ref.init_dictionary(1, (16, 16), (16, 16), seed=4)
    cfg = ref.Cfg(beta=0.05, max_admm=200, normalize=0)
    z_r, st_r, s_r = ref.solve_coding(x[0], d, cfg)
    z_g, st_g, s_g = dcsc.solve_coding(x[0], d, dcsc.SolverConfig(beta=0.05, max_admm=200, normalize=0))
    assert s_g["admm_iters"] == s_r["admm_iters"]
    assert rel(z_g, z_r) <= FP64_TOL and rel(st_g.lam, st_r[2]) <= FP64_TOL


def test_support_larger_than_grid_is_a_dimension_error():
    with pytest.raises(dcsc.DimensionError):
        dcsc.Context(1, (16, 16), 2, (17, 3), dcsc.SolverConfig(normalize=0), 64)


def test_coding_image_subranges_are_independent():
    # batched coding over [n0, n1) equals coding each image alone (pipeline.cpp:221-227)
    x, d = problem(4, (20, 20), 4, 5)
    sc = dcsc.SolverConfig(beta=0.1, max_admm=150, normalize=0)
    with dcsc.Context(4, (20, 20), 4, (5, 5), sc, 64) as ctx:
        ctx.set_signals(x)
        ctx.set_dictionary(d)
        s_a = ctx.coding(1, 3)
        _, z_a, lam_a = ctx.get_coding_state(1, 3)
        s_b = ctx.coding(0, 4)
        _, z_b, _ = ctx.get_coding_state(0, 4)
    for i, n in enumerate((1, 2)):
        z1, st1, s1 = dcsc.solve_coding(x[n], d, sc)
        assert s_a[i]["admm_iters"] == s1["admm_iters"]
        assert rel(z_a[i], z1) <= 1e-12 and rel(lam_a[i], st1.lam) <= 1e-12
    # the second call warm-starts images 1, 2 from their state and cold-starts 0, 3
    assert s_b[1]["admm_iters"] <= s_a[0]["admm_iters"]


def test_huge_beta_gives_zero_maps_and_lambda_minus_x():
    x, d = problem(1, (20, 20), 4, 5)
    z, st, s = dcsc.solve_coding(x[0], d, dcsc.SolverConfig(beta=1e6, rho=1.0, max_admm=500, normalize=0))
    assert np.all(z == 0)
    # a property of the converged iterate, not a reference comparison: ADMM stops at its
    # relative tolerance (coding.cpp:264-283), so lambda equals -x to that tolerance only
    assert rel(st.lam, -x[0]) <= 1e-3
    z_r, st_r, s_r = ref.solve_coding(x[0], d, ref.Cfg(beta=1e6, rho=1.0, max_admm=500, normalize=0))
    assert s["admm_iters"] == s_r["admm_iters"] and rel(st.lam, st_r[2]) <= FP64_TOL


def test_learning_correlation_fp64_matches_reference():
    # LearningOperator::correlation (learning.cpp:124-134), a13 of SURVEY.md 8(a)
    x, d = problem(3, (16, 20), 4, 5)
    maps = coded_maps(x, d, 0.1)
    rng = np.random.default_rng(4)
    v = rng.standard_normal(x.shape)
    out_r = ref.learning_correlation(maps, (5, 5), v)
    with dcsc.Context(3, (16, 20), 4, (5, 5), dcsc.SolverConfig(normalize=0), 64) as ctx:
        ctx.set_signals(x)
        ctx.set_maps(maps)
        out_g = ctx.learning_correlation(v)
    assert rel(out_g, out_r) <= 1e-12


# ---------------------------------------------------------------- stateless ops (coding.hpp:45-66, learning.hpp:81-95)
def test_stateless_coding_ops_fp64_match_reference():
    x, d = problem(2, (20, 20), 4, 5)
    rng = np.random.default_rng(11)
    theta = rng.standard_normal((2, 4, 20, 20)) * 0.1
    z = rng.standard_normal((2, 4, 20, 20)) * 0.1
    lam = rng.standard_normal((2, 20, 20))
    with dcsc.Context(2, (20, 20), 4, (5, 5), dcsc.SolverConfig(rho=0.3, normalize=0), 64) as ctx:
        ctx.set_signals(x)
        ctx.set_dictionary(d)
        lg = ctx.lambda_update(theta, z)
        tg = ctx.dictionary_adjoint(lam)
    for n in range(2):
        assert rel(lg[n], ref.lambda_update(x[n], d, theta[n], z[n], 0.3)) <= 1e-12
        assert rel(tg[n], ref.dictionary_adjoint(d, lam[n])) <= 1e-12


def test_stateless_learning_ops_fp64_match_reference():
    x, d = problem(3, (16, 20), 4, 5)
    maps = coded_maps(x, d, 0.1)
    mu = np.array([1.0, 0.3, 2.0, 0.7])
    g0 = np.zeros_like(x)
    with dcsc.Context(3, (16, 20), 4, (5, 5), dcsc.SolverConfig(normalize=0), 64) as ctx:
        ctx.set_signals(x)
        ctx.set_maps(maps)
        g_g, it_g, cv_g = ctx.gamma_solve(mu, g0)
        g_r, it_r, cv_r = ref.gamma_solve(maps, (5, 5), mu, 1e-6, x, 1e-6, 300, g0)
        d_g = ctx.d_recover(g_r, mu)  # same gamma on both sides
    assert cv_g == cv_r and abs(it_g - it_r) <= 2
    assert rel(g_g, g_r) <= 1e-7  # CG stops at rel. residual 1e-6 (learning.cpp:156)
    assert rel(d_g, ref.d_recover(maps, (5, 5), g_r, mu)) <= 1e-12


def test_c4_shaped_run_fp32_matches_reference():
    """A C4-shaped slice (BASELINE configs[4]: 64x64 FP32, K=32 filters 7x7,
    p=0.005, sigma=0.05) for 2 outer iterations of run_csc against the oracle on
    the same FP32-rounded inputs: objectives and dictionary <= 1e-4."""
    x, _ = dcsc.synth_generate(12, (64, 64), 32, 7, 0.005, 0.05, 20250917, True)
    kw = dict(beta=0.5, max_outer=2, normalize=0, seed=20250917, tol=1e-300, max_admm=120, max_mu_iters=10,
              cg_max=60)
    r = ref.run(x, 32, (7, 7), ref.Cfg(**kw))
    g = dcsc.run_csc(x, 32, (7, 7), dcsc.SolverConfig(**kw), precision=32)
    compare_runs(g, r, FP32_TOL)
    assert rel(g["dict"], r["dict"]) <= FP32_TOL
