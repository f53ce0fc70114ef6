"""GPU parity of the multi-channel (J > 1, TCSC / Joint channel mode) path.

The checker is the reference's own TCSC translation unit (proj/src/tcsc.cpp)
compiled into oracle/_ref (oracle/Makefile, Eigen-API shim), called through
oracle/ref.py on identical inputs. Tolerances as for J = 1: FP64 <= 1e-9
relative for coding (learning / runs 1e-7 like test_gpu_parity.py, CG
iteration counts may differ by a step), FP32 objective <= 1e-4.
"""
import numpy as np
import pytest

from oracle import ref
from paper_1709_09479_b200 import dcsc

pytestmark = pytest.mark.gpu

FP64_TOL = 1e-9


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def problem(N, J, grid, K, m, seed=5, fp32=False):
    rng = np.random.default_rng(seed)
    # J-channel synthetic images: shared sparse maps through a random J-channel dictionary + noise
    dt = rng.standard_normal((K, J, m, m))
    dt /= np.sqrt((dt ** 2).sum(axis=(1, 2, 3), keepdims=True))
    z = rng.laplace(size=(N, K) + grid) * (rng.random((N, K) + grid) < 0.03)
    dh = np.fft.fft2(np.pad(dt, ((0, 0), (0, 0), (0, grid[0] - m), (0, grid[1] - m))))
    x = np.fft.ifft2(np.einsum("kjhw,nkhw->njhw", dh, np.fft.fft2(z))).real
    x += 0.01 * rng.standard_normal(x.shape)
    if fp32:
        x = x.astype(np.float32).astype(np.float64)
    d0 = ref.init_dictionary_j(K, J, (m, m), grid, seed=3)
    return x, d0


@pytest.mark.parametrize("J,grid,K,m,beta", [(2, (20, 20), 4, 5, 0.1), (3, (16, 20), 3, 3, 0.05),
                                             (4, (16, 16), 2, 3, 0.1)])
def test_tcsc_coding_fp64_matches_reference(J, grid, K, m, beta):
    x, d = problem(1, J, grid, K, m)
    cfg = ref.Cfg(beta=beta, max_admm=300, normalize=0)
    z_r, st_r, s_r = ref.solve_coding_tcsc(x[0], d, cfg)
    sc = dcsc.SolverConfig(beta=beta, max_admm=300, normalize=0)
    z_g, st_g, s_g = dcsc.solve_coding_tcsc(x[0], d, sc, precision=64)
    assert s_g["admm_iters"] == s_r["admm_iters"]
    assert s_g["converged"] == s_r["converged"]
    assert rel(z_g, z_r) <= FP64_TOL
    assert rel(st_g.theta, st_r[0]) <= FP64_TOL
    assert rel(st_g.lam, st_r[2]) <= FP64_TOL
    for key in ("dual_objective", "primal_residual", "z_change", "theta_change"):
        assert abs(s_g[key] - s_r[key]) <= FP64_TOL * max(abs(s_r[key]), 1e-12) + 1e-13, key
    # warm restart from the returned state
    z_r2, _, s_r2 = ref.solve_coding_tcsc(x[0], d * 0.9, cfg, st_r)
    z_g2, _, s_g2 = dcsc.solve_coding_tcsc(x[0], d * 0.9, sc, st_g, precision=64)
    assert s_g2["admm_iters"] == s_r2["admm_iters"]
    assert rel(z_g2, z_r2) <= FP64_TOL


def test_tcsc_woodbury_regime_fp64():  # K < J: the reference's Auto route is Woodbury
    x, d = problem(1, 5, (16, 16), 2, 3, seed=9)
    cfg = ref.Cfg(beta=0.1, max_admm=200, normalize=0)
    z_r, st_r, s_r = ref.solve_coding_tcsc(x[0], d, cfg)
    z_g, st_g, s_g = dcsc.solve_coding_tcsc(x[0], d, dcsc.SolverConfig(beta=0.1, max_admm=200, normalize=0))
    assert s_g["admm_iters"] == s_r["admm_iters"]
    assert rel(z_g, z_r) <= FP64_TOL and rel(st_g.lam, st_r[2]) <= FP64_TOL


def test_tcsc_zero_signal_and_degenerate_dictionary():
    x, d = problem(1, 3, (20, 20), 4, 5)
    z, _, s = dcsc.solve_coding_tcsc(np.zeros_like(x[0]), d, dcsc.SolverConfig(normalize=0))
    assert np.all(z == 0) and s["converged"]
    z, st, s = dcsc.solve_coding_tcsc(x[0], np.zeros_like(d), dcsc.SolverConfig(normalize=0))
    assert s["degenerate_dictionary"] and np.all(z == 0) and np.allclose(st.lam, -x[0])


def test_tcsc_coding_fp32_matches_reference():
    x, d = problem(1, 3, (64, 64), 8, 7, fp32=True)
    cfg = ref.Cfg(beta=0.1, max_admm=60, normalize=0)
    z_r, _, s_r = ref.solve_coding_tcsc(x[0], d, cfg)
    z_g, _, s_g = dcsc.solve_coding_tcsc(x[0], d, dcsc.SolverConfig(beta=0.1, max_admm=60, normalize=0), precision=32)
    assert s_g["admm_iters"] == s_r["admm_iters"]
    og = ref.objective_j(x[0], d, z_g, 0.1)
    orf = ref.objective_j(x[0], d, z_r, 0.1)
    assert abs(og[2] - orf[2]) <= 1e-4 * abs(orf[2])


def test_tcsc_objective_fp64_matches_reference():
    x, d = problem(2, 3, (20, 20), 4, 5)
    rng = np.random.default_rng(5)
    z = rng.standard_normal((2, 4, 20, 20)) * (rng.random((2, 4, 20, 20)) < 0.1)
    with dcsc.Context(2, (20, 20), 4, (5, 5), dcsc.SolverConfig(beta=0.3, normalize=0), 64, channels=3) as ctx:
        ctx.set_signals(x)
        ctx.set_dictionary(d)
        ctx.set_maps(z)
        og = ctx.objective()
        ld = ctx.learning_data_term()
    for n in range(2):
        orf = ref.objective_j(x[n], d, z[n], 0.3)
        for a, b in zip(og[n], orf):
            assert abs(a - b) <= FP64_TOL * abs(b)
    assert abs(ld - (og[0][0] + og[1][0])) <= FP64_TOL * ld


@pytest.mark.parametrize("J", [2, 3])
def test_tcsc_learning_fp64_matches_reference(J):
    x, d = problem(3, J, (20, 20), 4, 5)
    cfg = ref.Cfg(beta=0.1, max_admm=200, normalize=0)
    maps = np.stack([ref.solve_coding_tcsc(xi, d, cfg)[0] for xi in x])
    d_r, st_r, s_r = ref.solve_learning_j(x, maps, (5, 5), cfg)
    d_g, st_g, s_g = dcsc.solve_learning(x, maps, (5, 5), dcsc.SolverConfig(beta=0.1, normalize=0), precision=64)
    assert d_g.shape == d_r.shape
    assert s_g["mu_iters"] == s_r["mu_iters"]
    assert abs(s_g["cg_iters"] - s_r["cg_iters"]) <= max(2 * J, 0.02 * s_r["cg_iters"])
    assert rel(d_g, d_r) <= 1e-7
    assert rel(st_g.mu, st_r[1]) <= 1e-7
    assert rel(st_g.gamma, st_r[0]) <= 1e-6


def test_tcsc_run_fp64_matches_reference():
    x, _ = problem(3, 3, (20, 20), 6, 5, seed=8)
    cfg = ref.Cfg(beta=0.2, max_outer=3, max_admm=150, normalize=1, seed=11, tol=1e-300)
    r = ref.run_j(x, 6, (5, 5), cfg)
    g = dcsc.run_csc(x, 6, (5, 5), dcsc.SolverConfig(beta=0.2, max_outer=3, max_admm=150, normalize=1, seed=11,
                                                     tol=1e-300), precision=64)
    assert len(g["trace"]) == len(r["trace"])
    for a, b in zip(g["trace"], r["trace"]):
        assert a["phase"] == b["phase"] and a["admm_iters"] == b["admm_iters"] and a["mu_iters"] == b["mu_iters"]
        for key in ("total", "data_term", "l1_term"):
            assert abs(a[key] - b[key]) <= 1e-8 * abs(b[key]), (a, b, key)
    assert rel(g["dict"], r["dict"]) <= 1e-7


# ---------------------------------------------------------------- reconstruct / encode
@pytest.mark.parametrize("J,prec,tol", [(1, 64, 1e-12), (3, 64, 1e-12), (1, 32, 2e-5), (3, 32, 2e-5)])
def test_reconstruct_matches_reference(J, prec, tol):
    rng = np.random.default_rng(J + prec)
    K, m, grid = 5, 5, (20, 20)
    d = rng.standard_normal((K, J, m, m)) if J > 1 else rng.standard_normal((K, m, m))
    z = rng.standard_normal((K,) + grid) * (rng.random((K,) + grid) < 0.1)
    assert rel(dcsc.reconstruct(d, z, precision=prec), ref.reconstruct(d, z)) <= tol


def test_encode_matches_reference_cli_path():
    x, d = problem(1, 3, (20, 20), 4, 5, seed=12)
    cfg = dcsc.SolverConfig(beta=0.1, max_admm=200, normalize=1)
    z, obj, st = dcsc.encode(x[0], d, cfg)
    xn = dcsc.Context(1, (20, 20), 4, (5, 5), cfg, 64, channels=3)
    xn.set_signals(x[0][None])
    xnorm = xn.get_signals()[0]
    xn.close()
    z_r, _, s_r = ref.solve_coding_tcsc(xnorm, d, ref.Cfg(beta=0.1, max_admm=200, normalize=0))
    assert st["admm_iters"] == s_r["admm_iters"]
    assert rel(z, z_r) <= FP64_TOL
    o_r = ref.objective_j(xnorm, d, z_r, 0.1)
    assert abs(obj[2] - o_r[2]) <= FP64_TOL * abs(o_r[2])


# ---------------------------------------------------------------- cluster grid families (J > 1)
@pytest.mark.parametrize("J,grid,K,m,prec", [(2, (128, 128), 3, 11, 64), (3, (256, 256), 2, 11, 32)])
def test_tcsc_coding_cluster_family_matches_reference(J, grid, K, m, prec):
    """Joint mode on the 4-CTA cluster families (FP64 128x128, FP32 256x256): the
    generator sums conj(d_hat_jk) lambda_hat_j over channels and the pass stores
    w_hat_k for the per-bin J x J solves (tcsc.cpp:101-171)."""
    x, d = problem(1, J, grid, K, m, seed=9, fp32=prec == 32)
    cfg = ref.Cfg(beta=0.1, max_admm=40, normalize=0)
    z_r, st_r, s_r = ref.solve_coding_tcsc(x[0], d, cfg)
    sc = dcsc.SolverConfig(beta=0.1, max_admm=40, normalize=0)
    z_g, st_g, s_g = dcsc.solve_coding_tcsc(x[0], d, sc, precision=prec)
    if prec == 64:
        assert s_g["admm_iters"] == s_r["admm_iters"]
        assert rel(z_g, z_r) <= FP64_TOL
        assert rel(st_g.lam, st_r[2]) <= FP64_TOL
        assert abs(s_g["dual_objective"] - s_r["dual_objective"]) <= FP64_TOL * abs(s_r["dual_objective"])
    else:
        assert abs(s_g["dual_objective"] - s_r["dual_objective"]) <= 1e-4 * abs(s_r["dual_objective"])
        og = dcsc.evaluate_objective(x[0], d, z_g, 0.1, precision=32)
        orf = ref.objective_j(x[0], d, z_r, 0.1)
        assert abs(og[2] - orf[2]) <= 1e-4 * abs(orf[2])


def test_tcsc_run_cluster_family_fp64_matches_reference():
    """run_csc in Joint mode (J = 2) on the FP64 128x128 cluster family: coding,
    objective (tc_objective over the stored z_hat), learning, 2 outer iterations."""
    x, _ = problem(2, 2, (128, 128), 3, 11, seed=12)
    kw = dict(beta=0.1, max_outer=2, normalize=0, seed=7, tol=1e-300, max_admm=40, max_mu_iters=6, cg_max=40)
    r = ref.run_j(x, 3, (11, 11), ref.Cfg(**kw))
    g = dcsc.run_csc(x, 3, (11, 11), dcsc.SolverConfig(**kw), precision=64)
    assert len(g["trace"]) == len(r["trace"])
    for a, b in zip(g["trace"], r["trace"]):
        assert a["admm_iters"] == b["admm_iters"]
        for key in ("total", "data_term", "l1_term"):
            assert abs(a[key] - b[key]) <= 1e-8 * abs(b[key]), (key, a, b)
    assert rel(g["dict"], r["dicts"][-1]) <= 1e-7
