"""CPU: pin the oracle before trusting it.

1. The FFTW3 shim under the compiled reference passes the reference's own
   spectral known answers (proj/tests/test_spectral.cpp) and matches numpy.fft.
2. The instrumented run_csc replica equals the reference's run_csc bit for bit.
3. The numpy restatement (oracle/dcsc_np.py) agrees with the compiled reference.
4. The compiled reference reproduces the committed golden fixtures.
"""
import os

import numpy as np
import pytest

from oracle import dcsc_np, ref
from paper_1709_09479_b200 import dcsc

GOLD = os.path.join(os.path.dirname(__file__), "golden")

pytestmark = pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")


def direct_dft(x):
    """O(D^2) DFT (oracle.cpp:79-99 restated)."""
    dims = x.shape
    idx = np.array(np.unravel_index(np.arange(x.size), dims)).T
    ph = np.zeros((x.size, x.size))
    for a, n in enumerate(dims):
        ph += np.outer(idx[:, a], idx[:, a]) / n
    return (np.exp(-2j * np.pi * ph) @ x.ravel()).reshape(dims)


def test_dft_impulse_is_all_ones():  # test_spectral.cpp:15-23
    x = np.zeros((4, 6))
    x[0, 0] = 1
    assert np.abs(ref.forward_dft(x) - 1).max() < 1e-14


def test_dft_constant():  # test_spectral.cpp:25-32
    x = np.full((5, 4), 2.5)
    X = ref.forward_dft(x)
    assert abs(X[0, 0] - 50.0) < 1e-12
    X[0, 0] = 0
    assert np.abs(X).max() < 1e-12


@pytest.mark.parametrize("shape", [(8,), (4, 6), (3, 4, 2)])
def test_dft_matches_direct(shape):  # test_spectral.cpp:34-44
    x = np.random.default_rng(1).standard_normal(shape)
    assert np.abs(ref.forward_dft(x) - direct_dft(x)).max() < 1e-10


@pytest.mark.parametrize("shape", [(16, 16), (100, 100), (128, 128), (20, 16), (7, 9)])
def test_dft_round_trip_and_numpy(shape):  # test_spectral.cpp:46-59
    x = np.random.default_rng(2).standard_normal(shape)
    X = ref.forward_dft(x)
    assert np.abs(X - np.fft.fftn(x)).max() < 1e-12 * np.abs(X).max()
    assert np.abs(ref.inverse_dft(X) - x).max() < 1e-12


def test_inverse_all_ones_is_impulse():  # test_spectral.cpp:61-74
    x = ref.inverse_dft(np.ones((4, 4), dtype=np.complex128))
    e = np.zeros((4, 4))
    e[0, 0] = 1
    assert np.abs(x - e).max() < 1e-14


def test_inverse_residue_guard_throws():  # test_spectral.cpp:76-80
    s = np.zeros((4, 4), dtype=np.complex128)
    s[1, 0] = 1j
    with pytest.raises(RuntimeError):
        ref.inverse_dft(s)


def test_parseval():  # test_spectral.cpp:149-159
    x = np.random.default_rng(3).standard_normal((12, 10))
    X = ref.forward_dft(x)
    assert abs((x * x).sum() - (np.abs(X) ** 2).sum() / x.size) < 1e-10


def test_init_dictionary_restatement_matches():
    d_ref = ref.init_dictionary(5, (3, 4), (10, 10), 42)
    d_np = dcsc_np.init_dictionary(5, (3, 4), 42)
    assert np.array_equal(d_ref, d_np)


def small_problem(N=2, grid=(16, 20), K=3, m=5, seed=7):
    x, _ = dcsc.synth_generate(N, grid, K, m, 0.05, 0.01, seed, False)
    d = ref.init_dictionary(K, (m, m), grid, 3)
    return x, d


def test_numpy_coding_matches_reference():
    x, d = small_problem()
    z_r, (th_r, _, lam_r), s_r = ref.solve_coding(x[0], d, ref.Cfg(beta=0.1, max_admm=150, normalize=0))
    z_n, th_n, lam_n, s_n = dcsc_np.solve_coding(x[0], d, 0.1, 0.1, 150)
    assert s_r["admm_iters"] == s_n["admm_iters"]
    assert np.abs(z_r - z_n).max() <= 1e-10 * np.abs(z_r).max()
    assert np.abs(lam_r - lam_n).max() <= 1e-10 * np.abs(lam_r).max()
    assert abs(s_r["dual_objective"] - s_n["dual_objective"]) <= 1e-10 * abs(s_r["dual_objective"])


def test_numpy_learning_matches_reference():
    x, d = small_problem()
    maps = np.stack([ref.solve_coding(xi, d, ref.Cfg(beta=0.1, max_admm=100, normalize=0))[0] for xi in x])
    d_r, (g_r, mu_r), s_r = ref.solve_learning(x, maps, (5, 5), ref.Cfg(beta=0.1, normalize=0))
    cfg = dict(mu_floor=1e-6, cg_tol=1e-6, cg_max=300, max_mu_iters=60)
    d_n, g_n, mu_n, s_n = dcsc_np.solve_learning(x, maps, (5, 5), cfg)
    assert s_r["mu_iters"] == s_n["mu_iters"]
    assert np.abs(d_r - d_n).max() <= 1e-8 * np.abs(d_r).max()
    assert np.abs(mu_r - mu_n).max() <= 1e-8 * np.abs(mu_r).max()


def test_numpy_objective_matches_reference():
    x, d = small_problem()
    z = np.random.default_rng(4).standard_normal((3, 16, 20)) * 0.1
    a = ref.objective(x[0], d, z, 0.3)
    b = dcsc_np.objective(x[0], d, z, 0.3)
    assert abs(a[0] - b[0]) <= 1e-11 * a[0] and abs(a[1] - b[1]) <= 1e-12 * a[1]


def test_learning_apply_matches_numpy():
    x, d = small_problem()
    maps = np.random.default_rng(5).standard_normal((2, 3, 16, 20)) * (np.random.default_rng(6).random((2, 3, 16, 20)) < 0.2)
    mu = np.array([1.0, 0.5, 3e-7])
    v = np.random.default_rng(7).standard_normal((2, 16, 20))
    op = dcsc_np.LearningOperator(maps, (5, 5), 1e-6)
    op.set_mu(mu)
    a = ref.learning_apply(maps, (5, 5), mu, 1e-6, v)
    assert np.abs(a - op.apply(v)).max() <= 1e-11 * np.abs(a).max()


def test_replica_equals_run_csc_bitwise():
    ref.set_threads(1)
    x, _ = dcsc.synth_generate(2, (16, 16), 4, 3, 0.05, 0.01, 9, False)
    cfg = ref.Cfg(beta=0.2, max_outer=2, normalize=1, seed=5, max_admm=80)
    a = ref.run(x, 4, (3, 3), cfg)
    b = ref.run_csc(x, 4, (3, 3), cfg)
    ref.set_threads(0)
    assert len(a["trace"]) == len(b["trace"])
    for r1, r2 in zip(a["trace"], b["trace"]):
        for k in ("total", "data_term", "l1_term", "residual_norm", "admm_iters", "cg_iters"):
            assert r1[k] == r2[k], k
    assert np.array_equal(a["dict"], b["dict"])
    assert np.array_equal(a["maps"], b["maps"])


def test_numpy_run_matches_reference():
    x, _ = dcsc.synth_generate(2, (16, 16), 4, 3, 0.05, 0.01, 9, False)
    cfgr = ref.Cfg(beta=0.2, max_outer=2, normalize=0, seed=5, max_admm=80, tol=1e-300)
    a = ref.run(x, 4, (3, 3), cfgr)
    b = dcsc_np.run_csc(x, 4, (3, 3), dict(beta=0.2, rho=0.1, max_outer=2, max_admm=80, seed=5, tol=1e-300,
                                           mu_floor=1e-6, cg_tol=1e-6, cg_max=300, max_mu_iters=60))
    for r1, r2 in zip(a["trace"], b["trace"]):
        assert abs(r1["total"] - r2["total"]) <= 1e-9 * abs(r1["total"])
    assert np.abs(a["dict"] - b["dict"]).max() <= 1e-8


def test_reference_reproduces_golden_small():
    g = np.load(os.path.join(GOLD, "run_small_fp64.npz"))
    c = g["cfg"]
    cfg = ref.Cfg(beta=c[0], rho=c[1], tol=c[2], max_outer=int(c[3]), max_admm=int(c[4]), max_mu_iters=int(c[5]),
                  cg_tol=c[6], cg_max=int(c[7]), mu_floor=c[8], seed=int(c[9]), normalize=int(c[10]))
    N, H, W, K, m = (int(v) for v in g["shape"])
    x, _ = dcsc.synth_generate(N, (H, W), K, m, *g["gen"][:2], int(g["gen"][2]), bool(g["gen"][3]))
    assert np.array_equal(x, g["x"])  # the generator is pinned too
    r = ref.run(x, K, (m, m), cfg)
    keys = list(g["trace_keys"])
    for row, grow in zip(r["trace"], g["trace"]):
        for k in ("total", "data_term", "l1_term"):
            assert abs(row[k] - grow[keys.index(k)]) <= 1e-12 * abs(grow[keys.index(k)])
        assert row["admm_iters"] == grow[keys.index("admm_iters")]
