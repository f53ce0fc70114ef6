"""CPU: pin the multi-channel (J > 1, TCSC) oracle.

The reference's TCSC translation unit (proj/src/tcsc.cpp) is compiled unmodified
into oracle/_ref against the Eigen-API shim (oracle/eigen_shim/). These tests
restate the reference's own TCSC known answers (proj/tests/test_tcsc.cpp) on
the compiled library and check the numpy restatement (oracle/dcsc_np.py
solve_coding_tcsc) against it.
"""
import numpy as np
import pytest

from oracle import dcsc_np, ref

pytestmark = pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")


def _case(seed, J=3, H=12, W=10, K=4, m=3):
    rng = np.random.default_rng(seed)
    return rng.standard_normal((J, H, W)), rng.standard_normal((K, J, m, m))


def test_tcsc_at_j1_is_the_scalar_path():  # test_tcsc.cpp:91-110
    x, d = _case(0, J=1)
    cfg = ref.Cfg(beta=0.2, max_admm=30, normalize=0)
    z1, (_, _, l1), s1 = ref.solve_coding_tcsc(x, d, cfg)
    zs, (_, _, ls), ss = ref.solve_coding(x[0], d[:, 0], cfg)
    assert np.abs(z1 - zs).max() <= 1e-12 * max(np.abs(zs).max(), 1.0)
    assert np.abs(l1[0] - ls).max() <= 1e-12
    assert s1["admm_iters"] == ss["admm_iters"]


def test_woodbury_and_direct_agree():  # test_tcsc.cpp:167-182
    x, d = _case(1, J=5, K=2)  # K < J: Auto picks Woodbury
    cfg = ref.Cfg(beta=0.2, max_admm=25, normalize=0)
    zd, (_, _, ld), _ = ref.solve_coding_tcsc(x, d, cfg, method=1)
    zw, (_, _, lw), _ = ref.solve_coding_tcsc(x, d, cfg, method=2)
    assert np.abs(zd - zw).max() < 1e-9
    assert np.abs(ld - lw).max() < 1e-9


def test_zero_signal_codes_to_zero():  # test_tcsc.cpp:186-195
    _, d = _case(2)
    z, _, s = ref.solve_coding_tcsc(np.zeros((3, 12, 10)), d, ref.Cfg(beta=0.2, normalize=0))
    assert not z.any() and s["converged"]


def test_dominating_beta_gives_lambda_minus_x():  # test_tcsc.cpp:198-221
    x, d = _case(3, J=2, H=6, W=6, K=2)
    d /= np.sqrt((d ** 2).sum(axis=(1, 2, 3), keepdims=True))  # unit filters (test_util.hpp)
    dh = np.fft.fft2(dcsc_np.pad(d, x.shape[1:]))
    dtx = np.fft.ifft2(np.einsum("kjhw,jhw->khw", np.conj(dh), np.fft.fft2(x))).real
    beta = 1.5 * np.abs(dtx).max()
    z, (_, _, lam), _ = ref.solve_coding_tcsc(x, d, ref.Cfg(beta=beta, rho=0.5, max_admm=4000, normalize=0))
    assert np.abs(z).max() < 1e-8
    assert np.abs(lam + x).max() < 1e-3


@pytest.mark.parametrize("J,K", [(2, 3), (3, 4), (4, 2)])
def test_numpy_tcsc_matches_reference(J, K):
    x, d = _case(10 + J, J=J, K=K)
    cfg = ref.Cfg(beta=0.3, max_admm=40, normalize=0)
    z, (th, _, lam), s = ref.solve_coding_tcsc(x, d, cfg)
    z2, th2, lam2, s2 = dcsc_np.solve_coding_tcsc(x, d, 0.3, 0.1, 40)
    scale = max(np.abs(z).max(), 1.0)
    assert np.abs(z - z2).max() <= 1e-10 * scale
    assert np.abs(th - th2).max() <= 1e-10
    assert np.abs(lam - lam2).max() <= 1e-10 * max(np.abs(lam).max(), 1.0)
    assert s["admm_iters"] == s2["admm_iters"]
    assert abs(s["dual_objective"] - s2["dual_objective"]) <= 1e-10 * abs(s["dual_objective"])


def test_joint_learning_at_j1_is_solve_learning():  # test_tcsc.cpp:304-312
    rng = np.random.default_rng(4)
    xs = rng.standard_normal((3, 1, 12, 10))
    maps = rng.standard_normal((3, 4, 12, 10)) * (rng.random((3, 4, 12, 10)) < 0.05)
    cfg = ref.Cfg(normalize=0, max_mu_iters=5)
    d1, _, _ = ref.solve_learning_j(xs, maps, (3, 3), cfg)
    d2, _, _ = ref.solve_learning(xs[:, 0], maps, (3, 3), cfg)
    assert np.array_equal(d1[:, 0], d2)


def test_zero_channel_learns_zero_slices():  # test_tcsc.cpp:315-326
    rng = np.random.default_rng(5)
    xs = rng.standard_normal((3, 2, 12, 10))
    xs[:, 1] = 0.0
    maps = rng.standard_normal((3, 4, 12, 10)) * (rng.random((3, 4, 12, 10)) < 0.05)
    d, _, _ = ref.solve_learning_j(xs, maps, (3, 3), ref.Cfg(normalize=0, max_mu_iters=5))
    assert not d[:, 1].any()


def test_joint_replica_equals_run_csc():
    rng = np.random.default_rng(6)
    xs = rng.standard_normal((3, 3, 12, 10))
    cfg = ref.Cfg(beta=0.1, max_admm=30, max_outer=2, normalize=1, seed=3)
    ref.set_threads(1)
    try:
        a = ref.run_j(xs, 4, (3, 3), cfg)
        b = ref.run_csc_j(xs, 4, (3, 3), cfg)
    finally:
        ref.set_threads(0)
    assert len(a["trace"]) == len(b["trace"])
    for ra, rb in zip(a["trace"], b["trace"]):
        assert ra["total"] == rb["total"] and ra["admm_iters"] == rb["admm_iters"]
    assert np.array_equal(a["dict"], b["dict"]) and np.array_equal(a["maps"], b["maps"])


def test_reference_reproduces_golden_tcsc():
    import os
    from paper_1709_09479_b200 import dcsc
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "run_tcsc_j3_fp64.npz"))
    c = g["cfg"]
    cfg = ref.Cfg(beta=c[0], rho=c[1], tol=c[2], max_outer=int(c[3]), max_admm=int(c[4]), max_mu_iters=int(c[5]),
                  cg_tol=c[6], cg_max=int(c[7]), mu_floor=c[8], seed=int(c[9]), normalize=int(c[10]))
    N, H, W, K, m, J = (int(v) for v in g["shape"])
    p, sigma, seed = float(g["gen"][0]), float(g["gen"][1]), int(g["gen"][2])
    x = np.stack([dcsc.synth_generate(N, (H, W), K, m, p, sigma, seed + j, False)[0] for j in range(J)], axis=1)
    assert np.array_equal(x, g["x"])
    r = ref.run_j(x, K, (m, m), cfg)
    keys = list(g["trace_keys"])
    for row, grow in zip(r["trace"], g["trace"]):
        for k in ("total", "data_term", "l1_term"):
            assert abs(row[k] - grow[keys.index(k)]) <= 1e-12 * abs(grow[keys.index(k)])
        assert row["admm_iters"] == grow[keys.index("admm_iters")]
