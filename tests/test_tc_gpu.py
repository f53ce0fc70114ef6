"""The tensor-core spatial coding pass (kernels_tc.cuh) on the GPU.

It replaces the per-filter c2r / prox / r2c of the FFT pass by two tcgen05
GEMMs per 128-pixel tile (correlation of lambda with every filter; adjoint
convolution of w) with FP32 operands split into two scaled f16 halves (three
products). Checked here: it is the path that runs on the 256 x 256 FP32
family, it agrees with the FFT pass (DCSC_TC=0) and with the reference oracle
on the same inputs at the north-star FP32 tolerance (1e-4) with equal
iteration counts, including padded filter counts (K < 64, K = 40) and the
first-iteration theta of a warm state that is not ADMM-consistent.
"""
import numpy as np
import pytest

from oracle import ref
from paper_1709_09479_b200 import dcsc

pytestmark = pytest.mark.gpu
TOL = 1e-4


def rel(a, b):
    return float(np.abs(np.asarray(a) - np.asarray(b)).max() / max(np.abs(np.asarray(b)).max(), 1e-300))


def run_coding(monkeypatch, tc, x, d, K, admm, theta=None, z=None, m=11):
    monkeypatch.setenv("DCSC_TC", "1" if tc else "0")
    N = x.shape[0]
    cfg = dcsc.SolverConfig(beta=0.5, rho=0.1, max_admm=admm, normalize=0)
    with dcsc.Context(N, x.shape[1:], K, (m, m), cfg, 32) as ctx:
        assert ctx.coding_path() == ("tensor" if tc else "fft")
        ctx.set_signals(x)
        ctx.set_dictionary(d)
        if theta is not None or z is not None:
            ctx.set_coding_state(theta, z)
        st = ctx.coding()
        th, zz, lam = ctx.get_coding_state()
    return st, th, zz, lam


@pytest.mark.parametrize("grid,K,m", [((256, 256), 128, 11), ((256, 256), 40, 11), ((128, 128), 64, 11),
                                      ((128, 128), 20, 11), ((100, 100), 100, 11), ((80, 80), 24, 11),
                                      ((64, 64), 32, 7), ((64, 64), 12, 7)])
def test_tc_pass_matches_fft_pass(monkeypatch, grid, K, m):
    """256 x 256: the cluster family (row-major u); 128 x 128, 100 x 100 and 80 x 80
    (one row per 128-lane tile, idle lanes past the row) and 64 x 64 (tiles of two
    rows, 7 x 7 supports padded to 64 taps): the single-CTA family, whose
    column-major pixel-pair u planes the pass converts around each coding call."""
    x, _ = dcsc.synth_generate(3, grid, K, m, 0.01, 0.01, 11, True)
    d = ref.init_dictionary(K, (m, m), grid, seed=5)
    a = run_coding(monkeypatch, True, x, d, K, 30, m=m)
    b = run_coding(monkeypatch, False, x, d, K, 30, m=m)
    assert [s["admm_iters"] for s in a[0]] == [s["admm_iters"] for s in b[0]]
    for key in ("primal_residual", "z_change", "theta_change", "dual_objective", "dual_infeasibility"):
        va = np.array([s[key] for s in a[0]])
        vb = np.array([s[key] for s in b[0]])
        assert np.abs(va - vb).max() <= TOL * max(np.abs(vb).max(), 1e-30), key
    assert rel(a[2], b[2]) <= TOL          # z
    assert rel(a[3], b[3]) <= TOL          # lambda
    # different arithmetic (spatial tensor-core GEMMs vs FFTs): not bit-identical
    assert not np.array_equal(a[2], b[2])


def test_tc_pass_full_filter_count_matches_reference(monkeypatch):
    """K = 128 (no padded filters, the C3 shape) against the reference's admm_coding."""
    K, admm = 128, 6
    x, _ = dcsc.synth_generate(1, (256, 256), K, 11, 0.01, 0.01, 17, True)
    d = ref.init_dictionary(K, (11, 11), (256, 256), seed=9)
    z_r, _, s_r = ref.solve_coding(x[0], d, ref.Cfg(beta=0.5, rho=0.1, max_admm=admm, normalize=0))
    st, th, z, lam = run_coding(monkeypatch, True, x, d, K, admm)
    assert st[0]["admm_iters"] == s_r["admm_iters"]
    for key in ("primal_residual", "z_change", "theta_change", "dual_objective"):
        assert abs(st[0][key] - s_r[key]) <= TOL * max(abs(s_r[key]), 1e-30), key
    assert rel(z[0], z_r) <= TOL


@pytest.mark.parametrize("kind", ["theta_outside_box", "theta_only"])
def test_tc_inconsistent_warm_state_matches_reference(monkeypatch, kind):
    """theta0 variant of the pass: theta itself is the first iteration's theta_old."""
    K, beta, rho = 6, 0.5, 0.1
    x, _ = dcsc.synth_generate(1, (256, 256), K, 11, 0.02, 0.01, 23, True)
    d = ref.init_dictionary(K, (11, 11), (256, 256), seed=4)
    rng = np.random.default_rng(8)
    if kind == "theta_outside_box":
        theta = rng.standard_normal((K, 256, 256)).astype(np.float32).astype(np.float64)
        z = (rng.standard_normal((K, 256, 256)) * 0.01).astype(np.float32).astype(np.float64)
    else:
        theta = rng.uniform(-beta, beta, (K, 256, 256)).astype(np.float32).astype(np.float64)
        z = np.zeros((K, 256, 256))
    for admm in (1, 8):
        z_r, (_, _, lam_r), s_r = ref.solve_coding(x[0], d, ref.Cfg(beta=beta, rho=rho, max_admm=admm, normalize=0),
                                                   (theta, z, np.zeros((256, 256))))
        st, _, z_g, lam_g = run_coding(monkeypatch, True, x, d, K, admm, theta[None], z[None])
        assert st[0]["admm_iters"] == s_r["admm_iters"]
        for key in ("theta_change", "z_change", "primal_residual"):
            assert abs(st[0][key] - s_r[key]) <= TOL * max(abs(s_r[key]), 1e-30), (admm, key)
        assert rel(z_g[0], z_r) <= TOL, admm
        assert rel(lam_g[0], lam_r) <= TOL, admm


def test_tc_pass_is_chosen_for_large_batches_only(monkeypatch):
    """Default (DCSC_TC unset): the tensor-core pass for batches of >= 2 work
    items per SM (C3: 512 images), the FFT pass for small ones; DCSC_TC=0 never."""
    monkeypatch.delenv("DCSC_TC", raising=False)
    cfg = dcsc.SolverConfig(max_admm=1, normalize=0)
    with dcsc.Context(512, (256, 256), 128, (11, 11), cfg, 32) as ctx:
        assert ctx.coding_path() == "tensor"
    with dcsc.Context(2, (256, 256), 128, (11, 11), cfg, 32) as ctx:
        assert ctx.coding_path() == "fft"
    with dcsc.Context(512, (128, 128), 64, (11, 11), cfg, 64) as ctx:  # FP64: FFT pass only
        assert ctx.coding_path() == "fft"
    monkeypatch.setenv("DCSC_TC", "0")
    with dcsc.Context(512, (256, 256), 128, (11, 11), cfg, 32) as ctx:
        assert ctx.coding_path() == "fft"
