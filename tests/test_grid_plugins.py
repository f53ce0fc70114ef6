"""Grid plugins (build.build_grid / dcsc_cuda_load_grid): the reference plans any grid at
run time (spectral.cpp:16-47); here a grid outside the built-in families is one more
engine instantiation compiled into its own library and found by the dispatcher.

CPU part: argument checks, the cross-compile of one small plugin, and that the main
library finds it by name (no compute). GPU part: rectangular FP64 40 x 60 and FP32 96 x 96
(radix plans 8x5 / 10x3 and 16x6 / 16x3 from the greedy factorisation) against the oracle:
DFT, coding, run_csc; the 96 x 96 grid also on the tensor-core pass."""
import ctypes as C
import os

import numpy as np
import pytest

from paper_1709_09479_b200 import build


def test_build_grid_rejects_unsupported_grids():
    with pytest.raises(ValueError):
        build.build_grid(64, 28, 28)    # 28 = 4 x 7
    with pytest.raises(ValueError):
        build.build_grid(64, 30, 45)    # odd width
    with pytest.raises(ValueError):
        build.build_grid(32, 200, 200)  # plane exceeds one CTA's shared memory
    with pytest.raises(ValueError):
        build.build_grid(16, 32, 32)


def test_plugin_builds_and_is_found_by_name():
    path = build.build_grid(64, 24, 24)
    assert os.path.exists(path)
    lib = C.CDLL(os.path.join(os.path.dirname(build.LIB), "libdcsc_cuda.so"))
    assert lib.dcsc_cuda_supported_grid(24, 24, 64) == 1     # found in lib/grids by name
    assert lib.dcsc_cuda_supported_grid(24, 24, 32) == 0     # no FP32 plugin for it
    assert lib.dcsc_cuda_supported_grid(28, 28, 64) == 0
    assert lib.dcsc_cuda_load_grid(path.encode()) == 0       # explicit registration: idempotent
    assert lib.dcsc_cuda_load_grid(b"/nonexistent/libdcsc_grid.so") != 0
    plug = C.CDLL(path)
    p, h, w = C.c_int(), C.c_int(), C.c_int()
    plug.dcsc_grid_info(C.byref(p), C.byref(h), C.byref(w))
    assert (p.value, h.value, w.value) == (64, 24, 24)


# ---------------------------------------------------------------- GPU
def rel(a, b):
    return float(np.abs(np.asarray(a) - np.asarray(b)).max() / max(np.abs(b).max(), 1e-300))


@pytest.fixture(scope="module")
def plugins():
    from paper_1709_09479_b200 import dcsc
    dcsc.build_grid(40, 60, 64)
    dcsc.build_grid(96, 96, 32)
    return dcsc


@pytest.mark.gpu
@pytest.mark.parametrize("H,W,prec", [(40, 60, 64), (96, 96, 32)])
def test_plugin_dft_matches_reference(plugins, H, W, prec):
    from oracle import ref
    dcsc = plugins
    assert dcsc.supported_grid(H, W, prec)
    rng = np.random.default_rng(H + W)
    x = rng.standard_normal((3, H, W))
    if prec == 32:
        x = x.astype(np.float32).astype(np.float64)
    g = dcsc.forward_dft2(x, prec)
    r = np.stack([ref.forward_dft(xi) for xi in x])[..., : W // 2 + 1]
    tol = 1e-13 if prec == 64 else 2e-6
    assert rel(g.view(np.float64), r.view(np.float64)) <= tol
    assert rel(dcsc.inverse_dft2(g, W, prec), x) <= tol


@pytest.mark.gpu
def test_plugin_rectangular_fp64_coding_and_run_match_reference(plugins):
    from oracle import ref
    dcsc = plugins
    H, W, K, m = 40, 60, 5, 5
    x, _ = dcsc.synth_generate(3, (H, W), K, m, 0.02, 0.01, 3, False)
    d = ref.init_dictionary(K, (m, m), (H, W), seed=4)
    cfg = dict(beta=0.3, max_admm=80, normalize=0)
    z_r, st_r, s_r = ref.solve_coding(x[0], d, ref.Cfg(**cfg))
    z_g, st_g, s_g = dcsc.solve_coding(x[0], d, dcsc.SolverConfig(**cfg), precision=64)
    assert s_g["admm_iters"] == s_r["admm_iters"]
    assert rel(z_g, z_r) <= 1e-9 and rel(st_g.lam, st_r[2]) <= 1e-9
    kw = dict(beta=0.3, max_outer=3, normalize=0, seed=5, tol=1e-300, max_admm=80)
    r = ref.run(x, K, (m, m), ref.Cfg(**kw))
    g = dcsc.run_csc(x, K, (m, m), dcsc.SolverConfig(**kw), precision=64)
    for a, b in zip(g["trace"], r["trace"]):
        for key in ("total", "data_term", "l1_term"):
            assert abs(a[key] - b[key]) <= 1e-9 * abs(b[key])
        assert a["admm_iters"] == b["admm_iters"] and a["mu_iters"] == b["mu_iters"]
    assert rel(g["dict"], r["dict"]) <= 1e-8
    # the reference's error behaviour holds on a plugin grid too (types.hpp:24-38)
    with pytest.raises(dcsc.DimensionError):
        dcsc.run_csc(x, K, (H + 1, 3), dcsc.SolverConfig(**kw), precision=64)


@pytest.mark.gpu
@pytest.mark.parametrize("tc", [False, True])
def test_plugin_fp32_96_coding_matches_reference(plugins, monkeypatch, tc):
    """96 x 96 FP32: the FFT pass, and the tensor-core pass on a single-row family the
    built-in set does not have (96 live lanes of each 128-lane tile)."""
    from oracle import ref
    dcsc = plugins
    monkeypatch.setenv("DCSC_TC", "1" if tc else "0")
    K, m = 24, 11
    x, _ = dcsc.synth_generate(2, (96, 96), K, m, 0.01, 0.01, 7, True)
    d = ref.init_dictionary(K, (m, m), (96, 96), seed=5)
    cfg = dcsc.SolverConfig(beta=0.5, rho=0.1, max_admm=30, normalize=0)
    with dcsc.Context(2, (96, 96), K, (m, m), cfg, 32) as ctx:
        assert ctx.coding_path() == ("tensor" if tc else "fft")
        ctx.set_signals(x)
        ctx.set_dictionary(d)
        st = ctx.coding()
        _, z, lam = ctx.get_coding_state()
    for n in range(2):
        z_r, st_r, s_r = ref.solve_coding(x[n], d, ref.Cfg(beta=0.5, rho=0.1, max_admm=30, normalize=0))
        assert st[n]["admm_iters"] == s_r["admm_iters"]
        assert abs(st[n]["dual_objective"] - s_r["dual_objective"]) <= 1e-4 * abs(s_r["dual_objective"])
        assert rel(z[n], z_r) <= 1e-4 and rel(lam[n], st_r[2]) <= 1e-4
