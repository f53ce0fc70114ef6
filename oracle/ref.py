"""ctypes binding of oracle/_ref/libdcsc_ref.so (TEST INFRASTRUCTURE ONLY).

The library is the UNMODIFIED reference solver (proj/src/{types,parallel,
spectral,objective,coding,learning,pipeline,tensor_io,trace_io,tcsc}.cpp) built
by oracle/Makefile against the FFTW3-API shim and (tcsc.cpp) the Eigen-API shim.
Multi-channel (J > 1) entry points take signals as (N, J, H, W), dictionaries
as (K, J, mh, mw) and run the reference's TCSC path (Joint channel mode). Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference leg may import this module; it is the checker,
never the thing measured as the product.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "libdcsc_ref.so")


class RefCfg(C.Structure):
    _fields_ = [
        ("beta", C.c_double), ("rho", C.c_double), ("tol", C.c_double),
        ("max_outer", C.c_int), ("max_admm", C.c_int), ("max_mu_iters", C.c_int),
        ("cg_tol", C.c_double), ("cg_max", C.c_int), ("mu_floor", C.c_double),
        ("seed", C.c_uint64), ("normalize", C.c_int),
    ]


class RefCodingStats(C.Structure):
    _fields_ = [
        ("admm_iters", C.c_int), ("converged", C.c_int), ("degenerate_dictionary", C.c_int),
        ("dual_rescaled", C.c_int), ("primal_residual", C.c_double), ("theta_change", C.c_double),
        ("z_change", C.c_double), ("dual_objective", C.c_double), ("dual_infeasibility", C.c_double),
    ]


class RefLearningStats(C.Structure):
    _fields_ = [
        ("mu_iters", C.c_int), ("cg_iters", C.c_long), ("cg_iters_first", C.c_long),
        ("converged", C.c_int), ("degenerate", C.c_int), ("mu_clamped", C.c_int),
        ("cg_budget_hit", C.c_int), ("rescaled_filters", C.c_int), ("n_dead", C.c_int),
    ]


class RefTraceRow(C.Structure):
    _fields_ = [
        ("outer_iter", C.c_int), ("phase", C.c_int), ("total", C.c_double),
        ("data_term", C.c_double), ("l1_term", C.c_double), ("residual_norm", C.c_double),
        ("admm_iters", C.c_long), ("cg_iters", C.c_long), ("mu_iters", C.c_int),
        ("elapsed_ms", C.c_double), ("wall_ms", C.c_double), ("l0", C.c_long),
    ]


@dataclass
class Cfg:
    """Mirror of dcsc::SolverConfig (proj/include/dcsc/types.hpp:96-110)."""
    beta: float = 0.5
    rho: float = 0.1
    tol: float = 1e-3
    max_outer: int = 50
    max_admm: int = 500
    max_mu_iters: int = 60
    cg_tol: float = 1e-6
    cg_max: int = 300
    mu_floor: float = 1e-6
    seed: int = 0
    normalize: int = 1  # 0 None, 1 Global, 2 Local

    def c(self) -> RefCfg:
        return RefCfg(self.beta, self.rho, self.tol, self.max_outer, self.max_admm,
                      self.max_mu_iters, self.cg_tol, self.cg_max, self.mu_floor,
                      self.seed, self.normalize)


_lib = None


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise RuntimeError(f"oracle reference library missing: {LIB_PATH} (run make -C oracle)")
        _lib = C.CDLL(LIB_PATH)
    return _lib


def _p(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _check(rc):
    if rc != 0:
        buf = C.create_string_buffer(1024)
        lib().ref_last_error(buf, 1024)
        raise RuntimeError(f"reference error {rc}: {buf.value.decode()}")


def set_threads(n: int) -> int:
    return lib().ref_set_threads(int(n))


def forward_dft(x: np.ndarray) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float64)
    dims = (C.c_int * x.ndim)(*x.shape)
    out = np.zeros(x.shape, dtype=np.complex128)
    _check(lib().ref_forward_dft(x.ndim, dims, _p(x), out.ctypes.data_as(C.POINTER(C.c_double))))
    return out


def inverse_dft(s: np.ndarray) -> np.ndarray:
    s = np.ascontiguousarray(s, dtype=np.complex128)
    dims = (C.c_int * s.ndim)(*s.shape)
    out = np.zeros(s.shape, dtype=np.float64)
    _check(lib().ref_inverse_dft(s.ndim, dims, s.ctypes.data_as(C.POINTER(C.c_double)), _p(out)))
    return out


def init_dictionary(K: int, m: tuple[int, int], grid: tuple[int, int], seed: int) -> np.ndarray:
    out = np.zeros((K, m[0], m[1]))
    _check(lib().ref_init_dictionary(K, m[0], m[1], grid[0], grid[1], C.c_uint64(seed), _p(out)))
    return out


def solve_coding(x, d, cfg: Cfg, state=None):
    """solve_coding (proj/src/coding.cpp:333-356). state = (theta, z, lambda) or None."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    d = np.ascontiguousarray(d, dtype=np.float64)
    H, W = x.shape
    K, mh, mw = d.shape
    if state is None:
        theta = np.zeros((K, H, W)); z = np.zeros((K, H, W)); lam = np.zeros((H, W)); warm = 0
    else:
        theta, z, lam = (np.array(a, dtype=np.float64, copy=True) for a in state); warm = 1
    st = RefCodingStats()
    c = cfg.c()
    _check(lib().ref_solve_coding(H, W, _p(x), K, mh, mw, _p(d), C.byref(c), warm,
                                  _p(theta), _p(z), _p(lam), C.byref(st)))
    stats = {f: getattr(st, f) for f, _ in RefCodingStats._fields_}
    return z.copy(), (theta, z, lam), stats


def solve_learning(xs, maps, support, cfg: Cfg, state=None):
    """solve_learning (proj/src/learning.cpp:227-355). state = (gamma N*D, mu K) or None."""
    xs = np.ascontiguousarray(xs, dtype=np.float64)
    maps = np.ascontiguousarray(maps, dtype=np.float64)
    N, H, W = xs.shape
    K = maps.shape[1]
    if state is None:
        gamma = np.zeros((N, H, W)); mu = np.ones(K); warm = 0
    else:
        gamma = np.array(state[0], dtype=np.float64, copy=True).reshape(N, H, W)
        mu = np.array(state[1], dtype=np.float64, copy=True); warm = 1
    d = np.zeros((K, support[0], support[1]))
    st = RefLearningStats()
    c = cfg.c()
    _check(lib().ref_solve_learning(N, H, W, _p(xs), K, _p(maps), support[0], support[1],
                                    C.byref(c), warm, _p(gamma), _p(mu), _p(d), C.byref(st)))
    stats = {f: getattr(st, f) for f, _ in RefLearningStats._fields_}
    return d, (gamma, mu), stats


def objective(x, d, z, beta):
    """evaluate_objective (proj/src/objective.cpp:59-81) -> (data, l1, total, residual_norm)."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    d = np.ascontiguousarray(d, dtype=np.float64)
    z = np.ascontiguousarray(z, dtype=np.float64)
    out = np.zeros(4)
    H, W = x.shape
    K, mh, mw = d.shape
    _check(lib().ref_objective(H, W, _p(x), K, mh, mw, _p(d), _p(z), C.c_double(beta), _p(out)))
    return tuple(out)


def learning_apply(maps, support, mu, mu_floor, v):
    """LearningOperator::apply (proj/src/learning.cpp:83-122)."""
    maps = np.ascontiguousarray(maps, dtype=np.float64)
    v = np.ascontiguousarray(v, dtype=np.float64)
    mu = np.ascontiguousarray(mu, dtype=np.float64)
    N, K, H, W = maps.shape
    out = np.zeros_like(v)
    _check(lib().ref_learning_apply(N, H, W, K, _p(maps), support[0], support[1], _p(mu),
                                    C.c_double(mu_floor), _p(v), _p(out)))
    return out


def run(xs, K, support, cfg: Cfg, dump_dicts=True, want_maps=True):
    """Instrumented run_csc replica (oracle/ref_capi.cpp:ref_run_ext). Besides the
    trace and the per-outer dictionaries it returns, per outer iteration, the
    near-tie counts of the accepted maps' soft-threshold argument (bands
    1e-7, 1e-6, 1e-5, 1e-4 relative to beta) and the acceptance flags (N image
    flags, then the dictionary flag)."""
    xs = np.ascontiguousarray(xs, dtype=np.float64)
    N, H, W = xs.shape
    mh, mw = support
    rows = (RefTraceRow * (2 * max(cfg.max_outer, 1)))()
    n_outer = C.c_int(0)
    dict_iter = np.zeros((cfg.max_outer + 1, K, mh, mw)) if dump_dicts else None
    maps = np.zeros((N, K, H, W)) if want_maps else None
    dfin = np.zeros((K, mh, mw))
    ties = np.zeros((max(cfg.max_outer, 1), 4), dtype=np.int64)
    acc = np.zeros((max(cfg.max_outer, 1), N + 1), dtype=np.int32)
    c = cfg.c()
    _check(lib().ref_run_ext(C.byref(c), N, H, W, _p(xs), K, mh, mw, rows, C.byref(n_outer),
                             _p(dict_iter) if dump_dicts else None, _p(maps) if want_maps else None, _p(dfin),
                             ties.ctypes.data_as(C.POINTER(C.c_long)), acc.ctypes.data_as(C.POINTER(C.c_int))))
    trace = [{f: getattr(rows[i], f) for f, _ in RefTraceRow._fields_} for i in range(2 * n_outer.value)]
    return {"trace": trace, "n_outer": n_outer.value,
            "dicts": dict_iter[: n_outer.value + 1] if dump_dicts else None,
            "maps": maps, "dict": dfin, "ties": ties[: n_outer.value], "accepts": acc[: n_outer.value]}


def set_parallel_objective(on: bool) -> None:
    """Golden generation only: the replica evaluates per-image objectives in
    parallel (identical values; the reference itself runs them serially)."""
    lib().ref_set_parallel_objective(int(on))


def synth_generate(n_images, grid, filters, m, p, sigma, seed, round_fp32, first=0):
    """The seeded BASELINE generator (paper_1709_09479_b200/csrc/synth.cpp, host
    only) compiled into this library, so the reference arm and the golden
    scripts never load the CUDA library. Same values as dcsc.synth_generate."""
    H, W = grid
    x = np.zeros((n_images, H, W))
    d = np.zeros((filters, m, m))
    rc = lib().dcsc_synth_generate_range(first, n_images, H, W, filters, m, C.c_double(p), C.c_double(sigma),
                                         C.c_uint64(seed), int(round_fp32), _p(x), _p(d))
    if rc != 0:
        raise ValueError("synth_generate: bad arguments")
    return x, d


def run_csc(xs, K, support, cfg: Cfg):
    """The reference's own run_csc (proj/src/pipeline.cpp:158-301)."""
    xs = np.ascontiguousarray(xs, dtype=np.float64)
    N, H, W = xs.shape
    mh, mw = support
    rows = (RefTraceRow * (2 * max(cfg.max_outer, 1)))()
    n_rows = C.c_int(0)
    dfin = np.zeros((K, mh, mw))
    maps = np.zeros((N, K, H, W))
    c = cfg.c()
    _check(lib().ref_run_csc(C.byref(c), N, H, W, _p(xs), K, mh, mw, rows, C.byref(n_rows),
                             _p(dfin), _p(maps)))
    trace = [{f: getattr(rows[i], f) for f, _ in RefTraceRow._fields_} for i in range(n_rows.value)]
    return {"trace": trace, "dict": dfin, "maps": maps}


def coding_batch(xs, d, cfg: Cfg, want_maps=False):
    """solve_coding over all images, OpenMP-parallel over images (pipeline.cpp:221-227)."""
    xs = np.ascontiguousarray(xs, dtype=np.float64)
    d = np.ascontiguousarray(d, dtype=np.float64)
    N, H, W = xs.shape
    K, mh, mw = d.shape
    iters = np.zeros(N, dtype=np.int32)
    maps = np.zeros((N, K, H, W)) if want_maps else None
    c = cfg.c()
    _check(lib().ref_coding_batch(N, H, W, _p(xs), K, mh, mw, _p(d), C.byref(c),
                                  _p(maps) if want_maps else None,
                                  iters.ctypes.data_as(C.POINTER(C.c_int))))
    return iters, maps


def write_tensor(path, values):
    """The reference's CSCT writer (tensor_io.cpp:45-60)."""
    v = np.ascontiguousarray(values, dtype=np.float64)
    dims = (C.c_uint64 * v.ndim)(*v.shape)
    _check(lib().ref_write_tensor(path.encode(), v.ndim, dims, _p(v)))


def read_tensor(path, shape):
    out = np.zeros(shape)
    _check(lib().ref_read_tensor(path.encode(), _p(out), C.c_uint64(out.size)))
    return out


def write_trace_csv(path, trace):
    """The reference's trace CSV writer (trace_io.cpp:15-30)."""
    rows = (RefTraceRow * max(len(trace), 1))()
    for i, t in enumerate(trace):
        for f, _ in RefTraceRow._fields_:
            setattr(rows[i], f, t.get(f, 0))
    _check(lib().ref_write_trace_csv(path.encode(), rows, len(trace)))


# ---------------------------------------------------------------- J channels
def init_dictionary_j(K: int, J: int, m: tuple[int, int], grid: tuple[int, int], seed: int) -> np.ndarray:
    out = np.zeros((K, J, m[0], m[1]))
    _check(lib().ref_init_dictionary_j(K, J, m[0], m[1], grid[0], grid[1], C.c_uint64(seed), _p(out)))
    return out


def solve_coding_tcsc(x, d, cfg: Cfg, state=None, method: int = 0):
    """solve_coding_tcsc (proj/src/tcsc.cpp:211-230). x (J,H,W), d (K,J,mh,mw);
    state = (theta K*D, z K*D, lambda J*D) or None. method 0 Auto, 1 Direct, 2 Woodbury."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    d = np.ascontiguousarray(d, dtype=np.float64)
    J, H, W = x.shape
    K, Jd, mh, mw = d.shape
    assert Jd == J
    if state is None:
        theta = np.zeros((K, H, W)); z = np.zeros((K, H, W)); lam = np.zeros((J, H, W)); warm = 0
    else:
        theta, z, lam = (np.array(a, dtype=np.float64, copy=True) for a in state); warm = 1
    st = RefCodingStats()
    c = cfg.c()
    _check(lib().ref_solve_coding_tcsc(H, W, J, _p(x), K, mh, mw, _p(d), C.byref(c), warm,
                                       _p(theta), _p(z), _p(lam), int(method), C.byref(st)))
    stats = {f: getattr(st, f) for f, _ in RefCodingStats._fields_}
    return z.copy(), (theta, z, lam), stats


def solve_learning_j(xs, maps, support, cfg: Cfg, state=None):
    """solve_learning / solve_learning_tcsc over J-channel images xs (N,J,H,W);
    state = (gamma (J,N,H,W), mu K) or None. Returns d (K,J,mh,mw)."""
    xs = np.ascontiguousarray(xs, dtype=np.float64)
    maps = np.ascontiguousarray(maps, dtype=np.float64)
    N, J, H, W = xs.shape
    K = maps.shape[1]
    if state is None:
        gamma = np.zeros((J, N, H, W)); mu = np.ones(K); warm = 0
    else:
        gamma = np.array(state[0], dtype=np.float64, copy=True).reshape(J, N, H, W)
        mu = np.array(state[1], dtype=np.float64, copy=True); warm = 1
    d = np.zeros((K, J, support[0], support[1]))
    st = RefLearningStats()
    c = cfg.c()
    _check(lib().ref_solve_learning_j(N, H, W, J, _p(xs), K, _p(maps), support[0], support[1],
                                      C.byref(c), warm, _p(gamma), _p(mu), _p(d), C.byref(st)))
    stats = {f: getattr(st, f) for f, _ in RefLearningStats._fields_}
    return d, (gamma, mu), stats


def objective_j(x, d, z, beta):
    """evaluate_objective of a J-channel image x (J,H,W) with d (K,J,mh,mw)."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    d = np.ascontiguousarray(d, dtype=np.float64)
    z = np.ascontiguousarray(z, dtype=np.float64)
    out = np.zeros(4)
    J, H, W = x.shape
    K, _, mh, mw = d.shape
    _check(lib().ref_objective_j(H, W, J, _p(x), K, mh, mw, _p(d), _p(z), C.c_double(beta), _p(out)))
    return tuple(out)


def run_j(xs, K, support, cfg: Cfg, dump_dicts=True):
    """Instrumented run_csc replica on J-channel signals xs (N,J,H,W), Joint mode for J > 1."""
    xs = np.ascontiguousarray(xs, dtype=np.float64)
    N, J, H, W = xs.shape
    mh, mw = support
    rows = (RefTraceRow * (2 * max(cfg.max_outer, 1)))()
    n_outer = C.c_int(0)
    dict_iter = np.zeros((cfg.max_outer + 1, K, J, mh, mw)) if dump_dicts else None
    maps = np.zeros((N, K, H, W))
    dfin = np.zeros((K, J, mh, mw))
    c = cfg.c()
    _check(lib().ref_run_j(C.byref(c), N, H, W, J, _p(xs), K, mh, mw, rows, C.byref(n_outer),
                           _p(dict_iter) if dump_dicts else None, _p(maps), _p(dfin), None, None))
    trace = [{f: getattr(rows[i], f) for f, _ in RefTraceRow._fields_} for i in range(2 * n_outer.value)]
    return {"trace": trace, "n_outer": n_outer.value,
            "dicts": dict_iter[: n_outer.value + 1] if dump_dicts else None,
            "maps": maps, "dict": dfin}


def run_csc_j(xs, K, support, cfg: Cfg):
    """The reference's own run_csc on J-channel signals (Joint mode for J > 1)."""
    xs = np.ascontiguousarray(xs, dtype=np.float64)
    N, J, H, W = xs.shape
    mh, mw = support
    rows = (RefTraceRow * (2 * max(cfg.max_outer, 1)))()
    n_rows = C.c_int(0)
    dfin = np.zeros((K, J, mh, mw))
    maps = np.zeros((N, K, H, W))
    c = cfg.c()
    _check(lib().ref_run_csc_j(C.byref(c), N, H, W, J, _p(xs), K, mh, mw, rows, C.byref(n_rows),
                               _p(dfin), _p(maps)))
    trace = [{f: getattr(rows[i], f) for f, _ in RefTraceRow._fields_} for i in range(n_rows.value)]
    return {"trace": trace, "dict": dfin, "maps": maps}


def coding_batch_j(xs, d, cfg: Cfg, want_maps=False):
    """solve_coding_tcsc over J-channel images xs (N,J,H,W), d (K,J,mh,mw), OpenMP over images."""
    xs = np.ascontiguousarray(xs, dtype=np.float64)
    d = np.ascontiguousarray(d, dtype=np.float64)
    N, J, H, W = xs.shape
    K, _, mh, mw = d.shape
    iters = np.zeros(N, dtype=np.int32)
    maps = np.zeros((N, K, H, W)) if want_maps else None
    c = cfg.c()
    _check(lib().ref_coding_batch_j(N, H, W, J, _p(xs), K, mh, mw, _p(d), C.byref(c),
                                    _p(maps) if want_maps else None,
                                    iters.ctypes.data_as(C.POINTER(C.c_int))))
    return iters, maps


def reconstruct(d, z):
    """reconstruct (objective.cpp:39-57): d (K,mh,mw) or (K,J,mh,mw), z (K,H,W)."""
    d = np.ascontiguousarray(d, dtype=np.float64)
    z = np.ascontiguousarray(z, dtype=np.float64)
    J = d.shape[1] if d.ndim == 4 else 1
    K, mh, mw = d.shape[0], d.shape[-2], d.shape[-1]
    _, H, W = z.shape
    out = np.zeros((J, H, W))
    _check(lib().ref_reconstruct_j(H, W, J, K, mh, mw, _p(d), _p(z), _p(out)))
    return out if d.ndim == 4 else out[0]


def learning_correlation(maps, support, v):
    """LearningOperator::correlation (learning.cpp:124-134) for every filter: (K, mh, mw)."""
    maps = np.ascontiguousarray(maps, dtype=np.float64)
    v = np.ascontiguousarray(v, dtype=np.float64)
    N, K, H, W = maps.shape
    out = np.zeros((K, support[0], support[1]))
    _check(lib().ref_learning_correlation(N, H, W, K, _p(maps), support[0], support[1], _p(v), _p(out)))
    return out


# ---------------------------------------------------------------- stateless ops (J = 1)
def lambda_update(x, d, theta, z, rho):
    """lambda_update (coding.cpp:103-124) for one image."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    d = np.ascontiguousarray(d, dtype=np.float64)
    H, W = x.shape
    K, mh, mw = d.shape
    out = np.zeros((H, W))
    _check(lib().ref_lambda_update(H, W, _p(x), K, mh, mw, _p(d), _p(np.ascontiguousarray(theta, dtype=np.float64)),
                                   _p(np.ascontiguousarray(z, dtype=np.float64)), C.c_double(rho), _p(out)))
    return out


def dictionary_adjoint(d, lam):
    """apply_dictionary_adjoint (coding.cpp:126-135): (K, H, W)."""
    d = np.ascontiguousarray(d, dtype=np.float64)
    lam = np.ascontiguousarray(lam, dtype=np.float64)
    K, mh, mw = d.shape
    H, W = lam.shape
    out = np.zeros((K, H, W))
    _check(lib().ref_dictionary_adjoint(H, W, K, mh, mw, _p(d), _p(lam), _p(out)))
    return out


def gamma_solve(maps, support, mu, mu_floor, x, cg_tol, cg_max, gamma):
    """gamma_solve (learning.cpp:136-185) on the stacked system; gamma is the warm start."""
    maps = np.ascontiguousarray(maps, dtype=np.float64)
    N, K, H, W = maps.shape
    g = np.array(gamma, dtype=np.float64, copy=True).reshape(N, H, W)
    it, conv = C.c_int(), C.c_int()
    _check(lib().ref_gamma_solve(N, H, W, K, _p(maps), support[0], support[1],
                                 _p(np.ascontiguousarray(mu, dtype=np.float64)), C.c_double(mu_floor),
                                 _p(np.ascontiguousarray(x, dtype=np.float64)), C.c_double(cg_tol), int(cg_max),
                                 _p(g), C.byref(it), C.byref(conv)))
    return g, it.value, bool(conv.value)


def d_recover(maps, support, gamma, mu):
    """d_recover (learning.cpp:187-216): (K, mh, mw)."""
    maps = np.ascontiguousarray(maps, dtype=np.float64)
    N, K, H, W = maps.shape
    out = np.zeros((K, support[0], support[1]))
    _check(lib().ref_d_recover(N, H, W, K, _p(maps), support[0], support[1],
                               _p(np.ascontiguousarray(gamma, dtype=np.float64)),
                               _p(np.ascontiguousarray(mu, dtype=np.float64)), _p(out)))
    return out


def time_learning(maps, support, n_apply=2):
    """Wall ms of the reference's LearningOperator build and of one apply (bench.py cpu baseline)."""
    maps = np.ascontiguousarray(maps, dtype=np.float64)
    N, K, H, W = maps.shape
    b, a = C.c_double(), C.c_double()
    _check(lib().ref_time_learning(N, H, W, K, _p(maps), support[0], support[1], int(n_apply), C.byref(b),
                                   C.byref(a)))
    return b.value, a.value
