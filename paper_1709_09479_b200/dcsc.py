"""Host-side mirror of the reference solver API over the C-ABI (include/dcsc_cuda.h).

Names, argument meaning and error behaviour follow the reference C++ API
(/root/reference/proj/include/dcsc/{coding,learning,pipeline,objective}.hpp):
  solve_coding(x, d, cfg, state)            coding.hpp:74-77
  solve_learning(xs, maps, support, cfg, state)  learning.hpp:99-104
  evaluate_objective(x, d, z, beta)         objective.hpp:14-15
  run_csc(xs, filters, support, cfg)        pipeline.hpp:58
Errors map to the reference exception classes (types.hpp:24-38).
The CUDA library is mandatory: there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

PKG = os.path.dirname(os.path.abspath(__file__))
# DCSC_LIB selects an experiment build (build.py tag=...); default: the in-tree library
LIB_PATH = os.environ.get("DCSC_LIB") or os.path.join(PKG, "lib", "libdcsc_cuda.so")


class IoError(RuntimeError):
    pass


class DimensionError(RuntimeError):
    pass


class NumericError(RuntimeError):
    pass


class CudaError(RuntimeError):
    pass


class InvalidArgument(ValueError):
    pass


_ERRS = {1: DimensionError, 2: NumericError, 3: CudaError, 4: InvalidArgument, 5: IoError}


class _SolverConfig(C.Structure):
    _fields_ = [
        ("beta", C.c_double), ("rho", C.c_double), ("tol", C.c_double),
        ("max_outer", C.c_int), ("max_admm", C.c_int), ("max_mu_iters", C.c_int),
        ("cg_tol", C.c_double), ("cg_max", C.c_int), ("mu_floor", C.c_double),
        ("seed", C.c_uint64), ("normalize", C.c_int),
    ]


class _Opts(C.Structure):
    _fields_ = [
        ("n_images", C.c_int), ("height", C.c_int), ("width", C.c_int), ("filters", C.c_int),
        ("support_h", C.c_int), ("support_w", C.c_int), ("precision", C.c_int), ("device", C.c_int),
        ("cfg", _SolverConfig), ("channels", C.c_int),
    ]


class CodingStats(C.Structure):
    _fields_ = [
        ("admm_iters", C.c_int), ("converged", C.c_int), ("degenerate_dictionary", C.c_int),
        ("dual_rescaled", C.c_int), ("primal_residual", C.c_double), ("theta_change", C.c_double),
        ("z_change", C.c_double), ("dual_objective", C.c_double), ("dual_infeasibility", C.c_double),
    ]

    def asdict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class LearningStats(C.Structure):
    _fields_ = [
        ("mu_iters", C.c_int), ("cg_iters", C.c_long), ("cg_iters_first", C.c_long),
        ("converged", C.c_int), ("degenerate", C.c_int), ("mu_clamped", C.c_int),
        ("cg_budget_hit", C.c_int), ("rescaled_filters", C.c_int), ("n_dead", C.c_int),
    ]

    def asdict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class Objective(C.Structure):
    _fields_ = [("data_term", C.c_double), ("l1_term", C.c_double), ("total", C.c_double),
                ("residual_norm", C.c_double)]


class TraceRow(C.Structure):
    _fields_ = [
        ("outer_iter", C.c_int), ("phase", C.c_int), ("total", C.c_double),
        ("data_term", C.c_double), ("l1_term", C.c_double), ("residual_norm", C.c_double),
        ("admm_iters", C.c_long), ("cg_iters", C.c_long), ("mu_iters", C.c_int),
        ("elapsed_ms", C.c_double), ("wall_ms", C.c_double), ("l0", C.c_long),
    ]

    def asdict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


@dataclass
class SolverConfig:
    """dcsc::SolverConfig (types.hpp:96-110); normalize 0 None / 1 Global / 2 Local."""
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
    normalize: int = 1

    def c(self) -> _SolverConfig:
        return _SolverConfig(self.beta, self.rho, self.tol, self.max_outer, self.max_admm,
                             self.max_mu_iters, self.cg_tol, self.cg_max, self.mu_floor,
                             self.seed, self.normalize)


_lib = None
EXPORTS = [
    "dcsc_cuda_last_error", "dcsc_cuda_supported_grid", "dcsc_cuda_load_grid", "dcsc_cuda_create", "dcsc_cuda_destroy",
    "dcsc_cuda_synchronize", "dcsc_cuda_set_signals", "dcsc_cuda_get_signals",
    "dcsc_cuda_set_dictionary", "dcsc_cuda_get_dictionary", "dcsc_cuda_init_variables",
    "dcsc_cuda_set_coding_state", "dcsc_cuda_get_coding_state", "dcsc_cuda_coding",
    "dcsc_cuda_set_maps", "dcsc_cuda_get_maps", "dcsc_cuda_set_learning_state",
    "dcsc_cuda_get_learning_state", "dcsc_cuda_learning", "dcsc_cuda_learning_apply",
    "dcsc_cuda_objective", "dcsc_cuda_learning_data_term", "dcsc_cuda_run",
    "dcsc_cuda_dft2_forward", "dcsc_cuda_dft2_inverse", "dcsc_cuda_kernel_launches",
    "dcsc_cuda_set_profiling", "dcsc_cuda_kernel_time", "dcsc_cuda_event_mark",
    "dcsc_cuda_event_elapsed", "dcsc_cuda_device_bytes", "dcsc_synth_generate",
    "dcsc_cuda_nccl_unique_id", "dcsc_cuda_set_comm_nccl", "dcsc_cuda_set_comm_callback",
    "dcsc_io_last_error", "dcsc_io_write_tensor", "dcsc_io_read_tensor_header", "dcsc_io_read_tensor",
    "dcsc_io_write_trace_csv", "dcsc_io_read_trace_csv", "dcsc_cuda_fft_timing", "dcsc_cuda_reconstruct",
    "dcsc_synth_dataset", "dcsc_synth_generate_range", "dcsc_cuda_learning_correlation",
    "dcsc_cuda_dictionary_adjoint", "dcsc_cuda_lambda_update", "dcsc_cuda_gamma_solve", "dcsc_cuda_d_recover",
    "dcsc_cuda_run_begin", "dcsc_cuda_run_step", "dcsc_cuda_run_accepts", "dcsc_cuda_signal_flags",
    "dcsc_cuda_set_learning_layout", "dcsc_cuda_coding_path",
]

ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, C.POINTER(C.c_double), C.c_size_t, C.c_void_p)


def shard_range(n_images: int, world: int, rank: int) -> tuple[int, int]:
    """Images [n0, n1) owned by `rank` (contiguous, sizes differ by at most one)."""
    base, extra = divmod(n_images, world)
    n0 = rank * base + min(rank, extra)
    return n0, n0 + base + (1 if rank < extra else 0)


def nccl_unique_id() -> bytes:
    buf = (C.c_ubyte * 128)()
    _err(lib().dcsc_cuda_nccl_unique_id(buf, 128))
    return bytes(buf)


def gloo_allreduce_fn(group=None):
    """Host all-reduce callback over torch.distributed (gloo): in-place sum."""
    import torch
    import torch.distributed as dist

    def fn(ptr, n, _user):
        try:
            arr = np.ctypeslib.as_array(ptr, shape=(n,))
            t = torch.from_numpy(arr)  # shares memory with the C buffer
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
            return 0
        except Exception:  # never raise through the C frame
            return 1

    return fn


def lib():
    """Load the in-tree CUDA library; raise if it is missing (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"CUDA extension missing: {LIB_PATH}; run __graft_entry__.build()")
        _lib = C.CDLL(LIB_PATH)
        _lib.dcsc_cuda_create.argtypes = [C.POINTER(_Opts), C.POINTER(C.c_void_p)]
        for name in EXPORTS:
            getattr(_lib, name).restype = C.c_int
    return _lib


def _err(rc: int):
    if rc == 0:
        return
    buf = C.create_string_buffer(2048)
    lib().dcsc_cuda_last_error(buf, 2048)
    raise _ERRS.get(rc, RuntimeError)(buf.value.decode())


def _dp(a: np.ndarray | None):
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def supported_grid(h: int, w: int, precision: int) -> bool:
    """True when a kernel family for this grid is compiled in or a grid plugin for it is found."""
    return bool(lib().dcsc_cuda_supported_grid(h, w, precision))


def build_grid(h: int, w: int, precision: int = 64) -> str:
    """Compile (once; needs nvcc) and register the engine plugin for a grid outside the built-in
    families: any even w with h and w/2 factoring into 2, 3 and 5 whose half-spectrum plane fits
    one CTA's shared memory. The reference plans any grid at run time (spectral.cpp:16-47)."""
    from . import build as _build
    path = _build.build_grid(precision, h, w)
    load_grid(path)
    return path


def load_grid(path: str):
    """Register a grid plugin library built elsewhere (dcsc_cuda_load_grid)."""
    _err(lib().dcsc_cuda_load_grid(path.encode()))


class Context:
    """Device-resident CSC state (the opaque dcsc_cuda_ctx)."""

    def __init__(self, n_images: int, grid: tuple[int, int], filters: int, support: tuple[int, int],
                 cfg: SolverConfig | None = None, precision: int = 64, device: int = 0, channels: int = 1):
        self.cfg = cfg or SolverConfig()
        self.N, (self.H, self.W), self.K = n_images, grid, filters
        self.J = max(1, int(channels))
        self.mh, self.mw = support
        self.D = self.H * self.W
        self.M = self.mh * self.mw
        self.precision = precision
        o = _Opts(n_images, grid[0], grid[1], filters, support[0], support[1], precision, device,
                  self.cfg.c(), self.J)
        h = C.c_void_p()
        _err(lib().dcsc_cuda_create(C.byref(o), C.byref(h)))
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            lib().dcsc_cuda_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # -- data
    def set_signals(self, xs):
        xs = _f64(xs)
        assert xs.size == self.N * self.J * self.D
        _err(lib().dcsc_cuda_set_signals(self._h, _dp(xs)))

    def _sig_shape(self, lead):
        return lead + ((self.J,) if self.J > 1 else ()) + (self.H, self.W)

    def signal_flags(self):
        """Per image: True when normalisation met a constant input (pipeline.cpp:177-183)."""
        out = np.zeros(self.N, dtype=np.int32)
        _err(lib().dcsc_cuda_signal_flags(self._h, out.ctypes.data_as(C.POINTER(C.c_int))))
        return out.astype(bool)

    def get_signals(self):
        out = np.zeros(self._sig_shape((self.N,)))
        _err(lib().dcsc_cuda_get_signals(self._h, _dp(out)))
        return out

    def set_dictionary(self, d):
        d = _f64(d)
        assert d.size == self.K * self.J * self.M
        _err(lib().dcsc_cuda_set_dictionary(self._h, _dp(d)))

    def _dict_shape(self):
        return (self.K,) + ((self.J,) if self.J > 1 else ()) + (self.mh, self.mw)

    def get_dictionary(self):
        out = np.zeros(self._dict_shape())
        _err(lib().dcsc_cuda_get_dictionary(self._h, _dp(out)))
        return out

    def init_variables(self):
        _err(lib().dcsc_cuda_init_variables(self._h))

    def set_coding_state(self, theta=None, z=None, n0=0, n1=None):
        n1 = self.N if n1 is None else n1
        th = None if theta is None else _f64(theta)
        zz = None if z is None else _f64(z)
        _err(lib().dcsc_cuda_set_coding_state(self._h, n0, n1, _dp(th), _dp(zz)))

    def get_coding_state(self, n0=0, n1=None):
        n1 = self.N if n1 is None else n1
        cnt = n1 - n0
        th = np.zeros((cnt, self.K, self.H, self.W))
        z = np.zeros_like(th)
        lam = np.zeros(self._sig_shape((cnt,)))
        _err(lib().dcsc_cuda_get_coding_state(self._h, n0, n1, _dp(th), _dp(z), _dp(lam)))
        return th, z, lam

    def coding(self, n0=0, n1=None):
        n1 = self.N if n1 is None else n1
        st = (CodingStats * (n1 - n0))()
        _err(lib().dcsc_cuda_coding(self._h, n0, n1, st))
        return [s.asdict() for s in st]

    def set_maps(self, z, n0=0, n1=None):
        n1 = self.N if n1 is None else n1
        _err(lib().dcsc_cuda_set_maps(self._h, n0, n1, _dp(_f64(z))))

    def get_maps(self, n0=0, n1=None):
        n1 = self.N if n1 is None else n1
        out = np.zeros((n1 - n0, self.K, self.H, self.W))
        _err(lib().dcsc_cuda_get_maps(self._h, n0, n1, _dp(out)))
        return out

    def set_learning_state(self, gamma=None, mu=None):
        g = None if gamma is None else _f64(gamma)
        m = None if mu is None else _f64(mu)
        _err(lib().dcsc_cuda_set_learning_state(self._h, _dp(g), _dp(m)))

    def get_learning_state(self):
        g = np.zeros(((self.J,) if self.J > 1 else ()) + (self.N, self.H, self.W))
        m = np.zeros(self.K)
        _err(lib().dcsc_cuda_get_learning_state(self._h, _dp(g), _dp(m)))
        return g, m

    def learning(self):
        d = np.zeros(self._dict_shape())
        st = LearningStats()
        _err(lib().dcsc_cuda_learning(self._h, _dp(d), C.byref(st)))
        return d, st.asdict()

    def learning_apply(self, mu, v):
        mu = _f64(mu)
        v = _f64(v)
        out = np.zeros_like(v)
        _err(lib().dcsc_cuda_learning_apply(self._h, _dp(mu), _dp(v), _dp(out)))
        return out

    # -- stateless ops (coding.hpp:45-66, learning.hpp:81-95)
    def dictionary_adjoint(self, lam, n0=0, n1=None):
        """D^T lambda (apply_dictionary_adjoint): lam (n, [J,] H, W) -> (n, K, H, W)."""
        n1 = self.N if n1 is None else n1
        lam = _f64(lam)
        out = np.zeros((n1 - n0, self.K, self.H, self.W))
        _err(lib().dcsc_cuda_dictionary_adjoint(self._h, n0, n1, _dp(lam), _dp(out)))
        return out

    def lambda_update(self, theta, z, n0=0, n1=None):
        """lambda_update (coding.cpp:103-124): theta, z (n, K, H, W) -> lambda (n, [J,] H, W)."""
        n1 = self.N if n1 is None else n1
        out = np.zeros(self._sig_shape((n1 - n0,)))
        _err(lib().dcsc_cuda_lambda_update(self._h, n0, n1, _dp(_f64(theta)), _dp(_f64(z)), _dp(out)))
        return out

    def gamma_solve(self, mu, gamma, channel=0):
        """gamma_solve (learning.cpp:136-185): returns (gamma, iters, converged)."""
        g = np.array(gamma, dtype=np.float64, copy=True).reshape(self.N, self.H, self.W)
        it, conv = C.c_int(), C.c_int()
        _err(lib().dcsc_cuda_gamma_solve(self._h, channel, _dp(_f64(mu)), _dp(g), C.byref(it), C.byref(conv)))
        return g, it.value, bool(conv.value)

    def d_recover(self, gamma, mu, channel=0):
        """d_recover (learning.cpp:187-216): (K, mh, mw) for one channel's gamma."""
        out = np.zeros((self.K, self.mh, self.mw))
        _err(lib().dcsc_cuda_d_recover(self._h, channel, _dp(_f64(gamma)), _dp(_f64(mu)), _dp(out)))
        return out

    def learning_correlation(self, v):
        """LearningOperator::correlation (learning.cpp:124-134) for all filters: (K, mh, mw)."""
        v = _f64(v)
        out = np.zeros((self.K, self.mh, self.mw))
        _err(lib().dcsc_cuda_learning_correlation(self._h, _dp(v), _dp(out)))
        return out

    def objective(self, d=None):
        out = (Objective * self.N)()
        dd = None if d is None else _f64(d)
        _err(lib().dcsc_cuda_objective(self._h, _dp(dd), out))
        return [(o.data_term, o.l1_term, o.total, o.residual_norm) for o in out]

    def learning_data_term(self, d=None):
        v = C.c_double()
        dd = None if d is None else _f64(d)
        _err(lib().dcsc_cuda_learning_data_term(self._h, _dp(dd), C.byref(v)))
        return v.value

    def reconstruct(self, d=None, n0=0, n1=None):
        """dcsc::reconstruct (objective.cpp:39-57) of the accepted maps of images [n0, n1)."""
        n1 = self.N if n1 is None else n1
        out = np.zeros(self._sig_shape((n1 - n0,)))
        dd = None if d is None else _f64(d)
        _err(lib().dcsc_cuda_reconstruct(self._h, _dp(dd), n0, n1, _dp(out)))
        return out

    def run(self, max_outer: int):
        rows = (TraceRow * (2 * max(max_outer, 1)))()
        n = C.c_int()
        conv = C.c_int()
        _err(lib().dcsc_cuda_run(self._h, max_outer, rows, C.byref(n), C.byref(conv)))
        return [rows[i].asdict() for i in range(n.value)], bool(conv.value)

    def run_begin(self):
        """run_csc's set-up (pipeline.cpp:169-213): init_variables + initial objectives."""
        _err(lib().dcsc_cuda_run_begin(self._h))

    def run_step(self):
        """The next run_csc outer iteration (pipeline.cpp:216-299): (coding row, learning row), converged."""
        rows = (TraceRow * 2)()
        conv = C.c_int()
        _err(lib().dcsc_cuda_run_step(self._h, rows, C.byref(conv)))
        return [rows[0].asdict(), rows[1].asdict()], bool(conv.value)

    def run_accepts(self):
        """Acceptance flags of the last run_step: (per-image array, dictionary flag)."""
        img = np.zeros(self.N, dtype=np.int32)
        dacc = C.c_int()
        _err(lib().dcsc_cuda_run_accepts(self._h, img.ctypes.data_as(C.POINTER(C.c_int)), C.byref(dacc)))
        return img, bool(dacc.value)

    # -- multi-rank
    def set_comm_nccl(self, world: int, rank: int, uid: bytes):
        buf = (C.c_ubyte * len(uid)).from_buffer_copy(uid)
        _err(lib().dcsc_cuda_set_comm_nccl(self._h, world, rank, buf, len(uid)))

    def set_comm_callback(self, world: int, rank: int, fn):
        self._cb = ALLREDUCE_FN(fn)  # keep the trampoline alive
        _err(lib().dcsc_cuda_set_comm_callback(self._h, world, rank, self._cb, None))

    # -- measurement
    def set_learning_layout(self, layout: str):
        """'image' (default) or 'freq': frequency-sharded learning across ranks (after set_comm_*)."""
        _err(lib().dcsc_cuda_set_learning_layout(self._h, {"image": 0, "freq": 1}[layout]))

    def synchronize(self):
        _err(lib().dcsc_cuda_synchronize(self._h))

    def kernel_launches(self) -> int:
        v = C.c_longlong()
        _err(lib().dcsc_cuda_kernel_launches(self._h, C.byref(v)))
        return v.value

    def set_profiling(self, on: int):
        """0 off, 1 every launch, 2 coding-pass launches only."""
        _err(lib().dcsc_cuda_set_profiling(self._h, int(on)))

    def kernel_time(self, family: int):
        ms = C.c_double()
        n = C.c_longlong()
        _err(lib().dcsc_cuda_kernel_time(self._h, family, C.byref(ms), C.byref(n)))
        return ms.value, n.value

    def event_mark(self, slot: int):
        _err(lib().dcsc_cuda_event_mark(self._h, slot))

    def event_elapsed(self, a: int, b: int) -> float:
        v = C.c_double()
        _err(lib().dcsc_cuda_event_elapsed(self._h, a, b, C.byref(v)))
        return v.value

    def device_bytes(self) -> int:
        v = C.c_size_t()
        _err(lib().dcsc_cuda_device_bytes(self._h, C.byref(v)))
        return v.value

    def coding_path(self) -> str:
        """'fft' (fused FFT coding pass) or 'tensor' (tcgen05 spatial pass)."""
        v = C.c_int()
        _err(lib().dcsc_cuda_coding_path(self._h, C.byref(v)))
        return "tensor" if v.value == 1 else "fft"


# ---------------------------------------------------------------- reference-shaped API
@dataclass
class CodingDualState:
    """dcsc::CodingDualState (coding.hpp:15-25): lambda D, theta K*D, z K*D."""
    theta: np.ndarray | None = None
    z: np.ndarray | None = None
    lam: np.ndarray | None = None

    def initialized(self) -> bool:
        return self.z is not None


@dataclass
class LearningDualState:
    """dcsc::LearningDualState (learning.hpp:15-23)."""
    gamma: np.ndarray | None = None
    mu: np.ndarray | None = None
    mu_iters_total: int = 0
    cg_iters_total: int = 0


def solve_coding(x, d, cfg: SolverConfig, state: CodingDualState | None = None, precision: int = 64):
    """solve_coding (coding.cpp:333-356) for one image; returns (maps, state, stats)."""
    x = _f64(x)
    d = _f64(d)
    if x.ndim != 2:
        raise DimensionError("solve_coding expects a single-channel 2-D signal; use solve_coding_tcsc")
    K, mh, mw = d.shape
    H, W = x.shape
    if mh > H or mw > W:
        raise DimensionError("filter support larger than the signal grid")
    c = SolverConfig(**{**cfg.__dict__, "normalize": 0})
    with Context(1, (H, W), K, (mh, mw), c, precision) as ctx:
        ctx.set_signals(x[None])
        ctx.set_dictionary(d)
        state = state or CodingDualState()
        if state.initialized():
            ctx.set_coding_state(state.theta[None], state.z[None])
        stats = ctx.coding()[0]
        th, z, lam = ctx.get_coding_state()
    return z[0].copy(), CodingDualState(th[0], z[0], lam[0]), stats


def solve_coding_tcsc(x, d, cfg: SolverConfig, state: CodingDualState | None = None, precision: int = 64):
    """solve_coding_tcsc (tcsc.cpp:211-230) for one J-channel image x (J,H,W)
    with d (K,J,mh,mw); returns (maps, state, stats). lambda is (J,H,W)."""
    x = _f64(x)
    d = _f64(d)
    if x.ndim != 3 or d.ndim != 4 or d.shape[1] != x.shape[0]:
        raise DimensionError("solve_coding_tcsc: signal and dictionary channel counts differ")
    J, H, W = x.shape
    K, _, mh, mw = d.shape
    if mh > H or mw > W:
        raise DimensionError("filter support larger than the signal grid")
    c = SolverConfig(**{**cfg.__dict__, "normalize": 0})
    with Context(1, (H, W), K, (mh, mw), c, precision, channels=J) as ctx:
        ctx.set_signals(x[None])
        ctx.set_dictionary(d)
        state = state or CodingDualState()
        if state.initialized():
            ctx.set_coding_state(state.theta[None], state.z[None])
        stats = ctx.coding()[0]
        th, z, lam = ctx.get_coding_state()
    lam = lam[0].reshape(J, H, W)
    return z[0].copy(), CodingDualState(th[0], z[0], lam), stats


def solve_learning(xs, maps, support, cfg: SolverConfig, state: LearningDualState | None = None,
                   precision: int = 64):
    """solve_learning (learning.cpp:227-355); returns (dictionary, state, stats)."""
    xs = _f64(xs)
    maps = _f64(maps)
    J = xs.shape[1] if xs.ndim == 4 else 1
    N, H, W = xs.shape[0], xs.shape[-2], xs.shape[-1]
    K = maps.shape[1]
    c = SolverConfig(**{**cfg.__dict__, "normalize": 0})
    with Context(N, (H, W), K, tuple(support), c, precision, channels=J) as ctx:
        ctx.set_signals(xs)
        ctx.set_maps(maps)
        state = state or LearningDualState()
        ctx.set_learning_state(state.gamma, state.mu)
        d, stats = ctx.learning()
        g, mu = ctx.get_learning_state()
    st = LearningDualState(g, mu, state.mu_iters_total + stats["mu_iters"],
                           state.cg_iters_total + stats["cg_iters"])
    return d, st, stats


def evaluate_objective(x, d, z, beta, precision: int = 64):
    """evaluate_objective (objective.cpp:59-81) -> (data, l1, total, residual_norm).
    J-channel: x (J,H,W), d (K,J,mh,mw)."""
    x = _f64(x)
    d = _f64(d)
    J = x.shape[0] if x.ndim == 3 else 1
    K, mh, mw = d.shape[0], d.shape[-2], d.shape[-1]
    H, W = x.shape[-2], x.shape[-1]
    with Context(1, (H, W), K, (mh, mw), SolverConfig(beta=beta, normalize=0), precision, channels=J) as ctx:
        ctx.set_signals(x[None])
        ctx.set_maps(_f64(z)[None])
        return ctx.objective(d)[0]


def reconstruct(d, z, precision: int = 64):
    """reconstruct (objective.cpp:39-57): one image from maps z (K,H,W) and a
    dictionary d (K,mh,mw) or (K,J,mh,mw); returns (H,W) or (J,H,W)."""
    d = _f64(d)
    z = _f64(z)
    J = d.shape[1] if d.ndim == 4 else 1
    K, mh, mw = d.shape[0], d.shape[-2], d.shape[-1]
    if z.shape[0] != K:
        raise DimensionError("dictionary and maps disagree on the filter count")
    H, W = z.shape[-2], z.shape[-1]
    with Context(1, (H, W), K, (mh, mw), SolverConfig(normalize=0), precision, channels=J) as ctx:
        ctx.set_maps(z[None])
        return ctx.reconstruct(d)[0]


def encode(x, d, cfg: SolverConfig, precision: int = 64):
    """The reference CLI's `encode` (csc_main.cpp:147-172) on the GPU: normalise
    x per cfg.normalize, code it (TCSC when d has J > 1 channels), evaluate the
    objective. Returns (maps, objective (data, l1, total, residual), stats)."""
    x = _f64(x)
    d = _f64(d)
    J = d.shape[1] if d.ndim == 4 else 1
    K, mh, mw = d.shape[0], d.shape[-2], d.shape[-1]
    H, W = x.shape[-2], x.shape[-1]
    with Context(1, (H, W), K, (mh, mw), cfg, precision, channels=J) as ctx:
        ctx.set_signals(x[None])
        ctx.set_dictionary(d)
        stats = ctx.coding()[0]
        _, z, _ = ctx.get_coding_state()
        ctx.set_maps(z)
        obj = ctx.objective()[0]
    return z[0], obj, stats


def run_csc(xs, filters: int, support, cfg: SolverConfig, precision: int = 64, names=None):
    """run_csc (pipeline.cpp:158-301): returns dict(trace, dict, maps, converged, warnings).
    xs (N,H,W) or (N,J,H,W); J > 1 is the Joint channel mode (TCSC). `warnings`
    follows RunResult::warnings (pipeline.cpp:177-183) for constant inputs."""
    xs = _f64(xs)
    J = xs.shape[1] if xs.ndim == 4 else 1
    N, H, W = xs.shape[0], xs.shape[-2], xs.shape[-1]
    with Context(N, (H, W), filters, tuple(support), cfg, precision, channels=J) as ctx:
        ctx.set_signals(xs)
        flags = ctx.signal_flags()
        warnings = [f"normalize: constant input '{names[n] if names is not None and n < len(names) else n}' "
                    "mapped to zeros" for n in range(N) if flags[n]]
        trace, conv = ctx.run(cfg.max_outer)
        return {"trace": trace, "dict": ctx.get_dictionary(), "maps": ctx.get_maps(),
                "converged": conv, "warnings": warnings}


def forward_dft2(x, precision: int = 64):
    """Half-spectrum forward DFT of a batch of real planes (spectral.cpp:59-74)."""
    x = _f64(x)
    B, H, W = x.shape
    out = np.zeros((B, H, W // 2 + 1), dtype=np.complex128)
    _err(lib().dcsc_cuda_dft2_forward(H, W, precision, B, _dp(x), out.ctypes.data_as(C.POINTER(C.c_double))))
    return out


def inverse_dft2(s, width: int, precision: int = 64):
    """Inverse of forward_dft2 (1/D scaled, real output; spectral.cpp:76-104)."""
    s = np.ascontiguousarray(s, dtype=np.complex128)
    B, H, Wh = s.shape
    out = np.zeros((B, H, width))
    _err(lib().dcsc_cuda_dft2_inverse(H, width, precision, B, s.ctypes.data_as(C.POINTER(C.c_double)), _dp(out)))
    return out


def fft_timing(grid, precision: int, batch: int, iters: int = 20):
    """Device-timed batched r2c / c2r of our FFT engine (ms per batch call)."""
    a, b = C.c_double(), C.c_double()
    _err(lib().dcsc_cuda_fft_timing(grid[0], grid[1], precision, batch, iters, C.byref(a), C.byref(b)))
    return a.value, b.value


def synth_generate(n_images, grid, filters, m, p, sigma, seed, round_fp32, first=0):
    """Synthetic BASELINE data; host-only, no GPU needed.
    Images [first, first + n_images) of the seeded dataset."""
    H, W = grid
    x = np.zeros((n_images, H, W))
    d = np.zeros((filters, m, m))
    _err(lib().dcsc_synth_generate_range(first, n_images, H, W, filters, m, C.c_double(p), C.c_double(sigma),
                                         C.c_uint64(seed), int(round_fp32), _dp(x), _dp(d)))
    return x, d


# ---------------------------------------------------------------- on-disk formats
def synth_dataset(n_images: int, channels: int, grid, seed: int) -> np.ndarray:
    """synthetic_dataset (bench.cpp:9-21): (N, H, W) or (N, J, H, W) uniform [0, 1)."""
    out = np.zeros((n_images, channels, grid[0], grid[1]))
    _err(lib().dcsc_synth_dataset(n_images, channels, grid[0], grid[1], C.c_uint64(seed), _dp(out)))
    return out if channels > 1 else out[:, 0]


def _io(rc: int):
    if rc == 0:
        return
    buf = C.create_string_buffer(2048)
    lib().dcsc_io_last_error(buf, 2048)
    raise IoError(buf.value.decode())


def write_tensor(path: str, values) -> None:
    """CSCT tensor writer (tensor_io.cpp:45-60): dims = values.shape."""
    v = _f64(values)
    dims = (C.c_uint64 * v.ndim)(*v.shape)
    _io(lib().dcsc_io_write_tensor(path.encode(), v.ndim, dims, _dp(v)))


def read_tensor(path: str) -> np.ndarray:
    """CSCT tensor reader (tensor_io.cpp:62-90)."""
    nd = C.c_int()
    dims = (C.c_uint64 * 255)()
    cnt = C.c_uint64()
    _io(lib().dcsc_io_read_tensor_header(path.encode(), C.byref(nd), dims, C.byref(cnt)))
    out = np.zeros(tuple(dims[i] for i in range(nd.value)))
    _io(lib().dcsc_io_read_tensor(path.encode(), _dp(out), cnt))
    return out


def write_trace_csv(path: str, trace) -> None:
    """Trace CSV writer (trace_io.cpp:15-30); trace = list of row dicts."""
    rows = (TraceRow * max(len(trace), 1))()
    for i, r in enumerate(trace):
        for f, _ in TraceRow._fields_:
            setattr(rows[i], f, r.get(f, 0))
    _io(lib().dcsc_io_write_trace_csv(path.encode(), rows, len(trace)))


def read_trace_csv(path: str, max_rows: int = 100000):
    """Trace CSV reader (trace_io.cpp:32-76)."""
    rows = (TraceRow * max_rows)()
    n = C.c_int()
    _io(lib().dcsc_io_read_trace_csv(path.encode(), rows, max_rows, C.byref(n)))
    return [rows[i].asdict() for i in range(n.value)]
