// The C-ABI of the B200 dual-domain CSC path (include/dcsc_cuda.h): argument
// checks, error mapping (no exception crosses the boundary), grid dispatch to
// the per-grid engines (engine_impl.cuh, instantiated in inst_*.cu) and the
// multi-rank reducers (NCCL, dlopen'ed; or a host all-reduce callback).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "dcsc_cuda.h"
#include "engine_shared.h"

using namespace dcsc_engine;

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return DCSC_OK;
  } catch (const DimErr& e) {
    g_err = e.what();
    return DCSC_ERR_DIMENSION;
  } catch (const NumErr& e) {
    g_err = e.what();
    return DCSC_ERR_NUMERIC;
  } catch (const CudaErr& e) {
    g_err = e.what();
    return DCSC_ERR_CUDA;
  } catch (const std::exception& e) {
    g_err = e.what();
    return DCSC_ERR_INVALID;
  }
}

void validate_cfg(const dcsc_solver_config& c) {  // types.cpp:106-114
  if (!(c.beta > 0)) throw InvErr("beta must be > 0");
  if (!(c.rho > 0)) throw InvErr("rho must be > 0");
  if (!(c.tol > 0)) throw InvErr("tol must be > 0");
  if (!(c.mu_floor > 0)) throw InvErr("mu_floor must be > 0");
  if (c.max_outer < 0 || c.max_admm < 1 || c.max_mu_iters < 1 || c.cg_max < 1)
    throw InvErr("iteration caps must be positive");
  if (!(c.cg_tol > 0)) throw InvErr("cg_tol must be > 0");
}


struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  const char* (*getErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*groupStart)() = nullptr;
  ncclResult_t (*groupEnd)() = nullptr;
};

NcclApi& nccl_api() {
  static NcclApi api;
  if (!api.h) {
    api.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!api.h) throw CudaErr(std::string("NCCL: dlopen(libnccl.so.2) failed: ") + dlerror());
    api.getUniqueId = reinterpret_cast<decltype(api.getUniqueId)>(dlsym(api.h, "ncclGetUniqueId"));
    api.commInitRank = reinterpret_cast<decltype(api.commInitRank)>(dlsym(api.h, "ncclCommInitRank"));
    api.allReduce = reinterpret_cast<decltype(api.allReduce)>(dlsym(api.h, "ncclAllReduce"));
    api.commDestroy = reinterpret_cast<decltype(api.commDestroy)>(dlsym(api.h, "ncclCommDestroy"));
    api.getErrorString = reinterpret_cast<decltype(api.getErrorString)>(dlsym(api.h, "ncclGetErrorString"));
    api.send = reinterpret_cast<decltype(api.send)>(dlsym(api.h, "ncclSend"));
    api.recv = reinterpret_cast<decltype(api.recv)>(dlsym(api.h, "ncclRecv"));
    api.groupStart = reinterpret_cast<decltype(api.groupStart)>(dlsym(api.h, "ncclGroupStart"));
    api.groupEnd = reinterpret_cast<decltype(api.groupEnd)>(dlsym(api.h, "ncclGroupEnd"));
    if (!api.getUniqueId || !api.commInitRank || !api.allReduce || !api.commDestroy)
      throw CudaErr("NCCL: missing symbols in libnccl.so.2");
  }
  return api;
}

#define NCK(x)                                                                                        \
  do {                                                                                                \
    ncclResult_t r_ = (x);                                                                            \
    if (r_ != ncclSuccess)                                                                            \
      throw CudaErr(std::string("NCCL ") + #x + ": " +                                               \
                    (nccl_api().getErrorString ? nccl_api().getErrorString(r_) : std::to_string(r_))); \
  } while (0)

struct NcclReducer final : Reducer {
  ncclComm_t comm = nullptr;
  NcclReducer(int w, int r, const unsigned char* id, size_t len) {
    if (len < sizeof(ncclUniqueId)) throw InvErr("NCCL unique id too short");
    world = w;
    rank = r;
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    NCK(nccl_api().commInitRank(&comm, w, uid, r));
  }
  ~NcclReducer() override {
    if (comm) nccl_api().commDestroy(comm);
  }
  void allreduce(double* dev, size_t n, cudaStream_t st) override {
    NCK(nccl_api().allReduce(dev, dev, n, ncclDouble, ncclSum, comm, st));
  }
  // grouped point-to-point all-to-all (NCCL 2.27 has no ncclAllToAll)
  void alltoall(const void* send, const size_t* sbytes, void* recv, const size_t* rbytes,
                cudaStream_t st) override {
    NcclApi& api = nccl_api();
    if (!api.send || !api.recv || !api.groupStart || !api.groupEnd) throw CudaErr("NCCL: no ncclSend/ncclRecv");
    size_t so = 0, ro = 0;
    NCK(api.groupStart());
    for (int q = 0; q < world; ++q) {
      if (sbytes[q]) NCK(api.send(static_cast<const char*>(send) + so, sbytes[q], ncclInt8, q, comm, st));
      if (rbytes[q]) NCK(api.recv(static_cast<char*>(recv) + ro, rbytes[q], ncclInt8, q, comm, st));
      so += sbytes[q];
      ro += rbytes[q];
    }
    NCK(api.groupEnd());
  }
};

struct HostReducer final : Reducer {
  dcsc_allreduce_fn fn;
  void* user;
  std::vector<double> host;
  HostReducer(int w, int r, dcsc_allreduce_fn f, void* u) : fn(f), user(u) {
    world = w;
    rank = r;
  }
  void allreduce(double* dev, size_t n, cudaStream_t st) override {
    host.resize(n);
    CK(cudaMemcpyAsync(host.data(), dev, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (fn(host.data(), n, user) != 0) throw CudaErr("host all-reduce callback failed");
    CK(cudaMemcpyAsync(dev, host.data(), sizeof(double) * n, cudaMemcpyHostToDevice, st));
    CK(cudaStreamSynchronize(st));
  }
  // all-to-all through the sum callback (tests with ranks sharing one GPU):
  // the size matrix first, then per destination one zero-padded buffer of
  // every source's block, summed over ranks
  void alltoall(const void* send, const size_t* sbytes, void* recv, const size_t* rbytes,
                cudaStream_t st) override {
    std::vector<double> sz((size_t)world * world, 0.0);
    for (int q = 0; q < world; ++q) sz[(size_t)rank * world + q] = (double)sbytes[q];
    if (fn(sz.data(), sz.size(), user) != 0) throw CudaErr("host all-reduce callback failed");
    size_t so = 0;
    for (int q = 0; q < world; ++q) {
      size_t tot = 0, mine = 0;
      for (int r = 0; r < world; ++r) {
        if (r == rank) mine = tot;
        tot += (size_t)sz[(size_t)r * world + q];
      }
      std::vector<double> buf(tot / 8, 0.0);
      if (sbytes[q]) {
        CK(cudaMemcpyAsync(reinterpret_cast<char*>(buf.data()) + mine, static_cast<const char*>(send) + so,
                           sbytes[q], cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
      }
      if (fn(buf.data(), buf.size(), user) != 0) throw CudaErr("host all-reduce callback failed");
      if (q == rank) {
        size_t want = 0;
        for (int r = 0; r < world; ++r) want += rbytes[r];
        if (want != tot) throw CudaErr("all-to-all size mismatch");
        CK(cudaMemcpyAsync(recv, buf.data(), tot, cudaMemcpyHostToDevice, st));
        CK(cudaStreamSynchronize(st));
      }
      so += sbytes[q];
    }
  }
};
int prec_of(const char* t) { return std::strcmp(t, "double") == 0 ? 64 : 32; }

// ---- grid plugins: one engine instantiation unit per shared library (DCSC_GRID_PLUGIN in
// engine_impl.cuh, built by paper_1709_09479_b200/build.py build_grid) for grids outside
// DCSC_SIZES. Loaded explicitly (dcsc_cuda_load_grid) or found by name next to this
// library (<dir>/grids/libdcsc_grid_f{32,64}_{H}x{W}.so, or $DCSC_GRID_DIR).
struct GridPlugin {
  int prec, H, W;
  void* (*make)(const dcsc_cuda_opts*);
  void (*dft)(int, int, const double*, double*);
  void (*fft_timing)(int, int, double*, double*);
};
std::vector<GridPlugin>& plugins() {
  static std::vector<GridPlugin> v;
  return v;
}
std::mutex& plugin_mutex() {
  static std::mutex m;
  return m;
}
const GridPlugin* load_plugin(const std::string& path, bool must_exist) {
  void* h = dlopen(path.c_str(), RTLD_NOW | RTLD_LOCAL);
  if (!h) {
    if (must_exist) throw InvErr("cannot load grid plugin " + path + ": " + dlerror());
    return nullptr;
  }
  auto info = reinterpret_cast<void (*)(int*, int*, int*)>(dlsym(h, "dcsc_grid_info"));
  GridPlugin g{};
  g.make = reinterpret_cast<void* (*)(const dcsc_cuda_opts*)>(dlsym(h, "dcsc_grid_make"));
  g.dft = reinterpret_cast<void (*)(int, int, const double*, double*)>(dlsym(h, "dcsc_grid_dft"));
  g.fft_timing = reinterpret_cast<void (*)(int, int, double*, double*)>(dlsym(h, "dcsc_grid_fft_timing"));
  if (!info || !g.make || !g.dft || !g.fft_timing) {
    dlclose(h);
    throw InvErr(path + " is not a dcsc grid plugin");
  }
  info(&g.prec, &g.H, &g.W);
  for (const GridPlugin& q : plugins())
    if (q.prec == g.prec && q.H == g.H && q.W == g.W) return &q;  // already registered
  plugins().push_back(g);
  return &plugins().back();
}
std::string own_dir() {
  Dl_info di;
  if (!dladdr(reinterpret_cast<const void*>(&prec_of), &di) || !di.dli_fname) return ".";
  std::string p = di.dli_fname;
  const size_t k = p.rfind('/');
  return k == std::string::npos ? "." : p.substr(0, k);
}
const GridPlugin* find_plugin(int H, int W, int prec) {
  std::lock_guard<std::mutex> lk(plugin_mutex());
  for (const GridPlugin& q : plugins())
    if (q.prec == prec && q.H == H && q.W == W) return &q;
  const std::string name = "libdcsc_grid_f" + std::to_string(prec) + "_" + std::to_string(H) + "x" +
                           std::to_string(W) + ".so";
  if (const char* d = std::getenv("DCSC_GRID_DIR"))
    if (const GridPlugin* g = load_plugin(std::string(d) + "/" + name, false)) return g;
  return load_plugin(own_dir() + "/grids/" + name, false);
}

std::unique_ptr<EngineBase> make_engine(const dcsc_cuda_opts& o) {
#define DCSC_MAKE(Rt, Hh, Ww) \
  if (o.precision == prec_of(#Rt) && o.height == Hh && o.width == Ww) return make_engine_##Rt##_##Hh##_##Ww(o);
  DCSC_SIZES(DCSC_MAKE)
#undef DCSC_MAKE
  if (const GridPlugin* g = find_plugin(o.height, o.width, o.precision))
    return std::unique_ptr<EngineBase>(static_cast<EngineBase*>(g->make(&o)));
  throw DimErr("no compiled kernel family for grid " + std::to_string(o.height) + "x" + std::to_string(o.width) +
               " at FP" + std::to_string(o.precision) +
               " (build a grid plugin: python -m paper_1709_09479_b200.build --grid " + std::to_string(o.precision) +
               " " + std::to_string(o.height) + " " + std::to_string(o.width) + ")");
}

bool supported(int H, int W, int prec) {
#define DCSC_SUP(Rt, Hh, Ww) \
  if (prec == prec_of(#Rt) && H == Hh && W == Ww) return true;
  DCSC_SIZES(DCSC_SUP)
#undef DCSC_SUP
  return find_plugin(H, W, prec) != nullptr;
}

void fft_timing_dispatch(int H, int W, int prec, int batch, int iters, double* r2c, double* c2r) {
#define DCSC_FT(Rt, Hh, Ww)                                 \
  if (prec == prec_of(#Rt) && H == Hh && W == Ww) {        \
    fft_timing_##Rt##_##Hh##_##Ww(batch, iters, r2c, c2r); \
    return;                                                 \
  }
  DCSC_SIZES(DCSC_FT)
#undef DCSC_FT
  if (const GridPlugin* g = find_plugin(H, W, prec)) return g->fft_timing(batch, iters, r2c, c2r);
  throw DimErr("no compiled FFT for this grid/precision");
}

void dft_dispatch(int H, int W, int prec, bool inverse, int batch, const double* in, double* out) {
#define DCSC_DFT(Rt, Hh, Ww)                           \
  if (prec == prec_of(#Rt) && H == Hh && W == Ww) {    \
    dft_batch_##Rt##_##Hh##_##Ww(inverse, batch, in, out); \
    return;                                            \
  }
  DCSC_SIZES(DCSC_DFT)
#undef DCSC_DFT
  if (const GridPlugin* g = find_plugin(H, W, prec)) return g->dft(inverse ? 1 : 0, batch, in, out);
  throw DimErr("no compiled FFT for this grid/precision");
}

}  // namespace

struct dcsc_cuda_ctx {
  std::unique_ptr<EngineBase> eng;
};

#define CTX_CHECK                                         \
  if (!ctx || !ctx->eng) {                                \
    g_err = "null context";                               \
    return DCSC_ERR_INVALID;                              \
  }

extern "C" {

int dcsc_cuda_last_error(char* buf, size_t len) {
  if (buf && len) {
    std::strncpy(buf, g_err.c_str(), len - 1);
    buf[len - 1] = 0;
  }
  return (int)g_err.size();
}

int dcsc_cuda_supported_grid(int height, int width, int precision) {
  int ok = 0;
  guarded([&] { ok = supported(height, width, precision) ? 1 : 0; });
  return ok;
}

int dcsc_cuda_load_grid(const char* path) {
  return guarded([&] {
    if (!path) throw InvErr("null argument");
    std::lock_guard<std::mutex> lk(plugin_mutex());
    load_plugin(path, true);
  });
}

int dcsc_cuda_create(const dcsc_cuda_opts* opts, dcsc_cuda_ctx** out) {
  return guarded([&] {
    if (!opts || !out) throw InvErr("null argument");
    validate_cfg(opts->cfg);
    if (opts->n_images < 1) throw InvErr("dataset is empty");
    if (opts->filters < 1) throw InvErr("filter count must be >= 1");
    if (opts->support_h < 1 || opts->support_w < 1 || opts->support_h > opts->height ||
        opts->support_w > opts->width)
      throw DimErr("filter support must fit inside the grid");
    if (opts->precision != 32 && opts->precision != 64) throw InvErr("precision must be 32 or 64");
    if (opts->cfg.normalize < 0 || opts->cfg.normalize > 2) throw InvErr("normalize must be 0, 1 or 2");
    if (opts->channels < 0) throw InvErr("channel count must be >= 0");
    auto* c = new dcsc_cuda_ctx;
    try {
      c->eng = make_engine(*opts);
    } catch (...) {
      delete c;
      throw;
    }
    *out = c;
  });
}

int dcsc_cuda_destroy(dcsc_cuda_ctx* ctx) {
  return guarded([&] { delete ctx; });
}

int dcsc_cuda_synchronize(dcsc_cuda_ctx* ctx) {
  CTX_CHECK
  return guarded([&] { ctx->eng->synchronize(); });
}

int dcsc_cuda_set_signals(dcsc_cuda_ctx* ctx, const double* x) {
  CTX_CHECK
  return guarded([&] { ctx->eng->set_signals(x); });
}
int dcsc_cuda_get_signals(dcsc_cuda_ctx* ctx, double* x) {
  CTX_CHECK
  return guarded([&] { ctx->eng->get_signals(x); });
}
int dcsc_cuda_set_dictionary(dcsc_cuda_ctx* ctx, const double* d) {
  CTX_CHECK
  return guarded([&] { ctx->eng->set_dictionary(d); });
}
int dcsc_cuda_get_dictionary(dcsc_cuda_ctx* ctx, double* d) {
  CTX_CHECK
  return guarded([&] { ctx->eng->get_dictionary(d); });
}
int dcsc_cuda_init_variables(dcsc_cuda_ctx* ctx) {
  CTX_CHECK
  return guarded([&] { ctx->eng->init_variables(); });
}
int dcsc_cuda_set_coding_state(dcsc_cuda_ctx* ctx, int n0, int n1, const double* theta, const double* z) {
  CTX_CHECK
  return guarded([&] { ctx->eng->set_coding_state(n0, n1, theta, z); });
}
int dcsc_cuda_get_coding_state(dcsc_cuda_ctx* ctx, int n0, int n1, double* theta, double* z, double* lambda) {
  CTX_CHECK
  return guarded([&] { ctx->eng->get_coding_state(n0, n1, theta, z, lambda); });
}
int dcsc_cuda_coding(dcsc_cuda_ctx* ctx, int n0, int n1, dcsc_coding_stats* stats) {
  CTX_CHECK
  return guarded([&] { ctx->eng->coding(n0, n1, stats); });
}
int dcsc_cuda_set_maps(dcsc_cuda_ctx* ctx, int n0, int n1, const double* z) {
  CTX_CHECK
  return guarded([&] { ctx->eng->set_maps(n0, n1, z); });
}
int dcsc_cuda_get_maps(dcsc_cuda_ctx* ctx, int n0, int n1, double* z) {
  CTX_CHECK
  return guarded([&] { ctx->eng->get_maps(n0, n1, z); });
}
int dcsc_cuda_set_learning_state(dcsc_cuda_ctx* ctx, const double* gamma, const double* mu) {
  CTX_CHECK
  return guarded([&] { ctx->eng->set_learning_state(gamma, mu); });
}
int dcsc_cuda_get_learning_state(dcsc_cuda_ctx* ctx, double* gamma, double* mu) {
  CTX_CHECK
  return guarded([&] { ctx->eng->get_learning_state(gamma, mu); });
}
int dcsc_cuda_learning(dcsc_cuda_ctx* ctx, double* d_out, dcsc_learning_stats* stats) {
  CTX_CHECK
  return guarded([&] { ctx->eng->learning(d_out, stats); });
}
int dcsc_cuda_dictionary_adjoint(dcsc_cuda_ctx* ctx, int n0, int n1, const double* lambda, double* out) {
  return guarded([&] {
    if (!ctx || !lambda || !out) throw InvErr("null argument");
    ctx->eng->dictionary_adjoint(n0, n1, lambda, out);
  });
}

int dcsc_cuda_lambda_update(dcsc_cuda_ctx* ctx, int n0, int n1, const double* theta, const double* z, double* out) {
  return guarded([&] {
    if (!ctx || !theta || !z || !out) throw InvErr("null argument");
    ctx->eng->lambda_update_op(n0, n1, theta, z, out);
  });
}

int dcsc_cuda_gamma_solve(dcsc_cuda_ctx* ctx, int channel, const double* mu, double* gamma, int* iters,
                          int* converged) {
  return guarded([&] {
    if (!ctx || !mu || !gamma) throw InvErr("null argument");
    ctx->eng->gamma_solve_op(channel, mu, gamma, iters, converged);
  });
}

int dcsc_cuda_d_recover(dcsc_cuda_ctx* ctx, int channel, const double* gamma, const double* mu, double* out) {
  return guarded([&] {
    if (!ctx || !gamma || !mu || !out) throw InvErr("null argument");
    ctx->eng->d_recover_op(channel, gamma, mu, out);
  });
}

int dcsc_cuda_learning_correlation(dcsc_cuda_ctx* ctx, const double* v, double* out) {
  return guarded([&] {
    if (!ctx || !v || !out) throw InvErr("null argument");
    ctx->eng->learning_correlation(v, out);
  });
}

int dcsc_cuda_learning_apply(dcsc_cuda_ctx* ctx, const double* mu, const double* v, double* out) {
  CTX_CHECK
  return guarded([&] { ctx->eng->learning_apply(mu, v, out); });
}
int dcsc_cuda_objective(dcsc_cuda_ctx* ctx, const double* d, dcsc_objective* per_image) {
  CTX_CHECK
  return guarded([&] { ctx->eng->objective(d, per_image); });
}
int dcsc_cuda_learning_data_term(dcsc_cuda_ctx* ctx, const double* d, double* data) {
  CTX_CHECK
  return guarded([&] { ctx->eng->learning_data_term(d, data); });
}
int dcsc_cuda_reconstruct(dcsc_cuda_ctx* ctx, const double* d, int n0, int n1, double* out) {
  return guarded([&] {
    if (!ctx || !out) throw InvErr("null argument");
    ctx->eng->reconstruct(d, n0, n1, out);
  });
}

int dcsc_cuda_run(dcsc_cuda_ctx* ctx, int max_outer, dcsc_trace_row* rows, int* n_rows, int* converged) {
  CTX_CHECK
  return guarded([&] { ctx->eng->run(max_outer, rows, n_rows, converged); });
}
int dcsc_cuda_signal_flags(dcsc_cuda_ctx* ctx, int* degenerate) {
  CTX_CHECK
  return guarded([&] {
    if (!degenerate) throw InvErr("null argument");
    ctx->eng->signal_flags(degenerate);
  });
}
int dcsc_cuda_run_begin(dcsc_cuda_ctx* ctx) {
  CTX_CHECK
  return guarded([&] { ctx->eng->run_begin(); });
}
int dcsc_cuda_run_step(dcsc_cuda_ctx* ctx, dcsc_trace_row* rows, int* converged) {
  CTX_CHECK
  return guarded([&] {
    if (!rows) throw InvErr("null argument");
    const int c = ctx->eng->run_step(rows);
    if (converged) *converged = c;
  });
}
int dcsc_cuda_set_learning_layout(dcsc_cuda_ctx* ctx, int layout) {
  CTX_CHECK
  return guarded([&] {
    if (layout != 0 && layout != 1) throw InvErr("learning layout: 0 image-sharded, 1 frequency-sharded");
    ctx->eng->set_learning_layout(layout);
  });
}
int dcsc_cuda_run_accepts(dcsc_cuda_ctx* ctx, int* image_accept, int* dict_accept) {
  CTX_CHECK
  return guarded([&] { ctx->eng->run_accepts(image_accept, dict_accept); });
}
int dcsc_cuda_dft2_forward(int height, int width, int precision, int batch, const double* in, double* out) {
  return guarded([&] { dft_dispatch(height, width, precision, false, batch, in, out); });
}
int dcsc_cuda_dft2_inverse(int height, int width, int precision, int batch, const double* in, double* out) {
  return guarded([&] { dft_dispatch(height, width, precision, true, batch, in, out); });
}
int dcsc_cuda_fft_timing(int height, int width, int precision, int batch, int iters, double* ms_r2c,
                         double* ms_c2r) {
  return guarded([&] { fft_timing_dispatch(height, width, precision, batch, iters, ms_r2c, ms_c2r); });
}
int dcsc_cuda_kernel_launches(dcsc_cuda_ctx* ctx, long long* count) {
  CTX_CHECK
  *count = ctx->eng->launches;
  return DCSC_OK;
}
int dcsc_cuda_set_profiling(dcsc_cuda_ctx* ctx, int enable) {
  CTX_CHECK
  return guarded([&] { ctx->eng->set_profiling(enable); });
}
int dcsc_cuda_kernel_time(dcsc_cuda_ctx* ctx, int family, double* total_ms, long long* launches) {
  CTX_CHECK
  return guarded([&] { ctx->eng->kernel_time(family, total_ms, launches); });
}
int dcsc_cuda_event_mark(dcsc_cuda_ctx* ctx, int slot) {
  CTX_CHECK
  return guarded([&] { ctx->eng->event_mark(slot); });
}
int dcsc_cuda_event_elapsed(dcsc_cuda_ctx* ctx, int a, int b, double* ms) {
  CTX_CHECK
  return guarded([&] { *ms = ctx->eng->event_elapsed(a, b); });
}
int dcsc_cuda_nccl_unique_id(unsigned char* out, size_t len) {
  return guarded([&] {
    if (len < sizeof(ncclUniqueId)) throw InvErr("buffer shorter than ncclUniqueId");
    ncclUniqueId id;
    NCK(nccl_api().getUniqueId(&id));
    std::memcpy(out, &id, sizeof(id));
  });
}
int dcsc_cuda_set_comm_nccl(dcsc_cuda_ctx* ctx, int world, int rank, const unsigned char* id, size_t len) {
  CTX_CHECK
  return guarded([&] {
    if (world < 1 || rank < 0 || rank >= world) throw InvErr("bad world/rank");
    const char* f = std::getenv("DCSC_FORCE_MULTI");
    const bool force = f && f[0] == '1';
    if (world == 1 && !force) {
      ctx->eng->set_reducer(nullptr);
      return;
    }
    auto r = std::make_unique<NcclReducer>(world, rank, id, len);
    r->forced = world == 1;
    ctx->eng->set_reducer(std::move(r));
  });
}
int dcsc_cuda_set_comm_callback(dcsc_cuda_ctx* ctx, int world, int rank, dcsc_allreduce_fn fn, void* user) {
  CTX_CHECK
  return guarded([&] {
    if (world < 1 || rank < 0 || rank >= world || !fn) throw InvErr("bad world/rank/callback");
    ctx->eng->set_reducer(std::make_unique<HostReducer>(world, rank, fn, user));
  });
}
int dcsc_cuda_device_bytes(dcsc_cuda_ctx* ctx, size_t* bytes) {
  CTX_CHECK
  *bytes = ctx->eng->device_bytes;
  return DCSC_OK;
}

int dcsc_cuda_coding_path(dcsc_cuda_ctx* ctx, int* path) {
  CTX_CHECK
  *path = ctx->eng->coding_path;
  return DCSC_OK;
}

}  // extern "C"
