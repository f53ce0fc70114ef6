// Types shared by the C-ABI translation unit (engine.cu) and the per-grid
// engine instantiation units (inst_*.cu): error types, the multi-rank reducer
// interface, the engine interface and the compiled grid/precision table.
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <memory>
#include <stdexcept>
#include <string>

#include "dcsc_cuda.h"

namespace dcsc_engine {

struct DimErr : std::runtime_error { using std::runtime_error::runtime_error; };
struct NumErr : std::runtime_error { using std::runtime_error::runtime_error; };
struct CudaErr : std::runtime_error { using std::runtime_error::runtime_error; };
struct InvErr : std::runtime_error { using std::runtime_error::runtime_error; };

#define CK(x)                                                                                  \
  do {                                                                                         \
    cudaError_t e_ = (x);                                                                      \
    if (e_ != cudaSuccess) throw CudaErr(std::string(#x) + ": " + cudaGetErrorString(e_));     \
  } while (0)

// Learning is image-sharded like coding by default (no z_hat all-to-all): the
// K x M cropped correlations (each rank crops its own partial), the CG scalars
// and the trace sums are all-reduced. The frequency-sharded layout
// (set_learning_layout(1)) moves z_hat and x_hat to frequency-major blocks by
// one all-to-all per outer iteration and keeps the crop all-reduce.
// NCCL is dlopen'ed (libnccl.so.2) so a process that already loaded torch's
// NCCL shares it; the host-callback reducer lets ranks that share one GPU be
// tested with host-side (gloo) reductions.
struct Reducer {
  int world = 1, rank = 0;
  // DCSC_FORCE_MULTI=1 (tests): a 1-rank communicator still takes the
  // multi-rank code paths, so the NCCL reducer runs end to end on one GPU
  bool forced = false;
  virtual ~Reducer() = default;
  virtual void allreduce(double* dev, size_t n, cudaStream_t st) = 0;  // in-place sum
  // all-to-all of device byte blocks: `send` holds `world` consecutive blocks
  // (block q -> rank q, sbytes[q]); `recv` gets `world` consecutive blocks
  // (from rank q, rbytes[q]). Sizes are multiples of 8 bytes.
  virtual void alltoall(const void* send, const size_t* sbytes, void* recv, const size_t* rbytes,
                        cudaStream_t st) = 0;
};

// ---------------------------------------------------------------- interface
class EngineBase {
 public:
  virtual ~EngineBase() = default;
  virtual void set_signals(const double* x) = 0;
  virtual void get_signals(double* x) = 0;
  virtual void signal_flags(int* degenerate) = 0;
  virtual void set_dictionary(const double* d) = 0;
  virtual void get_dictionary(double* d) = 0;
  virtual void init_variables() = 0;
  virtual void set_coding_state(int n0, int n1, const double* theta, const double* z) = 0;
  virtual void get_coding_state(int n0, int n1, double* theta, double* z, double* lambda) = 0;
  virtual void coding(int n0, int n1, dcsc_coding_stats* stats) = 0;
  virtual void set_maps(int n0, int n1, const double* z) = 0;
  virtual void get_maps(int n0, int n1, double* z) = 0;
  virtual void set_learning_state(const double* gamma, const double* mu) = 0;
  virtual void get_learning_state(double* gamma, double* mu) = 0;
  virtual void learning(double* d_out, dcsc_learning_stats* st) = 0;
  virtual void learning_apply(const double* mu, const double* v, double* out) = 0;
  virtual void objective(const double* d, dcsc_objective* per_image) = 0;
  virtual void learning_data_term(const double* d, double* data) = 0;
  virtual void reconstruct(const double* d, int n0, int n1, double* out) = 0;
  virtual void learning_correlation(const double* v, double* out) = 0;
  virtual void dictionary_adjoint(int n0, int n1, const double* lam, double* out) = 0;
  virtual void lambda_update_op(int n0, int n1, const double* theta, const double* z, double* out) = 0;
  virtual void gamma_solve_op(int channel, const double* mu, double* gamma, int* iters, int* converged) = 0;
  virtual void d_recover_op(int channel, const double* gamma, const double* mu, double* out) = 0;
  virtual void run(int max_outer, dcsc_trace_row* rows, int* n_rows, int* converged) = 0;
  virtual void run_begin() = 0;
  virtual int run_step(dcsc_trace_row* rows) = 0;
  virtual void run_accepts(int* image_accept, int* dict_accept) = 0;
  virtual void set_learning_layout(int freq) = 0;
  virtual void synchronize() = 0;
  virtual void set_profiling(int on) = 0;
  virtual void kernel_time(int fam, double* ms, long long* n) = 0;
  virtual void event_mark(int slot) = 0;
  virtual double event_elapsed(int a, int b) = 0;
  void set_reducer(std::unique_ptr<Reducer> r) { red_ = std::move(r); }
  bool multi() const { return red_ && (red_->world > 1 || red_->forced); }
  long long launches = 0;
 protected:
  std::unique_ptr<Reducer> red_;
 public:
  size_t device_bytes = 0;
  int coding_path = 0;  // ADMM coding iteration: 0 FFT pass (kernels*.cuh), 1 tensor-core spatial pass (kernels_tc.cuh)
};

// ---------------------------------------------------------------- size table
// Adding a grid: one X(...) line here, a DCSC_ENGINE_INSTANTIATE in an
// inst_*.cu unit, and PlanFor<H>, PlanFor<W/2> radix plans (fft2d.cuh) built
// from radices 2, 3, 4, 5, 6, 8, 10, 16.
#define DCSC_SIZES(X) \
  X(double, 16, 16)   \
  X(double, 16, 20)   \
  X(double, 20, 20)   \
  X(double, 32, 32)   \
  X(double, 48, 48)   \
  X(double, 64, 64)   \
  X(double, 100, 100) \
  X(double, 128, 128) \
  X(float, 16, 16)    \
  X(float, 16, 20)    \
  X(float, 20, 20)    \
  X(float, 32, 32)    \
  X(float, 48, 48)    \
  X(float, 64, 64)    \
  X(float, 80, 80)    \
  X(float, 100, 100)  \
  X(float, 128, 128)  \
  X(float, 256, 256)
// per-grid entry points, defined by DCSC_ENGINE_INSTANTIATE in inst_*.cu
#define DCSC_DECL(Rt, Hh, Ww)                                                                  \
  std::unique_ptr<EngineBase> make_engine_##Rt##_##Hh##_##Ww(const dcsc_cuda_opts& o);          \
  void dft_batch_##Rt##_##Hh##_##Ww(bool inverse, int batch, const double* in, double* out);    \
  void fft_timing_##Rt##_##Hh##_##Ww(int batch, int iters, double* ms_r2c, double* ms_c2r);
DCSC_SIZES(DCSC_DECL)
#undef DCSC_DECL

}  // namespace dcsc_engine
