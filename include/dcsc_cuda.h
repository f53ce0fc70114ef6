/* dcsc_cuda.h — C-ABI of the B200 (sm_100a) dual-domain CSC hot path.
 *
 * Drop-in boundary for the reference's solver API (arXiv 1709.09479
 * reference, /root/reference/proj). No exceptions or torch types cross it:
 * every entry returns a status code; dcsc_cuda_last_error() gives the message.
 * Plain host pointers and sizes only; all hot-path state stays device-resident
 * between calls inside the opaque context.
 *
 * Entry point -> reference interface it replaces:
 *   dcsc_cuda_create / _destroy     dcsc::SolverConfig + RunConfig
 *                                   (include/dcsc/types.hpp:96-110,
 *                                    include/dcsc/pipeline.hpp:19-26)
 *   dcsc_cuda_set_signals           Dataset signals + dcsc::normalize
 *                                   (pipeline.hpp:13-16, 32; pipeline.cpp:78-121)
 *   dcsc_cuda_set_dictionary/get    dcsc::Dictionary (types.hpp:62-78)
 *   dcsc_cuda_init_dictionary       dcsc::init_variables (pipeline.hpp:44-45;
 *                                   pipeline.cpp:123-156)
 *   dcsc_cuda_set/get_coding_state  dcsc::CodingDualState (coding.hpp:15-25)
 *   dcsc_cuda_coding                dcsc::solve_coding (coding.hpp:74-77),
 *                                   batched over images: replaces the OpenMP
 *                                   loop at pipeline.cpp:221-227; with
 *                                   channels > 1 dcsc::solve_coding_tcsc
 *                                   (tcsc.hpp:53-60, pipeline.cpp:222-224)
 *   dcsc_cuda_set/get_maps          dcsc::SparseMaps (types.hpp:81-94)
 *   dcsc_cuda_set/get_learning_state dcsc::LearningDualState (learning.hpp:15-23)
 *   dcsc_cuda_learning              dcsc::solve_learning (learning.hpp:99-104);
 *                                   channels > 1: solve_learning_tcsc (tcsc.hpp:62-68)
 *   dcsc_cuda_objective             dcsc::evaluate_objective (objective.hpp:14-15)
 *   dcsc_cuda_learning_data_term    dcsc::learning_data_term (objective.hpp:18-19)
 *   dcsc_cuda_reconstruct           dcsc::reconstruct (objective.hpp:11)
 *   dcsc_cuda_learning_apply        dcsc::LearningOperator::apply (learning.hpp:57)
 *   dcsc_cuda_learning_correlation  dcsc::LearningOperator::correlation (learning.hpp:59-60)
 *   dcsc_cuda_run                   dcsc::run_csc (pipeline.hpp:58) + trace rows
 *                                   (types.hpp:122-136, trace_io.hpp)
 *   dcsc_cuda_run_begin / _step     the same run_csc outer loop
 *                                   (pipeline.cpp:216-299), one iteration per call
 *   dcsc_cuda_dft2_forward/_inverse dcsc::forward_dft / inverse_dft
 *                                   (spectral.hpp:27-38), half-spectrum form
 */
#ifndef DCSC_CUDA_H
#define DCSC_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes (mirroring the reference's exception classes, types.hpp:24-38) */
#define DCSC_OK 0
#define DCSC_ERR_DIMENSION 1 /* dcsc::DimensionError */
#define DCSC_ERR_NUMERIC 2   /* dcsc::NumericError */
#define DCSC_ERR_CUDA 3      /* CUDA / NCCL failure */
#define DCSC_ERR_INVALID 4   /* std::invalid_argument from validate() */
#define DCSC_ERR_IO 5        /* dcsc::IoError */

typedef struct dcsc_cuda_ctx dcsc_cuda_ctx;

/* dcsc::SolverConfig (types.hpp:96-110); normalize: 0 None, 1 Global, 2 Local */
typedef struct {
  double beta, rho, tol;
  int max_outer, max_admm, max_mu_iters;
  double cg_tol;
  int cg_max;
  double mu_floor;
  uint64_t seed;
  int normalize;
} dcsc_solver_config;

typedef struct {
  int n_images;            /* N */
  int height, width;       /* grid H x W (row-major, last axis fastest) */
  int filters;             /* K */
  int support_h, support_w;
  int precision;           /* 32 or 64: storage/FFT precision; reductions are FP64 */
  int device;              /* CUDA device ordinal */
  dcsc_solver_config cfg;
  int channels;            /* J (0 or 1 = single channel). J > 1 runs the
                              reference's Joint channel mode: TCSC coding
                              (tcsc.hpp: per-bin J x J block solves) and
                              per-channel learning (solve_learning_tcsc) */
} dcsc_cuda_opts;

/* dcsc::CodingStats (coding.hpp:27-37) */
typedef struct {
  int admm_iters, converged, degenerate_dictionary, dual_rescaled;
  double primal_residual, theta_change, z_change, dual_objective, dual_infeasibility;
} dcsc_coding_stats;

/* dcsc::LearningStats (learning.hpp:25-35); dead filters reported by count */
typedef struct {
  int mu_iters;
  long cg_iters, cg_iters_first;
  int converged, degenerate, mu_clamped, cg_budget_hit, rescaled_filters, n_dead;
} dcsc_learning_stats;

/* dcsc::ObjectiveBreakdown (types.hpp:112-117) */
typedef struct {
  double data_term, l1_term, total, residual_norm;
} dcsc_objective;

/* dcsc::TraceRow (types.hpp:122-129) + mu_iters, wall time, l0 of the maps */
typedef struct {
  int outer_iter, phase; /* phase 0 coding, 1 learning */
  double total, data_term, l1_term, residual_norm;
  long admm_iters, cg_iters;
  int mu_iters;
  double elapsed_ms; /* solver call only (the reference's timer) */
  double wall_ms;    /* whole half-step incl. objective bookkeeping */
  long l0;           /* non-zero entries of the accepted maps */
} dcsc_trace_row;

int dcsc_cuda_last_error(char* buf, size_t len);
/* 1 when a kernel family for this grid / precision is compiled in */
int dcsc_cuda_supported_grid(int height, int width, int precision);
/* The reference plans any grid at run time (spectral.cpp:16-47, DftPlan). Here every grid is a
 * compiled kernel family: the built-in ones (DCSC_SIZES), plus grid plugins - one shared library
 * per (precision, H, W), any even W with H and W/2 factoring into 2, 3, 5 and a half-spectrum
 * plane that fits shared memory - built by `python -m paper_1709_09479_b200.build --grid P H W`.
 * A plugin named libdcsc_grid_f<P>_<H>x<W>.so in <library dir>/grids or $DCSC_GRID_DIR is found by
 * dcsc_cuda_create on its own; dcsc_cuda_load_grid registers one from any path. */
int dcsc_cuda_load_grid(const char* path);

int dcsc_cuda_create(const dcsc_cuda_opts* opts, dcsc_cuda_ctx** out);
int dcsc_cuda_destroy(dcsc_cuda_ctx* ctx);
int dcsc_cuda_synchronize(dcsc_cuda_ctx* ctx);

/* signals x: N*J*H*W doubles (image-major, then channel); normalised per
 * cfg.normalize (pipeline.cpp:78-121) */
int dcsc_cuda_set_signals(dcsc_cuda_ctx* ctx, const double* x);
int dcsc_cuda_get_signals(dcsc_cuda_ctx* ctx, double* x);
/* per image (N ints): 1 when the last set_signals' normalisation met a constant
 * input (dcsc::normalize's degenerate flag, pipeline.cpp:84-121; run_csc turns
 * it into RunResult::warnings, pipeline.cpp:177-183) */
int dcsc_cuda_signal_flags(dcsc_cuda_ctx* ctx, int* degenerate);
/* dictionary: K*J*mh*mw doubles (filter-major, Dictionary::filter(k, j)) */
int dcsc_cuda_set_dictionary(dcsc_cuda_ctx* ctx, const double* d);
int dcsc_cuda_get_dictionary(dcsc_cuda_ctx* ctx, double* d);
/* init_variables: seeded dictionary, zero maps / coding state, gamma = 0, mu = 1 */
int dcsc_cuda_init_variables(dcsc_cuda_ctx* ctx);

/* warm coding state for images [n0, n1): theta, z (K*D each per image), NULL = zeros;
 * get also returns lambda (J*D per image) */
int dcsc_cuda_set_coding_state(dcsc_cuda_ctx* ctx, int n0, int n1, const double* theta,
                               const double* z);
int dcsc_cuda_get_coding_state(dcsc_cuda_ctx* ctx, int n0, int n1, double* theta, double* z,
                               double* lambda);
/* solve_coding for images [n0, n1) against the context dictionary */
int dcsc_cuda_coding(dcsc_cuda_ctx* ctx, int n0, int n1, dcsc_coding_stats* stats);

/* accepted maps used by learning / objective: K*D per image */
int dcsc_cuda_set_maps(dcsc_cuda_ctx* ctx, int n0, int n1, const double* z);
int dcsc_cuda_get_maps(dcsc_cuda_ctx* ctx, int n0, int n1, double* z);

/* learning warm state: gamma J*N*D (channel-major; NULL = zeros), mu K (NULL = ones) */
int dcsc_cuda_set_learning_state(dcsc_cuda_ctx* ctx, const double* gamma, const double* mu);
int dcsc_cuda_get_learning_state(dcsc_cuda_ctx* ctx, double* gamma, double* mu);
/* solve_learning over all images' maps; writes the candidate dictionary
 * (K*mh*mw) to d_out without installing it */
int dcsc_cuda_learning(dcsc_cuda_ctx* ctx, double* d_out, dcsc_learning_stats* stats);
/* reconstruct (objective.cpp:39-57) of the accepted maps of images [n0, n1)
 * with dictionary d (K*J*M; NULL = the context dictionary): out (n1-n0)*J*D.
 * GPU side of the reference CLI's `reconstruct` / `encode` (csc_main.cpp:147-202) */
int dcsc_cuda_reconstruct(dcsc_cuda_ctx* ctx, const double* d, int n0, int n1, double* out);
/* Stateless ops (coding.hpp:45-66, learning.hpp:81-95, tcsc.hpp:38-51), for
 * replaying iterations; they leave the context's coding / learning state as is.
 * apply_dictionary_adjoint / block_dictionary_adjoint: lambda (n1-n0)*J*D ->
 * D^T lambda (n1-n0)*K*D against the context dictionary */
int dcsc_cuda_dictionary_adjoint(dcsc_cuda_ctx* ctx, int n0, int n1, const double* lambda, double* out);
/* lambda_update / lambda_update_blocked: theta, z (n1-n0)*K*D -> lambda (n1-n0)*J*D
 * against the context's signals and dictionary */
int dcsc_cuda_lambda_update(dcsc_cuda_ctx* ctx, int n0, int n1, const double* theta, const double* z,
                            double* out);
/* gamma_solve on one channel with the given mu (K): gamma N*D warm start in /
 * solution out over the accepted maps */
int dcsc_cuda_gamma_solve(dcsc_cuda_ctx* ctx, int channel, const double* mu, double* gamma, int* iters,
                          int* converged);
/* d_recover: gamma N*D (one channel), mu K -> K*mh*mw */
int dcsc_cuda_d_recover(dcsc_cuda_ctx* ctx, int channel, const double* gamma, const double* mu, double* out);
/* LearningOperator::correlation (learning.cpp:124-134) for every filter k:
 * sum_n S_k Z_nk^T v_n over the accepted maps, v N*D (this rank's images; summed
 * over ranks), out K*mh*mw */
int dcsc_cuda_learning_correlation(dcsc_cuda_ctx* ctx, const double* v, double* out);
/* LearningOperator::apply with the given mu on N*D vectors */
int dcsc_cuda_learning_apply(dcsc_cuda_ctx* ctx, const double* mu, const double* v, double* out);

/* evaluate_objective(x_n, d, maps_n) for every image; d NULL = context dictionary */
int dcsc_cuda_objective(dcsc_cuda_ctx* ctx, const double* d, dcsc_objective* per_image);
/* learning_data_term(xs, d, maps) */
int dcsc_cuda_learning_data_term(dcsc_cuda_ctx* ctx, const double* d, double* data);

/* run_csc from init_variables: rows needs 2*max_outer entries */
int dcsc_cuda_run(dcsc_cuda_ctx* ctx, int max_outer, dcsc_trace_row* rows, int* n_rows,
                  int* converged);

/* run_csc one outer iteration at a time (the same arithmetic as
 * dcsc_cuda_run): run_begin = init_variables + the initial objectives
 * (pipeline.cpp:169-213); each run_step is the next outer iteration
 * (pipeline.cpp:216-299), rows needs 2 entries (coding, learning);
 * *converged = 1 when the run's stop test (pipeline.cpp:290-298) is met */
int dcsc_cuda_run_begin(dcsc_cuda_ctx* ctx);
int dcsc_cuda_run_step(dcsc_cuda_ctx* ctx, dcsc_trace_row* rows, int* converged);
/* acceptance decisions of the last run_step: image_accept (this rank's N
 * images, pipeline.cpp:236), dict_accept (pipeline.cpp:272); either may be NULL */
int dcsc_cuda_run_accepts(dcsc_cuda_ctx* ctx, int* image_accept, int* dict_accept);

/* standalone half-spectrum DFTs of a batch of H x W real planes:
 * forward writes batch * H * (W/2+1) complex (interleaved re,im) */
int dcsc_cuda_dft2_forward(int height, int width, int precision, int batch, const double* in,
                           double* out);
int dcsc_cuda_dft2_inverse(int height, int width, int precision, int batch, const double* in,
                           double* out);

/* device-timed batched r2c / c2r of random planes (mean ms per batch call),
 * the comparator hook against cuFFT (scripts/fft_comparator.py) */
int dcsc_cuda_fft_timing(int height, int width, int precision, int batch, int iters, double* ms_r2c,
                         double* ms_c2r);

/* measurement: kernels launched by this context so far; per-kernel-family
 * CUDA-event timing (family: 0 coding_pass ADMM, 1 lambda_update,
 * 2 learning contractions — the z_hat streams contract_c / contract_out, one
 * z_hat read per launch —, 3 learning mask step, 4 other) */
int dcsc_cuda_kernel_launches(dcsc_cuda_ctx* ctx, long long* count);
/* per-launch CUDA-event timing on the library stream: 0 off, 1 every launch,
 * 2 coding-pass launches only (cheap enough to leave on in a timed region),
 * 3 coding-pass launches + the learning z_hat streams (families 0 and 2) */
int dcsc_cuda_set_profiling(dcsc_cuda_ctx* ctx, int enable);
int dcsc_cuda_kernel_time(dcsc_cuda_ctx* ctx, int family, double* total_ms, long long* launches);
/* device-event timer on the context stream: mark(slot), elapsed(slot a, slot b) */
int dcsc_cuda_event_mark(dcsc_cuda_ctx* ctx, int slot);
int dcsc_cuda_event_elapsed(dcsc_cuda_ctx* ctx, int a, int b, double* ms);
/* bytes of device memory held by the context */
int dcsc_cuda_device_bytes(dcsc_cuda_ctx* ctx, size_t* bytes);

/* Which ADMM coding iteration the context runs (no reference counterpart:
 * the reference has one, admm_coding, coding.cpp:166-329):
 * 0 = the fused FFT pass (half-spectrum c2r / prox / r2c per filter),
 * 1 = the tensor-core spatial pass (FP32 grids 256^2, 128^2, 100^2, 80^2
 *     with 11 x 11 supports and 64^2 with 7 x 7, K <= 128, one channel),
 *     for a coding call over all the context's images. It runs for batches of
 *     at least two work items per SM; DCSC_TC=1 forces it whenever it
 *     applies, DCSC_TC=0 disables it. */
int dcsc_cuda_coding_path(dcsc_cuda_ctx* ctx, int* path);

/* multi-rank: one context per GPU holds its shard of images; learning sums
 * its K x NB correlations and the CG / trace scalars over ranks.
 * dcsc_cuda_nccl_unique_id: rank 0 creates the id (>= 128 bytes) and ships it
 * to the other ranks (e.g. torch.distributed broadcast); each rank then calls
 * dcsc_cuda_set_comm_nccl. dcsc_cuda_set_comm_callback installs a host-side
 * in-place sum (for testing ranks that share one GPU, e.g. over gloo). */
typedef int (*dcsc_allreduce_fn)(double* buf, size_t n, void* user);
int dcsc_cuda_nccl_unique_id(unsigned char* out, size_t len);
int dcsc_cuda_set_comm_nccl(dcsc_cuda_ctx* ctx, int world, int rank, const unsigned char* id, size_t len);
int dcsc_cuda_set_comm_callback(dcsc_cuda_ctx* ctx, int world, int rank, dcsc_allreduce_fn fn, void* user);
/* learning layout across ranks (call after set_comm_*; J = 1):
 * 0 image-sharded (default): each rank keeps z_hat of its own images, the
 *   K x M cropped correlations are all-reduced per operator apply;
 * 1 frequency-sharded (BASELINE.json north_star): after coding, one
 *   all-to-all (grouped ncclSend/ncclRecv) moves z_hat (and x_hat) from
 *   image-major to frequency-major blocks, so each rank runs CG over all N
 *   images on 1/world of the bins; the cropped correlations are still
 *   all-reduced (crop(iDFT(sum_r c_r)) = sum_r crop(iDFT(c_r))) and the
 *   per-image learning data terms are all-reduced. Learning-state get/set is
 *   not available in this layout. A no-op on one rank. */
int dcsc_cuda_set_learning_layout(dcsc_cuda_ctx* ctx, int layout);

/* On-disk formats, byte-compatible with the reference (host only):
 * CSCT tensors (tensor_io.hpp:1-30; tensor_io.cpp:45-90) and the
 * convergence-trace CSV (trace_io.hpp; trace_io.cpp:11-76). Errors return
 * DCSC_ERR_IO with the message in dcsc_io_last_error. */
int dcsc_io_last_error(char* buf, size_t len);
int dcsc_io_write_tensor(const char* path, int ndim, const uint64_t* dims, const double* values);
int dcsc_io_read_tensor_header(const char* path, int* ndim, uint64_t* dims /* 255 */, uint64_t* count);
int dcsc_io_read_tensor(const char* path, double* values, uint64_t count);
int dcsc_io_write_trace_csv(const char* path, const dcsc_trace_row* rows, int n);
int dcsc_io_read_trace_csv(const char* path, dcsc_trace_row* rows, int max_rows, int* n_rows);

/* synthetic BASELINE data (host only, no GPU): x N*H*W, d_true K*m*m */
int dcsc_synth_generate(int n_images, int height, int width, int filters, int m, double p,
                        double sigma, uint64_t seed, int round_fp32, double* x, double* d_true);
/* images [n0, n0 + n_images) of the same seeded dataset (per-image streams) */
int dcsc_synth_generate_range(int n0, int n_images, int height, int width, int filters, int m, double p,
                              double sigma, uint64_t seed, int round_fp32, double* x, double* d_true);
/* the reference bench harness's dataset (bench.cpp:9-21): uniform [0,1) values
 * from one mt19937_64(seed), N*J*H*W doubles */
int dcsc_synth_dataset(int n_images, int channels, int height, int width, uint64_t seed, double* x);

#ifdef __cplusplus
}
#endif

#endif /* DCSC_CUDA_H */
