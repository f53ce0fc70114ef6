// C-ABI over the UNMODIFIED reference hot-path translation units
// (TEST INFRASTRUCTURE ONLY: loaded by tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference leg; never by the product).
//
// oracle/Makefile compiles /root/reference/proj/src/{types,parallel,spectral,
// objective,coding,learning,pipeline,tensor_io,trace_io,tcsc}.cpp in place (no
// sources are copied) against oracle/fftw3.h + oracle/fftw_shim.c and (tcsc.cpp)
// the Eigen-API shim oracle/eigen_shim/, links this file, and writes
// oracle/_ref/libdcsc_ref.so. The *_j entry points take J channels (signals
// N x J x D, dictionary K x J x M, lambda J x D, gamma J x N x D); J > 1 runs
// the reference's TCSC path (Joint channel mode, pipeline.cpp:168).
//
// ref_run() is an instrumented replica of dcsc::run_csc
// (proj/src/pipeline.cpp:158-301) assembled ONLY from the reference's public
// functions (normalize, init_variables, solve_coding, evaluate_objective,
// solve_learning, learning_data_term). It exists because run_csc returns only
// the final state; the replica additionally dumps the per-outer-iteration
// dictionary, the l0 count of the maps and mu_iters. tests/ assert that its
// trace equals run_csc's (ref_run_csc) bit for bit at one thread.
#ifdef _OPENMP
#include <omp.h>
#endif
#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "dcsc/coding.hpp"
#include "dcsc/learning.hpp"
#include "dcsc/objective.hpp"
#include "dcsc/parallel.hpp"
#include "dcsc/pipeline.hpp"
#include "dcsc/spectral.hpp"
#include "dcsc/tcsc.hpp"
#include "dcsc/tensor_io.hpp"
#include "dcsc/trace_io.hpp"
#include "dcsc/types.hpp"

using namespace dcsc;

extern "C" {

struct ref_cfg {
  double beta, rho, tol;
  int max_outer, max_admm, max_mu_iters;
  double cg_tol;
  int cg_max;
  double mu_floor;
  std::uint64_t seed;
  int normalize;  // 0 None, 1 Global, 2 Local
};

struct ref_coding_stats {
  int admm_iters, converged, degenerate_dictionary, dual_rescaled;
  double primal_residual, theta_change, z_change, dual_objective, dual_infeasibility;
};

struct ref_learning_stats {
  int mu_iters;
  long cg_iters, cg_iters_first;
  int converged, degenerate, mu_clamped, cg_budget_hit, rescaled_filters, n_dead;
};

struct ref_trace_row {
  int outer_iter, phase;
  double total, data_term, l1_term, residual_norm;
  long admm_iters, cg_iters;
  int mu_iters;
  double elapsed_ms;  // reference timer: solver call only
  double wall_ms;     // whole half-step including objective bookkeeping
  long l0;            // |z| > 1e-12 * max|z| over the accepted maps (coding rows)
};

}  // extern "C"

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const DimensionError& e) {
    g_err = e.what();
    return 1;
  } catch (const NumericError& e) {
    g_err = e.what();
    return 2;
  } catch (const IoError& e) {
    g_err = e.what();
    return 5;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 4;
  }
}

SolverConfig to_cfg(const ref_cfg* c) {
  SolverConfig s;
  s.beta = c->beta;
  s.rho = c->rho;
  s.tol = c->tol;
  s.max_outer = c->max_outer;
  s.max_admm = c->max_admm;
  s.max_mu_iters = c->max_mu_iters;
  s.cg_tol = c->cg_tol;
  s.cg_max = c->cg_max;
  s.mu_floor = c->mu_floor;
  s.seed = c->seed;
  s.normalize = c->normalize == 0 ? NormalizeMode::None
                : c->normalize == 1 ? NormalizeMode::Global
                                    : NormalizeMode::Local;
  return s;
}

double now_ms() {
  using clock = std::chrono::steady_clock;
  return std::chrono::duration<double, std::milli>(clock::now().time_since_epoch()).count();
}

Dictionary make_dict(int K, int mh, int mw, const double* d, int J = 1) {
  Dictionary dict(K, {mh, mw}, J);
  std::copy(d, d + dict.values.size(), dict.values.begin());
  return dict;
}

SignalTensor make_signal(int H, int W, const double* x, int J = 1) {
  SignalTensor s({H, W}, J);
  std::copy(x, x + s.values.size(), s.values.begin());
  return s;
}

void put_coding_stats(const CodingStats& s, ref_coding_stats* st) {
  if (!st) return;
  st->admm_iters = s.admm_iters;
  st->converged = s.converged;
  st->degenerate_dictionary = s.degenerate_dictionary;
  st->dual_rescaled = s.dual_rescaled;
  st->primal_residual = s.primal_residual;
  st->theta_change = s.theta_change;
  st->z_change = s.z_change;
  st->dual_objective = s.dual_objective;
  st->dual_infeasibility = s.dual_infeasibility;
}

void put_learning_stats(const LearningStats& s, ref_learning_stats* st) {
  if (!st) return;
  st->mu_iters = s.mu_iters;
  st->cg_iters = s.cg_iters;
  st->cg_iters_first = s.cg_iters_first;
  st->converged = s.converged;
  st->degenerate = s.degenerate;
  st->mu_clamped = s.mu_clamped;
  st->cg_budget_hit = s.cg_budget_hit;
  st->rescaled_filters = s.rescaled_filters;
  st->n_dead = static_cast<int>(s.dead_filters.size());
}

long count_l0(const std::vector<SparseMaps>& maps) {
  double mx = 0.0;
  for (const auto& m : maps)
    for (double v : m.values) mx = std::max(mx, std::abs(v));
  const double thr = 1e-12 * mx;
  long c = 0;
  for (const auto& m : maps)
    for (double v : m.values)
      if (std::abs(v) > thr) ++c;
  return c;
}

}  // namespace

extern "C" {

int ref_last_error(char* buf, std::size_t len) {
  if (buf && len) {
    std::strncpy(buf, g_err.c_str(), len - 1);
    buf[len - 1] = 0;
  }
  return static_cast<int>(g_err.size());
}

int ref_set_threads(int n) {
  // par::max_threads() is capped by omp_get_max_threads(), which a launcher's
  // OMP_NUM_THREADS=1 (torchrun's default) would pin to 1: raise the OpenMP
  // thread budget of this (calling) thread too.
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#endif
  par::set_max_threads(n);
  return par::max_threads();
}

// rank-D forward DFT of a real grid: out is D interleaved complex values.
int ref_forward_dft(int rank, const int* dims, const double* in, double* out) {
  return guarded([&] {
    GridDims g(dims, dims + rank);
    const std::size_t n = grid_count(g);
    Spectrum s = forward_dft(g, std::span<const double>(in, n));
    std::memcpy(out, s.values.data(), n * sizeof(std::complex<double>));
  });
}

// rank-D inverse DFT (1/D, real part kept, residue guard) of a full spectrum.
int ref_inverse_dft(int rank, const int* dims, const double* in, double* out) {
  return guarded([&] {
    GridDims g(dims, dims + rank);
    Spectrum s(g);
    std::memcpy(s.values.data(), in, s.values.size() * sizeof(std::complex<double>));
    inverse_dft(s, std::span<double>(out, s.values.size()));
  });
}

int ref_init_dictionary_j(int K, int J, int mh, int mw, int H, int W, std::uint64_t seed, double* out) {
  return guarded([&] {
    RunConfig rc;
    rc.solver.seed = seed;
    rc.filters = K;
    rc.support = {mh, mw};
    rc.channel_mode = J > 1 ? ChannelMode::Joint : ChannelMode::Separate;
    InitVariables v = init_variables(rc, {H, W}, J, 1);
    std::copy(v.dict.values.begin(), v.dict.values.end(), out);
  });
}

int ref_init_dictionary(int K, int mh, int mw, int H, int W, std::uint64_t seed, double* out) {
  return ref_init_dictionary_j(K, 1, mh, mw, H, W, seed, out);
}

// One solve_coding call. theta/z/lambda are in/out warm state (K*D, K*D, D);
// warm = 0 starts from the reference's empty state.
int ref_solve_coding(int H, int W, const double* x, int K, int mh, int mw, const double* d,
                     const ref_cfg* cfg, int warm, double* theta, double* z, double* lambda,
                     ref_coding_stats* st) {
  return guarded([&] {
    const SignalTensor xs = make_signal(H, W, x);
    const Dictionary dict = make_dict(K, mh, mw, d);
    const std::size_t D = static_cast<std::size_t>(H) * W;
    CodingDualState state;
    if (warm) {
      state.theta.assign(theta, theta + K * D);
      state.z.assign(z, z + K * D);
      state.lambda.assign(lambda, lambda + D);
    }
    CodingStats s;
    solve_coding(xs, dict, to_cfg(cfg), state, &s);
    std::copy(state.theta.begin(), state.theta.end(), theta);
    std::copy(state.z.begin(), state.z.end(), z);
    std::copy(state.lambda.begin(), state.lambda.end(), lambda);
    put_coding_stats(s, st);
  });
}

// solve_coding_tcsc (tcsc.cpp) on a J-channel signal x (J*D); d is K*J*M;
// lambda is J*D. method: 0 Auto, 1 Direct, 2 Woodbury.
int ref_solve_coding_tcsc(int H, int W, int J, const double* x, int K, int mh, int mw, const double* d,
                          const ref_cfg* cfg, int warm, double* theta, double* z, double* lambda,
                          int method, ref_coding_stats* st) {
  return guarded([&] {
    const SignalTensor xs = make_signal(H, W, x, J);
    const Dictionary dict = make_dict(K, mh, mw, d, J);
    const std::size_t D = static_cast<std::size_t>(H) * W;
    CodingDualState state;
    if (warm) {
      state.theta.assign(theta, theta + K * D);
      state.z.assign(z, z + K * D);
      state.lambda.assign(lambda, lambda + J * D);
    }
    CodingStats s;
    const BlockSolveMethod m = method == 1   ? BlockSolveMethod::Direct
                               : method == 2 ? BlockSolveMethod::Woodbury
                                             : BlockSolveMethod::Auto;
    solve_coding_tcsc(xs, dict, to_cfg(cfg), state, &s, m);
    std::copy(state.theta.begin(), state.theta.end(), theta);
    std::copy(state.z.begin(), state.z.end(), z);
    std::copy(state.lambda.begin(), state.lambda.end(), lambda);
    put_coding_stats(s, st);
  });
}

// solve_coding over N images from the empty state, OpenMP-parallel over
// images exactly as run_csc's coding half-step (pipeline.cpp:221-227).
// Used by bench.py as the reference CPU arm. iters_out: per-image ADMM iterations.
int ref_coding_batch(int N, int H, int W, const double* xs, int K, int mh, int mw,
                     const double* d, const ref_cfg* cfg, double* maps_out, int* iters_out) {
  return guarded([&] {
    const std::size_t D = static_cast<std::size_t>(H) * W;
    const Dictionary dict = make_dict(K, mh, mw, d);
    const SolverConfig sc = to_cfg(cfg);
    std::vector<SignalTensor> sig;
    for (int n = 0; n < N; ++n) sig.push_back(make_signal(H, W, xs + n * D));
    std::vector<SparseMaps> out(N);
    std::vector<CodingStats> st(N);
    std::vector<CodingDualState> state(N);
    par::parallel_for(N, [&](std::int64_t n) { out[n] = solve_coding(sig[n], dict, sc, state[n], &st[n]); });
    for (int n = 0; n < N; ++n) {
      if (iters_out) iters_out[n] = st[n].admm_iters;
      if (maps_out) std::copy(out[n].values.begin(), out[n].values.end(), maps_out + n * K * D);
    }
  });
}

// solve_coding_tcsc over N J-channel images (xs N*J*D, d K*J*M) from the empty
// state, OpenMP-parallel over images (pipeline.cpp:221-227, Joint mode).
int ref_coding_batch_j(int N, int H, int W, int J, const double* xs, int K, int mh, int mw,
                       const double* d, const ref_cfg* cfg, double* maps_out, int* iters_out) {
  return guarded([&] {
    const std::size_t D = static_cast<std::size_t>(H) * W;
    const Dictionary dict = make_dict(K, mh, mw, d, J);
    const SolverConfig sc = to_cfg(cfg);
    std::vector<SignalTensor> sig;
    for (int n = 0; n < N; ++n) sig.push_back(make_signal(H, W, xs + n * J * D, J));
    std::vector<SparseMaps> out(N);
    std::vector<CodingStats> st(N);
    std::vector<CodingDualState> state(N);
    par::parallel_for(N, [&](std::int64_t n) {
      out[n] = J > 1 ? solve_coding_tcsc(sig[n], dict, sc, state[n], &st[n])
                     : solve_coding(sig[n], dict, sc, state[n], &st[n]);
    });
    for (int n = 0; n < N; ++n) {
      if (iters_out) iters_out[n] = st[n].admm_iters;
      if (maps_out) std::copy(out[n].values.begin(), out[n].values.end(), maps_out + n * K * D);
    }
  });
}

// One solve_learning call over N J-channel images (xs N*J*D). gamma (J*N*D,
// channel-major) / mu (K) are in/out warm state; warm = 0 starts from the
// empty state. d_out receives K*J*M values.
int ref_solve_learning_j(int N, int H, int W, int J, const double* xs, int K, const double* maps, int mh,
                         int mw, const ref_cfg* cfg, int warm, double* gamma, double* mu, double* d_out,
                         ref_learning_stats* st) {
  return guarded([&] {
    const std::size_t D = static_cast<std::size_t>(H) * W;
    std::vector<SignalTensor> sig;
    std::vector<SparseMaps> zs;
    for (int n = 0; n < N; ++n) {
      sig.push_back(make_signal(H, W, xs + n * J * D, J));
      SparseMaps m(K, {H, W});
      std::copy(maps + n * K * D, maps + (n + 1) * K * D, m.values.begin());
      zs.push_back(std::move(m));
    }
    LearningDualState state;
    if (warm) {
      state.gamma.clear();
      for (int j = 0; j < J; ++j)
        state.gamma.emplace_back(gamma + j * N * D, gamma + (j + 1) * N * D);
      state.mu.assign(mu, mu + K);
    }
    LearningStats s;
    Dictionary dict = J > 1 ? solve_learning_tcsc(sig, zs, {mh, mw}, to_cfg(cfg), state, &s)
                            : solve_learning(sig, zs, {mh, mw}, to_cfg(cfg), state, &s);
    std::copy(dict.values.begin(), dict.values.end(), d_out);
    for (int j = 0; j < (int)state.gamma.size() && j < J; ++j)
      std::copy(state.gamma[j].begin(), state.gamma[j].end(), gamma + j * N * D);
    std::copy(state.mu.begin(), state.mu.end(), mu);
    put_learning_stats(s, st);
  });
}

int ref_solve_learning(int N, int H, int W, const double* xs, int K, const double* maps, int mh,
                       int mw, const ref_cfg* cfg, int warm, double* gamma, double* mu,
                       double* d_out, ref_learning_stats* st) {
  return ref_solve_learning_j(N, H, W, 1, xs, K, maps, mh, mw, cfg, warm, gamma, mu, d_out, st);
}

// evaluate_objective for one J-channel image: out = {data_term, l1_term, total, residual_norm}
int ref_objective_j(int H, int W, int J, const double* x, int K, int mh, int mw, const double* d,
                    const double* z, double beta, double* out) {
  return guarded([&] {
    SparseMaps m(K, {H, W});
    std::copy(z, z + m.values.size(), m.values.begin());
    const ObjectiveBreakdown b =
        evaluate_objective(make_signal(H, W, x, J), make_dict(K, mh, mw, d, J), m, beta);
    out[0] = b.data_term;
    out[1] = b.l1_term;
    out[2] = b.total;
    out[3] = b.residual_norm;
  });
}

// reconstruct (objective.cpp:39-57): out J*D from d (K*J*M) and maps z (K*D)
int ref_reconstruct_j(int H, int W, int J, int K, int mh, int mw, const double* d, const double* z,
                      double* out) {
  return guarded([&] {
    SparseMaps m(K, {H, W});
    std::copy(z, z + m.values.size(), m.values.begin());
    const SignalTensor r = reconstruct(make_dict(K, mh, mw, d, J), m);
    std::copy(r.values.begin(), r.values.end(), out);
  });
}

int ref_objective(int H, int W, const double* x, int K, int mh, int mw, const double* d,
                  const double* z, double beta, double* out) {
  return ref_objective_j(H, W, 1, x, K, mh, mw, d, z, beta, out);
}

// LearningOperator::apply (proj/src/learning.cpp:83-122) on stacked N*D vectors.
int ref_learning_apply(int N, int H, int W, int K, const double* maps, int mh, int mw,
                       const double* mu, double mu_floor, const double* v, double* out) {
  return guarded([&] {
    const std::size_t D = static_cast<std::size_t>(H) * W;
    std::vector<SparseMaps> zs;
    for (int n = 0; n < N; ++n) {
      SparseMaps m(K, {H, W});
      std::copy(maps + n * K * D, maps + (n + 1) * K * D, m.values.begin());
      zs.push_back(std::move(m));
    }
    LearningOperator op(zs, {mh, mw}, mu_floor);
    op.set_mu(std::span<const double>(mu, K));
    op.apply(std::span<const double>(v, N * D), std::span<double>(out, N * D));
  });
}

// Stateless ops (coding.hpp:45-66, learning.hpp:81-95) for one J = 1 image /
// the stacked learning system, for the GPU stateless-op parity tests.
int ref_lambda_update(int H, int W, const double* x, int K, int mh, int mw, const double* d, const double* theta,
                      const double* z, double rho, double* out) {
  return guarded([&] {
    const GridDims g{H, W};
    const std::size_t D = static_cast<std::size_t>(H) * W;
    const Dictionary dict = make_dict(K, mh, mw, d);
    std::vector<Spectrum> dh, th, zh;
    for (int k = 0; k < K; ++k) {
      dh.push_back(filter_spectrum(dict, k, 0, g));
      th.push_back(forward_dft(g, std::span<const double>(theta + k * D, D)));
      zh.push_back(forward_dft(g, std::span<const double>(z + k * D, D)));
    }
    const Spectrum xh = forward_dft(g, std::span<const double>(x, D));
    const std::vector<double> lam = lambda_update(dh, th, zh, xh, rho);
    std::copy(lam.begin(), lam.end(), out);
  });
}

int ref_dictionary_adjoint(int H, int W, int K, int mh, int mw, const double* d, const double* lambda, double* out) {
  return guarded([&] {
    const GridDims g{H, W};
    const std::size_t D = static_cast<std::size_t>(H) * W;
    const Dictionary dict = make_dict(K, mh, mw, d);
    std::vector<Spectrum> dh;
    for (int k = 0; k < K; ++k) dh.push_back(filter_spectrum(dict, k, 0, g));
    const std::vector<double> t = apply_dictionary_adjoint(dh, forward_dft(g, std::span<const double>(lambda, D)));
    std::copy(t.begin(), t.end(), out);
  });
}

int ref_gamma_solve(int N, int H, int W, int K, const double* maps, int mh, int mw, const double* mu,
                    double mu_floor, const double* x, double cg_tol, int cg_max, double* gamma, int* iters,
                    int* converged) {
  return guarded([&] {
    const std::size_t D = static_cast<std::size_t>(H) * W;
    std::vector<SparseMaps> zs;
    for (int n = 0; n < N; ++n) {
      SparseMaps m(K, {H, W});
      std::copy(maps + n * K * D, maps + (n + 1) * K * D, m.values.begin());
      zs.push_back(std::move(m));
    }
    LearningOperator op(zs, {mh, mw}, mu_floor);
    op.set_mu(std::span<const double>(mu, K));
    const CgResult r = gamma_solve(op, std::span<const double>(x, N * D), cg_tol, cg_max,
                                   std::span<double>(gamma, N * D));
    *iters = r.iters;
    *converged = r.converged;
  });
}

int ref_d_recover(int N, int H, int W, int K, const double* maps, int mh, int mw, const double* gamma,
                  const double* mu, double* out) {
  return guarded([&] {
    const std::size_t D = static_cast<std::size_t>(H) * W;
    std::vector<SparseMaps> zs;
    for (int n = 0; n < N; ++n) {
      SparseMaps m(K, {H, W});
      std::copy(maps + n * K * D, maps + (n + 1) * K * D, m.values.begin());
      zs.push_back(std::move(m));
    }
    LearningOperator op(zs, {mh, mw}, 1e-300);
    const auto dk = d_recover(op, std::span<const double>(gamma, N * D), std::span<const double>(mu, K));
    const std::size_t M = static_cast<std::size_t>(mh) * mw;
    for (int k = 0; k < K; ++k) std::copy(dk[k].begin(), dk[k].end(), out + k * M);
  });
}

// CPU-baseline unit costs of the reference learning step (bench.py): wall ms to
// build the LearningOperator (learning.cpp:24-64: N*K forward FFTs) and the mean
// wall ms of one LearningOperator::apply (learning.cpp:83-122) over n_apply calls.
int ref_time_learning(int N, int H, int W, int K, const double* maps, int mh, int mw, int n_apply,
                      double* build_ms, double* apply_ms) {
  return guarded([&] {
    const std::size_t D = static_cast<std::size_t>(H) * W;
    std::vector<SparseMaps> zs;
    for (int n = 0; n < N; ++n) {
      SparseMaps m(K, {H, W});
      std::copy(maps + n * K * D, maps + (n + 1) * K * D, m.values.begin());
      zs.push_back(std::move(m));
    }
    const double t0 = now_ms();
    LearningOperator op(zs, {mh, mw}, 1e-6);
    const double t1 = now_ms();
    std::vector<double> mu(K, 1.0), v(N * D, 0.0), out(N * D);
    for (std::size_t i = 0; i < v.size(); ++i) v[i] = std::sin(0.37 * static_cast<double>(i));
    op.set_mu(std::span<const double>(mu.data(), K));
    for (int a = 0; a < n_apply; ++a)
      op.apply(std::span<const double>(v.data(), N * D), std::span<double>(out.data(), N * D));
    const double t2 = now_ms();
    *build_ms = t1 - t0;
    *apply_ms = (t2 - t1) / std::max(n_apply, 1);
  });
}

// LearningOperator::correlation (learning.cpp:124-134) for every filter: out K*M.
int ref_learning_correlation(int N, int H, int W, int K, const double* maps, int mh, int mw, const double* v,
                             double* out) {
  return guarded([&] {
    const std::size_t D = static_cast<std::size_t>(H) * W;
    std::vector<SparseMaps> zs;
    for (int n = 0; n < N; ++n) {
      SparseMaps m(K, {H, W});
      std::copy(maps + n * K * D, maps + (n + 1) * K * D, m.values.begin());
      zs.push_back(std::move(m));
    }
    LearningOperator op(zs, {mh, mw}, 1e-6);
    const std::size_t M = static_cast<std::size_t>(mh) * mw;
    for (int k = 0; k < K; ++k) {
      const std::vector<double> c = op.correlation(k, std::span<const double>(v, N * D));
      std::copy(c.begin(), c.end(), out + k * M);
    }
  });
}

// Instrumented replica of run_csc (see header comment). xs are the RAW signals;
// normalisation follows cfg->normalize exactly as run_csc does. rows must hold
// 2*max_outer entries. dict_iter (optional) receives (max_outer+1)*K*M values:
// the initial dictionary then the accepted dictionary after each outer
// iteration. maps_out (optional) receives the final N*K*D maps, dict_out the
// final K*M dictionary. Returns the number of outer iterations run in *n_outer.
// J > 1: Joint channel mode (solve_coding_tcsc), signals N*J*D, dictionary K*J*M.
//
// Parity instrumentation (optional, NULL = off): ties_out receives 4 counts per
// outer iteration — entries of the accepted maps' soft-threshold argument
// u = theta - z/rho (so z = -rho soft(u, beta), coding.cpp:237-246) with
// ||u| - beta| <= delta * beta for delta = 1e-7, 1e-6, 1e-5, 1e-4 (the support
// near-ties); accept_out receives N + 1 flags per outer iteration — the
// per-image coding acceptances (pipeline.cpp:236) then the dictionary
// acceptance (pipeline.cpp:272).
static int g_parallel_objective = 0;  // golden generation only: objective passes over images in parallel
int ref_set_parallel_objective(int on) {
  g_parallel_objective = on;
  return 0;
}

int ref_run_j(const ref_cfg* cfgp, int N, int H, int W, int J, const double* xs_raw, int K, int mh,
              int mw, ref_trace_row* rows, int* n_outer, double* dict_iter, double* maps_out,
              double* dict_out, long* ties_out, int* accept_out) {
  return guarded([&] {
    RunConfig cfg;
    cfg.solver = to_cfg(cfgp);
    cfg.filters = K;
    cfg.support = {mh, mw};
    cfg.channel_mode = J > 1 ? ChannelMode::Joint : ChannelMode::Separate;
    const bool tcsc = J > 1;
    const std::size_t D = static_cast<std::size_t>(H) * W;
    const double beta = cfg.solver.beta;
    const double tau = cfg.solver.tol;
    std::vector<SignalTensor> xs(N);
    for (int n = 0; n < N; ++n)
      xs[n] = normalize(make_signal(H, W, xs_raw + n * J * D, J), cfg.solver.normalize);

    InitVariables vars = init_variables(cfg, {H, W}, J, N);
    Dictionary dict = vars.dict;
    std::vector<SparseMaps> maps = vars.maps;
    const std::size_t KM = dict.values.size();
    if (dict_iter) std::copy(dict.values.begin(), dict.values.end(), dict_iter);
    *n_outer = 0;

    auto total_objective = [&]() {
      ObjectiveBreakdown sum;
      for (int n = 0; n < N; ++n) {
        const ObjectiveBreakdown b = evaluate_objective(xs[n], dict, maps[n], beta);
        sum.data_term += b.data_term;
        sum.l1_term += b.l1_term;
        sum.residual_norm += b.residual_norm * b.residual_norm;
      }
      sum.total = sum.data_term + sum.l1_term;
      sum.residual_norm = std::sqrt(sum.residual_norm);
      return sum;
    };
    double prev_total = total_objective().total;
    std::vector<ObjectiveBreakdown> image_obj(N);
    for (int n = 0; n < N; ++n) image_obj[n] = evaluate_objective(xs[n], dict, maps[n], beta);
    // near-tie counts of each image's accepted maps (4 bands), see header
    std::vector<std::array<long, 4>> ties(N, std::array<long, 4>{0, 0, 0, 0});
    auto count_ties = [&](const CodingDualState& st) {
      std::array<long, 4> t{0, 0, 0, 0};
      const double inv_rho = 1.0 / cfg.solver.rho;
      const double bands[4] = {1e-7, 1e-6, 1e-5, 1e-4};
      for (std::size_t i = 0; i < st.theta.size(); ++i) {
        const double u = st.theta[i] - st.z[i] * inv_rho;
        const double gap = std::abs(std::abs(u) - beta);
        for (int b = 0; b < 4; ++b) t[b] += gap <= bands[b] * beta ? 1 : 0;
      }
      return t;
    };

    int row = 0;
    for (int outer = 1; outer <= cfg.solver.max_outer; ++outer) {
      const double wall0 = now_ms();
      std::vector<SparseMaps> cand(N);
      std::vector<CodingStats> cs(N);
      const double c0 = now_ms();
      par::parallel_for(N, [&](std::int64_t n) {
        cand[n] = tcsc ? solve_coding_tcsc(xs[n], dict, cfg.solver, vars.coding[n], &cs[n])
                       : solve_coding(xs[n], dict, cfg.solver, vars.coding[n], &cs[n]);
      });
      const double coding_ms = now_ms() - c0;
      long admm_total = 0;
      double z_change_sq = 0.0, z_norm_sq = 0.0;
      std::vector<ObjectiveBreakdown> cobj(N);
      if (g_parallel_objective)
        par::parallel_for(N, [&](std::int64_t n) { cobj[n] = evaluate_objective(xs[n], dict, cand[n], beta); });
      for (int n = 0; n < N; ++n) {
        admm_total += cs[n].admm_iters;
        const ObjectiveBreakdown c = g_parallel_objective ? cobj[n] : evaluate_objective(xs[n], dict, cand[n], beta);
        if (!std::isfinite(c.total)) throw NumericError("non-finite objective (coding)");
        if (accept_out) accept_out[(size_t)(outer - 1) * (N + 1) + n] = c.total <= image_obj[n].total ? 1 : 0;
        if (c.total <= image_obj[n].total) {
          if (ties_out && !tcsc) ties[n] = count_ties(vars.coding[n]);
          for (std::size_t i = 0; i < cand[n].values.size(); ++i) {
            const double delta = cand[n].values[i] - maps[n].values[i];
            z_change_sq += delta * delta;
          }
          maps[n] = std::move(cand[n]);
          image_obj[n] = c;
        }
        for (double v : maps[n].values) z_norm_sq += v * v;
      }
      ObjectiveBreakdown after_coding;
      for (int n = 0; n < N; ++n) {
        after_coding.data_term += image_obj[n].data_term;
        after_coding.l1_term += image_obj[n].l1_term;
        after_coding.residual_norm += image_obj[n].residual_norm * image_obj[n].residual_norm;
      }
      after_coding.total = after_coding.data_term + after_coding.l1_term;
      after_coding.residual_norm = std::sqrt(after_coding.residual_norm);
      const double wall1 = now_ms();
      rows[row++] = {outer, 0, after_coding.total, after_coding.data_term, after_coding.l1_term,
                     after_coding.residual_norm, admm_total, 0, 0, coding_ms, wall1 - wall0,
                     count_l0(maps)};
      if (ties_out)
        for (int b = 0; b < 4; ++b) {
          long t = 0;
          for (int n = 0; n < N; ++n) t += ties[n][b];
          ties_out[(size_t)(outer - 1) * 4 + b] = t;
        }

      LearningStats ls;
      const double l0 = now_ms();
      Dictionary dc = tcsc ? solve_learning_tcsc(xs, maps, cfg.support, cfg.solver, vars.learning, &ls)
                           : solve_learning(xs, maps, cfg.support, cfg.solver, vars.learning, &ls);
      const double learning_ms = now_ms() - l0;
      double d_change_sq = 0.0, d_norm_sq = 0.0;
      ObjectiveBreakdown after_learning = after_coding;
      const double cand_data = learning_data_term(xs, dc, maps);
      if (!std::isfinite(cand_data + after_coding.l1_term))
        throw NumericError("non-finite objective (learning)");
      if (accept_out) accept_out[(size_t)(outer - 1) * (N + 1) + N] = cand_data <= after_coding.data_term ? 1 : 0;
      if (cand_data <= after_coding.data_term) {
        for (std::size_t i = 0; i < dc.values.size(); ++i) {
          const double delta = dc.values[i] - dict.values[i];
          d_change_sq += delta * delta;
        }
        dict = std::move(dc);
        after_learning.data_term = cand_data;
        after_learning.total = cand_data + after_coding.l1_term;
        after_learning.residual_norm = std::sqrt(2.0 * cand_data);
        if (g_parallel_objective)
          par::parallel_for(N, [&](std::int64_t n) { image_obj[n] = evaluate_objective(xs[n], dict, maps[n], beta); });
        else
          for (int n = 0; n < N; ++n) image_obj[n] = evaluate_objective(xs[n], dict, maps[n], beta);
      }
      for (double v : dict.values) d_norm_sq += v * v;
      const double wall2 = now_ms();
      rows[row++] = {outer, 1, after_learning.total, after_learning.data_term,
                     after_learning.l1_term, after_learning.residual_norm, 0, ls.cg_iters,
                     ls.mu_iters, learning_ms, wall2 - wall1, count_l0(maps)};
      if (dict_iter) std::copy(dict.values.begin(), dict.values.end(), dict_iter + outer * KM);
      *n_outer = outer;

      const double obj_change =
          std::abs(prev_total - after_learning.total) / std::max(std::abs(prev_total), 1e-30);
      const double z_change = std::sqrt(z_change_sq) / std::max(std::sqrt(z_norm_sq), 1.0);
      const double d_change = std::sqrt(d_change_sq) / std::max(std::sqrt(d_norm_sq), 1.0);
      prev_total = after_learning.total;
      if (obj_change <= tau && z_change <= tau && d_change <= tau) break;
    }
    if (maps_out)
      for (int n = 0; n < N; ++n) std::copy(maps[n].values.begin(), maps[n].values.end(), maps_out + n * K * D);
    if (dict_out) std::copy(dict.values.begin(), dict.values.end(), dict_out);
  });
}

int ref_run(const ref_cfg* cfgp, int N, int H, int W, const double* xs_raw, int K, int mh,
            int mw, ref_trace_row* rows, int* n_outer, double* dict_iter, double* maps_out,
            double* dict_out) {
  return ref_run_j(cfgp, N, H, W, 1, xs_raw, K, mh, mw, rows, n_outer, dict_iter, maps_out, dict_out, nullptr,
                   nullptr);
}

int ref_run_ext(const ref_cfg* cfgp, int N, int H, int W, const double* xs_raw, int K, int mh, int mw,
                ref_trace_row* rows, int* n_outer, double* dict_iter, double* maps_out, double* dict_out,
                long* ties_out, int* accept_out) {
  return ref_run_j(cfgp, N, H, W, 1, xs_raw, K, mh, mw, rows, n_outer, dict_iter, maps_out, dict_out, ties_out,
                   accept_out);
}

// The reference's CSCT writer/reader (tensor_io.cpp:45-90) and trace CSV
// writer (trace_io.cpp:15-30), for byte-compatibility tests of the product's.
int ref_write_tensor(const char* path, int ndim, const std::uint64_t* dims, const double* values) {
  return guarded([&] {
    TensorData t;
    t.dims.assign(dims, dims + ndim);
    std::uint64_t n = 1;
    for (auto d : t.dims) n *= d;
    t.values.assign(values, values + n);
    write_tensor(path, t);
  });
}

int ref_read_tensor(const char* path, double* values, std::uint64_t count) {
  return guarded([&] {
    TensorData t = read_tensor(path);
    if (t.values.size() != count) throw IoError("count mismatch");
    std::copy(t.values.begin(), t.values.end(), values);
  });
}

int ref_write_trace_csv(const char* path, const ref_trace_row* rows, int n) {
  return guarded([&] {
    ConvergenceTrace tr;
    for (int i = 0; i < n; ++i) {
      TraceRow r;
      r.outer_iter = rows[i].outer_iter;
      r.phase = rows[i].phase == 0 ? Phase::Coding : Phase::Learning;
      r.objective.total = rows[i].total;
      r.objective.data_term = rows[i].data_term;
      r.objective.l1_term = rows[i].l1_term;
      r.admm_iters = rows[i].admm_iters;
      r.cg_iters = rows[i].cg_iters;
      r.elapsed_ms = rows[i].elapsed_ms;
      tr.rows.push_back(r);
    }
    write_trace_csv(std::string(path), tr);
  });
}

// The reference's own run_csc, for checking the replica (trace rows only).
int ref_run_csc_j(const ref_cfg* cfgp, int N, int H, int W, int J, const double* xs_raw, int K, int mh,
                  int mw, ref_trace_row* rows, int* n_rows, double* dict_out, double* maps_out) {
  return guarded([&] {
    RunConfig cfg;
    cfg.solver = to_cfg(cfgp);
    cfg.filters = K;
    cfg.support = {mh, mw};
    cfg.channel_mode = J > 1 ? ChannelMode::Joint : ChannelMode::Separate;
    const std::size_t D = static_cast<std::size_t>(H) * W;
    Dataset data;
    for (int n = 0; n < N; ++n) data.signals.push_back(make_signal(H, W, xs_raw + n * J * D, J));
    RunResult r = run_csc(cfg, data);
    *n_rows = static_cast<int>(r.trace.rows.size());
    for (std::size_t i = 0; i < r.trace.rows.size(); ++i) {
      const TraceRow& t = r.trace.rows[i];
      rows[i] = {t.outer_iter, t.phase == Phase::Coding ? 0 : 1, t.objective.total,
                 t.objective.data_term, t.objective.l1_term, t.objective.residual_norm,
                 t.admm_iters, t.cg_iters, 0, t.elapsed_ms, 0.0, 0};
    }
    if (dict_out) std::copy(r.dict.values.begin(), r.dict.values.end(), dict_out);
    if (maps_out)
      for (int n = 0; n < N; ++n) std::copy(r.maps[n].values.begin(), r.maps[n].values.end(), maps_out + n * K * D);
  });
}

int ref_run_csc(const ref_cfg* cfgp, int N, int H, int W, const double* xs_raw, int K, int mh,
                int mw, ref_trace_row* rows, int* n_rows, double* dict_out, double* maps_out) {
  return ref_run_csc_j(cfgp, N, H, W, 1, xs_raw, K, mh, mw, rows, n_rows, dict_out, maps_out);
}

}  // extern "C"
