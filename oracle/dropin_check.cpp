// Drop-in demonstration (TEST INFRASTRUCTURE): the same reference program calls
// dcsc::run_csc (the reference, CPU) and dcsc::cuda::run_csc (include/dcsc_cuda.hpp
// over the CUDA C-ABI) on identical data and compares the traces and dictionaries.
// Built by oracle/Makefile (target dropin) against the reference headers; run by
// tests/test_dropin_gpu.py. Exit code 0 = within tolerance.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "dcsc/pipeline.hpp"
#include "dcsc_cuda.hpp"

// Error behaviour: the reference and the drop-in must throw the same exception
// type for the same bad input (types.hpp:24-38, pipeline.cpp:66-80,159-167).
template <class F>
static const char* thrown(F&& f) {
  try {
    f();
  } catch (const dcsc::DimensionError&) {
    return "DimensionError";
  } catch (const dcsc::NumericError&) {
    return "NumericError";
  } catch (const std::invalid_argument&) {
    return "invalid_argument";
  } catch (const std::exception&) {
    return "other";
  }
  return "none";
}

static int check_errors() {
  auto signal = [](int h, int w, double fill) {
    dcsc::SignalTensor x({h, w}, 1);
    for (std::size_t i = 0; i < x.values.size(); ++i) x.values[i] = fill + 0.001 * static_cast<double>(i % 7);
    return x;
  };
  dcsc::RunConfig cfg;
  cfg.filters = 2;
  cfg.support = {3, 3};
  cfg.solver.max_outer = 1;
  struct Case {
    const char* name;
    dcsc::Dataset data;
    dcsc::RunConfig cfg;
  };
  std::vector<Case> cases;
  cases.push_back({"empty dataset", dcsc::Dataset{}, cfg});
  {
    dcsc::Dataset d;
    d.signals = {signal(16, 16, 0.1), signal(20, 20, 0.2)};
    d.names = {"a", "b"};
    cases.push_back({"ragged dataset", d, cfg});
  }
  {
    dcsc::Dataset d;
    d.signals = {signal(16, 16, 0.1)};
    d.signals[0].values[5] = std::nan("");
    d.names = {"nan"};
    cases.push_back({"non-finite signal", d, cfg});
  }
  {
    dcsc::Dataset d;
    d.signals = {signal(16, 16, 0.1)};
    d.names = {"a"};
    dcsc::RunConfig big = cfg;
    big.support = {17, 3};
    cases.push_back({"support larger than grid", d, big});
    dcsc::RunConfig nofilt = cfg;
    nofilt.filters = 0;
    cases.push_back({"no filters", d, nofilt});
    dcsc::RunConfig badbeta = cfg;
    badbeta.solver.beta = -1.0;
    cases.push_back({"negative beta", d, badbeta});
  }
  bool ok = true;
  std::printf("{\"errors\": [");
  for (std::size_t i = 0; i < cases.size(); ++i) {
    const char* a = thrown([&] { dcsc::run_csc(cases[i].cfg, cases[i].data); });
    const char* b = thrown([&] { dcsc::cuda::run_csc(cases[i].cfg, cases[i].data); });
    const bool same = std::string(a) == b && std::string(a) != "none";
    ok = ok && same;
    std::printf("%s{\"case\": \"%s\", \"reference\": \"%s\", \"cuda\": \"%s\"}", i ? ", " : "", cases[i].name, a, b);
  }
  std::printf("], \"ok\": %s}\n", ok ? "true" : "false");
  return ok ? 0 : 1;
}

// The reference's own call pattern (pipeline.cpp:221-227): solve_coding once
// per image from OpenMP threads, warm states carried over two sweeps, then
// solve_learning; dcsc::cuda's per-thread cached contexts against the
// reference's sequential calls (FP64, identical iteration counts, <= 1e-9).
static int check_threads() {
  const int N = 12, H = 20, W = 20, K = 4, m = 5;
  std::mt19937_64 rng(7);
  std::vector<dcsc::SignalTensor> xs;
  for (int n = 0; n < N; ++n) {
    dcsc::SignalTensor x({H, W}, 1);
    for (double& v : x.values) v = static_cast<double>(rng() >> 11) * 0x1.0p-53 - 0.5;
    xs.push_back(x);
  }
  dcsc::Dictionary d(K, {m, m}, 1);
  for (double& v : d.values) v = static_cast<double>(rng() >> 11) * 0x1.0p-53 - 0.5;
  dcsc::SolverConfig cfg;
  cfg.beta = 0.1;
  cfg.max_admm = 60;
  std::vector<dcsc::CodingDualState> sa(N), sb(N);
  std::vector<dcsc::SparseMaps> za(N), zb(N);
  std::vector<dcsc::CodingStats> ca(N), cb(N);
  double worst = 0.0;
  bool iters_ok = true;
  for (int sweep = 0; sweep < 2; ++sweep) {
    for (int n = 0; n < N; ++n) za[n] = dcsc::solve_coding(xs[n], d, cfg, sa[n], &ca[n]);
#pragma omp parallel for schedule(dynamic, 1) num_threads(4)
    for (int n = 0; n < N; ++n) zb[n] = dcsc::cuda::solve_coding(xs[n], d, cfg, sb[n], &cb[n]);
    for (int n = 0; n < N; ++n) {
      iters_ok = iters_ok && ca[n].admm_iters == cb[n].admm_iters;
      double zm = 0.0, dz = 0.0;
      for (std::size_t i = 0; i < za[n].values.size(); ++i) {
        zm = std::max(zm, std::abs(za[n].values[i]));
        dz = std::max(dz, std::abs(za[n].values[i] - zb[n].values[i]));
      }
      worst = std::max(worst, dz / std::max(zm, 1e-300));
    }
  }
  dcsc::LearningDualState la, lb;
  const dcsc::Dictionary da = dcsc::solve_learning(xs, za, {m, m}, cfg, la);
  const dcsc::Dictionary db = dcsc::cuda::solve_learning(xs, zb, {m, m}, cfg, lb);
  double dmax = 0.0, dref = 0.0;
  for (std::size_t i = 0; i < da.values.size(); ++i) {
    dmax = std::max(dmax, std::abs(da.values[i] - db.values[i]));
    dref = std::max(dref, std::abs(da.values[i]));
  }
  const bool ok = iters_ok && worst <= 1e-9 && dmax <= 1e-7 * dref;
  std::printf("{\"threads\": 4, \"ok\": %s, \"iters_equal\": %s, \"max_rel_z\": %.3e, \"max_rel_dict\": %.3e}\n",
              ok ? "true" : "false", iters_ok ? "true" : "false", worst, dmax / std::max(dref, 1e-300));
  return ok ? 0 : 1;
}

// usage: dropin_check [outer] [channels]   (channels > 1: Joint mode, TCSC)
//        dropin_check errors               (exception parity on bad inputs)
//        dropin_check threads              (per-image calls from OpenMP threads)
int main(int argc, char** argv) {
  if (argc > 1 && std::string(argv[1]) == "errors") return check_errors();
  if (argc > 1 && std::string(argv[1]) == "threads") return check_threads();
  const int N = 3, H = 20, W = 20, K = 6, m = 5, outer = argc > 1 ? std::atoi(argv[1]) : 3;
  const int J = argc > 2 ? std::atoi(argv[2]) : 1;
  dcsc::Dataset data;
  std::mt19937_64 rng(123);
  for (int n = 0; n < N; ++n) {
    dcsc::SignalTensor x({H, W}, J);
    for (double& v : x.values) v = static_cast<double>(rng() >> 11) * 0x1.0p-53 - 0.5;
    data.signals.push_back(x);
  }
  dcsc::RunConfig cfg;
  cfg.filters = K;
  cfg.support = {m, m};
  cfg.channel_mode = J > 1 ? dcsc::ChannelMode::Joint : dcsc::ChannelMode::Separate;
  cfg.solver.beta = 0.2;
  cfg.solver.max_outer = outer;
  cfg.solver.tol = 1e-300;
  cfg.solver.seed = 17;  // default Global normalisation on both sides
  const dcsc::RunResult a = dcsc::run_csc(cfg, data);
  const dcsc::RunResult b = dcsc::cuda::run_csc(cfg, data);
  double worst = 0.0;
  if (a.trace.rows.size() != b.trace.rows.size()) {
    std::printf("{\"ok\": false, \"reason\": \"trace length\"}\n");
    return 1;
  }
  for (std::size_t i = 0; i < a.trace.rows.size(); ++i) {
    const double ra = a.trace.rows[i].objective.total, rb = b.trace.rows[i].objective.total;
    worst = std::max(worst, std::abs(ra - rb) / std::abs(ra));
    if (a.trace.rows[i].admm_iters != b.trace.rows[i].admm_iters) {
      std::printf("{\"ok\": false, \"reason\": \"admm_iters row %zu: %ld vs %ld\"}\n", i,
                  a.trace.rows[i].admm_iters, b.trace.rows[i].admm_iters);
      return 1;
    }
  }
  double dmax = 0.0, dref = 0.0;
  for (std::size_t i = 0; i < a.dict.values.size(); ++i) {
    dmax = std::max(dmax, std::abs(a.dict.values[i] - b.dict.values[i]));
    dref = std::max(dref, std::abs(a.dict.values[i]));
  }
  const bool ok = worst <= 1e-9 && dmax <= 1e-8 * dref;
  std::printf("{\"ok\": %s, \"channels\": %d, \"rows\": %zu, \"max_rel_objective\": %.3e, \"max_rel_dict\": %.3e}\n",
              ok ? "true" : "false", J, a.trace.rows.size(), worst, dmax / dref);
  return ok ? 0 : 1;
}
