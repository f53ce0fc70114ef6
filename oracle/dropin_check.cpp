// Drop-in demonstration (TEST INFRASTRUCTURE): the same reference program calls
// dcsc::run_csc (the reference, CPU) and dcsc::cuda::run_csc (include/dcsc_cuda.hpp
// over the CUDA C-ABI) on identical data and compares the traces and dictionaries.
// Built by oracle/Makefile (target dropin) against the reference headers; run by
// tests/test_dropin_gpu.py. Exit code 0 = within tolerance.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>

#include "dcsc/pipeline.hpp"
#include "dcsc_cuda.hpp"

// usage: dropin_check [outer] [channels]   (channels > 1: Joint mode, TCSC)
int main(int argc, char** argv) {
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
