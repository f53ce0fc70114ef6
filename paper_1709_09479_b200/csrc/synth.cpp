// Synthetic BASELINE.json data, host only.
//
// Seeded std::mt19937_64 streams with explicit transforms so the values are
// identical across compilers and machines:
//   uniform  u = (rng() >> 11) * 2^-53                (as pipeline.cpp:131-132)
//   normal   sqrt(-2 ln(1-u1)) cos(2 pi u2)           (Box-Muller, one per pair)
//   laplace  -sgn(u-1/2) ln(1 - 2|u-1/2|)
//   bernoulli [u < p]
// Streams: filters = seed ^ S1; image n maps = mix(seed, 2, n); image n noise =
// mix(seed, 3, n), so images generate independently (in parallel).
// Ground-truth filters ~ N(0,1), unit l2; maps z_nk = Bernoulli(p) Laplace(0,1);
// x_n = sum_k pad(d_k) * z_nk (circular, corner placement of
// spectral.cpp:106-122, accumulation order of objective.cpp:21-35) + N(0, sigma^2),
// then zero-meaned; optionally rounded to FP32 (both arms see the same values).
#include <cmath>
#include <cstdint>
#include <random>
#include <vector>

#include "dcsc_cuda.h"

namespace {

inline double uni(std::mt19937_64& r) { return static_cast<double>(r() >> 11) * 0x1.0p-53; }

inline double normal(std::mt19937_64& r) {
  const double u1 = uni(r), u2 = uni(r);
  return std::sqrt(-2.0 * std::log(1.0 - u1)) * std::cos(6.283185307179586476925286766559 * u2);
}

inline double laplace(std::mt19937_64& r) {
  const double u = uni(r) - 0.5;
  const double s = u < 0 ? -1.0 : (u > 0 ? 1.0 : 0.0);
  return -s * std::log(1.0 - 2.0 * std::fabs(u));
}

inline std::uint64_t mix(std::uint64_t seed, std::uint64_t stream, std::uint64_t idx) {
  std::uint64_t z = seed + 0x9E3779B97F4A7C15ULL * (stream * 0x100000001B3ULL + idx + 1);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

}  // namespace

// Images [n0, n0 + N) of the seeded dataset (each image has its own streams,
// so any range is generated independently of the others).
extern "C" int dcsc_synth_generate_range(int n0, int N, int H, int W, int K, int m, double p, double sigma,
                                         std::uint64_t seed, int round_fp32, double* x, double* d_true) {
  if (n0 < 0 || N < 1 || H < 1 || W < 1 || K < 1 || m < 1 || m > H || m > W) return DCSC_ERR_DIMENSION;
  const int M = m * m;
  std::vector<double> d(static_cast<size_t>(K) * M);
  {
    std::mt19937_64 rf(mix(seed, 1, 0));
    for (int k = 0; k < K; ++k) {
      double sq = 0.0;
      for (int i = 0; i < M; ++i) {
        const double v = normal(rf);
        d[static_cast<size_t>(k) * M + i] = v;
        sq += v * v;
      }
      const double nrm = std::sqrt(sq);
      for (int i = 0; i < M; ++i) d[static_cast<size_t>(k) * M + i] /= nrm;
    }
  }
  if (d_true)
    for (size_t i = 0; i < d.size(); ++i) d_true[i] = d[i];
  const size_t D = static_cast<size_t>(H) * W;
#pragma omp parallel for schedule(dynamic, 1)
  for (int img = 0; img < N; ++img) {
    const std::uint64_t n = static_cast<std::uint64_t>(n0) + static_cast<std::uint64_t>(img);
    std::mt19937_64 rm(mix(seed, 2, n));
    std::mt19937_64 re(mix(seed, 3, n));
    double* xn = x + static_cast<size_t>(img) * D;
    for (size_t i = 0; i < D; ++i) xn[i] = 0.0;
    for (int k = 0; k < K; ++k) {
      const double* dk = d.data() + static_cast<size_t>(k) * M;
      for (int r = 0; r < H; ++r)
        for (int c = 0; c < W; ++c) {
          if (!(uni(rm) < p)) continue;
          const double v = laplace(rm);
          for (int a = 0; a < m; ++a) {
            const int rr = (r + a) % H;
            for (int b = 0; b < m; ++b) xn[static_cast<size_t>(rr) * W + (c + b) % W] += dk[a * m + b] * v;
          }
        }
    }
    double mean = 0.0;
    for (size_t i = 0; i < D; ++i) {
      xn[i] += sigma * normal(re);
      mean += xn[i];
    }
    mean /= static_cast<double>(D);
    for (size_t i = 0; i < D; ++i) {
      const double v = xn[i] - mean;
      xn[i] = round_fp32 ? static_cast<double>(static_cast<float>(v)) : v;
    }
  }
  return DCSC_OK;
}

// The reference bench harness's dataset (bench.cpp:9-21): one mt19937_64
// seeded with `seed`, values u = (rng() >> 11) * 2^-53 in [0, 1), drawn image
// by image in row-major order. x: N*J*H*W.
extern "C" int dcsc_synth_dataset(int N, int J, int H, int W, std::uint64_t seed, double* x) {
  if (N < 1 || J < 1 || H < 1 || W < 1 || !x) return DCSC_ERR_DIMENSION;
  std::mt19937_64 rng(seed);
  const std::size_t total = (std::size_t)N * J * H * W;
  for (std::size_t i = 0; i < total; ++i) x[i] = static_cast<double>(rng() >> 11) * 0x1.0p-53;
  return DCSC_OK;
}

extern "C" int dcsc_synth_generate(int N, int H, int W, int K, int m, double p, double sigma,
                                   std::uint64_t seed, int round_fp32, double* x, double* d_true) {
  return dcsc_synth_generate_range(0, N, H, W, K, m, p, sigma, seed, round_fp32, x, d_true);
}
