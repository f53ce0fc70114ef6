// Engine<R, H, W>: host orchestration of the B200 dual-domain CSC path for one
// compiled grid/precision. Included by the per-grid instantiation units
// (inst_*.cu) so the kernel families compile in parallel; the C-ABI lives in
// engine.cu. One Engine keeps every hot-path buffer device-resident; the host
// only makes the discrete decisions the reference makes on scalars (stop tests,
// acceptance, the mu settle test) from FP64 reductions read back per iteration.
#pragma once
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "dcsc_cuda.h"
#include "kernels.cuh"
#include "kernels_cluster.cuh"
#include "kernels_tc.cuh"
#include "tcsc_kernels.cuh"

using namespace dcsc_cuda;
#include "engine_shared.h"

using namespace dcsc_engine;

namespace {

double now_ms() {
  using clock = std::chrono::steady_clock;
  return std::chrono::duration<double, std::milli>(clock::now().time_since_epoch()).count();
}

struct DevMem {
  void* p = nullptr;
  size_t bytes = 0;
  DevMem() = default;
  DevMem(const DevMem&) = delete;
  DevMem& operator=(const DevMem&) = delete;
  ~DevMem() {
    if (p) cudaFree(p);
  }
  void alloc(size_t b) {
    if (p) {
      cudaFree(p);
      p = nullptr;
    }
    bytes = b;
    if (b) CK(cudaMalloc(&p, b));
  }
  template <class T> T* as() const { return static_cast<T*>(p); }
};

void require_finite(const double* v, size_t n, const char* what) {  // types.cpp:26-29
  for (size_t i = 0; i < n; ++i)
    if (!std::isfinite(v[i])) throw NumErr(std::string(what) + " contains a non-finite value");
}

constexpr double kFilterNormTol = 1e-3;  // learning.cpp:14

// Kernel families for the per-launch CUDA-event profiler.
enum Family { kFamCoding = 0, kFamLambda = 1, kFamContract = 2, kFamMask = 3, kFamOther = 4, kFamCount = 5 };

// Circular Gaussian blur (sigma in samples, truncated at 4 sigma) along both
// axes, as pipeline.cpp:26-57 does for local contrast normalisation.
std::vector<double> gaussian_blur(int H, int W, const double* v, double sigma) {
  const int radius = static_cast<int>(std::ceil(4.0 * sigma));
  std::vector<double> ker(2 * radius + 1);
  double ks = 0.0;
  for (int i = -radius; i <= radius; ++i) {
    ker[i + radius] = std::exp(-0.5 * (i * i) / (sigma * sigma));
    ks += ker[i + radius];
  }
  for (double& k : ker) k /= ks;
  std::vector<double> cur(v, v + (size_t)H * W), next(cur.size());
  const int dims[2] = {H, W};
  for (int axis = 0; axis < 2; ++axis) {
    const int n = dims[axis];
    for (int r = 0; r < H; ++r)
      for (int c = 0; c < W; ++c) {
        double acc = 0.0;
        const int c0 = axis == 0 ? r : c;
        for (int i = -radius; i <= radius; ++i) {
          int cc = (c0 + i) % n;
          if (cc < 0) cc += n;
          acc += ker[i + radius] * (axis == 0 ? cur[(size_t)cc * W + c] : cur[(size_t)r * W + cc]);
        }
        next[(size_t)r * W + c] = acc;
      }
    cur.swap(next);
  }
  return cur;
}

// dcsc::normalize (pipeline.cpp:78-121) for one J-channel image: Global uses
// the mean / std of all J*D values, Local runs per channel.
// *degen: the reference's degenerate flag (constant input, pipeline.cpp:90-93, 111-115).
void normalize_image(int mode, int H, int W, const double* in, double* out, int J = 1, bool* degen = nullptr) {
  if (mode == 2 && J > 1) {
    for (int j = 0; j < J; ++j)
      normalize_image(mode, H, W, in + (size_t)j * H * W, out + (size_t)j * H * W, 1, degen);
    return;
  }
  const size_t D = (size_t)H * W * J;  // None / Global act on all J*D values
  if (mode == 0) {
    std::copy(in, in + D, out);
    return;
  }
  if (mode == 1) {
    double m = 0.0;
    for (size_t i = 0; i < D; ++i) m += in[i];
    m /= (double)D;
    double var = 0.0;
    for (size_t i = 0; i < D; ++i) var += (in[i] - m) * (in[i] - m);
    const double sd = std::sqrt(var / (double)D);
    if (sd < 1e-8) {
      std::fill(out, out + D, 0.0);
      if (degen) *degen = true;
      return;
    }
    for (size_t i = 0; i < D; ++i) out[i] = (in[i] - m) / sd;
    return;
  }
  const std::vector<double> lm = gaussian_blur(H, W, in, 3.0);
  std::vector<double> sq(D);
  for (size_t i = 0; i < D; ++i) sq[i] = in[i] * in[i];
  const std::vector<double> ls = gaussian_blur(H, W, sq.data(), 3.0);
  std::vector<double> lsd(D);
  double fl = 0.0;
  for (size_t i = 0; i < D; ++i) {
    lsd[i] = std::sqrt(std::max(ls[i] - lm[i] * lm[i], 0.0));
    fl += lsd[i];
  }
  fl /= (double)D;
  if (fl < 1e-8) {
    for (size_t i = 0; i < D; ++i) out[i] = in[i] - lm[i];
    if (degen) *degen = true;
    return;
  }
  for (size_t i = 0; i < D; ++i) out[i] = (in[i] - lm[i]) / std::max(lsd[i], fl);
}


#ifndef DCSC_KC
#define DCSC_KC 8  // filters per contract_c CTA (v_hat reuse)
#endif

#ifndef DCSC_T128
#define DCSC_T128 512  // threads per CTA of the 128x128 family (experiment knob)
#endif
constexpr int pick_threads(int H, int W) {
  return H * W == 128 * 128 ? DCSC_T128 : (H * W >= 100 * 100 ? 512 : (H * W >= 64 * 64 ? 256 : 128));
}
#ifndef DCSC_T100D
#define DCSC_T100D 512  // threads per CTA of the FP64 100x100 family (experiment knob)
#endif
template <class R>
constexpr int pick_threads_r(int H, int W) {
  return (sizeof(R) == 8 && H * W == 100 * 100) ? DCSC_T100D : pick_threads(H, W);
}

// Kernel family per compiled grid: one CTA per plane (Plane), or a 4-CTA
// cluster per plane (ClusterPlane) when the half spectrum exceeds smem.
template <class R, int H, int W>
struct KernelFamily {
  static constexpr bool cluster = false;
  static constexpr int CL = 1;
  using P = Plane<R, H, W, pick_threads_r<R>(H, W)>;
};
template <>
struct KernelFamily<double, 128, 128> {  // FP64 128x128: 133 KB per plane buffer
  static constexpr bool cluster = true;
  static constexpr int CL = 4;
  using P = ClusterPlane<double, 128, 128, 4, 256>;
};
template <>
struct KernelFamily<float, 256, 256> {
  static constexpr bool cluster = true;
#ifndef DCSC_CL256
#define DCSC_CL256 4
#endif
  static constexpr int CL = DCSC_CL256;
  using P = ClusterPlane<float, 256, 256, CL, (CL == 8 ? 256 : 512)>;
};

template <class R, int H, int W>
class Engine final : public EngineBase {
 public:
  using F = KernelFamily<R, H, W>;
  using P = typename F::P;
  static constexpr bool CLU = F::cluster;
  static constexpr int CLN = F::CL;
  static constexpr int T = P::T;
  using C = cx<R>;
  static constexpr int NB = P::NB, D = P::D, Wh = P::Wh;
  static constexpr int TBV = 256;  // block size of the streaming kernels

  template <class Q = P>
  static constexpr size_t smem_coding() {
    if constexpr (CLU) return SmemCl<Q>::coding; else return Smem<Q>::coding;
  }
  template <class Q = P>
  static constexpr size_t smem_plain() {
    if constexpr (CLU) return SmemCl<Q>::plain; else return Smem<Q>::two;
  }
  template <int MODE>
  static void launch_coding(int G, int cnt, cudaStream_t st, const CodingArgs<R>& a) {
    if constexpr (CLU) {
      if (a.J > 1)
        coding_pass_cl<P, MODE, true><<<dim3(G * CLN, cnt), T, smem_coding(), st>>>(a);
      else
        coding_pass_cl<P, MODE><<<dim3(G * CLN, cnt), T, smem_coding(), st>>>(a);
    } else {
      if (MODE == kPassAdmm && a.J == 2)  // common channel counts: compile-time loops
        coding_pass<P, MODE, true, 2><<<dim3(G, cnt), T, smem_coding(), st>>>(a);
      else if (MODE == kPassAdmm && a.J == 3)
        coding_pass<P, MODE, true, 3><<<dim3(G, cnt), T, smem_coding(), st>>>(a);
      else if (MODE == kPassAdmm && a.J == 4)
        coding_pass<P, MODE, true, 4><<<dim3(G, cnt), T, smem_coding(), st>>>(a);
      else if (a.J > 1)
        coding_pass<P, MODE, true><<<dim3(G, cnt), T, smem_coding(), st>>>(a);
      else
        coding_pass<P, MODE><<<dim3(G, cnt), T, smem_coding(), st>>>(a);
    }
  }
  // Tensor-core spatial coding iteration (kernels_tc.cuh): FP32 planes whose
  // rows split into 128-pixel tiles, 11 x 11 supports, K <= 128, J = 1.
  // The pass works on row-major u planes: the cluster family's own layout; the
  // single-CTA family (column-major pixel pairs) runs it on a row-major copy
  // (tu_) converted once before and after each coding call.
  static constexpr int kTcRB = H % 16 == 0 ? 16 : 20;  // band rows (C2's 100 x 100: 20)
  static constexpr bool kTcFamily = std::is_same<R, float>::value && H % kTcRB == 0 &&
                                    ((W % 128 == 0 && (W / 128 == 1 || (W / 128) % 2 == 0)) || W == 64 ||
                                     (W > 64 && W < 128 && W % 4 == 0));
  // compiled support (square) and filter-slot counts per family: 64 x 64 (C4) runs
  // 7 x 7 supports with 32 / 64 filter slots, the wider grids 11 x 11 with 64 / 128
  // (single-row families 80 / 100: 112 slots for C2's K = 100)
  static constexpr int kTcM = W == 64 ? 7 : 11, kTcKFa = W == 64 ? 32 : 64,
                       kTcKFb = W == 64 ? 64 : ((W > 64 && W < 128) ? 112 : 128);
  // epilogue warps: 16 (two per TMEM lane quarter) where the per-tile epilogue is long (256 x 256 with
  // 128 filter slots, the single-row 100 / 80 families with 112), 8 at 128 x 128 and 64 x 64 (measured)
#ifdef DCSC_TC_EW
  static constexpr int kTcEW = DCSC_TC_EW;
#else
  static constexpr int kTcEW = (W == 128 || W == 64) ? 8 : 16;
#endif
  template <int KF>
  using TG = TcGeom<H, W, KF, kTcM, kTcM, kTcRB, kTcEW>;
  template <int KF>
  static void set_tc_attr() {
    const int sm = (int)TG<KF>::smem;
    CK(cudaFuncSetAttribute((const void*)coding_pass_tc<TG<KF>, true, false>,
                            cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
    CK(cudaFuncSetAttribute((const void*)coding_pass_tc<TG<KF>, true, true>,
                            cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
    CK(cudaFuncSetAttribute((const void*)coding_pass_tc<TG<KF>, false, false>,
                            cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
    CK(cudaFuncSetAttribute((const void*)coding_pass_tc<TG<KF>, false, true>,
                            cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
  }
  template <int KF>
  void launch_tc(int grid, const TcArgs& a, cudaStream_t st) {
    constexpr size_t sm = TG<KF>::smem;
    const bool full = a.K == KF, t0 = a.theta0 != nullptr;
    if (full && !t0)
      coding_pass_tc<TG<KF>, true, false><<<grid, TG<KF>::THREADS, sm, st>>>(a);
    else if (full)
      coding_pass_tc<TG<KF>, true, true><<<grid, TG<KF>::THREADS, sm, st>>>(a);
    else if (!t0)
      coding_pass_tc<TG<KF>, false, false><<<grid, TG<KF>::THREADS, sm, st>>>(a);
    else
      coding_pass_tc<TG<KF>, false, true><<<grid, TG<KF>::THREADS, sm, st>>>(a);
  }
  // persistent pipelined r2c / c2r (SmemPipe) when the staging buffer fits and
  // the planes are 16-byte aligned storage-precision planes: grid = resident slots
  static int pipe_grid(const void* fn, size_t smem, int count) {
    int dev = 0, sms = 148, per = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, T, smem) != cudaSuccess || per < 1) per = 1;
    cudaGetLastError();
    return std::max(1, std::min(count, sms * per));
  }
  static bool aligned16(const void* p, size_t stride_bytes) {
    return (reinterpret_cast<uintptr_t>(p) % 16) == 0 && stride_bytes % 16 == 0;
  }
  template <class SRC>
  static void launch_r2c(int count, cudaStream_t st, const SRC* src, size_t ss, C* dst, size_t ds, const C* tw,
                         int* live, int live_mod) {
    if constexpr (CLU) {
      // persistent: as many clusters as fit at once, each walking planes
      static int slots = 0;
      if (!slots) {
        cudaLaunchConfig_t lc{};
        lc.gridDim = dim3(CLN, 1, 1);
        lc.blockDim = dim3(T, 1, 1);
        lc.dynamicSmemBytes = smem_plain();
        int ncl = 0;
        slots = (cudaOccupancyMaxActiveClusters(&ncl, (void*)r2c_planes_cl<P, SRC>, &lc) == cudaSuccess && ncl > 0)
                    ? ncl : 32;
        cudaGetLastError();
      }
      const int g = std::max(1, std::min(count, slots));
      r2c_planes_cl<P, SRC><<<g * CLN, T, smem_plain(), st>>>(src, ss, dst, ds, tw, live, live_mod, count);
    } else {
      if constexpr (std::is_same<SRC, R>::value && SmemPipe<P>::r2c_ok) {
        if (!std::getenv("DCSC_NO_FFT_PIPE") && aligned16(src, ss * sizeof(R))) {
          constexpr size_t sm = SmemPipe<P>::r2c;
          const int g = pipe_grid((const void*)r2c_planes_pipe<P>, sm, count);
          r2c_planes_pipe<P><<<g, T, sm, st>>>(src, ss, dst, ds, tw, live, live_mod, count);
          return;
        }
      }
      r2c_planes<P, SRC><<<count, T, smem_plain(), st>>>(src, ss, dst, ds, tw, live, live_mod);
    }
  }
  template <class DST>
  static void launch_c2r(int count, cudaStream_t st, const C* src, size_t ss, DST* dst, size_t ds, const C* tw) {
    if constexpr (CLU) {
      static int slots = 0;
      if (!slots) {
        cudaLaunchConfig_t lc{};
        lc.gridDim = dim3(CLN, 1, 1);
        lc.blockDim = dim3(T, 1, 1);
        lc.dynamicSmemBytes = smem_plain();
        int ncl = 0;
        slots = (cudaOccupancyMaxActiveClusters(&ncl, (void*)c2r_planes_cl<P, DST>, &lc) == cudaSuccess && ncl > 0)
                    ? ncl : 32;
        cudaGetLastError();
      }
      const int g = std::max(1, std::min(count, slots));
      c2r_planes_cl<P, DST><<<g * CLN, T, smem_plain(), st>>>(src, ss, dst, ds, tw, nullptr, count);
    } else {
      if constexpr (std::is_same<DST, R>::value && SmemPipe<P>::c2r_ok) {
        if (!std::getenv("DCSC_NO_FFT_PIPE") && aligned16(src, ss * sizeof(C)) && aligned16(dst, ds * sizeof(R))) {
          constexpr size_t sm = SmemPipe<P>::c2r;
          const int g = pipe_grid((const void*)c2r_planes_pipe<P>, sm, count);
          c2r_planes_pipe<P><<<g, T, sm, st>>>(src, ss, dst, ds, tw, count);
          return;
        }
      }
      c2r_planes<P, DST><<<count, T, smem_plain(), st>>>(src, ss, dst, ds, tw, nullptr);
    }
  }
  static void launch_filters(int K, cudaStream_t st, const double* d, int mh, int mw, C* dst, const C* tw) {
    if constexpr (CLU)
      r2c_filters_cl<P><<<K * CLN, T, smem_plain(), st>>>(d, mh, mw, dst, tw);
    else
      r2c_filters<P><<<K, T, smem_plain(), st>>>(d, mh, mw, dst, tw);
  }
  static void launch_mask(int K, cudaStream_t st, const C* c, C* phat, double* d_out, const int* live,
                          const double* mu, int mh, int mw, int mode, const C* tw, const int* done) {
    if constexpr (CLU)
      mask_step_cl<P><<<K * CLN, T, smem_plain(), st>>>(c, phat, d_out, live, mu, mh, mw, mode, tw, done);
    else
      mask_step<P><<<K, T, smem_plain(), st>>>(c, phat, d_out, live, mu, mh, mw, mode, tw, done);
  }
  static void set_attributes() {
    auto big = [](const void* fn, size_t bytes) {
      if (bytes > 48 * 1024) CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    };
    if constexpr (kTcFamily) {
      set_tc_attr<kTcKFa>();
      set_tc_attr<kTcKFb>();
    }
    if constexpr (CLU) {
      big((const void*)coding_pass_cl<P, kPassAdmm>, smem_coding());
      big((const void*)coding_pass_cl<P, kPassPrologue>, smem_coding());
      big((const void*)coding_pass_cl<P, kPassObjective>, smem_coding());
      big((const void*)coding_pass_cl<P, kPassMaps>, smem_coding());
      big((const void*)coding_pass_cl<P, kPassAdmm, true>, smem_coding());
      big((const void*)coding_pass_cl<P, kPassPrologue, true>, smem_coding());
      big((const void*)coding_pass_cl<P, kPassObjective, true>, smem_coding());
      big((const void*)coding_pass_cl<P, kPassMaps, true>, smem_coding());
      big((const void*)r2c_planes_cl<P, R>, smem_plain());
      big((const void*)r2c_planes_cl<P, double>, smem_plain());
      big((const void*)c2r_planes_cl<P, R>, smem_plain());
      big((const void*)c2r_planes_cl<P, double>, smem_plain());
      big((const void*)r2c_filters_cl<P>, smem_plain());
      big((const void*)mask_step_cl<P>, smem_plain());
    } else {
      big((const void*)coding_pass<P, kPassAdmm>, smem_coding());
      big((const void*)coding_pass<P, kPassPrologue>, smem_coding());
      big((const void*)coding_pass<P, kPassObjective>, smem_coding());
      big((const void*)coding_pass<P, kPassMaps>, smem_coding());
      big((const void*)coding_pass<P, kPassAdmm, true>, smem_coding());
      big((const void*)coding_pass<P, kPassAdmm, true, 2>, smem_coding());
      big((const void*)coding_pass<P, kPassAdmm, true, 3>, smem_coding());
      big((const void*)coding_pass<P, kPassAdmm, true, 4>, smem_coding());
      big((const void*)coding_pass<P, kPassPrologue, true>, smem_coding());
      big((const void*)coding_pass<P, kPassObjective, true>, smem_coding());
      big((const void*)coding_pass<P, kPassMaps, true>, smem_coding());
      big((const void*)r2c_planes<P, R>, smem_plain());
      big((const void*)r2c_planes<P, double>, smem_plain());
      big((const void*)c2r_planes<P, R>, smem_plain());
      big((const void*)c2r_planes<P, double>, smem_plain());
      big((const void*)r2c_filters<P>, smem_plain());
      big((const void*)mask_step<P>, smem_plain());
      if constexpr (SmemPipe<P>::r2c_ok) big((const void*)r2c_planes_pipe<P>, SmemPipe<P>::r2c);
      if constexpr (SmemPipe<P>::c2r_ok) big((const void*)c2r_planes_pipe<P>, SmemPipe<P>::c2r);
    }
  }

  explicit Engine(const dcsc_cuda_opts& o) : o_(o), cfg_(o.cfg) {
    N_ = o.n_images;
    K_ = o.filters;
    J_ = std::max(1, o.channels);
    if (J_ > kMaxChannels) throw DimErr("at most " + std::to_string(kMaxChannels) + " channels are supported");
    if constexpr (CLU) {  // the cropped support must sit in the first rank's row block
      if (o.support_h > P::ROWS)
        throw DimErr("filter support taller than " + std::to_string(P::ROWS) + " rows on the cluster grid family");
    }
    mh_ = o.support_h;
    mw_ = o.support_w;
    M_ = mh_ * mw_;
    CK(cudaSetDevice(o.device));
    CK(cudaStreamCreateWithFlags(&st_, cudaStreamNonBlocking));
    CK(cudaMallocHost(&pin_, 1 << 20));
    setup_attributes();
    // Filter groups per image: a CTA runs kpg filters; pick G minimising the
    // makespan ceil(N*G / slots) * (ceil(K/G) + 1): wave quantisation plus a
    // per-CTA overhead of about one filter's worth (partial spectrum write and
    // re-read, twiddles, the epilogue). Ties -> fewer groups.
    {
      int sms = 148, per_sm = 1;
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, o.device);
      long slots;
      if constexpr (CLU) {
        // clusters must sit inside one GPC: ask the runtime how many fit at
        // once (4-CTA clusters strand SMs on GPCs whose SM count is not a
        // multiple of 4) instead of assuming sms / CLN
        slots = sms / CLN;
        cudaLaunchConfig_t lc{};
        lc.gridDim = dim3(CLN, 1, 1);
        lc.blockDim = dim3(T, 1, 1);
        lc.dynamicSmemBytes = smem_coding();
        int ncl = 0;
        if (cudaOccupancyMaxActiveClusters(&ncl, (void*)coding_pass_cl<P, kPassAdmm>, &lc) == cudaSuccess && ncl > 0)
          slots = ncl;
        cudaGetLastError();
      } else {
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, coding_pass<P, kPassAdmm>, T, smem_coding()));
        slots = (long)sms * std::max(per_sm, 1);
      }
      long best = -1;
      int bestG = 1;
      for (int G = 1; G <= K_; ++G) {
        const int kpg = (K_ + G - 1) / G;
        if ((K_ + kpg - 1) / kpg != G) continue;  // G must be realisable
        const long waves = ((long)N_ * G + slots - 1) / slots;
        const long span = waves * (kpg + 1);
        if (best < 0 || span < best) {
          best = span;
          bestG = G;
        }
      }
      if (const char* e = std::getenv("DCSC_GROUPS")) {  // experiment override
        const int g = std::atoi(e);
        if (g >= 1 && g <= K_) bestG = g;
      }
      kpg_ = (K_ + bestG - 1) / bestG;
      G_ = (K_ + kpg_ - 1) / kpg_;
      if (std::getenv("DCSC_VERBOSE"))
        std::fprintf(stderr, "dcsc: N=%d K=%d slots=%ld groups G=%d (%d filters per CTA)\n", N_, K_, slots, G_, kpg_);
    }
    // twiddles (forward roots) in long double, rounded once
    std::vector<C> tw(P::TW_LEN);
    fill_twiddles<P>(tw.data());
    dtw_.alloc(sizeof(C) * P::TW_LEN);
    CK(cudaMemcpy(dtw_.p, tw.data(), sizeof(C) * P::TW_LEN, cudaMemcpyHostToDevice));

    const size_t nD = (size_t)N_ * D, nNB = (size_t)N_ * NB;
    x_.alloc(sizeof(R) * nD * J_);                    // N x J x D
    xhat_.alloc(sizeof(C) * nNB * J_);                // J x N x NB (channel-major)
    dhat_.alloc(sizeof(C) * (size_t)J_ * K_ * NB);    // J x K x NB (channel-major)
    dcand_.alloc(sizeof(C) * (size_t)J_ * K_ * NB);
    if constexpr (CLU) {
      if (J_ == 1) dhat_rb_.alloc((size_t)K_ * CLN * P::buffer_bytes);  // rank-blocked d_hat (cl_rank_block)
    }
    sigma_.alloc(sizeof(R) * NB);
    u_.alloc(sizeof(R) * nD * K_);
    maps_.alloc(sizeof(R) * nD * K_);
    lamhat_.alloc(sizeof(C) * nNB * J_);              // N x J x NB
    lam_.alloc(sizeof(R) * nD * J_);                  // N x J x D
    if (J_ > 1) {
      ginv_.alloc(sizeof(C) * (size_t)NB * J_ * J_);
      what_.alloc(sizeof(C) * nNB * K_);
    }
    part_.alloc(sizeof(C) * (size_t)N_ * G_ * NB);
    sums_.alloc(sizeof(double) * (size_t)N_ * G_ * CLN * kSums);
    conv_.alloc(sizeof(int) * N_);
    cnt_.alloc(sizeof(unsigned) * N_);
    CK(cudaMemset(cnt_.p, 0, cnt_.bytes));
    img_.alloc(sizeof(ImageAdmm) * N_);
    dual_.alloc(sizeof(double) * N_);
    infeas_.alloc(sizeof(double) * N_);
    resc_.alloc(sizeof(int) * N_);
    odata_.alloc(sizeof(double) * N_);
    ol1_.alloc(sizeof(double) * N_);
    accept_.alloc(sizeof(int) * N_);
    gam_.alloc(sizeof(C) * nNB * J_);                 // J x N x NB
    r_.alloc(sizeof(C) * nNB);
    p_.alloc(sizeof(C) * nNB);
    ap_.alloc(sizeof(C) * nNB);
    cvec_.alloc(sizeof(C) * (size_t)K_ * NB);
    // contract_c splits the image sum only as far as needed to fill the GPU
    // (~4 CTAs of 256 threads per SM): every split adds a K x NB FP64 partial
    // plane written and re-read per CG apply (C3: 1 GB at 16 splits)
    {
      int sms = 148;
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, o.device);
      const long base = (long)((NB + TBV - 1) / TBV) * ((K_ + DCSC_KC - 1) / DCSC_KC);
      const double want = std::max(1.0, 4.0 * sms / (double)base);
      const long p2 = 1L << (int)std::lround(std::log2(want));  // nearest power of two (measured: C4 16 > 17)
      csplit_ = (int)std::max(1L, std::min({p2, 64L, (long)N_}));
      if (const char* e = std::getenv("DCSC_CSPLIT")) {  // experiment override
        const int v = std::atoi(e);
        if (v >= 1 && v <= std::min(64, N_)) csplit_ = v;
      }
    }
    cpart_.alloc(sizeof(double2) * (size_t)csplit_ * K_ * NB);
    phat_.alloc(sizeof(C) * (size_t)K_ * NB);
    live_.alloc(sizeof(int) * K_);
    dmu_.alloc(sizeof(double) * K_);
    dwk_.alloc(sizeof(double) * K_);
    dd_.alloc(sizeof(double) * (size_t)K_ * M_);
    ddict_.alloc(sizeof(double) * (size_t)J_ * K_ * M_);
    cg_.alloc(sizeof(CgState));
    cgcnt_.alloc(sizeof(unsigned) * 2);
    {
      int sms = 148;
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, o.device);
      fused_rows_ = 8 * sms;  // blocks of a fused CG launch: ~8 resident x 256 threads per SM
    }
    no_cg_fuse_ = std::getenv("DCSC_NO_CG_FUSE") != nullptr;
    CK(cudaMemsetAsync(cgcnt_.p, 0, cgcnt_.bytes, st_));
    hred_.alloc(sizeof(double) * std::max(64, K_ + 8));
    tiles_ = (NB + TBV - 1) / TBV;
    const size_t vec_blocks = (nNB + TBV - 1) / TBV;
    accept_chunks_ = std::max(1, std::min(64, (int)((size_t)K_ * D / (TBV * 8))));
    const size_t np = std::max({(size_t)N_ * tiles_, vec_blocks, (size_t)N_ * accept_chunks_});
    partial_.alloc(sizeof(double) * np);
    partial2_.alloc(sizeof(double) * (size_t)N_ * accept_chunks_);
    l0_.alloc(sizeof(unsigned long long) * (size_t)N_ * accept_chunks_);
    device_bytes = x_.bytes + xhat_.bytes + dhat_.bytes + dcand_.bytes + sigma_.bytes + u_.bytes +
                   maps_.bytes + lamhat_.bytes + lam_.bytes + part_.bytes + sums_.bytes + gam_.bytes +
                   3 * r_.bytes + cvec_.bytes + phat_.bytes + partial_.bytes + ginv_.bytes + what_.bytes +
                   dhat_rb_.bytes;
    if constexpr (kTcFamily) {
      // DCSC_TC: 0 = FFT pass, 1 = tensor-core pass whenever it applies; unset =
      // tensor-core pass for coding calls with at least two work items per SM
      // (smaller batches leave SMs idle and the FFT pass wins)
      const char* e = std::getenv("DCSC_TC");
      tc_force_ = e && e[0] == '1';
      tc_ = J_ == 1 && mh_ == kTcM && mw_ == kTcM && K_ <= kTcKFb && !(e && e[0] == '0');
      if (tc_) {
        using G = TG<kTcKFb>;  // band geometry does not depend on the filter count
        tc_kf_ = K_ <= kTcKFa ? kTcKFa : kTcKFb;
        tlam16_.alloc(sizeof(uint32_t) * (size_t)N_ * D);
        tlscale_.alloc(sizeof(float) * (size_t)N_);
        tdsplit_.alloc((size_t)2 * tc_kf_ * G::TP * 2);
        tspart_.alloc(sizeof(float) * (size_t)N_ * G::NBANDS * G::SR * W);
        tbsums_.alloc(sizeof(double) * (size_t)N_ * G::NBANDS * kSums);
        tupd_.alloc(sizeof(int) * (size_t)N_);
        tzmax_.alloc(sizeof(float) * (size_t)N_ * G::NBANDS * G::TPI * 4 * G::HV);
        if (!CLU) tu_.alloc(sizeof(float) * (size_t)N_ * K_ * D);
        device_bytes += tlam16_.bytes + tlscale_.bytes + tdsplit_.bytes + tspart_.bytes + tbsums_.bytes + tu_.bytes +
                        tzmax_.bytes;
        CK(cudaDeviceGetAttribute(&tc_grid_, cudaDevAttrMultiProcessorCount, o.device));
        // TMA map of u as [N*K planes][D pixels] FP32, box 16 planes x 128 pixels
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult qr;
        CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr));
        if (!fn || qr != cudaDriverEntryPointSuccess) throw std::runtime_error("cuTensorMapEncodeTiled unavailable");
        const cuuint64_t gdim[2] = {(cuuint64_t)D, (cuuint64_t)N_ * K_};
        const cuuint64_t gstr[1] = {(cuuint64_t)D * sizeof(float)};
        const cuuint32_t box[2] = {128u, 16u}, estr[2] = {1u, 1u};
        const CUresult cr = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn)(
            &tc_umap_, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, CLU ? u_.p : tu_.p, gdim, gstr, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (cr != CUDA_SUCCESS) throw std::runtime_error("cuTensorMapEncodeTiled failed: " + std::to_string((int)cr));
        CK(cudaStreamCreateWithFlags(&st2_, cudaStreamNonBlocking));
        coding_path = tc_use(N_) ? 1 : 0;
        if (std::getenv("DCSC_VERBOSE"))
          std::fprintf(stderr, "dcsc: tensor-core coding pass available (KF=%d), used for all %d images: %d\n", tc_kf_,
                       N_, coding_path);
      }
    }
    CK(cudaMemsetAsync(u_.p, 0, u_.bytes, st_));
    CK(cudaMemsetAsync(maps_.p, 0, maps_.bytes, st_));
    CK(cudaMemsetAsync(lam_.p, 0, lam_.bytes, st_));
    CK(cudaMemsetAsync(gam_.p, 0, gam_.bytes, st_));
    CK(cudaMemsetAsync(x_.p, 0, x_.bytes, st_));
    CK(cudaMemsetAsync(xhat_.p, 0, xhat_.bytes, st_));
    dict_.assign((size_t)K_ * J_ * M_, 0.0);
    u_zero_.assign(N_, 1);
    mu_.assign(K_, 1.0);
    xnorm2_.assign(N_, 0.0);
    xnorm2c_.assign((size_t)N_ * J_, 0.0);
    xh_ch_ = xhat_.as<C>();
    gam_ch_ = gam_.as<C>();
    CK(cudaStreamSynchronize(st_));
  }

  ~Engine() override {
    for (auto& e : evpool_) cudaEventDestroy(e);
    for (auto& e : marks_)
      if (e) cudaEventDestroy(e);
    if (pin_) cudaFreeHost(pin_);
    if (xstage_) cudaFreeHost(xstage_);
    if (st_) cudaStreamDestroy(st_);
    if (st2_) cudaStreamDestroy(st2_);
  }

  // ------------------------------------------------------------ launches
  // per-launch profiling events come from a pool reused across profiling
  // windows (creating two events per launch costs microseconds of host time,
  // which shows up in wall-clock traces of launch-dense phases)
  cudaEvent_t pooled_event() {
    if (evused_ == evpool_.size()) {
      cudaEvent_t e;
      CK(cudaEventCreate(&e));
      evpool_.push_back(e);
    }
    return evpool_[evused_++];
  }
  template <class F>
  void launch(int fam, F&& f, cudaStream_t s = nullptr) {
    if (!s) s = st_;
    cudaEvent_t a = nullptr, b = nullptr;
    const bool prof = profiling_ == 1 || (profiling_ >= 2 && fam == kFamCoding) || (profiling_ == 3 && fam == kFamContract);
    if (prof) {
      a = pooled_event();
      b = pooled_event();
      CK(cudaEventRecord(a, s));
    }
    f();
    CK(cudaGetLastError());
    if (prof) {
      CK(cudaEventRecord(b, s));
      prof_.push_back({fam, a, b});
    }
    ++launches;
  }

  void setup_attributes() { set_attributes(); }

  CodingArgs<R> cargs(const C* dhat, int n_off) {
    CodingArgs<R> a;
    a.dhat = dhat;
    a.J = J_;
    a.what = what_.as<C>() ? what_.as<C>() + (size_t)n_off * K_ * NB : nullptr;
    a.u = u_.as<R>() + (size_t)n_off * K_ * D;
    a.maps = maps_.as<R>() + (size_t)n_off * K_ * D;
    a.part = part_.as<C>() + (size_t)n_off * G_ * NB;
    a.sums = sums_.as<double>() + (size_t)n_off * G_ * CLN * kSums;
    a.conv = conv_.as<int>() + n_off;
    a.lamhat = lamhat_.as<C>() + (size_t)n_off * J_ * NB;
    a.K = K_;
    a.G = G_;
    a.kpg = kpg_;
    a.rho = R(cfg_.rho);
    a.beta = R(cfg_.beta);
    a.tw = dtw_.as<C>();
    a.cnt = cnt_.as<unsigned>() + n_off;
    a.conv_w = conv_.as<int>() + n_off;
    a.xhat = xhat_.as<C>() + (size_t)n_off * NB;
    a.sigma = sigma_.as<R>();
    a.lamhat_w = lamhat_.as<C>() + (size_t)n_off * J_ * NB;
    a.img = img_.as<ImageAdmm>() + n_off;
    a.dhat_rb = (dhat == dhat_.as<C>() && dhat_rb_.p) ? dhat_rb_.as<C>() : nullptr;
    a.iter = 0;
    a.is_last = 0;
    a.theta0 = use_theta0_ ? theta0_.as<R>() + (size_t)n_off * K_ * D : nullptr;
    return a;
  }

  template <int MODE>
  void coding_launch(const C* dhat, int n0, int cnt, int iter = 0, int is_last = 0) {
    CodingArgs<R> a = cargs(dhat, n0);
    a.iter = iter;
    a.is_last = is_last;
    launch(MODE == kPassAdmm ? kFamCoding : kFamOther, [&] { launch_coding<MODE>(G_, cnt, st_, a); });
  }

  // single-CTA family: u planes of images [n0, n0 + cnt) between the column-major
  // pair layout (u_) and the row-major copy the tensor-core pass works on (tu_)
  void tc_convert_u(int n0, int cnt, bool to_rows) {
    if constexpr (kTcFamily && !CLU) {
      const long planes = (long)cnt * K_;
      for (long p0 = 0; p0 < planes; p0 += 32768) {  // gridDim.z <= 65535
        const int np = (int)std::min(32768L, planes - p0);
        float2* u2 = reinterpret_cast<float2*>(u_.as<float>() + ((size_t)n0 * K_ + p0) * D);
        float2* t2 = reinterpret_cast<float2*>(tu_.as<float>() + ((size_t)n0 * K_ + p0) * D);
        launch(kFamOther, [&] {
          if (to_rows)
            tc_pair_transpose<true><<<dim3((H + 31) / 32, (W / 2 + 31) / 32, np), dim3(32, 8), 0, st_>>>(
                u2, t2, H, W / 2);
          else
            tc_pair_transpose<false><<<dim3((W / 2 + 31) / 32, (H + 31) / 32, np), dim3(32, 8), 0, st_>>>(
                t2, u2, H, W / 2);
        });
      }
    }
  }
  // max |z/rho| per warp-tile of the stored u: the pass's bound for W's f16 scale
  void tc_zmax(int n0, int cnt) {
    if constexpr (kTcFamily) {
      using G = TG<kTcKFb>;
      launch(kFamOther, [&] {
        tc_zmax_init<G><<<dim3(G::NBANDS * G::TPI, cnt), 128, 0, st_>>>(
            (CLU ? u_.as<float>() : tu_.as<float>()) + (size_t)n0 * K_ * D,
            tzmax_.as<float>() + (size_t)n0 * G::NBANDS * G::TPI * 4 * G::HV, K_, (float)cfg_.beta);
      });
    }
  }
  bool tc_use(int cnt) const {
    if constexpr (kTcFamily) {
      return tc_ && (tc_force_ || (long)cnt * TG<kTcKFb>::NBANDS >= 2L * tc_grid_);
    }
    return false;
  }
  // lambda_hat -> spatial lambda -> scaled f16 hi / lo planes for the tensor-core pass
  void tc_lambda_spatial(int n0, int cnt, cudaStream_t s = nullptr) {
    if constexpr (kTcFamily) {
      if (!s) s = st_;
      launch(kFamOther, [&] {
        launch_c2r<R>(cnt, s, lamhat_.as<C>() + (size_t)n0 * NB, NB, lam_.as<R>() + (size_t)n0 * D, D, dtw_.as<C>());
      }, s);
      launch(kFamLambda, [&] {
        tc_lam_split<D><<<cnt, 512, 0, s>>>(lam_.as<R>() + (size_t)n0 * D, tlam16_.as<uint32_t>() + (size_t)n0 * D,
                                            tlscale_.as<float>() + n0);
      }, s);
    }
  }
  // One ADMM iteration of images [n0, n0 + cnt) on the tensor-core path:
  // spatial pass (t, prox, s = sum_k d_k * w_k) -> band sums -> DFT(s) ->
  // stop test + lambda_hat (lambda_update, coding.cpp:264-283, :25-37) ->
  // spatial lambda for the next iteration.
  void tc_iteration(int n0, int cnt, int it, bool last, cudaStream_t st = nullptr) {
    if constexpr (kTcFamily) {
      if (!st) st = st_;
      using G = TG<kTcKFb>;
      TcArgs a;
      a.lam16 = tlam16_.as<uint32_t>() + (size_t)n0 * D;
      a.lam_scale = tlscale_.as<float>() + n0;
      a.dsplit = tdsplit_.as<__half>();
      a.d_scale = tc_dscale_;
      a.u = (CLU ? u_.as<float>() : tu_.as<float>()) + (size_t)n0 * K_ * D;
      a.theta0 = use_theta0_ ? theta0_.as<float>() + (size_t)n0 * K_ * D : nullptr;
      a.spart = tspart_.as<float>() + (size_t)n0 * G::NBANDS * G::SR * W;
      a.bsums = tbsums_.as<double>() + (size_t)n0 * G::NBANDS * kSums;
      a.conv = conv_.as<int>() + n0;
      a.zmax = tzmax_.as<float>() + (size_t)n0 * G::NBANDS * G::TPI * 4 * G::HV;
      a.tbound = tc_tbound_;
      a.N = cnt;
      a.K = K_;
      a.rho = (float)cfg_.rho;
      a.beta = (float)cfg_.beta;
      a.umap = tc_umap_;
      a.plane0 = n0 * K_;
      const int grid = std::min(tc_grid_, cnt * G::NBANDS);
      launch(kFamCoding, [&] {
        if (tc_kf_ == kTcKFa)
          launch_tc<kTcKFa>(grid, a, st);
        else
          launch_tc<kTcKFb>(grid, a, st);
      }, st);
      R* s = lam_.as<R>() + (size_t)n0 * D;          // s reuses the spatial lambda planes
      C* spec = part_.as<C>() + (size_t)n0 * NB;      // one partial spectrum per image (G = 1)
      double* sm1 = sums_.as<double>() + (size_t)n0 * kSums;
      int* upd = tupd_.as<int>() + n0;
      launch(kFamLambda, [&] {
        tc_band_reduce<G><<<dim3(16, cnt), 256, 0, st>>>(a.spart, a.bsums, conv_.as<int>() + n0, s,
                                                        img_.as<ImageAdmm>() + n0, upd, it, last ? 1 : 0);
      }, st);
      (void)sm1;
      if (last) return;
      launch(kFamOther, [&] {
        launch_r2c<R>(cnt, st, s, D, spec, NB, dtw_.as<C>(), nullptr, 1);
      }, st);
      launch(kFamLambda, [&] {
        tc_lambda_apply<R><<<dim3(32, cnt), 256, 0, st>>>(spec, xhat_.as<C>() + (size_t)n0 * NB, sigma_.as<R>(),
                                                         lamhat_.as<C>() + (size_t)n0 * NB, upd, NB, R(cfg_.rho));
      }, st);
      tc_lambda_spatial(n0, cnt, st);
    }
  }

  void r2c(const void* src, bool src_double, size_t src_stride, C* dst, size_t dst_stride, int count,
           int* live = nullptr, int live_mod = 1) {
    if (count <= 0) return;
    launch(kFamOther, [&] {
      if (src_double)
        launch_r2c<double>(count, st_, static_cast<const double*>(src), src_stride, dst, dst_stride, dtw_.as<C>(),
                           live, live_mod);
      else
        launch_r2c<R>(count, st_, static_cast<const R*>(src), src_stride, dst, dst_stride, dtw_.as<C>(), live,
                      live_mod);
    });
  }

  template <class DST>
  void c2r(const C* src, size_t src_stride, DST* dst, size_t dst_stride, int count) {
    if (count <= 0) return;
    launch(kFamOther, [&] { launch_c2r<DST>(count, st_, src, src_stride, dst, dst_stride, dtw_.as<C>()); });
  }

  // host dictionary K x J x M (Dictionary::filter(k, j), types.cpp:60-68) ->
  // device spectra J x K x NB (channel-major: channel j's K planes contiguous)
  void upload_dict_spectra(const double* d, C* dst) {
    const double* src = d;
    if (J_ > 1) {
      dstage_.resize((size_t)J_ * K_ * M_);
      for (int k = 0; k < K_; ++k)
        for (int j = 0; j < J_; ++j)
          std::copy(d + ((size_t)k * J_ + j) * M_, d + ((size_t)k * J_ + j + 1) * M_,
                    dstage_.data() + ((size_t)j * K_ + k) * M_);
      src = dstage_.data();
    }
    CK(cudaMemcpyAsync(ddict_.p, src, sizeof(double) * J_ * K_ * M_, cudaMemcpyHostToDevice, st_));
    launch(kFamOther, [&] { launch_filters(J_ * K_, st_, ddict_.as<double>(), mh_, mw_, dst, dtw_.as<C>()); });
    CK(cudaStreamSynchronize(st_));  // dstage_ is reused
  }

  // ------------------------------------------------------------ API
  void set_signals(const double* x) override {
    const size_t nD = (size_t)N_ * J_ * D;
    // host side parallel over images: validate, normalise (pipeline.cpp:78-121),
    // round to the storage precision into pinned staging, per-image (and
    // per-channel) norms of the stored values (what the oracle sees)
    int bad = 0;
#pragma omp parallel for reduction(| : bad)
    for (long i = 0; i < (long)nD; ++i) bad |= !std::isfinite(x[i]);
    if (bad) throw NumErr("signal contains a non-finite value");
    if (!xstage_ || xstage_bytes_ < sizeof(R) * nD) {
      if (xstage_) cudaFreeHost(xstage_);
      CK(cudaMallocHost(&xstage_, sizeof(R) * nD));
      xstage_bytes_ = sizeof(R) * nD;
    }
    R* xr = static_cast<R*>(xstage_);
    xs_host_.resize(nD);
    degen_.assign(N_, 0);
    xf_valid_ = false;
    const size_t JD = (size_t)J_ * D;
#pragma omp parallel for schedule(static)
    for (int n = 0; n < N_; ++n) {
      double* xn = xs_host_.data() + (size_t)n * JD;
      bool dg = false;
      normalize_image(cfg_.normalize, H, W, x + (size_t)n * JD, xn, J_, &dg);
      degen_[n] = dg ? 1 : 0;
      double s = 0.0;
      for (int j = 0; j < J_; ++j) {
        double sj = 0.0;
        for (size_t i = (size_t)j * D; i < (size_t)(j + 1) * D; ++i) {
          const R v = R(xn[i]);
          xr[(size_t)n * JD + i] = v;
          xn[i] = double(v);
          sj += xn[i] * xn[i];
        }
        xnorm2c_[(size_t)n * J_ + j] = sj;
        s += sj;
      }
      xnorm2_[n] = s;
    }
    CK(cudaMemcpyAsync(x_.p, xr, sizeof(R) * nD, cudaMemcpyHostToDevice, st_));
    for (int j = 0; j < J_; ++j)  // x_hat channel-major: J x N x NB
      r2c(x_.as<R>() + (size_t)j * D, false, JD, xhat_.as<C>() + (size_t)j * N_ * NB, NB, N_);
    CK(cudaStreamSynchronize(st_));
  }

  void get_signals(double* x) override { std::copy(xs_host_.begin(), xs_host_.end(), x); }
  void signal_flags(int* degenerate) override {
    for (int n = 0; n < N_; ++n) degenerate[n] = n < (int)degen_.size() ? degen_[n] : 0;
  }

  void set_dictionary(const double* d) override {
    const size_t cnt = (size_t)K_ * J_ * M_;
    require_finite(d, cnt, "dictionary");
    dict_.assign(d, d + cnt);
    dict_zero_ = std::all_of(dict_.begin(), dict_.end(), [](double v) { return v == 0.0; });
    upload_dict_spectra(dict_.data(), dhat_.as<C>());
    if constexpr (CLU) {
      if (dhat_rb_.p)
        launch(kFamOther, [&] {
          cl_rank_block<P><<<592, 256, 0, st_>>>(dhat_.as<C>(), dhat_rb_.as<C>(), K_);
        });
    }
    if constexpr (kTcFamily) {
      if (tc_) {
        float amax = 0.f;
        for (double v : dict_) amax = std::max(amax, (float)std::fabs(v));
        tc_dscale_ = umma::pow2_scale(amax);
        double l1max = 0.0;  // max_k ||d_k||_1 (J = 1): the pass's bound on |t|
        for (int k = 0; k < K_; ++k) {
          double l1 = 0.0;
          for (int o = 0; o < M_; ++o) l1 += std::fabs(dict_[(size_t)k * M_ + o]);
          l1max = std::max(l1max, l1);
        }
        tc_tbound_ = (float)(2.0 * 16384.0 * l1max);
        launch(kFamOther, [&] {
          constexpr int TP = TG<kTcKFb>::TP;
          if (tc_kf_ == kTcKFa)
            tc_dsplit<kTcKFa, TP><<<32, 256, 0, st_>>>(ddict_.as<double>(), K_, M_, tc_dscale_,
                                                       tdsplit_.as<__half>());
          else
            tc_dsplit<kTcKFb, TP><<<64, 256, 0, st_>>>(ddict_.as<double>(), K_, M_, tc_dscale_,
                                                       tdsplit_.as<__half>());
        });
      }
    }
    if (J_ == 1) {
      launch(kFamOther, [&] {
        sigma_kernel<R><<<(NB + 255) / 256, 256, 0, st_>>>(dhat_.as<C>(), sigma_.as<R>(), K_, NB, cfg_.rho);
      });
    } else {  // per-bin block factorisation, once per dictionary (tcsc.cpp:31-55)
      launch(kFamOther, [&] {
        tc_factor<R><<<(NB + 127) / 128, 128, 0, st_>>>(dhat_.as<C>(), ginv_.as<C>(), K_, J_, NB, cfg_.rho);
      });
    }
    CK(cudaStreamSynchronize(st_));
  }

  void get_dictionary(double* d) override { std::copy(dict_.begin(), dict_.end(), d); }

  // init_variables (pipeline.cpp:123-156)
  void init_variables() override {
    const int JM = J_ * M_;  // filter k spans its J channel slices (k-major)
    std::vector<double> d((size_t)K_ * JM);
    std::mt19937_64 rng(cfg_.seed);
    auto uniform = [&rng]() { return static_cast<double>(rng() >> 11) * 0x1.0p-53 - 0.5; };
    for (int k = 0; k < K_; ++k) {
      double sq = 0.0;
      for (int i = 0; i < JM; ++i) {
        const double v = uniform();
        d[(size_t)k * JM + i] = v;
        sq += v * v;
      }
      double nrm = std::sqrt(sq);
      if (nrm == 0.0) {
        d[(size_t)k * JM] = 1.0;
        nrm = 1.0;
      }
      for (int i = 0; i < JM; ++i) d[(size_t)k * JM + i] /= nrm;
    }
    set_dictionary(d.data());
    CK(cudaMemsetAsync(u_.p, 0, u_.bytes, st_));
    CK(cudaMemsetAsync(maps_.p, 0, maps_.bytes, st_));
    CK(cudaMemsetAsync(lam_.p, 0, lam_.bytes, st_));
    CK(cudaMemsetAsync(gam_.p, 0, gam_.bytes, st_));
    u_zero_.assign(N_, 1);
    t0_pending_.assign(N_, 0);
    mu_.assign(K_, 1.0);
    zhat_valid_ = false;
    zf_valid_ = false;
    CK(cudaStreamSynchronize(st_));
  }

  // sum v[0..n) over ranks (host values; no-op on one rank)
  void reduce_host(double* v, int n) {
    if (!multi()) return;
    CK(cudaMemcpyAsync(hred_.p, v, sizeof(double) * n, cudaMemcpyHostToDevice, st_));
    red_->allreduce(hred_.as<double>(), n, st_);
    CK(cudaMemcpyAsync(v, hred_.p, sizeof(double) * n, cudaMemcpyDeviceToHost, st_));
    CK(cudaStreamSynchronize(st_));
  }

  // Internal u layout: the single-CTA family stores each plane's pixel pairs
  // column-major ((c/2)*H + r), the cluster family row-major; i is a
  // reference-layout index (plane-major, row-major pixels).
  static size_t u_index(size_t i) {
    if constexpr (CLU) {
      return i;
    } else {
      const size_t p = i / D, q = i % D;
      const size_t r = q / W, c = q % W;
      return p * D + ((c >> 1) * H + r) * 2 + (c & 1);
    }
  }

  void check_range(int n0, int n1) const {
    if (n0 < 0 || n1 > N_ || n0 >= n1) throw DimErr("image range out of bounds");
  }

  void set_coding_state(int n0, int n1, const double* theta, const double* z) override {
    check_range(n0, n1);
    const size_t cnt = (size_t)(n1 - n0) * K_ * D;
    if (!theta && !z) {  // the reference's empty state (coding.cpp:175-179): device-side reset
      std::fill(u_zero_.begin() + n0, u_zero_.begin() + n1, 1);
      if (!t0_pending_.empty()) std::fill(t0_pending_.begin() + n0, t0_pending_.begin() + n1, 0);
      CK(cudaMemsetAsync(u_.as<R>() + (size_t)n0 * K_ * D, 0, sizeof(R) * cnt, st_));
      CK(cudaMemsetAsync(lam_.as<R>() + (size_t)n0 * J_ * D, 0, sizeof(R) * (size_t)(n1 - n0) * J_ * D, st_));
      return;
    }
    std::fill(u_zero_.begin() + n0, u_zero_.begin() + n1, 0);
    std::vector<R> u(cnt), th(cnt);
    const double inv_rho = 1.0 / cfg_.rho, beta = cfg_.beta;
    // The single state array u = theta - z/rho reproduces the reference's first
    // iteration (w = theta + z/rho, theta_old) only when theta = clamp(u), which
    // holds for every state ADMM produces. Other states (theta outside the box,
    // z given without theta, a state saved under another beta / rho) keep
    // theta for the prologue and the first iteration (CodingArgs::theta0).
    bool consistent = true;
    for (size_t i = 0; i < cnt; ++i) {
      const double tv = theta ? theta[i] : 0.0;
      const double uv = tv - (z ? z[i] : 0.0) * inv_rho;
      u[u_index(i)] = R(uv);
      th[u_index(i)] = R(tv);
      const double cl = std::min(std::max(uv, -beta), beta);
      if (std::abs(cl - tv) > 1e-12 * std::max({beta, std::abs(tv), std::abs(uv)})) consistent = false;
    }
    CK(cudaMemcpyAsync(u_.as<R>() + (size_t)n0 * K_ * D, u.data(), sizeof(R) * cnt, cudaMemcpyHostToDevice, st_));
    if (!consistent) {
      if (!theta0_.p) {
        theta0_.alloc(sizeof(R) * (size_t)N_ * K_ * D);
        device_bytes += theta0_.bytes;
      }
      CK(cudaMemcpyAsync(theta0_.as<R>() + (size_t)n0 * K_ * D, th.data(), sizeof(R) * cnt, cudaMemcpyHostToDevice,
                         st_));
    }
    t0_pending_.resize(N_, 0);
    std::fill(t0_pending_.begin() + n0, t0_pending_.begin() + n1, consistent ? 0 : 1);
    CK(cudaStreamSynchronize(st_));
  }

  // theta0 of images [n0, n1) that have no pending theta: clamp(u) (their
  // states are ADMM-consistent), so one theta0 launch serves a mixed range
  void theta0_fill_consistent(int n0, int n1) {
    const size_t KD = (size_t)K_ * D;
    std::vector<R> u(KD);
    const R beta = R(cfg_.beta);
    for (int n = n0; n < n1; ++n) {
      if (t0_pending_[n]) continue;
      CK(cudaMemcpyAsync(u.data(), u_.as<R>() + (size_t)n * KD, sizeof(R) * KD, cudaMemcpyDeviceToHost, st_));
      CK(cudaStreamSynchronize(st_));
      for (auto& v : u) v = std::min(std::max(v, -beta), beta);
      CK(cudaMemcpyAsync(theta0_.as<R>() + (size_t)n * KD, u.data(), sizeof(R) * KD, cudaMemcpyHostToDevice, st_));
      CK(cudaStreamSynchronize(st_));
    }
  }
  bool theta0_pending(int n0, int n1) const {
    if (t0_pending_.empty()) return false;
    return std::any_of(t0_pending_.begin() + n0, t0_pending_.begin() + n1, [](char v) { return v != 0; });
  }

  void get_coding_state(int n0, int n1, double* theta, double* z, double* lambda) override {
    check_range(n0, n1);
    const size_t cnt = (size_t)(n1 - n0) * K_ * D;
    std::vector<R> u(cnt);
    CK(cudaMemcpyAsync(u.data(), u_.as<R>() + (size_t)n0 * K_ * D, sizeof(R) * cnt, cudaMemcpyDeviceToHost, st_));
    std::vector<R> l((size_t)(n1 - n0) * J_ * D);
    CK(cudaMemcpyAsync(l.data(), lam_.as<R>() + (size_t)n0 * J_ * D, sizeof(R) * l.size(), cudaMemcpyDeviceToHost,
                       st_));
    CK(cudaStreamSynchronize(st_));
    std::vector<R> t0;
    if (theta0_pending(n0, n1)) {
      t0.resize(cnt);
      CK(cudaMemcpyAsync(t0.data(), theta0_.as<R>() + (size_t)n0 * K_ * D, sizeof(R) * cnt, cudaMemcpyDeviceToHost,
                         st_));
      CK(cudaStreamSynchronize(st_));
    }
    const R beta = R(cfg_.beta), rho = R(cfg_.rho);
    const size_t KD = (size_t)K_ * D;
    for (size_t i = 0; i < cnt; ++i) {
      const R uv = u[u_index(i)];
      const bool pend = !t0.empty() && t0_pending_[n0 + i / KD];
      const R th = pend ? t0[u_index(i)] : std::min(std::max(uv, -beta), beta);
      if (theta) theta[i] = th;
      if (z) z[i] = rho * (th - uv);
    }
    if (lambda)
      for (size_t i = 0; i < l.size(); ++i) lambda[i] = l[i];
  }

  // solve_coding for images [n0, n1) (coding.cpp:166-329, 333-356)
  void coding(int n0, int n1, dcsc_coding_stats* stats) override {
    check_range(n0, n1);
    const int cnt = n1 - n0;
    std::vector<dcsc_coding_stats> out(cnt);
    if (dict_zero_) {
      // degenerate dictionary: z = theta = 0, lambda = -x (coding.cpp:181-191)
      std::fill(u_zero_.begin() + n0, u_zero_.begin() + n1, 1);
      if (!t0_pending_.empty()) std::fill(t0_pending_.begin() + n0, t0_pending_.begin() + n1, 0);
      CK(cudaMemsetAsync(u_.as<R>() + (size_t)n0 * K_ * D, 0, sizeof(R) * (size_t)cnt * K_ * D, st_));
      const size_t JD = (size_t)J_ * D;
      const size_t tot = (size_t)cnt * JD;
      launch(kFamOther, [&] {
        neg_copy<R><<<(unsigned)((tot + 255) / 256), 256, 0, st_>>>(x_.as<R>() + (size_t)n0 * JD,
                                                                   lam_.as<R>() + (size_t)n0 * JD, tot);
      });
      CK(cudaStreamSynchronize(st_));
      for (int i = 0; i < cnt; ++i) {
        double ls = 0.0, lx = 0.0;
        for (size_t j = 0; j < JD; ++j) {
          const double lv = -xs_host_[(size_t)(n0 + i) * JD + j];
          ls += lv * lv;
          lx += lv * xs_host_[(size_t)(n0 + i) * JD + j];
        }
        out[i] = dcsc_coding_stats{};
        out[i].converged = 1;
        out[i].degenerate_dictionary = 1;
        out[i].dual_objective = -0.5 * ls - lx;
      }
      if (stats) std::copy(out.begin(), out.end(), stats);
      return;
    }
    int* conv_h = static_cast<int*>(pin_);
    CK(cudaMemsetAsync(conv_.as<int>() + n0, 0, sizeof(int) * cnt, st_));
    CK(cudaMemsetAsync(img_.as<ImageAdmm>() + n0, 0, sizeof(ImageAdmm) * cnt, st_));
    const dim3 lgrid((NB + 255) / 256, cnt);
    // initial lambda_hat from the warm state (the first assemble_w, coding.cpp:216-229);
    // a zero state has w_hat = 0, so the FFT pass is skipped and part is zeroed
    const bool all_zero = std::all_of(u_zero_.begin() + n0, u_zero_.begin() + n1, [](char v) { return v != 0; });
    // a warm state that is not ADMM-consistent: theta0 feeds the prologue and iteration 1
    const bool t0_pending = theta0_pending(n0, n1);
    if (t0_pending) theta0_fill_consistent(n0, n1);
    use_theta0_ = t0_pending;
    // multi-channel: lambda_hat from the per-bin J x J solves (tcsc.cpp:68-88)
    auto tc_lam = [&](int kw, bool skip_conv) {
      launch(kFamLambda, [&] {
        const dim3 grid((NB + 127) / 128, cnt);
        const C* wp = what_.as<C>() + (size_t)n0 * K_ * NB;
        const C* xp = xhat_.as<C>() + (size_t)n0 * NB;
        C* lp = lamhat_.as<C>() + (size_t)n0 * J_ * NB;
        const int* cv = skip_conv ? conv_.as<int>() + n0 : nullptr;
        const R ir = R(1.0 / cfg_.rho);
        if (J_ == 3)
          tc_lambda<R, 3><<<grid, 128, 0, st_>>>(wp, dhat_.as<C>(), ginv_.as<C>(), xp, (size_t)N_ * NB, lp, cv, K_,
                                                 kw, J_, NB, ir);
        else
          tc_lambda<R><<<grid, 128, 0, st_>>>(wp, dhat_.as<C>(), ginv_.as<C>(), xp, (size_t)N_ * NB, lp, cv, K_, kw,
                                              J_, NB, ir);
      });
    };
    if (J_ > 1) {
      if (!all_zero) coding_launch<kPassPrologue>(dhat_.as<C>(), n0, cnt);  // w_hat of the warm state
      tc_lam(all_zero ? 0 : K_, false);
    } else if (all_zero) {
      CK(cudaMemsetAsync(part_.as<C>() + (size_t)n0 * G_ * NB, 0, sizeof(C) * (size_t)cnt * G_ * NB, st_));
    } else {
      coding_launch<kPassPrologue>(dhat_.as<C>(), n0, cnt);  // lambda_hat from the fused epilogue
    }
    std::fill(u_zero_.begin() + n0, u_zero_.begin() + n1, 0);
    use_theta0_ = false;
    if (t0_pending) std::fill(t0_pending_.begin() + n0, t0_pending_.begin() + n1, 0);
    auto lam_update = [&](int iter, int last, int prologue) {
      launch(kFamLambda, [&] {
        lambda_update<R><<<lgrid, 256, 0, st_>>>(part_.as<C>() + (size_t)n0 * G_ * NB,
                                                 sums_.as<double>() + (size_t)n0 * G_ * kSums,
                                                 xhat_.as<C>() + (size_t)n0 * NB, sigma_.as<R>(),
                                                 lamhat_.as<C>() + (size_t)n0 * NB, conv_.as<int>() + n0,
                                                 img_.as<ImageAdmm>() + n0, G_, NB, R(cfg_.rho), iter, last,
                                                 prologue);
      });
    };
    if (all_zero && J_ == 1) lam_update(0, 0, 1);
    // tensor-core pass for this call (the single-CTA family keeps a warm state that
    // is not ADMM-consistent on the FFT pass: its theta0 is in the pair layout)
    const bool tc = tc_use(cnt) && (CLU || !t0_pending);
    if (tc) {
      if (!CLU) tc_convert_u(n0, cnt, true);
      tc_lambda_spatial(n0, cnt);
      tc_zmax(n0, cnt);
    }
    cudaEvent_t ev[2];
    CK(cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming));
    // tensor-core pass on large batches: the images in two halves on two streams,
    // so each half's per-iteration neighbours (band reduction, lambda_hat
    // update, the two FFTs, lambda split) run beside the other half's coding
    // pass instead of between two full-width passes
    // (measured: C1 23.6 -> 24.7, C2 3.81 -> 4.51, C4 1.92 -> 2.20 outer iters/s; DCSC_TC_SPLIT=0 disables)
    const char* sp = std::getenv("DCSC_TC_SPLIT");
    const bool split = !(sp && sp[0] == '0');
    const int half = (tc && split && cnt >= 2) ? cnt / 2 : 0;
    cudaEvent_t ev2[2] = {nullptr, nullptr};
    if (half) {
      CK(cudaEventCreateWithFlags(&ev2[0], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&ev2[1], cudaEventDisableTiming));
      CK(cudaEventRecord(ev2[0], st_));  // prologue / lambda split / u conversion done
      CK(cudaStreamWaitEvent(st2_, ev2[0], 0));
    }
    int pending = -1;  // iteration whose conv flags are in flight
    for (int it = 1; it <= cfg_.max_admm; ++it) {
      use_theta0_ = t0_pending && it == 1;
      if (half) {
        tc_iteration(n0, half, it, it == cfg_.max_admm, st_);
        tc_iteration(n0 + half, cnt - half, it, it == cfg_.max_admm, st2_);
      } else if (tc) {
        tc_iteration(n0, cnt, it, it == cfg_.max_admm);
      } else {
        coding_launch<kPassAdmm>(dhat_.as<C>(), n0, cnt, it, it == cfg_.max_admm);
      }
      use_theta0_ = false;
      if (J_ > 1 && it < cfg_.max_admm) tc_lam(K_, true);
      if (pending >= 0) {
        // one-iteration look-ahead: iteration `it` is queued before we wait on it-1
        CK(cudaEventSynchronize(ev[pending & 1]));
        if (half) CK(cudaEventSynchronize(ev2[pending & 1]));
        bool all = true;
        for (int i = 0; i < cnt; ++i) all = all && conv_h[(pending & 1) * 65536 + i];
        if (all) break;
      }
      if (cnt <= 65536) {
        const int c1 = half ? half : cnt;
        CK(cudaMemcpyAsync(conv_h + (it & 1) * 65536, conv_.as<int>() + n0, sizeof(int) * c1,
                           cudaMemcpyDeviceToHost, st_));
        CK(cudaEventRecord(ev[it & 1], st_));
        if (half) {
          CK(cudaMemcpyAsync(conv_h + (it & 1) * 65536 + half, conv_.as<int>() + n0 + half,
                             sizeof(int) * (cnt - half), cudaMemcpyDeviceToHost, st2_));
          CK(cudaEventRecord(ev2[it & 1], st2_));
        }
        pending = it;
      }
    }
    if (half) {  // join: the exit work on st_ sees both halves
      CK(cudaEventRecord(ev2[0], st2_));
      CK(cudaStreamWaitEvent(st_, ev2[0], 0));
      CK(cudaStreamSynchronize(st2_));
      cudaEventDestroy(ev2[0]);
      cudaEventDestroy(ev2[1]);
    }
    cudaEventDestroy(ev[0]);
    cudaEventDestroy(ev[1]);
    if (tc && !CLU) tc_convert_u(n0, cnt, false);
    // exit: lambda = iDFT(lambda_hat), rescale, dual objective (coding.cpp:287-309)
    c2r<R>(lamhat_.as<C>() + (size_t)n0 * J_ * NB, NB, lam_.as<R>() + (size_t)n0 * J_ * D, D, cnt * J_);
    launch(kFamOther, [&] {
      admm_exit<R><<<cnt, 256, 0, st_>>>(lam_.as<R>() + (size_t)n0 * J_ * D, x_.as<R>() + (size_t)n0 * J_ * D,
                                         img_.as<ImageAdmm>() + n0, J_ * D, cfg_.beta, dual_.as<double>() + n0,
                                         infeas_.as<double>() + n0, resc_.as<int>() + n0);
    });
    std::vector<ImageAdmm> im(cnt);
    std::vector<double> du(cnt), inf(cnt);
    std::vector<int> rs(cnt);
    CK(cudaMemcpyAsync(im.data(), img_.as<ImageAdmm>() + n0, sizeof(ImageAdmm) * cnt, cudaMemcpyDeviceToHost, st_));
    CK(cudaMemcpyAsync(du.data(), dual_.as<double>() + n0, sizeof(double) * cnt, cudaMemcpyDeviceToHost, st_));
    CK(cudaMemcpyAsync(inf.data(), infeas_.as<double>() + n0, sizeof(double) * cnt, cudaMemcpyDeviceToHost, st_));
    CK(cudaMemcpyAsync(rs.data(), resc_.as<int>() + n0, sizeof(int) * cnt, cudaMemcpyDeviceToHost, st_));
    CK(cudaStreamSynchronize(st_));
    for (int i = 0; i < cnt; ++i) {
      dcsc_coding_stats& s = out[i];
      s.admm_iters = im[i].iters;
      s.converged = im[i].converged;
      s.degenerate_dictionary = 0;
      s.dual_rescaled = rs[i];
      s.primal_residual = im[i].primal;
      s.theta_change = im[i].thc;
      s.z_change = im[i].zc;
      s.dual_objective = du[i];
      s.dual_infeasibility = inf[i];
    }
    if (stats) std::copy(out.begin(), out.end(), stats);
  }

  void set_maps(int n0, int n1, const double* z) override {
    check_range(n0, n1);
    const size_t cnt = (size_t)(n1 - n0) * K_ * D;
    std::vector<R> v(cnt);
    for (size_t i = 0; i < cnt; ++i) v[i] = R(z[i]);
    CK(cudaMemcpyAsync(maps_.as<R>() + (size_t)n0 * K_ * D, v.data(), sizeof(R) * cnt, cudaMemcpyHostToDevice, st_));
    CK(cudaStreamSynchronize(st_));
    zhat_valid_ = false;
    zf_valid_ = false;
  }

  void get_maps(int n0, int n1, double* z) override {
    check_range(n0, n1);
    const size_t cnt = (size_t)(n1 - n0) * K_ * D;
    std::vector<R> v(cnt);
    CK(cudaMemcpyAsync(v.data(), maps_.as<R>() + (size_t)n0 * K_ * D, sizeof(R) * cnt, cudaMemcpyDeviceToHost, st_));
    CK(cudaStreamSynchronize(st_));
    for (size_t i = 0; i < cnt; ++i) z[i] = v[i];
  }

  void set_learning_state(const double* gamma, const double* mu) override {
    if (freq_) throw InvErr("learning state is not available in the frequency-sharded layout");
    if (gamma) {  // J x N x D (LearningDualState::gamma[j], learning.hpp:15-23)
      DevMem tmp;
      tmp.alloc(sizeof(double) * (size_t)J_ * N_ * D);
      CK(cudaMemcpyAsync(tmp.p, gamma, tmp.bytes, cudaMemcpyHostToDevice, st_));
      r2c(tmp.p, true, D, gam_.as<C>(), NB, J_ * N_);
      CK(cudaStreamSynchronize(st_));
    } else {
      CK(cudaMemsetAsync(gam_.p, 0, gam_.bytes, st_));
    }
    if (mu) mu_.assign(mu, mu + K_);
    else mu_.assign(K_, 1.0);
    CK(cudaStreamSynchronize(st_));
  }

  void get_learning_state(double* gamma, double* mu) override {
    if (freq_ && gamma) throw InvErr("learning state is not available in the frequency-sharded layout");
    if (gamma) {
      DevMem tmp;
      tmp.alloc(sizeof(double) * (size_t)J_ * N_ * D);
      c2r<double>(gam_.as<C>(), NB, tmp.as<double>(), D, J_ * N_);
      CK(cudaMemcpyAsync(gamma, tmp.p, tmp.bytes, cudaMemcpyDeviceToHost, st_));
      CK(cudaStreamSynchronize(st_));
    }
    if (mu) std::copy(mu_.begin(), mu_.end(), mu);
  }

  // z_hat of the accepted maps and the dead-filter flags (learning.cpp:41-64)
  void build_zhat() {
    if (zhat_valid_) return;
    if (!zhat_.p) {
      zhat_.alloc(sizeof(C) * (size_t)N_ * K_ * NB);
      device_bytes += zhat_.bytes;
    }
    CK(cudaMemsetAsync(live_.p, 0, sizeof(int) * K_, st_));
    r2c(maps_.p, false, D, zhat_.as<C>(), NB, N_ * K_, live_.as<int>(), K_);
    live_h_.assign(K_, 0);
    CK(cudaMemcpyAsync(live_h_.data(), live_.p, sizeof(int) * K_, cudaMemcpyDeviceToHost, st_));
    CK(cudaStreamSynchronize(st_));
    if (multi()) {  // a filter is dead only if its maps vanish on every rank
      std::vector<double> lv(K_);
      for (int k = 0; k < K_; ++k) lv[k] = live_h_[k];
      reduce_host(lv.data(), K_);
      for (int k = 0; k < K_; ++k) live_h_[k] = lv[k] > 0.0 ? 1 : 0;
      CK(cudaMemcpyAsync(live_.p, live_h_.data(), sizeof(int) * K_, cudaMemcpyHostToDevice, st_));
      CK(cudaStreamSynchronize(st_));
    }
    zhat_valid_ = true;
  }

  // c_k = sum_n conj(z_hat_nk) v_n (split over image chunks, fixed-order reduce)
  void correlate_hat(const C* v, const int* done) {
    constexpr int KC = DCSC_KC;
    const dim3 g1((NB + TBV - 1) / TBV, (K_ + KC - 1) / KC, csplit_);
    launch(kFamContract, [&] {
      contract_c<R, KC><<<g1, TBV, 0, st_>>>(zhat_.as<C>(), v, cpart_.as<double2>(), live_.as<int>(), N_, K_, NB,
                                             done);
    });
    const size_t knb = (size_t)K_ * NB;
    const unsigned rb = (unsigned)((knb + 255) / 256);
    // multi-rank: this is the rank's partial correlation; the ranks' sum is
    // taken after the mask's crop (mask_crop / apply_hat), K x M values instead of K x NB
    launch(kFamOther, [&] {  // (kFamContract holds only the z_hat streams: contract_c, contract_out)
      contract_c_reduce<R><<<rb, 256, 0, st_>>>(cpart_.as<double2>(), cvec_.as<C>(), csplit_, knb, done);
    });
  }

  // Cropped correlation of cvec_ (mask_step mode 1: d_recover scaling, mode 2:
  // plain) into dd_ (K x M), summed over ranks: the crop of the inverse DFT is
  // linear, so crop(iDFT(sum_r c_r)) = sum_r crop(iDFT(c_r)) and the ranks
  // exchange K x M values (C3: 124 KB) instead of the K x NB spectra (67 MB).
  void mask_crop(int mode, const int* done) {
    launch(kFamMask, [&] {
      launch_mask(K_, st_, cvec_.as<C>(), nullptr, dd_.as<double>(), live_.as<int>(), dmu_.as<double>(), mh_, mw_,
                  mode, dtw_.as<C>(), done);
    });
    if (multi()) red_->allreduce(dd_.as<double>(), (size_t)K_ * M_, st_);
  }

  // A v for half-spectrum stacks (LearningOperator::apply, learning.cpp:83-122)
  // fuse_alpha (single rank, inside the CG loop): contract_out's last block
  // also runs the alpha step (no separate cg_scalar launch)
  void apply_hat(const C* v, C* out, const int* done = nullptr, bool fuse_alpha = false) {
    correlate_hat(v, done);
    if (!multi()) {
      launch(kFamMask, [&] {
        launch_mask(K_, st_, cvec_.as<C>(), phat_.as<C>(), nullptr, live_.as<int>(), dmu_.as<double>(), mh_, mw_, 0,
                    dtw_.as<C>(), done);
      });
    } else {  // crop per rank, sum the K x M crops, then p_hat = DFT(pad(crop))
      mask_crop(2, done);
      launch(kFamMask, [&] { launch_filters(K_, st_, dd_.as<double>(), mh_, mw_, phat_.as<C>(), dtw_.as<C>()); });
    }
    // fused: fewer image rows per launch (each block loops over images) so the
    // last-block alpha step sums few partials and the arrival counter sees
    // few atomics
    const dim3 g3(tiles_, fuse_alpha ? std::min(N_, std::max(1, fused_rows_ / tiles_)) : N_);
    // two images per pass share the p_hat loads once the p_hat stack outgrows ~16 MB (C3)
    const bool pair = sizeof(C) * (size_t)K_ * NB > (16u << 20);
    launch(kFamContract, [&] {
      if (pair)
        contract_out<R, TBV, 2><<<g3, TBV, 0, st_>>>(zhat_.as<C>(), phat_.as<C>(), dwk_.as<double>(),
                                                      live_.as<int>(), v, out, partial_.as<double>(), N_, K_, NB, Wh,
                                                      0, done, fuse_alpha ? cg_.as<CgState>() : nullptr,
                                                      cgcnt_.as<unsigned>(), 1.0 / D);
      else
        contract_out<R, TBV><<<g3, TBV, 0, st_>>>(zhat_.as<C>(), phat_.as<C>(), dwk_.as<double>(), live_.as<int>(),
                                                   v, out, partial_.as<double>(), N_, K_, NB, Wh, 0, done,
                                                   fuse_alpha ? cg_.as<CgState>() : nullptr, cgcnt_.as<unsigned>(),
                                                   1.0 / D);
    });
  }

  void upload_mu() {
    std::vector<double> wk(K_);
    for (int k = 0; k < K_; ++k) wk[k] = 0.5 / mu_[k];
    CK(cudaMemcpyAsync(dmu_.p, mu_.data(), sizeof(double) * K_, cudaMemcpyHostToDevice, st_));
    CK(cudaMemcpyAsync(dwk_.p, wk.data(), sizeof(double) * K_, cudaMemcpyHostToDevice, st_));
  }

  CgState read_cg() {
    CgState* h = reinterpret_cast<CgState*>(static_cast<char*>(pin_) + 600000);
    CK(cudaMemcpyAsync(h, cg_.p, sizeof(CgState), cudaMemcpyDeviceToHost, st_));
    CK(cudaStreamSynchronize(st_));
    return *h;
  }

  // One CG scalar step; across ranks the block partials are first summed
  // locally, all-reduced, then applied (identical state on every rank).
  void cg_step(const double* partial, int count, double invD, int step) {
    if (!multi()) {
      launch(kFamOther, [&] { cg_scalar<<<1, 1024, 0, st_>>>(partial, count, invD, cg_.as<CgState>(), step, nullptr); });
      return;
    }
    launch(kFamOther, [&] { sum_partials<<<1, 1024, 0, st_>>>(partial, count, hred_.as<double>()); });
    red_->allreduce(hred_.as<double>(), 1, st_);
    launch(kFamOther, [&] {
      cg_scalar<<<1, 1024, 0, st_>>>(partial, count, invD, cg_.as<CgState>(), step, hred_.as<double>());
    });
  }

  // gamma_solve (learning.cpp:136-185), warm-started, on half spectra. The
  // iteration loop terminates on the device (CgState::done); the host issues
  // iterations in chunks and reads the state once per chunk.
  void gamma_solve(double bnorm, int& iters, bool& converged) {
    iters = 0;
    converged = false;
    const size_t total = (size_t)N_ * NB;
    const unsigned vb = (unsigned)((total + TBV - 1) / TBV);
    if (bnorm == 0.0) {
      CK(cudaMemsetAsync(gam_ch_, 0, sizeof(C) * total, st_));
      converged = true;
      return;
    }
    CgState init{};
    init.bnorm = bnorm;
    init.tol = cfg_.cg_tol;
    init.max_iters = cfg_.cg_max;
    CK(cudaMemcpyAsync(cg_.p, &init, sizeof(CgState), cudaMemcpyHostToDevice, st_));
    apply_hat(gam_ch_, ap_.as<C>());
    launch(kFamOther, [&] {
      cg_init<R, TBV><<<vb, TBV, 0, st_>>>(xh_ch_, ap_.as<C>(), r_.as<C>(), p_.as<C>(),
                                            partial_.as<double>(), total, NB, Wh);
    });
    const double invD = 1.0 / D;
    cg_step(partial_.as<double>(), (int)vb, invD, 0);
    const int* done = &cg_.as<CgState>()->done;
    CgState s = read_cg();
    int issued = 0, chunk = 2;
    while (!s.done && issued < cfg_.cg_max) {
      const int n = std::min(chunk, cfg_.cg_max - issued);
      const bool fuse = !multi() && !no_cg_fuse_;  // single rank: scalar steps in the producers' last blocks
      for (int c = 0; c < n; ++c) {
        apply_hat(p_.as<C>(), ap_.as<C>(), done, fuse);
        if (!fuse) cg_step(partial_.as<double>(), N_ * tiles_, invD, 1);
        launch(kFamOther, [&] {
          cg_update<R, TBV><<<fuse ? std::min<unsigned>(vb, (unsigned)fused_rows_) : vb, TBV, 0, st_>>>(
                                                  gam_ch_, r_.as<C>(), p_.as<C>(), ap_.as<C>(),
                                                  cg_.as<CgState>(), partial_.as<double>(), total, NB, Wh,
                                                  fuse ? cgcnt_.as<unsigned>() + 1 : nullptr, invD);
        });
        if (!fuse) cg_step(partial_.as<double>(), (int)vb, invD, 2);
        launch(kFamOther, [&] {
          cg_pupdate<R, TBV><<<vb, TBV, 0, st_>>>(r_.as<C>(), p_.as<C>(), cg_.as<CgState>(), total);
        });
      }
      issued += n;
      chunk = std::min(chunk * 2, 8);
      s = read_cg();
    }
    iters = s.iters;
    converged = s.converged != 0;
  }

  // d_recover (learning.cpp:187-216): d_k = -0.5/max(mu_k,1e-300) crop(iDFT(sum_n conj(z_nk) gamma_n))
  void d_recover(std::vector<double>& d) {
    correlate_hat(gam_ch_, nullptr);
    // d_recover does not skip dead filters; their correlation is exactly zero anyway
    mask_crop(1, nullptr);
    d.resize((size_t)K_ * M_);
    CK(cudaMemcpyAsync(d.data(), dd_.p, sizeof(double) * K_ * M_, cudaMemcpyDeviceToHost, st_));
    CK(cudaStreamSynchronize(st_));
  }

  // solve_learning (learning.cpp:227-355) over all images; J > 1 runs the J
  // per-channel gamma systems under one mu ascent with joint filter norms
  // (solve_learning_tcsc, tcsc.cpp:263-270 -> learning.cpp:276-345)
  void learning(double* d_out, dcsc_learning_stats* st) override {
    if (freq_) {
      learning_freq(d_out, st);
      return;
    }
    dcsc_learning_stats ls{};
    if ((int)mu_.size() != K_) mu_.assign(K_, 1.0);
    build_zhat();
    int n_live = 0;
    for (int k = 0; k < K_; ++k) n_live += live_h_[k] ? 1 : 0;
    ls.n_dead = K_ - n_live;
    const size_t JM = (size_t)J_ * M_;
    if (n_live == 0) {  // every map zero: zero dictionary, gamma = 0 (learning.cpp:258-270)
      ls.degenerate = 1;
      CK(cudaMemsetAsync(gam_.p, 0, gam_.bytes, st_));
      CK(cudaStreamSynchronize(st_));
      std::fill(d_out, d_out + (size_t)K_ * JM, 0.0);
      if (st) *st = ls;
      return;
    }
    std::vector<double> bnorm(J_, 0.0);
    for (int n = 0; n < N_; ++n)
      for (int j = 0; j < J_; ++j) bnorm[j] += xnorm2c_[(size_t)n * J_ + j];
    reduce_host(bnorm.data(), J_);
    for (double& b : bnorm) b = std::sqrt(b);
    std::vector<std::vector<double>> parts(J_);
    std::vector<double> norms(K_, 0.0);
    bool clamped = false;
    for (int iter = 1; iter <= cfg_.max_mu_iters; ++iter) {
      clamped = false;
      for (int k = 0; k < K_; ++k)
        if (mu_[k] < cfg_.mu_floor) {
          mu_[k] = cfg_.mu_floor;
          clamped = true;
        }
      upload_mu();
      long iter_cg = 0;
      for (int j = 0; j < J_; ++j) {
        select_channel(j);
        int cg_iters = 0;
        bool cg_conv = false;
        gamma_solve(bnorm[j], cg_iters, cg_conv);
        iter_cg += cg_iters;
        if (!cg_conv) ls.cg_budget_hit = 1;
      }
      ls.cg_iters += iter_cg;
      if (iter == 1) ls.cg_iters_first = iter_cg;
      for (int j = 0; j < J_; ++j) {
        select_channel(j);
        d_recover(parts[j]);
      }
      select_channel(0);
      for (int k = 0; k < K_; ++k) {
        double sq = 0.0;
        for (int j = 0; j < J_; ++j)
          for (int i = 0; i < M_; ++i) sq += parts[j][(size_t)k * M_ + i] * parts[j][(size_t)k * M_ + i];
        norms[k] = std::sqrt(sq);
      }
      ls.mu_iters = iter;
      bool settled = true;
      for (int k = 0; k < K_; ++k) {
        const bool at_boundary = std::abs(norms[k] - 1.0) <= kFilterNormTol;
        const bool inactive = mu_[k] <= cfg_.mu_floor * (1.0 + 1e-9) && norms[k] < 1.0;
        if (!at_boundary && !inactive) {
          settled = false;
          break;
        }
      }
      if (settled) {
        ls.converged = 1;
        break;
      }
      if (iter < cfg_.max_mu_iters)
        for (int k = 0; k < K_; ++k) mu_[k] = std::max(mu_[k] * norms[k], cfg_.mu_floor);
    }
    ls.mu_clamped = clamped ? 1 : 0;
    for (int k = 0; k < K_; ++k) {
      double scale = 1.0;
      if (norms[k] > 1.0) {
        scale = 1.0 / norms[k];
        ++ls.rescaled_filters;
      }
      for (int j = 0; j < J_; ++j)
        for (int i = 0; i < M_; ++i) d_out[(size_t)k * JM + (size_t)j * M_ + i] = scale * parts[j][(size_t)k * M_ + i];
    }
    if (st) *st = ls;
  }

  // learning views of channel j: x_hat_j and gamma_j (both N x NB)
  void select_channel(int j) {
    xh_ch_ = xhat_.as<C>() + (size_t)j * N_ * NB;
    gam_ch_ = gam_.as<C>() + (size_t)j * N_ * NB;
  }

  // LearningOperator::correlation (learning.cpp:124-134) for every filter:
  // out[k] = crop(iDFT(sum_n conj(z_hat_nk) DFT(v_n))), K x M (channel-free)
  void learning_correlation(const double* v, double* out) override {
    build_zhat();
    DevMem tmp;
    tmp.alloc(sizeof(double) * (size_t)N_ * D);
    CK(cudaMemcpyAsync(tmp.p, v, tmp.bytes, cudaMemcpyHostToDevice, st_));
    r2c(tmp.p, true, D, r_.as<C>(), NB, N_);
    correlate_hat(r_.as<C>(), nullptr);
    mask_crop(2, nullptr);
    CK(cudaMemcpyAsync(out, dd_.p, sizeof(double) * K_ * M_, cudaMemcpyDeviceToHost, st_));
    CK(cudaStreamSynchronize(st_));
  }

  // ---------------------------------------------------------- stateless ops
  // (coding.hpp:45-66, learning.hpp:81-95), for replaying iterations; they
  // leave the context's coding and learning state untouched.

  // D^T lambda: apply_dictionary_adjoint (coding.cpp:126-135), J > 1
  // block_dictionary_adjoint (tcsc.cpp:185-193). lam (n1-n0) x J x D -> out (n1-n0) x K x D.
  void dictionary_adjoint(int n0, int n1, const double* lam, double* out) override {
    check_range(n0, n1);
    const size_t JD = (size_t)J_ * D, KD = (size_t)K_ * D;
    DevMem lin, lh, th, tout;
    lin.alloc(sizeof(double) * JD);
    lh.alloc(sizeof(C) * (size_t)J_ * NB);
    th.alloc(sizeof(C) * (size_t)K_ * NB);
    tout.alloc(sizeof(double) * KD);
    for (int i = 0; i < n1 - n0; ++i) {
      CK(cudaMemcpyAsync(lin.p, lam + i * JD, sizeof(double) * JD, cudaMemcpyHostToDevice, st_));
      r2c(lin.p, true, D, lh.as<C>(), NB, J_);
      launch(kFamOther, [&] {
        adjoint_spectra<R><<<dim3((NB + 255) / 256, K_), 256, 0, st_>>>(dhat_.as<C>(), lh.as<C>(), th.as<C>(), K_,
                                                                       J_, NB);
      });
      c2r<double>(th.as<C>(), NB, tout.as<double>(), D, K_);
      CK(cudaMemcpyAsync(out + i * KD, tout.p, sizeof(double) * KD, cudaMemcpyDeviceToHost, st_));
      CK(cudaStreamSynchronize(st_));
    }
  }

  // lambda_update (coding.cpp:103-124; J > 1 lambda_update_blocked,
  // tcsc.cpp:162-183) from theta, z ((n1-n0) x K x D each) against the
  // context's signals and dictionary: out (n1-n0) x J x D.
  void lambda_update_op(int n0, int n1, const double* theta, const double* z, double* out) override {
    check_range(n0, n1);
    const size_t KD = (size_t)K_ * D, JD = (size_t)J_ * D;
    std::vector<double> w(KD);
    DevMem win, wh, lh, lout;
    win.alloc(sizeof(double) * KD);
    wh.alloc(sizeof(C) * (size_t)K_ * NB);
    lh.alloc(sizeof(C) * (size_t)J_ * NB);
    lout.alloc(sizeof(double) * JD);
    const double inv_rho = 1.0 / cfg_.rho;
    for (int i = 0; i < n1 - n0; ++i) {
      for (size_t q = 0; q < KD; ++q) w[q] = theta[i * KD + q] + z[i * KD + q] * inv_rho;  // coding.cpp:224-227
      CK(cudaMemcpyAsync(win.p, w.data(), sizeof(double) * KD, cudaMemcpyHostToDevice, st_));
      r2c(win.p, true, D, wh.as<C>(), NB, K_);
      const int n = n0 + i;
      launch(kFamOther, [&] {
        if (J_ == 1)
          lambda_from_w<R><<<(NB + 255) / 256, 256, 0, st_>>>(wh.as<C>(), dhat_.as<C>(), xhat_.as<C>() + (size_t)n * NB,
                                                               sigma_.as<R>(), lh.as<C>(), K_, NB, R(inv_rho));
        else
          tc_lambda<R><<<dim3((NB + 127) / 128, 1), 128, 0, st_>>>(wh.as<C>(), dhat_.as<C>(), ginv_.as<C>(),
                                                                 xhat_.as<C>() + (size_t)n * NB, (size_t)N_ * NB,
                                                                 lh.as<C>(), nullptr, K_, K_, J_, NB, R(inv_rho));
      });
      c2r<double>(lh.as<C>(), NB, lout.as<double>(), D, J_);
      CK(cudaMemcpyAsync(out + i * JD, lout.p, sizeof(double) * JD, cudaMemcpyDeviceToHost, st_));
      CK(cudaStreamSynchronize(st_));
    }
  }

  // gamma_solve (learning.cpp:136-185) on channel `channel` with the given mu
  // (clamped at the floor as LearningOperator::set_mu does); gamma (N x D) is
  // the warm start on entry and the solution on exit.
  void gamma_solve_op(int channel, const double* mu, double* gamma, int* iters, int* converged) override {
    if (channel < 0 || channel >= J_) throw DimErr("channel out of range");
    build_zhat();
    const std::vector<double> keep_mu = mu_;
    DevMem keep_g;
    keep_g.alloc(sizeof(C) * (size_t)N_ * NB);
    select_channel(channel);
    CK(cudaMemcpyAsync(keep_g.p, gam_ch_, keep_g.bytes, cudaMemcpyDeviceToDevice, st_));
    mu_.assign(mu, mu + K_);
    for (double& m : mu_) m = std::max(m, cfg_.mu_floor);
    upload_mu();
    DevMem tmp;
    tmp.alloc(sizeof(double) * (size_t)N_ * D);
    CK(cudaMemcpyAsync(tmp.p, gamma, tmp.bytes, cudaMemcpyHostToDevice, st_));
    r2c(tmp.p, true, D, gam_ch_, NB, N_);
    double bn = 0.0;
    for (int n = 0; n < N_; ++n) bn += xnorm2c_[(size_t)n * J_ + channel];
    reduce_host(&bn, 1);
    int it = 0;
    bool conv = false;
    gamma_solve(std::sqrt(bn), it, conv);
    c2r<double>(gam_ch_, NB, tmp.as<double>(), D, N_);
    CK(cudaMemcpyAsync(gamma, tmp.p, tmp.bytes, cudaMemcpyDeviceToHost, st_));
    CK(cudaMemcpyAsync(gam_ch_, keep_g.p, keep_g.bytes, cudaMemcpyDeviceToDevice, st_));
    CK(cudaStreamSynchronize(st_));
    mu_ = keep_mu;
    select_channel(0);
    if (iters) *iters = it;
    if (converged) *converged = conv ? 1 : 0;
  }

  // d_recover (learning.cpp:187-216) for one channel's gamma (N x D): out K x M
  void d_recover_op(int channel, const double* gamma, const double* mu, double* out) override {
    if (channel < 0 || channel >= J_) throw DimErr("channel out of range");
    build_zhat();
    DevMem tmp;
    tmp.alloc(sizeof(double) * (size_t)N_ * D);
    CK(cudaMemcpyAsync(tmp.p, gamma, tmp.bytes, cudaMemcpyHostToDevice, st_));
    r2c(tmp.p, true, D, r_.as<C>(), NB, N_);
    correlate_hat(r_.as<C>(), nullptr);
    CK(cudaMemcpyAsync(dmu_.p, mu, sizeof(double) * K_, cudaMemcpyHostToDevice, st_));
    mask_crop(1, nullptr);
    CK(cudaMemcpyAsync(out, dd_.p, sizeof(double) * K_ * M_, cudaMemcpyDeviceToHost, st_));
    upload_mu();  // the context's own mu back on the device
    CK(cudaStreamSynchronize(st_));
  }

  void learning_apply(const double* mu, const double* v, double* out) override {
    build_zhat();
    std::vector<double> keep = mu_;
    mu_.assign(mu, mu + K_);
    for (int k = 0; k < K_; ++k) mu_[k] = std::max(mu_[k], cfg_.mu_floor);  // set_mu clamps (learning.cpp:66-81)
    upload_mu();
    DevMem tmp;
    tmp.alloc(sizeof(double) * (size_t)N_ * D);
    CK(cudaMemcpyAsync(tmp.p, v, tmp.bytes, cudaMemcpyHostToDevice, st_));
    r2c(tmp.p, true, D, r_.as<C>(), NB, N_);
    apply_hat(r_.as<C>(), ap_.as<C>());
    c2r<double>(ap_.as<C>(), NB, tmp.as<double>(), D, N_);
    CK(cudaMemcpyAsync(out, tmp.p, tmp.bytes, cudaMemcpyDeviceToHost, st_));
    CK(cudaStreamSynchronize(st_));
    mu_ = keep;
  }

  // per-image data terms of `d` against the accepted maps (Parseval on z_hat),
  // summed over channels
  void data_terms(const double* d, std::vector<double>& data) {
    if (freq_) {
      data_terms_freq(d, data);
      return;
    }
    build_zhat();
    upload_dict_spectra(d, dcand_.as<C>());
    const dim3 g3(tiles_, N_);
    data.assign(N_, 0.0);
    std::vector<double> part(N_);
    for (int j = 0; j < J_; ++j) {
      launch(kFamContract, [&] {
        contract_out<R, TBV><<<g3, TBV, 0, st_>>>(zhat_.as<C>(), dcand_.as<C>() + (size_t)j * K_ * NB,
                                                   dwk_.as<double>(), live_.as<int>(),
                                                   xhat_.as<C>() + (size_t)j * N_ * NB, nullptr,
                                                   partial_.as<double>(), N_, K_, NB, Wh, 1, nullptr);
      });
      launch(kFamOther, [&] {
        per_image_reduce<<<N_, 256, 0, st_>>>(partial_.as<double>(), tiles_, 0.5 / D, odata_.as<double>());
      });
      CK(cudaMemcpyAsync(part.data(), odata_.p, sizeof(double) * N_, cudaMemcpyDeviceToHost, st_));
      CK(cudaStreamSynchronize(st_));
      for (int n = 0; n < N_; ++n) data[n] += part[n];
    }
  }

  void learning_data_term(const double* d, double* out) override {
    std::vector<double> data;
    data_terms(d ? d : dict_.data(), data);
    double s = 0.0;
    for (double v : data) s += v;
    reduce_host(&s, 1);
    *out = s;
  }

  // per-image objective of a map source (coding candidates in u, or the accepted maps)
  template <int MODE>
  void objective_pass(const C* dhat, std::vector<double>& data, std::vector<double>& l1) {
    coding_launch<MODE>(dhat, 0, N_);
    if (J_ > 1) {
      launch(kFamOther, [&] {
        tc_objective<R><<<N_, 256, 0, st_>>>(what_.as<C>(), dhat, xhat_.as<C>(), (size_t)N_ * NB, sums_.as<double>(),
                                             G_ * CLN, K_, J_, NB, Wh, 1.0 / D, cfg_.beta, odata_.as<double>(),
                                             ol1_.as<double>());
      });
    } else {
      launch(kFamOther, [&] {
        objective_reduce<R><<<N_, 256, 0, st_>>>(part_.as<C>(), sums_.as<double>(), xhat_.as<C>(), G_, G_ * CLN,
                                                 NB, Wh, 1.0 / D, cfg_.beta, odata_.as<double>(), ol1_.as<double>());
      });
    }
    data.resize(N_);
    l1.resize(N_);
    CK(cudaMemcpyAsync(data.data(), odata_.p, sizeof(double) * N_, cudaMemcpyDeviceToHost, st_));
    CK(cudaMemcpyAsync(l1.data(), ol1_.p, sizeof(double) * N_, cudaMemcpyDeviceToHost, st_));
    CK(cudaStreamSynchronize(st_));
  }

  void objective(const double* d, dcsc_objective* per_image) override {
    const C* dh = dhat_.as<C>();
    if (d) {
      upload_dict_spectra(d, dcand_.as<C>());
      dh = dcand_.as<C>();
    }
    std::vector<double> data, l1;
    objective_pass<kPassMaps>(dh, data, l1);
    for (int n = 0; n < N_; ++n) {
      per_image[n].data_term = data[n];
      per_image[n].l1_term = l1[n];
      per_image[n].total = data[n] + l1[n];
      per_image[n].residual_norm = std::sqrt(2.0 * data[n]);
      if (!std::isfinite(per_image[n].total)) throw NumErr("objective is not finite");
    }
  }

  // reconstruct (objective.cpp:39-57) of the accepted maps of images [n0, n1)
  // with `d` (NULL = the context dictionary): out is (n1-n0) x J x D
  void reconstruct(const double* d, int n0, int n1, double* out) override {
    check_range(n0, n1);
    const int cnt = n1 - n0;
    const C* dh = dhat_.as<C>();
    if (d) {
      require_finite(d, (size_t)K_ * J_ * M_, "dictionary");
      upload_dict_spectra(d, dcand_.as<C>());
      dh = dcand_.as<C>();
    }
    coding_launch<kPassMaps>(dh, n0, cnt);
    DevMem spec, sp;
    spec.alloc(sizeof(C) * (size_t)cnt * J_ * NB);
    sp.alloc(sizeof(double) * (size_t)cnt * J_ * D);
    launch(kFamOther, [&] {
      recon_spectrum<R><<<dim3((NB + 255) / 256, cnt), 256, 0, st_>>>(
          part_.as<C>() + (size_t)n0 * G_ * NB, what_.as<C>() ? what_.as<C>() + (size_t)n0 * K_ * NB : nullptr, dh,
          spec.as<C>(), J_, K_, G_, NB);
    });
    c2r<double>(spec.as<C>(), NB, sp.as<double>(), D, cnt * J_);
    CK(cudaMemcpyAsync(out, sp.p, sp.bytes, cudaMemcpyDeviceToHost, st_));
    CK(cudaStreamSynchronize(st_));
  }

  // run_csc (pipeline.cpp:158-301) from init_variables, split into a
  // begin (init_variables + the initial per-image objectives, :169-213) and
  // one outer iteration per step (:216-299), so a caller can take the outer
  // loop one iteration at a time (bench, per-outer parity dumps) without
  // re-initialising
  void run_begin() override {
    init_variables();
    run_img_.assign(N_, dcsc_objective{});
    double dsum = 0.0;
    for (int n = 0; n < N_; ++n) {
      run_img_[n].data_term = 0.5 * xnorm2_[n];  // maps are zero: reconstruct = 0
      run_img_[n].l1_term = 0.0;
      run_img_[n].total = run_img_[n].data_term;
      run_img_[n].residual_norm = std::sqrt(xnorm2_[n]);
      dsum += run_img_[n].data_term;
    }
    reduce_host(&dsum, 1);
    run_prev_total_ = dsum;
    run_outer_ = 0;
    run_ready_ = true;
  }

  // one outer iteration; rows[0] = coding row, rows[1] = learning row;
  // returns 1 when the run's stop test (pipeline.cpp:290-298) is met
  int run_step(dcsc_trace_row* rows) override {
    if (!run_ready_) throw InvErr("run_step before run_begin");
    const int outer = ++run_outer_;
    std::vector<dcsc_objective>& img = run_img_;
    std::vector<dcsc_coding_stats> cs(N_);
    std::vector<int> acc(N_);
    const double w0 = now_ms();
    coding(0, N_, cs.data());
    const double coding_ms = now_ms() - w0;
    std::vector<double> cdata, cl1;
    objective_pass<kPassObjective>(dhat_.as<C>(), cdata, cl1);
    long admm_total = 0;
    for (int n = 0; n < N_; ++n) {
      admm_total += cs[n].admm_iters;
      const double tot = cdata[n] + cl1[n];
      if (!std::isfinite(tot))
        throw NumErr("non-finite objective at outer iteration " + std::to_string(outer) + ", coding phase");
      acc[n] = tot <= img[n].total ? 1 : 0;
      if (acc[n]) img[n] = {cdata[n], cl1[n], tot, std::sqrt(2.0 * cdata[n])};
    }
    double zc2 = 0.0, zn2 = 0.0;
    long l0 = 0;
    accept(acc, zc2, zn2, l0);
    run_acc_ = acc;
    zhat_valid_ = false;
    zf_valid_ = false;
    dcsc_objective after{};
    for (int n = 0; n < N_; ++n) {
      after.data_term += img[n].data_term;
      after.l1_term += img[n].l1_term;
      after.residual_norm += img[n].residual_norm * img[n].residual_norm;
    }
    {
      double s[7] = {after.data_term, after.l1_term, after.residual_norm, (double)admm_total, zc2, zn2, (double)l0};
      reduce_host(s, 7);
      after.data_term = s[0];
      after.l1_term = s[1];
      after.residual_norm = s[2];
      admm_total = (long)s[3];
      zc2 = s[4];
      zn2 = s[5];
      l0 = (long)s[6];
    }
    after.total = after.data_term + after.l1_term;
    after.residual_norm = std::sqrt(after.residual_norm);
    const double w1 = now_ms();
    rows[0] = {outer, 0, after.total, after.data_term, after.l1_term, after.residual_norm,
               admm_total, 0, 0, coding_ms, w1 - w0, l0};

    dcsc_learning_stats ls{};
    std::vector<double> dc((size_t)K_ * J_ * M_);
    learning(dc.data(), &ls);
    const double learning_ms = now_ms() - w1;
    std::vector<double> data;
    data_terms(dc.data(), data);
    double cand = 0.0;
    for (double v : data) cand += v;
    reduce_host(&cand, 1);
    if (!std::isfinite(cand + after.l1_term))
      throw NumErr("non-finite objective at outer iteration " + std::to_string(outer) + ", learning phase");
    dcsc_objective afterl = after;
    double dc2 = 0.0, dn2 = 0.0;
    run_dacc_ = cand <= after.data_term ? 1 : 0;
    if (cand <= after.data_term) {
      for (size_t i = 0; i < dc.size(); ++i) {
        const double dl = dc[i] - dict_[i];
        dc2 += dl * dl;
      }
      set_dictionary(dc.data());
      afterl.data_term = cand;
      afterl.total = cand + after.l1_term;
      afterl.residual_norm = std::sqrt(2.0 * cand);
      for (int n = 0; n < N_; ++n)
        img[n] = {data[n], img[n].l1_term, data[n] + img[n].l1_term, std::sqrt(2.0 * data[n])};
    }
    for (double v : dict_) dn2 += v * v;
    const double w2 = now_ms();
    rows[1] = {outer, 1, afterl.total, afterl.data_term, afterl.l1_term, afterl.residual_norm,
               0, ls.cg_iters, ls.mu_iters, learning_ms, w2 - w1, l0};
    const double prev = run_prev_total_;
    const double obj_change = std::abs(prev - afterl.total) / std::max(std::abs(prev), 1e-30);
    const double z_change = std::sqrt(zc2) / std::max(std::sqrt(zn2), 1.0);
    const double d_change = std::sqrt(dc2) / std::max(std::sqrt(dn2), 1.0);
    run_prev_total_ = afterl.total;
    return (obj_change <= cfg_.tol && z_change <= cfg_.tol && d_change <= cfg_.tol) ? 1 : 0;
  }

  // acceptance decisions of the last run_step: per image (pipeline.cpp:236), dictionary (:272)
  void run_accepts(int* image_accept, int* dict_accept) override {
    if (image_accept) std::copy(run_acc_.begin(), run_acc_.end(), image_accept);
    if (dict_accept) *dict_accept = run_dacc_;
  }

  void run(int max_outer, dcsc_trace_row* rows, int* n_rows, int* converged) override {
    *n_rows = 0;
    *converged = 0;
    run_begin();
    for (int outer = 1; outer <= max_outer; ++outer) {
      const int done = run_step(rows + 2 * (outer - 1));
      *n_rows = 2 * outer;
      if (done) {
        *converged = 1;
        break;
      }
    }
  }

  // ---------------------------------------------------- frequency-sharded learning
  // (BASELINE.json north_star). Rank r owns the half-spectrum
  // bins [b0_r, b0_r + nbl_r), b0_r = r NB / world, for ALL images: after
  // coding, one all-to-all (grouped ncclSend/ncclRecv) moves z_hat from
  // image-major [N_r][K][NB] to frequency-major [N_tot][K][nbl] (x_hat once per
  // set_signals). The contractions (learning.cpp:97-121) and the CG vector
  // updates then run on the local bins of every image; the mask step needs all
  // bins of c_k, and the crop of an inverse DFT is linear, so each rank crops
  // the inverse DFT of its local bins (zero elsewhere) and the K x M crops are
  // all-reduced as in the image-sharded layout (d_recover identically); the
  // CG scalars (Parseval with the bins' global weights) and the per-image
  // learning data terms (objective.cpp:83-95) are all-reduced.
  void set_learning_layout(int freq) override {
    freq_ = false;
    if (!freq || !multi()) return;
    if (J_ != 1) throw DimErr("frequency-sharded learning supports single-channel data");
    const int world = red_->world, rank = red_->rank;
    std::vector<double> nr(world, 0.0);
    nr[rank] = N_;
    reduce_host(nr.data(), world);
    fn_rank_.assign(world, 0);
    fntot_ = 0;
    fnoff_ = 0;
    for (int q = 0; q < world; ++q) {
      fn_rank_[q] = (long)nr[q];
      if (q < rank) fnoff_ += (int)fn_rank_[q];
      fntot_ += (int)fn_rank_[q];
    }
    fb0_ = (int)((long)rank * NB / world);
    fnbl_ = (int)((long)(rank + 1) * NB / world) - fb0_;
    ftiles_ = (fnbl_ + TBV - 1) / TBV;
    const size_t vec = (size_t)fntot_ * fnbl_;
    zf_.alloc(sizeof(C) * vec * K_);
    xf_.alloc(sizeof(C) * vec);
    gf_.alloc(sizeof(C) * vec);
    rf_.alloc(sizeof(C) * vec);
    pf_.alloc(sizeof(C) * vec);
    apf_.alloc(sizeof(C) * vec);
    fsend_.alloc(sizeof(C) * (size_t)N_ * K_ * NB);
    fpart_.alloc(sizeof(double) * std::max((size_t)fntot_ * ftiles_, (vec + TBV - 1) / TBV));
    fodata_.alloc(sizeof(double) * fntot_);
    {
      int sms = 148;
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, o_.device);
      const long base = (long)ftiles_ * ((K_ + DCSC_KC - 1) / DCSC_KC);
      const double want = std::max(1.0, 4.0 * sms / (double)base);
      const long p2 = 1L << (int)std::lround(std::log2(want));
      fcsplit_ = (int)std::max(1L, std::min({p2, 64L, (long)fntot_}));
    }
    fcpart_.alloc(sizeof(double2) * (size_t)fcsplit_ * K_ * fnbl_);
    device_bytes += zf_.bytes + 5 * xf_.bytes + fsend_.bytes + fcpart_.bytes;
    CK(cudaMemsetAsync(gf_.p, 0, gf_.bytes, st_));
    CK(cudaStreamSynchronize(st_));
    zf_valid_ = xf_valid_ = false;
    freq_ = true;
  }

  // image-major [planes_r][NB] on every rank -> frequency-major [sum_r planes_r][nbl]
  // (`per_image` planes per image)
  void to_freq(const C* src, C* dst, int per_image) {
    const int world = red_->world;
    const size_t planes = (size_t)N_ * per_image;
    launch(kFamOther, [&] {
      pack_bins<C><<<1184, 256, 0, st_>>>(src, fsend_.as<C>(), planes, NB, world);
    });
    std::vector<size_t> sb(world), rb(world);
    for (int q = 0; q < world; ++q) {
      const long b0 = (long)q * NB / world, b1 = (long)(q + 1) * NB / world;
      sb[q] = sizeof(C) * planes * (size_t)(b1 - b0);
      rb[q] = sizeof(C) * (size_t)fn_rank_[q] * per_image * (size_t)fnbl_;
    }
    red_->alltoall(fsend_.p, sb.data(), dst, rb.data(), st_);
  }

  void freq_operands() {
    build_zhat();
    if (!zf_valid_) {
      to_freq(zhat_.as<C>(), zf_.as<C>(), K_);
      zf_valid_ = true;
    }
    if (!xf_valid_) {
      to_freq(xhat_.as<C>(), xf_.as<C>(), 1);
      xf_valid_ = true;
    }
  }

  // c_k on the local bins of every image -> full K x NB spectra (zero elsewhere)
  void correlate_freq(const C* v, const int* done) {
    constexpr int KC = DCSC_KC;
    const dim3 g1(ftiles_, (K_ + KC - 1) / KC, fcsplit_);
    launch(kFamContract, [&] {
      contract_c<R, KC><<<g1, TBV, 0, st_>>>(zf_.as<C>(), v, fcpart_.as<double2>(), live_.as<int>(), fntot_, K_,
                                             fnbl_, done);
    });
    const size_t knbl = (size_t)K_ * fnbl_;
    launch(kFamOther, [&] {
      contract_c_reduce_off<R><<<(unsigned)((knbl + 255) / 256), 256, 0, st_>>>(
          fcpart_.as<double2>(), cvec_.as<C>(), fcsplit_, knbl, done, fnbl_, NB, fb0_);
    });
  }

  void apply_freq(const C* v, C* out, const int* done) {
    correlate_freq(v, done);
    mask_crop(2, done);  // crops of the local-bin inverse DFTs, summed over ranks
    launch(kFamMask, [&] { launch_filters(K_, st_, dd_.as<double>(), mh_, mw_, phat_.as<C>(), dtw_.as<C>()); });
    launch(kFamContract, [&] {
      contract_out<R, TBV><<<dim3(ftiles_, fntot_), TBV, 0, st_>>>(
          zf_.as<C>(), phat_.as<C>() + fb0_, dwk_.as<double>(), live_.as<int>(), v, out, fpart_.as<double>(), fntot_,
          K_, fnbl_, Wh, 0, done, nullptr, nullptr, 0.0, fb0_, NB);
    });
  }

  // gamma_solve (learning.cpp:136-185) on the local bins of all images
  void gamma_solve_freq(double bnorm, int& iters, bool& converged) {
    iters = 0;
    converged = false;
    const size_t total = (size_t)fntot_ * fnbl_;
    const unsigned vb = (unsigned)((total + TBV - 1) / TBV);
    if (bnorm == 0.0) {
      CK(cudaMemsetAsync(gf_.p, 0, gf_.bytes, st_));
      converged = true;
      return;
    }
    CgState init{};
    init.bnorm = bnorm;
    init.tol = cfg_.cg_tol;
    init.max_iters = cfg_.cg_max;
    CK(cudaMemcpyAsync(cg_.p, &init, sizeof(CgState), cudaMemcpyHostToDevice, st_));
    apply_freq(gf_.as<C>(), apf_.as<C>(), nullptr);
    launch(kFamOther, [&] {
      cg_init<R, TBV><<<vb, TBV, 0, st_>>>(xf_.as<C>(), apf_.as<C>(), rf_.as<C>(), pf_.as<C>(),
                                            fpart_.as<double>(), total, fnbl_, Wh, fb0_);
    });
    const double invD = 1.0 / D;
    cg_step(fpart_.as<double>(), (int)vb, invD, 0);
    const int* done = &cg_.as<CgState>()->done;
    CgState s = read_cg();
    int issued = 0, chunk = 2;
    while (!s.done && issued < cfg_.cg_max) {
      const int n = std::min(chunk, cfg_.cg_max - issued);
      for (int c = 0; c < n; ++c) {
        apply_freq(pf_.as<C>(), apf_.as<C>(), done);
        cg_step(fpart_.as<double>(), fntot_ * ftiles_, invD, 1);
        launch(kFamOther, [&] {
          cg_update<R, TBV><<<vb, TBV, 0, st_>>>(gf_.as<C>(), rf_.as<C>(), pf_.as<C>(), apf_.as<C>(),
                                                  cg_.as<CgState>(), fpart_.as<double>(), total, fnbl_, Wh, nullptr,
                                                  invD, fb0_);
        });
        cg_step(fpart_.as<double>(), (int)vb, invD, 2);
        launch(kFamOther, [&] {
          cg_pupdate<R, TBV><<<vb, TBV, 0, st_>>>(rf_.as<C>(), pf_.as<C>(), cg_.as<CgState>(), total);
        });
      }
      issued += n;
      chunk = std::min(chunk * 2, 8);
      s = read_cg();
    }
    iters = s.iters;
    converged = s.converged != 0;
  }

  // solve_learning (learning.cpp:227-355), frequency-sharded (J = 1)
  void learning_freq(double* d_out, dcsc_learning_stats* st) {
    dcsc_learning_stats ls{};
    if ((int)mu_.size() != K_) mu_.assign(K_, 1.0);
    freq_operands();
    CK(cudaMemsetAsync(cvec_.p, 0, cvec_.bytes, st_));  // bins outside [b0, b0 + nbl) stay zero
    int n_live = 0;
    for (int k = 0; k < K_; ++k) n_live += live_h_[k] ? 1 : 0;
    ls.n_dead = K_ - n_live;
    if (n_live == 0) {  // learning.cpp:258-270
      ls.degenerate = 1;
      CK(cudaMemsetAsync(gf_.p, 0, gf_.bytes, st_));
      CK(cudaStreamSynchronize(st_));
      std::fill(d_out, d_out + (size_t)K_ * M_, 0.0);
      if (st) *st = ls;
      return;
    }
    double bnorm = 0.0;
    for (int n = 0; n < N_; ++n) bnorm += xnorm2c_[n];
    reduce_host(&bnorm, 1);
    bnorm = std::sqrt(bnorm);
    std::vector<double> part, norms(K_, 0.0);
    bool clamped = false;
    for (int iter = 1; iter <= cfg_.max_mu_iters; ++iter) {
      clamped = false;
      for (int k = 0; k < K_; ++k)
        if (mu_[k] < cfg_.mu_floor) {
          mu_[k] = cfg_.mu_floor;
          clamped = true;
        }
      upload_mu();
      int cg_iters = 0;
      bool cg_conv = false;
      gamma_solve_freq(bnorm, cg_iters, cg_conv);
      if (!cg_conv) ls.cg_budget_hit = 1;
      ls.cg_iters += cg_iters;
      if (iter == 1) ls.cg_iters_first = cg_iters;
      correlate_freq(gf_.as<C>(), nullptr);  // d_recover (learning.cpp:187-216)
      mask_crop(1, nullptr);
      part.resize((size_t)K_ * M_);
      CK(cudaMemcpyAsync(part.data(), dd_.p, sizeof(double) * K_ * M_, cudaMemcpyDeviceToHost, st_));
      CK(cudaStreamSynchronize(st_));
      for (int k = 0; k < K_; ++k) {
        double sq = 0.0;
        for (int i = 0; i < M_; ++i) sq += part[(size_t)k * M_ + i] * part[(size_t)k * M_ + i];
        norms[k] = std::sqrt(sq);
      }
      ls.mu_iters = iter;
      bool settled = true;
      for (int k = 0; k < K_; ++k) {
        const bool at_boundary = std::abs(norms[k] - 1.0) <= kFilterNormTol;
        const bool inactive = mu_[k] <= cfg_.mu_floor * (1.0 + 1e-9) && norms[k] < 1.0;
        if (!at_boundary && !inactive) {
          settled = false;
          break;
        }
      }
      if (settled) {
        ls.converged = 1;
        break;
      }
      if (iter < cfg_.max_mu_iters)
        for (int k = 0; k < K_; ++k) mu_[k] = std::max(mu_[k] * norms[k], cfg_.mu_floor);
    }
    ls.mu_clamped = clamped ? 1 : 0;
    for (int k = 0; k < K_; ++k) {
      double scale = 1.0;
      if (norms[k] > 1.0) {
        scale = 1.0 / norms[k];
        ++ls.rescaled_filters;
      }
      for (int i = 0; i < M_; ++i) d_out[(size_t)k * M_ + i] = scale * part[(size_t)k * M_ + i];
    }
    if (st) *st = ls;
  }

  // per-image learning data terms (objective.cpp:83-95) of this rank's images
  void data_terms_freq(const double* d, std::vector<double>& data) {
    freq_operands();
    upload_dict_spectra(d, dcand_.as<C>());
    launch(kFamContract, [&] {
      contract_out<R, TBV><<<dim3(ftiles_, fntot_), TBV, 0, st_>>>(
          zf_.as<C>(), dcand_.as<C>() + fb0_, dwk_.as<double>(), live_.as<int>(), xf_.as<C>(), nullptr,
          fpart_.as<double>(), fntot_, K_, fnbl_, Wh, 1, nullptr, nullptr, nullptr, 0.0, fb0_, NB);
    });
    launch(kFamOther, [&] {
      per_image_reduce<<<fntot_, 256, 0, st_>>>(fpart_.as<double>(), ftiles_, 0.5 / D, fodata_.as<double>());
    });
    red_->allreduce(fodata_.as<double>(), fntot_, st_);
    std::vector<double> all(fntot_);
    CK(cudaMemcpyAsync(all.data(), fodata_.p, sizeof(double) * fntot_, cudaMemcpyDeviceToHost, st_));
    CK(cudaStreamSynchronize(st_));
    data.assign(all.begin() + fnoff_, all.begin() + fnoff_ + N_);
  }

  // accept-only-descent for the coding half-step (pipeline.cpp:231-247)
  void accept(const std::vector<int>& acc, double& zc2, double& zn2, long& l0) {
    CK(cudaMemcpyAsync(accept_.p, acc.data(), sizeof(int) * N_, cudaMemcpyHostToDevice, st_));
    const dim3 g(accept_chunks_, N_);
    launch(kFamOther, [&] {
      accept_maps<R, TBV, !CLU><<<g, TBV, 0, st_>>>(u_.as<R>(), maps_.as<R>(), accept_.as<int>(), (size_t)K_ * D,
                                                     cfg_.rho, cfg_.beta, partial_.as<double>(),
                                                     partial2_.as<double>(), l0_.as<unsigned long long>(), P::H, P::W);
    });
    const size_t cnt = (size_t)N_ * accept_chunks_;
    std::vector<double> a(cnt), b(cnt);
    std::vector<unsigned long long> c(cnt);
    CK(cudaMemcpyAsync(a.data(), partial_.p, sizeof(double) * cnt, cudaMemcpyDeviceToHost, st_));
    CK(cudaMemcpyAsync(b.data(), partial2_.p, sizeof(double) * cnt, cudaMemcpyDeviceToHost, st_));
    CK(cudaMemcpyAsync(c.data(), l0_.p, sizeof(unsigned long long) * cnt, cudaMemcpyDeviceToHost, st_));
    CK(cudaStreamSynchronize(st_));
    zc2 = zn2 = 0.0;
    l0 = 0;
    for (size_t i = 0; i < cnt; ++i) {
      zc2 += a[i];
      zn2 += b[i];
      l0 += (long)c[i];
    }
  }

  void synchronize() override { CK(cudaStreamSynchronize(st_)); }

  void set_profiling(int on) override {
    CK(cudaStreamSynchronize(st_));
    prof_.clear();
    evused_ = 0;
    profiling_ = on;  // 1: every launch, 2: coding-pass launches only, 3: coding pass + z_hat streams
  }

  void kernel_time(int fam, double* ms, long long* n) override {
    CK(cudaStreamSynchronize(st_));
    double t = 0.0;
    long long c = 0;
    for (auto& e : prof_)
      if (e.fam == fam) {
        float x = 0.f;
        CK(cudaEventElapsedTime(&x, e.a, e.b));
        t += x;
        ++c;
      }
    *ms = t;
    *n = c;
  }

  void event_mark(int slot) override {
    if (slot < 0 || slot >= 64) throw InvErr("event slot out of range");
    if ((int)marks_.size() < 64) marks_.resize(64, nullptr);
    if (!marks_[slot]) CK(cudaEventCreate(&marks_[slot]));
    CK(cudaEventRecord(marks_[slot], st_));
  }

  double event_elapsed(int a, int b) override {
    if (a < 0 || b < 0 || a >= (int)marks_.size() || b >= (int)marks_.size() || !marks_[a] || !marks_[b])
      throw InvErr("event slot not marked");
    CK(cudaEventSynchronize(marks_[b]));
    float x = 0.f;
    CK(cudaEventElapsedTime(&x, marks_[a], marks_[b]));
    return x;
  }

 private:
  struct Prof {
    int fam;
    cudaEvent_t a, b;
  };
  dcsc_cuda_opts o_;
  dcsc_solver_config cfg_;
  int N_, K_, J_ = 1, mh_, mw_, M_, G_, kpg_, tiles_, accept_chunks_, csplit_ = 1, fused_rows_ = 1184;
  bool no_cg_fuse_ = false;
  cudaStream_t st_ = nullptr;
  cudaStream_t st2_ = nullptr;  // second half of a tensor-core coding batch
  void* pin_ = nullptr;
  DevMem dtw_, x_, xhat_, dhat_, dcand_, sigma_, u_, maps_, lamhat_, lam_, part_, sums_, conv_, img_, dual_,
      infeas_, resc_, cnt_, odata_, ol1_, accept_, gam_, r_, p_, ap_, cvec_, phat_, live_, dmu_, dwk_, dd_, ddict_, cg_,
      partial_, partial2_, l0_, zhat_, cpart_, hred_, ginv_, what_, cgcnt_, dhat_rb_, theta0_;
  std::vector<char> t0_pending_;  // per image: theta0_ holds a not ADMM-consistent warm theta
  // frequency-sharded learning (set_learning_layout)
  bool freq_ = false, zf_valid_ = false, xf_valid_ = false;
  int fb0_ = 0, fnbl_ = 0, fntot_ = 0, fnoff_ = 0, ftiles_ = 0, fcsplit_ = 1;
  std::vector<long> fn_rank_;
  DevMem zf_, xf_, gf_, rf_, pf_, apf_, fsend_, fpart_, fodata_, fcpart_;
  bool use_theta0_ = false;
  // tensor-core coding pass (kernels_tc.cuh)
  bool tc_ = false, tc_force_ = false;
  int tc_kf_ = 128, tc_grid_ = 148;
  float tc_dscale_ = 1.f, tc_tbound_ = 0.f;
  DevMem tlam16_, tlscale_, tdsplit_, tspart_, tbsums_, tu_, tupd_, tzmax_;
  CUtensorMap tc_umap_{};
  std::vector<double> dict_, mu_, xnorm2_, xnorm2c_, xs_host_, dstage_;
  std::vector<int> degen_;  // per image: normalisation met a constant input
  C* xh_ch_ = nullptr;   // learning view: x_hat of the current channel (N x NB)
  C* gam_ch_ = nullptr;  // learning view: gamma_hat of the current channel
  std::vector<int> live_h_;
  std::vector<char> u_zero_;  // per image: ADMM state known to be exactly zero
  void* xstage_ = nullptr;    // pinned staging of the signals (host -> device)
  size_t xstage_bytes_ = 0;
  bool dict_zero_ = false, zhat_valid_ = false;
  int profiling_ = 0;
  std::vector<Prof> prof_;
  std::vector<dcsc_objective> run_img_;  // per-image objectives of the run in progress
  double run_prev_total_ = 0.0;
  int run_outer_ = 0;
  bool run_ready_ = false;
  std::vector<int> run_acc_;
  int run_dacc_ = 0;
  std::vector<cudaEvent_t> evpool_;
  size_t evused_ = 0;
  std::vector<cudaEvent_t> marks_;
};

// Standalone half-spectrum DFTs
template <class R, int H, int W>
void dft_batch(bool inverse, int batch, const double* in, double* out) {
  using E = Engine<R, H, W>;
  using P = typename E::P;
  using C = cx<R>;
  constexpr int NB = P::NB, D = P::D;
  static bool attr = false;
  if (!attr) {
    E::set_attributes();
    attr = true;
  }
  std::vector<C> tw(P::TW_LEN);
  fill_twiddles<P>(tw.data());
  DevMem dtw, din, dout, spec;
  dtw.alloc(sizeof(C) * P::TW_LEN);
  CK(cudaMemcpy(dtw.p, tw.data(), dtw.bytes, cudaMemcpyHostToDevice));
  spec.alloc(sizeof(C) * (size_t)batch * NB);
  // FP32 families run the storage-precision kernels the engine uses (the
  // input rounded to float once, as set_signals does; the output widened)
  constexpr bool narrow = !std::is_same<R, double>::value;
  if (!inverse) {
    if constexpr (narrow) {
      std::vector<R> hin((size_t)batch * D);
      for (size_t i = 0; i < hin.size(); ++i) hin[i] = R(in[i]);
      din.alloc(sizeof(R) * hin.size());
      CK(cudaMemcpy(din.p, hin.data(), din.bytes, cudaMemcpyHostToDevice));
      E::template launch_r2c<R>(batch, 0, din.as<R>(), D, spec.as<C>(), NB, dtw.as<C>(), nullptr, 1);
    } else {
      din.alloc(sizeof(double) * (size_t)batch * D);
      CK(cudaMemcpy(din.p, in, din.bytes, cudaMemcpyHostToDevice));
      E::template launch_r2c<double>(batch, 0, din.as<double>(), D, spec.as<C>(), NB, dtw.as<C>(), nullptr, 1);
    }
    CK(cudaGetLastError());
    std::vector<C> h((size_t)batch * NB);
    CK(cudaMemcpy(h.data(), spec.p, spec.bytes, cudaMemcpyDeviceToHost));
    for (size_t i = 0; i < h.size(); ++i) {
      out[2 * i] = h[i].x;
      out[2 * i + 1] = h[i].y;
    }
  } else {
    std::vector<C> h((size_t)batch * NB);
    for (size_t i = 0; i < h.size(); ++i) h[i] = mk<C>(R(in[2 * i]), R(in[2 * i + 1]));
    CK(cudaMemcpy(spec.p, h.data(), spec.bytes, cudaMemcpyHostToDevice));
    if constexpr (narrow) {
      dout.alloc(sizeof(R) * (size_t)batch * D);
      E::template launch_c2r<R>(batch, 0, spec.as<C>(), NB, dout.as<R>(), D, dtw.as<C>());
      CK(cudaGetLastError());
      std::vector<R> hout((size_t)batch * D);
      CK(cudaMemcpy(hout.data(), dout.p, dout.bytes, cudaMemcpyDeviceToHost));
      for (size_t i = 0; i < hout.size(); ++i) out[i] = double(hout[i]);
    } else {
      dout.alloc(sizeof(double) * (size_t)batch * D);
      E::template launch_c2r<double>(batch, 0, spec.as<C>(), NB, dout.as<double>(), D, dtw.as<C>());
      CK(cudaGetLastError());
      CK(cudaMemcpy(out, dout.p, dout.bytes, cudaMemcpyDeviceToHost));
    }
  }
  CK(cudaDeviceSynchronize());
}

// Device-timed batched r2c and c2r of `batch` planes (random data), for the
// cuFFT comparator (scripts/fft_comparator.py). Returns the mean ms per call.
template <class R, int H, int W>
void fft_timing(int batch, int iters, double* ms_r2c, double* ms_c2r) {
  using E = Engine<R, H, W>;
  using P = typename E::P;
  using C = cx<R>;
  constexpr int NB = P::NB, D = P::D;
  E::set_attributes();
  std::vector<C> tw(P::TW_LEN);
  fill_twiddles<P>(tw.data());
  DevMem dtw, real, spec;
  dtw.alloc(sizeof(C) * P::TW_LEN);
  CK(cudaMemcpy(dtw.p, tw.data(), dtw.bytes, cudaMemcpyHostToDevice));
  real.alloc(sizeof(R) * (size_t)batch * D);
  spec.alloc(sizeof(C) * (size_t)batch * NB);
  std::vector<R> h((size_t)batch * D);
  std::mt19937_64 rng(1);
  for (auto& v : h) v = R(static_cast<double>(rng() >> 11) * 0x1.0p-53 - 0.5);
  CK(cudaMemcpy(real.p, h.data(), real.bytes, cudaMemcpyHostToDevice));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  auto time_it = [&](auto&& f) {
    for (int i = 0; i < 3; ++i) f();
    CK(cudaEventRecord(a));
    for (int i = 0; i < iters; ++i) f();
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, a, b));
    return (double)ms / iters;
  };
  *ms_r2c = time_it([&] {
    E::template launch_r2c<R>(batch, 0, real.as<R>(), D, spec.as<C>(), NB, dtw.as<C>(), nullptr, 1);
  });
  *ms_c2r = time_it([&] { E::template launch_c2r<R>(batch, 0, spec.as<C>(), NB, real.as<R>(), D, dtw.as<C>()); });
  CK(cudaGetLastError());
  cudaEventDestroy(a);
  cudaEventDestroy(b);
}

}  // namespace

#define DCSC_ENGINE_INSTANTIATE(Rt, Hh, Ww)                                                    \
  namespace dcsc_engine {                                                                      \
  std::unique_ptr<EngineBase> make_engine_##Rt##_##Hh##_##Ww(const dcsc_cuda_opts& o) {         \
    return std::make_unique<Engine<Rt, Hh, Ww>>(o);                                            \
  }                                                                                            \
  void dft_batch_##Rt##_##Hh##_##Ww(bool inverse, int batch, const double* in, double* out) {   \
    dft_batch<Rt, Hh, Ww>(inverse, batch, in, out);                                            \
  }                                                                                            \
  void fft_timing_##Rt##_##Hh##_##Ww(int batch, int iters, double* ms_r2c, double* ms_c2r) {   \
    fft_timing<Rt, Hh, Ww>(batch, iters, ms_r2c, ms_c2r);                                      \
  }                                                                                            \
  }

// A grid plugin: the engine of one more (precision, H, W) as its own shared library, found by
// engine.cu's dispatcher (find_plugin) through these four C symbols.
#define DCSC_GRID_PLUGIN(Rt, Hh, Ww)                                                              \
  DCSC_ENGINE_INSTANTIATE(Rt, Hh, Ww)                                                              \
  extern "C" void dcsc_grid_info(int* prec, int* h, int* w) {                                      \
    *prec = sizeof(Rt) == 8 ? 64 : 32;                                                             \
    *h = Hh;                                                                                       \
    *w = Ww;                                                                                       \
  }                                                                                                \
  extern "C" void* dcsc_grid_make(const dcsc_cuda_opts* o) {                                       \
    return static_cast<dcsc_engine::EngineBase*>(dcsc_engine::make_engine_##Rt##_##Hh##_##Ww(*o).release()); \
  }                                                                                                \
  extern "C" void dcsc_grid_dft(int inverse, int batch, const double* in, double* out) {           \
    dcsc_engine::dft_batch_##Rt##_##Hh##_##Ww(inverse != 0, batch, in, out);                       \
  }                                                                                                \
  extern "C" void dcsc_grid_fft_timing(int batch, int iters, double* ms_r2c, double* ms_c2r) {     \
    dcsc_engine::fft_timing_##Rt##_##Hh##_##Ww(batch, iters, ms_r2c, ms_c2r);                      \
  }
