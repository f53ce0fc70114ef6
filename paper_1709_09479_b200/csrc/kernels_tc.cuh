// Spatial-domain ADMM coding iteration on the 5th-generation tensor cores.
//
// The reference forms, per ADMM iteration and filter k (coding.cpp:223-263),
//   t_k = iDFT(conj(d_hat_k) lambda_hat)          (correlate, coding.cpp:77-86)
//   prox on (theta, z) with t_k                    (coding.cpp:237-251)
//   acc = sum_k d_hat_k DFT(theta_k + z_k / rho)   (lambda_from_w, coding.cpp:25-37)
// With the filters' m x m support at the plane corner (filter_spectrum) the two
// spectral products are circular correlations / convolutions with m*m taps:
//   t_k[p] = sum_o d_k[o] lambda[p + o],  s[p] = sum_k sum_o d_k[o] w_k[p - o],
// and DFT(s) = sum_k d_hat_k w_hat_k exactly. Over all filters at once they are
// two GEMMs per tile of 128 pixels (a row segment, a row pair at W = 64, or one
// row with idle lanes for 64 < W < 128):
//   GEMM-1  T[p][k] = sum_o L[p][o] D[k][o]    L = im2col(lambda) (M=128, N=KF, K=TP taps)
//   GEMM-2  Z[p][o] = sum_k W[p][k] D[k][o]    W = w of the tile   (M=128, N=TP taps, K=KF)
// followed by the col2im sum s[p + o] += Z[p][o]. Both run on tcgen05 with the
// pixel operand in tensor memory and the dictionary in shared memory (one
// copy serves GEMM-1 K-major and GEMM-2 MN-major), accumulating in FP32; each
// FP32 operand is split into two scaled f16 (x*s = hi + lo + O(2^-22 |x*s|)) and
// three products (hi*hi + hi*lo + lo*hi) restore FP32-level accuracy. lambda
// is scaled per image, the dictionary per dictionary, w per pixel (a row of W).
// The per-image FFT work that remains is one r2c of s and one c2r of lambda_hat
// per iteration instead of a c2r + r2c per filter.
//
// Persistent kernel, one CTA per SM, 10 warps: warp 0 issues the GEMMs (a
// converged warp, one elected lane, uniform operands); warps 1-8 are two
// epilogue groups of 4 warps (one per TMEM lane quarter = 32 pixels), each
// owning one of two tensor-memory slots (256 columns: A operand = im2col then
// W; accumulator = T then Z) and alternate tiles, so one group's epilogue
// overlaps the other group's GEMMs; warp 9 streams u by 2-D TMA into one
// shared-memory ring per group (plus L2 tensor prefetches ahead).
// Work item = (image, band of RB tile rows); deterministic: every sum has a
// fixed order (per-warp col2im strips, strips and bands summed in index order).
#pragma once
#include <cuda.h>

#include <type_traits>

#include "kernels.cuh"
#include "umma.cuh"

namespace dcsc_cuda {

#ifdef DCSC_TC_TRACE  // per-phase globaltimer trace of one epilogue warp (CTA 0, group 0, warp 1), a few tiles
#define TCT(slot)                                                                              \
  if (blockIdx.x == 0 && (threadIdx.x & 31) == 0 && e == 0 && t >= 2 && t < 8) {              \
    unsigned long long tt_;                                                                    \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt_));                                   \
    tr[(t - 2) / 2][slot] = tt_;                                                               \
  }
#else
#define TCT(slot)
#endif

constexpr int kTcTaps = 128;                       // GEMM-1 K / GEMM-2 N (taps padded)
// epilogue warps per CTA (TcGeom::EW): 8 = one warp per (group, TMEM lane quarter); 16 = two, which
// split the filters (prox) and the taps (im2col, col2im) of the quarter's 32 pixels. DCSC_TC_EW forces one.
constexpr int kTcStripW = 44;                      // col2im strip row stride (floats) >= 32 + MW - 1
constexpr int kTcUSlots = 6;                       // u staging ring depth per epilogue group
#ifndef DCSC_TC_UPREFETCH  // experiment overrides (build.build(defines=[...]))
#define DCSC_TC_UPREFETCH 8
#endif
#ifndef DCSC_TC_MMA_SLEEP
#define DCSC_TC_MMA_SLEEP 40
#endif
constexpr int kTcUPrefetch = DCSC_TC_UPREFETCH;    // chunks ahead an L2 prefetch of u rows is issued

struct TcArgs {
  CUtensorMap umap;        // u as [N*K planes][D pixels] FP32, box [16 planes][128 pixels]
  int plane0;              // umap plane of (image 0 of this launch, filter 0)
  const uint32_t* lam16;   // N x 2 x H x W/2 words: f16 pairs of lambda * lam_scale[n] (hi plane, lo plane)
  const float* lam_scale;  // N
  const __half* dsplit;    // 2 x KF x 128 f16 core-matrix grid of d * d_scale (hi, lo)
  float d_scale;
  float* u;                // N x K x H x W ADMM state u = t - z/rho
  const float* theta0;     // N x K x H x W (first iteration's theta_old) or nullptr
  float* spart;            // N x NBANDS x SR x W col2im band partials
  double* bsums;           // N x NBANDS x kSums stop-test partial sums
  const int* conv;         // N
  float* zmax;             // N x NBANDS x TPI x 4 x HV: per warp and tile, max_k |z/rho| of the stored u (written each pass)
  float tbound;            // |t| <= tbound / lam_scale[n] (2 * 2^14 * max_k ||d_k||_1)
  int N, K;
  float rho, beta;
};

template <int H_, int W_, int KF_, int MH_, int MW_, int RB_, int EW_>
struct TcGeom {
  static constexpr int H = H_, W = W_, KF = KF_, MH = MH_, MW = MW_, RB = RB_;
  static constexpr int EW = EW_;                   // epilogue warps: 8 or 16
  static constexpr int HV = EW / 8;                // warps per (group, lane quarter)
  static constexpr int THREADS = 32 * (EW + 2);    // MMA warp, epilogue warps, u streaming warp
  // w's f16 split with packed FMUL2 / FADD2 (bit-identical to the scalar form): measured +1.0% at C3 and
  // +1.7% at C1, -0.7% at C2 (100^2) and -1.1% at C4 (64^2) -> the 256^2 and 128^2 families only
#ifdef DCSC_TC_SCALAR_SPLIT
  static constexpr bool PSPLIT = false;
#else
  static constexpr bool PSPLIT = W_ >= 128;
#endif
  static_assert(EW == 8 || EW == 16, "epilogue warps");
  static constexpr int D = H * W;
  // a 128-lane tile is RPT image rows x WT pixels: row segments of 128 (W a multiple of 128),
  // row pairs (W = 64), or one row with 128 - W idle lanes (64 < W < 128)
  static constexpr int WT = W < 128 ? W : 128;
  static constexpr int RPT = W <= 64 ? 128 / W : 1;
  static constexpr int VALID = WT * RPT;           // live lanes of a tile
  static constexpr int TPR = W / WT;               // tiles per row (tile rows of RPT image rows)
  static constexpr int NBANDS = H / RB;
  static constexpr int TPI = (RB / RPT) * TPR;     // tiles per work item
  static constexpr int SR = RB + MH - 1;           // rows a band's col2im touches / lambda rows it reads
  static constexpr int LWW = W / 2 + 8;            // lambda band row: W halves + 16 wrap halves, in words
  static constexpr int NSS = TPR == 1 ? 2 : TPR;   // strip sets (per tile column; per epilogue group if TPR == 1)
  static constexpr int NSTRIP = NSS * 4;
  static constexpr int STRIP = SR * kTcStripW;
  static constexpr int TAPS = MH * MW;
  static constexpr int TP = TAPS <= 64 ? 64 : 128;  // taps padded: GEMM-1 K, GEMM-2 N
  static_assert((W % 128 == 0 && (TPR == 1 || TPR % 2 == 0)) || W == 64 || (W > 64 && W < 128 && W % 4 == 0),
                "128-lane tiles: row segments, row pairs, or single rows");
  static_assert(H % RB == 0 && RB % RPT == 0 && RB >= MH - 1 && TPI % 2 == 0, "band geometry");
  static_assert(TAPS <= kTcTaps && 32 + MW - 1 <= kTcStripW && MW <= 16 && MW < W, "filter support");
  static_assert(KF % 16 == 0 && KF >= 32 && KF <= 128, "filters per pass");
  static constexpr size_t d_bytes = (size_t)2 * KF * TP * 2;
  static constexpr size_t lam_off = d_bytes;
  static constexpr size_t lam_bytes = (size_t)2 * SR * LWW * 4;
  static constexpr size_t strip_off = (lam_off + lam_bytes + 15) / 16 * 16;
  static constexpr size_t strip_bytes = (size_t)NSTRIP * STRIP * 4;
  static constexpr size_t red_off = strip_off + strip_bytes;
  static constexpr size_t red_bytes = (size_t)8 * EW * 8;
  // u staging: per epilogue group a ring of kTcUSlots chunks of 16 filter rows x 128 pixels (TMA bulk copies)
  static constexpr size_t ubuf_off = (red_off + red_bytes + 127) / 128 * 128;
  static constexpr size_t ubuf_bytes = (size_t)2 * kTcUSlots * 16 * 128 * 4;
  static constexpr size_t bar_off = ubuf_off + ubuf_bytes;
  static constexpr size_t smem = bar_off + (size_t)(10 + 4 * kTcUSlots) * 8;  // barriers + TMEM slot
};

// Packed FP32 pairs (FADD2 / FMUL2 / FFMA2): half the issue slots of scalar FP32.
struct F2 {
  unsigned long long u;
};
__device__ __forceinline__ F2 f2(float x, float y) {
  F2 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r.u) : "f"(x), "f"(y));
  return r;
}
__device__ __forceinline__ float f2x(F2 a) {
  float x, y;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(x), "=f"(y) : "l"(a.u));
  return x;
}
__device__ __forceinline__ float f2y(F2 a) {
  float x, y;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(x), "=f"(y) : "l"(a.u));
  return y;
}
__device__ __forceinline__ F2 add2(F2 a, F2 b) {
  F2 r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r.u) : "l"(a.u), "l"(b.u));
  return r;
}
__device__ __forceinline__ F2 sub2(F2 a, F2 b) {
  F2 r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r.u) : "l"(a.u), "l"(b.u));
  return r;
}
__device__ __forceinline__ F2 mul2(F2 a, F2 b) {
  F2 r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r.u) : "l"(a.u), "l"(b.u));
  return r;
}
__device__ __forceinline__ F2 fma2(F2 a, F2 b, F2 c) {
  F2 r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r.u) : "l"(a.u), "l"(b.u), "l"(c.u));
  return r;
}

__device__ __forceinline__ void mbar_arrive1(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_test(unsigned long long* bar, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{\n.reg .pred p;\nmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_addr(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// Wait for a GEMM's commit (1-2 us): a plain try_wait loop re-issues every ~36 cycles (ncu: 12% of the
// pass's executed warp instructions were these two spin loops). DCSC_TC_WAIT: 0 plain loop, 1 try_wait with a
// suspend-time hint, 2 nanosleep back-off between tries.
#ifndef DCSC_TC_WAIT
#define DCSC_TC_WAIT 0
#endif
#ifndef DCSC_TC_WAIT_NS
#define DCSC_TC_WAIT_NS 200
#endif
__device__ __forceinline__ void mbar_wait_gemm(unsigned long long* bar, unsigned parity) {
#if DCSC_TC_WAIT == 1
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAITG_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      "@!p bra WAITG_%=;\n"
      "}\n" ::"r"(smem_addr(bar)),
      "r"(parity), "r"((unsigned)DCSC_TC_WAIT_NS)
      : "memory");
#elif DCSC_TC_WAIT == 2
  while (!mbar_test(bar, parity)) __nanosleep(DCSC_TC_WAIT_NS);
#else
  mbar_wait(bar, parity);
#endif
}
template <int THREADS>
__device__ __forceinline__ void epi_sync() {
  asm volatile("bar.sync 1, %0;" ::"n"(THREADS) : "memory");
}
__device__ __forceinline__ uint32_t lds_u16(const void* p) {
  unsigned short v;
  asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(smem_addr(p)));
  return v;
}

// im2col row of one pixel (tap o = oy*MW + ox, lambda[r + oy][c + ox]) as f16
// pairs (o = 2j, 2j+1) -> tensor-memory columns j (hi) and 64 + j (lo).
// `row` = this tile row's first band row (hi plane; the lo plane follows at
// +SR*LWW words), cb = c >> 1, par = c & 1. Pairs inside one tap row are two
// word loads + a byte permute; pairs across tap rows two half loads.
template <class G>
__device__ __forceinline__ void tc_build_im2col(const uint32_t* row, int c, uint32_t A, int h) {
  constexpr int MW = G::MW, TAPS = G::TAPS, LWW = G::LWW, SR = G::SR, TP = G::TP;
  const int cb = c >> 1, par = c & 1;
  const uint32_t sel_e = par ? 0x5432u : 0x3210u;  // pair starting at an even tap column offset
  const uint32_t sel_o = par ? 0x3210u : 0x5432u;
#pragma unroll
  for (int ch = 0; ch < TP / 32; ++ch) {
    if (G::HV > 1 && (ch % G::HV) != h) continue;  // 32-tap chunks alternate between the quarter's warps
    uint32_t vv[2][16];
#pragma unroll
    for (int pl = 0; pl < 2; ++pl) {
      const uint32_t* rp = row + pl * SR * LWW;
#pragma unroll
      for (int jj = 0; jj < 16; ++jj) {
        const int o0 = 2 * (ch * 16 + jj), o1 = o0 + 1;
        uint32_t val = 0;
        if (o0 < TAPS) {
          const int oy0 = o0 / MW, ox0 = o0 % MW;
          if (o1 < TAPS && o1 / MW == oy0) {
            const uint32_t* p = rp + oy0 * LWW + cb;
            if ((ox0 & 1) == 0) {
              val = __byte_perm(p[ox0 / 2], p[ox0 / 2 + 1], sel_e);
            } else {
              val = __byte_perm(p[par + (ox0 - 1) / 2], p[par + (ox0 - 1) / 2 + 1], sel_o);
            }
          } else {
            const unsigned short* hr = reinterpret_cast<const unsigned short*>(rp);
            const uint32_t lo = lds_u16(hr + oy0 * 2 * LWW + c + ox0);
            uint32_t hi = 0;
            if (o1 < TAPS) hi = lds_u16(hr + (o1 / MW) * 2 * LWW + c + (o1 % MW));
            val = lo | (hi << 16);
          }
        }
        vv[pl][jj] = val;
      }
    }
    umma::st16(A + ch * 16, vv[0]);
    umma::st16(A + 64 + ch * 16, vv[1]);
  }
}

// tensor-memory columns [C0, C0 + N) of this warp's lanes -> v[0 .. N) (largest power-of-two pieces first)
template <int N>
__device__ __forceinline__ void tc_ld_cols(uint32_t taddr, uint32_t* v) {
  if constexpr (N >= 32) {
    umma::ld32(taddr, *reinterpret_cast<uint32_t(*)[32]>(v));
    tc_ld_cols<N - 32>(taddr + 32, v + 32);
  } else if constexpr (N >= 16) {
    umma::ld16(taddr, *reinterpret_cast<uint32_t(*)[16]>(v));
    tc_ld_cols<N - 16>(taddr + 16, v + 16);
  } else if constexpr (N >= 8) {
    umma::ld8(taddr, *reinterpret_cast<uint32_t(*)[8]>(v));
    tc_ld_cols<N - 8>(taddr + 8, v + 8);
  } else if constexpr (N >= 4) {
    umma::ld4(taddr, *reinterpret_cast<uint32_t(*)[4]>(v));
    tc_ld_cols<N - 4>(taddr + 4, v + 4);
  } else if constexpr (N >= 2) {
    umma::ld2(taddr, *reinterpret_cast<uint32_t(*)[2]>(v));
    tc_ld_cols<N - 2>(taddr + 2, v + 2);
  } else if constexpr (N == 1) {
    umma::ld1(taddr, v[0]);
  }
}

// col2im of tap rows [OY0, OY1): s[r + oy][c + ox] += Z[p][oy * MW + ox] * zsc into this warp's
// strip rows. Taps (oy, ox) of one ox touch distinct strip rows: OY1 - OY0 independent
// read-modify-writes between warp syncs (lanes overlap only along ox).
template <class G, int OY0, int OY1>
__device__ __forceinline__ void tc_col2im(uint32_t ACC, float* S, float zsc, bool live) {
  constexpr int MW = G::MW, C0 = OY0 * MW, NV = (OY1 - OY0) * MW;
  uint32_t v[NV];
  tc_ld_cols<NV>(ACC + C0, v);
  umma::wait_ld();
#pragma unroll
  for (int ox = 0; ox < MW; ++ox) {
#pragma unroll
    for (int oy = OY0; oy < OY1; ++oy) {
      float* sp = S + oy * kTcStripW + ox;
      if (live) *sp = fmaf(__uint_as_float(v[(oy - OY0) * MW + ox]), zsc, *sp);
    }
    __syncwarp();
  }
}

// FULL: K == KF (no padded filters); T0: a.theta0 is set (first iteration of a
// warm state that is not ADMM-consistent).
template <class G, bool FULL, bool T0>
__global__ void __launch_bounds__(G::THREADS, 1) coding_pass_tc(const __grid_constant__ TcArgs a) {
  constexpr int H = G::H, W = G::W, KF = G::KF, MW = G::MW, RB = G::RB, D = G::D, TPR = G::TPR, TP = G::TP,
                WT = G::WT, RPT = G::RPT,
                NBANDS = G::NBANDS, TPI = G::TPI, SR = G::SR, LWW = G::LWW, TAPS = G::TAPS;
  extern __shared__ __align__(1024) unsigned char sm[];
  const __half* Ds = reinterpret_cast<const __half*>(sm);
  uint32_t* LAM = reinterpret_cast<uint32_t*>(sm + G::lam_off);
  float* STR = reinterpret_cast<float*>(sm + G::strip_off);
  double* RED = reinterpret_cast<double*>(sm + G::red_off);
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(sm + G::bar_off);
  unsigned long long *a_full = bars, *t_full = bars + 2, *w_full = bars + 4, *z_full = bars + 6, *dbar = bars + 8;
  unsigned long long *ufull = bars + 9, *uempty = bars + 9 + 2 * kTcUSlots;  // [group][slot]
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 9 + 4 * kTcUSlots);
  float* UB = reinterpret_cast<float*>(sm + G::ubuf_off);
  // warp index through a shuffle: provably warp-uniform, so role branches keep
  // the MMA operands in uniform registers (no per-instruction lane loops)
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;

  if (warp == 0) umma::tmem_alloc<512>(tslot);
  if (threadIdx.x == 32) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(a_full + i, 4 * G::HV);
      mbar_init(w_full + i, 4 * G::HV);
      mbar_init(t_full + i, 1);
      mbar_init(z_full + i, 1);
    }
    mbar_init(dbar, 1);
    for (int i = 0; i < 2 * kTcUSlots; ++i) {
      mbar_init(ufull + i, 1);
      mbar_init(uempty + i, 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  umma::fence_before_sync();
  __syncthreads();
  umma::fence_after_sync();
  const uint32_t tbase = *tslot;
  if (tbase != 0u) __trap();  // 512 columns allocated by the only CTA on the SM start at column 0
  const int items = a.N * NBANDS;

  constexpr int NCU = KF / 16, NCHUNK = (TPI / 2) * NCU;  // u chunks per item and group
  if (warp == 0 || warp == G::EW + 1) {
    // ===== producer warps: GEMM issue (warp 0, lane 0); u row streaming by TMA (last warp) =====
    if (warp == 0 && lane == 0) {
      mbar_expect_tx(dbar, (unsigned)G::d_bytes);
      static_assert(G::d_bytes % 8192 == 0, "dictionary split in 8 KB bulk copies");
      for (int i = 0; i < (int)(G::d_bytes / 8192); ++i)
        bulk_g2s(const_cast<__half*>(Ds) + i * 4096, a.dsplit + i * 4096, 8192u, dbar);
      mbar_wait(dbar, 0);
    }
    __syncwarp();
    const uint32_t dh = umma::smem_u32(Ds), dl = dh + KF * TP * 2;
    constexpr uint32_t id1 = umma::idesc_f16(128, KF, 0), id2 = umma::idesc_f16(128, TP, 1);
    constexpr uint32_t FGS = (uint32_t)TP * 16u;  // bytes per filter group (8 filters x TP taps) in the D grid
    // the CTA owns all 512 TMEM columns, so the allocation starts at address 0
    // (checked below); slot addresses are then warp-uniform immediates
    // slot as a compile-time constant: TMEM addresses become immediates
    auto gemm1s = [&](auto S) {
      constexpr uint32_t A = 256u * decltype(S)::value, acc = A + 128u;
      umma::fence_after_sync();
#pragma unroll
      for (int j = 0; j < TP / 16; ++j) {  // K = taps; B K-major: LBO 128 B (taps), SBO FGS (filters)
        const uint64_t bh = umma::sdesc(dh + 256u * j, 128u, FGS), bl = umma::sdesc(dl + 256u * j, 128u, FGS);
        umma::mma_ts_warp(acc, A + 8u * j, bh, id1, j > 0);
        umma::mma_ts_warp(acc, A + 8u * j, bl, id1, 1u);
        umma::mma_ts_warp(acc, A + 64u + 8u * j, bh, id1, 1u);
      }
      umma::commit_warp(t_full + decltype(S)::value);
    };
    auto gemm2s = [&](auto S) {
      constexpr uint32_t A = 256u * decltype(S)::value, acc = A + 128u;
      umma::fence_after_sync();
#pragma unroll
      for (int j = 0; j < KF / 16; ++j) {  // K = filters; B MN-major: LBO FGS (filters), SBO 128 B (taps)
        const uint64_t bh = umma::sdesc(dh + 2u * FGS * j, FGS, 128u), bl = umma::sdesc(dl + 2u * FGS * j, FGS, 128u);
        umma::mma_ts_warp(acc, A + 8u * j, bh, id2, j > 0);
        umma::mma_ts_warp(acc, A + 8u * j, bl, id2, 1u);
        umma::mma_ts_warp(acc, A + 64u + 8u * j, bh, id2, 1u);
      }
      umma::commit_warp(z_full + decltype(S)::value);
    };
    auto gemm1 = [&](uint32_t gg) {
      if (gg & 1u) gemm1s(std::integral_constant<uint32_t, 1>{}); else gemm1s(std::integral_constant<uint32_t, 0>{});
    };
    auto gemm2 = [&](uint32_t gg) {
      if (gg & 1u) gemm2s(std::integral_constant<uint32_t, 1>{}); else gemm2s(std::integral_constant<uint32_t, 0>{});
    };
    int ntiles = 0;
    for (int item = blockIdx.x; item < items; item += gridDim.x)
      if (!a.conv[item / NBANDS]) ntiles += TPI;
    // per group: next chunk (item, index within the item) and its ring sequence number
    int c_item[2], c_i[2];
    uint32_t c_seq[2] = {0u, 0u};
    auto next_active = [&](int item) {
      while (item < items && a.conv[item / NBANDS]) item += gridDim.x;
      return item;
    };
    c_item[0] = c_item[1] = next_active(blockIdx.x);
    c_i[0] = c_i[1] = 0;
    uint32_t n1 = 0, n2 = 0;
    auto lane0_test = [&](unsigned long long* bar, unsigned par) {
      int r = 0;
      if (lane == 0) r = mbar_test(bar, par) ? 1 : 0;
      return __shfl_sync(0xffffffffu, r, 0) != 0;
    };
    if (warp == 0) {
      // GEMMs: whichever is ready first (GEMM-1 of the next tile, GEMM-2 of the oldest pending)
      // whole warp, converged: decisions from lane 0's barrier tests, MMAs by an elected lane
      while ((int)n2 < ntiles) {
        if ((int)n1 < ntiles && lane0_test(a_full + (n1 & 1u), (n1 >> 1) & 1u)) {
          gemm1(n1++);
        } else if (n2 < n1 && lane0_test(w_full + (n2 & 1u), (n2 >> 1) & 1u)) {
          gemm2(n2++);
        } else {
          __nanosleep(DCSC_TC_MMA_SLEEP);  // keep the polling off the epilogue warps' issue slots
        }
      }
    } else
    while (c_item[0] < items || c_item[1] < items) {
      const uint32_t seq0 = c_seq[0] + c_seq[1];
      // u rows: chunk i of an item = tile e + 2 (i / NCU), filter rows 16 (i % NCU) .. + 16
      for (int e = 0; e < 2; ++e) {
        while (c_item[e] < items) {  // every free ring slot
        const uint32_t ci = c_seq[e], sl = ci % kTcUSlots;
        if (ci >= (uint32_t)kTcUSlots && !lane0_test(uempty + e * kTcUSlots + sl, ((ci / kTcUSlots) - 1) & 1u))
          break;
        const int n = c_item[e] / NBANDS, b = c_item[e] % NBANDS, i = c_i[e];
        const int t = e + 2 * (i / NCU), k0 = 16 * (i % NCU);
        const int r = b * RB + (t / TPR) * RPT, c0 = (t % TPR) * 128;  // the tile's first pixel
        const int nv = FULL ? 16 : max(0, min(16, a.K - k0));
        unsigned long long* fb = ufull + e * kTcUSlots + sl;
        (void)nv;
        if (lane == 0 && i + kTcUPrefetch < NCHUNK) {  // the same group's chunk kTcUPrefetch ahead -> L2
          const int ip = i + kTcUPrefetch;
          const int tp = e + 2 * (ip / NCU), kp = 16 * (ip % NCU);
          asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global [%0, {%1, %2}];" ::"l"(&a.umap),
                       "r"((b * RB + (tp / TPR) * RPT) * W + (tp % TPR) * 128), "r"(a.plane0 + n * a.K + kp)
                       : "memory");
        }
        if (lane == 0) {  // one 2-D TMA: 16 planes x 128 pixels (rows past the last plane are zero-filled)
          mbar_expect_tx(fb, 16u * 128u * 4u);
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                  smem_addr(UB + (size_t)(e * kTcUSlots + sl) * 16 * 128)),
              "l"(&a.umap), "r"(r * W + c0), "r"(a.plane0 + n * a.K + k0), "r"(smem_addr(fb))
              : "memory");
        }
        __syncwarp();
        ++c_seq[e];
        if (++c_i[e] == NCHUNK) {
          c_i[e] = 0;
          c_item[e] = next_active(c_item[e] + gridDim.x);
        }
        }
      }
      if (c_seq[0] + c_seq[1] == seq0) __nanosleep(32);
    }
  } else {
    // ===== epilogue groups =====
    // warp -> (group e, half h, lane quarter q = warp % 4: the TMEM lanes a warp may access)
    const int ew = warp - 1, e = (ew >> 2) & 1, h = ew >> 3, q = warp & 3, p = 32 * q + lane, et = threadIdx.x - 32;
    const uint32_t lane_off = (uint32_t)(32 * q) << 16;
    const uint32_t A = tbase + 256u * e + lane_off, ACC = A + 128u;
    const float rho = a.rho, beta = a.beta;
    uint32_t g = 0, uc = 0;  // tiles / u chunks (per group) of this CTA's earlier items
    for (int item = blockIdx.x; item < items; item += gridDim.x) {
      const int n = item / NBANDS, b = item % NBANDS;
      if (a.conv[n]) continue;
      epi_sync<32 * G::EW>();  // previous item's strips flushed
      {            // lambda band rows b*RB .. b*RB + SR - 1 (mod H), wrap-padded by 16 halves
        const uint32_t* src = a.lam16 + (size_t)n * 2 * (D / 2);
        for (int i = et; i < 2 * SR * LWW; i += 32 * G::EW) {
          const int pl = i / (SR * LWW), rr = (i / LWW) % SR, wi = i % LWW;
          const int gr = (b * RB + rr) % H, sc = wi < W / 2 ? wi : wi - W / 2;
          LAM[i] = __ldg(src + ((size_t)pl * H + gr) * (W / 2) + sc);
        }
        float4* z4 = reinterpret_cast<float4*>(STR);
        for (int i = et; i < G::NSTRIP * G::STRIP / 4; i += 32 * G::EW) z4[i] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
      epi_sync<32 * G::EW>();
      if (et == 0 && item + (int)gridDim.x < items) {  // next item's lambda band -> L2 (both f16 planes)
        const int n2 = (item + gridDim.x) / NBANDS, b2 = (item + gridDim.x) % NBANDS;
        const int rows = min(SR, H - b2 * RB);  // the wrapped rows (from row 0) are the next bands' anyway
        for (int pl = 0; pl < 2; ++pl)
          prefetch_l2_bulk(a.lam16 + ((size_t)(n2 * 2 + pl) * H + b2 * RB) * (W / 2), (unsigned)(rows * W * 2));
      }
      const float lsc = __ldg(a.lam_scale + n);
      const float tsc = 1.f / (lsc * a.d_scale);
      const float tb = a.tbound / lsc;
      const float dinv = 1.f / a.d_scale;
      double st[7] = {0, 0, 0, 0, 0, 0, 0};
      float* const ubase = a.u + (size_t)n * a.K * D;
      const float* const t0base = a.theta0 ? a.theta0 + (size_t)n * a.K * D : nullptr;
      // u rows arrive in this group's ring by TMA (producer warp); every warp
      // releases a slot once it holds the chunk in registers
      float* const ring = UB + (size_t)e * kTcUSlots * 16 * 128;
      unsigned long long* const uf = ufull + e * kTcUSlots;
      unsigned long long* const ue = uempty + e * kTcUSlots;
      // chunk cix (item-relative, group order: tile-major, filter chunks inside); chunks
      // alternate between the quarter's warps, each released by the four warps that read it
      auto take_chunk = [&](float (&uo)[16], int cix) {
        const uint32_t ci = uc + (uint32_t)cix, sl = ci % kTcUSlots;
        mbar_wait(uf + sl, (ci / kTcUSlots) & 1u);
        const float* src = ring + (size_t)sl * 16 * 128 + p;
#pragma unroll
        for (int j = 0; j < 16; ++j) uo[j] = src[j * 128];
        __syncwarp();
        if (lane == 0) mbar_arrive1(ue + sl);
      };
#ifdef DCSC_TC_TRACE
      unsigned long long tr[3][8] = {};
#endif
      for (int t = e; t < TPI; t += 2) {
        TCT(0)
        const uint32_t gg = g + t, ph = (gg >> 1) & 1u;
        const int tc = t % TPR;
        const bool live = p < G::VALID;           // lanes past a short row (64 < W < 128) carry zeros
        const int pc = live ? p : p - G::VALID;   // in-row stand-in for a dead lane's addresses
        const int rl = (t / TPR) * RPT + pc / WT;  // this pixel's band-local row
        const int r = b * RB + rl, c = tc * 128 + pc % WT;
        float* const up = ubase + (size_t)r * W + c;
        const float* const t0p = t0base ? t0base + (size_t)r * W + c : nullptr;
        // --- im2col(lambda) -> A
        tc_build_im2col<G>(LAM + rl * LWW, c, A, h);
        umma::wait_st();
        umma::fence_before_sync();
        __syncwarp();
        if (lane == 0) mbar_arrive1(a_full + e);
        TCT(1)
        // --- prox on T, w -> A (two f16 planes, per-pixel scale)
        // stop-test sums (coding.cpp:237-259): sum dz^2 = rho^2 sum (theta' - t)^2 and
        // sum z'^2 = rho^2 sum (theta' - u')^2 are scaled once per tile
        // per-pair accumulators (packed FP32), folded once per tile
        F2 a0 = f2(0.f, 0.f), a1 = a0, a2 = a0, a4 = a0, a5 = a0;
        float f6 = 0.f, wmax = 0.f, zm = 0.f;
        // W's per-pixel f16 scale from a bound known before the prox (not T0):
        // |w| = |2 theta' - u'| <= beta + |u'| <= beta + |t| + |z_old / rho|, with
        // |t| <= ||d_k||_1 max|lambda| (tb) and max_k |z_old / rho| of this warp's
        // pixels recorded by the previous pass (zmax) -> w is split as it is formed
        float* const zslot = a.zmax + ((((size_t)n * NBANDS + b) * TPI + t) * 4 + q) * G::HV;
        const float zprev = G::HV > 1 ? fmaxf(zslot[0], zslot[G::HV - 1]) : zslot[0];
        const float sw_pred = T0 ? 1.f : umma::pow2_scale(beta + tb + zprev);
        const float tsl = live ? tsc : 0.f;  // dead lanes: t = u = 0, so w = 0 and no stop-test share
        const F2 tsc2 = f2(tsl, tsl);
        mbar_wait_gemm(t_full + e, ph);
        umma::fence_after_sync();
        TCT(2)
#pragma unroll 1
        // filter chunks alternate between the quarter's warps; the theta0 variant needs max|w| over
        // all filters of a pixel, so there the first warp of the quarter takes every chunk
        for (int ch = T0 ? (h == 0 ? 0 : KF / 16) : h; ch < KF / 16; ch += T0 ? 1 : G::HV) {
          float ucur[16], tcur[16];
          take_chunk(ucur, ((t - e) >> 1) * NCU + ch);
          if constexpr (T0) {
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              const int k = ch * 16 + j;
              tcur[j] = ((FULL || k < a.K) && live) ? __ldg(t0p + (size_t)k * D) : 0.f;
            }
          }
          uint32_t v[16], vh[8], vl[8];
          umma::ld16(ACC + ch * 16, v);
          umma::wait_ld();
#pragma unroll
          for (int jj = 0; jj < 8; ++jj) {
            const int k0 = ch * 16 + 2 * jj;
            const float u0 = ((FULL || k0 < a.K) && live) ? ucur[2 * jj] : 0.f;
            const float u1 = ((FULL || k0 + 1 < a.K) && live) ? ucur[2 * jj + 1] : 0.f;
            const F2 t = mul2(f2(__uint_as_float(v[2 * jj]), __uint_as_float(v[2 * jj + 1])), tsc2);
            float o0, o1;
            if constexpr (T0) {
              o0 = tcur[2 * jj];
              o1 = tcur[2 * jj + 1];
            } else {
              o0 = fminf(fmaxf(u0, -beta), beta);
              o1 = fminf(fmaxf(u1, -beta), beta);
            }
            const F2 tho = f2(o0, o1);
            const F2 un = sub2(t, sub2(tho, f2(u0, u1)));  // u' = t - (theta_old - u)
            const float un0 = f2x(un), un1 = f2y(un);
            const F2 th = f2(fminf(fmaxf(un0, -beta), beta), fminf(fmaxf(un1, -beta), beta));
            const F2 d_tt = sub2(th, t), d_z = sub2(th, un), dth = sub2(th, tho);
            a0 = fma2(d_tt, d_tt, a0);
            a1 = fma2(th, th, a1);
            a2 = fma2(t, t, a2);
            a4 = fma2(d_z, d_z, a4);
            a5 = fma2(dth, dth, a5);
            f6 = fmaxf(f6, fmaxf(fabsf(f2x(t)), fabsf(f2y(t))));
            zm = fmaxf(zm, fmaxf(fabsf(f2x(d_z)), fabsf(f2y(d_z))));
            const F2 w = add2(th, d_z);  // w = theta' + z'/rho = 2 theta' - u'
            const float w0 = f2x(w), w1 = f2y(w);
            if constexpr (T0) {
              wmax = fmaxf(wmax, fmaxf(fabsf(w0), fabsf(w1)));
            } else {
              if constexpr (G::PSPLIT) {  // split2x2's roundings with the scale and the remainder as packed FP32
                const F2 ws = mul2(w, f2(sw_pred, sw_pred));
                const __half2 hh = __float22half2_rn(make_float2(f2x(ws), f2y(ws)));
                const float2 hb = __half22float2(hh);
                const F2 rem = sub2(ws, f2(hb.x, hb.y));
                const __half2 ll = __float22half2_rn(make_float2(f2x(rem), f2y(rem)));
                vh[jj] = *reinterpret_cast<const uint32_t*>(&hh);
                vl[jj] = *reinterpret_cast<const uint32_t*>(&ll);
              } else {
                umma::split2x2(w0, w1, sw_pred, vh[jj], vl[jj]);
              }
            }
            if ((FULL || k0 < a.K) && live) __stcs(up + (size_t)k0 * D, un0);
            if ((FULL || k0 + 1 < a.K) && live) __stcs(up + (size_t)(k0 + 1) * D, un1);
            v[2 * jj] = __float_as_uint(w0);
            v[2 * jj + 1] = __float_as_uint(w1);
          }
          if constexpr (T0) {
            umma::st16(ACC + ch * 16, v);
          } else {  // filter pairs 8 ch .. 8 ch + 7 -> W columns (hi, lo)
            umma::st8(A + ch * 8, vh);
            umma::st8(A + 64 + ch * 8, vl);
          }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) zm = fmaxf(zm, __shfl_xor_sync(0xffffffffu, zm, o));
        const float f0 = f2x(a0) + f2y(a0), f1 = f2x(a1) + f2y(a1), f2_ = f2x(a2) + f2y(a2),
                    f4 = f2x(a4) + f2y(a4), f5 = f2x(a5) + f2y(a5);
        TCT(3)
        umma::wait_st();
        const float sw = T0 ? umma::pow2_scale(wmax) : sw_pred;
#pragma unroll 1
        for (int ch = 0; ch < (T0 && h == 0 ? KF / 32 : 0); ++ch) {
          uint32_t v[32];
          umma::ld32(ACC + ch * 32, v);
          umma::wait_ld();
          uint32_t vh[16], vl[16];
#pragma unroll
          for (int jj = 0; jj < 16; ++jj)
            umma::split2x2(__uint_as_float(v[2 * jj]), __uint_as_float(v[2 * jj + 1]), sw, vh[jj], vl[jj]);
          umma::st16(A + ch * 16, vh);
          umma::st16(A + 64 + ch * 16, vl);
        }
        if (T0 && KF % 32 != 0 && h == 0) {  // a last chunk of 16 filter slots (KF = 112)
          uint32_t v[16];
          umma::ld16(ACC + (KF / 32) * 32, v);
          umma::wait_ld();
          uint32_t vh[8], vl[8];
#pragma unroll
          for (int jj = 0; jj < 8; ++jj)
            umma::split2x2(__uint_as_float(v[2 * jj]), __uint_as_float(v[2 * jj + 1]), sw, vh[jj], vl[jj]);
          umma::st8(A + (KF / 32) * 16, vh);
          umma::st8(A + 64 + (KF / 32) * 16, vl);
        }
        umma::wait_st();
        umma::fence_before_sync();
        __syncwarp();
        if (lane == 0) mbar_arrive1(w_full + e);
        TCT(4)
        const float rho2 = rho * rho;
        st[0] += (double)f0; st[1] += (double)f1; st[2] += (double)f2_; st[3] += (double)(rho2 * f0);
        st[4] += (double)(rho2 * f4); st[5] += (double)f5; st[6] = fmax(st[6], (double)f6);
        // --- col2im: s[r + oy][c + ox] += Z[p][o] into this warp's strip
        const float zsc = dinv / sw;
        float* const S = STR + ((TPR == 1 ? e : tc) * 4 + q) * G::STRIP + rl * kTcStripW + lane;  // warp-uniform row
        mbar_wait_gemm(z_full + e, ph);
        umma::fence_after_sync();
        if (lane == 0) zslot[h] = zm;  // both of the quarter's warps have read the previous record by now
        TCT(5)
        // the quarter's warps split the tap rows (disjoint strip rows): oy in [0, MH0) and [MH0, MH)
        // (theta0 variant: W's scale is known to the quarter's first warp only, which takes both parts)
        if constexpr (G::HV == 1) {
          tc_col2im<G, 0, G::MH>(ACC, S, zsc, live);
        } else {
          if (h == 0) tc_col2im<G, 0, (G::MH + 1) / 2>(ACC, S, zsc, live);
          if (T0 ? h == 0 : h == 1) tc_col2im<G, (G::MH + 1) / 2, G::MH>(ACC, S, zsc, live);
        }
        TCT(6)
      }
#ifdef DCSC_TC_TRACE
      if (blockIdx.x == 0 && (threadIdx.x & 31) == 0 && e == 0 && item == (int)blockIdx.x)
        for (int f = 0; f < 3; ++f)
          printf("TCT warp %d tile %d: start %llu build %llu waitG1 %llu epi1 %llu split %llu waitG2 %llu col2im %llu\n",
                 warp, 2 + 2 * f, tr[f][0] % 1000000, tr[f][1] - tr[f][0], tr[f][2] - tr[f][1], tr[f][3] - tr[f][2],
                 tr[f][4] - tr[f][3], tr[f][5] - tr[f][4], tr[f][6] - tr[f][5]);
#endif
      g += TPI;
      uc += NCHUNK;
      // --- stop-test partial sums of the item (fixed order)
#pragma unroll
      for (int i = 0; i < 7; ++i) {
        double x = st[i];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const double y = __shfl_xor_sync(0xffffffffu, x, o);
          x = i == 6 ? fmax(x, y) : x + y;
        }
        if (lane == 0) RED[ew * 8 + i] = x;
      }
      epi_sync<32 * G::EW>();
      if (et == 0) {
        double* o = a.bsums + ((size_t)n * NBANDS + b) * kSums;
        for (int i = 0; i < 7; ++i) {
          double x = 0.0;
          for (int w2 = 0; w2 < G::EW; ++w2) x = i == 6 ? fmax(x, RED[w2 * 8 + i]) : x + RED[w2 * 8 + i];
          o[i] = x;
        }
        o[7] = 0.0;
      }
      // --- strips -> band partial (strips summed in index order)
      float* dst = a.spart + ((size_t)n * NBANDS + b) * SR * W;
#ifndef DCSC_TC_STRIP_GENERIC  // build override: the general loop everywhere (bit-identity check)
      if constexpr (TPR >= 2) {
        // row segments of 128: strip j = s2 * 4 + q2 starts at column 32 j, so a column reads its own strip
        // and, in its first MW - 1 columns, the spill-over of the previous one (cyclic). Two terms: the sum
        // (0 + a) + b equals the index-order sum of the general loop below bit for bit.
        static_assert(G::NSTRIP * 32 == W, "one strip per 32 columns");
        for (int i = et; i < SR * W; i += 32 * G::EW) {
          const int lr = i / W, col = i % W, j = col >> 5, off = col & 31;
          const float* sp = STR + lr * kTcStripW + off;
          float v = 0.f + sp[j * G::STRIP];
          if (off < MW - 1) v += sp[((j + G::NSTRIP - 1) % G::NSTRIP) * G::STRIP + 32];
          dst[i] = v;
        }
      } else
#endif
      for (int i = et; i < SR * W; i += 32 * G::EW) {
        const int lr = i / W, col = i % W;
        float v = 0.f;
#pragma unroll
        for (int s2 = 0; s2 < G::NSS; ++s2)
#pragma unroll
          for (int q2 = 0; q2 < 4; ++q2) {
            int off = col - ((TPR == 1 ? 0 : s2 * 128) + (32 * q2) % WT);
            if (off < 0) off += W;
            if (off < 32 + MW - 1) v += STR[(s2 * 4 + q2) * G::STRIP + lr * kTcStripW + off];
          }
        dst[i] = v;
      }
    }
  }
  umma::fence_before_sync();
  __syncthreads();
  if (warp == 0) {
    umma::fence_after_sync();
    umma::tmem_free<512>(tbase);
  }
}

// zmax of a stored u (coding_pass_tc's per warp-tile record, recomputed at the
// start of a coding call): max_k |clamp(u, beta) - u| over the 32 pixels that
// epilogue warp q handles in tile t of band b. Block (b * TPI + t, n), 128 threads.
template <class G>
__global__ void __launch_bounds__(128) tc_zmax_init(const float* __restrict__ u, float* __restrict__ zmax, int K,
                                                    float beta) {
  constexpr int W = G::W, D = G::D, TPR = G::TPR, WT = G::WT, RPT = G::RPT, RB = G::RB, TPI = G::TPI;
  const int n = blockIdx.y, b = blockIdx.x / TPI, t = blockIdx.x % TPI;
  const int p = threadIdx.x, lane = p & 31, q = p >> 5;
  const bool live = p < G::VALID;
  const int pc = live ? p : p - G::VALID;
  const int r = b * RB + (t / TPR) * RPT + pc / WT, c = (t % TPR) * 128 + pc % WT;
  const float* up = u + (size_t)n * K * D + (size_t)r * W + c;
  float m = 0.f;
  if (live)
    for (int k = 0; k < K; ++k) {
      const float v = __ldg(up + (size_t)k * D);
      m = fmaxf(m, fabsf(fminf(fmaxf(v, -beta), beta) - v));
    }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (lane == 0)
    for (int hh = 0; hh < G::HV; ++hh) zmax[(((size_t)n * gridDim.x + blockIdx.x) * 4 + q) * G::HV + hh] = m;
}

// s[n] = sum of the band partials (each output row from its own band and the
// previous one, in that order). Block (0, n) also reduces the stop-test sums
// over bands (fixed order) and runs the stop test of coding.cpp:264-283 once
// per image: ImageAdmm stats, conv[n], and upd[n] = "form the next lambda_hat".
template <class G>
__global__ void tc_band_reduce(const float* __restrict__ spart, const double* __restrict__ bsums, int* conv,
                               float* __restrict__ s, ImageAdmm* img, int* upd, int iter, int is_last) {
  constexpr int W = G::W, RB = G::RB, SR = G::SR, NBANDS = G::NBANDS, D = G::D;
  const int n = blockIdx.y;
  if (conv[n]) {
    if (blockIdx.x == 0 && threadIdx.x == 0) upd[n] = 0;
    return;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    double tt = 0, th = 0, t2 = 0, dz2 = 0, z2 = 0, dth = 0, tinf = 0;
    for (int bb = 0; bb < NBANDS; ++bb) {
      const double* o = bsums + ((size_t)n * NBANDS + bb) * kSums;
      tt += o[0]; th += o[1]; t2 += o[2]; dz2 += o[3]; z2 += o[4]; dth += o[5];
      tinf = fmax(tinf, o[6]);
    }
    const double denom = fmax(fmax(sqrt(th), sqrt(t2)), 1.0);
    const double primal = sqrt(tt) / denom;
    const double zc = sqrt(dz2) / fmax(sqrt(z2), 1.0);
    const double thc = sqrt(dth) / fmax(sqrt(th), 1.0);
    const bool stop = primal <= kAdmmRelTol && zc <= kAdmmRelTol && thc <= kAdmmRelTol;
    ImageAdmm& m = img[n];
    m.iters = iter;
    m.primal = primal;
    m.zc = zc;
    m.thc = thc;
    m.tinf = tinf;
    if (stop) m.converged = 1;
    upd[n] = (stop || is_last) ? 0 : 1;
    if (stop) conv[n] = 1;  // blocks of this launch that miss it write an s nobody reads
  }
  const float4* sp = reinterpret_cast<const float4*>(spart + (size_t)n * NBANDS * SR * W);
  float4* so = reinterpret_cast<float4*>(s + (size_t)n * D);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < D / 4; i += gridDim.x * blockDim.x) {
    const int r = (4 * i) / W, c4 = i % (W / 4);
    const int b0 = r / RB, lr0 = r - b0 * RB;
    const int bp = (b0 + NBANDS - 1) % NBANDS, lrp = lr0 + RB;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (lrp < SR) v = sp[((size_t)bp * SR + lrp) * (W / 4) + c4];
    const float4 w = sp[((size_t)b0 * SR + lr0) * (W / 4) + c4];
    v.x += w.x; v.y += w.y; v.z += w.z; v.w += w.w;
    so[i] = v;
  }
}

// lambda_hat = (DFT(s) - x_hat / rho) / sigma (lambda_from_w, coding.cpp:25-37) for
// the images whose stop test asked for the next iteration (upd[n])
template <class R>
__global__ void tc_lambda_apply(const cx<R>* __restrict__ shat, const cx<R>* __restrict__ xhat,
                                const R* __restrict__ sigma, cx<R>* __restrict__ lamhat, const int* __restrict__ upd,
                                int NB, R rho) {
  const int n = blockIdx.y;
  if (!upd[n]) return;
  const R inv_rho = R(1) / rho;
  for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < NB; b += gridDim.x * blockDim.x) {
    const cx<R> a = shat[(size_t)n * NB + b], xv = xhat[(size_t)n * NB + b];
    const R sg = sigma[b];
    lamhat[(size_t)n * NB + b] = mk<cx<R>>((a.x - xv.x * inv_rho) / sg, (a.y - xv.y * inv_rho) / sg);
  }
}

// lambda (spatial, per image) -> f16 hi / lo pair planes scaled by a power of
// two that maps max|lambda| to [2^13, 2^14).
template <int D>
__global__ void tc_lam_split(const float* __restrict__ lam, uint32_t* __restrict__ lam16, float* __restrict__ scale) {
  __shared__ float red[32];
  const int n = blockIdx.x;
  const float2* l2 = reinterpret_cast<const float2*>(lam + (size_t)n * D);
  float m = 0.f;
  for (int i = threadIdx.x; i < D / 2; i += blockDim.x) {
    const float2 v = l2[i];
    m = fmaxf(m, fmaxf(fabsf(v.x), fabsf(v.y)));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    m = threadIdx.x < (int)(blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (threadIdx.x == 0) red[0] = m;
  }
  __syncthreads();
  const float sc = umma::pow2_scale(red[0]);
  if (threadIdx.x == 0) scale[n] = sc;
  uint32_t* hi = lam16 + (size_t)n * D;
  uint32_t* lo = hi + D / 2;
  for (int i = threadIdx.x; i < D / 2; i += blockDim.x) {
    const float2 v = l2[i];
    umma::split2x2(v.x, v.y, sc, hi[i], lo[i]);
  }
}

// u planes of the single-CTA family (column-major pixel pairs: pair (r, m) at
// m*H + r) <-> row-major planes for the tensor-core pass: a float2 transpose of
// each [W/2][H] plane through 32 x 32 shared tiles. TO_ROWS: pairs -> rows.
template <bool TO_ROWS>
__global__ void tc_pair_transpose(const float2* __restrict__ src, float2* __restrict__ dst, int H, int W2) {
  __shared__ float2 t[32][33];
  const size_t plane = (size_t)blockIdx.z * H * W2;
  // TO_ROWS: src [W2][H] -> dst [H][W2]; else src [H][W2] -> dst [W2][H]
  const int R0 = TO_ROWS ? W2 : H, C0 = TO_ROWS ? H : W2;  // src rows x cols
  const int br = blockIdx.y * 32, bc = blockIdx.x * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int r = br + i, c = bc + threadIdx.x;
    if (r < R0 && c < C0) t[i][threadIdx.x] = src[plane + (size_t)r * C0 + c];
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int r = bc + i, c = br + threadIdx.x;  // dst [C0][R0]
    if (r < C0 && c < R0) dst[plane + (size_t)r * R0 + c] = t[threadIdx.x][i];
  }
}

// dictionary K x TAPS (FP64, tap o = y*MW + x) -> f16 hi / lo core-matrix grid:
// element (k, o) at ((k/8)*(TP/8) + o/8)*64 + (k%8)*8 + o%8 halves; zero padded to KF x TP.
template <int KF, int TP>
__global__ void tc_dsplit(const double* __restrict__ d, int K, int taps, float scale, __half* __restrict__ out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < KF * TP; i += gridDim.x * blockDim.x) {
    const int k = i / TP, o = i % TP;
    const float v = (k < K && o < taps) ? (float)d[(size_t)k * taps + o] : 0.f;
    __half hi, lo;
    umma::split2(v, scale, hi, lo);
    const int idx = (((k >> 3) * (TP / 8) + (o >> 3)) * 8 + (k & 7)) * 8 + (o & 7);
    out[idx] = hi;
    out[KF * TP + idx] = lo;
  }
}

}  // namespace dcsc_cuda
