// Device kernels of the dual-domain CSC hot path, templated on the plane type
// P = Plane<R, H, W, T> (fft2d.cuh). Reference anchors are cited per kernel.
#pragma once
#include "fft2d.cuh"

namespace dcsc_cuda {

constexpr double kAdmmRelTol = 1e-4;  // proj/include/dcsc/coding.hpp:41

enum PassMode : int {
  kPassAdmm = 0,      // one full ADMM iteration for a filter group
  kPassPrologue = 1,  // w = theta + z/rho from the stored state -> acc (initial lambda)
  kPassObjective = 2, // z from the ADMM state -> acc = sum_k d_hat_k z_hat_k, l1
  kPassMaps = 3,      // z from the accepted-maps buffer -> acc, l1
};

// Per-(image, group) partial sums written by coding_pass, in slot order:
// 0 sum (theta'-t)^2, 1 sum theta'^2, 2 sum t^2, 3 sum dz^2, 4 sum z'^2,
// 5 sum dtheta^2, 6 max|t|, 7 unused. (proj/src/coding.cpp:237-259)
// Objective modes: 0 = sum |z|.
constexpr int kSums = 8;

// Per-image ADMM bookkeeping written by the last CTA of the image (coding_pass epilogue) or lambda_update.
struct ImageAdmm {
  int iters;
  int converged;
  double primal, zc, thc, tinf;
};

template <class R>
struct CodingArgs {
  const cx<R>* dhat;    // K x NB filter spectra
  const cx<R>* lamhat;  // N x NB current lambda_hat
  R* u;                 // N x K x D ADMM state u = t - z/rho (theta = clamp(u), z = rho(theta-u))
  const R* maps;        // N x K x D accepted maps (kPassMaps)
  cx<R>* part;          // N x G x NB partial sum_k d_hat_k w_hat_k
  double* sums;         // N x G x kSums
  const int* conv;      // N: nonzero = this image's ADMM has stopped
  int K, G, kpg;
  R rho, beta;
  const cx<R>* tw;      // twiddle table (global)
  // fused lambda update (last CTA of each image, see lambda_epilogue)
  unsigned* cnt;        // N arrival counters, zero between launches
  int* conv_w;          // conv, writable
  const cx<R>* xhat;    // N x NB
  const R* sigma;       // NB
  cx<R>* lamhat_w;      // N x NB
  struct ImageAdmm* img;
  int iter, is_last;
  // multi-channel (TCSC, J > 1) passes: dhat is J x K x NB (channel-major),
  // lamhat N x J x NB; the pass stores w_hat_k to what (N x K x NB) instead of
  // accumulating, and the per-bin J x J solve runs in tc_lambda.
  int J;
  cx<R>* what;
  // cluster family (J = 1): d_hat in the rank-blocked layout K x CL x [H][CS]
  // (cl_rank_block), so a rank's generator slice is one contiguous TMA copy;
  // nullptr: the generator reads d_hat from L2
  const cx<R>* dhat_rb;
  // warm state whose theta is not clamp(theta - z/rho) (set_coding_state of a
  // state not produced by ADMM): theta (u layout) for the prologue's
  // w = theta + z/rho and the first iteration's theta_old; nullptr otherwise
  const R* theta0;
};

// Bulk prefetch of a contiguous global range into L2 (sm_90+ TMA engine op).
__device__ __forceinline__ void prefetch_l2_bulk(const void* p, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// ---- TMA bulk copies (cp.async.bulk) with mbarrier completion (sm_90+/sm_100a)
__device__ __forceinline__ unsigned smem_addr(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_addr(dst)),
               "l"(src), "r"(bytes), "r"(smem_addr(bar))
               : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_addr(src)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

template <class P>
struct Smem {
  static constexpr size_t tw_bytes = sizeof(typename P::C) * (P::TW_LEN + P::H);  // + COL0
  static constexpr size_t two = 2 * P::buffer_bytes + tw_bytes;
  static constexpr size_t three = 3 * P::buffer_bytes + tw_bytes;
  // per-filter ADMM state staged in smem by one TMA bulk copy (dense H x M pairs)
  static constexpr int US = P::M;
  static constexpr size_t u_bytes = sizeof(typename P::C) * P::H * US;
  static constexpr size_t u_off = (two + 127) / 128 * 128;
  // Preferred: lambda_hat of the CTA's image resident in smem for the whole
  // filter group (one TMA load per CTA; the generated t_hat stage then reads
  // only d_hat from L2) and u read straight from L2/HBM in the fused row stage
  // (column-major pairs: coalesced). Fallback when that does not fit: stage
  // each filter's u plane by TMA.
  static constexpr size_t lam_bytes = sizeof(typename P::C) * P::NB;
  static constexpr bool lam_smem = u_off + lam_bytes <= 220 * 1024;
  static constexpr bool stage_u = !lam_smem && u_off + u_bytes <= 220 * 1024;
  static constexpr size_t coding = lam_smem ? u_off + lam_bytes : (stage_u ? u_off + u_bytes : two);
};

// ----------------------------------------------------------------------------
// The fused coding kernel. One CTA = (image n, filter group g); for each filter:
//   t_hat = conj(d_hat_k) lambda_hat           (coding.cpp:77-86, correlate)
//     generated inside the first inverse column stage (no smem pass)
//   t = iDFT(t_hat)                            (coding.cpp:234)
//   theta' = clamp(t - z/rho), z' = z + rho(theta'-t)   (coding.cpp:237-246)
//     in closed form on u: u' = t - z/rho, theta' = clamp(u'), z' = rho(theta'-u')
//   w = theta' + z'/rho = 2 theta' - u'  ->  w_hat = DFT(w)
//     (one forward FFT replaces DFT(theta) and DFT(z), coding.cpp:260-261,224-227)
//   acc += d_hat_k w_hat_k  inside the last forward column stage
//                                              (lambda_from_w numerator, coding.cpp:25-37)
// The last CTA of each image runs the stop test and the lambda_hat update.
// ----------------------------------------------------------------------------
// TC (multi-channel, J > 1, tcsc.cpp:121-171): t_hat_k = sum_j conj(d_hat_jk)
// lambda_hat_j in the generator, w_hat_k stored to a.what by the last forward
// column stage, and the epilogue only runs the stop test (tc_lambda solves
// the per-bin J x J systems).
// JT > 0: the channel count as a compile-time constant (the t_hat generator's
// channel loop is then unrolled and its 2J loads per bin issued together).
template <class P, int MODE, bool TC = false, int JT = 0>
__global__ void __launch_bounds__(P::T) coding_pass(CodingArgs<typename P::R> a) {
  using R = typename P::R;
  using C = typename P::C;
  constexpr int H = P::H, W = P::W, Wh = P::Wh, NB = P::NB, D = P::D, T = P::T, M = P::M;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ double red[kSums * (T / 32)];
  C* B0 = reinterpret_cast<C*>(smem_raw);
  C* B1 = B0 + NB;
  C* TW = B1 + NB;
  C* COL0 = TW + P::TW_LEN;
  constexpr bool STAGE = (MODE == kPassAdmm) && !TC && Smem<P>::stage_u;
  constexpr int US = Smem<P>::US;
  C* U = reinterpret_cast<C*>(smem_raw + Smem<P>::u_off);
  __shared__ __align__(8) unsigned long long ubar_s;
  unsigned long long* ubar = &ubar_s;
  unsigned uphase = 0;
  const int n = blockIdx.y, g = blockIdx.x;
  if (MODE == kPassAdmm && a.conv[n]) return;

  constexpr bool LAMS = (MODE == kPassAdmm) && !TC && Smem<P>::lam_smem;
  C* LAM = reinterpret_cast<C*>(smem_raw + Smem<P>::u_off);
  // With lambda_hat in smem, the t_hat stage's only global operand is d_hat:
  // each filter's d_hat plane is staged into the free plane buffer by one TMA
  // bulk copy issued at the start of the previous filter's last forward column
  // stage (which reads only the other buffer), so its L2 latency overlaps
  // that stage. The column-0 epilogue's d_hat(r, 0), d_hat(r, W/2) are
  // fetched into registers at the same point (d0, dM).
  constexpr bool PREF = LAMS;
  __shared__ __align__(8) unsigned long long dbar_s;
  unsigned long long* dbar = &dbar_s;
  unsigned dphase = 0;
  C* stg = B1;  // buffer holding the staged d_hat of the current filter
  C d0 = mk<C>(R(0), R(0)), dMv = mk<C>(R(0), R(0));
  P::load_twiddles(TW, a.tw);
  if ((STAGE || LAMS) && threadIdx.x == 0) {
    mbar_init(ubar, 1);
    if (PREF) mbar_init(dbar, 1);
    fence_async_smem();
  }
  __syncthreads();
  if constexpr (LAMS) {
    if (threadIdx.x == 0) {
      mbar_expect_tx(ubar, (unsigned)(sizeof(C) * NB));
      bulk_g2s(LAM, a.lamhat + (size_t)n * NB, (unsigned)(sizeof(C) * NB), ubar);
      if (PREF && g * a.kpg < a.K) {
        mbar_expect_tx(dbar, (unsigned)(sizeof(C) * NB));
        bulk_g2s(stg, a.dhat + (size_t)g * a.kpg * NB, (unsigned)(sizeof(C) * NB), dbar);
      }
    }
    mbar_wait(ubar, 0);
  }
  // sum_k d_hat_k w_hat_k for this group, in registers of the bins' owners
  C acc[P::LAST_IPT][P::LAST_R];
#pragma unroll
  for (int i = 0; i < P::LAST_IPT; ++i)
#pragma unroll
    for (int s = 0; s < P::LAST_R; ++s) acc[i][s] = mk<C>(R(0), R(0));
  C acc0 = mk<C>(R(0), R(0)), accN = mk<C>(R(0), R(0));  // bins (tid, 0), (tid, W/2)

  const R rho = a.rho, beta = a.beta, invD = R(1) / R(D);
  // per-thread stop-test sums over the CTA's filters, in the storage precision
  // (FP32: <= 32 terms per filter x kpg filters per thread before the FP64 block
  // reduction); Σdz² = ρ²·Σ(θ'−t)² and Σz'² = ρ²·Σ(z'/ρ)² are formed at the end
  R s0 = 0, s1 = 0, s2 = 0, s4 = 0, s5 = 0, s6 = 0;
  const int k0 = g * a.kpg;
  const int k1 = min(a.K, k0 + a.kpg);
  // TC: forward column pass of the row FFTs in z, natural bins of w_hat_k -> a.what
  auto store_what = [&](C* z, C* other, int k) {
    C* wk = a.what + ((size_t)n * a.K + k) * NB;
    P::cols_fwd(z, other, TW, COL0, [](int, int) { return 0; }, [&](int r, int c, C v, int) { wk[r * Wh + c] = v; });
    if (threadIdx.x < H) {
      C x0, xn;
      P::template unpack_col0<1>(COL0, threadIdx.x, x0, xn);
      wk[threadIdx.x * Wh] = x0;
      wk[threadIdx.x * Wh + M] = xn;
    }
  };
  for (int k = k0; k < k1; ++k) {
    const C* __restrict__ dk = a.dhat + (size_t)k * NB;
    C* work;
    if constexpr (MODE == kPassAdmm) {
      C* __restrict__ uk = reinterpret_cast<C*>(a.u + ((size_t)n * a.K + k) * D);  // pixel pairs
      const C* __restrict__ t0k =
          a.theta0 ? reinterpret_cast<const C*>(a.theta0 + ((size_t)n * a.K + k) * D) : nullptr;
      const C* __restrict__ lam = a.lamhat + (size_t)n * NB;
      if constexpr (STAGE) {
        // TMA: this filter's u rows -> U (padded rows); lands during the inverse FFT
        if (threadIdx.x == 0) {
          bulk_wait_read0();  // the previous filter's U store has drained
          mbar_expect_tx(ubar, (unsigned)(sizeof(C) * H * M));
          bulk_g2s(U, uk, sizeof(C) * H * M, ubar);
        }
      } else if (threadIdx.x == 0) {
        prefetch_l2_bulk(uk, sizeof(R) * D);
      }
      if (threadIdx.x == 0 && k + 1 < k1) prefetch_l2_bulk(dk + NB, sizeof(C) * NB);
      C* cs;
      if constexpr (TC) {
        const int J = JT > 0 ? JT : a.J;
        cs = P::template cols_inv<true, true>(B0, B1, TW, [&](int r, int c) {
          const int b = r * Wh + c;
          C t = mk<C>(R(0), R(0));
#pragma unroll
          for (int j = 0; j < J; ++j)
            t = cadd(t, cmulc(__ldg(a.dhat + ((size_t)j * a.K + k) * NB + b), __ldg(a.lamhat + ((size_t)n * J + j) * NB + b)));
          return t;
        });
      } else if constexpr (PREF) {
        mbar_wait(dbar, dphase);
        dphase ^= 1u;
        const C* sd = stg;
        cs = P::template cols_inv<false>(stg == B0 ? B1 : B0, stg, TW, [&](int r, int c) {
          const int b = r * Wh + c;
          return cmulc(sd[b], LAM[b]);
        });
      } else {
        cs = P::cols_inv(B0, B1, TW, [&](int r, int c) {
          const int b = r * Wh + c;
          return cmulc(__ldg(dk + b), LAMS ? LAM[b] : __ldg(lam + b));
        });
      }
      C* hin = P::rows_inv_head(cs, cs == B0 ? B1 : B0, TW);
      C* fout = (hin == B0) ? B1 : B0;
      // fused: last inverse row stage -> prox on u -> first forward row stage,
      // in registers. u is stored column-major per plane (pair m, row r at
      // m*H + r) so lanes over rows read U / u conflict-free and coalesced.
      if constexpr (STAGE) mbar_wait(ubar, uphase);
      uphase ^= 1u;
      {
        constexpr int RX = P::RX, J = M / RX;
        const C* twr = TW + P::TW_ROW;
        R& f0 = s0; R& f1 = s1; R& f2 = s2; R& f4 = s4; R& f5 = s5; R& f6 = s6;
#pragma unroll 1
        for (int it = threadIdx.x; it < H * J; it += T) {
          const int r = it % H, j = it / H;
          C x[RX];
#pragma unroll
          for (int q = 0; q < RX; ++q)
            x[q] = (P::RI_N == 1) ? P::pre(hin, TW, r, j + q * J) : hin[r * Wh + j + q * J];
          if constexpr (P::RI_N > 1) stage_twiddle<C, RX, 1, true>(x, twr, j);
          dft<RX, true>(x);
#pragma unroll
          for (int s = 0; s < RX; ++s) {
            C* up = (STAGE ? U : uk) + (j + s * J) * H + r;
            const C uv = STAGE ? *up : __ldcs(up);  // u streams through once: evict-first
            const R tv[2] = {x[s].x * invD, x[s].y * invD};
            const R uo[2] = {uv.x, uv.y};
            C t0v = mk<C>(R(0), R(0));
            if (t0k) t0v = __ldg(t0k + (j + s * J) * H + r);
            const R t0[2] = {t0v.x, t0v.y};
            R wv[2], un2[2];
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const R t = tv[e];
              const R th_o = t0k ? t0[e] : fmin(fmax(uo[e], -beta), beta);
              const R un = t - (th_o - uo[e]);           // u' = t - z/rho
              const R th = fmin(fmax(un, -beta), beta);  // theta' = clamp(u')
              const R ez = th - un;                      // z' / rho
              const R d_tt = th - t;                     // (z' - z) / rho
              const R dth = th - th_o;
              f0 += d_tt * d_tt;                         // sum dz^2 = rho^2 f0 (slot 3)
              f1 += th * th;
              f2 += t * t;
              f4 += ez * ez;                             // sum z'^2 = rho^2 f4
              f5 += dth * dth;
              f6 = fmax(f6, fabs(t));
              wv[e] = th + ez;                           // w = theta' + z'/rho
              un2[e] = un;
            }
            if constexpr (STAGE) *up = mk<C>(un2[0], un2[1]);
            else __stcs(up, mk<C>(un2[0], un2[1]));
            x[s] = mk<C>(wv[0], wv[1]);
          }
          dft<RX, false>(x);  // first forward row stage (NS = 1)
#pragma unroll
          for (int s = 0; s < RX; ++s) fout[r * Wh + j * RX + s] = x[s];
        }
      }
      if constexpr (STAGE) fence_async_smem();
      __syncthreads();
      if constexpr (STAGE) {
        if (threadIdx.x == 0) {
          bulk_s2g(uk, U, sizeof(C) * H * M);
          bulk_commit();
        }
      }
      C* z = P::rows_fwd_tail(fout, hin, TW);
      if constexpr (TC) {
        store_what(z, z == B0 ? B1 : B0, k);
        continue;
      }
      P::cols_fwd_acc(z, z == B0 ? B1 : B0, TW, COL0, dk, acc, [&](C* freebuf) {
        if constexpr (PREF) {
          if (threadIdx.x < H) {
            d0 = __ldg(dk + threadIdx.x * Wh);
            dMv = __ldg(dk + threadIdx.x * Wh + M);
          }
          stg = freebuf;
          if (threadIdx.x == 0 && k + 1 < k1) {
            fence_async_smem();
            mbar_expect_tx(dbar, (unsigned)(sizeof(C) * NB));
            bulk_g2s(freebuf, dk + NB, (unsigned)(sizeof(C) * NB), dbar);
          }
        }
      });
      if (threadIdx.x < H) {
        const int r = threadIdx.x;
        C x0, xn;
        P::template unpack_col0<1>(COL0, r, x0, xn);
        if constexpr (PREF) {
          acc0 = cadd(acc0, cmul(d0, x0));
          accN = cadd(accN, cmul(dMv, xn));
        } else {
          acc0 = cadd(acc0, cmul(__ldg(dk + r * Wh), x0));
          accN = cadd(accN, cmul(__ldg(dk + r * Wh + M), xn));
        }
      }
      continue;
    } else {
      const C* __restrict__ src = reinterpret_cast<const C*>(
          (MODE == kPassMaps) ? a.maps + ((size_t)n * a.K + k) * D : a.u + ((size_t)n * a.K + k) * D);
      const C* __restrict__ t0k =
          (MODE == kPassPrologue && a.theta0) ? reinterpret_cast<const C*>(a.theta0 + ((size_t)n * a.K + k) * D)
                                              : nullptr;
      for (int it = threadIdx.x; it < H * M; it += T) {
        const int r = it / M, m = it % M;
        // maps are row-major [r][c]; u is column-major pairs [m][r]
        const C v = (MODE == kPassMaps) ? src[it] : src[m * H + r];
        R w0, w1;
        if constexpr (MODE == kPassPrologue) {
          // w = theta + z/rho = 2 theta - u (theta = clamp(u) for an ADMM-produced state)
          const C th = t0k ? t0k[m * H + r] : mk<C>(fmin(fmax(v.x, -beta), beta), fmin(fmax(v.y, -beta), beta));
          w0 = R(2) * th.x - v.x;
          w1 = R(2) * th.y - v.y;
        } else if constexpr (MODE == kPassObjective) {
          w0 = rho * (fmin(fmax(v.x, -beta), beta) - v.x);
          w1 = rho * (fmin(fmax(v.y, -beta), beta) - v.y);
          s0 += fabs(w0) + fabs(w1);
        } else {
          w0 = v.x;
          w1 = v.y;
          s0 += fabs(w0) + fabs(w1);
        }
        B0[r * Wh + m] = mk<C>(w0, w1);
      }
      __syncthreads();
      work = B0;
    }
    // forward r2c of w with acc += d_hat_k w_hat_k fused into the last column stage
    C* other = (work == B0) ? B1 : B0;
    C* z = P::rows_fwd(work, other, TW);
    if constexpr (TC) {
      store_what(z, z == work ? other : work, k);
      continue;
    }
    P::cols_fwd_acc(z, z == work ? other : work, TW, COL0, dk, acc, [](C*) {});
    static_assert(H <= T, "column-0 owners: one thread per row");
    if (threadIdx.x < H) {
      const int r = threadIdx.x;
      C x0, xn;
      P::template unpack_col0<1>(COL0, r, x0, xn);
      acc0 = cadd(acc0, cmul(__ldg(dk + r * Wh), x0));
      accN = cadd(accN, cmul(__ldg(dk + r * Wh + M), xn));
    }
  }
  if (STAGE && threadIdx.x == 0) bulk_wait0();  // u stores complete before the CTA retires
  if constexpr (!TC) {
    C* dst = a.part + ((size_t)n * a.G + g) * NB;
#pragma unroll
    for (int i = 0; i < P::LAST_IPT; ++i) {
      const int it = threadIdx.x + i * T;
      if (it >= P::LAST_ITEMS || it % M == 0) continue;
#pragma unroll
      for (int s = 0; s < P::LAST_R; ++s) {
        int r, c;
        P::acc_bin(i, s, r, c);
        dst[r * Wh + c] = acc[i][s];
      }
    }
    if (threadIdx.x < H) {
      dst[threadIdx.x * Wh] = acc0;
      dst[threadIdx.x * Wh + M] = accN;
    }
  }
  // reductions of the partial sums (FP64)
  const double rr2 = (double)rho * (double)rho;
  double v[7] = {(double)s0, (double)s1, (double)s2, MODE == kPassAdmm ? rr2 * (double)s0 : 0.0,
                 rr2 * (double)s4, (double)s5, 0.0};
  block_sum<T, 7>(v, red);
  const double mx = block_max((double)s6, red, T);
  if (threadIdx.x == 0) {
    double* o = a.sums + ((size_t)n * a.G + g) * kSums;
    for (int i = 0; i < 6; ++i) o[i] = v[i];
    o[6] = mx;
    o[7] = 0.0;
  }
  if constexpr (MODE == kPassAdmm || MODE == kPassPrologue) {
    // Last CTA of image n to finish reduces the G partials: stop test
    // (coding.cpp:264-283) and lambda_hat = (sum - x_hat/rho)/sigma (:25-37).
    __shared__ int last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
      const unsigned prev = atomicAdd(a.cnt + n, 1u);
      last = prev == (unsigned)(a.G - 1);
      if (last) a.cnt[n] = 0;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    bool stop = false;
    if (MODE == kPassAdmm) {
      double tt = 0, th = 0, t2 = 0, dz2 = 0, z2 = 0, dth = 0, tinf = 0;
      for (int gg = 0; gg < a.G; ++gg) {
        const double* s = a.sums + ((size_t)n * a.G + gg) * kSums;
        tt += __ldcg(s + 0); th += __ldcg(s + 1); t2 += __ldcg(s + 2); dz2 += __ldcg(s + 3);
        z2 += __ldcg(s + 4); dth += __ldcg(s + 5);
        tinf = fmax(tinf, __ldcg(s + 6));
      }
      const double denom = fmax(fmax(sqrt(th), sqrt(t2)), 1.0);
      const double primal = sqrt(tt) / denom;
      const double zc = sqrt(dz2) / fmax(sqrt(z2), 1.0);
      const double thc = sqrt(dth) / fmax(sqrt(th), 1.0);
      stop = primal <= kAdmmRelTol && zc <= kAdmmRelTol && thc <= kAdmmRelTol;
      if (threadIdx.x == 0) {
        ImageAdmm& m = a.img[n];
        m.iters = a.iter;
        m.primal = primal;
        m.zc = zc;
        m.thc = thc;
        m.tinf = tinf;
        if (stop) {
          m.converged = 1;
          a.conv_w[n] = 1;
        }
      }
    }
    if (TC || stop || (MODE == kPassAdmm && a.is_last)) return;
    const R inv_rho = R(1) / rho;
    const C* pn = a.part + (size_t)n * a.G * NB;
    for (int b = threadIdx.x; b < NB; b += T) {
      C acc = __ldcg(pn + b);  // L2 view of the other CTAs' partials
      for (int gg = 1; gg < a.G; ++gg) acc = cadd(acc, __ldcg(pn + (size_t)gg * NB + b));
      const C xv = a.xhat[(size_t)n * NB + b];
      const R s = a.sigma[b];
      a.lamhat_w[(size_t)n * NB + b] = mk<C>((acc.x - xv.x * inv_rho) / s, (acc.y - xv.y * inv_rho) / s);
    }
  }
}

// ----------------------------------------------------------------------------
// lambda_hat = (sum_g part_g - x_hat / rho) / sigma    (coding.cpp:25-37)
// preceded by the per-image stop test on the iteration's partial sums
// (coding.cpp:264-283). A converging or final iteration keeps lambda_hat.
// ----------------------------------------------------------------------------
template <class R>
__global__ void lambda_update(const cx<R>* __restrict__ part, const double* __restrict__ sums,
                              const cx<R>* __restrict__ xhat, const R* __restrict__ sigma,
                              cx<R>* __restrict__ lamhat, int* conv, ImageAdmm* img, int G, int NB,
                              R rho, int iter, int is_last, int prologue) {
  using C = cx<R>;
  const int n = blockIdx.y;
  if (!prologue && conv[n]) return;
  bool stop = false;
  if (!prologue) {
    double tt = 0, th = 0, t2 = 0, dz2 = 0, z2 = 0, dth = 0, tinf = 0;
    for (int g = 0; g < G; ++g) {
      const double* s = sums + ((size_t)n * G + g) * kSums;
      tt += s[0]; th += s[1]; t2 += s[2]; dz2 += s[3]; z2 += s[4]; dth += s[5];
      tinf = fmax(tinf, s[6]);
    }
    const double denom = fmax(fmax(sqrt(th), sqrt(t2)), 1.0);
    const double primal = sqrt(tt) / denom;
    const double zc = sqrt(dz2) / fmax(sqrt(z2), 1.0);
    const double thc = sqrt(dth) / fmax(sqrt(th), 1.0);
    stop = primal <= kAdmmRelTol && zc <= kAdmmRelTol && thc <= kAdmmRelTol;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      ImageAdmm& m = img[n];
      m.iters = iter;
      m.primal = primal;
      m.zc = zc;
      m.thc = thc;
      m.tinf = tinf;
      if (stop) {
        m.converged = 1;
        conv[n] = 1;
      }
    }
  }
  if (stop || is_last) return;
  const R inv_rho = R(1) / rho;
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= NB) return;
  C acc = part[((size_t)n * G) * NB + b];
  for (int g = 1; g < G; ++g) acc = cadd(acc, part[((size_t)n * G + g) * NB + b]);
  const C xv = xhat[(size_t)n * NB + b];
  const R s = sigma[b];
  lamhat[(size_t)n * NB + b] = mk<C>((acc.x - xv.x * inv_rho) / s, (acc.y - xv.y * inv_rho) / s);
}

// ----------------------------------------------------------------------------
// Batched r2c of real planes (x_hat, z_hat, padded filters) and c2r.
// ----------------------------------------------------------------------------
// Shared tail: forward FFT of the spatial pairs in B0, NSL spectrum to `d`.
template <class P>
__device__ __forceinline__ void forward_to_global(typename P::C* B0, typename P::C* B1, const typename P::C* TW,
                                                  typename P::C* COL0, typename P::C* __restrict__ d) {
  using C = typename P::C;
  constexpr int Wh = P::Wh, M = P::M, H = P::H, T = P::T;
  C* z = P::rows_fwd(B0, B1, TW);
  P::cols_fwd(z, z == B0 ? B1 : B0, TW, COL0, [](int, int) { return 0; },
              [&](int r, int c, C v, int) { d[r * Wh + c] = v; });
  for (int r = threadIdx.x; r < H; r += T) {
    C x0, xn;
    P::template unpack_col0<1>(COL0, r, x0, xn);
    d[r * Wh] = x0;
    d[r * Wh + M] = xn;
  }
}

template <class P, class SRC>
__global__ void __launch_bounds__(P::T)
r2c_planes(const SRC* __restrict__ src, size_t src_stride, cx<typename P::R>* __restrict__ dst,
           size_t dst_stride, const cx<typename P::R>* tw, int* live_flags, int live_mod) {
  using R = typename P::R;
  using C = typename P::C;
  constexpr int H = P::H, W = P::W, Wh = P::Wh, NB = P::NB, T = P::T, M = P::M;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  C* B0 = reinterpret_cast<C*>(smem_raw);
  C* B1 = B0 + NB;
  C* TW = B1 + NB;
  C* COL0 = TW + P::TW_LEN;
  const int p = blockIdx.x;
  P::load_twiddles(TW, tw);
  const SRC* s = src + (size_t)p * src_stride;
  int any = 0;
  for (int it = threadIdx.x; it < H * M; it += T) {
    const int r = it / M, m = it % M;
    R v0, v1;
    if constexpr (std::is_same<SRC, R>::value) {  // pixel pair as one vector load
      const C v = reinterpret_cast<const C*>(s)[it];
      v0 = v.x;
      v1 = v.y;
    } else {
      v0 = R(s[r * W + 2 * m]);
      v1 = R(s[r * W + 2 * m + 1]);
    }
    any |= (v0 != R(0)) | (v1 != R(0));
    B0[r * Wh + m] = mk<C>(v0, v1);
  }
  __syncthreads();
  if (live_flags) {
    any = __syncthreads_or(any);
    if (threadIdx.x == 0 && any) atomicOr(live_flags + (p % live_mod), 1);
  }
  forward_to_global<P>(B0, B1, TW, COL0, dst + (size_t)p * dst_stride);
}

// Persistent, pipelined batched transforms: one CTA per SM slot walks planes
// p = blockIdx.x, + gridDim.x, ...; the next plane's input streams into a
// staging buffer by one TMA bulk copy while the current plane transforms, so
// the HBM read overlaps the FFT instead of preceding it (the one-CTA-per-plane
// kernels above serialise load -> FFT -> store on each SM).
template <class P>
struct SmemPipe {
  using R = typename P::R;
  using C = typename P::C;
  static constexpr size_t stg_off = (Smem<P>::two + 127) / 128 * 128;
  static constexpr size_t r2c = stg_off + sizeof(R) * P::D;   // + real plane
  static constexpr size_t c2r = stg_off + sizeof(C) * P::NB;  // + half spectrum
  static constexpr bool r2c_ok = r2c <= 220 * 1024 && (sizeof(R) * P::D) % 16 == 0;
  static constexpr bool c2r_ok = c2r <= 220 * 1024 && (sizeof(C) * P::NB) % 16 == 0;
};

template <class P>
__global__ void __launch_bounds__(P::T)
r2c_planes_pipe(const typename P::R* __restrict__ src, size_t src_stride, cx<typename P::R>* __restrict__ dst,
                size_t dst_stride, const cx<typename P::R>* tw, int* live_flags, int live_mod, int count) {
  using R = typename P::R;
  using C = typename P::C;
  constexpr int H = P::H, Wh = P::Wh, NB = P::NB, T = P::T, M = P::M;
  constexpr unsigned BYTES = sizeof(R) * P::D;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ __align__(8) unsigned long long bar_s;
  C* B0 = reinterpret_cast<C*>(smem_raw);
  C* B1 = B0 + NB;
  C* TW = B1 + NB;
  C* COL0 = TW + P::TW_LEN;
  const C* STG = reinterpret_cast<const C*>(smem_raw + SmemPipe<P>::stg_off);
  unsigned long long* bar = &bar_s;
  P::load_twiddles(TW, tw);
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_async_smem();
  }
  __syncthreads();
  int p = blockIdx.x;
  if (threadIdx.x == 0 && p < count) {
    mbar_expect_tx(bar, BYTES);
    bulk_g2s((void*)STG, src + (size_t)p * src_stride, BYTES, bar);
  }
  unsigned phase = 0;
  for (; p < count; p += gridDim.x) {
    mbar_wait(bar, phase);
    phase ^= 1u;
    int any = 0;
    for (int it = threadIdx.x; it < H * M; it += T) {  // pixel pairs -> [H][Wh]
      const C v = STG[it];
      any |= (v.x != R(0)) | (v.y != R(0));
      B0[(it / M) * Wh + it % M] = v;
    }
    if (live_flags) {
      any = __syncthreads_or(any);
      if (threadIdx.x == 0 && any) atomicOr(live_flags + (p % live_mod), 1);
    } else {
      __syncthreads();
    }
    const int nx = p + gridDim.x;
    if (threadIdx.x == 0 && nx < count) {  // staging consumed: the next plane streams in
      fence_async_smem();
      mbar_expect_tx(bar, BYTES);
      bulk_g2s((void*)STG, src + (size_t)nx * src_stride, BYTES, bar);
    }
    forward_to_global<P>(B0, B1, TW, COL0, dst + (size_t)p * dst_stride);
    __syncthreads();
  }
}

template <class P>
__global__ void __launch_bounds__(P::T)
c2r_planes_pipe(const cx<typename P::R>* __restrict__ src, size_t src_stride, typename P::R* __restrict__ dst,
                size_t dst_stride, const cx<typename P::R>* tw, int count) {
  using R = typename P::R;
  using C = typename P::C;
  constexpr int H = P::H, Wh = P::Wh, NB = P::NB, T = P::T, D = P::D, M = P::M;
  constexpr unsigned BYTES = sizeof(C) * NB;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ __align__(8) unsigned long long bar_s;
  C* B0 = reinterpret_cast<C*>(smem_raw);
  C* B1 = B0 + NB;
  C* TW = B1 + NB;
  C* STG = reinterpret_cast<C*>(smem_raw + SmemPipe<P>::stg_off);
  unsigned long long* bar = &bar_s;
  P::load_twiddles(TW, tw);
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_async_smem();
  }
  __syncthreads();
  int p = blockIdx.x;
  if (threadIdx.x == 0 && p < count) {
    mbar_expect_tx(bar, BYTES);
    bulk_g2s(STG, src + (size_t)p * src_stride, BYTES, bar);
  }
  unsigned phase = 0;
  const R sc = R(1.0 / (double)D);
  for (; p < count; p += gridDim.x) {
    mbar_wait(bar, phase);
    phase ^= 1u;
    // the first column stage reads the staged spectrum; cols_inv syncs after it
    C* c = P::template cols_inv<false>(B0, B1, TW, [&](int r, int cc) { return STG[r * Wh + cc]; });
    const int nx = p + gridDim.x;
    if (threadIdx.x == 0 && nx < count) {  // staging consumed: the next spectrum streams in
      fence_async_smem();
      mbar_expect_tx(bar, BYTES);
      bulk_g2s(STG, src + (size_t)nx * src_stride, BYTES, bar);
    }
    C* sp = P::rows_inv(c, c == B0 ? B1 : B0, TW);
    C* o = reinterpret_cast<C*>(dst + (size_t)p * dst_stride);
    for (int it = threadIdx.x; it < H * M; it += T) {
      const C v = sp[(it / M) * Wh + it % M];
      o[it] = mk<C>(v.x * sc, v.y * sc);
    }
    __syncthreads();
  }
}

// Zero-padded filters (corner placement, spectral.cpp:106-122) -> spectra.
template <class P>
__global__ void __launch_bounds__(P::T)
r2c_filters(const double* __restrict__ d, int mh, int mw, cx<typename P::R>* __restrict__ dst,
            const cx<typename P::R>* tw) {
  using R = typename P::R;
  using C = typename P::C;
  constexpr int H = P::H, Wh = P::Wh, NB = P::NB, T = P::T, M = P::M;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  C* B0 = reinterpret_cast<C*>(smem_raw);
  C* B1 = B0 + NB;
  C* TW = B1 + NB;
  C* COL0 = TW + P::TW_LEN;
  const int k = blockIdx.x;
  P::load_twiddles(TW, tw);
  const double* f = d + (size_t)k * mh * mw;
  for (int it = threadIdx.x; it < H * M; it += T) {
    const int r = it / M, m = it % M;
    const int c0 = 2 * m, c1 = c0 + 1;
    const R v0 = (r < mh && c0 < mw) ? R(f[r * mw + c0]) : R(0);
    const R v1 = (r < mh && c1 < mw) ? R(f[r * mw + c1]) : R(0);
    B0[r * Wh + m] = mk<C>(v0, v1);
  }
  __syncthreads();
  forward_to_global<P>(B0, B1, TW, COL0, dst + (size_t)k * NB);
}

// Batched c2r of NSL spectra (scaled by `scale`/D) into real planes.
template <class P, class DST>
__global__ void __launch_bounds__(P::T)
c2r_planes(const cx<typename P::R>* __restrict__ src, size_t src_stride, DST* __restrict__ dst,
           size_t dst_stride, const cx<typename P::R>* tw, const double* scale) {
  using R = typename P::R;
  using C = typename P::C;
  constexpr int H = P::H, W = P::W, Wh = P::Wh, NB = P::NB, T = P::T, D = P::D, M = P::M;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  C* B0 = reinterpret_cast<C*>(smem_raw);
  C* B1 = B0 + NB;
  C* TW = B1 + NB;
  const int p = blockIdx.x;
  P::load_twiddles(TW, tw);
  __syncthreads();
  const C* s = src + (size_t)p * src_stride;
  C* sp = P::inverse(B0, B1, TW, [&](int r, int c) { return s[r * Wh + c]; });
  const R sc = R((scale ? scale[p] : 1.0) / (double)D);
  DST* o = dst + (size_t)p * dst_stride;
  for (int it = threadIdx.x; it < H * M; it += T) {
    const int r = it / M, m = it % M;
    const C v = sp[r * Wh + m];
    if constexpr (std::is_same<DST, R>::value) {
      reinterpret_cast<C*>(o)[it] = mk<C>(v.x * sc, v.y * sc);
    } else {
      o[r * W + 2 * m] = DST(v.x * sc);
      o[r * W + 2 * m + 1] = DST(v.y * sc);
    }
  }
}

// ----------------------------------------------------------------------------
// Learning: the support-mask step of LearningOperator::apply
// (learning.cpp:96-107): p_hat_k = DFT(mask . iDFT(c_k)), and the crop of
// d_recover (learning.cpp:205-214): d_k = -0.5/max(mu_k,1e-300) crop(iDFT(c_k)).
// mode 0: mask -> p_hat (NSL); mode 1: crop -> d_out (K x mh x mw, double).
// ----------------------------------------------------------------------------
template <class P>
__global__ void __launch_bounds__(P::T)
mask_step(const cx<typename P::R>* __restrict__ c, cx<typename P::R>* __restrict__ phat,
          double* __restrict__ d_out, const int* live, const double* mu, int mh, int mw, int mode,
          const cx<typename P::R>* tw, const int* done) {
  if (done && *done) return;
  using R = typename P::R;
  using C = typename P::C;
  constexpr int H = P::H, Wh = P::Wh, NB = P::NB, T = P::T, D = P::D, M = P::M;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  C* B0 = reinterpret_cast<C*>(smem_raw);
  C* B1 = B0 + NB;
  C* TW = B1 + NB;
  C* COL0 = TW + P::TW_LEN;
  const int k = blockIdx.x;
  if (!live[k]) {  // dead filter: skipped by the operator (learning.cpp:96)
    if (mode == 0) {
      for (int i = threadIdx.x; i < NB; i += T) phat[(size_t)k * NB + i] = mk<C>(R(0), R(0));
    } else {
      for (int i = threadIdx.x; i < mh * mw; i += T) d_out[(size_t)k * mh * mw + i] = 0.0;
    }
    return;
  }
  P::load_twiddles(TW, tw);
  __syncthreads();
  const C* s = c + (size_t)k * NB;
  C* sp = P::inverse(B0, B1, TW, [&](int r, int cc) { return s[r * Wh + cc]; });
  const R invD = R(1) / R(D);
  if (mode != 0) {  // 1: d_recover (-0.5/mu scaling), 2: plain cropped correlation
    const double scale = mode == 2 ? 1.0 : -0.5 / fmax(mu[k], 1e-300);
    for (int i = threadIdx.x; i < mh * mw; i += T) {
      const int r = i / mw, cc = i % mw;
      const C v = sp[r * Wh + cc / 2];
      const R val = ((cc & 1) ? v.y : v.x) * invD;
      d_out[(size_t)k * mh * mw + i] = scale * (double)val;
    }
    return;
  }
  for (int it = threadIdx.x; it < H * M; it += T) {
    const int r = it / M, m = it % M;
    const C v = sp[r * Wh + m];
    const bool rin = r < mh;
    const R v0 = (rin && 2 * m < mw) ? v.x * invD : R(0);
    const R v1 = (rin && 2 * m + 1 < mw) ? v.y * invD : R(0);
    sp[r * Wh + m] = mk<C>(v0, v1);
  }
  __syncthreads();
  C* other = (sp == B0) ? B1 : B0;
  forward_to_global<P>(sp, other, TW, COL0, phat + (size_t)k * NB);
}

// Parseval weight of a half-spectrum bin: columns 0 and W/2 are their own
// mirrors (weight 1), every other bin stands for itself and its conjugate.
__device__ __forceinline__ double bin_weight(int b, int Wh) {
  const int c = b % Wh;
  return (c == 0 || c == Wh - 1) ? 1.0 : 2.0;
}

// c_k(w) = sum_n conj(z_hat_nk(w)) v_hat_n(w)   (learning.cpp:97-102, 204-209)
// The image sum is split over gridDim.z chunks (FP64 partials, fixed-order
// second pass in contract_c_reduce) so that N >> 1 still fills the machine.
template <class R, int KC>
__global__ void __launch_bounds__(256)
contract_c(const cx<R>* __restrict__ zhat, const cx<R>* __restrict__ v, double2* __restrict__ cpart,
           const int* __restrict__ live, int N, int K, int NB, const int* done) {
  if (done && *done) return;
  using C = cx<R>;
  // CTA = (bin tile, chunk of KC filters, image chunk); v_hat_n(b) is loaded
  // once per image and reused for the KC filters.
  const int k0 = blockIdx.y * KC;
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= NB) return;
  const int per = (N + gridDim.z - 1) / gridDim.z;
  const int n0 = blockIdx.z * per, n1 = min(N, n0 + per);
  double ar[KC], ai[KC];
#pragma unroll
  for (int q = 0; q < KC; ++q) ar[q] = ai[q] = 0.0;
  const size_t zs = (size_t)K * NB;
  const C* zp = zhat + (size_t)k0 * NB + b;
  const int kn = min(KC, K - k0);
  if (kn == KC) {
#pragma unroll 2
    for (int n = n0; n < n1; ++n) {
      const C x = __ldg(v + (size_t)n * NB + b);
      C z[KC];
#pragma unroll
      for (int q = 0; q < KC; ++q) z[q] = __ldcs(zp + (size_t)n * zs + (size_t)q * NB);
#pragma unroll
      for (int q = 0; q < KC; ++q) {
        ar[q] += (double)z[q].x * (double)x.x + (double)z[q].y * (double)x.y;
        ai[q] += (double)z[q].x * (double)x.y - (double)z[q].y * (double)x.x;
      }
    }
  } else {
    for (int n = n0; n < n1; ++n) {
      const C x = __ldg(v + (size_t)n * NB + b);
#pragma unroll
      for (int q = 0; q < KC; ++q) {
        if (q < kn) {
          const C z = __ldg(zp + (size_t)n * zs + (size_t)q * NB);
          ar[q] += (double)z.x * (double)x.x + (double)z.y * (double)x.y;
          ai[q] += (double)z.x * (double)x.y - (double)z.y * (double)x.x;
        }
      }
    }
  }
#pragma unroll
  for (int q = 0; q < KC; ++q) {
    if (q >= kn) break;
    // dead filters: exactly zero (the operator skips them, learning.cpp:96)
    const bool lv = live[k0 + q] != 0;
    cpart[((size_t)blockIdx.z * K + k0 + q) * NB + b] = make_double2(lv ? ar[q] : 0.0, lv ? ai[q] : 0.0);
  }
}

template <class R>
__global__ void contract_c_reduce(const double2* __restrict__ cpart, cx<R>* __restrict__ c, int splits, size_t KNB,
                                  const int* done) {
  if (done && *done) return;
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= KNB) return;
  double ar = 0.0, ai = 0.0;
  for (int s = 0; s < splits; ++s) {
    const double2 p = cpart[(size_t)s * KNB + i];
    ar += p.x;
    ai += p.y;
  }
  c[i] = mk<cx<R>>(R(ar), R(ai));
}

// frequency-sharded learning: the local-bin correlations (K x NBL) into the
// full K x NBF spectra at bin offset b0 (the other bins stay zero)
template <class R>
__global__ void contract_c_reduce_off(const double2* __restrict__ cpart, cx<R>* __restrict__ c, int splits,
                                      size_t KNBL, const int* done, int NBL, int NBF, int b0) {
  if (done && *done) return;
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= KNBL) return;
  double ar = 0.0, ai = 0.0;
  for (int s = 0; s < splits; ++s) {
    const double2 p = cpart[(size_t)s * KNBL + i];
    ar += p.x;
    ai += p.y;
  }
  const size_t k = i / NBL, b = i % NBL;
  c[k * NBF + b0 + b] = mk<cx<R>>(R(ar), R(ai));
}

// image-major spectra src [planes][NB] -> per-destination blocks for the
// frequency all-to-all: bins [b0_q, b0_q + nbl_q) of every plane go to block q
// (offset planes * b0_q, layout [planes][nbl_q]); b0_q = q NB / world
template <class C>
__global__ void pack_bins(const C* __restrict__ src, C* __restrict__ dst, size_t planes, int NB, int world) {
  const size_t total = planes * (size_t)NB;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    const size_t p = i / NB;
    const int b = (int)(i % NB);
    int q = world - 1;
    while ((long)q * NB / world > b) --q;
    const int b0 = (int)((long)q * NB / world), nbl = (int)((long)(q + 1) * NB / world) - b0;
    dst[planes * (size_t)b0 + p * (size_t)nbl + (b - b0)] = src[i];
  }
}

// single-block fixed-order sum of block partials into out[0]
static __global__ void sum_partials(const double* partial, int count, double* out) {
  __shared__ double red[32];
  double v = 0.0;
  for (int i = threadIdx.x; i < count; i += blockDim.x) v += partial[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < (int)(blockDim.x / 32); ++w) s += red[w];
    out[0] = s;
  }
}

struct CgState {
  double rr, pap, alpha, beta, rel, bnorm, tol;
  int bad, done, iters, max_iters, converged, pad;
};

// Single-block scalar step of CG. step 0: rr from the initial residual (done
// when already below tol); step 1: pap -> alpha (pAp <= 0 stops, gamma
// untouched, learning.cpp:166); step 2: rr_new -> rel, beta, iteration count.
// Run by one whole block (the cg_scalar kernel, or the last block of the
// kernel that produced the partials).
__device__ __forceinline__ void cg_scalar_block(const double* partial, int count, double invD, CgState* st, int step,
                                                const double* presum) {
  __shared__ double red[32];
  if (step != 0 && st->done) return;
  if (presum) count = 0;  // already summed (over ranks)
  double v = 0.0;
  // fixed-order strided partial sums, then a fixed-order tree: deterministic
  for (int i = threadIdx.x; i < count; i += blockDim.x) v += __ldcg(partial + i);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x != 0) return;
  double s = 0.0;
  for (int w = 0; w < (int)(blockDim.x / 32); ++w) s += red[w];
  if (presum) s = presum[0];
  s *= invD;
  if (step == 0) {
    st->rr = s;
    st->rel = sqrt(s) / st->bnorm;
    st->bad = 0;
    st->iters = 0;
    st->converged = st->rel <= st->tol;
    st->done = st->converged;
  } else if (step == 1) {
    st->pap = s;
    if (s <= 0.0) {
      st->bad = 1;
      st->done = 1;
    } else {
      st->alpha = st->rr / s;
    }
  } else {
    st->iters += 1;
    st->rel = sqrt(s) / st->bnorm;
    st->beta = s / st->rr;
    st->rr = s;
    if (st->rel <= st->tol) {
      st->converged = 1;
      st->done = 1;
    } else if (st->iters >= st->max_iters) {
      st->done = 1;
    }
  }
}

// After a block has written its partial: true in the block that arrives last
// (its partial reads then see every block's write). The counter is reset.
__device__ __forceinline__ bool last_block_arrive(unsigned* counter, unsigned total) {
  __shared__ int am_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned prev = atomicAdd(counter, 1u);
    am_last = prev == total - 1;
    if (am_last) *counter = 0;
  }
  __syncthreads();
  if (am_last) __threadfence();
  return am_last != 0;
}

// out_n = v_n + sum_k (0.5/mu_k) z_hat_nk p_hat_k (learning.cpp:109-121, in the
// frequency domain), with the block partial of <v, out> (Parseval, FP64).
// mode 1 (learning data term): y_n = sum_k d_hat_k z_hat_nk, partial of
// |y_n - x_hat_n|^2 weighted, no identity (objective.cpp:83-95).
template <class R, int TB, int NI = 1>
__global__ void __launch_bounds__(TB)
contract_out(const cx<R>* __restrict__ zhat, const cx<R>* __restrict__ p, const double* __restrict__ wk,
             const int* __restrict__ live, const cx<R>* __restrict__ v, cx<R>* __restrict__ out,
             double* __restrict__ partial, int N, int K, int NB, int Wh, int mode, const int* done,
             CgState* cgst = nullptr, unsigned* cnt = nullptr, double invD = 0.0, int b0 = 0, int pstride = 0) {
  // b0 / pstride (frequency-sharded learning): the NB bins are [b0, b0 + NB)
  // of the full half spectrum, p points at bin b0 of K spectra pstride apart
  using C = cx<R>;
  __shared__ double red[TB / 32];
  if (done && *done) return;
  const int b = blockIdx.x * TB + threadIdx.x;
  double dot = 0.0;
  // images n = blockIdx.y, + gridDim.y, ...: one image per block unless the
  // caller (fused CG apply) launches fewer rows to keep the partial count small.
  // NI images per pass share each p_hat load (NI = 2 pays when the p_hat
  // stack is far beyond L1 reuse, C3: 5.89 vs 6.11 s of contractions per outer
  // iteration; at C2/C4 NI = 1 is 3-5% faster). Same accumulation order.
  for (int n = blockIdx.y; n < N; n += NI * gridDim.y) {
  if (b < NB) {
    // Dead filters have identically zero z_hat (and p_hat), so summing them
    // adds exact zeros: no per-filter branch, loads batched 8 deep.
    double ar[NI], ai[NI];
    const C* zp[NI];
    bool ok[NI];
#pragma unroll
    for (int i = 0; i < NI; ++i) {
      const int ni = n + i * gridDim.y;
      ok[i] = ni < N;
      zp[i] = zhat + (size_t)(ok[i] ? ni : n) * K * NB + b;
      ar[i] = ai[i] = 0.0;
    }
    const C* pp = p + b;
    const size_t PS = pstride ? (size_t)pstride : (size_t)NB;
    constexpr int U = 8;
    int k = 0;
    for (; k + U <= K; k += U) {
      C z[NI][U], q[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
#pragma unroll
        for (int i = 0; i < NI; ++i) z[i][u] = __ldcs(zp[i] + (size_t)(k + u) * NB);  // streaming: keep p_hat in L2
        q[u] = __ldg(pp + (size_t)(k + u) * PS);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const double w = mode == 0 ? wk[k + u] : 1.0;
#pragma unroll
        for (int i = 0; i < NI; ++i) {
          ar[i] += w * ((double)z[i][u].x * (double)q[u].x - (double)z[i][u].y * (double)q[u].y);
          ai[i] += w * ((double)z[i][u].x * (double)q[u].y + (double)z[i][u].y * (double)q[u].x);
        }
      }
    }
    for (; k < K; ++k) {
      const C q = __ldg(pp + (size_t)k * PS);
      const double w = mode == 0 ? wk[k] : 1.0;
#pragma unroll
      for (int i = 0; i < NI; ++i) {
        const C z = __ldcs(zp[i] + (size_t)k * NB);
        ar[i] += w * ((double)z.x * (double)q.x - (double)z.y * (double)q.y);
        ai[i] += w * ((double)z.x * (double)q.y + (double)z.y * (double)q.x);
      }
    }
    (void)live;
#pragma unroll
    for (int i = 0; i < NI; ++i) {
      if (!ok[i]) continue;
      const size_t o_n = (size_t)(n + i * gridDim.y) * NB + b;
      const C vv = v[o_n];
      if (mode == 0) {
        const C o = mk<C>(R((double)vv.x + ar[i]), R((double)vv.y + ai[i]));
        out[o_n] = o;
        dot += bin_weight(b0 + b, Wh) * ((double)vv.x * (double)o.x + (double)vv.y * (double)o.y);
      } else {
        const double rr = ar[i] - (double)vv.x, ri = ai[i] - (double)vv.y;
        dot += bin_weight(b0 + b, Wh) * (rr * rr + ri * ri);
      }
    }
  }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = dot;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < TB / 32; ++w) s += red[w];
    partial[(size_t)blockIdx.y * gridDim.x + blockIdx.x] = s;
  }
  // single-rank CG: the last block turns the <p, Ap> partials into alpha
  if (cgst && last_block_arrive(cnt, gridDim.x * gridDim.y))
    cg_scalar_block(partial, gridDim.x * gridDim.y, invD, cgst, 1, nullptr);
}

// ----------------------------------------------------------------------------
// CG vector kernels on half spectra (gamma_solve, learning.cpp:136-185).
// Dot products are spatial via Parseval: <a,b> = (1/D) sum_bins wt Re(conj(a) b).
// ----------------------------------------------------------------------------
template <int TB>
__device__ __forceinline__ void block_partial(double v, double* out_slot) {
  __shared__ double red[TB / 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < TB / 32; ++w) s += red[w];
    *out_slot = s;
  }
}

// r = -x_hat - ap ; p = r ; partial of rr
template <class R, int TB>
__global__ void __launch_bounds__(TB)
cg_init(const cx<R>* __restrict__ xhat, const cx<R>* __restrict__ ap, cx<R>* __restrict__ r,
        cx<R>* __restrict__ p, double* partial, size_t total, int NB, int Wh, int b0 = 0) {
  using C = cx<R>;
  const size_t i = (size_t)blockIdx.x * TB + threadIdx.x;
  double v = 0.0;
  if (i < total) {
    const C x = xhat[i], a = ap[i];
    const C rv = mk<C>(-x.x - a.x, -x.y - a.y);
    r[i] = rv;
    p[i] = rv;
    v = bin_weight(b0 + (int)(i % (size_t)NB), Wh) * ((double)rv.x * rv.x + (double)rv.y * rv.y);
  }
  block_partial<TB>(v, partial + blockIdx.x);
}

// Device-resident CG scalars. `done` stops every CG kernel (device-side loop
// termination): set when the relative residual reaches tol, when pAp <= 0
// (learning.cpp:166) or when the budget is spent.

// gamma += alpha p ; r -= alpha ap ; partial of rr_new
template <class R, int TB>
__global__ void __launch_bounds__(TB)
cg_update(cx<R>* __restrict__ gam, cx<R>* __restrict__ r, const cx<R>* __restrict__ p,
          const cx<R>* __restrict__ ap, CgState* st, double* partial, size_t total, int NB,
          int Wh, unsigned* cnt = nullptr, double invD = 0.0, int b0 = 0) {
  using C = cx<R>;
  if (st->done) return;
  double v = 0.0;
  const double al = st->alpha;
  for (size_t i = (size_t)blockIdx.x * TB + threadIdx.x; i < total; i += (size_t)gridDim.x * TB) {
    const C pv = p[i], av = ap[i], gv = gam[i], rv0 = r[i];
    gam[i] = mk<C>(R(gv.x + al * pv.x), R(gv.y + al * pv.y));
    const C rv = mk<C>(R(rv0.x - al * av.x), R(rv0.y - al * av.y));
    r[i] = rv;
    v += bin_weight(b0 + (int)(i % (size_t)NB), Wh) * ((double)rv.x * rv.x + (double)rv.y * rv.y);
  }
  block_partial<TB>(v, partial + blockIdx.x);
  // single-rank CG: the last block turns the rr partials into beta / stop
  if (cnt && last_block_arrive(cnt, gridDim.x)) cg_scalar_block(partial, gridDim.x, invD, st, 2, nullptr);
}

// p = r + beta p
template <class R, int TB>
__global__ void __launch_bounds__(TB)
cg_pupdate(const cx<R>* __restrict__ r, cx<R>* __restrict__ p, const CgState* st, size_t total) {
  using C = cx<R>;
  const size_t i = (size_t)blockIdx.x * TB + threadIdx.x;
  if (i >= total || st->done) return;
  const double be = st->beta;
  const C rv = r[i], pv = p[i];
  p[i] = mk<C>(R(rv.x + be * pv.x), R(rv.y + be * pv.y));
}

static __global__ void cg_scalar(const double* partial, int count, double invD, CgState* st, int step,
                          const double* presum) {
  cg_scalar_block(partial, count, invD, st, step, presum);
}

// Per-image sum of block partials (learning data term / objective), out[n] = 0.5*invD*sum.
static __global__ void per_image_reduce(const double* partial, int tiles, double scale, double* out) {
  __shared__ double red[32];
  const int n = blockIdx.x;
  double v = 0.0;
  for (int i = threadIdx.x; i < tiles; i += blockDim.x) v += partial[(size_t)n * tiles + i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < (int)(blockDim.x / 32); ++w) s += red[w];
    out[n] = scale * s;
  }
}

// Coding objective: data_n = 1/2 ||sum_k d_k * z_k - x||^2 by Parseval on the
// reduced partial spectra; l1_n = beta * sum |z| (objective.cpp:59-81).
template <class R>
__global__ void objective_reduce(const cx<R>* __restrict__ part, const double* __restrict__ sums,
                                 const cx<R>* __restrict__ xhat, int G, int slots, int NB, int Wh, double invD,
                                 double beta, double* data, double* l1) {
  using C = cx<R>;
  __shared__ double red[32];
  const int n = blockIdx.x;
  double v = 0.0;
  for (int b = threadIdx.x; b < NB; b += blockDim.x) {
    C acc = part[((size_t)n * G) * NB + b];
    for (int g = 1; g < G; ++g) acc = cadd(acc, part[((size_t)n * G + g) * NB + b]);
    const C x = xhat[(size_t)n * NB + b];
    const double rr = (double)acc.x - (double)x.x, ri = (double)acc.y - (double)x.y;
    v += bin_weight(b, Wh) * (rr * rr + ri * ri);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < (int)(blockDim.x / 32); ++w) s += red[w];
    data[n] = 0.5 * invD * s;
    double a = 0.0;
    for (int g = 0; g < slots; ++g) a += sums[((size_t)n * slots + g) * kSums];
    l1[n] = beta * a;
  }
}

// ADMM exit (coding.cpp:287-309): lambda = iDFT(lambda_hat) (done by c2r into
// `lam`), rescale by beta/max|t| when infeasible, dual objective. One CTA/image.
template <class R>
__global__ void admm_exit(R* __restrict__ lam, const R* __restrict__ x, const ImageAdmm* img,
                          int D, double beta, double* dual_obj, double* infeas, int* rescaled) {
  __shared__ double red[64];
  const int n = blockIdx.x;
  const double tinf = img[n].tinf;
  const bool resc = tinf > beta;
  const R scale = resc ? R(beta / tinf) : R(1);
  double a = 0.0, b = 0.0;
  R* l = lam + (size_t)n * D;
  const R* xv = x + (size_t)n * D;
  for (int i = threadIdx.x; i < D; i += blockDim.x) {
    R v = l[i];
    if (resc) {
      v *= scale;
      l[i] = v;
    }
    a += (double)v * (double)v;
    b += (double)v * (double)xv[i];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
  }
  if ((threadIdx.x & 31) == 0) {
    red[threadIdx.x >> 5] = a;
    red[32 + (threadIdx.x >> 5)] = b;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double sa = 0.0, sb = 0.0;
    for (int w = 0; w < (int)(blockDim.x / 32); ++w) {
      sa += red[w];
      sb += red[32 + w];
    }
    dual_obj[n] = -0.5 * sa - sb;
    infeas[n] = fmax(0.0, tinf - beta);
    rescaled[n] = resc ? 1 : 0;
  }
}

// sigma(w) = sum_k |d_hat_k(w)|^2 + 1/rho  (coding.cpp:15-21), FP64 accumulation
template <class R>
__global__ void sigma_kernel(const cx<R>* __restrict__ dhat, R* __restrict__ sigma, int K, int NB,
                             double rho) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= NB) return;
  double s = 1.0 / rho;
  for (int k = 0; k < K; ++k) {
    const cx<R> d = dhat[(size_t)k * NB + b];
    s += (double)d.x * d.x + (double)d.y * d.y;
  }
  sigma[b] = R(s);
}

// Accept coded maps (pipeline.cpp:236-246): for accepted images maps = z_cand
// (closed form from u); block partials of sum (cand-old)^2 over accepted images,
// sum maps^2 and the l0 count over all images. grid (chunks, N).
template <class R, int TB, bool UT>
__global__ void __launch_bounds__(TB)
accept_maps(const R* __restrict__ u, R* __restrict__ maps, const int* __restrict__ accept,
            size_t per_image, double rho, double beta, double* part_dz, double* part_zz,
            unsigned long long* l0, int H, int W) {
  const int n = blockIdx.y;
  const bool acc = accept[n] != 0;
  double dz = 0.0, zz = 0.0;
  unsigned long long cnt = 0;
  const R rr = R(rho), bb = R(beta);
  const R* up = u + (size_t)n * per_image;
  R* mp = maps + (size_t)n * per_image;
  for (size_t i = (size_t)blockIdx.x * TB + threadIdx.x; i < per_image; i += (size_t)gridDim.x * TB) {
    R m = mp[i];
    if (acc) {
      size_t ui = i;
      if (UT) {  // u planes are column-major pixel pairs: (r, c) -> ((c/2) H + r) * 2 + (c & 1)
        const size_t D = (size_t)H * W, p = i / D, q = i % D;
        const int r = (int)(q / W), c = (int)(q % W);
        ui = p * D + ((size_t)(c >> 1) * H + r) * 2 + (c & 1);
      }
      const R uv = up[ui];
      const R zc = rr * (fmin(fmax(uv, -bb), bb) - uv);
      const double d = (double)zc - (double)m;
      dz += d * d;
      m = zc;
      mp[i] = m;
    }
    zz += (double)m * (double)m;
    cnt += (m != R(0));
  }
  __shared__ double red[2][TB / 32];
  __shared__ unsigned long long redc[TB / 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    dz += __shfl_xor_sync(0xffffffffu, dz, o);
    zz += __shfl_xor_sync(0xffffffffu, zz, o);
    cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  }
  if ((threadIdx.x & 31) == 0) {
    red[0][threadIdx.x >> 5] = dz;
    red[1][threadIdx.x >> 5] = zz;
    redc[threadIdx.x >> 5] = cnt;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, b = 0.0;
    unsigned long long c = 0;
    for (int w = 0; w < TB / 32; ++w) {
      a += red[0][w];
      b += red[1][w];
      c += redc[w];
    }
    const size_t slot = (size_t)n * gridDim.x + blockIdx.x;
    part_dz[slot] = a;
    part_zz[slot] = b;
    l0[slot] = c;
  }
}

// lambda = -x for the degenerate (all-zero) dictionary (coding.cpp:181-191)
template <class R>
__global__ void neg_copy(const R* __restrict__ x, R* __restrict__ lam, size_t total) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < total) lam[i] = -x[i];
}

template <class R>
__global__ void to_real(const double* __restrict__ src, R* __restrict__ dst, size_t total) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < total) dst[i] = R(src[i]);
}

}  // namespace dcsc_cuda
