// Cluster (multi-CTA per plane) variants of the hot-path kernels for planes
// whose half spectrum exceeds one CTA's shared memory (C3: 256 x 256 FP32).
// Same algorithms and reference anchors as kernels.cuh; the FFT work of one
// plane is split over a CP::CL-CTA cluster (fft2d_cluster.cuh), the two
// transposes per plane are TMA bulk block exchanges between the CTAs' shared
// memories (cl_issue_exchange).
//
// Buffers (3 x [BUF] complex per CTA): X, Y, Z. One plane round trip:
//   cols_inv      gen -> X -> Y            (Y = send blocks of exchange I)
//   exchange I    Y -> peers' Z            (Z = [CL src][ROWS][CS])
//   rows_inv      Z -> X -> Z              (Z = spatial rows)
//   prox / load   Z in place
//   rows_fwd      Z -> X -> Z (send layout; exchange F)
//   exchange F    Z -> peers' Y            (Y = [H][CS] column buffer)
//   cols_fwd      Y -> X -> consumer
#pragma once
#include "fft2d_cluster.cuh"
#include "kernels.cuh"

namespace dcsc_cuda {

#ifdef DCSC_CL_TRACE
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define CLT(slot) \
  if (threadIdx.x == 0 && blockIdx.y == 0 && blockIdx.x < CL && k >= k0 + 2 && k < k0 + 5) tt[k - k0 - 2][slot] = gtimer();
#else
#define CLT(slot)
#endif

template <class CP>
struct SmemCl {
  using C = typename CP::C;
  static constexpr size_t bufs = 3 * CP::buffer_bytes;
  static constexpr size_t tw_off = bufs;
  static constexpr size_t col0_off = tw_off + sizeof(C) * CP::TW_LEN;
  static constexpr size_t plain = col0_off + sizeof(C) * CP::H;
  // coding pass: lambda_hat columns 0 and W/2 of the CTA's image (rank 0
  // pre-packs its generator column from them) and a column of ones
  static constexpr size_t lamc_off = plain;
  static constexpr size_t coding = lamc_off + 2 * sizeof(C) * CP::H;
};

// The split cluster barriers only guard buffer reuse (write-after-read): all
// data moves by TMA pushes completed on the receiver's mbarrier, and the
// reads a rank retires before arriving have been consumed by then. So the
// arrive needs no release fence (relaxed; the MEMBAR it implied cost ~5% of a
// 256x256 coding pass). Build with -DDCSC_CL_ARRIVE_RELAXED=0 for release.
#ifndef DCSC_CL_ARRIVE_RELAXED
#define DCSC_CL_ARRIVE_RELAXED 1
#endif
__device__ __forceinline__ void cluster_arrive() {
#if DCSC_CL_ARRIVE_RELAXED
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
#else
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
#endif
}
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }
__device__ __forceinline__ void fence_mbar_init_cluster() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// Bulk copy of `bytes` from this CTA's smem to the same-offset address `dst`
// in peer CTA `peer`; completion is counted on the peer's mbarrier `bar`.
__device__ __forceinline__ void bulk_s2peer(void* dst, unsigned peer, const void* src, unsigned bytes,
                                            unsigned long long* bar) {
  unsigned d, b;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(d) : "r"(smem_addr(dst)), "r"(peer));
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(b) : "r"(smem_addr(bar)), "r"(peer));
  asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   d),
               "r"(smem_addr(src)), "r"(bytes), "r"(b)
               : "memory");
}

// Block q of snd -> slot `rank` of peer q's stg (one bulk copy per peer; the
// rank's own block is not copied, consumers read it from snd). The caller has made snd visible to the async proxy
// (fence_async_smem + __syncthreads) and knows every peer's stg is free.
template <class CP>
__device__ __forceinline__ void cl_issue_exchange(const typename CP::C* snd, typename CP::C* stg, unsigned rank,
                                                  unsigned long long* bar) {
  if (threadIdx.x == 0) mbar_expect_tx(bar, (CP::CL - 1) * CP::block_bytes);
  if (threadIdx.x < CP::CL && threadIdx.x != rank) {
    const unsigned q = threadIdx.x;
    bulk_s2peer(stg + rank * CP::BLOCK, q, snd + q * CP::BLOCK, CP::block_bytes, bar);
  }
}

// Fully synchronised exchange (single-plane helper kernels).
template <class CP>
__device__ __forceinline__ void cl_exchange_sync(const typename CP::C* snd, typename CP::C* stg, unsigned rank,
                                                 unsigned long long* bar, unsigned& phase) {
  fence_async_smem();
  __syncthreads();
  cluster_sync_all();  // every rank: send blocks written, staging free
  cl_issue_exchange<CP>(snd, stg, rank, bar);
  mbar_wait(bar, phase);
  phase ^= 1u;
  cluster_sync_all();  // every block delivered: send buffers reusable
}

template <class CP>
__device__ __forceinline__ void cl_init_exchange(unsigned long long* bar) {
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_mbar_init_cluster();
  }
  __syncthreads();
}

// The fused coding kernel (see coding_pass in kernels.cuh) with each plane's
// FFTs split over a cluster: rank c owns rows [c*ROWS, ...) of u / w and
// columns col_of(c, .) of the spectra. blockIdx.x = group * CL + rank.
// Cluster barrier phases are split (arrive early, wait late): B_I (after the
// staged blocks of exchange I are consumed) is awaited before exchange F is
// issued, B_F (after exchange F's blocks are consumed) before the next
// filter's exchange I / plane load — two barriers per filter, each with a
// pass of slack.
// d_hat (K x NB) -> rank-blocked copy K x CL x [H][CS]: slot cl < COLS holds
// column col_of(c, cl) of rank c, slot COLS column W/2 (rank 0's packed pair
// partner; zero elsewhere). Built once per dictionary (set_dictionary).
template <class CP>
__global__ void cl_rank_block(const cx<typename CP::R>* __restrict__ dhat, cx<typename CP::R>* __restrict__ out,
                              int K) {
  using C = typename CP::C;
  constexpr int H = CP::H, CS = CP::CS, COLS = CP::COLS, CL = CP::CL, Wh = CP::Wh, M = CP::M, NB = CP::NB;
  constexpr int RB = (int)(CP::buffer_bytes / sizeof(C));  // slice stride = the smem buffer stride
  static_assert(CP::BUF == H * CS, "rank block = one column buffer");
  const size_t total = (size_t)K * CL * RB;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    const int e = (int)(i % RB);
    const int c = (int)((i / RB) % CL);
    const size_t k = i / ((size_t)RB * CL);
    const int r = e / CS, cl = e % CS;
    C v = mk<C>(typename CP::R(0), typename CP::R(0));
    if (e >= H * CS) {
      // padding to the buffer stride
    } else if (cl < COLS)
      v = dhat[k * NB + r * Wh + CP::col_of((unsigned)c, cl)];
    else if (c == 0)
      v = dhat[k * NB + r * Wh + M];
    out[i] = v;
  }
}

#ifndef DCSC_CL_PROX_UNROLL
#define DCSC_CL_PROX_UNROLL 16
#endif
constexpr int kClProxUnroll = DCSC_CL_PROX_UNROLL;  // u loads in flight per thread in the prox loop

// TC (multi-channel, J > 1, the reference's Joint mode, tcsc.cpp:101-171): the
// generator forms t_hat_k = sum_j conj(d_hat_jk) lambda_hat_j from L2, and the
// last forward column stage stores w_hat_k (z_hat_k in the objective / maps
// passes) to a.what instead of accumulating; tc_lambda / tc_objective do the
// per-bin J x J work (tcsc_kernels.cuh).
template <class CP, int MODE, bool TC = false>
__global__ void __cluster_dims__(CP::CL, 1, 1) __launch_bounds__(CP::T)
    coding_pass_cl(CodingArgs<typename CP::R> a) {
  using R = typename CP::R;
  using C = typename CP::C;
  using SM = SmemCl<CP>;
  constexpr int H = CP::H, M = CP::M, Wh = CP::Wh, NB = CP::NB, D = CP::D, T = CP::T, CL = CP::CL;
  constexpr int ROWS = CP::ROWS, COLS = CP::COLS, CS = CP::CS;
  constexpr int BS = CP::buffer_bytes / sizeof(C);
  static_assert(BS >= CP::BUF, "rank-blocked d_hat stride (cl_rank_block) = buffer stride");
  constexpr bool ADMM = MODE == kPassAdmm;
  using S = Split<typename CP::ColPlan>;
  static_assert(CountStages<typename CP::ColPlan>::value == 2, "two-stage column plan (X -> Y)");
  static_assert(CountStages<typename CP::RowPlan>::value == 2, "two-stage row plan (Z -> X -> Z)");

  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ double red[kSums * (T / 32)];
  __shared__ __align__(8) unsigned long long xbar_s;
  C* X = reinterpret_cast<C*>(smem_raw);
  C* Y = X + BS;
  C* Z = Y + BS;
  C* TW = reinterpret_cast<C*>(smem_raw + SM::tw_off);
  C* COL0 = reinterpret_cast<C*>(smem_raw + SM::col0_off);
  unsigned long long* xbar = &xbar_s;
  unsigned xphase = 0;
  const unsigned rank = cluster_rank();
  const int g = blockIdx.x / CL, n = blockIdx.y;
  const int r0 = rank * ROWS;
  if (ADMM && a.conv[n]) return;  // the whole cluster sees the same flag

  CP::load_twiddles(TW, a.tw);
  // The generator's d_hat slice of each filter is staged by one TMA copy into
  // Y (rank-blocked layout) while the previous filter's last stage runs; Y is
  // free then (exchange F's blocks consumed) and no peer writes it before this
  // rank's own next-filter exchange (B_I). Only lambda_hat is read from L2.
  __shared__ __align__(8) unsigned long long dbar_s;
  unsigned long long* dbar = &dbar_s;
  unsigned dphase = 0;
  const bool DST = ADMM && !TC && a.dhat_rb != nullptr;
  const int k0s = (int)(blockIdx.x / CL) * a.kpg;
  // rank 0's packed generator column P(r) = t(r, 0) + i t(r, W/2), t = conj(d) lambda:
  // rank 0 pre-packs conj(P) into the staged d_hat slot 0 per filter, and the
  // generator multiplies it by a lambda of ones, so no lane issues partner loads
  C* LAMC = reinterpret_cast<C*>(smem_raw + SM::lamc_off);
  if (DST && rank == 0 && threadIdx.x < H) {
    const C* lamn = a.lamhat + (size_t)n * NB;
    LAMC[threadIdx.x] = lamn[threadIdx.x * Wh];
    LAMC[H + threadIdx.x] = lamn[threadIdx.x * Wh + M];
  }
  if (DST && threadIdx.x == 0) mbar_init(dbar, 1);
  cl_init_exchange<CP>(xbar);  // (fences the mbarrier inits, syncs the CTA)
  if (DST && threadIdx.x == 0 && k0s < a.K) {
    mbar_expect_tx(dbar, (unsigned)(sizeof(C) * BS));
    bulk_g2s(Y, a.dhat_rb + ((size_t)k0s * CL + rank) * BS, (unsigned)(sizeof(C) * BS), dbar);
  }
  cluster_arrive();  // matched by the wait before the first filter's exchange

  constexpr int RL = S::last, JL = H / RL, ITEMS_L = COLS * JL;
  static_assert(ITEMS_L <= T, "one last-stage item per thread");
  C acc[RL];
#pragma unroll
  for (int s = 0; s < RL; ++s) acc[s] = mk<C>(R(0), R(0));
  C acc0 = mk<C>(R(0), R(0)), accN = mk<C>(R(0), R(0));

  const R rho = a.rho, beta = a.beta, invD = R(1) / R(D);
  // non-ADMM passes: the l1 sum in s0; ADMM: the seven stop-test sums are
  // reduced per filter over each warp (FP32 shuffles over 32 lanes x 32 terms)
  // and accumulated in FP64 per warp in shared memory, so no FP64 running sums
  // occupy registers across the filter loop (they spilled)
  double s0 = 0, s1 = 0, s2 = 0, s3 = 0, s4 = 0, s5 = 0, s6 = 0;
  __shared__ double wsum[T / 32][8];
  if (ADMM && threadIdx.x < (T / 32) * 8) (&wsum[0][0])[threadIdx.x] = 0.0;
  const int k0 = g * a.kpg;
  const int k1 = min(a.K, k0 + a.kpg);
#ifdef DCSC_CL_TRACE
  unsigned long long tt[3][14] = {};
#endif
  for (int k = k0; k < k1; ++k) {
#ifdef DCSC_CL_TRACE
    if (threadIdx.x == 0 && blockIdx.y == 0 && blockIdx.x < CL && k >= k0 + 2 && k < k0 + 5) tt[k - k0 - 2][6] = gtimer();
#endif
    const C* __restrict__ dk = a.dhat + (size_t)k * NB;
    if constexpr (ADMM) {
      C* __restrict__ uk = reinterpret_cast<C*>(a.u + ((size_t)n * a.K + k) * D) + (size_t)r0 * M;
      const C* __restrict__ t0k =
          a.theta0 ? reinterpret_cast<const C*>(a.theta0 + ((size_t)n * a.K + k) * D) + (size_t)r0 * M : nullptr;
      const C* __restrict__ lam = a.lamhat + (size_t)n * NB;
      if (threadIdx.x == 0) {
        prefetch_l2_bulk(uk, sizeof(C) * ROWS * M);
        if (k + 1 < k1) prefetch_l2_bulk(dk + NB, sizeof(C) * NB);
      }
      if (DST) {
        mbar_wait(dbar, dphase);
        dphase ^= 1u;
        CLT(12)
        if (rank == 0) {
          for (int r = threadIdx.x; r < H; r += T) {  // one row per thread
            const C p0 = cmulc(Y[r * CS], LAMC[r]), pm = cmulc(Y[r * CS + COLS], LAMC[H + r]);
            Y[r * CS] = cconj(CP::pack_col0(p0, pm));
          }
          __syncthreads();
        }
        const C one = mk<C>(R(1), R(0));
        CP::cols_inv_gen_prepacked(X, rank, [&](int r, int c) {
          unsigned cr;
          int cl;
          CP::owner_of(c, cr, cl);
          // c = 0 (rank 0): slot 0 holds conj(P) and multiplies 1
          const C lv = c == 0 ? one : __ldg(lam + r * Wh + c);
          return cmulc(Y[r * CS + cl], lv);
        });
        CLT(13)
        CP::cols_inv_rest(X, Y, TW);
      } else if constexpr (TC) {
        const int J = a.J;
        CP::cols_inv(X, Y, TW, rank, [&](int r, int c) {
          const int b = r * Wh + c;
          C t = mk<C>(R(0), R(0));
          for (int j = 0; j < J; ++j)
            t = cadd(t, cmulc(__ldg(a.dhat + ((size_t)j * a.K + k) * NB + b),
                              __ldg(a.lamhat + ((size_t)n * J + j) * NB + b)));
          return t;
        });
      } else {
        CP::cols_inv(X, Y, TW, rank, [&](int r, int c) {
          const int b = r * Wh + c;
          return cmulc(__ldg(dk + b), __ldg(lam + b));
        });
      }
      fence_async_smem();
      __syncthreads();
      CLT(0)
      cluster_wait();  // B_F (previous filter): peers' Z free
      CLT(1)
      cl_issue_exchange<CP>(Y, Z, rank, xbar);
      mbar_wait(xbar, xphase);
      CLT(2)
      xphase ^= 1u;
      CP::rows_inv_first(Z, Y, rank, X, TW);
      __syncthreads();
      CLT(7)
      cluster_arrive();  // B_I: my Z consumed, my incoming blocks complete
      CP::rows_inv_rest(X, Z, TW);
      CLT(8)
      R f0 = 0, f1 = 0, f2 = 0, f3 = 0, f4 = 0, f5 = 0, f6 = 0;
      auto prox_elem = [&](const R t, const R u_old, const R t0e, R& w_out, R& u_out) {
        const R th_o = t0k ? t0e : fmin(fmax(u_old, -beta), beta);
        const R un = t - (th_o - u_old);
        const R th = fmin(fmax(un, -beta), beta);
        const R zn = rho * (th - un);
        const R d_tt = th - t;
        const R dz = rho * d_tt;
        const R dth = th - th_o;
        f0 += d_tt * d_tt;
        f1 += th * th;
        f2 += t * t;
        f3 += dz * dz;
        f4 += zn * zn;
        f5 += dth * dth;
        f6 = fmax(f6, fabs(t));
        w_out = R(2) * th - un;
        u_out = un;
      };
      if constexpr (sizeof(R) == 4) {
        // FP32: two pixel pairs per item, u as 16-byte vectors (half the LDG /
        // STG instructions of the 8-byte form)
        float4* __restrict__ uk4 = reinterpret_cast<float4*>(uk);
        const float4* __restrict__ t0k4 = reinterpret_cast<const float4*>(t0k);
#pragma unroll 8
        for (int it = threadIdx.x; it < ROWS * M / 2; it += T) {
          const int rl = (2 * it) / M, m = (2 * it) % M;
          const float4 u4 = __ldcs(uk4 + it);  // u streams through once: evict-first (keeps d_hat, lambda_hat in L2)
          float4 t04 = make_float4(0.f, 0.f, 0.f, 0.f);
          if (t0k) t04 = __ldg(t0k4 + it);
          const C va = Z[rl * Wh + m], vb = Z[rl * Wh + m + 1];
          float4 o4;
          C wa, wb;
          prox_elem(va.x * invD, u4.x, t04.x, wa.x, o4.x);
          prox_elem(va.y * invD, u4.y, t04.y, wa.y, o4.y);
          prox_elem(vb.x * invD, u4.z, t04.z, wb.x, o4.z);
          prox_elem(vb.y * invD, u4.w, t04.w, wb.y, o4.w);
          __stcs(uk4 + it, o4);
          Z[rl * Wh + m] = wa;
          Z[rl * Wh + m + 1] = wb;
        }
      } else {
#pragma unroll kClProxUnroll
        for (int it = threadIdx.x; it < ROWS * M; it += T) {
          const int rl = it / M, m = it % M;
          const C uv = __ldcs(uk + it);
          C t0v = mk<C>(R(0), R(0));
          if (t0k) t0v = __ldg(t0k + it);
          const C v = Z[rl * Wh + m];
          C w, un;
          prox_elem(v.x * invD, uv.x, t0v.x, w.x, un.x);
          prox_elem(v.y * invD, uv.y, t0v.y, w.y, un.y);
          __stcs(uk + it, un);
          Z[rl * Wh + m] = w;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        f0 += __shfl_xor_sync(0xffffffffu, f0, o);
        f1 += __shfl_xor_sync(0xffffffffu, f1, o);
        f2 += __shfl_xor_sync(0xffffffffu, f2, o);
        f3 += __shfl_xor_sync(0xffffffffu, f3, o);
        f4 += __shfl_xor_sync(0xffffffffu, f4, o);
        f5 += __shfl_xor_sync(0xffffffffu, f5, o);
        f6 = fmax(f6, __shfl_xor_sync(0xffffffffu, f6, o));
      }
      if ((threadIdx.x & 31) == 0) {
        double* ws = wsum[threadIdx.x >> 5];
        ws[0] += (double)f0; ws[1] += (double)f1; ws[2] += (double)f2; ws[3] += (double)f3;
        ws[4] += (double)f4; ws[5] += (double)f5; ws[6] = fmax(ws[6], (double)f6);
      }
      __syncthreads();
      CLT(9)
    } else {
      const C* __restrict__ src = reinterpret_cast<const C*>(
          (MODE == kPassMaps) ? a.maps + ((size_t)n * a.K + k) * D : a.u + ((size_t)n * a.K + k) * D) +
          (size_t)r0 * M;
      const C* __restrict__ t0k = (MODE == kPassPrologue && a.theta0)
                                      ? reinterpret_cast<const C*>(a.theta0 + ((size_t)n * a.K + k) * D) + (size_t)r0 * M
                                      : nullptr;
      cluster_wait();  // B_F (previous filter): my Z no longer read by peers' copies
      for (int it = threadIdx.x; it < ROWS * M; it += T) {
        const int rl = it / M, m = it % M;
        const C v = src[it];
        R w0, w1;
        if constexpr (MODE == kPassPrologue) {
          // w = theta + z/rho = 2 theta - u (theta = clamp(u) for an ADMM-produced state)
          const C th = t0k ? t0k[it] : mk<C>(fmin(fmax(v.x, -beta), beta), fmin(fmax(v.y, -beta), beta));
          w0 = R(2) * th.x - v.x;
          w1 = R(2) * th.y - v.y;
        } else if constexpr (MODE == kPassObjective) {
          w0 = rho * (fmin(fmax(v.x, -beta), beta) - v.x);
          w1 = rho * (fmin(fmax(v.y, -beta), beta) - v.y);
          s0 += (double)fabs(w0) + (double)fabs(w1);
        } else {
          w0 = v.x;
          w1 = v.y;
          s0 += (double)fabs(w0) + (double)fabs(w1);
        }
        Z[rl * Wh + m] = mk<C>(w0, w1);
      }
      __syncthreads();
    }
    // forward: local rows into the send layout, exchange F, column pass
    CP::rows_fwd_to_send(Z, X, Z, TW);
    fence_async_smem();
    __syncthreads();
    CLT(3)
    if constexpr (ADMM) cluster_wait();  // B_I: peers' Y free (else covered by the wait at the filter start)
    CLT(4)
    cl_issue_exchange<CP>(Z, Y, rank, xbar);
    mbar_wait(xbar, xphase);
    CLT(5)
    xphase ^= 1u;
    CP::cols_fwd_first(Y, Z, X, TW, rank);
    __syncthreads();
    CLT(10)
    cluster_arrive();  // B_F: my Y consumed, my incoming blocks complete
    if (DST && threadIdx.x == 0 && k + 1 < k1) {  // next filter's d_hat slice -> Y
      fence_async_smem();
      mbar_expect_tx(dbar, (unsigned)(sizeof(C) * BS));
      bulk_g2s(Y, a.dhat_rb + ((size_t)(k + 1) * CL + rank) * BS, (unsigned)(sizeof(C) * BS), dbar);
    }
    // column-0 epilogue operands (rank 0) fetched with the last stage's loads,
    // so rank 0 does not trail its peers by an L2 round trip every filter
    C d0 = mk<C>(R(0), R(0)), dMv = mk<C>(R(0), R(0));
    if (!TC && rank == 0 && threadIdx.x < H) {
      d0 = __ldg(dk + threadIdx.x * Wh);
      dMv = __ldg(dk + threadIdx.x * Wh + M);
    }
    C* const wk = TC ? a.what + ((size_t)n * a.K + k) * NB : nullptr;
    {
      const C* twc = TW + CP::TW_COL;
      const int it = threadIdx.x;
      if (it < ITEMS_L) {
        const int cl = it % COLS, j = it / COLS;
        const int col = CP::col_of(rank, cl);
        C pv[RL];
        if (!TC && col != 0) {
#pragma unroll
          for (int s = 0; s < RL; ++s)
            pv[s] = __ldg(dk + (j + s * JL) * Wh + col);
        }
        C x[RL];
#pragma unroll
        for (int q = 0; q < RL; ++q) x[q] = X[(j + q * JL) * CS + cl];
        if constexpr (JL > 1) stage_twiddle<C, RL, H / (JL * RL), false>(x, twc, j);
        dft<RL, false>(x);
        if (col == 0) {
#pragma unroll
          for (int s = 0; s < RL; ++s) COL0[j + s * JL] = x[s];
        } else if constexpr (TC) {  // w_hat_k (z_hat_k) at the natural bins of this rank's columns
#pragma unroll
          for (int s = 0; s < RL; ++s) wk[(j + s * JL) * Wh + col] = x[s];
        } else {
#pragma unroll
          for (int s = 0; s < RL; ++s) acc[s] = cadd(acc[s], cmul(pv[s], x[s]));
        }
      }
      __syncthreads();
      CLT(11)
    }
    if (rank == 0 && threadIdx.x < H) {
      const int r = threadIdx.x;
      C x0, xn;
      CP::unpack_col0(COL0, r, x0, xn);
      if constexpr (TC) {
        wk[r * Wh] = x0;
        wk[r * Wh + M] = xn;
      } else {
        acc0 = cadd(acc0, cmul(d0, x0));
        accN = cadd(accN, cmul(dMv, xn));
      }
    }
  }
#ifdef DCSC_CL_TRACE
  if (ADMM && threadIdx.x == 0 && blockIdx.y == 0 && blockIdx.x < CL)
    for (int f = 0; f < 3; ++f)
      printf("CLT f=%d rank=%u start=%llu ready_I=%llu bf_I=%llu recv_I=%llu rif=%llu rir=%llu prox=%llu "
             "ready_F=%llu bi_F=%llu recv_F=%llu cff=%llu last=%llu dwait=%llu gen1=%llu\n", f, rank, tt[f][6], tt[f][0],
             tt[f][1], tt[f][2], tt[f][7], tt[f][8], tt[f][9], tt[f][3], tt[f][4], tt[f][5], tt[f][10], tt[f][11],
             tt[f][12], tt[f][13]);
#endif
  cluster_wait();  // last B_F: every block delivered, no peer addresses this CTA's smem
  if constexpr (!TC) {
    C* dst = a.part + ((size_t)n * a.G + g) * NB;
    const int it = threadIdx.x;
    if (it < ITEMS_L) {
      const int cl = it % COLS, j = it / COLS;
      const int col = CP::col_of(rank, cl);
      if (col != 0) {
#pragma unroll
        for (int s = 0; s < RL; ++s) dst[(j + s * JL) * Wh + col] = acc[s];
      }
    }
    if (rank == 0 && threadIdx.x < H) {
      dst[threadIdx.x * Wh] = acc0;
      dst[threadIdx.x * Wh + M] = accN;
    }
  }
  if constexpr (ADMM) {
    __syncthreads();
    if ((threadIdx.x & 31) == 0) {
      const double* ws = wsum[threadIdx.x >> 5];
      s0 = ws[0]; s1 = ws[1]; s2 = ws[2]; s3 = ws[3]; s4 = ws[4]; s5 = ws[5]; s6 = ws[6];
    }
  }
  double v[7] = {s0, s1, s2, s3, s4, s5, 0.0};
  block_sum<T, 7>(v, red);
  const double mx = block_max(s6, red, T);
  const int GS = a.G * CL;  // sum slots / arrivals per image
  if (threadIdx.x == 0) {
    double* o = a.sums + ((size_t)n * GS + blockIdx.x) * kSums;
    for (int i = 0; i < 6; ++i) o[i] = v[i];
    o[6] = mx;
    o[7] = 0.0;
  }
  if constexpr (MODE == kPassAdmm || MODE == kPassPrologue) {
    __shared__ int last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
      const unsigned prev = atomicAdd(a.cnt + n, 1u);
      last = prev == (unsigned)(GS - 1);
      if (last) a.cnt[n] = 0;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    bool stop = false;
    if (MODE == kPassAdmm) {
      double tt = 0, th = 0, t2 = 0, dz2 = 0, z2 = 0, dth = 0, tinf = 0;
      for (int gg = 0; gg < GS; ++gg) {
        const double* s = a.sums + ((size_t)n * GS + gg) * kSums;
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
        ImageAdmm& mm = a.img[n];
        mm.iters = a.iter;
        mm.primal = primal;
        mm.zc = zc;
        mm.thc = thc;
        mm.tinf = tinf;
        if (stop) {
          mm.converged = 1;
          a.conv_w[n] = 1;
        }
      }
    }
    if (TC || stop || (MODE == kPassAdmm && a.is_last)) return;  // TC: lambda_hat from tc_lambda
    const R inv_rho = R(1) / rho;
    const C* pn = a.part + (size_t)n * a.G * NB;
    for (int b = threadIdx.x; b < NB; b += T) {
      C accb = __ldcg(pn + b);
      for (int gg = 1; gg < a.G; ++gg) accb = cadd(accb, __ldcg(pn + (size_t)gg * NB + b));
      const C xv = a.xhat[(size_t)n * NB + b];
      const R s = a.sigma[b];
      a.lamhat_w[(size_t)n * NB + b] = mk<C>((accb.x - xv.x * inv_rho) / s, (accb.y - xv.y * inv_rho) / s);
    }
  }
}

// Single-plane helpers. Buffers as above; every exchange fully synchronised.
template <class CP>
struct ClBufs {
  using C = typename CP::C;
  C *X, *Y, *Z, *TW, *COL0;
  unsigned long long* bar;
  unsigned phase;
  __device__ ClBufs(unsigned char* raw, unsigned long long* b) : bar(b), phase(0) {
    constexpr int BS = CP::buffer_bytes / sizeof(C);
    X = reinterpret_cast<C*>(raw);
    Y = X + BS;
    Z = Y + BS;
    TW = reinterpret_cast<C*>(raw + SmemCl<CP>::tw_off);
    COL0 = reinterpret_cast<C*>(raw + SmemCl<CP>::col0_off);
  }
};

// Forward of this CTA's rows (spatial pairs in Z) to a global NSL spectrum d;
// every rank stores its own columns, rank 0 the packed pair.
template <class CP>
__device__ __forceinline__ void cl_forward_to_global(ClBufs<CP>& b, unsigned rank, typename CP::C* __restrict__ d) {
  using C = typename CP::C;
  constexpr int Wh = CP::Wh, M = CP::M, H = CP::H, T = CP::T;
  CP::rows_fwd_to_send(b.Z, b.X, b.Z, b.TW);
  cl_exchange_sync<CP>(b.Z, b.Y, rank, b.bar, b.phase);
  CP::cols_fwd_first(b.Y, b.Z, b.X, b.TW, rank);
  __syncthreads();
  CP::cols_fwd_rest(b.X, b.Y, b.TW, rank, b.COL0, [](int, int) { return 0; },
                    [&](int r, int c, C v, int) { d[r * Wh + c] = v; });
  if (rank == 0)
    for (int r = threadIdx.x; r < H; r += T) {
      C x0, xn;
      CP::unpack_col0(b.COL0, r, x0, xn);
      d[r * Wh] = x0;
      d[r * Wh + M] = xn;
    }
}

// Inverse of a global NSL spectrum (gen) into this CTA's rows; the spatial
// pairs (times D) end in Z.
template <class CP, class GEN>
__device__ __forceinline__ void cl_inverse(ClBufs<CP>& b, unsigned rank, GEN&& gen) {
  CP::cols_inv(b.X, b.Y, b.TW, rank, gen);
  cl_exchange_sync<CP>(b.Y, b.Z, rank, b.bar, b.phase);
  CP::rows_inv_first(b.Z, b.Y, rank, b.X, b.TW);
  __syncthreads();
  CP::rows_inv_rest(b.X, b.Z, b.TW);
}

template <class CP, class SRC>
__global__ void __cluster_dims__(CP::CL, 1, 1) __launch_bounds__(CP::T)
    r2c_planes_cl(const SRC* __restrict__ src, size_t src_stride, cx<typename CP::R>* __restrict__ dst,
                  size_t dst_stride, const cx<typename CP::R>* tw, int* live_flags, int live_mod, int count) {
  using R = typename CP::R;
  using C = typename CP::C;
  constexpr int W = CP::W, Wh = CP::Wh, T = CP::T, M = CP::M, ROWS = CP::ROWS;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ __align__(8) unsigned long long bar_s;
  ClBufs<CP> b(smem_raw, &bar_s);
  const unsigned rank = cluster_rank();
  const int r0 = rank * ROWS;
  CP::load_twiddles(b.TW, tw);
  cl_init_exchange<CP>(b.bar);
  // persistent over planes (grid = resident clusters): the next plane's rows of
  // this rank are prefetched into L2 while the current plane transforms
  const int stride = gridDim.x / CP::CL;
  for (int p = blockIdx.x / CP::CL; p < count; p += stride) {
    const SRC* s = src + (size_t)p * src_stride + (size_t)r0 * W;
    if (threadIdx.x == 0 && p + stride < count)
      prefetch_l2_bulk(src + (size_t)(p + stride) * src_stride + (size_t)r0 * W, sizeof(SRC) * ROWS * W);
    int any = 0;
    for (int it = threadIdx.x; it < ROWS * M; it += T) {
      const int rl = it / M, m = it % M;
      R v0, v1;
      if constexpr (std::is_same<SRC, R>::value) {  // pixel pair as one vector load
        const C v = reinterpret_cast<const C*>(s)[it];
        v0 = v.x;
        v1 = v.y;
      } else {
        v0 = R(s[rl * W + 2 * m]);
        v1 = R(s[rl * W + 2 * m + 1]);
      }
      any |= (v0 != R(0)) | (v1 != R(0));
      b.Z[rl * Wh + m] = mk<C>(v0, v1);
    }
    any = __syncthreads_or(any);
    if (live_flags && threadIdx.x == 0 && any) atomicOr(live_flags + (p % live_mod), 1);
    cl_forward_to_global<CP>(b, rank, dst + (size_t)p * dst_stride);
    __syncthreads();
  }
}

template <class CP>
__global__ void __cluster_dims__(CP::CL, 1, 1) __launch_bounds__(CP::T)
    r2c_filters_cl(const double* __restrict__ d, int mh, int mw, cx<typename CP::R>* __restrict__ dst,
                   const cx<typename CP::R>* tw) {
  using R = typename CP::R;
  using C = typename CP::C;
  constexpr int Wh = CP::Wh, T = CP::T, M = CP::M, ROWS = CP::ROWS, NB = CP::NB;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ __align__(8) unsigned long long bar_s;
  ClBufs<CP> b(smem_raw, &bar_s);
  const unsigned rank = cluster_rank();
  const int k = blockIdx.x / CP::CL, r0 = rank * ROWS;
  CP::load_twiddles(b.TW, tw);
  cl_init_exchange<CP>(b.bar);
  const double* f = d + (size_t)k * mh * mw;
  for (int it = threadIdx.x; it < ROWS * M; it += T) {
    const int rl = it / M, m = it % M, r = r0 + rl;
    const int c0 = 2 * m, c1 = c0 + 1;
    const R v0 = (r < mh && c0 < mw) ? R(f[r * mw + c0]) : R(0);
    const R v1 = (r < mh && c1 < mw) ? R(f[r * mw + c1]) : R(0);
    b.Z[rl * Wh + m] = mk<C>(v0, v1);
  }
  __syncthreads();
  cl_forward_to_global<CP>(b, rank, dst + (size_t)k * NB);
}

template <class CP, class DST>
__global__ void __cluster_dims__(CP::CL, 1, 1) __launch_bounds__(CP::T)
    c2r_planes_cl(const cx<typename CP::R>* __restrict__ src, size_t src_stride, DST* __restrict__ dst,
                  size_t dst_stride, const cx<typename CP::R>* tw, const double* scale, int count) {
  using R = typename CP::R;
  using C = typename CP::C;
  constexpr int W = CP::W, Wh = CP::Wh, T = CP::T, M = CP::M, ROWS = CP::ROWS, D = CP::D;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ __align__(8) unsigned long long bar_s;
  ClBufs<CP> b(smem_raw, &bar_s);
  const unsigned rank = cluster_rank();
  const int r0 = rank * ROWS;
  CP::load_twiddles(b.TW, tw);
  cl_init_exchange<CP>(b.bar);
  // persistent over planes; each rank prefetches a quarter (its row block) of
  // the next plane's spectrum into L2 while the current plane transforms
  const int stride = gridDim.x / CP::CL;
  for (int p = blockIdx.x / CP::CL; p < count; p += stride) {
    const C* s = src + (size_t)p * src_stride;
    if (threadIdx.x == 0 && p + stride < count)
      prefetch_l2_bulk(src + (size_t)(p + stride) * src_stride + (size_t)r0 * Wh, sizeof(C) * ROWS * Wh);
    cl_inverse<CP>(b, rank, [&](int r, int c) { return s[r * Wh + c]; });
    const R sc = R((scale ? scale[p] : 1.0) / (double)D);
    DST* o = dst + (size_t)p * dst_stride + (size_t)r0 * W;
    for (int it = threadIdx.x; it < ROWS * M; it += T) {
      const int rl = it / M, m = it % M;
      const C v = b.Z[rl * Wh + m];
      if constexpr (std::is_same<DST, R>::value) {
        reinterpret_cast<C*>(o)[it] = mk<C>(v.x * sc, v.y * sc);
      } else {
        o[rl * W + 2 * m] = DST(v.x * sc);
        o[rl * W + 2 * m + 1] = DST(v.y * sc);
      }
    }
    __syncthreads();
  }
}

template <class CP>
__global__ void __cluster_dims__(CP::CL, 1, 1) __launch_bounds__(CP::T)
    mask_step_cl(const cx<typename CP::R>* __restrict__ c, cx<typename CP::R>* __restrict__ phat,
                 double* __restrict__ d_out, const int* live, const double* mu, int mh, int mw, int mode,
                 const cx<typename CP::R>* tw, const int* done) {
  using R = typename CP::R;
  using C = typename CP::C;
  constexpr int Wh = CP::Wh, T = CP::T, M = CP::M, ROWS = CP::ROWS, D = CP::D, NB = CP::NB;
  if (done && *done) return;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ __align__(8) unsigned long long bar_s;
  const unsigned rank = cluster_rank();
  const int k = blockIdx.x / CP::CL, r0 = rank * ROWS;
  if (!live[k]) {
    if (mode == 0) {
      for (int i = threadIdx.x + rank * T; i < NB; i += T * CP::CL) phat[(size_t)k * NB + i] = mk<C>(R(0), R(0));
    } else if (rank == 0) {
      for (int i = threadIdx.x; i < mh * mw; i += T) d_out[(size_t)k * mh * mw + i] = 0.0;
    }
    return;
  }
  ClBufs<CP> b(smem_raw, &bar_s);
  CP::load_twiddles(b.TW, tw);
  cl_init_exchange<CP>(b.bar);
  const C* s = c + (size_t)k * NB;
  cl_inverse<CP>(b, rank, [&](int r, int cc) { return s[r * Wh + cc]; });
  const R invD = R(1) / R(D);
  if (mode != 0) {  // 1: d_recover (-0.5/mu scaling), 2: plain cropped correlation
    if (rank == 0) {  // the support rows (mh <= ROWS) live in rank 0
      const double scale = mode == 2 ? 1.0 : -0.5 / fmax(mu[k], 1e-300);
      for (int i = threadIdx.x; i < mh * mw; i += T) {
        const int r = i / mw, cc = i % mw;
        const C v = b.Z[r * Wh + cc / 2];
        const R val = ((cc & 1) ? v.y : v.x) * invD;
        d_out[(size_t)k * mh * mw + i] = scale * (double)val;
      }
    }
    return;
  }
  for (int it = threadIdx.x; it < ROWS * M; it += T) {
    const int rl = it / M, m = it % M;
    const C v = b.Z[rl * Wh + m];
    const bool rin = r0 + rl < mh;
    const R v0 = (rin && 2 * m < mw) ? v.x * invD : R(0);
    const R v1 = (rin && 2 * m + 1 < mw) ? v.y * invD : R(0);
    b.Z[rl * Wh + m] = mk<C>(v0, v1);
  }
  __syncthreads();
  cl_forward_to_global<CP>(b, rank, phat + (size_t)k * NB);
}

}  // namespace dcsc_cuda
