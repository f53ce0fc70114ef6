// Cluster (multi-CTA per plane) variants of the hot-path kernels for planes
// whose half spectrum exceeds one CTA's shared memory (C3: 256 x 256 FP32).
// Same algorithms and reference anchors as kernels.cuh; the FFT work of one
// plane is split over a CP::CL-CTA cluster (fft2d_cluster.cuh).
#pragma once
#include "fft2d_cluster.cuh"
#include "kernels.cuh"

namespace dcsc_cuda {

template <class CP>
struct SmemCl {
  using C = typename CP::C;
  static constexpr size_t bufs = 2 * CP::buffer_bytes;
  static constexpr size_t tw_off = bufs;
  static constexpr size_t col0_off = tw_off + sizeof(C) * CP::TW_LEN;
  static constexpr size_t u_off = (col0_off + sizeof(C) * CP::H + 127) / 128 * 128;
  static constexpr size_t u_bytes = sizeof(C) * CP::ROWS * CP::M;  // this CTA's rows of u (pixel pairs)
  static constexpr size_t plain = u_off;
  static constexpr size_t coding = u_off + u_bytes;
};

// The fused coding kernel (see coding_pass in kernels.cuh) with each plane's
// FFTs split over a cluster: rank c owns rows [c*ROWS, ...) of u / w and
// columns [c*COLS, ...) of the spectra. blockIdx.x = group * CL + rank.
template <class CP, int MODE>
__global__ void __cluster_dims__(CP::CL, 1, 1) __launch_bounds__(CP::T)
    coding_pass_cl(CodingArgs<typename CP::R> a) {
  using R = typename CP::R;
  using C = typename CP::C;
  using SM = SmemCl<CP>;
  constexpr int H = CP::H, M = CP::M, Wh = CP::Wh, NB = CP::NB, D = CP::D, T = CP::T, CL = CP::CL;
  constexpr int ROWS = CP::ROWS, COLS = CP::COLS;
  constexpr bool ADMM = MODE == kPassAdmm;

  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ double red[kSums * (T / 32)];
  __shared__ __align__(8) unsigned long long ubar_s;
  C* B0 = reinterpret_cast<C*>(smem_raw);
  C* B1 = B0 + CP::BUF;
  C* TW = reinterpret_cast<C*>(smem_raw + SM::tw_off);
  C* COL0 = reinterpret_cast<C*>(smem_raw + SM::col0_off);
  C* U = reinterpret_cast<C*>(smem_raw + SM::u_off);
  unsigned long long* ubar = &ubar_s;
  unsigned uphase = 0;
  const unsigned rank = cluster_rank();
  const int g = blockIdx.x / CL, n = blockIdx.y;
  const int r0 = rank * ROWS;
  if (ADMM && a.conv[n]) return;  // the whole cluster sees the same flag

  CP::load_twiddles(TW, a.tw);
  if (ADMM && threadIdx.x == 0) {
    mbar_init(ubar, 1);
    fence_async_smem();
  }
  __syncthreads();

  using S = Split<typename CP::ColPlan>;
  constexpr int RL = S::last, JL = H / RL, ITEMS_L = COLS * JL;
  static_assert(ITEMS_L <= T, "one last-stage item per thread");
  C acc[RL];
#pragma unroll
  for (int s = 0; s < RL; ++s) acc[s] = mk<C>(R(0), R(0));
  C acc0 = mk<C>(R(0), R(0)), accN = mk<C>(R(0), R(0));

  const R rho = a.rho, beta = a.beta, invD = R(1) / R(D);
  double s0 = 0, s1 = 0, s2 = 0, s3 = 0, s4 = 0, s5 = 0, s6 = 0;
  const int k0 = g * a.kpg;
  const int k1 = min(a.K, k0 + a.kpg);
  for (int k = k0; k < k1; ++k) {
    const C* __restrict__ dk = a.dhat + (size_t)k * NB;
    C* w;  // buffer holding this CTA's rows of w (spatial pairs)
    if constexpr (ADMM) {
      C* __restrict__ uk = reinterpret_cast<C*>(a.u + ((size_t)n * a.K + k) * D) + (size_t)r0 * M;
      const C* __restrict__ lam = a.lamhat + (size_t)n * NB;
      if (threadIdx.x == 0) {
        bulk_wait_read0();
        mbar_expect_tx(ubar, (unsigned)SM::u_bytes);
        bulk_g2s(U, uk, (unsigned)SM::u_bytes, ubar);
        if (k + 1 < k1) prefetch_l2_bulk(dk + NB, sizeof(C) * NB);
      }
      C* cs = CP::cols_inv(B0, B1, TW, rank, [&](int r, int c) {
        const int b = r * Wh + c;
        return cmulc(__ldg(dk + b), __ldg(lam + b));
      });
      C* ob = (cs == B0) ? B1 : B0;
      cluster_sync_all();  // every rank's column results are in place
      CP::rows_inv_first(cs, ob, TW, rank);
      __syncthreads();
      cluster_sync_all();  // every rank is done reading cs
      C* sp = CP::rows_inv_rest(ob, cs, TW);
      mbar_wait(ubar, uphase);
      uphase ^= 1u;
      R f0 = 0, f1 = 0, f2 = 0, f3 = 0, f4 = 0, f5 = 0, f6 = 0;
#pragma unroll 4
      for (int it = threadIdx.x; it < ROWS * M; it += T) {
        const int rl = it / M, m = it % M;
        const C uv = U[it];
        const C v = sp[rl * Wh + m];
        const R tv[2] = {v.x * invD, v.y * invD};
        const R uo[2] = {uv.x, uv.y};
        R wv[2], un2[2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const R t = tv[e];
          const R th_o = fmin(fmax(uo[e], -beta), beta);
          const R un = t - (th_o - uo[e]);
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
          wv[e] = R(2) * th - un;
          un2[e] = un;
        }
        U[it] = mk<C>(un2[0], un2[1]);
        sp[rl * Wh + m] = mk<C>(wv[0], wv[1]);
      }
      s0 += (double)f0; s1 += (double)f1; s2 += (double)f2; s3 += (double)f3;
      s4 += (double)f4; s5 += (double)f5; s6 = fmax(s6, (double)f6);
      fence_async_smem();
      __syncthreads();
      if (threadIdx.x == 0) {
        bulk_s2g(uk, U, (unsigned)SM::u_bytes);
        bulk_commit();
      }
      w = sp;
    } else {
      const C* __restrict__ src = reinterpret_cast<const C*>(
          (MODE == kPassMaps) ? a.maps + ((size_t)n * a.K + k) * D : a.u + ((size_t)n * a.K + k) * D) +
          (size_t)r0 * M;
      for (int it = threadIdx.x; it < ROWS * M; it += T) {
        const int rl = it / M, m = it % M;
        const C v = src[it];
        R w0, w1;
        if constexpr (MODE == kPassPrologue) {
          w0 = R(2) * fmin(fmax(v.x, -beta), beta) - v.x;
          w1 = R(2) * fmin(fmax(v.y, -beta), beta) - v.y;
        } else if constexpr (MODE == kPassObjective) {
          w0 = rho * (fmin(fmax(v.x, -beta), beta) - v.x);
          w1 = rho * (fmin(fmax(v.y, -beta), beta) - v.y);
          s0 += (double)fabs(w0) + (double)fabs(w1);
        } else {
          w0 = v.x;
          w1 = v.y;
          s0 += (double)fabs(w0) + (double)fabs(w1);
        }
        B0[rl * Wh + m] = mk<C>(w0, w1);
      }
      __syncthreads();
      w = B0;
    }
    // forward: local rows, transposing first column stage, accumulating last stage
    C* z = CP::rows_fwd(w, w == B0 ? B1 : B0, TW);
    C* zo = (z == B0) ? B1 : B0;
    cluster_sync_all();  // every rank's row results are in place
    CP::cols_fwd_first(z, zo, TW, rank);
    __syncthreads();
    cluster_sync_all();  // every rank is done reading z
    {
      // middle stages (none for a two-stage plan) then the accumulating last stage
      using Mid = typename Split<typename S::tail>::init;
      const C* twc = TW + CP::TW_COL;
      C* in = run_stages<C, H, false, COLS, CP::CS, 1, T, S::first>(zo, z, twc, Mid{});
      const int it = threadIdx.x;
      if (it < ITEMS_L) {
        const int cl = it % COLS, j = it / COLS;
        const int col = CP::col_of(rank, cl);
        C pv[RL];
        if (col != 0) {
#pragma unroll
          for (int s = 0; s < RL; ++s) pv[s] = __ldg(dk + (j + s * JL) * Wh + col);
        }
        C x[RL];
#pragma unroll
        for (int q = 0; q < RL; ++q) x[q] = in[(j + q * JL) * CP::CS + cl];
        if constexpr (JL > 1) stage_twiddle<C, RL, H / (JL * RL), false>(x, twc, j);
        dft<RL, false>(x);
        if (col == 0) {
#pragma unroll
          for (int s = 0; s < RL; ++s) COL0[j + s * JL] = x[s];
        } else {
#pragma unroll
          for (int s = 0; s < RL; ++s) acc[s] = cadd(acc[s], cmul(pv[s], x[s]));
        }
      }
      __syncthreads();
    }
    if (rank == 0 && threadIdx.x < H) {
      const int r = threadIdx.x;
      C x0, xn;
      CP::unpack_col0(COL0, r, x0, xn);
      acc0 = cadd(acc0, cmul(__ldg(dk + r * Wh), x0));
      accN = cadd(accN, cmul(__ldg(dk + r * Wh + M), xn));
    }
  }
  if (ADMM && threadIdx.x == 0) bulk_wait0();
  {
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
  cluster_sync_all();  // no rank exits while a peer may still address its smem
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
    if (stop || (MODE == kPassAdmm && a.is_last)) return;
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

// Forward of this CTA's rows (spatial pairs already in B0) to a global NSL
// spectrum d; every rank stores its own columns, rank 0 the packed pair.
template <class CP>
__device__ __forceinline__ void cl_forward_to_global(typename CP::C* B0, typename CP::C* B1,
                                                     const typename CP::C* TW, typename CP::C* COL0,
                                                     unsigned rank, typename CP::C* __restrict__ d) {
  using C = typename CP::C;
  constexpr int Wh = CP::Wh, M = CP::M, H = CP::H, T = CP::T;
  C* z = CP::rows_fwd(B0, B1, TW);
  C* zo = (z == B0) ? B1 : B0;
  cluster_sync_all();
  CP::cols_fwd_first(z, zo, TW, rank);
  __syncthreads();
  cluster_sync_all();
  CP::cols_fwd_rest(zo, z, TW, rank, COL0, [](int, int) { return 0; },
                    [&](int r, int c, C v, int) { d[r * Wh + c] = v; });
  if (rank == 0)
    for (int r = threadIdx.x; r < H; r += T) {
      C x0, xn;
      CP::unpack_col0(COL0, r, x0, xn);
      d[r * Wh] = x0;
      d[r * Wh + M] = xn;
    }
}

// Inverse of a global NSL spectrum (gen) into this CTA's rows; returns the
// buffer with the spatial pairs (times D).
template <class CP, class GEN>
__device__ __forceinline__ typename CP::C* cl_inverse(typename CP::C* B0, typename CP::C* B1,
                                                      const typename CP::C* TW, unsigned rank, GEN&& gen) {
  using C = typename CP::C;
  C* cs = CP::cols_inv(B0, B1, TW, rank, gen);
  C* ob = (cs == B0) ? B1 : B0;
  cluster_sync_all();
  CP::rows_inv_first(cs, ob, TW, rank);
  __syncthreads();
  cluster_sync_all();
  return CP::rows_inv_rest(ob, cs, TW);
}

template <class CP, class SRC>
__global__ void __cluster_dims__(CP::CL, 1, 1) __launch_bounds__(CP::T)
    r2c_planes_cl(const SRC* __restrict__ src, size_t src_stride, cx<typename CP::R>* __restrict__ dst,
                  size_t dst_stride, const cx<typename CP::R>* tw, int* live_flags, int live_mod) {
  using R = typename CP::R;
  using C = typename CP::C;
  using SM = SmemCl<CP>;
  constexpr int W = CP::W, Wh = CP::Wh, T = CP::T, M = CP::M, ROWS = CP::ROWS;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  C* B0 = reinterpret_cast<C*>(smem_raw);
  C* B1 = B0 + CP::BUF;
  C* TW = reinterpret_cast<C*>(smem_raw + SM::tw_off);
  C* COL0 = reinterpret_cast<C*>(smem_raw + SM::col0_off);
  const unsigned rank = cluster_rank();
  const int p = blockIdx.x / CP::CL, r0 = rank * ROWS;
  CP::load_twiddles(TW, tw);
  const SRC* s = src + (size_t)p * src_stride;
  int any = 0;
  for (int it = threadIdx.x; it < ROWS * M; it += T) {
    const int rl = it / M, m = it % M;
    const R v0 = R(s[(r0 + rl) * W + 2 * m]), v1 = R(s[(r0 + rl) * W + 2 * m + 1]);
    any |= (v0 != R(0)) | (v1 != R(0));
    B0[rl * Wh + m] = mk<C>(v0, v1);
  }
  any = __syncthreads_or(any);
  if (live_flags && threadIdx.x == 0 && any) atomicOr(live_flags + (p % live_mod), 1);
  cl_forward_to_global<CP>(B0, B1, TW, COL0, rank, dst + (size_t)p * dst_stride);
  cluster_sync_all();
}

template <class CP>
__global__ void __cluster_dims__(CP::CL, 1, 1) __launch_bounds__(CP::T)
    r2c_filters_cl(const double* __restrict__ d, int mh, int mw, cx<typename CP::R>* __restrict__ dst,
                   const cx<typename CP::R>* tw) {
  using R = typename CP::R;
  using C = typename CP::C;
  using SM = SmemCl<CP>;
  constexpr int Wh = CP::Wh, T = CP::T, M = CP::M, ROWS = CP::ROWS, NB = CP::NB;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  C* B0 = reinterpret_cast<C*>(smem_raw);
  C* B1 = B0 + CP::BUF;
  C* TW = reinterpret_cast<C*>(smem_raw + SM::tw_off);
  C* COL0 = reinterpret_cast<C*>(smem_raw + SM::col0_off);
  const unsigned rank = cluster_rank();
  const int k = blockIdx.x / CP::CL, r0 = rank * ROWS;
  CP::load_twiddles(TW, tw);
  const double* f = d + (size_t)k * mh * mw;
  for (int it = threadIdx.x; it < ROWS * M; it += T) {
    const int rl = it / M, m = it % M, r = r0 + rl;
    const int c0 = 2 * m, c1 = c0 + 1;
    const R v0 = (r < mh && c0 < mw) ? R(f[r * mw + c0]) : R(0);
    const R v1 = (r < mh && c1 < mw) ? R(f[r * mw + c1]) : R(0);
    B0[rl * Wh + m] = mk<C>(v0, v1);
  }
  __syncthreads();
  cl_forward_to_global<CP>(B0, B1, TW, COL0, rank, dst + (size_t)k * NB);
  cluster_sync_all();
}

template <class CP, class DST>
__global__ void __cluster_dims__(CP::CL, 1, 1) __launch_bounds__(CP::T)
    c2r_planes_cl(const cx<typename CP::R>* __restrict__ src, size_t src_stride, DST* __restrict__ dst,
                  size_t dst_stride, const cx<typename CP::R>* tw, const double* scale) {
  using R = typename CP::R;
  using C = typename CP::C;
  using SM = SmemCl<CP>;
  constexpr int W = CP::W, Wh = CP::Wh, T = CP::T, M = CP::M, ROWS = CP::ROWS, D = CP::D;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  C* B0 = reinterpret_cast<C*>(smem_raw);
  C* B1 = B0 + CP::BUF;
  C* TW = reinterpret_cast<C*>(smem_raw + SM::tw_off);
  const unsigned rank = cluster_rank();
  const int p = blockIdx.x / CP::CL, r0 = rank * ROWS;
  CP::load_twiddles(TW, tw);
  __syncthreads();
  const C* s = src + (size_t)p * src_stride;
  C* sp = cl_inverse<CP>(B0, B1, TW, rank, [&](int r, int c) { return s[r * Wh + c]; });
  const R sc = R((scale ? scale[p] : 1.0) / (double)D);
  DST* o = dst + (size_t)p * dst_stride;
  for (int it = threadIdx.x; it < ROWS * M; it += T) {
    const int rl = it / M, m = it % M;
    const C v = sp[rl * Wh + m];
    o[(r0 + rl) * W + 2 * m] = DST(v.x * sc);
    o[(r0 + rl) * W + 2 * m + 1] = DST(v.y * sc);
  }
  cluster_sync_all();
}

template <class CP>
__global__ void __cluster_dims__(CP::CL, 1, 1) __launch_bounds__(CP::T)
    mask_step_cl(const cx<typename CP::R>* __restrict__ c, cx<typename CP::R>* __restrict__ phat,
                 double* __restrict__ d_out, const int* live, const double* mu, int mh, int mw, int mode,
                 const cx<typename CP::R>* tw, const int* done) {
  using R = typename CP::R;
  using C = typename CP::C;
  using SM = SmemCl<CP>;
  constexpr int Wh = CP::Wh, T = CP::T, M = CP::M, ROWS = CP::ROWS, D = CP::D, NB = CP::NB;
  if (done && *done) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  C* B0 = reinterpret_cast<C*>(smem_raw);
  C* B1 = B0 + CP::BUF;
  C* TW = reinterpret_cast<C*>(smem_raw + SM::tw_off);
  C* COL0 = reinterpret_cast<C*>(smem_raw + SM::col0_off);
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
  CP::load_twiddles(TW, tw);
  __syncthreads();
  const C* s = c + (size_t)k * NB;
  C* sp = cl_inverse<CP>(B0, B1, TW, rank, [&](int r, int cc) { return s[r * Wh + cc]; });
  const R invD = R(1) / R(D);
  if (mode == 1) {
    if (rank == 0) {  // the support rows (mh <= ROWS) live in rank 0
      const double scale = -0.5 / fmax(mu[k], 1e-300);
      for (int i = threadIdx.x; i < mh * mw; i += T) {
        const int r = i / mw, cc = i % mw;
        const C v = sp[r * Wh + cc / 2];
        const R val = ((cc & 1) ? v.y : v.x) * invD;
        d_out[(size_t)k * mh * mw + i] = scale * (double)val;
      }
    }
    cluster_sync_all();
    return;
  }
  for (int it = threadIdx.x; it < ROWS * M; it += T) {
    const int rl = it / M, m = it % M;
    const C v = sp[rl * Wh + m];
    const bool rin = r0 + rl < mh;
    const R v0 = (rin && 2 * m < mw) ? v.x * invD : R(0);
    const R v1 = (rin && 2 * m + 1 < mw) ? v.y * invD : R(0);
    sp[rl * Wh + m] = mk<C>(v0, v1);
  }
  __syncthreads();
  C* other = (sp == B0) ? B1 : B0;
  cl_forward_to_global<CP>(sp, other, TW, COL0, rank, phat + (size_t)k * NB);
  cluster_sync_all();
}

}  // namespace dcsc_cuda
