// 2-D real FFT of one H x W plane split over a CL-CTA thread-block cluster
// (sm_90+/sm_100a distributed shared memory), for planes whose half spectrum
// does not fit one CTA's shared memory (C3: 256 x 256 FP32 = 258 KB).
//
// Ownership inside the cluster (rank c):
//   column passes: COLS = W/(2 CL) of the W/2 transformed columns, all H rows,
//                  local layout [H][CS] (CS = COLS + 1, odd stride). Columns are
//                  owned in mirror pairs (c, W/2 - c) so that the r2c/c2r pre/post
//                  processing of a bin and of its mirror happen in one rank
//                  (col_of / owner_of). Column 0 (rank 0) carries the packed pair
//                  X[.][0] + i X[.][W/2].
//   row passes:    rows [c*ROWS, (c+1)*ROWS), local layout [ROWS][Wh].
// Transposes are block exchanges: a column buffer [H][CS] is CL contiguous
// blocks [ROWS][CS] (block q = rank q's rows), and each block travels to its
// rank with one TMA bulk copy into the peer's staging buffer
// (cp.async.bulk.shared::cluster.shared::cta, completion counted on the
// receiver's mbarrier; kernels_cluster.cuh). The staging buffer then reads as
// [CL src][ROWS][CS] — i.e. exactly the [H][CS] column layout after the
// forward exchange — and the first stage of the next pass loads from it with
// the r2c/c2r pre/post-processing pairs (k, W/2-k) fused; the forward row pass
// stores its last stage straight into the send layout. No remote loads go
// through the LSU. Conventions are those of fft2d.cuh (Plane).
#pragma once
#include "fft2d.cuh"

namespace dcsc_cuda {

__device__ __forceinline__ unsigned cluster_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <class Rt, int H_, int W_, int CL_, int T_>
struct ClusterPlane {
  using R = Rt;
  using C = cx<Rt>;
  static constexpr int H = H_, W = W_, T = T_, CL = CL_;
  static constexpr int M = W / 2, Wh = M + 1, NB = H * Wh, D = H * W;
  static constexpr int ROWS = H / CL, COLS = M / CL, CS = COLS + 1;
  static constexpr int BLOCK = ROWS * CS;  // complex per exchanged block
  static_assert(H % CL == 0 && M % CL == 0, "cluster split");
  static_assert((BLOCK * sizeof(C)) % 16 == 0, "bulk copies move multiples of 16 bytes");
  static constexpr int BUF = (H * CS > ROWS * Wh) ? H * CS : ROWS * Wh;  // complex per buffer
  static constexpr size_t buffer_bytes = (sizeof(C) * BUF + 127) / 128 * 128;
  static constexpr unsigned block_bytes = sizeof(C) * BLOCK;
  using RowPlan = typename PlanFor<M>::type;
  using RowPlanI = typename Reverse<RowPlan>::type;
  using ColPlan = typename PlanFor<H>::type;
  static constexpr int TW_ROW = 0, TW_COL = M, TW_PP = M + H;
  static constexpr int TW_LEN = 2 * M + H + 1;
  static_assert(CountStages<ColPlan>::value >= 2, "column plan needs a first and a last stage");
  static_assert(CountStages<RowPlan>::value >= 2, "row plan needs a first and a last stage");

  __device__ static __forceinline__ void load_twiddles(C* tw_s, const C* __restrict__ tw_g) {
    for (int i = threadIdx.x; i < TW_LEN; i += T) tw_s[i] = tw_g[i];
  }
  __device__ static __forceinline__ C pack_col0(C x0, C xn) { return mk<C>(x0.x - xn.y, x0.y + xn.x); }

  // ---- pair ownership of the transformed columns [0, M) ----
  // pair p = min(k, M-k) in [0, M/2]; rank c owns pairs [c*HP, (c+1)*HP),
  // rank 0 also the self-mirror column M/2. Local index cl < HP is the pair's
  // low column, cl >= HP its mirror (rank 0: cl = 0 -> column 0 (packed),
  // cl = HP -> column M/2).
  static constexpr int HP = COLS / 2;
  static_assert(CL * HP * 2 == M, "pairs per rank");
  __device__ static __forceinline__ int col_of(unsigned c, int cl) {
    if (c == 0) {
      if (cl == 0) return 0;
      if (cl == HP) return M / 2;
      return cl < HP ? cl : M - (cl - HP);
    }
    const int p = (int)c * HP + (cl % HP);
    return cl < HP ? p : M - p;
  }
  __device__ static __forceinline__ void owner_of(int k, unsigned& c, int& cl) {
    const int p = k <= M / 2 ? k : M - k;
    if (p == M / 2) {
      c = 0;
      cl = HP;
    } else {
      c = (unsigned)(p / HP);
      cl = (p % HP) + (k <= M / 2 ? 0 : HP);
    }
  }
  // offset of (row-local rl, column k) in a staging buffer [CL][ROWS][CS]
  __device__ static __forceinline__ int stage_off(int rl, int k) {
    unsigned c;
    int cl;
    owner_of(k, c, cl);
    return (int)c * BLOCK + rl * CS + cl;
  }
  // element (rl, k) of the staged blocks; block `rank` stays in `self`
  __device__ static __forceinline__ C staged(const C* stg, const C* self, unsigned rank, int rl, int k) {
    unsigned c;
    int cl;
    owner_of(k, c, cl);
    return (c == rank ? self : stg)[(int)c * BLOCK + rl * CS + cl];
  }

  // ---- inverse: column pass (local columns), input generated from global ----
  // gen(r, col) returns natural bin (r, col), col in [0, M]. Returns the
  // column-pass result buffer (a or b), layout [H][CS].
  template <class GEN>
  __device__ static __forceinline__ void cols_inv_gen(C* a, unsigned rank, GEN&& gen) {
    using S = Split<ColPlan>;
    gen_first_stage_inv<C, H, S::first, COLS, T>(
        M, [&](int cl) { return col_of(rank, cl); }, gen, [](C x0, C xn) { return pack_col0(x0, xn); },
        [&](int l, int i, C v) { a[i * CS + l] = v; });
    __syncthreads();
  }
  // generator whose packed column 0 is produced by gen(r, 0) itself (no
  // partner column loads): every lane issues the same loads
  template <class GEN>
  __device__ static __forceinline__ void cols_inv_gen_prepacked(C* a, unsigned rank, GEN&& gen) {
    using S = Split<ColPlan>;
    constexpr int R = S::first, J = H / R, ITEMS = COLS * J;
#pragma unroll 1
    for (int it = threadIdx.x; it < ITEMS; it += T) {
      const int line = it % COLS, j = it / COLS;
      const int col = col_of(rank, line);
      C x[R];
#pragma unroll
      for (int q = 0; q < R; ++q) x[q] = gen(j + q * J, col);
      dft<R, true>(x);
#pragma unroll
      for (int s = 0; s < R; ++s) a[(j * R + s) * CS + line] = x[s];
    }
    __syncthreads();
  }
  __device__ static __forceinline__ C* cols_inv_rest(C* a, C* b, const C* tw) {
    using S = Split<ColPlan>;
    return run_stages<C, H, true, COLS, CS, 1, T, S::first>(a, b, tw + TW_COL, typename S::tail{});
  }
  template <class GEN>
  __device__ static __forceinline__ C* cols_inv(C* a, C* b, const C* tw, unsigned rank, GEN&& gen) {
    cols_inv_gen(a, rank, gen);
    return cols_inv_rest(a, b, tw);
  }

  __device__ static __forceinline__ C pre_pair(C xk, C xm, C w) {  // w = W_W^k
    const C s = mk<C>(xk.x + xm.x, xk.y - xm.y);                  // X[k] + conj X[M-k]
    const C d = mk<C>(xk.x - xm.x, xk.y + xm.y);                  // X[k] - conj X[M-k]
    const C wd = cmulc(w, d);
    return mk<C>(s.x - wd.y, s.y + wd.x);
  }
  // ---- inverse row pass, first stage: reads the received column blocks
  // `stg` [CL][ROWS][CS] with the c2r pre-processing fused; writes `out`
  // [ROWS][Wh]. Butterflies go in mirror pairs (j, J-j) — and (0, J/2), both
  // self-mirrored — so every staged element is loaded once.
  // The block of this rank itself is read from its own send buffer `self`
  // (it is not copied).
  __device__ static __forceinline__ void rows_inv_first(const C* stg, const C* self, unsigned rank, C* out,
                                                        const C* tw) {
    using S = Split<RowPlanI>;
    constexpr int R = S::first, J = M / R, TASKS = ROWS * (J / 2);
    static_assert(J % 2 == 0, "paired butterflies");
#pragma unroll 1
    for (int task = threadIdx.x; task < TASKS; task += T) {
      const int rl = task % ROWS, t = task / ROWS;
      const int ja = t == 0 ? 0 : t, jb = t == 0 ? J / 2 : J - t;
      C a[R], b[R];
#pragma unroll
      for (int q = 0; q < R; ++q) {
        a[q] = staged(stg, self, rank, rl, ja + J * q);
        b[q] = staged(stg, self, rank, rl, jb + J * q);
      }
      C xa[R], xb[R];
#pragma unroll
      for (int q = 0; q < R; ++q) {
        const int ka = ja + J * q, kb = jb + J * q;
        if (t == 0) {
          // item 0: mirror of J q is item 0 at R-q (q = 0: packed column 0)
          xa[q] = (q == 0) ? mk<C>(a[0].x + a[0].y, a[0].x - a[0].y) : pre_pair(a[q], a[R - q], tw[TW_PP + ka]);
          // item J/2: self-mirrored at R-1-q
          xb[q] = pre_pair(b[q], b[R - 1 - q], tw[TW_PP + kb]);
        } else {
          xa[q] = pre_pair(a[q], b[R - 1 - q], tw[TW_PP + ka]);
          xb[q] = pre_pair(b[q], a[R - 1 - q], tw[TW_PP + kb]);
        }
      }
      dft<R, true>(xa);
      dft<R, true>(xb);
#pragma unroll
      for (int s2 = 0; s2 < R; ++s2) {
        out[rl * Wh + ja * R + s2] = xa[s2];
        out[rl * Wh + jb * R + s2] = xb[s2];
      }
    }
  }
  // remaining inverse row stages (local), input in a; returns result buffer
  __device__ static __forceinline__ C* rows_inv_rest(C* a, C* b, const C* tw) {
    using S = Split<RowPlanI>;
    return run_stages<C, M, true, ROWS, 1, Wh, T, S::first>(a, b, tw + TW_ROW, typename S::tail{});
  }

  // ---- forward row pass (local rows): spatial pairs in `a`, scratch `b`;
  // the last stage stores into the send layout snd [CL dst][ROWS][CS]
  // (column k of row rl -> its owner's block). snd may alias `a`.
  __device__ static __forceinline__ void rows_fwd_to_send(C* a, C* b, C* snd, const C* tw) {
    using S = Split<RowPlan>;
    static_assert(CountStages<RowPlan>::value == 2, "two-stage row plan: a -> b -> snd");
    constexpr int RL = S::last;
    constexpr int NSL = M / RL;
    stockham<C, M, S::first, 1, false, ROWS, T>(
        tw + TW_ROW, [&](int l, int i) { return a[l * Wh + i]; }, [&](int l, int i, C v) { b[l * Wh + i] = v; });
    __syncthreads();
    stockham<C, M, RL, NSL, false, ROWS, T>(
        tw + TW_ROW, [&](int l, int i) { return b[l * Wh + i]; },
        [&](int l, int i, C v) { snd[stage_off(l, i)] = v; });
    __syncthreads();
  }

  // ---- forward column pass, first stage: reads the received column buffer
  // zc [H][CS] (rows of every rank, this rank's columns) with the r2c
  // post-processing fused. The two columns of a mirror pair are produced
  // together from one load of Z[c] and Z[M-c]: X[c] = E + w O,
  // X[M-c] = conj(E - w O). Writes `out` [H][CS].
  // Rows of this rank itself are read from its own send buffer `self`.
  __device__ static __forceinline__ void cols_fwd_first(const C* zc, const C* self, C* out, const C* tw,
                                                        unsigned rank) {
    using S = Split<ColPlan>;
    constexpr int R = S::first, J = H / R, TASKS = HP * J;
#pragma unroll 1
    for (int task = threadIdx.x; task < TASKS; task += T) {
      const int pl = task % HP, j = task / HP;
      // rank 0 / pl 0: column 0 (packed) and column M/2; otherwise pair (pl, pl + HP)
      const bool special = rank == 0 && pl == 0;
      const int cla = pl, clb = pl + HP;
      const int cola = col_of(rank, cla);  // low column (0 for the special task)
      C z1[R], z2[R];
#pragma unroll
      for (int q = 0; q < R; ++q) {
        const int r = j + q * J;
        const C* base = (r / ROWS == (int)rank) ? self : zc;
        z1[q] = base[r * CS + cla];
        z2[q] = base[r * CS + clb];
      }
      C xa[R], xb[R];
      if (special) {
        const C wm = tw[TW_PP + M / 2];
#pragma unroll
        for (int q = 0; q < R; ++q) {
          xa[q] = mk<C>(z1[q].x + z1[q].y, z1[q].x - z1[q].y);
          const C e = mk<C>(z2[q].x, R_(0));  // (Z + conj Z)/2
          const C o = mk<C>(z2[q].y, R_(0));  // -i/2 (Z - conj Z)
          xb[q] = cadd(e, cmul(wm, o));
        }
      } else {
        const C w = tw[TW_PP + cola];
#pragma unroll
        for (int q = 0; q < R; ++q) {
          const C e = mk<C>(R_(0.5) * (z1[q].x + z2[q].x), R_(0.5) * (z1[q].y - z2[q].y));
          const C o = mk<C>(R_(0.5) * (z1[q].y + z2[q].y), R_(0.5) * (z2[q].x - z1[q].x));
          const C wo = cmul(w, o);
          xa[q] = cadd(e, wo);
          xb[q] = cconj(csub(e, wo));
        }
      }
      dft<R, false>(xa);
      dft<R, false>(xb);
#pragma unroll
      for (int s2 = 0; s2 < R; ++s2) {
        out[(j * R + s2) * CS + cla] = xa[s2];
        out[(j * R + s2) * CS + clb] = xb[s2];
      }
    }
  }
  using R_ = Rt;

  // Middle column stages + the last one handed to cons(r, col, v, pre(r, col))
  // (col != 0); the packed column 0 (rank 0, local column 0) goes to col0[r].
  // Input (first-stage output) in a. Ends with __syncthreads().
  template <class PRE, class CONS>
  __device__ static __forceinline__ void cols_fwd_rest(C* a, C* b, const C* tw, unsigned rank, C* col0, PRE&& pre,
                                                      CONS&& cons) {
    using S = Split<ColPlan>;
    constexpr int R1 = S::first, RL = S::last, NSL = H / RL, J = H / RL, ITEMS = COLS * J;
    using Mid = typename Split<typename S::tail>::init;
    const C* twc = tw + TW_COL;
    C* in = run_stages<C, H, false, COLS, CS, 1, T, R1>(a, b, twc, Mid{});
#pragma unroll 1
    for (int it = threadIdx.x; it < ITEMS; it += T) {
      const int cl = it % COLS, j = it / COLS;
      const int col = col_of(rank, cl);
      using PT = decltype(pre(0, 1));
      PT pv[RL];
      if (col != 0) {
#pragma unroll
        for (int s = 0; s < RL; ++s) pv[s] = pre(j + s * NSL, col);
      }
      C x[RL];
#pragma unroll
      for (int q = 0; q < RL; ++q) x[q] = in[(j + q * J) * CS + cl];
      if constexpr (NSL > 1) stage_twiddle<C, RL, H / (NSL * RL), false>(x, twc, j);
      dft<RL, false>(x);
      if (col == 0) {
#pragma unroll
        for (int s = 0; s < RL; ++s) col0[j + s * NSL] = x[s];
      } else {
#pragma unroll
        for (int s = 0; s < RL; ++s) cons(j + s * NSL, col, x[s], pv[s]);
      }
    }
    __syncthreads();
  }

  template <int STRIDE = 1>
  __device__ static __forceinline__ void unpack_col0(const C* pcl, int r, C& x0, C& xn) {
    const C y = pcl[r * STRIDE];
    const C ym = pcl[((H - r) % H) * STRIDE];
    x0 = mk<C>(R(0.5) * (y.x + ym.x), R(0.5) * (y.y - ym.y));
    xn = mk<C>(R(0.5) * (y.y + ym.y), R(0.5) * (ym.x - y.x));
  }
};

}  // namespace dcsc_cuda
