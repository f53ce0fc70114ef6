// Shared-memory 2-D real FFT engine for one H x W plane per CTA (sm_100a).
//
// Replaces the reference's FFTW c2c transforms (proj/src/spectral.cpp:59-104)
// with half-spectrum r2c/c2r transforms. The reference always transforms real
// data (forward_dft copies a real slice, spectral.cpp:65-66) and keeps only the
// real part of every inverse (spectral.cpp:86-92), so all spectra it forms are
// Hermitian and the H x (W/2+1) half spectrum carries the same information.
// Conventions match the reference: unnormalised forward (sign -1), inverse
// scaled by 1/D applied by the caller (spectral.cpp:85).
//
// Layouts (complex elements, row-major):
//  * NSL  natural spectral layout [H][Wh], Wh = W/2+1 — the global layout of
//         every spectrum (d_hat, x_hat, lambda_hat, z_hat, CG vectors).
//  * PCL  packed column layout: NSL with columns 0 and W/2 (both spectra of
//         real columns after the row pass) packed as one complex column
//         P = X0 + i*XN in column 0; only columns [0, W/2) are transformed.
//  * RPL  row-pair layout [H/2][W+1]: pair a holds rows 2a (real part) and
//         2a+1 (imag part); the odd line stride W+1 keeps lane-per-line
//         accesses bank-conflict free.
// Forward:  RPL(real) -rows-> RPL(spec) -unpack-> PCL -cols-> PCL(spec)
// Inverse:  PCL(spec) -cols^-1-> PCL -pack-> RPL -rows^-1-> RPL(real * D)
// Producers write PCL directly (packing columns 0/W/2); consumers unpack
// column 0 on read (pcl_bin). Every 1-D pass is a Stockham autosort radix
// sequence executed out of place between two smem buffers (one sync/stage).
#pragma once
#include <cmath>
#include <type_traits>
#include <utility>

#include "common.cuh"

namespace dcsc_cuda {

// ---------------------------------------------------------------- constexpr trig
constexpr double kPi = 3.14159265358979323846264338327950288;

constexpr double taylor_sin(double x) {
  double term = x, sum = x;
  for (int n = 1; n < 20; ++n) {
    term *= -x * x / ((2.0 * n) * (2.0 * n + 1.0));
    sum += term;
  }
  return sum;
}
constexpr double taylor_cos(double x) {
  double term = 1.0, sum = 1.0;
  for (int n = 1; n < 20; ++n) {
    term *= -x * x / ((2.0 * n - 1.0) * (2.0 * n));
    sum += term;
  }
  return sum;
}
// cos / sin of 2*pi*m/n, reduced to the first octant for accuracy
constexpr double kcos(int m, int n);
constexpr double ksin(int m, int n) {
  m %= n;
  if (m < 0) m += n;
  if (2 * m > n) return -ksin(n - m, n);          // sin(2pi - x) = -sin x
  if (4 * m > n) return kcos(n - 4 * m, 4 * n);   // sin x = cos(pi/2 - x)
  return taylor_sin(2.0 * kPi * m / n);
}
constexpr double kcos(int m, int n) {
  m %= n;
  if (m < 0) m += n;
  if (2 * m > n) return kcos(n - m, n);           // cos(2pi - x) = cos x
  if (4 * m > n) return -kcos(n - 2 * m, 2 * n);  // cos x = -cos(pi - x)
  if (8 * m > n) return ksin(n - 4 * m, 4 * n);   // cos x = sin(pi/2 - x)
  return taylor_cos(2.0 * kPi * m / n);
}

template <int B, int E, class F>
__device__ __forceinline__ void sfor(F&& f) {
  if constexpr (B < E) {
    f(std::integral_constant<int, B>{});
    sfor<B + 1, E>(f);
  }
}

// ---------------------------------------------------------------- register DFTs
template <int R, bool INV, class C> __device__ __forceinline__ void dft(C* x);

// x * W_N^m (forward) or x * W_N^-m (inverse), W_N = exp(-2 pi i / N)
template <int N, int M, bool INV, class C>
__device__ __forceinline__ C twiddle_const(C x) {
  constexpr int m = M % N;
  if constexpr (m == 0) {
    return x;
  } else if constexpr (2 * m == N) {
    return mk<C>(-x.x, -x.y);
  } else if constexpr (4 * m == N) {
    return mul_mi<INV>(x);
  } else if constexpr (4 * m == 3 * N) {
    return mul_mi<!INV>(x);
  } else {
    using Rt = decltype(C::x);
    constexpr double c = kcos(m, N);
    constexpr double s = INV ? ksin(m, N) : -ksin(m, N);
    return mk<C>(x.x * Rt(c) - x.y * Rt(s), x.x * Rt(s) + x.y * Rt(c));
  }
}

template <int R1, int R2, bool INV, class C>
__device__ __forceinline__ void dft_2lvl(C* x) {
  constexpr int N = R1 * R2;
  C y[N];
  sfor<0, R2>([&](auto n2c) {
    constexpr int n2 = decltype(n2c)::value;
    C t[R1];
    sfor<0, R1>([&](auto n1c) { t[decltype(n1c)::value] = x[R2 * decltype(n1c)::value + n2]; });
    dft<R1, INV>(t);
    sfor<0, R1>([&](auto k1c) {
      constexpr int k1 = decltype(k1c)::value;
      y[n2 * R1 + k1] = twiddle_const<N, n2 * k1, INV>(t[k1]);
    });
  });
  sfor<0, R1>([&](auto k1c) {
    constexpr int k1 = decltype(k1c)::value;
    C t[R2];
    sfor<0, R2>([&](auto n2c) { t[decltype(n2c)::value] = y[decltype(n2c)::value * R1 + k1]; });
    dft<R2, INV>(t);
    sfor<0, R2>([&](auto k2c) { x[k1 + R1 * decltype(k2c)::value] = t[decltype(k2c)::value]; });
  });
}

template <int R, bool INV, class C>
__device__ __forceinline__ void dft(C* x) {
  using Rt = decltype(C::x);
  if constexpr (R == 1) {
  } else if constexpr (R == 2) {
    const C a = x[0], b = x[1];
    x[0] = cadd(a, b);
    x[1] = csub(a, b);
  } else if constexpr (R == 3) {
    constexpr Rt c = Rt(-0.5);
    constexpr Rt s = Rt(0.86602540378443864676372317075294);
    const C t = cadd(x[1], x[2]);
    const C m = mk<C>(x[0].x + c * t.x, x[0].y + c * t.y);
    const C d = mk<C>((x[1].x - x[2].x) * s, (x[1].y - x[2].y) * s);
    x[0] = cadd(x[0], t);
    // forward: X1 = m - i d, X2 = m + i d
    const C md = mul_mi<INV>(d);
    x[1] = cadd(m, md);
    x[2] = csub(m, md);
  } else if constexpr (R == 4) {
    const C t0 = cadd(x[0], x[2]), t1 = csub(x[0], x[2]);
    const C t2 = cadd(x[1], x[3]), t3 = mul_mi<INV>(csub(x[1], x[3]));
    x[0] = cadd(t0, t2);
    x[2] = csub(t0, t2);
    x[1] = cadd(t1, t3);
    x[3] = csub(t1, t3);
  } else if constexpr (R == 5) {
    constexpr Rt c1 = Rt(0.30901699437494742410229341718282);
    constexpr Rt c2 = Rt(-0.80901699437494742410229341718282);
    constexpr Rt s1 = Rt(0.95105651629515357211643933337938);
    constexpr Rt s2 = Rt(0.58778525229247312916870595463907);
    const C a1 = cadd(x[1], x[4]), a2 = cadd(x[2], x[3]);
    const C b1 = csub(x[1], x[4]), b2 = csub(x[2], x[3]);
    const C m1 = mk<C>(x[0].x + c1 * a1.x + c2 * a2.x, x[0].y + c1 * a1.y + c2 * a2.y);
    const C m2 = mk<C>(x[0].x + c2 * a1.x + c1 * a2.x, x[0].y + c2 * a1.y + c1 * a2.y);
    const C n1 = mul_mi<INV>(mk<C>(s1 * b1.x + s2 * b2.x, s1 * b1.y + s2 * b2.y));
    const C n2 = mul_mi<INV>(mk<C>(s2 * b1.x - s1 * b2.x, s2 * b1.y - s1 * b2.y));
    x[0] = cadd(x[0], cadd(a1, a2));
    x[1] = cadd(m1, n1);
    x[4] = csub(m1, n1);
    x[2] = cadd(m2, n2);
    x[3] = csub(m2, n2);
  } else if constexpr (R == 8) {
    dft_2lvl<4, 2, INV>(x);
  } else if constexpr (R == 16) {
    dft_2lvl<4, 4, INV>(x);
  } else if constexpr (R == 10) {
    dft_2lvl<2, 5, INV>(x);
  } else if constexpr (R == 6) {
    dft_2lvl<2, 3, INV>(x);
  } else {
    static_assert(R == 2, "unsupported radix");
  }
}

// ---------------------------------------------------------------- radix plans
template <int... Rs> struct RadixList {};

// Any length whose prime factors are 2, 3 and 5 has a plan: the tuned lists below for the
// compiled families, otherwise greedy from the largest radix {16, 10, 8, 6, 5, 4, 3, 2} that
// divides what is left (grid plugins, build.build_grid).
template <int R, class L> struct PrependR;
template <int R, int... Rs> struct PrependR<R, RadixList<Rs...>> { using type = RadixList<R, Rs...>; };
constexpr int greedy_radix(int L) {
  constexpr int rs[8] = {16, 10, 8, 6, 5, 4, 3, 2};
  for (int i = 0; i < 8; ++i)
    if (L % rs[i] == 0) return rs[i];
  return 0;
}
template <int L> struct PlanFor {
  static constexpr int R = greedy_radix(L);
  static_assert(R != 0, "FFT length must factor into 2, 3 and 5");
  using type = typename PrependR<R, typename PlanFor<L / R>::type>::type;
};
template <> struct PlanFor<1> { using type = RadixList<>; };
template <> struct PlanFor<8> { using type = RadixList<8>; };
template <> struct PlanFor<10> { using type = RadixList<10>; };
template <> struct PlanFor<12> { using type = RadixList<4, 3>; };
template <> struct PlanFor<16> { using type = RadixList<16>; };
template <> struct PlanFor<20> { using type = RadixList<4, 5>; };
template <> struct PlanFor<24> { using type = RadixList<8, 3>; };
template <> struct PlanFor<32> { using type = RadixList<8, 4>; };
template <> struct PlanFor<40> { using type = RadixList<8, 5>; };
template <> struct PlanFor<48> { using type = RadixList<16, 3>; };
template <> struct PlanFor<50> { using type = RadixList<10, 5>; };
template <> struct PlanFor<64> { using type = RadixList<8, 8>; };
template <> struct PlanFor<80> { using type = RadixList<16, 5>; };
template <> struct PlanFor<100> { using type = RadixList<10, 10>; };
template <> struct PlanFor<128> { using type = RadixList<16, 8>; };
template <> struct PlanFor<256> { using type = RadixList<16, 16>; };

template <class L> struct CountStages;
template <int... Rs> struct CountStages<RadixList<Rs...>> { static constexpr int value = sizeof...(Rs); };
template <int R, class L> struct Prepend;
template <int R, int... Rs> struct Prepend<R, RadixList<Rs...>> { using type = RadixList<R, Rs...>; };
template <class L, int R> struct Append;
template <int R, int... Rs> struct Append<RadixList<Rs...>, R> { using type = RadixList<Rs..., R>; };
template <class L> struct Reverse;
template <> struct Reverse<RadixList<>> { using type = RadixList<>; };
template <int R, int... Rs> struct Reverse<RadixList<R, Rs...>> {
  using type = typename Append<typename Reverse<RadixList<Rs...>>::type, R>::type;
};
template <class L> struct Split;
template <int R> struct Split<RadixList<R>> {
  static constexpr int first = R, last = R;
  using tail = RadixList<>;
  using init = RadixList<>;
};
template <int R, int R2, int... Rs> struct Split<RadixList<R, R2, Rs...>> {
  using rest = Split<RadixList<R2, Rs...>>;
  static constexpr int first = R, last = rest::last;
  using tail = RadixList<R2, Rs...>;
  using init = typename Prepend<R, typename rest::init>::type;
};

// Stage twiddles x[q] *= W_L^(q k STEP), read straight from the smem table:
// lanes of a warp share k, so every load is a single-wavefront broadcast and
// costs one issue slot (cheaper than composing powers with complex multiplies
// once the kernel is issue-bound).
template <class C, int R, int STEP, bool INV>
__device__ __forceinline__ void stage_twiddle(C* x, const C* __restrict__ tw, int k) {
  sfor<1, R>([&](auto qc) {
    constexpr int q = decltype(qc)::value;
    const C w = tw[q * k * STEP];
    x[q] = INV ? cmulc(w, x[q]) : cmul(x[q], w);
  });
}

// One Stockham stage over LINES lines of length L, radix R, NS = product of
// the radices already applied. load(line, idx) / store(line, idx, v) address
// the data (plain smem or fused producers/consumers). Lanes run over lines.
template <class C, int L, int R, int NS, bool INV, int LINES, int T, class LOAD, class STORE>
__device__ __forceinline__ void stockham(const C* __restrict__ tw, LOAD&& load, STORE&& store) {
  constexpr int J = L / R;
  constexpr int ITEMS = LINES * J;
#pragma unroll 1
  for (int it = threadIdx.x; it < ITEMS; it += T) {
    const int b = it % LINES;
    const int j = it / LINES;
    const int k = j % NS;
    C x[R];
#pragma unroll
    for (int q = 0; q < R; ++q) x[q] = load(b, j + q * J);
    if constexpr (NS > 1) stage_twiddle<C, R, L / (NS * R), INV>(x, tw, k);
    dft<R, INV>(x);
    const int o = (j / NS) * NS * R + k;
#pragma unroll
    for (int s = 0; s < R; ++s) store(b, o + s * NS, x[s]);
  }
}

// Plain smem stages for every radix in the list (ping-pong, one sync each);
// returns the buffer holding the result.
template <class C, int L, bool INV, int LINES, int ES, int LS, int T, int NS>
__device__ __forceinline__ C* run_stages(C* a, C*, const C*, RadixList<>) {
  return a;
}
template <class C, int L, bool INV, int LINES, int ES, int LS, int T, int NS, int R, int... Rest>
__device__ __forceinline__ C* run_stages(C* a, C* b, const C* tw, RadixList<R, Rest...>) {
  stockham<C, L, R, NS, INV, LINES, T>(
      tw, [&](int l, int i) { return a[l * LS + i * ES]; }, [&](int l, int i, C v) { b[l * LS + i * ES] = v; });
  __syncthreads();
  return run_stages<C, L, INV, LINES, ES, LS, T, NS * R>(b, a, tw, RadixList<Rest...>{});
}

// First inverse column stage (NS = 1) with its input generated: item `it` is
// column line col_of(it % LINES), output rows j*R + s of that line go to
// store(line, j*R + s). gen(r, c) returns natural bin (r, c); column 0 carries
// the packed pair gen(r, 0), gen(r, N0) (pack). The column-0 branch is
// uniform over the item, so it is taken once per item and every generator
// load of the item is issued before the first use (with a per-element
// ternary the compiler serialised one global round trip per element).
template <class C, int L, int R, int LINES, int T, bool SPLIT = false, class COLOF, class GEN, class PACK,
          class STORE>
__device__ __forceinline__ void gen_first_stage_inv(int N0, COLOF&& col_of, GEN&& gen, PACK&& pack,
                                                    STORE&& store) {
  constexpr int J = L / R;
  constexpr int ITEMS = LINES * J;
#pragma unroll 1
  for (int it = threadIdx.x; it < ITEMS; it += T) {
    const int line = it % LINES, j = it / LINES;
    const int col = col_of(line);
    C x[R];
    if constexpr (SPLIT) {
      // one load batch per branch path (heavy multi-channel generators: the
      // merged form below costs registers there, c1j3 2.38 -> 2.92 ms)
      if (col == 0) {
        C g0[R], gn[R];
#pragma unroll
        for (int q = 0; q < R; ++q) {
          g0[q] = gen(j + q * J, 0);
          gn[q] = gen(j + q * J, N0);
        }
#pragma unroll
        for (int q = 0; q < R; ++q) x[q] = pack(g0[q], gn[q]);
      } else {
#pragma unroll
        for (int q = 0; q < R; ++q) x[q] = gen(j + q * J, col);
      }
    } else {
      // every lane issues its item's loads; the column-0 lane (one per warp in
      // some layouts, e.g. rank 0 of a cluster) adds the partner column's
      // loads on top, so a warp pays one load round trip, not one per branch
      // path (c3s 1.268 -> 1.247 ms, C0 0.186 -> 0.180 ms)
#pragma unroll
      for (int q = 0; q < R; ++q) x[q] = gen(j + q * J, col);
      if (col == 0) {
        C gn[R];
#pragma unroll
        for (int q = 0; q < R; ++q) gn[q] = gen(j + q * J, N0);
#pragma unroll
        for (int q = 0; q < R; ++q) x[q] = pack(x[q], gn[q]);
      }
    }
    dft<R, true>(x);
#pragma unroll
    for (int s = 0; s < R; ++s) store(line, j * R + s, x[s]);
  }
}

template <int A, int B> struct Prod;
template <class L> struct ListProd;
template <> struct ListProd<RadixList<>> { static constexpr int value = 1; };
template <int R, int... Rs> struct ListProd<RadixList<R, Rs...>> {
  static constexpr int value = R * ListProd<RadixList<Rs...>>::value;
};

// ---------------------------------------------------------------- 2-D plane
// Layout (one buffer = NB complex): [H][Wh], Wh = W/2 + 1 (odd line stride
// for W = 0 mod 4, so lane-per-line accesses are bank-conflict free).
//  * spectral: natural half spectrum X[r][c], c in [0, W/2]; during the
//    column passes column 0 holds the packed pair P = X[.][0] + i X[.][W/2]
//    (both are spectra of real columns) and only columns [0, W/2) transform.
//  * spatial: element [r][m], m < W/2, holds (x[r][2m], x[r][2m+1]).
// Row transforms are W/2-point complex FFTs of those pairs with the r2c/c2r
// pre/post-processing X[k] <-> (Z[k], Z[W/2-k]) fused into the adjacent
// column stage (forward) or the first row stage (inverse).
template <class Rt, int H_, int W_, int T_>
struct Plane {
  using R = Rt;
  using C = cx<Rt>;
  static constexpr int H = H_, W = W_, T = T_;
  static constexpr int M = W / 2;     // row FFT length
  static constexpr int Wh = M + 1;
  static constexpr int NB = H * Wh;  // complex elements per plane buffer
  static constexpr int D = H * W;
  static constexpr int HALF = H * M;  // column-pass items (columns [0, W/2))
  static_assert(W % 2 == 0, "even grid width only");
  using RowPlan = typename PlanFor<M>::type;
  using ColPlan = typename PlanFor<H>::type;
  // twiddles: [0,M) row roots W_M^j, [M, M+H) column roots W_H^j,
  // [M+H, 2M+H+1) pre/post-processing roots W_W^k, k = 0..M
  static constexpr int TW_ROW = 0, TW_COL = M, TW_PP = M + H;
  static constexpr int TW_LEN = 2 * M + H + 1;
  static constexpr size_t buffer_bytes = sizeof(C) * NB;

  __device__ static __forceinline__ void load_twiddles(C* tw_s, const C* __restrict__ tw_g) {
    for (int i = threadIdx.x; i < TW_LEN; i += T) tw_s[i] = tw_g[i];
  }

  // --- spatial element (r, m) <-> real pixels (r, 2m), (r, 2m+1)
  __device__ static __forceinline__ int sidx(int r, int m) { return r * Wh + m; }

  // --- forward ---------------------------------------------------------
  // Row FFTs (length M) of the spatial pairs in `a`; returns the buffer with Z.
  __device__ static __forceinline__ C* rows_fwd(C* a, C* b, const C* tw) {
    return run_stages<C, M, false, H, 1, Wh, T, 1>(a, b, tw + TW_ROW, RowPlan{});
  }

  // r2c post-processing of row r at column c (natural bin) from the row FFT Z:
  // X[c] = E + W_W^c O, E = (Z[c] + conj Z[M-c])/2, O = -i/2 (Z[c] - conj Z[M-c]).
  // Column 0 returns the packed pair (X[0], X[M]) = (Re Z0 + Im Z0, Re Z0 - Im Z0).
  __device__ static __forceinline__ C post(const C* z, const C* tw, int r, int c) {
    const C z1 = z[r * Wh + c];
    if (c == 0) return mk<C>(z1.x + z1.y, z1.x - z1.y);
    const C z2 = z[r * Wh + (M - c)];
    // z2c = conj(z2); E = (z1 + z2c)/2 ; O = -i/2 (z1 - z2c)
    const C e = mk<C>(R(0.5) * (z1.x + z2.x), R(0.5) * (z1.y - z2.y));
    const C o = mk<C>(R(0.5) * (z1.y + z2.y), R(0.5) * (z2.x - z1.x));
    return cadd(e, cmul(tw[TW_PP + c], o));
  }

  // Forward column pass over Z (row-FFT output in `z`): the first stage applies
  // the r2c post-processing on load; the last stage hands every output to
  // cons(r, c, v, pre(r, c)) (c in [1, M)), column 0 (packed Y) goes to col0[r].
  // `z` and `b` are both clobbered. Ends with __syncthreads().
  template <class PRE, class CONS>
  __device__ static __forceinline__ void cols_fwd(C* z, C* b, const C* tw, C* col0, PRE&& pre, CONS&& cons) {
    using S = Split<ColPlan>;
    constexpr int NST = CountStages<ColPlan>::value;
    const C* twc = tw + TW_COL;
    auto consume_store = [&](auto&& load, auto nsc, auto rc) {
      constexpr int NS = decltype(nsc)::value, R = decltype(rc)::value;
      constexpr int J = H / R;
      constexpr int ITEMS = M * J;
#pragma unroll 1
      for (int it = threadIdx.x; it < ITEMS; it += T) {
        const int col = it % M, j = it / M;  // outputs rows j + s*NS (j < NS)
        using PT = decltype(pre(0, 1));
        PT pv[R];
        if (col != 0) {
#pragma unroll
          for (int s = 0; s < R; ++s) pv[s] = pre(j + s * NS, col);
        }
        C x[R];
#pragma unroll
        for (int q = 0; q < R; ++q) x[q] = load(col, j + q * J);
        if constexpr (NS > 1) stage_twiddle<C, R, H / (NS * R), false>(x, twc, j);
        dft<R, false>(x);
        if (col == 0) {
#pragma unroll
          for (int s = 0; s < R; ++s) col0[j + s * NS] = x[s];
        } else {
#pragma unroll
          for (int s = 0; s < R; ++s) cons(j + s * NS, col, x[s], pv[s]);
        }
      }
      __syncthreads();
    };
    auto post_load = [&](int col, int r) { return post(z, tw, r, col); };
    if constexpr (NST == 1) {
      consume_store(post_load, std::integral_constant<int, 1>{}, std::integral_constant<int, S::first>{});
    } else {
      constexpr int R1 = S::first;
      stockham<C, H, R1, 1, false, M, T>(twc, post_load, [&](int l, int i, C v) { b[i * Wh + l] = v; });
      __syncthreads();
      using Mid = typename Split<typename S::tail>::init;  // stages between first and last
      C* in = run_stages<C, H, false, M, Wh, 1, T, R1>(b, z, twc, Mid{});
      constexpr int NSL = H / S::last;
      consume_store([&](int l, int i) { return in[i * Wh + l]; }, std::integral_constant<int, NSL>{},
                    std::integral_constant<int, S::last>{});
    }
  }

  // Accumulating variant of cols_fwd for the coding pass: the last stage adds
  // d_hat(r,c) * X(r,c) into per-thread registers acc[i][s] (item i = tid + i*T,
  // output row j + s*NS). Bin ownership is fixed across calls, so acc lives in
  // registers for a whole filter group. Column 0 goes to col0 as in cols_fwd.
  static constexpr int LAST_R = Split<ColPlan>::last;
  static constexpr int LAST_NS = H / LAST_R;
  static constexpr int LAST_ITEMS = M * (H / LAST_R);
  static constexpr int LAST_IPT = (LAST_ITEMS + T - 1) / T;
  __device__ static __forceinline__ void acc_bin(int i, int s, int& r, int& c) {
    const int it = threadIdx.x + i * T;
    c = it % M;
    r = it / M + s * LAST_NS;
  }
  // `hook(free)` runs at the start of the last stage with the buffer that
  // stage does not read (the coding pass stages its next filter there).
  template <class HOOK>
  __device__ static __forceinline__ void cols_fwd_acc(C* z, C* b, const C* tw, C* col0, const C* __restrict__ dk,
                                                      C (&acc)[LAST_IPT][LAST_R], HOOK&& hook) {
    using S = Split<ColPlan>;
    constexpr int NST = CountStages<ColPlan>::value;
    constexpr int R = LAST_R, NS = LAST_NS, J = H / R;
    const C* twc = tw + TW_COL;
    auto last = [&](auto&& load, C* freebuf) {
      hook(freebuf);
#pragma unroll
      for (int i = 0; i < LAST_IPT; ++i) {
        const int it = threadIdx.x + i * T;
        if (LAST_IPT * T != LAST_ITEMS && it >= LAST_ITEMS) continue;
        const int col = it % M, j = it / M;
        C pv[R];
        if (col != 0) {
#pragma unroll
          for (int s = 0; s < R; ++s) pv[s] = __ldg(dk + (j + s * NS) * Wh + col);
        }
        C x[R];
#pragma unroll
        for (int q = 0; q < R; ++q) x[q] = load(col, j + q * J);
        if constexpr (NS > 1) stage_twiddle<C, R, H / (NS * R), false>(x, twc, j);
        dft<R, false>(x);
        if (col == 0) {
#pragma unroll
          for (int s = 0; s < R; ++s) col0[j + s * NS] = x[s];
        } else {
#pragma unroll
          for (int s = 0; s < R; ++s) acc[i][s] = cadd(acc[i][s], cmul(pv[s], x[s]));
        }
      }
      __syncthreads();
    };
    auto post_load = [&](int col, int r) { return post(z, tw, r, col); };
    if constexpr (NST == 1) {
      last(post_load, b);
    } else {
      constexpr int R1 = S::first;
      stockham<C, H, R1, 1, false, M, T>(twc, post_load, [&](int l, int i, C v) { b[i * Wh + l] = v; });
      __syncthreads();
      using Mid = typename Split<typename S::tail>::init;
      C* in = run_stages<C, H, false, M, Wh, 1, T, R1>(b, z, twc, Mid{});
      last([&](int l, int i) { return in[i * Wh + l]; }, in == b ? z : b);
    }
  }

  // --- fused row boundary (coding pass) ---------------------------------
  // The inverse row pass runs the forward plan reversed, so its last stage
  // (radix RX, outputs m = j + s*M/RX) lines up with the forward pass's first
  // stage (inputs m = j + q*M/RX): the prox can sit between them in registers.
  using RowPlanI = typename Reverse<RowPlan>::type;
  static constexpr int RI_N = CountStages<RowPlanI>::value;
  static constexpr int RX = Split<RowPlan>::first;
  static_assert(Split<RowPlanI>::last == RX, "plan reversal");
  // All inverse row stages but the last (the first applies the c2r
  // pre-processing); returns the last stage's input buffer (p itself if the
  // plan has a single stage, whose load then applies the pre-processing).
  __device__ static __forceinline__ C* rows_inv_head(C* p, C* b, const C* tw) {
    if constexpr (RI_N == 1) {
      return p;
    } else {
      using S = Split<RowPlanI>;
      constexpr int R1 = S::first;
      const C* twr = tw + TW_ROW;
      stockham<C, M, R1, 1, true, H, T>(
          twr, [&](int r, int k) { return pre(p, tw, r, k); }, [&](int l, int i, C v) { b[l * Wh + i] = v; });
      __syncthreads();
      using Mid = typename Split<typename S::tail>::init;
      return run_stages<C, M, true, H, 1, Wh, T, R1>(b, p, twr, Mid{});
    }
  }
  // Forward row stages after the first (the first is fused by the caller).
  __device__ static __forceinline__ C* rows_fwd_tail(C* a, C* b, const C* tw) {
    return run_stages<C, M, false, H, 1, Wh, T, RX>(a, b, tw + TW_ROW, typename Split<RowPlan>::tail{});
  }

  // --- inverse ---------------------------------------------------------
  // Inverse column pass with the first stage generating its input:
  // gen(r, c) returns natural bin (r, c), c in [0, M]; column 0 packs (r,0)+(r,M).
  // Returns the buffer holding the column-inverse result (PCL).
  // HOIST: column-0 branch taken once per item (gen_first_stage_inv) — for
  // generators that read global memory; generators that read only shared
  // memory (the staged coding pass) keep the per-element form, which the
  // compiler predicates (1% faster at 128x128).
  template <bool HOIST = true, bool SPLIT = false, class GEN>
  __device__ static __forceinline__ C* cols_inv(C* a, C* b, const C* tw, GEN&& gen) {
    using S = Split<ColPlan>;
    constexpr int R1 = S::first;
    const C* twc = tw + TW_COL;
    if constexpr (HOIST) {
      gen_first_stage_inv<C, H, R1, M, T, SPLIT>(
          M, [](int l) { return l; }, gen, [](C x0, C xn) { return pack_col0(x0, xn); },
          [&](int l, int i, C v) { a[i * Wh + l] = v; });
    } else {
      stockham<C, H, R1, 1, true, M, T>(
          twc, [&](int col, int r) { return col == 0 ? pack_col0(gen(r, 0), gen(r, M)) : gen(r, col); },
          [&](int l, int i, C v) { a[i * Wh + l] = v; });
    }
    __syncthreads();
    return run_stages<C, H, true, M, Wh, 1, T, R1>(a, b, twc, typename S::tail{});
  }

  // c2r pre-processing of row r at index k from the column-inverse result p:
  // Z'[k] = (A + Bc) + i W_W^-k (A - Bc), A = X[k], Bc = conj X[M-k];
  // X[0] = Re P, X[M] = Im P (packed column 0).
  __device__ static __forceinline__ C pre(const C* p, const C* tw, int r, int k) {
    if (k == 0) {
      const C q = p[r * Wh];
      return mk<C>(q.x + q.y, q.x - q.y);
    }
    const C a = p[r * Wh + k];
    const C bb = p[r * Wh + (M - k)];
    const C s = mk<C>(a.x + bb.x, a.y - bb.y);  // A + conj(B)
    const C d = mk<C>(a.x - bb.x, a.y + bb.y);  // A - conj(B)
    const C wd = cmulc(tw[TW_PP + k], d);       // W_W^-k (A - conj B)
    return mk<C>(s.x - wd.y, s.y + wd.x);       // s + i wd
  }

  // Inverse row pass (first stage applies the c2r pre-processing on load).
  // Input: column-inverse result in `p`; output: spatial pairs times D in the
  // returned buffer (p or b).
  __device__ static __forceinline__ C* rows_inv(C* p, C* b, const C* tw) {
    using S = Split<RowPlan>;
    constexpr int R1 = S::first;
    const C* twr = tw + TW_ROW;
    stockham<C, M, R1, 1, true, H, T>(
        twr, [&](int r, int k) { return pre(p, tw, r, k); }, [&](int l, int i, C v) { b[l * Wh + i] = v; });
    __syncthreads();
    return run_stages<C, M, true, H, 1, Wh, T, R1>(b, p, twr, typename S::tail{});
  }

  // Full inverse from a generator (used by c2r and the coding pass).
  template <class GEN>
  __device__ static __forceinline__ C* inverse(C* a, C* b, const C* tw, GEN&& gen) {
    C* c = cols_inv(a, b, tw, gen);
    return rows_inv(c, c == a ? b : a, tw);
  }

  // Natural bins (r,0) and (r,W/2) from a packed column-0 spectrum Y (stride STRIDE).
  template <int STRIDE = Wh>
  __device__ static __forceinline__ void unpack_col0(const C* pcl, int r, C& x0, C& xn) {
    const C y = pcl[r * STRIDE];
    const C ym = pcl[((H - r) % H) * STRIDE];
    x0 = mk<C>(R(0.5) * (y.x + ym.x), R(0.5) * (y.y - ym.y));
    xn = mk<C>(R(0.5) * (y.y + ym.y), R(0.5) * (ym.x - y.x));
  }
  // Packed column-0 entry from natural bins x0 (col 0) and xn (col W/2).
  __device__ static __forceinline__ C pack_col0(C x0, C xn) { return mk<C>(x0.x - xn.y, x0.y + xn.x); }
};

// Host-side twiddle table for Plane (forward roots, long double).
template <class P>
void fill_twiddles(typename P::C* tw) {
  using C = typename P::C;
  using R = typename P::R;
  auto root = [](long double num, long double den) {
    const long double a = -2.0L * 3.141592653589793238462643383279502884L * num / den;
    return mk<C>(R(std::cos(a)), R(std::sin(a)));
  };
  for (int j = 0; j < P::M; ++j) tw[P::TW_ROW + j] = root(j, P::M);
  for (int j = 0; j < P::H; ++j) tw[P::TW_COL + j] = root(j, P::H);
  for (int k = 0; k <= P::M; ++k) tw[P::TW_PP + k] = root(k, P::W);
}

}  // namespace dcsc_cuda
