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

template <int L> struct PlanFor;
template <> struct PlanFor<8> { using type = RadixList<8>; };
template <> struct PlanFor<12> { using type = RadixList<4, 3>; };
template <> struct PlanFor<16> { using type = RadixList<16>; };
template <> struct PlanFor<20> { using type = RadixList<4, 5>; };
template <> struct PlanFor<24> { using type = RadixList<8, 3>; };
template <> struct PlanFor<32> { using type = RadixList<8, 4>; };
template <> struct PlanFor<64> { using type = RadixList<8, 8>; };
template <> struct PlanFor<100> { using type = RadixList<10, 10>; };
template <> struct PlanFor<128> { using type = RadixList<16, 8>; };
template <> struct PlanFor<256> { using type = RadixList<16, 16>; };

// One Stockham stage over LINES lines of length L (elements at
// line*LS + idx*ES), radix R, NS = product of the radices already applied.
template <class C, int L, int R, int NS, bool INV, int LINES, int ES, int LS, int T>
__device__ __forceinline__ void stockham_stage(const C* __restrict__ in, C* __restrict__ out,
                                               const C* __restrict__ tw) {
  constexpr int J = L / R;
  constexpr int ITEMS = LINES * J;
  for (int it = threadIdx.x; it < ITEMS; it += T) {
    const int b = it % LINES;
    const int j = it / LINES;
    const int k = j % NS;
    C x[R];
#pragma unroll
    for (int q = 0; q < R; ++q) x[q] = in[b * LS + (j + q * J) * ES];
    if constexpr (NS > 1) {
#pragma unroll
      for (int q = 1; q < R; ++q) {
        const C w = tw[q * k * (L / (NS * R))];
        x[q] = INV ? cmulc(w, x[q]) : cmul(x[q], w);
      }
    }
    dft<R, INV>(x);
    const int o = (j / NS) * NS * R + k;
#pragma unroll
    for (int s = 0; s < R; ++s) out[b * LS + (o + s * NS) * ES] = x[s];
  }
}

// Runs every stage of RadixList; data starts in a, result pointer returned
// (a or b by stage parity). Ends with __syncthreads().
template <class C, int L, bool INV, int LINES, int ES, int LS, int T, int NS>
__device__ __forceinline__ C* run_stages(C* a, C*, const C*, RadixList<>) {
  return a;
}
template <class C, int L, bool INV, int LINES, int ES, int LS, int T, int NS, int R, int... Rest>
__device__ __forceinline__ C* run_stages(C* a, C* b, const C* tw, RadixList<R, Rest...>) {
  stockham_stage<C, L, R, NS, INV, LINES, ES, LS, T>(a, b, tw);
  __syncthreads();
  return run_stages<C, L, INV, LINES, ES, LS, T, NS * R>(b, a, tw, RadixList<Rest...>{});
}

template <int NSTAGES> struct Parity { static constexpr bool odd = NSTAGES & 1; };
template <class L> struct CountStages;
template <int... Rs> struct CountStages<RadixList<Rs...>> { static constexpr int value = sizeof...(Rs); };

template <int R, class L> struct Prepend;
template <int R, int... Rs> struct Prepend<R, RadixList<Rs...>> { using type = RadixList<R, Rs...>; };
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

// ---------------------------------------------------------------- 2-D plane
template <class Rt, int H_, int W_, int T_>
struct Plane {
  using R = Rt;
  using C = cx<Rt>;
  static constexpr int H = H_, W = W_, T = T_;
  static constexpr int Wh = W / 2 + 1;
  static constexpr int NB = H * Wh;      // complex elements in NSL / PCL (and smem buffer)
  static constexpr int RLS = W + 1;      // RPL line stride
  static constexpr int D = H * W;
  static constexpr int HALF = H * (W / 2);  // PCL items (columns [0, W/2))
  static_assert(H % 2 == 0 && W % 2 == 0, "even grid sizes only");
  static_assert((H / 2) * RLS <= NB, "RPL must fit in a plane buffer");
  using RowPlan = typename PlanFor<W>::type;
  using ColPlan = typename PlanFor<H>::type;
  static constexpr int ROW_STAGES = CountStages<RowPlan>::value;
  static constexpr int COL_STAGES = CountStages<ColPlan>::value;
  static constexpr bool SAME_TW = (H == W);
  static constexpr int TW_LEN = SAME_TW ? W : (W + H);
  static constexpr size_t buffer_bytes = sizeof(C) * NB;

  // twiddle tables (forward roots): tw_row[0..W), tw_col[0..H)
  __device__ static __forceinline__ const C* tw_row(const C* tw) { return tw; }
  __device__ static __forceinline__ const C* tw_col(const C* tw) { return SAME_TW ? tw : tw + W; }

  __device__ static __forceinline__ void load_twiddles(C* tw_s, const C* __restrict__ tw_g) {
    for (int i = threadIdx.x; i < TW_LEN; i += T) tw_s[i] = tw_g[i];
  }

  template <bool INV>
  __device__ static __forceinline__ C* rows(C* a, C* b, const C* tw) {
    return run_stages<C, W, INV, H / 2, 1, RLS, T, 1>(a, b, tw_row(tw), RowPlan{});
  }
  template <bool INV>
  __device__ static __forceinline__ C* cols(C* a, C* b, const C* tw) {
    return run_stages<C, H, INV, W / 2, Wh, 1, T, 1>(a, b, tw_col(tw), ColPlan{});
  }

  // RPL(spectral) in `src` -> PCL in `dst` (forward row unpack), then sync.
  __device__ static __forceinline__ void rows_to_cols(const C* __restrict__ src, C* __restrict__ dst) {
    constexpr int W2 = W / 2;
    for (int it = threadIdx.x; it < (H / 2) * W2; it += T) {
      const int a = it / W2, k = it % W2;
      const C* row = src + a * RLS;
      C* o0 = dst + (2 * a) * Wh;
      C* o1 = o0 + Wh;
      if (k == 0) {
        const C c0 = row[0], cn = row[W2];
        o0[0] = mk<C>(c0.x, cn.x);  // (X_{2a}[0], X_{2a}[W/2]) both real
        o1[0] = mk<C>(c0.y, cn.y);  // (X_{2a+1}[0], X_{2a+1}[W/2])
      } else {
        const C c = row[k], cm = row[W - k];
        // Xa = (C + conj(Cm))/2 ; Xb = -i/2 (C - conj(Cm))
        o0[k] = mk<C>(R(0.5) * (c.x + cm.x), R(0.5) * (c.y - cm.y));
        o1[k] = mk<C>(R(0.5) * (c.y + cm.y), R(0.5) * (cm.x - c.x));
      }
    }
    __syncthreads();
  }

  // PCL(spatial columns) in `src` -> RPL(spectral) in `dst` (inverse row pack), then sync.
  __device__ static __forceinline__ void cols_to_rows(const C* __restrict__ src, C* __restrict__ dst) {
    constexpr int W2 = W / 2;
    for (int it = threadIdx.x; it < (H / 2) * W; it += T) {
      const int a = it / W, k = it % W;
      const C* r0 = src + (2 * a) * Wh;
      const C* r1 = r0 + Wh;
      C xa, xb;
      if (k == 0) {
        xa = mk<C>(r0[0].x, R(0));
        xb = mk<C>(r1[0].x, R(0));
      } else if (k == W2) {
        xa = mk<C>(r0[0].y, R(0));
        xb = mk<C>(r1[0].y, R(0));
      } else if (k < W2) {
        xa = r0[k];
        xb = r1[k];
      } else {
        xa = cconj(r0[W - k]);
        xb = cconj(r1[W - k]);
      }
      // C = Xa + i Xb
      dst[a * RLS + k] = mk<C>(xa.x - xb.y, xa.y + xb.x);
    }
    __syncthreads();
  }

  // Forward r2c. Input: real plane in RPL in buffer a. Output: PCL spectrum
  // (returned pointer, a or b). Column 0 holds FFT_col(X0 + i XN).
  __device__ static __forceinline__ C* forward(C* a, C* b, const C* tw) {
    C* r = rows<false>(a, b, tw);
    C* o = (r == a) ? b : a;
    rows_to_cols(r, o);
    return cols<false>(o, r, tw);
  }

  // Inverse c2r (unscaled). Input: PCL spectrum in buffer a (column 0 packed).
  // Output: RPL real plane times D (returned pointer).
  __device__ static __forceinline__ C* inverse(C* a, C* b, const C* tw) {
    C* c = cols<true>(a, b, tw);
    C* o = (c == a) ? b : a;
    cols_to_rows(c, o);
    return rows<true>(o, c, tw);
  }

  // ---- fused column stages (coding hot loop) ----
  // Inverse column pass whose first Stockham stage generates its input on the
  // fly: gen(r, c) returns natural bin (r, c); column 0 packs (r,0)+(r,W/2).
  // Writes the first stage into `a`, runs the rest ping-pong; returns result.
  template <class GEN>
  __device__ static __forceinline__ C* cols_inv_generated(C* a, C* b, const C* tw, GEN&& gen) {
    using S = Split<ColPlan>;
    constexpr int R = S::first, J = H / R, LINES = W / 2, ITEMS = LINES * J;
#pragma unroll 1
    for (int it = threadIdx.x; it < ITEMS; it += T) {
      const int col = it % LINES, j = it / LINES;
      C x[R];
      if (col == 0) {
#pragma unroll
        for (int q = 0; q < R; ++q) x[q] = pack_col0(gen(j + q * J, 0), gen(j + q * J, W / 2));
      } else {
#pragma unroll
        for (int q = 0; q < R; ++q) x[q] = gen(j + q * J, col);
      }
      dft<R, true>(x);
#pragma unroll
      for (int s = 0; s < R; ++s) a[(j * R + s) * Wh + col] = x[s];
    }
    __syncthreads();
    return run_stages<C, H, true, W / 2, Wh, 1, T, R>(a, b, tw_col(tw), typename S::tail{});
  }

  // Forward column pass whose last Stockham stage hands each output to
  // cons(r, col, value, pre) instead of storing it; pre = prefetch(r, col) is
  // issued before the stage's smem reads. Column 0 outputs (the packed pair
  // spectrum Y) go to col0[r]; the caller unpacks them after a sync.
  template <class PRE, class CONS>
  __device__ static __forceinline__ void cols_fwd_consumed(C* a, C* b, const C* tw, C* col0, PRE&& pre,
                                                          CONS&& cons) {
    using S = Split<ColPlan>;
    constexpr int R = S::last, NS = H / R, J = H / R, LINES = W / 2, ITEMS = LINES * J;
    C* in = run_stages<C, H, false, W / 2, Wh, 1, T, 1>(a, b, tw_col(tw), typename S::init{});
    const C* twc = tw_col(tw);
#pragma unroll 1
    for (int it = threadIdx.x; it < ITEMS; it += T) {
      const int col = it % LINES, j = it / LINES;  // j < NS: outputs rows j + s*NS
      using PT = decltype(pre(0, 1));
      PT pv[R];
      if (col != 0) {
#pragma unroll
        for (int s = 0; s < R; ++s) pv[s] = pre(j + s * NS, col);
      }
      C x[R];
#pragma unroll
      for (int q = 0; q < R; ++q) x[q] = in[(j + q * J) * Wh + col];
      if constexpr (NS > 1) {
#pragma unroll
        for (int q = 1; q < R; ++q) x[q] = cmul(x[q], twc[q * j * (H / (NS * R))]);
      }
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
  }

  // Natural bins (r,0) and (r,W/2) from a forward PCL column 0.
  template <int STRIDE = Wh>
  __device__ static __forceinline__ void unpack_col0(const C* pcl, int r, C& x0, C& xn) {
    const C y = pcl[r * STRIDE];
    const C ym = pcl[((H - r) % H) * STRIDE];
    x0 = mk<C>(R(0.5) * (y.x + ym.x), R(0.5) * (y.y - ym.y));
    xn = mk<C>(R(0.5) * (y.y + ym.y), R(0.5) * (ym.x - y.x));
  }
  // PCL column-0 entry packing natural bins x0 (col 0) and xn (col W/2).
  __device__ static __forceinline__ C pack_col0(C x0, C xn) {
    return mk<C>(x0.x - xn.y, x0.y + xn.x);
  }
};

}  // namespace dcsc_cuda
