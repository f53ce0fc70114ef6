/* FFTW3-API shim (TEST INFRASTRUCTURE ONLY — never linked into the product).
 *
 * Restates the algorithm FFTW3 computes for the subset the reference uses
 * (proj/src/spectral.cpp:16-47 plan cache, :59-68 forward, :76-98 inverse):
 * an unnormalised, out-of-place, row-major N-D complex DFT with sign -1
 * (FFTW_FORWARD) or +1 (FFTW_BACKWARD). FFTW itself is not in this image and
 * its version is unpinned by the reference (proj/CMakeLists.txt:16-17).
 *
 * Algorithm: per axis, an iterative mixed-radix Stockham autosort transform
 * (radix 4, 2, 3, 5 butterflies, any remaining odd prime by a direct O(p^2)
 * butterfly) run over all the sequences of the axis at once, the innermost
 * loop over contiguous memory. Per-stage twiddles are tabulated once per plan
 * from sin/cos evaluated directly in double (exact at the quarter points, no
 * recurrences), so the transform is accurate to a few ulps * log(n). Executing a plan is thread-safe (all
 * scratch is per call), matching FFTW's "execute on fresh arrays" contract that
 * the reference relies on under OpenMP (spectral.cpp:16-18).
 *
 * Pinned by the reference's own known answers (tests/test_oracle_pins.py
 * restates proj/tests/test_spectral.cpp:15-80,137-177) and cross-checked
 * against numpy.fft.
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "fftw3.h"

typedef struct {
  double re, im;
} cplx;

/* One Stockham stage: radix r, ns = product of the radices already applied. */
typedef struct {
  int r, ns;
  cplx* tw; /* tw[k * r + q] = exp(sign 2 pi i q k / (ns r)), k < ns, q < r */
} stage;

typedef struct {
  int n, nst;
  stage st[64];
  cplx* root; /* root[q] = exp(sign 2 pi i q / r) for the generic odd-prime radix (largest r) */
} axis_plan;

struct fftw_plan_s {
  int rank;
  int sign;
  size_t total;
  int dims[16];
  axis_plan axes[16];
};

fftw_complex* fftw_alloc_complex(size_t n) {
  void* p = NULL;
  if (posix_memalign(&p, 64, (n ? n : 1) * sizeof(fftw_complex)) != 0) return NULL;
  return (fftw_complex*)p;
}

void fftw_free(void* p) { free(p); }

static const double kTwoPi = 6.283185307179586476925286766559;

/* exp(sign 2 pi i m / d), exact at the quarter points */
static cplx unit_root(long m, long d, int sign) {
  m %= d;
  if (m < 0) m += d;
  cplx w;
  if (m == 0) { w.re = 1; w.im = 0; return w; }
  if (4 * m == d) { w.re = 0; w.im = (double)sign; return w; }
  if (2 * m == d) { w.re = -1; w.im = 0; return w; }
  if (4 * m == 3 * d) { w.re = 0; w.im = -(double)sign; return w; }
  const double ang = kTwoPi * (double)m / (double)d;
  w.re = cos(ang);
  w.im = (double)sign * sin(ang);
  return w;
}

static int init_axis(axis_plan* a, int n, int sign) {
  a->n = n;
  a->nst = 0;
  a->root = NULL;
  int fac[64], nf = 0, m = n;
  while (m % 4 == 0) { fac[nf++] = 4; m /= 4; }
  while (m % 2 == 0) { fac[nf++] = 2; m /= 2; }
  for (int p = 3; m > 1; p += 2)
    while (m % p == 0) { fac[nf++] = p; m /= p; }
  int ns = 1, rmax = 1;
  for (int f = 0; f < nf; ++f) {
    const int r = fac[f];
    if (r > 64) return 0; /* primes above 64 are not needed by the reference sizes */
    stage* st = &a->st[a->nst++];
    st->r = r;
    st->ns = ns;
    st->tw = (cplx*)malloc((size_t)ns * r * sizeof(cplx));
    for (int k = 0; k < ns; ++k)
      for (int q = 0; q < r; ++q) st->tw[k * r + q] = unit_root((long)q * k, (long)ns * r, sign);
    ns *= r;
    if (r > rmax && r > 5) rmax = r;
  }
  if (rmax > 5) {
    a->root = (cplx*)malloc((size_t)rmax * sizeof(cplx));
    for (int q = 0; q < rmax; ++q) a->root[q] = unit_root(q, rmax, sign);
  }
  return 1;
}

static void free_axis(axis_plan* a) {
  for (int s = 0; s < a->nst; ++s) free(a->st[s].tw);
  free(a->root);
}

static inline cplx cmul(cplx a, cplx b) {
  cplx r = {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re};
  return r;
}
static inline cplx cadd(cplx a, cplx b) {
  cplx r = {a.re + b.re, a.im + b.im};
  return r;
}
static inline cplx csub(cplx a, cplx b) {
  cplx r = {a.re - b.re, a.im - b.im};
  return r;
}
/* multiply by sign * i */
static inline cplx mul_si(cplx a, double s) {
  cplx r = {-s * a.im, s * a.re};
  return r;
}

/* One Stockham stage over a batch of `bat` transforms: element (index j,
 * transform c) at x[j * es + c * bs]. Output index o = (j / ns) ns r + k + s ns. */
static void run_stage(const stage* st, int n, size_t bat, size_t es, size_t bs, const cplx* x, cplx* y, int sign,
                      const cplx* root) {
  const int r = st->r, ns = st->ns, J = n / r;
  const double sg = (double)sign;
  for (int j = 0; j < J; ++j) {
    const int k = j % ns;
    const size_t o = (size_t)(j / ns) * ns * r + k;
    const cplx* w = st->tw + (size_t)k * r;
    const cplx* xj = x + (size_t)j * es;
    cplx* yo = y + o * es;
    const size_t xs = (size_t)J * es, ys = (size_t)ns * es;
    if (r == 2) {
      for (size_t c = 0, cb = 0; c < bat; ++c, cb += bs) {
        const cplx a = xj[cb], b = k ? cmul(xj[xs + cb], w[1]) : xj[xs + cb];
        yo[cb] = cadd(a, b);
        yo[ys + cb] = csub(a, b);
      }
    } else if (r == 4) {
      for (size_t c = 0, cb = 0; c < bat; ++c, cb += bs) {
        const cplx x0 = xj[cb];
        const cplx x1 = k ? cmul(xj[xs + cb], w[1]) : xj[xs + cb];
        const cplx x2 = k ? cmul(xj[2 * xs + cb], w[2]) : xj[2 * xs + cb];
        const cplx x3 = k ? cmul(xj[3 * xs + cb], w[3]) : xj[3 * xs + cb];
        const cplx t0 = cadd(x0, x2), t1 = csub(x0, x2), t2 = cadd(x1, x3), t3 = mul_si(csub(x1, x3), sg);
        yo[cb] = cadd(t0, t2);
        yo[ys + cb] = cadd(t1, t3);
        yo[2 * ys + cb] = csub(t0, t2);
        yo[3 * ys + cb] = csub(t1, t3);
      }
    } else if (r == 3) {
      const double c1 = -0.5, s1 = sg * 0.86602540378443864676372317075294;
      for (size_t c = 0, cb = 0; c < bat; ++c, cb += bs) {
        const cplx x0 = xj[cb];
        const cplx x1 = k ? cmul(xj[xs + cb], w[1]) : xj[xs + cb];
        const cplx x2 = k ? cmul(xj[2 * xs + cb], w[2]) : xj[2 * xs + cb];
        const cplx t = cadd(x1, x2), d = csub(x1, x2);
        const cplx m = {x0.re + c1 * t.re, x0.im + c1 * t.im};
        const cplx e = {-s1 * d.im, s1 * d.re}; /* i s1 d */
        yo[cb] = cadd(x0, t);
        yo[ys + cb] = cadd(m, e);
        yo[2 * ys + cb] = csub(m, e);
      }
    } else if (r == 5) {
      const double c1 = 0.30901699437494742410229341718282, c2 = -0.80901699437494742410229341718282;
      const double s1 = sg * 0.95105651629515357211643933337938, s2 = sg * 0.58778525229247312916870595463907;
      for (size_t c = 0, cb = 0; c < bat; ++c, cb += bs) {
        const cplx x0 = xj[cb];
        const cplx x1 = k ? cmul(xj[xs + cb], w[1]) : xj[xs + cb];
        const cplx x2 = k ? cmul(xj[2 * xs + cb], w[2]) : xj[2 * xs + cb];
        const cplx x3 = k ? cmul(xj[3 * xs + cb], w[3]) : xj[3 * xs + cb];
        const cplx x4 = k ? cmul(xj[4 * xs + cb], w[4]) : xj[4 * xs + cb];
        const cplx a1 = cadd(x1, x4), a2 = cadd(x2, x3), b1 = csub(x1, x4), b2 = csub(x2, x3);
        const cplx m1 = {x0.re + c1 * a1.re + c2 * a2.re, x0.im + c1 * a1.im + c2 * a2.im};
        const cplx m2 = {x0.re + c2 * a1.re + c1 * a2.re, x0.im + c2 * a1.im + c1 * a2.im};
        /* i (s1 b1 + s2 b2), i (s2 b1 - s1 b2) */
        const cplx n1 = {-(s1 * b1.im + s2 * b2.im), s1 * b1.re + s2 * b2.re};
        const cplx n2 = {-(s2 * b1.im - s1 * b2.im), s2 * b1.re - s1 * b2.re};
        yo[cb] = cadd(x0, cadd(a1, a2));
        yo[ys + cb] = cadd(m1, n1);
        yo[4 * ys + cb] = csub(m1, n1);
        yo[2 * ys + cb] = cadd(m2, n2);
        yo[3 * ys + cb] = csub(m2, n2);
      }
    } else { /* generic odd prime: direct DFT_r of the twiddled inputs */
      cplx t[64];
      for (size_t c = 0, cb = 0; c < bat; ++c, cb += bs) {
        for (int q = 0; q < r; ++q) t[q] = (q && k) ? cmul(xj[q * xs + cb], w[q]) : xj[q * xs + cb];
        for (int s2 = 0; s2 < r; ++s2) {
          cplx acc = t[0];
          for (int q = 1; q < r; ++q) acc = cadd(acc, cmul(t[q], root[((long)q * s2) % r]));
          yo[s2 * ys + cb] = acc;
        }
      }
    }
  }
}

/* In-place transform of `bat` length-n sequences at x (element j of sequence c
 * at x[j * es + c * bs], the n * bat elements dense); scratch holds n * bat values. */
static void fft_batch(const axis_plan* ap, cplx* x, cplx* scratch, size_t bat, size_t es, size_t bs, int sign) {
  cplx* a = x;
  cplx* b = scratch;
  for (int s = 0; s < ap->nst; ++s) {
    run_stage(&ap->st[s], ap->n, bat, es, bs, a, b, sign, ap->root);
    cplx* t = a;
    a = b;
    b = t;
  }
  if (a != x) memcpy(x, a, (size_t)ap->n * bat * sizeof(cplx));
}

fftw_plan fftw_plan_dft(int rank, const int* n, fftw_complex* in, fftw_complex* out, int sign,
                        unsigned flags) {
  (void)in; (void)out; (void)flags;
  if (rank < 1 || rank > 16) return NULL;
  struct fftw_plan_s* p = (struct fftw_plan_s*)calloc(1, sizeof(*p));
  p->rank = rank;
  p->sign = sign;
  p->total = 1;
  for (int a = 0; a < rank; ++a) {
    if (n[a] < 1 || !init_axis(&p->axes[a], n[a], sign)) {
      for (int b = 0; b < a; ++b) free_axis(&p->axes[b]);
      free(p);
      return NULL;
    }
    p->dims[a] = n[a];
    p->total *= (size_t)n[a];
  }
  return p;
}

void fftw_destroy_plan(fftw_plan p) {
  if (!p) return;
  for (int a = 0; a < p->rank; ++a) free_axis(&p->axes[a]);
  free(p);
}

/* Per axis: the leading dims index independent blocks; within a block the
 * axis has stride `inner` (product of the later dims), so the block is `inner`
 * interleaved sequences of length n — transformed together, the innermost
 * loop running over contiguous memory. */
void fftw_execute_dft(const fftw_plan p, fftw_complex* in_, fftw_complex* out_) {
  const size_t total = p->total;
  cplx* out = (cplx*)out_;
  if ((void*)in_ != (void*)out_) memcpy(out, in_, total * sizeof(cplx));
  /* per-thread scratch, grown on demand (plans execute concurrently under OpenMP) */
  static _Thread_local cplx* scratch = NULL;
  static _Thread_local size_t scratch_n = 0;
  if (scratch_n < total) {
    free(scratch);
    scratch = (cplx*)malloc(total * sizeof(cplx));
    scratch_n = total;
  }
  size_t inner = total;
  for (int a = 0; a < p->rank; ++a) {
    const int n = p->dims[a];
    inner /= (size_t)n;
    if (n == 1) continue;
    const size_t outer = total / ((size_t)n * inner);
    if (inner == 1) /* last axis: all rows at once, the batch loop running over rows */
      fft_batch(&p->axes[a], out, scratch, outer, 1, (size_t)n, p->sign);
    else
      for (size_t o = 0; o < outer; ++o)
        fft_batch(&p->axes[a], out + o * (size_t)n * inner, scratch, inner, inner, 1, p->sign);
  }
}
