/* FFTW3-API shim (TEST INFRASTRUCTURE ONLY — never linked into the product).
 *
 * Restates the algorithm FFTW3 computes for the subset the reference uses
 * (proj/src/spectral.cpp:16-47 plan cache, :59-68 forward, :76-98 inverse):
 * an unnormalised, out-of-place, row-major N-D complex DFT with sign -1
 * (FFTW_FORWARD) or +1 (FFTW_BACKWARD). FFTW itself is not in this image and
 * its version is unpinned by the reference (proj/CMakeLists.txt:16-17).
 *
 * Algorithm: per axis, a recursive mixed-radix decimation-in-time
 * Cooley-Tukey transform (radix 4, 2, 3, 5, then any remaining prime by a
 * direct O(p^2) butterfly). Twiddles are tabulated once per plan from
 * sin/cos evaluated directly in double (no recurrences), so the transform is
 * accurate to a few ulps * log(n). Multi-dimensional transforms apply the 1-D
 * transform along each axis in turn. Executing a plan is thread-safe (all
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

typedef struct {
  int n;
  int nfac;
  int fac[64];
  cplx* w; /* w[j] = exp(sign * 2 pi i j / n) */
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

static void factorize(axis_plan* a) {
  int n = a->n;
  a->nfac = 0;
  while (n % 4 == 0) { a->fac[a->nfac++] = 4; n /= 4; }
  while (n % 2 == 0) { a->fac[a->nfac++] = 2; n /= 2; }
  for (int p = 3; n > 1; p += 2) {
    while (n % p == 0) { a->fac[a->nfac++] = p; n /= p; }
  }
  if (a->nfac == 0) a->fac[a->nfac++] = 1;
}

static void init_axis(axis_plan* a, int n, int sign) {
  a->n = n;
  factorize(a);
  a->w = (cplx*)malloc((size_t)n * sizeof(cplx));
  const double two_pi = 6.283185307179586476925286766559;
  for (int j = 0; j < n; ++j) {
    /* reduce the angle to the first octant-friendly form for accuracy */
    const double ang = two_pi * (double)j / (double)n;
    a->w[j].re = cos(ang);
    a->w[j].im = (double)sign * sin(ang);
  }
  /* exact values at the quarter points */
  if (n % 4 == 0) {
    a->w[0].re = 1; a->w[0].im = 0;
    a->w[n / 4].re = 0; a->w[n / 4].im = (double)sign;
    a->w[n / 2].re = -1; a->w[n / 2].im = 0;
    a->w[3 * n / 4].re = 0; a->w[3 * n / 4].im = -(double)sign;
  } else if (n % 2 == 0) {
    a->w[n / 2].re = -1; a->w[n / 2].im = 0;
  }
}

static inline cplx cmul(cplx a, cplx b) {
  cplx r = {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re};
  return r;
}

/* out[0..n) = DFT_n(in[0], in[is], ...), wst = N/n indexes the axis table. */
static void fft_rec(const cplx* in, size_t is, cplx* out, int n, const int* fac,
                    const axis_plan* ap, int wst, int sign) {
  if (n == 1) {
    out[0] = in[0];
    return;
  }
  const int r = fac[0];
  const int m = n / r;
  const int N = ap->n;
  const cplx* w = ap->w;
  for (int q = 0; q < r; ++q) fft_rec(in + (size_t)q * is, is * (size_t)r, out + (size_t)q * m, m, fac + 1, ap, wst * r, sign);

  if (r == 2) {
    for (int k = 0; k < m; ++k) {
      const cplx a = out[k];
      const cplx b = cmul(out[m + k], w[(size_t)k * wst % N]);
      out[k].re = a.re + b.re; out[k].im = a.im + b.im;
      out[m + k].re = a.re - b.re; out[m + k].im = a.im - b.im;
    }
    return;
  }
  if (r == 4) {
    const double s = (double)sign; /* W_4 = s*i */
    for (int k = 0; k < m; ++k) {
      const cplx x0 = out[k];
      const cplx x1 = cmul(out[m + k], w[(size_t)k * wst % N]);
      const cplx x2 = cmul(out[2 * m + k], w[(size_t)2 * k * wst % N]);
      const cplx x3 = cmul(out[3 * m + k], w[(size_t)3 * k * wst % N]);
      const cplx t0 = {x0.re + x2.re, x0.im + x2.im};
      const cplx t1 = {x0.re - x2.re, x0.im - x2.im};
      const cplx t2 = {x1.re + x3.re, x1.im + x3.im};
      const cplx t3 = {x1.re - x3.re, x1.im - x3.im};
      /* s*i*t3 */
      const cplx it3 = {-s * t3.im, s * t3.re};
      out[k].re = t0.re + t2.re; out[k].im = t0.im + t2.im;
      out[m + k].re = t1.re + it3.re; out[m + k].im = t1.im + it3.im;
      out[2 * m + k].re = t0.re - t2.re; out[2 * m + k].im = t0.im - t2.im;
      out[3 * m + k].re = t1.re - it3.re; out[3 * m + k].im = t1.im - it3.im;
    }
    return;
  }
  /* generic radix r: y_q = out[q m + k] W_n^{qk}; out[k + s m] = sum_q y_q W_r^{qs} */
  cplx y[64];
  cplx acc[64];
  for (int k = 0; k < m; ++k) {
    for (int q = 0; q < r; ++q) y[q] = q == 0 ? out[k] : cmul(out[(size_t)q * m + k], w[(size_t)q * k * wst % N]);
    for (int s2 = 0; s2 < r; ++s2) {
      cplx a = y[0];
      for (int q = 1; q < r; ++q) {
        const cplx t = cmul(y[q], w[((size_t)q * s2 % r) * (size_t)m * wst % N]);
        a.re += t.re; a.im += t.im;
      }
      acc[s2] = a;
    }
    for (int s2 = 0; s2 < r; ++s2) out[k + (size_t)s2 * m] = acc[s2];
  }
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
    if (n[a] < 1) { free(p); return NULL; }
    p->dims[a] = n[a];
    p->total *= (size_t)n[a];
    init_axis(&p->axes[a], n[a], sign);
    for (int f = 0; f < p->axes[a].nfac; ++f)
      if (p->axes[a].fac[f] > 64) { /* primes above 64 are not needed by the reference sizes */
        free(p); return NULL;
      }
  }
  return p;
}

void fftw_destroy_plan(fftw_plan p) {
  if (!p) return;
  for (int a = 0; a < p->rank; ++a) free(p->axes[a].w);
  free(p);
}

void fftw_execute_dft(const fftw_plan p, fftw_complex* in_, fftw_complex* out_) {
  const size_t total = p->total;
  cplx* out = (cplx*)out_;
  if ((void*)in_ != (void*)out_) memcpy(out, in_, total * sizeof(cplx));
  size_t maxn = 1;
  for (int a = 0; a < p->rank; ++a) if ((size_t)p->dims[a] > maxn) maxn = (size_t)p->dims[a];
  cplx* line = (cplx*)malloc(2 * maxn * sizeof(cplx));
  cplx* res = line + maxn;
  size_t inner = total; /* product of dims after axis a */
  for (int a = 0; a < p->rank; ++a) {
    const int n = p->dims[a];
    inner /= (size_t)n;
    const size_t outer = total / ((size_t)n * inner);
    const axis_plan* ap = &p->axes[a];
    if (n == 1) continue;
    for (size_t o = 0; o < outer; ++o) {
      for (size_t i = 0; i < inner; ++i) {
        cplx* base = out + o * (size_t)n * inner + i;
        if (inner == 1) {
          fft_rec(base, 1, res, n, ap->fac, ap, 1, p->sign);
          memcpy(base, res, (size_t)n * sizeof(cplx));
        } else {
          for (int j = 0; j < n; ++j) line[j] = base[(size_t)j * inner];
          fft_rec(line, 1, res, n, ap->fac, ap, 1, p->sign);
          for (int j = 0; j < n; ++j) base[(size_t)j * inner] = res[j];
        }
      }
    }
  }
  free(line);
}
