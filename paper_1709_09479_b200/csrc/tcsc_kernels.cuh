// Multi-channel (J > 1) coding kernels: the per-frequency block solves of the
// reference's TCSC path (proj/src/tcsc.cpp). Layouts: d_hat J x K x NB
// (channel-major), x_hat J x N x NB (channel-major), lambda_hat N x J x NB,
// w_hat N x K x NB, Ginv NB x J x J (row-major per bin).
#pragma once
#include "kernels.cuh"

namespace dcsc_cuda {

constexpr int kMaxChannels = 8;

// Ginv(w) = (D_hat(w) D_hat(w)^H + I/rho)^-1 per bin (tcsc.cpp:31-55). The
// reference factors by Cholesky (or K x K Woodbury when K < J, the same
// solution); here the J x J inverse is formed once per dictionary in FP64 by
// Cholesky and column solves, then applied as a matvec every iteration.
template <class R>
__global__ void tc_factor(const cx<R>* __restrict__ dhat, cx<R>* __restrict__ ginv, int K, int J, int NB,
                          double rho) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= NB) return;
  double2 G[kMaxChannels][kMaxChannels], L[kMaxChannels][kMaxChannels];
  for (int j = 0; j < J; ++j)
    for (int i = 0; i <= j; ++i) {
      double re = 0.0, im = 0.0;
      for (int k = 0; k < K; ++k) {
        const cx<R> a = dhat[((size_t)j * K + k) * NB + b];
        const cx<R> c = dhat[((size_t)i * K + k) * NB + b];
        re += (double)a.x * c.x + (double)a.y * c.y;  // a conj(c)
        im += (double)a.y * c.x - (double)a.x * c.y;
      }
      if (i == j) re += 1.0 / rho;
      G[j][i] = make_double2(re, im);
    }
  // G = L L^H (lower)
  for (int j = 0; j < J; ++j) {
    double d = G[j][j].x;
    for (int k = 0; k < j; ++k) d -= L[j][k].x * L[j][k].x + L[j][k].y * L[j][k].y;
    const double ljj = sqrt(d);
    L[j][j] = make_double2(ljj, 0.0);
    for (int i = j + 1; i < J; ++i) {
      double re = G[i][j].x, im = G[i][j].y;
      for (int k = 0; k < j; ++k) {  // - L[i][k] conj(L[j][k])
        re -= L[i][k].x * L[j][k].x + L[i][k].y * L[j][k].y;
        im -= L[i][k].y * L[j][k].x - L[i][k].x * L[j][k].y;
      }
      L[i][j] = make_double2(re / ljj, im / ljj);
    }
  }
  // columns of G^-1: solve L y = e_c, L^H x = y
  for (int c = 0; c < J; ++c) {
    double2 y[kMaxChannels], x[kMaxChannels];
    for (int i = 0; i < J; ++i) {
      double re = (i == c) ? 1.0 : 0.0, im = 0.0;
      for (int k = 0; k < i; ++k) {
        re -= L[i][k].x * y[k].x - L[i][k].y * y[k].y;
        im -= L[i][k].x * y[k].y + L[i][k].y * y[k].x;
      }
      y[i] = make_double2(re / L[i][i].x, im / L[i][i].x);
    }
    for (int i = J - 1; i >= 0; --i) {
      double re = y[i].x, im = y[i].y;
      for (int k = i + 1; k < J; ++k) {  // - conj(L[k][i]) x[k]
        re -= L[k][i].x * x[k].x + L[k][i].y * x[k].y;
        im -= L[k][i].x * x[k].y - L[k][i].y * x[k].x;
      }
      x[i] = make_double2(re / L[i][i].x, im / L[i][i].x);
    }
    for (int i = 0; i < J; ++i) ginv[((size_t)b * J + i) * J + c] = mk<cx<R>>(R(x[i].x), R(x[i].y));
  }
}

// lambda_hat_j(w) = sum_i Ginv_ji(w) r_i(w), r_j = sum_k d_hat_jk w_hat_k - x_hat_j / rho
// (tcsc.cpp:68-88). One thread per (bin, image); images whose ADMM stopped keep
// the lambda_hat of their last iteration (coding.cpp:287-291). kw = 0: w_hat = 0.
template <class R, int JT = 0>
__global__ void tc_lambda(const cx<R>* __restrict__ what, const cx<R>* __restrict__ dhat,
                          const cx<R>* __restrict__ ginv, const cx<R>* __restrict__ xhat, size_t xstride,
                          cx<R>* __restrict__ lamhat, const int* conv, int K, int kw, int Jr, int NB, R inv_rho) {
  using C = cx<R>;
  constexpr int JM = JT > 0 ? JT : kMaxChannels;  // register arrays sized for the compile-time count
  const int J = JT > 0 ? JT : Jr;
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  const int n = blockIdx.y;
  if (b >= NB || (conv && conv[n])) return;
  C r[JM];
#pragma unroll
  for (int j = 0; j < JM; ++j) r[j] = mk<C>(R(0), R(0));
#pragma unroll 4
  for (int k = 0; k < kw; ++k) {
    const C w = what[((size_t)n * K + k) * NB + b];
#pragma unroll
    for (int j = 0; j < JM; ++j)
      if (j < J) r[j] = cadd(r[j], cmul(dhat[((size_t)j * K + k) * NB + b], w));
  }
#pragma unroll
  for (int j = 0; j < JM; ++j)
    if (j < J) {
      const C xv = xhat[(size_t)j * xstride + (size_t)n * NB + b];
      r[j] = mk<C>(r[j].x - xv.x * inv_rho, r[j].y - xv.y * inv_rho);
    }
  const C* g = ginv + (size_t)b * J * J;
#pragma unroll
  for (int j = 0; j < JM; ++j) {
    if (j >= J) break;
    C l = mk<C>(R(0), R(0));
#pragma unroll
    for (int i = 0; i < JM; ++i)
      if (i < J) l = cadd(l, cmul(g[j * J + i], r[i]));
    lamhat[((size_t)n * J + j) * NB + b] = l;
  }
}

// Objective of J-channel images from w_hat = z_hat (N x K x NB): data_n =
// 1/2 sum_j ||sum_k d_k,j * z_k - x_j||^2 by Parseval on half spectra
// (objective.cpp:39-81); l1 from the pass's per-CTA |z| sums. One CTA/image.
template <class R>
__global__ void tc_objective(const cx<R>* __restrict__ what, const cx<R>* __restrict__ dhat,
                             const cx<R>* __restrict__ xhat, size_t xstride, const double* __restrict__ sums,
                             int slots, int K, int J, int NB, int Wh, double invD, double beta, double* data,
                             double* l1) {
  using C = cx<R>;
  __shared__ double red[32];
  const int n = blockIdx.x;
  double v = 0.0;
  for (int b = threadIdx.x; b < NB; b += blockDim.x) {
    for (int j = 0; j < J; ++j) {
      C acc = mk<C>(R(0), R(0));
      for (int k = 0; k < K; ++k)
        acc = cadd(acc, cmul(dhat[((size_t)j * K + k) * NB + b], what[((size_t)n * K + k) * NB + b]));
      const C x = xhat[(size_t)j * xstride + (size_t)n * NB + b];
      const double rr = (double)acc.x - (double)x.x, ri = (double)acc.y - (double)x.y;
      v += bin_weight(b, Wh) * (rr * rr + ri * ri);
    }
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

// Stateless-op helpers (coding.hpp:45-66). t_hat_k = sum_j conj(d_hat_jk)
// lambda_hat_j for one image (D^T lambda spectra, K planes).
template <class R>
__global__ void adjoint_spectra(const cx<R>* __restrict__ dhat, const cx<R>* __restrict__ lamhat,
                                cx<R>* __restrict__ out, int K, int J, int NB) {
  using C = cx<R>;
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  const int k = blockIdx.y;
  if (b >= NB) return;
  C t = mk<C>(R(0), R(0));
  for (int j = 0; j < J; ++j)
    t = cadd(t, cmulc(dhat[((size_t)j * K + k) * NB + b], lamhat[(size_t)j * NB + b]));
  out[(size_t)k * NB + b] = t;
}

// Single-channel lambda_hat = (sum_k d_hat_k w_hat_k - x_hat / rho) / sigma for
// one image from its w_hat planes (lambda_from_w, coding.cpp:25-37).
template <class R>
__global__ void lambda_from_w(const cx<R>* __restrict__ what, const cx<R>* __restrict__ dhat,
                              const cx<R>* __restrict__ xhat, const R* __restrict__ sigma, cx<R>* __restrict__ lamhat,
                              int K, int NB, R inv_rho) {
  using C = cx<R>;
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= NB) return;
  C acc = mk<C>(R(0), R(0));
  for (int k = 0; k < K; ++k) acc = cadd(acc, cmul(dhat[(size_t)k * NB + b], what[(size_t)k * NB + b]));
  const C xv = xhat[b];
  const R s = sigma[b];
  lamhat[b] = mk<C>((acc.x - xv.x * inv_rho) / s, (acc.y - xv.y * inv_rho) / s);
}

// Reconstruction spectrum y_n,j = sum_k d_hat_jk z_hat_nk (objective.cpp:39-57 in
// the Fourier basis): J = 1 sums the coding pass's G group partials (fixed
// order), J > 1 contracts the stored z_hat planes. out: N x J x NB.
template <class R>
__global__ void recon_spectrum(const cx<R>* __restrict__ part, const cx<R>* __restrict__ what,
                               const cx<R>* __restrict__ dhat, cx<R>* __restrict__ out, int J, int K, int G, int NB) {
  using C = cx<R>;
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  const int n = blockIdx.y;
  if (b >= NB) return;
  if (J == 1) {
    C acc = part[((size_t)n * G) * NB + b];
    for (int g = 1; g < G; ++g) acc = cadd(acc, part[((size_t)n * G + g) * NB + b]);
    out[(size_t)n * NB + b] = acc;
    return;
  }
  for (int j = 0; j < J; ++j) {
    C acc = mk<C>(R(0), R(0));
    for (int k = 0; k < K; ++k)
      acc = cadd(acc, cmul(dhat[((size_t)j * K + k) * NB + b], what[((size_t)n * K + k) * NB + b]));
    out[((size_t)n * J + j) * NB + b] = acc;
  }
}

}  // namespace dcsc_cuda
