// Shared device helpers: complex arithmetic on float2/double2 and
// block-level FP64 reductions.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

namespace dcsc_cuda {

template <class R> struct CT;
template <> struct CT<float> { using type = float2; };
template <> struct CT<double> { using type = double2; };
template <class R> using cx = typename CT<R>::type;

template <class C> __host__ __device__ __forceinline__ C mk(decltype(C::x) a, decltype(C::x) b) {
  C r; r.x = a; r.y = b; return r;
}
template <class C> __device__ __forceinline__ C cadd(C a, C b) { return mk<C>(a.x + b.x, a.y + b.y); }
template <class C> __device__ __forceinline__ C csub(C a, C b) { return mk<C>(a.x - b.x, a.y - b.y); }
template <class C> __device__ __forceinline__ C cmul(C a, C b) {
  return mk<C>(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
// conj(a) * b
template <class C> __device__ __forceinline__ C cmulc(C a, C b) {
  return mk<C>(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x);
}
template <class C> __device__ __forceinline__ C cconj(C a) { return mk<C>(a.x, -a.y); }
template <class C> __device__ __forceinline__ C cscale(C a, decltype(C::x) s) { return mk<C>(a.x * s, a.y * s); }
// multiply by -i (forward) / +i (inverse)
template <bool INV, class C> __device__ __forceinline__ C mul_mi(C a) {
  return INV ? mk<C>(-a.y, a.x) : mk<C>(a.y, -a.x);
}

// Block-wide sum of NV doubles held per thread; result valid in thread 0.
template <int T, int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV], double* scratch /* >= NV*T/32 */) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    double s = v[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) scratch[i * (T / 32) + warp] = s;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      double s = 0.0;
      for (int w = 0; w < T / 32; ++w) s += scratch[i * (T / 32) + w];
      v[i] = s;
    }
  }
  __syncthreads();
}

__device__ __forceinline__ double block_max(double v, double* scratch, int T) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  if (lane == 0) scratch[warp] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = 0.0;
    for (int w = 0; w < T / 32; ++w) m = fmax(m, scratch[w]);
    v = m;
  }
  __syncthreads();
  return v;
}

}  // namespace dcsc_cuda
