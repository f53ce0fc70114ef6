// Probe of the tcgen05 building blocks used by the spatial coding pass:
// A from tensor memory (f16 hi/lo split), B from a no-swizzle smem core-matrix
// grid used K-major (GEMM-1) and MN-major (GEMM-2), FP32 accumulators.
//   T[p][f] = sum_o A1[p][o] D[f][o]     (M=128 pixels, N=128 filters, K=128 taps)
//   Z[p][o] = sum_f W[p][f]  D[f][o]     (M=128 pixels, N=128 taps,    K=128 filters)
// Three products per K step (hi*hi + hi*lo + lo*hi). Test tool only.
#include <cuda_runtime.h>
#include "umma.cuh"

using namespace dcsc_cuda;

__device__ __forceinline__ void bar_init(unsigned long long* b, unsigned c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(umma::smem_u32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void bar_wait(unsigned long long* b, unsigned ph) {
  asm volatile(
      "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
          umma::smem_u32(b)),
      "r"(ph)
      : "memory");
}

__global__ void __launch_bounds__(128, 1)
    probe_kernel(const float* A1, const float* Dm, const float* Wm, float sA, float sD, float* T, float* Z,
                 int variant) {
  extern __shared__ __align__(1024) unsigned char dsm[];
  __half* Dh = reinterpret_cast<__half*>(dsm);
  __half* Dl = Dh + 128 * 128;
  __shared__ uint32_t tslot;
  __shared__ __align__(8) unsigned long long bar;
  const int p = threadIdx.x, w = p >> 5;
  if (w == 0) umma::tmem_alloc<512>(&tslot);
  if (p == 0) bar_init(&bar, 1);
  // D (filters x taps) -> core (fg, tg) at (fg*16 + tg)*128 B; row = filter, 8 taps per row
  for (int i = p; i < 128 * 128; i += 128) {
    const int f = i / 128, o = i % 128;
    const int idx = (((f >> 3) * 16 + (o >> 3)) * 8 + (f & 7)) * 8 + (o & 7);
    __half hi, lo;
    umma::split2(Dm[i], sD, hi, lo);
    Dh[idx] = hi;
    Dl[idx] = lo;
  }
  umma::fence_proxy_async();
  umma::fence_before_sync();
  __syncthreads();
  umma::fence_after_sync();
  const uint32_t base = tslot;
  const uint32_t lane_off = (uint32_t)(32 * w) << 16;
  // A1 row p -> cols [0,64) hi, [64,128) lo ; W row p -> [128,192) hi, [192,256) lo
  float sW = 0.f;
  for (int f = 0; f < 128; ++f) sW = fmaxf(sW, fabsf(Wm[p * 128 + f]));
  sW = umma::pow2_scale(sW);
  for (int part = 0; part < 2; ++part) {
    const float* src = part == 0 ? A1 + p * 128 : Wm + p * 128;
    const float sc = part == 0 ? sA : sW;
    for (int c = 0; c < 4; ++c) {
      uint32_t vh[16], vl[16];
      for (int j = 0; j < 16; ++j) {
        __half h0, l0, h1, l1;
        umma::split2(src[(c * 16 + j) * 2], sc, h0, l0);
        umma::split2(src[(c * 16 + j) * 2 + 1], sc, h1, l1);
        vh[j] = umma::pack2(h0, h1);
        vl[j] = umma::pack2(l0, l1);
      }
      umma::st16(base + lane_off + part * 128 + c * 16, vh);
      umma::st16(base + lane_off + part * 128 + 64 + c * 16, vl);
    }
  }
  umma::wait_st();
  umma::fence_before_sync();
  __syncthreads();
  umma::fence_after_sync();
  if (p == 0) {
    const uint32_t dh = umma::smem_u32(Dh), dl = umma::smem_u32(Dl);
    const uint32_t id1 = umma::idesc_f16(128, 128, 0), id2 = umma::idesc_f16(128, 128, 1);
    const int nprod = variant == 1 ? 1 : 3;
    for (int j = 0; j < 8; ++j) {  // GEMM-1: K = taps, B K-major (LBO 128 along taps, SBO 2048 along filters)
      const uint64_t bh = umma::sdesc(dh + j * 256, 128, 2048), bl = umma::sdesc(dl + j * 256, 128, 2048);
      umma::mma_ts(base + 256, base + 0 + j * 8, bh, id1, j > 0);
      if (nprod == 3) {
        umma::mma_ts(base + 256, base + 0 + j * 8, bl, id1, 1);
        umma::mma_ts(base + 256, base + 64 + j * 8, bh, id1, 1);
      }
    }
    for (int j = 0; j < 8; ++j) {  // GEMM-2: K = filters, B MN-major (LBO 2048 along filters, SBO 128 along taps)
      const uint64_t bh = umma::sdesc(dh + j * 4096, 2048, 128), bl = umma::sdesc(dl + j * 4096, 2048, 128);
      umma::mma_ts(base + 384, base + 128 + j * 8, bh, id2, j > 0);
      if (nprod == 3) {
        umma::mma_ts(base + 384, base + 128 + j * 8, bl, id2, 1);
        umma::mma_ts(base + 384, base + 192 + j * 8, bh, id2, 1);
      }
    }
    umma::commit(&bar);
  }
  __syncwarp();
  bar_wait(&bar, 0);
  umma::fence_after_sync();
  for (int c = 0; c < 4; ++c) {
    uint32_t v[32];
    umma::ld32(base + lane_off + 256 + c * 32, v);
    umma::wait_ld();
    for (int j = 0; j < 32; ++j) T[p * 128 + c * 32 + j] = __uint_as_float(v[j]) / (sA * sD);
    umma::ld32(base + lane_off + 384 + c * 32, v);
    umma::wait_ld();
    for (int j = 0; j < 32; ++j) Z[p * 128 + c * 32 + j] = __uint_as_float(v[j]) / (sW * sD);
  }
  umma::fence_before_sync();
  __syncthreads();
  if (w == 0) umma::tmem_free<512>(base);
}

__global__ void __launch_bounds__(128, 1) probe_time(int reps, long long* cyc) {
  extern __shared__ __align__(1024) unsigned char dsm[];
  __half* Dh = reinterpret_cast<__half*>(dsm);
  __shared__ uint32_t tslot;
  __shared__ __align__(8) unsigned long long bar;
  const int p = threadIdx.x, w = p >> 5;
  if (w == 0) umma::tmem_alloc<512>(&tslot);
  if (p == 0) bar_init(&bar, 1);
  for (int i = p; i < 2 * 128 * 128; i += 128) Dh[i] = __float2half(0.001f * (i % 7));
  umma::fence_proxy_async();
  umma::fence_before_sync();
  __syncthreads();
  umma::fence_after_sync();
  const uint32_t base = tslot;
  if (p == 0) {
    const uint32_t dh = umma::smem_u32(Dh), dl = dh + 128 * 128 * 2;
    const uint32_t id1 = umma::idesc_f16(128, 128, 0), id2 = umma::idesc_f16(128, 128, 1);
    unsigned ph = 0;
    for (int mode = 0; mode < 2; ++mode) {
      long long t0 = clock64();
      for (int r = 0; r < reps; ++r) {
        for (int j = 0; j < 8; ++j) {
          const uint64_t bh = mode == 0 ? umma::sdesc(dh + j * 256, 128, 2048) : umma::sdesc(dh + j * 4096, 2048, 128);
          const uint64_t bl = mode == 0 ? umma::sdesc(dl + j * 256, 128, 2048) : umma::sdesc(dl + j * 4096, 2048, 128);
          const uint32_t id = mode == 0 ? id1 : id2;
          umma::mma_ts(base + 256, base + j * 8, bh, id, j > 0);
          umma::mma_ts(base + 256, base + j * 8, bl, id, 1);
          umma::mma_ts(base + 256, base + 64 + j * 8, bh, id, 1);
        }
      }
      umma::commit(&bar);
      bar_wait(&bar, ph);
      ph ^= 1;
      cyc[mode] = clock64() - t0;
    }
  }
  umma::fence_before_sync();
  __syncthreads();
  if (w == 0) umma::tmem_free<512>(base);
}

extern "C" int umma_time(int reps, long long* out) {
  long long* d;
  cudaMalloc(&d, 16);
  cudaFuncSetAttribute(probe_time, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  probe_time<<<1, 128, 65536>>>(reps, d);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(out, d, 16, cudaMemcpyDeviceToHost);
  cudaFree(d);
  return (int)e;
}

extern "C" int umma_probe(const float* hA1, const float* hD, const float* hW, float sA, float sD, float* hT,
                          float* hZ, int variant) {
  float *A1, *Dm, *Wm, *T, *Z;
  const size_t b = sizeof(float) * 128 * 128;
  cudaMalloc(&A1, b); cudaMalloc(&Dm, b); cudaMalloc(&Wm, b); cudaMalloc(&T, b); cudaMalloc(&Z, b);
  cudaMemcpy(A1, hA1, b, cudaMemcpyHostToDevice);
  cudaMemcpy(Dm, hD, b, cudaMemcpyHostToDevice);
  cudaMemcpy(Wm, hW, b, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  probe_kernel<<<1, 128, 65536>>>(A1, Dm, Wm, sA, sD, T, Z, variant);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(hT, T, b, cudaMemcpyDeviceToHost);
  cudaMemcpy(hZ, Z, b, cudaMemcpyDeviceToHost);
  cudaFree(A1); cudaFree(Dm); cudaFree(Wm); cudaFree(T); cudaFree(Z);
  return (int)e;
}
