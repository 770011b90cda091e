// Microbenchmark: tcgen05.ld / tcgen05.st throughput per SM vs number of warps.
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2501_02573_b200/csrc/sm100.cuh"
using namespace linattn::sm100;

template <int MODE>
__global__ void bench(unsigned long long* out, int iters) {
  __shared__ uint32_t slot;
  const uint32_t warp = threadIdx.x / 32;
  if (warp == 0) tmem_alloc<512>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = slot;
  const uint32_t sub = warp % 4;
  const uint32_t colg = warp / 4;       // column group of this warp
  const uint32_t ta = tbase + ((sub * 32) << 16) + colg * 128;
  float acc = 0.f;
  __syncthreads();
  unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float v[32];
      if (MODE == 0) {
        tmem_ld32(ta + j * 32, v);
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 32; ++i) acc += v[i];
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = acc + i;
        tmem_st32(ta + j * 32, v);
      }
    }
    if (MODE == 1) tmem_wait_st();
  }
  __syncthreads();
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  if (acc == 12345.f) out[1000] = 1;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc<512>(tbase);
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 8192);
  const int iters = 1000;
  for (int mode = 0; mode < 2; ++mode)
    for (int warps : {4, 8, 16}) {
      if (mode == 0) bench<0><<<1, warps * 32>>>(d, iters); else bench<1><<<1, warps * 32>>>(d, iters);
      cudaDeviceSynchronize();
      if (mode == 0) bench<0><<<1, warps * 32>>>(d, iters); else bench<1><<<1, warps * 32>>>(d, iters);
      unsigned long long cyc;
      cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
      const double bytes = (double)warps * 32 * 128 * 4 * iters;   // 128 fp32 per thread per iter
      printf("%s warps=%2d  %.1f B/cycle/SM  (err=%s)\n", mode ? "st" : "ld", warps, bytes / cyc,
             cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
