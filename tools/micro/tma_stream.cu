// Microbenchmark: per-SM TMA streaming throughput with a STAGES-deep ring of 48 KiB stages
// (the configs[1] prefill's Q/K/V chunk), consumer releasing each stage immediately.
// usage: tma_stream <ctas> <stages>
#include <cstdio>
#include <cstdlib>
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include "../../paper_2501_02573_b200/csrc/sm100.cuh"
using namespace linattn::sm100;

constexpr int CHUNK = 64, D = 128, STAGE_BYTES = 3 * CHUNK * D * 2;

template <int STAGES>
__global__ void __launch_bounds__(64, 1) stream(const __grid_constant__ CUtensorMap tm, int nchunks,
                                                unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    fence_barrier_init();
  }
  __syncthreads();
  const int bh = blockIdx.x;
  unsigned long long t0 = clock64();
  if (warp == 0 && lane == 0) {
    for (int c = 0; c < nchunks; ++c) {
      const int s = c % STAGES;
      mbar_wait(&empty[s], ((c / STAGES) & 1) ^ 1);
      mbar_arrive_expect_tx(&full[s], STAGE_BYTES);
      for (int b = 0; b < 6; ++b)   // 6 boxes of 64 x 64 bf16 (Q, K, V chunks of a 128-wide head)
        tma_load_3d(smem + s * STAGE_BYTES + b * 8192, &tm, &full[s], (b % 2) * 64, c * CHUNK, bh * 3 + b / 2);
    }
  } else if (warp == 1 && lane == 0) {
    for (int c = 0; c < nchunks; ++c) {
      const int s = c % STAGES;
      mbar_wait(&full[s], (c / STAGES) & 1);
      mbar_arrive(&empty[s]);
    }
    out[blockIdx.x] = clock64() - t0;
  }
}

int main(int argc, char** argv) {
  const int ctas = argc > 1 ? atoi(argv[1]) : 148;
  const int stages = argc > 2 ? atoi(argv[2]) : 4;
  const int N = 8192, nchunks = N / CHUNK;
  const size_t elems = (size_t)ctas * 3 * N * D;
  void* buf;
  cudaMalloc(&buf, elems * 2);
  cudaMemset(buf, 0, elems * 2);
  unsigned long long* out;
  cudaMalloc(&out, ctas * 8);
  void* fnp = nullptr;
  cudaDriverEntryPointQueryResult qr;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &qr);
  auto fn = (PFN_cuTensorMapEncodeTiled_v12000)fnp;
  CUtensorMap tm;
  cuuint64_t dims[3] = {D, (cuuint64_t)N, (cuuint64_t)ctas * 3};
  cuuint64_t strides[2] = {D * 2, (cuuint64_t)N * D * 2};
  cuuint32_t box[3] = {64, 64, 1}, es[3] = {1, 1, 1};
  fn(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const size_t smem = (size_t)stages * STAGE_BYTES + 1024;
  auto run = [&]() {
    switch (stages) {
      case 2: cudaFuncSetAttribute(stream<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
              stream<2><<<ctas, 64, smem>>>(tm, nchunks, out); break;
      case 3: cudaFuncSetAttribute(stream<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
              stream<3><<<ctas, 64, smem>>>(tm, nchunks, out); break;
      default: cudaFuncSetAttribute(stream<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
              stream<4><<<ctas, 64, smem>>>(tm, nchunks, out); break;
    }
  };
  run();
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int i = 0; i < 5; ++i) run();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  ms /= 5;
  const double bytes = (double)ctas * nchunks * STAGE_BYTES;
  printf("ctas=%d stages=%d: %.3f ms, %.0f GB/s total, %.1f GB/s per CTA (%s)\n", ctas, stages, ms,
         bytes / ms / 1e6, bytes / ms / 1e6 / ctas, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
