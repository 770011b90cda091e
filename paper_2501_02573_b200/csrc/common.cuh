// Shared device helpers and the internal launcher interface.
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include "../../include/linattn_b200.h"

namespace linattn {

// gamma^n from log2(gamma): exact 1 at n == 0 (gamma^0 == 1 even for gamma == 0,
// reference masks.py:22 and masks.py:44-49); log2g == -inf gives 0 for n > 0.
__device__ __forceinline__ float gpow(float log2g, float n) {
  return n == 0.f ? 1.f : exp2f(n * log2g);
}

// Fast variant (ex2.approx) for the bf16 tensor-core path.
__device__ __forceinline__ float gpow_fast(float log2g, float n) {
  float r;
  float x = n * log2g;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return n == 0.f ? 1.f : r;
}

template <typename T> __device__ __forceinline__ float to_f32(T x);
template <> __device__ __forceinline__ float to_f32<float>(float x) { return x; }
template <> __device__ __forceinline__ float to_f32<__nv_bfloat16>(__nv_bfloat16 x) {
  return __bfloat162float(x);
}
template <typename T> __device__ __forceinline__ T from_f32(float x);
template <> __device__ __forceinline__ float from_f32<float>(float x) { return x; }
template <> __device__ __forceinline__ __nv_bfloat16 from_f32<__nv_bfloat16>(float x) {
  return __float2bfloat16_rn(x);
}

// ---- internal launchers (return cudaError_t of the launch) -------------------
struct ShapeArgs {
  int64_t B, H, N, dk, dv;
};

cudaError_t launch_prefill_simt(const void* q, const void* k, const void* v, void* o,
                                const float* log2g, const float* s_in, float* s_out,
                                const ShapeArgs& s, int dtype, bool state_only,
                                cudaStream_t stream);

// Returns cudaErrorNotSupported when the shape is outside the TC kernel's envelope.
cudaError_t launch_prefill_tc(const void* q, const void* k, const void* v, void* o,
                              const float* log2g, const float* s_in, float* s_out,
                              const ShapeArgs& s, bool state_only, cudaStream_t stream);
bool tc_supported(const ShapeArgs& s, int dtype);
void set_trace(void* buf);  // debug only: per-chunk clock64 trace of CTA (0,0), nullptr = off

cudaError_t launch_decode_step(const void* q, const void* k, const void* v, void* o,
                               float* state, const float* log2g, const ShapeArgs& s,
                               int dtype, cudaStream_t stream);

cudaError_t launch_prefix_combine(const float* gathered, float* s_in, const int64_t* seg_lens,
                                  int P, int rank, const float* log2g, const ShapeArgs& s,
                                  cudaStream_t stream);

void count_launch();

}  // namespace linattn
