// K3: one recurrent decode step for a batch of single tokens (memory-bound).
// Semantics of one iteration of the reference row recurrence (kernels.py:100-104):
//   S <- gamma S + k^T v ;  o = q S
// Every (b, h) state [dk][dv] fp32 is read once and written once per step with
// 128-bit coalesced accesses; all of a thread's state loads are issued before
// any is consumed so each SM keeps enough bytes in flight to saturate HBM.
#include "common.cuh"

namespace linattn {
namespace {

// Block size / rows per batch of in-flight loads: swept on B200 (configs[3]): 128 x 8 keeps the
// most 16-byte loads in flight per SM (small blocks -> more resident CTAs): 190 -> 168 us/step.
#ifndef DEC_NT
#define DEC_NT 128
#endif
#ifndef DEC_RB
#define DEC_RB 8
#endif
constexpr int NT = DEC_NT;
constexpr int RB = DEC_RB;  // state rows per thread per batch of in-flight loads

template <typename T, int VEC>
__global__ void __launch_bounds__(NT)
decode_step_kernel(const T* __restrict__ q, const T* __restrict__ k, const T* __restrict__ v,
                   T* __restrict__ o, float* __restrict__ state, const float* __restrict__ log2g,
                   int H, int dk, int dv) {
  extern __shared__ float sm[];
  float* qs = sm;            // [dk]
  float* ks = qs + dk;       // [dk]
  float* vs = ks + dk;       // [dv]
  float* part = vs + dv;     // [rg][dv]

  const int bh = blockIdx.x;
  const int tid = threadIdx.x;
  const float g = gpow(log2g[bh % H], 1.f);
  for (int i = tid; i < dk; i += NT) {
    qs[i] = to_f32(q[(size_t)bh * dk + i]);
    ks[i] = to_f32(k[(size_t)bh * dk + i]);
  }
  for (int j = tid; j < dv; j += NT) vs[j] = to_f32(v[(size_t)bh * dv + j]);
  __syncthreads();

  const int nvec = dv / VEC;                     // vectors per state row
  const int ct = nvec < NT ? nvec : NT;          // threads across columns
  const int rg = NT / ct;                        // row groups
  const int my_rg = tid / ct;
  float* st = state + (size_t)bh * dk * dv;

  if (my_rg < rg) for (int cv = tid % ct; cv < nvec; cv += ct) {
    float acc[VEC];
#pragma unroll
    for (int e = 0; e < VEC; ++e) acc[e] = 0.f;
    float vv[VEC];
#pragma unroll
    for (int e = 0; e < VEC; ++e) vv[e] = vs[cv * VEC + e];
    {
      for (int r0 = my_rg; r0 < dk; r0 += rg * RB) {
        float x[RB][VEC];
#pragma unroll
        for (int u = 0; u < RB; ++u) {
          const int r = r0 + u * rg;
          if (r < dk) {
            if constexpr (VEC == 4) {
              const float4 t4 = *reinterpret_cast<const float4*>(st + (size_t)r * dv + cv * 4);
              x[u][0] = t4.x; x[u][1] = t4.y; x[u][2] = t4.z; x[u][3] = t4.w;
            } else {
              x[u][0] = st[(size_t)r * dv + cv];
            }
          }
        }
#pragma unroll
        for (int u = 0; u < RB; ++u) {
          const int r = r0 + u * rg;
          if (r < dk) {
            const float kr = ks[r], qr = qs[r];
#pragma unroll
            for (int e = 0; e < VEC; ++e) {
              x[u][e] = fmaf(g, x[u][e], kr * vv[e]);
              acc[e] = fmaf(qr, x[u][e], acc[e]);
            }
            if constexpr (VEC == 4) {
              *reinterpret_cast<float4*>(st + (size_t)r * dv + cv * 4) =
                  make_float4(x[u][0], x[u][1], x[u][2], x[u][3]);
            } else {
              st[(size_t)r * dv + cv] = x[u][0];
            }
          }
        }
      }
    }
#pragma unroll
    for (int e = 0; e < VEC; ++e) part[my_rg * dv + cv * VEC + e] = acc[e];
  }
  __syncthreads();
  for (int j = tid; j < dv; j += NT) {
    float sacc = 0.f;
    for (int r = 0; r < rg; ++r) sacc += part[r * dv + j];
    o[(size_t)bh * dv + j] = from_f32<T>(sacc);
  }
}

template <typename T>
cudaError_t launch_t(const void* q, const void* k, const void* v, void* o, float* state,
                     const float* log2g, const ShapeArgs& s, cudaStream_t stream) {
  const bool vec4 = (s.dv % 4 == 0) && ((reinterpret_cast<uintptr_t>(state) & 15) == 0);
  const int nvec = (int)(vec4 ? s.dv / 4 : s.dv);
  const int ct = nvec < NT ? nvec : NT;
  const int rg = NT / ct;
  const size_t smem = sizeof(float) * (2 * s.dk + s.dv + (size_t)rg * s.dv);
  if (smem > 227 * 1024) return cudaErrorNotSupported;
  const unsigned grid = (unsigned)(s.B * s.H);
  if (vec4) {
    auto kern = decode_step_kernel<T, 4>;
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<grid, NT, smem, stream>>>((const T*)q, (const T*)k, (const T*)v, (T*)o, state, log2g,
                                     (int)s.H, (int)s.dk, (int)s.dv);
  } else {
    auto kern = decode_step_kernel<T, 1>;
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<grid, NT, smem, stream>>>((const T*)q, (const T*)k, (const T*)v, (T*)o, state, log2g,
                                     (int)s.H, (int)s.dk, (int)s.dv);
  }
  count_launch();
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_decode_step(const void* q, const void* k, const void* v, void* o,
                               float* state, const float* log2g, const ShapeArgs& s,
                               int dtype, cudaStream_t stream) {
  if (dtype == LINATTN_BF16)
    return launch_t<__nv_bfloat16>(q, k, v, o, state, log2g, s, stream);
  return launch_t<float>(q, k, v, o, state, log2g, s, stream);
}

}  // namespace linattn
