// K3: one recurrent decode step for a batch of single tokens (memory-bound).
// Semantics of one iteration of the reference row recurrence (kernels.py:100-104):
//   S <- gamma S + k^T v ;  o = q S
// Every (b, h) state [dk][dv] fp32 is read once and written once per step with
// 128-bit coalesced accesses; all of a thread's state loads are issued before
// any is consumed so each SM keeps enough bytes in flight to saturate HBM.
// Small batches (few (b, h) states): the dv columns of a state are split over blockIdx.y
// slices -- columns of o are independent, so no cross-CTA reduction -- to fill the SMs.
#include <algorithm>

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
                   int H, int dk, int dv, int dvs) {
  // this CTA: columns [c0, c0 + dvs) of state bh (dvs = dv unless the launch split the columns)
  extern __shared__ float sm[];
  float* qs = sm;            // [dk]
  float* ks = qs + dk;       // [dk]
  float* vs = ks + dk;       // [dvs]
  float* part = vs + dvs;    // [rg][dvs]

  const int bh = blockIdx.x;
  const int tid = threadIdx.x;
  const int c0 = blockIdx.y * dvs;
  const int ncol = min(dvs, dv - c0);
  const float g = gpow(log2g[bh % H], 1.f);
  for (int i = tid; i < dk; i += NT) {
    qs[i] = to_f32(q[(size_t)bh * dk + i]);
    ks[i] = to_f32(k[(size_t)bh * dk + i]);
  }
  for (int j = tid; j < ncol; j += NT) vs[j] = to_f32(v[(size_t)bh * dv + c0 + j]);
  __syncthreads();

  const int nvec = ncol / VEC;                   // vectors per state row slice
  const int nvs = dvs / VEC;                     // ... of a full slice (sets the thread layout)
  const int ct = nvs < NT ? nvs : NT;            // threads across columns
  const int rg = NT / ct;                        // row groups
  const int my_rg = tid / ct;
  float* st = state + (size_t)bh * dk * dv + c0;

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
    for (int e = 0; e < VEC; ++e) part[my_rg * dvs + cv * VEC + e] = acc[e];
  }
  __syncthreads();
  for (int j = tid; j < ncol; j += NT) {
    float sacc = 0.f;
    for (int r = 0; r < rg; ++r) sacc += part[r * dvs + j];
    o[(size_t)bh * dv + c0 + j] = from_f32<T>(sacc);
  }
}

template <typename T>
cudaError_t launch_t(const void* q, const void* k, const void* v, void* o, float* state,
                     const float* log2g, const ShapeArgs& s, cudaStream_t stream) {
  const bool vec4 = (s.dv % 4 == 0) && ((reinterpret_cast<uintptr_t>(state) & 15) == 0);
  // split the columns when (b, h) states alone leave SMs idle: about two CTAs per SM, slices of
  // at least 32 columns (one 128-byte row segment per slice)
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t bhn = s.B * s.H;
  int64_t slices = (2 * sms + bhn - 1) / bhn;
  slices = std::max<int64_t>(1, std::min<int64_t>(slices, s.dv / 32));
  int dvs = (int)((s.dv + slices - 1) / slices);
  if (vec4) dvs = (dvs + 3) / 4 * 4;
  slices = (s.dv + dvs - 1) / dvs;
  const int nvec = vec4 ? dvs / 4 : dvs;
  const int ct = nvec < NT ? nvec : NT;
  const int rg = NT / ct;
  const size_t smem = sizeof(float) * (2 * s.dk + dvs + (size_t)rg * dvs);
  if (smem > 227 * 1024) return cudaErrorNotSupported;
  const dim3 grid((unsigned)bhn, (unsigned)slices);
  if (vec4) {
    auto kern = decode_step_kernel<T, 4>;
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<grid, NT, smem, stream>>>((const T*)q, (const T*)k, (const T*)v, (T*)o, state, log2g,
                                     (int)s.H, (int)s.dk, (int)s.dv, dvs);
  } else {
    auto kern = decode_step_kernel<T, 1>;
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<grid, NT, smem, stream>>>((const T*)q, (const T*)k, (const T*)v, (T*)o, state, log2g,
                                     (int)s.H, (int)s.dk, (int)s.dv, dvs);
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
