// K5 (combine half): exclusive gamma-weighted prefix of gathered segment end states.
//   s_in = sum_{q < rank} gamma^(sum_{q < m < rank} L_m) * S_q
// evaluated as the scan acc <- gamma^(L_q) acc + S_q over q = 0 .. rank-1 (the
// recursion cross-term weights of the reference, kernels.py:185-189, applied
// across sequence segments).  Elementwise over [B, H, dk, dv]; float4 accesses.
// Every scan here batches its loads kLoads entries ahead: with one load in flight per thread
// these small kernels were DRAM-latency bound (ncu: 8 us for 8-15 MB).
#include <algorithm>

#include "common.cuh"

namespace linattn {
namespace {

constexpr int MAXP = 64;
constexpr int kLoads = 8;          // entries loaded ahead per thread
struct SegLens {
  long long len[MAXP];   // segment lengths in tokens (int64: exact past 2^24)
};

__global__ void prefix_combine_kernel(const float4* __restrict__ gathered, float4* __restrict__ s_in,
                                      SegLens lens, int rank, const float* __restrict__ log2g,
                                      int H, int64_t per_head4, int64_t per_rank4) {
  pdl_wait();
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= per_rank4) return;
  const int h = (int)((idx / per_head4) % H);
  const float lg = log2g[h];
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int p0 = 0; p0 < rank; p0 += kLoads) {
    float4 x[kLoads];
#pragma unroll
    for (int j = 0; j < kLoads; ++j)
      if (p0 + j < rank) x[j] = gathered[(int64_t)(p0 + j) * per_rank4 + idx];
#pragma unroll
    for (int j = 0; j < kLoads; ++j) {
      if (p0 + j >= rank) break;
      const float c = gpow_n(lg, lens.len[p0 + j]);
      acc.x = fmaf(c, acc.x, x[j].x);
      acc.y = fmaf(c, acc.y, x[j].y);
      acc.z = fmaf(c, acc.z, x[j].z);
      acc.w = fmaf(c, acc.w, x[j].w);
    }
  }
  s_in[idx] = acc;
}

__global__ void prefix_combine_kernel_scalar(const float* __restrict__ gathered, float* __restrict__ s_in,
                                             SegLens lens, int rank, const float* __restrict__ log2g,
                                             int H, int64_t per_head, int64_t per_rank) {
  pdl_wait();
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= per_rank) return;
  const int h = (int)((idx / per_head) % H);
  const float lg = log2g[h];
  float acc = 0.f;
  for (int p0 = 0; p0 < rank; p0 += kLoads) {
    float x[kLoads];
#pragma unroll
    for (int j = 0; j < kLoads; ++j)
      if (p0 + j < rank) x[j] = gathered[(int64_t)(p0 + j) * per_rank + idx];
#pragma unroll
    for (int j = 0; j < kLoads; ++j)
      if (p0 + j < rank) acc = fmaf(gpow_n(lg, lens.len[p0 + j]), acc, x[j]);
  }
  s_in[idx] = acc;
}

// out = gamma^pos s_in + sum_{q: hi_q <= pos} gamma^(pos - hi_q) loc[q], float4 over [B*H][dk][dv].
__global__ void state_at_kernel(const float4* __restrict__ loc, const float4* __restrict__ s_in,
                                float4* __restrict__ out, const SegArgs sa, int N, int pos,
                                const float* __restrict__ log2g, int H, int64_t per_head4,
                                int64_t per_state4) {
  pdl_wait();
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= per_state4) return;
  const float lg = log2g[(int)((idx / per_head4) % H)];
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  if (s_in) {
    const float w = gpow(lg, (float)pos);
    const float4 x = s_in[idx];
    acc = make_float4(w * x.x, w * x.y, w * x.z, w * x.w);
  }
  for (int q0 = 0; q0 < sa.nloc; q0 += kLoads) {
    float4 x[kLoads];
    float w[kLoads];
#pragma unroll
    for (int j = 0; j < kLoads; ++j) {
      w[j] = q0 + j < sa.nloc ? seg_loc_weight(sa, q0 + j, N, pos, lg) : -1.f;
      if (w[j] >= 0.f) x[j] = loc[(int64_t)(q0 + j) * per_state4 + idx];
    }
#pragma unroll
    for (int j = 0; j < kLoads; ++j) {
      if (w[j] < 0.f) continue;
      acc.x = fmaf(w[j], x[j].x, acc.x);
      acc.y = fmaf(w[j], x[j].y, acc.y);
      acc.z = fmaf(w[j], x[j].z, acc.z);
      acc.w = fmaf(w[j], x[j].w, acc.w);
    }
  }
  out[idx] = acc;
}

// incl[p] = state at H_p = min(N, (p+1)*seg_len) accumulated from the ordered local states:
// acc (state at `pos`) <- gamma^(hi_q - pos) acc + loc[q] for each entry q, emitted at each H_p.
__global__ void segment_prefix_kernel(const float4* __restrict__ loc, float4* __restrict__ incl,
                                      const SegArgs sa, int N, int seg_len, int nseg,
                                      const float* __restrict__ log2g, int H, int64_t per_head4,
                                      int64_t per_state4) {
  pdl_wait();
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= per_state4) return;
  const float lg = log2g[(int)((idx / per_head4) % H)];
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  int pos = 0, p = 0;
  auto seg_end = [&](int pp) { return (int)min((long long)(pp + 1) * seg_len, (long long)N); };
  auto emit = [&](int pp) {        // incl[pp] = state at its segment end, from the state at pos
    const float w = gpow(lg, (float)(seg_end(pp) - pos));
    incl[(int64_t)pp * per_state4 + idx] = make_float4(w * acc.x, w * acc.y, w * acc.z, w * acc.w);
  };
  // entries in token order; before folding entry q, emit every segment ending before it
  for (int q0 = 0; q0 < sa.nloc; q0 += kLoads) {
    float4 x[kLoads];
    int qhi[kLoads];
#pragma unroll
    for (int j = 0; j < kLoads; ++j) {
      int qlo = 0;
      qhi[j] = 0;
      if (q0 + j < sa.nloc) seg_bounds(sa.loc_seg_len, sa.loc_sub, sa.loc_m, q0 + j, N, qlo, qhi[j]);
      if (qhi[j] <= qlo) qhi[j] = -1;                    // past the end or an empty sub-segment
      else x[j] = loc[(int64_t)(q0 + j) * per_state4 + idx];
    }
#pragma unroll
    for (int j = 0; j < kLoads; ++j) {
      if (qhi[j] < 0) continue;
      for (; p < nseg && seg_end(p) < qhi[j]; ++p) emit(p);
      const float w = gpow(lg, (float)(qhi[j] - pos));
      acc = make_float4(fmaf(w, acc.x, x[j].x), fmaf(w, acc.y, x[j].y), fmaf(w, acc.z, x[j].z),
                        fmaf(w, acc.w, x[j].w));
      pos = qhi[j];
    }
  }
  for (; p < nseg; ++p) emit(p);
}

}  // namespace

cudaError_t launch_segment_prefix(const SegArgs& sa, float* incl, int64_t seg_len, int64_t nseg,
                                  const float* log2g, const ShapeArgs& s, cudaStream_t stream) {
  const int64_t per_head = s.dk * s.dv;
  if (per_head % 4 != 0) return cudaErrorNotSupported;
  for (const void* p : {(const void*)sa.loc, (const void*)incl})
    if (reinterpret_cast<uintptr_t>(p) & 15) return cudaErrorNotSupported;
  const int64_t n4 = s.B * s.H * per_head / 4;
  constexpr int NT = 256;
  cudaError_t err = launch_pdl(segment_prefix_kernel, dim3((unsigned)((n4 + NT - 1) / NT)), dim3(NT), 0, stream,
                               (const float4*)sa.loc, (float4*)incl, sa, (int)s.N,
                               (int)std::min<int64_t>(seg_len, 0x7fffffff), (int)nseg, log2g, (int)s.H,
                               per_head / 4, n4);
  count_launch();
  return err != cudaSuccess ? err : cudaGetLastError();
}

cudaError_t launch_state_at(const float* loc, const float* s_in, float* out, const SegArgs& sa,
                            int64_t pos, const float* log2g, const ShapeArgs& s, cudaStream_t stream) {
  const int64_t per_head = s.dk * s.dv;
  if (per_head % 4 != 0) return cudaErrorNotSupported;
  for (const void* p : {(const void*)loc, (const void*)s_in, (const void*)out})
    if (reinterpret_cast<uintptr_t>(p) & 15) return cudaErrorNotSupported;
  const int64_t n4 = s.B * s.H * per_head / 4;
  constexpr int NT = 256;
  state_at_kernel<<<(unsigned)((n4 + NT - 1) / NT), NT, 0, stream>>>(
      (const float4*)loc, (const float4*)s_in, (float4*)out, sa, (int)s.N, (int)pos, log2g, (int)s.H,
      per_head / 4, n4);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_prefix_combine(const float* gathered, float* s_in, const int64_t* seg_lens,
                                  int P, int rank, const float* log2g, const ShapeArgs& s,
                                  cudaStream_t stream) {
  if (P > MAXP || rank < 0 || rank >= P) return cudaErrorInvalidValue;
  SegLens lens{};
  for (int p = 0; p < P; ++p) lens.len[p] = (long long)seg_lens[p];
  const int64_t per_head = s.dk * s.dv;
  const int64_t per_rank = s.B * s.H * per_head;
  const bool vec = (per_head % 4 == 0) && ((reinterpret_cast<uintptr_t>(gathered) & 15) == 0) &&
                   ((reinterpret_cast<uintptr_t>(s_in) & 15) == 0);
  constexpr int NT = 256;
  if (vec) {
    const int64_t n4 = per_rank / 4;
    cudaError_t err = launch_pdl(prefix_combine_kernel, dim3((unsigned)((n4 + NT - 1) / NT)), dim3(NT), 0, stream,
                                 (const float4*)gathered, (float4*)s_in, lens, rank, log2g, (int)s.H,
                                 per_head / 4, n4);
    if (err != cudaSuccess) return err;
  } else {
    prefix_combine_kernel_scalar<<<(unsigned)((per_rank + NT - 1) / NT), NT, 0, stream>>>(
        gathered, s_in, lens, rank, log2g, (int)s.H, per_head, per_rank);
  }
  count_launch();
  return cudaGetLastError();
}

}  // namespace linattn
