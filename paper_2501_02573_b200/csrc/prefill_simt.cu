// K6: chunked prefill on the FP32 FFMA pipe (the fp32 parity mode and the
// general-shape kernel).  Same algebra as the reference two-level-block method
// (kernels.py:139-166) with chunk CH and 0-based in-chunk row t:
//   O_t   = sum_{s<=t} gamma^(t-s) (q_t . k_s) v_s  +  gamma^(t+1) q_t S
//   S    <- gamma^L S + sum_s gamma^(L-1-s) k_s^T v_s
// One CTA owns one (batch*head, dv-tile) unit and walks the sequence; the
// state tile S[dk][DVT] stays in shared memory for the whole walk.
#include "common.cuh"

namespace linattn {
namespace {

constexpr int CH = 32;    // chunk length
constexpr int DVT = 64;   // dv columns per CTA
constexpr int NT = 256;   // threads per CTA

template <typename T>
__global__ void __launch_bounds__(NT)
prefill_simt_kernel(const T* __restrict__ q, const T* __restrict__ k, const T* __restrict__ v,
                    T* __restrict__ o, const float* __restrict__ log2g,
                    const float* __restrict__ s_in, float* __restrict__ s_out,
                    int H, int N, int dk, int dv, int state_only, const SegArgs sa) {
  extern __shared__ float smem[];
  const int ldq = dk + 1;                     // padded rows: conflict-free column walks
  float* Qs = smem;                           // [CH][ldq]
  float* Ks = Qs + CH * ldq;                  // [CH][ldq]
  float* Vs = Ks + CH * ldq;                  // [CH][DVT]
  float* A = Vs + CH * DVT;                   // [CH][CH+1]
  float* S = A + CH * (CH + 1);               // [dk][DVT]
  float* w = S + (size_t)dk * DVT;            // [CH] gamma^(L-1-s)

  const int bh = blockIdx.y;
  const int h = bh % H;
  const int j0 = blockIdx.x * DVT;
  const int nj = min(DVT, dv - j0);
  const int tid = threadIdx.x;
  const float lg = log2g[h];
  int lo, hi;  // this CTA's token segment (SegArgs)
  seg_bounds(sa.seg_len, sa.sub, sa.m, blockIdx.z, N, lo, hi);
  const size_t per_state = (size_t)gridDim.y * dk * dv;   // one [B*H][dk][dv] state

  const T* qb = q + (size_t)bh * N * dk;
  const T* kb = k + (size_t)bh * N * dk;
  const T* vb = v + (size_t)bh * N * dv;
  T* ob = o ? o + (size_t)bh * N * dv : nullptr;

  {
    const float w_in = gpow(lg, (float)lo);
    for (int e = tid; e < dk * DVT; e += NT) {
      const int i = e / DVT, j = e % DVT;
      S[e] = (s_in && j < nj) ? w_in * s_in[((size_t)bh * dk + i) * dv + j0 + j] : 0.f;
    }
    for (int qi = 0; qi < sa.nloc; ++qi) {
      const float wq = seg_loc_weight(sa, qi, N, lo, lg);
      if (wq < 0.f) continue;
      const float* lq = sa.loc + qi * per_state;
      for (int e = tid; e < dk * DVT; e += NT) {
        const int i = e / DVT, j = e % DVT;
        if (j < nj) S[e] = fmaf(wq, lq[((size_t)bh * dk + i) * dv + j0 + j], S[e]);
      }
    }
  }

  for (int c0 = lo; c0 < hi; c0 += CH) {
    const int L = min(CH, hi - c0);
    __syncthreads();
    for (int e = tid; e < CH * dk; e += NT) {
      const int t = e / dk, i = e % dk;
      const bool in = t < L;
      Ks[t * ldq + i] = in ? to_f32(kb[(size_t)(c0 + t) * dk + i]) : 0.f;
      if (!state_only) Qs[t * ldq + i] = in ? to_f32(qb[(size_t)(c0 + t) * dk + i]) : 0.f;
    }
    for (int e = tid; e < CH * DVT; e += NT) {
      const int t = e / DVT, j = e % DVT;
      Vs[e] = (t < L && j < nj) ? to_f32(vb[(size_t)(c0 + t) * dv + j0 + j]) : 0.f;
    }
    if (tid < CH) w[tid] = tid < L ? gpow(lg, (float)(L - 1 - tid)) : 0.f;
    __syncthreads();

    if (!state_only) {
      // A[t][s] = (q_t . k_s) gamma^(t-s) for s <= t (intra-chunk masked scores)
      for (int e = tid; e < CH * CH; e += NT) {
        const int t = e / CH, s = e % CH;
        float acc = 0.f;
        if (s <= t && t < L) {
          const float* qr = Qs + t * ldq;
          const float* kr = Ks + s * ldq;
          for (int i = 0; i < dk; ++i) acc = fmaf(qr[i], kr[i], acc);
          acc *= gpow(lg, (float)(t - s));
        }
        A[t * (CH + 1) + s] = acc;
      }
      __syncthreads();
      // O_t = A_t V + gamma^(t+1) q_t S
      const int j = tid % DVT;
      for (int t = tid / DVT; t < L; t += NT / DVT) {
        float intra = 0.f, inter = 0.f;
        const float* ar = A + t * (CH + 1);
        for (int s = 0; s <= t; ++s) intra = fmaf(ar[s], Vs[s * DVT + j], intra);
        const float* qr = Qs + t * ldq;
        for (int i = 0; i < dk; ++i) inter = fmaf(qr[i], S[i * DVT + j], inter);
        if (j < nj)
          ob[(size_t)(c0 + t) * dv + j0 + j] = from_f32<T>(intra + gpow(lg, (float)(t + 1)) * inter);
      }
      __syncthreads();
    }
    // S <- gamma^L S + sum_s gamma^(L-1-s) k_s^T v_s
    const float carry = gpow(lg, (float)L);
    for (int e = tid; e < dk * DVT; e += NT) {
      const int i = e / DVT, j = e % DVT;
      float acc = 0.f;
      for (int s = 0; s < L; ++s) acc = fmaf(w[s] * Ks[s * ldq + i], Vs[s * DVT + j], acc);
      S[e] = fmaf(carry, S[e], acc);
    }
  }
  __syncthreads();
  if (s_out && (state_only || blockIdx.z == gridDim.z - 1)) {
    float* so = s_out + (state_only ? blockIdx.z * per_state : 0);
    for (int e = tid; e < dk * DVT; e += NT) {
      const int i = e / DVT, j = e % DVT;
      if (j < nj) so[((size_t)bh * dk + i) * dv + j0 + j] = S[e];
    }
  }
}

}  // namespace

cudaError_t launch_prefill_simt(const void* q, const void* k, const void* v, void* o,
                                const float* log2g, const float* s_in, float* s_out,
                                const ShapeArgs& s, int dtype, bool state_only,
                                const SegArgs& sa, int nz, cudaStream_t stream) {
  const size_t ldq = (size_t)s.dk + 1;
  const size_t smem = sizeof(float) * (2 * CH * ldq + CH * DVT + CH * (CH + 1) +
                                       (size_t)s.dk * DVT + CH);
  if (smem > 227 * 1024) return cudaErrorNotSupported;
  dim3 grid((unsigned)((s.dv + DVT - 1) / DVT), (unsigned)(s.B * s.H), (unsigned)nz);
  cudaError_t err;
  if (dtype == LINATTN_BF16) {
    auto kern = prefill_simt_kernel<__nv_bfloat16>;
    err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (err != cudaSuccess) return err;
    kern<<<grid, NT, smem, stream>>>((const __nv_bfloat16*)q, (const __nv_bfloat16*)k,
                                     (const __nv_bfloat16*)v, (__nv_bfloat16*)o, log2g, s_in,
                                     s_out, (int)s.H, (int)s.N, (int)s.dk, (int)s.dv, state_only, sa);
  } else {
    auto kern = prefill_simt_kernel<float>;
    err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (err != cudaSuccess) return err;
    kern<<<grid, NT, smem, stream>>>((const float*)q, (const float*)k, (const float*)v,
                                     (float*)o, log2g, s_in, s_out, (int)s.H, (int)s.N,
                                     (int)s.dk, (int)s.dv, state_only, sa);
  }
  count_launch();
  return cudaGetLastError();
}

}  // namespace linattn
