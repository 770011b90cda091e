// Row-based recurrence in one launch: the reference _row_based_slice (kernels.py:93-106),
//   for t in 0..N-1:  S <- gamma S + k_t^T v_t ;  o_t = q_t S
// One CTA per (b*h, 128-wide dv tile) walks the tokens with its fp32 state in registers:
// thread (row group rg, column quad cv) owns the contiguous rows rg*rpt .. rg*rpt+rpt-1
// (rpt = ceil(dk / RRG)) x columns 4cv..4cv+3, so its q and k values of a token are one
// contiguous run in shared memory (16-byte vector loads, broadcast across the warp).
// Tokens are staged TC at a time by cp.async one chunk ahead, and each token's o partials go to
// a [TC][RRG][128] shared buffer that is reduced once per chunk -- two barriers per TC tokens.
#include <type_traits>

#include "common.cuh"

namespace linattn {
namespace {

constexpr int RNT = 256;              // threads
constexpr int RDV = 128;              // dv columns per CTA
constexpr int RCQ = RDV / 4;          // column quads (32)
constexpr int RRG = RNT / RCQ;        // row groups (8)
#ifndef REC_TC
#define REC_TC 16
#endif

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// RMAXR = state rows per thread (16: dk <= 128, 32: dk <= 256); TC = tokens per staged chunk
template <typename T, int RMAXR, int TC>
__global__ void __launch_bounds__(RNT)
recurrent_kernel(const T* __restrict__ q, const T* __restrict__ k, const T* __restrict__ v,
                 T* __restrict__ o, const float* __restrict__ log2g, const float* __restrict__ s_in,
                 float* __restrict__ s_out, int H, int N, int dk, int dv) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  T* qs = reinterpret_cast<T*>(smem_raw);                  // [2][TC][dk]
  T* ks = qs + 2 * TC * dk;                                // [2][TC][dk]
  T* vs = ks + 2 * TC * dk;                                // [2][TC][RDV]
  float* part = reinterpret_cast<float*>(vs + 2 * TC * RDV);   // [TC][RRG][RDV]
  const int bh = blockIdx.y;
  const int j0 = blockIdx.x * RDV;
  const int nj = min(RDV, dv - j0);
  const int tid = threadIdx.x;
  const int cv = tid % RCQ, rg = tid / RCQ;
  const int rpt = (dk + RRG - 1) / RRG;                     // rows per thread
  const int row0 = rg * rpt;
  const int nrows = max(0, min(rpt, dk - row0));           // rows row0 .. row0+nrows-1
  constexpr int EV2 = 16 / sizeof(T);
  const bool vec = (rpt % EV2) == 0;                       // 16-byte aligned runs (dk % (8*EV2) == 0)
  const float g = gpow(log2g[bh % H], 1.f);
  const T* qb = q + (size_t)bh * N * dk;
  const T* kb = k + (size_t)bh * N * dk;
  const T* vvb = v + (size_t)bh * N * dv;
  T* ob = o + (size_t)bh * N * dv;
  constexpr int EV = 16 / sizeof(T);                        // elements per 16-byte piece

  float S[RMAXR][4];
#pragma unroll
  for (int r = 0; r < RMAXR; ++r)
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int i = row0 + r, j = 4 * cv + e;
      S[r][e] = (s_in && r < nrows && j < nj) ? s_in[((size_t)bh * dk + i) * dv + j0 + j] : 0.f;
    }
  // stage tokens [c0, c0 + TC) into buffer buf (rows past N and columns past nj are never read)
  auto stage = [&](int c0, int buf) {
    const int nt = min(TC, N - c0);
    const int qk_pieces = nt * dk / EV;
    for (int x = tid; x < qk_pieces; x += RNT) {
      cp_async16(qs + (size_t)buf * TC * dk + x * EV, qb + (size_t)c0 * dk + x * EV);
      cp_async16(ks + (size_t)buf * TC * dk + x * EV, kb + (size_t)c0 * dk + x * EV);
    }
    const int vrow = nj / EV;                                // pieces per token row of the tile
    for (int x = tid; x < nt * vrow; x += RNT) {
      const int t = x / vrow, p = x % vrow;
      cp_async16(vs + ((size_t)buf * TC + t) * RDV + p * EV, vvb + (size_t)(c0 + t) * dv + j0 + p * EV);
    }
    cp_async_commit();
  };
  const int nchunks = (N + TC - 1) / TC;
  float sig = 1.f, inv = 1.f;                                // lazy decay state (see token_loop)
  const float ginv = g >= 0x1p-30f ? 1.f / g : 0.f;
  if (nchunks > 0) stage(0, 0);
  for (int ci = 0; ci < nchunks; ++ci) {
    const int c0 = ci * TC, buf = ci & 1;
    const int nt = min(TC, N - c0);
    if (ci + 1 < nchunks) {
      stage(c0 + TC, buf ^ 1);
      cp_async_wait<1>();                                    // chunk ci landed (ci+1 in flight)
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();                                         // ... for every thread's pieces
    const T* qc = qs + (size_t)buf * TC * dk;
    const T* kc = ks + (size_t)buf * TC * dk;
    const T* vc = vs + (size_t)buf * TC * RDV;
    // Lazy decay (gamma > 0): keep T = S / sig with sig = gamma^(tokens since the last renorm), so
    // S <- gamma S + k^T v becomes T += (k / sig) v and o = (q sig) . T: one FMA per state element
    // for the update instead of an FMUL and an FMA.  T is renormalised (T <- sig T) before sig
    // underflows; gamma == 0 keeps the direct form.
    auto token_loop = [&](auto lazy_tag) {
     constexpr bool LAZY = decltype(lazy_tag)::value;
     for (int t = 0; t < nt; ++t) {
      float vv[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) vv[e] = 4 * cv + e < nj ? to_f32(vc[t * RDV + 4 * cv + e]) : 0.f;
      float acc[4] = {0.f, 0.f, 0.f, 0.f};
      float kscale = 1.f, qscale = 1.f;
      if constexpr (LAZY) {
        sig *= g;
        inv *= ginv;
        kscale = inv;
        qscale = sig;
      }
      const T* kt = kc + t * dk + row0;
      const T* qt = qc + t * dk + row0;
#pragma unroll
      for (int r0 = 0; r0 < RMAXR; r0 += EV2) {
        if (r0 >= nrows) break;
        T kb8[EV2], qb8[EV2];
        if (vec) {   // one 16-byte load each (all lanes of the warp read the same run)
          *reinterpret_cast<uint4*>(kb8) = *reinterpret_cast<const uint4*>(kt + r0);
          *reinterpret_cast<uint4*>(qb8) = *reinterpret_cast<const uint4*>(qt + r0);
        } else {
#pragma unroll
          for (int u = 0; u < EV2; ++u) {
            kb8[u] = r0 + u < nrows ? kt[r0 + u] : T(0.f);
            qb8[u] = r0 + u < nrows ? qt[r0 + u] : T(0.f);
          }
        }
#pragma unroll
        for (int u = 0; u < EV2; ++u) {
          const int r = r0 + u;
          const float kr = to_f32(kb8[u]) * kscale, qr = to_f32(qb8[u]) * qscale;
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            if constexpr (LAZY) S[r][e] = fmaf(kr, vv[e], S[r][e]);
            else S[r][e] = fmaf(g, S[r][e], kr * vv[e]);
            acc[e] = fmaf(qr, S[r][e], acc[e]);
          }
        }
      }
      *reinterpret_cast<float4*>(part + ((size_t)t * RRG + rg) * RDV + 4 * cv) =
          make_float4(acc[0], acc[1], acc[2], acc[3]);
      if constexpr (LAZY) {
        if (sig < 0x1p-30f) {                                // uniform: same gamma for the CTA
#pragma unroll
          for (int r = 0; r < RMAXR; ++r)
#pragma unroll
            for (int e = 0; e < 4; ++e) S[r][e] *= sig;
          sig = 1.f;
          inv = 1.f;
        }
      }
     }
    };
    // (fp32 inputs keep the direct form: the lazy variant spills there and measured slower)
    // gamma < 2^-30 keeps the direct form too: 1/gamma (and k / sig) would overflow to inf
    if constexpr (sizeof(T) == 2) {
      if (g >= 0x1p-30f) token_loop(std::true_type{});
      else token_loop(std::false_type{});
    } else {
      token_loop(std::false_type{});
    }
    __syncthreads();                                         // all partials of the chunk written
    for (int x = tid; x < nt * RDV; x += RNT) {
      const int t = x / RDV, j = x % RDV;
      if (j < nj) {
        float sacc = 0.f;
#pragma unroll
        for (int r = 0; r < RRG; ++r) sacc += part[((size_t)t * RRG + r) * RDV + j];
        ob[(size_t)(c0 + t) * dv + j0 + j] = from_f32<T>(sacc);
      }
    }
    __syncthreads();                                         // staging buffer and partials reusable
  }
  if (s_out) {
#pragma unroll
    for (int r = 0; r < RMAXR; ++r)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int i = row0 + r, j = 4 * cv + e;
        if (r < nrows && j < nj) s_out[((size_t)bh * dk + i) * dv + j0 + j] = sig * S[r][e];
      }
  }
}

template <typename T, int RMAXR, int TC>
cudaError_t launch_rows(const void* q, const void* k, const void* v, void* o, const float* log2g,
                        const float* s_in, float* s_out, const ShapeArgs& s, cudaStream_t stream) {
  const size_t smem = sizeof(T) * (4 * TC * (size_t)s.dk + 2 * TC * RDV) + sizeof(float) * TC * RRG * RDV;
  if (smem > 227 * 1024) return cudaErrorNotSupported;
  auto kern = recurrent_kernel<T, RMAXR, TC>;
  cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (err != cudaSuccess) return err;
  dim3 grid((unsigned)((s.dv + RDV - 1) / RDV), (unsigned)(s.B * s.H));
  kern<<<grid, RNT, smem, stream>>>((const T*)q, (const T*)k, (const T*)v, (T*)o, log2g, s_in, s_out, (int)s.H,
                                    (int)s.N, (int)s.dk, (int)s.dv);
  count_launch();
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_t(const void* q, const void* k, const void* v, void* o, const float* log2g,
                     const float* s_in, float* s_out, const ShapeArgs& s, cudaStream_t stream) {
  if (s.dk <= 16 * RRG) {
    cudaError_t e = launch_rows<T, 16, REC_TC>(q, k, v, o, log2g, s_in, s_out, s, stream);
    if (e != cudaErrorNotSupported) return e;
    return launch_rows<T, 16, 16>(q, k, v, o, log2g, s_in, s_out, s, stream);   // fp32 staging is bigger
  }
  return launch_rows<T, 32, 16>(q, k, v, o, log2g, s_in, s_out, s, stream);
}

}  // namespace

cudaError_t launch_recurrent(const void* q, const void* k, const void* v, void* o, const float* log2g,
                             const float* s_in, float* s_out, const ShapeArgs& s, int dtype,
                             cudaStream_t stream) {
  const int ev = dtype == LINATTN_BF16 ? 8 : 4;                // elements per 16-byte cp.async piece
  if (s.dk > 32 * RRG || s.dk % ev != 0 || s.dv % ev != 0) return cudaErrorNotSupported;
  for (const void* p : {q, k, v})
    if (reinterpret_cast<uintptr_t>(p) & 15) return cudaErrorNotSupported;
  if (dtype == LINATTN_BF16)
    return launch_t<__nv_bfloat16>(q, k, v, o, log2g, s_in, s_out, s, stream);
  return launch_t<float>(q, k, v, o, log2g, s_in, s_out, s, stream);
}

}  // namespace linattn
