// K6: chunked prefill on the FP32 FFMA pipe (the fp32 parity mode and the
// general-shape kernel).  Same algebra as the reference two-level-block method
// (kernels.py:139-166) with chunk CH and 0-based in-chunk row t:
//   O_t   = sum_{s<=t} gamma^(t-s) (q_t . k_s) v_s  +  gamma^(t+1) q_t S
//   S    <- gamma^L S + sum_s gamma^(L-1-s) k_s^T v_s
// One CTA owns one (batch*head, dv-tile) unit and walks the sequence; the
// state tile S[dk][DVT] stays in shared memory for the whole walk.
#include <cstdlib>

#include "common.cuh"

namespace linattn {
namespace {

constexpr int CH = 32;    // chunk length
constexpr int DVT = 64;   // dv columns per CTA
constexpr int NT = 256;   // threads per CTA
#ifndef SIMT_O44
#define SIMT_O44 1        // 4x4 output tiles with the dk reduction split in halves (0: 2x4 tiles)
#endif

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

// Register-blocked variant for dk % 8 == 0 (every shape the benchmarks use): each thread owns
// a small output tile per product so one shared-memory load feeds 2-8 FMAs instead of 0.5:
//   A  (CH x CH, over dk):   2 x 2 tile per thread, float4 loads along dk
//   O  (CH x 64, over CH + dk): 2 (t) x 4 (j) tile
//   S  (dk x 64, over CH):   8 (i) x 4 (j) tile, read-modify-write of the smem state
// Same chunking, masks, decay weights and summation split as prefill_simt_kernel.
// ASYNC (fp32 inputs, 16-byte aligned rows): the next chunk's K and V stream into a second
// buffer by cp.async while the current chunk computes, and the next Q into the single Q buffer
// once the output products are done with it -- the synchronous loads left the kernel stalled
// on global memory (ncu: long-scoreboard half of all issue cycles).
__device__ __forceinline__ void cp_async16_zfill(float* dst, const float* src, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void st_release_gpu_u32(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_gpu_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void cp_async_commit_group() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_one() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

// BAL: balanced persistent schedule (Balance mode 0, chunk CH, tile DVT): one CTA per resident
// slot walks its work list (head -> published hand-off state, whole units, seeded tail).
template <typename T, bool ASYNC, bool BAL>
__global__ void __launch_bounds__(NT)
prefill_simt_rb_kernel(const T* __restrict__ q, const T* __restrict__ k, const T* __restrict__ v,
                       T* __restrict__ o, const float* __restrict__ log2g,
                       const float* __restrict__ s_in, float* __restrict__ s_out,
                       int H, int N, int dk, int dv, int state_only, const SegArgs sa, const Balance bal) {
  static_assert(!ASYNC || sizeof(T) == 4, "cp.async staging copies fp32 rows");
  extern __shared__ __align__(16) float smem[];
  const int ld = dk + 4;                      // 16-byte rows, bank-spread
  constexpr int NB = ASYNC ? 2 : 1;           // K/V buffers
  float* Qs = smem;                           // [CH][ld]
  float* Ks = Qs + CH * ld;                   // [NB][CH][ld]
  float* Vs = Ks + NB * CH * ld;              // [NB][CH][DVT]
  float* A = Vs + NB * CH * DVT;              // [CH][CH+4]
  float* S = A + CH * (CH + 4);               // [dk][DVT]
  float* w = S + (size_t)dk * DVT;            // [CH] gamma^(L-1-s)
  float* gq = w + CH;                         // [CH] gamma^(t+1)
  float* red = gq + CH;                       // SIMT_O44: [128][16] partial outputs of the k halves
  constexpr int LA = CH + 4;

  const int tid = threadIdx.x;
  const size_t per_state = (size_t)gridDim.y * dk * dv;
  // thread tiles
  const int tA = 2 * (tid / 16), sA = 2 * (tid % 16);    // A: rows tA..tA+1, cols sA..sA+1
  const int tO = 2 * (tid / 16), jO = 4 * (tid % 16);    // O: rows tO..tO+1, cols jO..jO+3
  const int jS = 4 * (tid % 16);                          // S: rows i0..i0+7 (i0 = 8*(tid/16) + 128*r)

  __shared__ int s_ticket;
  int ticket = 0, nitems = 1;
  long long r0 = 0, r1 = 0;
  if constexpr (!BAL) pdl_wait();               // launched with programmatic dependent launch
  if constexpr (BAL) {
    if (tid == 0) s_ticket = (int)atomicAdd(bal.flags + gridDim.x, 1u);   // start order
    __syncthreads();
    ticket = s_ticket;
    nitems = balance_items(bal, ticket, r0, r1);
  }
  for (int it = 0; it < nitems; ++it) {
  WorkItem wi;
  if constexpr (BAL) {
    wi = balance_item(bal, N, ticket, it, r0, r1);
  } else {
    wi.bh = blockIdx.y;
    wi.j0 = blockIdx.x * DVT;
    seg_bounds(sa.seg_len, sa.sub, sa.m, blockIdx.z, N, wi.lo, wi.hi);
    wi.in_slot = wi.out_slot = -1;
  }
  const int bh = wi.bh;
  const int h = bh % H;
  const int j0 = wi.j0;
  const int nj = min(DVT, dv - j0);
  const int lo = wi.lo, hi = wi.hi;
  const float lg = log2g[h];
  const T* qb = q + (size_t)bh * N * dk;
  const T* kb = k + (size_t)bh * N * dk;
  const T* vb = v + (size_t)bh * N * dv;
  T* ob = o ? o + (size_t)bh * N * dv : nullptr;

  if (BAL && it > 0) __syncthreads();        // the previous item's end-state reads of S are done
  if (BAL && wi.in_slot >= 0) {
    // balanced tail: the previous range's head published the state at lo (s_in included)
    if (tid == 0)
      while (ld_acquire_gpu_u32(bal.flags + wi.in_slot) == 0u) __nanosleep(256);
    __syncthreads();
    const float* hp = bal.hst + (size_t)wi.in_slot * dk * DVT;
    for (int e = tid; e < dk * DVT; e += NT) S[e] = (e % DVT) < nj ? __ldcg(hp + e) : 0.f;
  } else {
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

  // async staging of rows [cc0, cc0 + CH): rows past the segment and columns past dv zero-fill
  // (width: global row length; ldd: smem row stride; rowlen: staged columns, ncols of them valid)
  auto stage_rows = [&](float* dst, const T* src, int cc0, int width, int ldd, int rowlen, int col0, int ncols) {
    const int Lc = min(CH, hi - cc0);
    const int per_row = rowlen / 4;
    for (int e = tid; e < CH * per_row; e += NT) {
      const int t = e / per_row, c4 = 4 * (e % per_row);
      const bool ok = t < Lc && c4 < ncols;
      const float* g = reinterpret_cast<const float*>(src) + (size_t)(cc0 + (ok ? t : 0)) * width + col0 + (ok ? c4 : 0);
      cp_async16_zfill(dst + t * ldd + c4, g, ok ? 16 : 0);
    }
  };
  if constexpr (ASYNC) {
    if (lo < hi) {
      if (!state_only) stage_rows(Qs, qb, lo, dk, ld, dk, 0, dk);
      stage_rows(Ks, kb, lo, dk, ld, dk, 0, dk);
      stage_rows(Vs, vb, lo, dv, DVT, DVT, j0, nj);
    }
    cp_async_commit_group();
  }
  int buf = 0;
  for (int c0 = lo; c0 < hi; c0 += CH, buf ^= (NB - 1)) {
    const int L = min(CH, hi - c0);
    __syncthreads();
    if constexpr (ASYNC) {
      // buffer buf^1 was last read by the previous chunk's state update (before the barrier)
      if (c0 + CH < hi) {
        stage_rows(Ks + (buf ^ 1) * CH * ld, kb, c0 + CH, dk, ld, dk, 0, dk);
        stage_rows(Vs + (buf ^ 1) * CH * DVT, vb, c0 + CH, dv, DVT, DVT, j0, nj);
      }
      cp_async_commit_group();
      cp_async_wait_one();               // this chunk's K, V (and Q) have landed for this thread
    } else {
      for (int e = tid; e < CH * dk; e += NT) {
        const int t = e / dk, i = e % dk;
        const bool in = t < L;
        Ks[t * ld + i] = in ? to_f32(kb[(size_t)(c0 + t) * dk + i]) : 0.f;
        if (!state_only) Qs[t * ld + i] = in ? to_f32(qb[(size_t)(c0 + t) * dk + i]) : 0.f;
      }
      for (int e = tid; e < CH * DVT; e += NT) {
        const int t = e / DVT, j = e % DVT;
        Vs[e] = (t < L && j < nj) ? to_f32(vb[(size_t)(c0 + t) * dv + j0 + j]) : 0.f;
      }
    }
    const float* Kc = Ks + buf * CH * ld;
    const float* Vc = Vs + buf * CH * DVT;
    if (tid < CH) {
      w[tid] = tid < L ? gpow(lg, (float)(L - 1 - tid)) : 0.f;
      gq[tid] = gpow(lg, (float)(tid + 1));
    }
    __syncthreads();

    if (!state_only) {
      // A[t][s] = (q_t . k_s) gamma^(t-s), s <= t < L
      {
        float a00 = 0.f, a01 = 0.f, a10 = 0.f, a11 = 0.f;
        if (sA <= tA + 1) {
          const float* q0 = Qs + tA * ld;
          const float* q1 = q0 + ld;
          const float* k0 = Kc + sA * ld;
          const float* k1 = k0 + ld;
          for (int i = 0; i < dk; i += 4) {
            const float4 x0 = *reinterpret_cast<const float4*>(q0 + i);
            const float4 x1 = *reinterpret_cast<const float4*>(q1 + i);
            const float4 y0 = *reinterpret_cast<const float4*>(k0 + i);
            const float4 y1 = *reinterpret_cast<const float4*>(k1 + i);
            a00 = fmaf(x0.x, y0.x, fmaf(x0.y, y0.y, fmaf(x0.z, y0.z, fmaf(x0.w, y0.w, a00))));
            a01 = fmaf(x0.x, y1.x, fmaf(x0.y, y1.y, fmaf(x0.z, y1.z, fmaf(x0.w, y1.w, a01))));
            a10 = fmaf(x1.x, y0.x, fmaf(x1.y, y0.y, fmaf(x1.z, y0.z, fmaf(x1.w, y0.w, a10))));
            a11 = fmaf(x1.x, y1.x, fmaf(x1.y, y1.y, fmaf(x1.z, y1.z, fmaf(x1.w, y1.w, a11))));
          }
        }
        const float r[2][2] = {{a00, a01}, {a10, a11}};
#pragma unroll
        for (int dt = 0; dt < 2; ++dt)
#pragma unroll
          for (int ds = 0; ds < 2; ++ds) {
            const int t = tA + dt, sc = sA + ds;
            A[t * LA + sc] = (sc <= t && t < L) ? r[dt][ds] * gpow(lg, (float)(t - sc)) : 0.f;
          }
      }
      __syncthreads();
      // O_t = A_t V + gamma^(t+1) q_t S   (rows tO, tO+1; columns jO..jO+3)
#if SIMT_O44
      {
        // 4 x 4 output tiles over 128 threads per half: each half reduces half of dk (and of
        // the intra sources), one float4 of Q / A per row feeds 16 FMAs, halves summed in smem
        const int kh = tid >> 7, tt = tid & 127;
        const int r0 = 4 * (tt >> 4), jq = 4 * (tt & 15);
        float in[4][4], ex[4][4];
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int e = 0; e < 4; ++e) in[r][e] = ex[r][e] = 0.f;
        auto step4 = [](float (&acc)[4], const float4 a, const float4& b0, const float4& b1,
                        const float4& b2, const float4& b3) {
          acc[0] = fmaf(a.x, b0.x, fmaf(a.y, b1.x, fmaf(a.z, b2.x, fmaf(a.w, b3.x, acc[0]))));
          acc[1] = fmaf(a.x, b0.y, fmaf(a.y, b1.y, fmaf(a.z, b2.y, fmaf(a.w, b3.y, acc[1]))));
          acc[2] = fmaf(a.x, b0.z, fmaf(a.y, b1.z, fmaf(a.z, b2.z, fmaf(a.w, b3.z, acc[2]))));
          acc[3] = fmaf(a.x, b0.w, fmaf(a.y, b1.w, fmaf(a.z, b2.w, fmaf(a.w, b3.w, acc[3]))));
        };
        const int sc_lo = kh * (CH / 2), sc_hi = min(sc_lo + CH / 2, r0 + 4);
        for (int sc = sc_lo; sc < sc_hi; sc += 4) {
          const float4 v0 = *reinterpret_cast<const float4*>(Vc + (sc + 0) * DVT + jq);
          const float4 v1 = *reinterpret_cast<const float4*>(Vc + (sc + 1) * DVT + jq);
          const float4 v2 = *reinterpret_cast<const float4*>(Vc + (sc + 2) * DVT + jq);
          const float4 v3 = *reinterpret_cast<const float4*>(Vc + (sc + 3) * DVT + jq);
#pragma unroll
          for (int r = 0; r < 4; ++r)
            step4(in[r], *reinterpret_cast<const float4*>(A + (r0 + r) * LA + sc), v0, v1, v2, v3);
        }
        const int k_lo = kh * (dk / 2);
        for (int i = k_lo; i < k_lo + dk / 2; i += 4) {
          const float4 s0 = *reinterpret_cast<const float4*>(S + (i + 0) * DVT + jq);
          const float4 s1 = *reinterpret_cast<const float4*>(S + (i + 1) * DVT + jq);
          const float4 s2 = *reinterpret_cast<const float4*>(S + (i + 2) * DVT + jq);
          const float4 s3 = *reinterpret_cast<const float4*>(S + (i + 3) * DVT + jq);
#pragma unroll
          for (int r = 0; r < 4; ++r)
            step4(ex[r], *reinterpret_cast<const float4*>(Qs + (r0 + r) * ld + i), s0, s1, s2, s3);
        }
        float4* rd = reinterpret_cast<float4*>(red) + tt * 4;
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const float g = gq[r0 + r];
          const float4 o4 = make_float4(fmaf(g, ex[r][0], in[r][0]), fmaf(g, ex[r][1], in[r][1]),
                                        fmaf(g, ex[r][2], in[r][2]), fmaf(g, ex[r][3], in[r][3]));
          if (kh == 1) rd[r] = o4;
          else {
            in[r][0] = o4.x; in[r][1] = o4.y; in[r][2] = o4.z; in[r][3] = o4.w;
          }
        }
        __syncthreads();
        if (kh == 0) {
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            const int t = r0 + r;
            if (t >= L) continue;
            const float4 p = rd[r];
            const float ov[4] = {in[r][0] + p.x, in[r][1] + p.y, in[r][2] + p.z, in[r][3] + p.w};
#pragma unroll
            for (int e = 0; e < 4; ++e)
              if (jq + e < nj) ob[(size_t)(c0 + t) * dv + j0 + jq + e] = from_f32<T>(ov[e]);
          }
        }
      }
#else
      {
        float in0[4] = {0.f, 0.f, 0.f, 0.f}, in1[4] = {0.f, 0.f, 0.f, 0.f};
        float ex0[4] = {0.f, 0.f, 0.f, 0.f}, ex1[4] = {0.f, 0.f, 0.f, 0.f};
        // four reduction steps per iteration: one float4 of A (or Q) per row feeds 16 FMAs
        // (A is zero above the diagonal, so the intra loop runs to the next multiple of 4)
        auto step4 = [](float (&acc)[4], const float4 a, const float4& b0, const float4& b1,
                        const float4& b2, const float4& b3) {
          acc[0] = fmaf(a.x, b0.x, fmaf(a.y, b1.x, fmaf(a.z, b2.x, fmaf(a.w, b3.x, acc[0]))));
          acc[1] = fmaf(a.x, b0.y, fmaf(a.y, b1.y, fmaf(a.z, b2.y, fmaf(a.w, b3.y, acc[1]))));
          acc[2] = fmaf(a.x, b0.z, fmaf(a.y, b1.z, fmaf(a.z, b2.z, fmaf(a.w, b3.z, acc[2]))));
          acc[3] = fmaf(a.x, b0.w, fmaf(a.y, b1.w, fmaf(a.z, b2.w, fmaf(a.w, b3.w, acc[3]))));
        };
        const int sc_end = min(CH, (tO + 2 + 3) & ~3);
        for (int sc = 0; sc < sc_end; sc += 4) {
          const float4 v0 = *reinterpret_cast<const float4*>(Vc + (sc + 0) * DVT + jO);
          const float4 v1 = *reinterpret_cast<const float4*>(Vc + (sc + 1) * DVT + jO);
          const float4 v2 = *reinterpret_cast<const float4*>(Vc + (sc + 2) * DVT + jO);
          const float4 v3 = *reinterpret_cast<const float4*>(Vc + (sc + 3) * DVT + jO);
          step4(in0, *reinterpret_cast<const float4*>(A + tO * LA + sc), v0, v1, v2, v3);
          step4(in1, *reinterpret_cast<const float4*>(A + (tO + 1) * LA + sc), v0, v1, v2, v3);
        }
        const float* q0 = Qs + tO * ld;
        const float* q1 = q0 + ld;
        for (int i = 0; i < dk; i += 4) {
          const float4 s0 = *reinterpret_cast<const float4*>(S + (i + 0) * DVT + jO);
          const float4 s1 = *reinterpret_cast<const float4*>(S + (i + 1) * DVT + jO);
          const float4 s2 = *reinterpret_cast<const float4*>(S + (i + 2) * DVT + jO);
          const float4 s3 = *reinterpret_cast<const float4*>(S + (i + 3) * DVT + jO);
          step4(ex0, *reinterpret_cast<const float4*>(q0 + i), s0, s1, s2, s3);
          step4(ex1, *reinterpret_cast<const float4*>(q1 + i), s0, s1, s2, s3);
        }
#pragma unroll
        for (int dt = 0; dt < 2; ++dt) {
          const int t = tO + dt;
          if (t >= L) continue;
          const float g = gq[t];
          const float* in = dt ? in1 : in0;
          const float* ex = dt ? ex1 : ex0;
#pragma unroll
          for (int e = 0; e < 4; ++e)
            if (jO + e < nj) ob[(size_t)(c0 + t) * dv + j0 + jO + e] = from_f32<T>(in[e] + g * ex[e]);
        }
      }
#endif
      __syncthreads();   // Q.S reads of S done before the update below
      if constexpr (ASYNC) {
        // every read of Q for this chunk is done: stream the next chunk's Q in behind the update
        if (c0 + CH < hi) stage_rows(Qs, qb, c0 + CH, dk, ld, dk, 0, dk);
        cp_async_commit_group();
      }
    }
    // S <- gamma^L S + sum_s gamma^(L-1-s) k_s^T v_s   (rows i0..i0+7, columns jS..jS+3)
    const float carry = gpow(lg, (float)L);
    for (int i0 = 8 * (tid / 16); i0 < dk; i0 += 8 * (NT / 16)) {
      float acc[8][4];
#pragma unroll
      for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[r][e] = 0.f;
      for (int sc = 0; sc < L; ++sc) {
        const float ws = w[sc];
        const float4 vv = *reinterpret_cast<const float4*>(Vc + sc * DVT + jS);
        const float4 ka = *reinterpret_cast<const float4*>(Kc + sc * ld + i0);
        const float4 kc = *reinterpret_cast<const float4*>(Kc + sc * ld + i0 + 4);
        const float kr[8] = {ws * ka.x, ws * ka.y, ws * ka.z, ws * ka.w, ws * kc.x, ws * kc.y, ws * kc.z, ws * kc.w};
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          acc[r][0] = fmaf(kr[r], vv.x, acc[r][0]);
          acc[r][1] = fmaf(kr[r], vv.y, acc[r][1]);
          acc[r][2] = fmaf(kr[r], vv.z, acc[r][2]);
          acc[r][3] = fmaf(kr[r], vv.w, acc[r][3]);
        }
      }
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        float4* sp = reinterpret_cast<float4*>(S + (i0 + r) * DVT + jS);
        float4 x = *sp;
        x.x = fmaf(carry, x.x, acc[r][0]);
        x.y = fmaf(carry, x.y, acc[r][1]);
        x.z = fmaf(carry, x.z, acc[r][2]);
        x.w = fmaf(carry, x.w, acc[r][3]);
        *sp = x;
      }
    }
  }
  __syncthreads();
  if (BAL && wi.out_slot >= 0) {
    // balanced head: publish the end state to the next range's tail
    float* hp = bal.hst + (size_t)wi.out_slot * dk * DVT;
    for (int e = tid; e < dk * DVT; e += NT) hp[e] = S[e];
    __threadfence();
    __syncthreads();
    if (tid == 0) st_release_gpu_u32(bal.flags + wi.out_slot, 1u);
  } else if (s_out && (BAL ? hi == N : (state_only || blockIdx.z == gridDim.z - 1))) {
    float* so = s_out + (state_only ? blockIdx.z * per_state : 0);
    for (int e = tid; e < dk * DVT; e += NT) {
      const int i = e / DVT, j = e % DVT;
      if (j < nj) so[((size_t)bh * dk + i) * dv + j0 + j] = S[e];
    }
  }
  }  // work items
}

}  // namespace

namespace {

// Register-blocked variant selection: 0 = none (plain kernel), 1 = synchronous loads, 2 = cp.async.
int rb_mode(const void* q, const void* k, const void* v, const ShapeArgs& s, int dtype, size_t& smem) {
  static const bool plain = getenv("LINATTN_SIMT_PLAIN") != nullptr;       // A/B switch
  static const bool sync_loads = getenv("LINATTN_SIMT_SYNC") != nullptr;   // A/B switch
  if (s.dk % 8 != 0 || plain) return 0;
  const bool async = !sync_loads && dtype == LINATTN_F32 && s.dv % 4 == 0 &&
                     !((reinterpret_cast<uintptr_t>(k) | reinterpret_cast<uintptr_t>(v) |
                        reinterpret_cast<uintptr_t>(q)) & 15);
  for (int nb = async ? 2 : 1; nb >= 1; --nb) {
    smem = sizeof(float) * ((1 + nb) * CH * ((size_t)s.dk + 4) + nb * CH * DVT + CH * (CH + 4) +
                            (size_t)s.dk * DVT + 2 * CH + (SIMT_O44 ? 128 * 16 : 0));
    if (smem <= 227 * 1024) return nb == 2 ? 2 : 1;
  }
  return 0;
}

template <bool BAL>
cudaError_t launch_rb(int mode, const void* q, const void* k, const void* v, void* o, const float* log2g,
                      const float* s_in, float* s_out, const ShapeArgs& s, int dtype, bool state_only,
                      const SegArgs& sa, const Balance& bal, dim3 grid, size_t smem, cudaStream_t stream) {
  auto go = [&](auto kern, auto tp) -> cudaError_t {
    using TT = typename decltype(tp)::type;
    cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (err != cudaSuccess) return err;
    if constexpr (BAL) {   // follows the memset of its flags: plain stream order
      kern<<<grid, NT, smem, stream>>>((const TT*)q, (const TT*)k, (const TT*)v, (TT*)o, log2g, s_in, s_out,
                                       (int)s.H, (int)s.N, (int)s.dk, (int)s.dv, state_only ? 1 : 0, sa, bal);
    } else {
      err = launch_pdl(kern, grid, dim3(NT), smem, stream, (const TT*)q, (const TT*)k, (const TT*)v, (TT*)o,
                       log2g, s_in, s_out, (int)s.H, (int)s.N, (int)s.dk, (int)s.dv, state_only ? 1 : 0, sa, bal);
      if (err != cudaSuccess) return err;
    }
    count_launch();
    return cudaGetLastError();
  };
  struct F { using type = float; };
  struct Hb { using type = __nv_bfloat16; };
  if (mode == 2) return go(prefill_simt_rb_kernel<float, true, BAL>, F{});
  if (dtype == LINATTN_BF16) return go(prefill_simt_rb_kernel<__nv_bfloat16, false, BAL>, Hb{});
  return go(prefill_simt_rb_kernel<float, false, BAL>, F{});
}

}  // namespace

cudaError_t launch_prefill_simt(const void* q, const void* k, const void* v, void* o,
                                const float* log2g, const float* s_in, float* s_out,
                                const ShapeArgs& s, int dtype, bool state_only,
                                const SegArgs& sa, int nz, cudaStream_t stream) {
  dim3 grid((unsigned)((s.dv + DVT - 1) / DVT), (unsigned)(s.B * s.H), (unsigned)nz);
  cudaError_t err;
  size_t smem_rb = 0;
  if (const int mode = rb_mode(q, k, v, s, dtype, smem_rb))
    return launch_rb<false>(mode, q, k, v, o, log2g, s_in, s_out, s, dtype, state_only, sa, Balance{}, grid,
                            smem_rb, stream);
  const size_t ldq = (size_t)s.dk + 1;
  const size_t smem = sizeof(float) * (2 * CH * ldq + CH * DVT + CH * (CH + 1) +
                                       (size_t)s.dk * DVT + CH);
  if (smem > 227 * 1024) return cudaErrorNotSupported;
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

namespace {
template <typename K>
int resident_per_sm(K kern, size_t smem) {
  int n = 0;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess ||
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, NT, smem) != cudaSuccess)
    return 0;
  return n;
}
}  // namespace

int simt_balance_slots(const void* q, const void* k, const void* v, const ShapeArgs& s, int dtype) {
  size_t smem = 0;
  const int mode = rb_mode(q, k, v, s, dtype, smem);
  if (mode == 0) return 0;
  const int per_sm = mode == 2 ? resident_per_sm(prefill_simt_rb_kernel<float, true, true>, smem)
                     : dtype == LINATTN_BF16 ? resident_per_sm(prefill_simt_rb_kernel<__nv_bfloat16, false, true>, smem)
                                             : resident_per_sm(prefill_simt_rb_kernel<float, false, true>, smem);
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
    return 0;
  return per_sm * sms;
}

size_t simt_balance_workspace_bytes(const ShapeArgs& s, int slots) {
  return 256 * (size_t)((slots + 1 + 63) / 64) + (size_t)slots * s.dk * DVT * sizeof(float);
}

cudaError_t launch_prefill_simt_balanced(const void* q, const void* k, const void* v, void* o,
                                         const float* log2g, const float* s_in, float* s_out,
                                         const ShapeArgs& s, int dtype, int slots, void* ws,
                                         cudaStream_t stream) {
  size_t smem = 0;
  const int mode = rb_mode(q, k, v, s, dtype, smem);
  const int64_t ntiles = (s.dv + DVT - 1) / DVT;
  const int64_t units = s.B * s.H * ntiles, nc = (s.N + CH - 1) / CH;
  const int64_t w = (units * nc + slots - 1) / slots;
  if (mode == 0 || w < nc || units * nc > (1LL << 31) - 1) return cudaErrorNotSupported;
  Balance bal;
  bal.on = 1;
  bal.units = (int)units;
  bal.nc = (int)nc;
  bal.w = (int)w;
  bal.ntiles = (int)ntiles;
  bal.chunk = CH;
  bal.tile = DVT;
  bal.flags = static_cast<unsigned*>(ws);
  bal.hst = reinterpret_cast<float*>(static_cast<uint8_t*>(ws) + 256 * (size_t)((slots + 1 + 63) / 64));
  const int used = (int)((units * nc + w - 1) / w);
  cudaError_t err = cudaMemsetAsync(ws, 0, sizeof(unsigned) * (slots + 1), stream);
  if (err != cudaSuccess) return err;
  return launch_rb<true>(mode, q, k, v, o, log2g, s_in, s_out, s, dtype, false, SegArgs{}, bal, dim3(used), smem,
                         stream);
}

}  // namespace linattn
