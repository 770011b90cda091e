// K6: the fp32 parity mode on the tensor cores -- 3xTF32 chunked prefill (tcgen05 kind::tf32).
//
// Same algebra and transposed layout as the bf16 kernel (prefill_tc.cu, v2) -- every accumulator
// has M = 128 TMEM lanes (lane = dv row d) -- with fp32 operands split into a tf32 "hi" part and a
// "lo" remainder, x = hi + lo with hi = x with its low 13 mantissa bits cleared, so each product
// a.b is computed as hi(a).hi(b) + hi(a).lo(b) + lo(a).hi(b) (the dropped lo.lo term is ~2^-22
// relative): three tf32 MMAs per product, fp32 accumulation in TMEM.  One chunk of C = 32 tokens:
//
//   MMA1  P^T[s][t]  = sum_i K[s][i] Q[t][i]                  (M=128 [32 live], N=32, K=dk)  x3
//   mask  P^T       *= gamma^(t-s) (t >= s) in fp32, split -> P^T hi | lo in smem
//   prep  K'[s]      = gamma^(L-1-s) K[s] in fp32, split;  lo parts of Q, K, V
//   MMA2  dS^T[d][i] = sum_s V[s][d] K'[s][i]                  (M=128, N=dk, K=32)          x3
//         Oi^T[d][t] = sum_s V[s][d] P^T[s][t]                 (M=128, N=32, K=32)          x3
//         Ox^T[d][t] = sum_i S^T[d][i] Q[t][i]                 (A = S^T hi|lo in TMEM)      x3
//   state S <- gamma^L S + dS  (fp32 registers of 8 state warps; hi/lo published to TMEM)
//   out   O[t][d] = Oi^T[d][t] + gamma^(t+1) Ox^T[d][t]  (fp32) -> smem -> TMA bulk store
//
// Reference: kernels.py:139-166 (two-level block, chunk L <= C with 1-based t), accumulated in
// fp32 and checked against the f64 oracle at 1e-4 (verify.py:14).  1xTF32 misses
// that bar (6.2e-4 measured); 3xTF32 meets it with ~1e-6.
//
// Why C = 32: the state S^T needs a hi and a lo copy in TMEM as the A operand of Ox (2 x dk
// columns), next to dS (dk), P^T, Oi and Ox (C each): 3 x 128 + 3 x 32 = 480 of 512 columns.
//
// MMA1 runs at M = 64 (rows 0-15 of the chunk land in TMEM lanes 0-15, rows 16-31 in lanes
// 32-47), halving the shared-memory reads of its A operand; the lo parts of Q and K are double
// buffered so the next chunk's operand prep overlaps this chunk's MMAs, and the tensor pipe
// issues MMA1 of chunk c+1 ahead of O_inter of chunk c.
//
// Warp roles (512 threads): 0-1 P^T mask + split (16 key rows each), 2-3 and 14-15 operand prep
// (lo parts, K', MN-major relayout), 4-11 running state + outputs (direct coalesced fp32 stores),
// 12 TMA producer, 13 MMA issuer / TMEM owner.
#include <cstdlib>
#include <mutex>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "sm100.cuh"

#ifndef TF32_BAL_ONEITEM
#define TF32_BAL_ONEITEM 0     // dev bisect: balance_item items, but a compile-time item count of 1
#endif
#ifndef TF32_V_ATOM32
#define TF32_V_ATOM32 0        // TMA writes V in the 32B-granule swizzle (CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B)
#endif
#ifndef TF32_BAL_PLAINITEM
#define TF32_BAL_PLAINITEM 0   // dev bisect: BAL instantiation with the plain one-unit-per-CTA items
#endif
#ifndef TF32_BAL_REGS
#define TF32_BAL_REGS 0
#endif
#ifndef TF32_BAL_PDL
#define TF32_BAL_PDL 0
#endif
#ifndef TF32_FUSE_DS_OI
#define TF32_FUSE_DS_OI 1      // dS^T = V^T K' and Oi^T = V^T P^T as one N = dk + 32 MMA group (V^T read once)
#endif
#ifndef TF32_TRACE
#define TF32_TRACE 0           // dev: per-chunk clock64 timeline of CTA (0,0,0) (tools/trace_tf32.py)
#endif
#ifndef TF32_L2_PREFETCH
#define TF32_L2_PREFETCH 1     // warm L2 with the chunk that will reuse a K|V stage
#endif
#ifndef TF32_TRUNC_INPLACE
#define TF32_TRUNC_INPLACE 0   // 1: also clear the low mantissa bits of the TMA-loaded hi operands (the
                               // MMA ignores them: bit-identical results measured on B200, so off)
#endif

namespace linattn {

PFN_cuTensorMapEncodeTiled_v12000 tf32_encode_fn();
float* g_tf32_dump = nullptr;   // debug: first-chunk intermediates of CTA (0, 0, 0), see linattn_debug_set_tf32_dump

namespace {

using namespace sm100;

namespace v4 {

constexpr int kC = 32;           // tokens per chunk
constexpr int kDVT = 128;        // dv rows per CTA (MMA M)
constexpr int kThreads = 512;
constexpr int kPrep = 128;       // operand-prep threads (warps 2, 3, 14, 15)
constexpr uint32_t kTmemCols = 512;
// dS (dk columns) and O_intra (32) are adjacent, so one MMA group with B = [K' | P^T] fills both
constexpr uint32_t T_P = 0, T_OX = 32, T_DS = 64, T_O = 224, T_SHI = 256, T_SLO = 384;

// Shared memory (1 KiB aligned).  Q/K/V tiles are TMA boxes of [32 rows][32 fp32] (4 KiB, 128-byte
// swizzle), column blocks 4 KiB apart.  MMA1 reads K as a 128-row A operand (rows 32..127 are
// don't-care), i.e. 12 KiB past the last K box: K is followed by V in the stage, Klo by Qlo.
// Two TMA rings: Q (QST stages, held until O_inter of its chunk) and K|V (KVST stages, released
// after O_intra), so the next K/V loads start a whole MMA1 + O_inter earlier than with one ring.
template <int DKP, int QST, int KVST>
struct Cfg {
  static constexpr int KB = DKP / 32;
  static constexpr int QK_BYTES = kC * DKP * 4;
  static constexpr int V_BYTES = kC * kDVT * 4;
  static constexpr int KV_BYTES = QK_BYTES + V_BYTES;              // K | V
  static constexpr int OFF_KV = QST * QK_BYTES;
  static constexpr int OFF_KLO = OFF_KV + KVST * KV_BYTES;         // Klo | Qlo[2], K-major
  static constexpr int OFF_QLO = OFF_KLO + QK_BYTES;
  // MN-major tf32 tiles, 32-column blocks 4 KiB apart: [K'hi | P^T hi] and [K'lo | P^T lo] are
  // each one contiguous B operand of N = dk + 32 (P^T [32 s][32 t]), then Vlo
  static constexpr int OFF_KPH = OFF_QLO + 2 * QK_BYTES;
  static constexpr int OFF_PH = OFF_KPH + QK_BYTES;
  static constexpr int OFF_KPL = OFF_PH + 4096;
  static constexpr int OFF_PL = OFF_KPL + QK_BYTES;
  static constexpr int OFF_VLO = OFF_PL + 4096;
  static constexpr int OFF_POW = OFF_VLO + V_BYTES;                // gamma^n, n = 0..32
  static constexpr int OFF_BAR = OFF_POW + 3 * 64 * 4;            // (three per-role tables)
  static constexpr int SMEM = OFF_BAR + 512 + 1024;
  // the 64-row A operand of MMA1 reads 4 KiB past the last K box (K then V in a K|V stage, Klo then Qlo)
  static_assert((KB + 1) * 4096 <= KV_BYTES && (KB + 1) * 4096 <= 3 * QK_BYTES, "A overread");
};

__device__ __forceinline__ float tf32_hi(float x) { return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); }

template <int DKP, int QST, int KVST, bool SO, bool BAL>
__global__ void __launch_bounds__(kThreads, 1)
prefill_tf32_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                    const __grid_constant__ CUtensorMap tm_v, float* __restrict__ o,
                    const float* __restrict__ log2g, const float* __restrict__ s_in, float* __restrict__ s_out,
                    int H, int N, int dk, int dv, const SegArgs sa, const Balance bal, float* __restrict__ dump,
                    unsigned long long* __restrict__ trace) {
  using G = Cfg<DKP, QST, KVST>;
  // O_intra accumulator: right after the dk columns of dS (the fused [dS | Oi] group writes both)
  constexpr uint32_t T_OI = TF32_FUSE_DS_OI ? T_DS + DKP : T_O;
  static_assert(T_OI + kC <= T_SHI, "TMEM columns");
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // aligned by pointer arithmetic (not via an integer cast) so ptxas keeps the shared address
  // space: LDS/STS instead of generic loads/stores
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full_q = reinterpret_cast<uint64_t*>(smem + G::OFF_BAR);
  uint64_t* empty_q = full_q + QST;
  uint64_t* full_kv = empty_q + QST;
  uint64_t* empty_kv = full_kv + KVST;
  uint64_t* prepA = empty_kv + KVST;     // [2] Klo, Qlo[b] written (128 arrivals)
  uint64_t* derA_free = prepA + 2;       // [2] Ox done with Qlo[b] (commit)
  uint64_t* klo_free = derA_free + 2;    // MMA1 done with Klo (commit)
  uint64_t* prepB = klo_free + 1;        // K'hi, K'lo, Vlo written (128)
  uint64_t* derB_free = prepB + 1;       // dS + Oi done with K'/Vlo (commit)
  uint64_t* mma1_bar = derB_free + 1;    // P^T in TMEM (commit)
  uint64_t* mask_bar = mma1_bar + 1;     // P^T hi/lo in smem, TMEM copy read (64)
  uint64_t* p_free = mask_bar + 1;       // Oi done with P^T hi/lo smem (commit)
  uint64_t* mma_s_bar = p_free + 1;      // dS ready (commit)
  uint64_t* ds_free = mma_s_bar + 1;     // dS read by the state warps (256)
  uint64_t* st_full = ds_free + 1;       // S hi/lo published in TMEM (256)
  uint64_t* mma_o_bar = st_full + 1;     // Oi + Ox done (commit)
  uint64_t* o_free = mma_o_bar + 1;      // O / Ox drained (256)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_free + 1);
  // work-list header {ticket, items, range start, range end}, re-read at item boundaries
  int* wl = reinterpret_cast<int*>(tmem_slot + 2);
  // per-role gamma^n tables (n = 0..32): mask | prep | state, each rewritten by its own role at
  // an item boundary (balanced ranges span heads)
  float* pw_mask = reinterpret_cast<float*>(smem + G::OFF_POW);
  float* pw_prep = pw_mask + 64;
  float* pw_st = pw_mask + 128;

  const uint32_t warp = warp_id();
  const uint32_t lane = threadIdx.x & 31;
  const size_t per_state = (size_t)gridDim.y * dk * dv;

  if (warp == 12 && lane == 0) {
    if constexpr (BAL) {   // tickets in start order: the range before ours is already running
      const int t = (int)atomicAdd(bal.flags + gridDim.x, 1u);
      long long r0 = 0, r1 = 0;
      wl[1] = balance_items(bal, t, r0, r1);
      wl[0] = t;
      reinterpret_cast<long long*>(wl)[1] = r0;
      reinterpret_cast<long long*>(wl)[2] = r1;
    } else {
      wl[1] = 1;
    }
    for (int i = 0; i < QST; ++i) {
      mbar_init(&full_q[i], 1);
      mbar_init(&empty_q[i], 1);
    }
    for (int i = 0; i < KVST; ++i) {
      mbar_init(&full_kv[i], 1);
      mbar_init(&empty_kv[i], 1);
    }
    mbar_init(klo_free, 1);
    for (int b = 0; b < 2; ++b) {
      mbar_init(&prepA[b], kPrep);
      mbar_init(&derA_free[b], 1);
    }
    mbar_init(prepB, kPrep);
    mbar_init(derB_free, 1);
    mbar_init(mma1_bar, 1);
    mbar_init(mask_bar, 64);
    mbar_init(p_free, 1);
    mbar_init(mma_s_bar, 1);
    mbar_init(ds_free, 256);
    mbar_init(st_full, 256);
    mbar_init(mma_o_bar, 1);
    mbar_init(o_free, 256);
    fence_barrier_init();
    if (!SO) tma_prefetch_desc(&tm_q);
    tma_prefetch_desc(&tm_k);
    tma_prefetch_desc(&tm_v);
  }
  if (warp == 13) tmem_alloc<kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  if constexpr (!BAL || TF32_BAL_PDL) pdl_wait();   // the prologue above overlapped the previous kernel's tail
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;
  const int nitems = BAL && !TF32_BAL_PLAINITEM && !TF32_BAL_ONEITEM ? wl[1] : 1;
#if TF32_BAL_REGS
  const int wl_t = wl[0];
  const long long wl_r0 = reinterpret_cast<const long long*>(wl)[1], wl_r1 = reinterpret_cast<const long long*>(wl)[2];
#endif
  auto item = [&](int k) {
    if constexpr (BAL && !TF32_BAL_PLAINITEM) {
#if TF32_BAL_REGS
      return balance_item(bal, N, wl_t, k, wl_r0, wl_r1);
#else
      const volatile int* v = wl;
      const volatile long long* r = reinterpret_cast<const volatile long long*>(wl);
      return balance_item(bal, N, v[0], k, r[1], r[2]);
#endif
    }
    WorkItem w;
    w.bh = TF32_BAL_PLAINITEM && BAL ? (TF32_BAL_PLAINITEM == 2 ? (blockIdx.x * 37) % gridDim.x
                                        : TF32_BAL_PLAINITEM == 3 ? wl[0] : blockIdx.x) : blockIdx.y;
    w.j0 = TF32_BAL_PLAINITEM && BAL ? 0 : blockIdx.x * kDVT;
    seg_bounds(sa.seg_len, sa.sub, sa.m, blockIdx.z, N, w.lo, w.hi);
    w.in_slot = w.out_slot = -1;
    return w;
  };
  auto item_chunks = [](const WorkItem& w) { return w.hi > w.lo ? (w.hi - w.lo + kC - 1) / kC : 0; };
  // rewrite a role's gamma table for the item's head (every role thread done with the old one first)
  auto load_table = [&](float* tab, const WorkItem& w, int it, int rank, int nthr, int bar_id) {
    if (it > 0) named_bar_sync(bar_id, nthr);
    const float lgi = log2g[w.bh % H];
    for (int n = rank; n <= kC; n += nthr) tab[n] = gpow(lgi, (float)n);
    named_bar_sync(bar_id, nthr);
  };
  const bool dumping = !BAL && dump != nullptr && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0;
  // debug: per-chunk clock64 of CTA (0,0,0), trace[event * 4096 + chunk] (tools/trace_tf32.py)
  const bool tracing = !BAL && trace != nullptr && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0;
#if TF32_TRACE
#define TF_TRACE(ev, c) do { if (tracing && lane == 0 && (c) < 4096) trace[(ev) * 4096 + (c)] = clock64(); } while (0)
#else
#define TF_TRACE(ev, c) do { (void)tracing; } while (0)   // build with -DTF32_TRACE=1 (tools/build_variant.sh)
#endif

  if (warp < 2) {
    // ------------------------------------------------------------ P^T mask + hi/lo split
    // M = 64 accumulator: key row s = 16 * warp + lane (lanes 0-15 of subpartitions 0 and 1)
    if (!SO) {
      const int srow = 16 * (int)warp + (int)(lane & 15);
      const bool live = lane < 16;
      uint8_t* ph = smem + G::OFF_PH;
      uint8_t* pl = smem + G::OFF_PL;
      int gc = 0;
      for (int it = 0; it < nitems; ++it) {
        const WorkItem w = item(it);
        load_table(pw_mask, w, it, (int)threadIdx.x, 64, 4);
        const int nch = item_chunks(w);
        for (int c = 0; c < nch; ++c, ++gc) {
          mbar_wait(mma1_bar, gc & 1);
          tc_fence_after();
          float p[32];
          tmem_ld32(tbase + ((32 * warp) << 16) + T_P, p);
          tmem_wait_ld();
          if (dumping && gc == 0 && live)
            for (int t = 0; t < 32; ++t) dump[64 + srow * 32 + t] = p[t];
          if (gc > 0) mbar_wait(p_free, (gc - 1) & 1);    // Oi(gc-1) has read the previous P^T
          if (live) {
            float hv[32], lv[32];
#pragma unroll
            for (int t = 0; t < 32; ++t) {
              const float x = t >= srow ? p[t] * pw_mask[t >= srow ? t - srow : 0] : 0.f;
              hv[t] = tf32_hi(x);
              lv[t] = x - hv[t];
            }
            // MN-major tf32 layout: 16-byte piece j of row s at granule (j/2) ^ (s & 3), half j & 1.
            // Rows s and s+4 share granule positions, so they store the two halves in opposite
            // order (jj ^ flip) and a quarter-warp never hits one bank twice.
            const int flip = (srow >> 2) & 1;
#pragma unroll
            for (int jj = 0; jj < 8; ++jj) {
              const int j = jj ^ flip;
              const int off = srow * 128 + (((((j >> 1) ^ (srow & 3)) << 1) | (j & 1)) << 4);
              const float4 h4 = flip ? make_float4(hv[4 * (jj ^ 1)], hv[4 * (jj ^ 1) + 1], hv[4 * (jj ^ 1) + 2], hv[4 * (jj ^ 1) + 3])
                                     : make_float4(hv[4 * jj], hv[4 * jj + 1], hv[4 * jj + 2], hv[4 * jj + 3]);
              const float4 l4 = flip ? make_float4(lv[4 * (jj ^ 1)], lv[4 * (jj ^ 1) + 1], lv[4 * (jj ^ 1) + 2], lv[4 * (jj ^ 1) + 3])
                                     : make_float4(lv[4 * jj], lv[4 * jj + 1], lv[4 * jj + 2], lv[4 * jj + 3]);
              *reinterpret_cast<float4*>(ph + off) = h4;
              *reinterpret_cast<float4*>(pl + off) = l4;
            }
          }
          fence_proxy_async_smem();
          tc_fence_before();
          mbar_arrive(mask_bar);
          if (warp == 0) TF_TRACE(9, gc);
        }
      }
    }
  } else if (warp < 4 || warp >= 14) {
    // ------------------------------------------------------------ operand prep (128 threads)
    const int pt = warp < 4 ? (int)threadIdx.x - 64 : (int)threadIdx.x - 384;
    int gc = 0;
    for (int it = 0; it < nitems; ++it) {
     const WorkItem w = item(it);
     load_table(pw_prep, w, it, pt, kPrep, 3);
     const int nch = item_chunks(w);
     for (int c = 0; c < nch; ++c, ++gc) {
      const int sq = gc % QST, skv = gc % KVST;
      const int b = gc & 1;
      const int L = min(kC, w.hi - w.lo - c * kC);
      uint8_t* qs = smem + sq * G::QK_BYTES;
      uint8_t* ks = smem + G::OFF_KV + skv * G::KV_BYTES;
      uint8_t* vs = ks + G::QK_BYTES;
      uint8_t* klo = smem + G::OFF_KLO;
      uint8_t* qlo = smem + G::OFF_QLO + b * G::QK_BYTES;
      mbar_wait(&full_kv[skv], (gc / KVST) & 1);
      if (!SO) {
        mbar_wait(&full_q[sq], (gc / QST) & 1);
        if (gc >= 2) mbar_wait(&derA_free[b], ((gc >> 1) - 1) & 1);
        if (gc >= 1) mbar_wait(klo_free, (gc - 1) & 1);
        // Klo, Qlo (and, with TF32_TRUNC_INPLACE, the hi parts truncated in place)
        for (int i = pt; i < 2 * G::QK_BYTES / 16; i += kPrep) {
          const bool isk = i < G::QK_BYTES / 16;
          const int off = (isk ? i : i - G::QK_BYTES / 16) * 16;
          float4* src = reinterpret_cast<float4*>((isk ? ks : qs) + off);
          float4* dst = reinterpret_cast<float4*>((isk ? klo : qlo) + off);
          float4 x = *src, h, l;
          h.x = tf32_hi(x.x); h.y = tf32_hi(x.y); h.z = tf32_hi(x.z); h.w = tf32_hi(x.w);
          l.x = x.x - h.x; l.y = x.y - h.y; l.z = x.z - h.z; l.w = x.w - h.w;
          *dst = l;
          if (TF32_TRUNC_INPLACE) *src = h;
        }
        fence_proxy_async_smem();
        mbar_arrive(&prepA[b]);
        if (warp == 2) TF_TRACE(10, gc);
      }
      if (gc > 0) mbar_wait(derB_free, (gc - 1) & 1);
      // Row units (a 128-byte row of one 32-column box): K' = gamma^(L-1-s) K (zero past the ragged
      // end) split into hi | lo, and V split into hi (in place) | lo -- both re-laid from the TMA's
      // 128B swizzle (16-byte chunk j of row r at j ^ (r & 7)) to the MN-major tf32 layout
      // (32-byte granule g at g ^ (r & 3)), the only MN-major layout kind::tf32 reads.
      if (!SO && TF32_TRUNC_INPLACE) named_bar_sync(5, kPrep);   // K' reads K truncated by other threads
      if (TF32_V_ATOM32) {   // V already in the MN-major tf32 layout: Vlo at the same positions
        for (int i = pt; i < G::V_BYTES / 16; i += kPrep) {
          float4* src = reinterpret_cast<float4*>(vs + i * 16);
          float4 x = *src, h, l;
          h.x = tf32_hi(x.x); h.y = tf32_hi(x.y); h.z = tf32_hi(x.z); h.w = tf32_hi(x.w);
          l.x = x.x - h.x; l.y = x.y - h.y; l.z = x.z - h.z; l.w = x.w - h.w;
          *reinterpret_cast<float4*>(smem + G::OFF_VLO + i * 16) = l;
          if (TF32_TRUNC_INPLACE) *src = h;
        }
      }
      for (int u = pt; u < (G::KB + (TF32_V_ATOM32 ? 0 : 4)) * kC; u += kPrep) {
        const bool isv = u >= G::KB * kC;
        const int uu = isv ? u - G::KB * kC : u;
        const int r = uu & (kC - 1);
        const int boff = (uu >> 5) * 4096 + r * 128;
        const uint8_t* src = (isv ? vs : ks) + boff;
        float4 x[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) x[j] = *reinterpret_cast<const float4*>(src + ((j ^ (r & 7)) << 4));
        float wgt = 1.f;
        if (!isv) {
          wgt = r < L ? pw_prep[r < L ? L - 1 - r : 0] : 0.f;
          if (!SO && TF32_TRUNC_INPLACE) {   // K = hi + lo exactly
            const uint8_t* ls = klo + boff;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const float4 l = *reinterpret_cast<const float4*>(ls + ((j ^ (r & 7)) << 4));
              x[j].x += l.x; x[j].y += l.y; x[j].z += l.z; x[j].w += l.w;
            }
          }
        }
        uint8_t* dh = isv ? vs + boff : smem + G::OFF_KPH + boff;
        uint8_t* dl = smem + (isv ? G::OFF_VLO : G::OFF_KPL) + boff;
        const int flip = (r >> 2) & 1;   // rows r and r+4 store their halves in opposite order
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) {
          const int j = jj ^ flip;
          float4 v4 = flip ? x[jj ^ 1] : x[jj], h, l;
          v4.x *= wgt; v4.y *= wgt; v4.z *= wgt; v4.w *= wgt;
          h.x = tf32_hi(v4.x); h.y = tf32_hi(v4.y); h.z = tf32_hi(v4.z); h.w = tf32_hi(v4.w);
          l.x = v4.x - h.x; l.y = v4.y - h.y; l.z = v4.z - h.z; l.w = v4.w - h.w;
          const int pos = ((((j >> 1) ^ (r & 3)) << 1) | (j & 1)) << 4;
          *reinterpret_cast<float4*>(dh + pos) = (isv && !TF32_TRUNC_INPLACE) ? v4 : h;
          *reinterpret_cast<float4*>(dl + pos) = l;
        }
      }
      fence_proxy_async_smem();
      if (dumping && gc == 0) {   // raw smem of K, V (stage 0), K'hi, Vlo after prep: 4 x 4096 floats
        named_bar_sync(5, kPrep);
        for (int i = pt; i < 4096; i += kPrep) {
          dump[20480 + i] = i < G::QK_BYTES / 4 ? reinterpret_cast<const float*>(ks)[i] : 0.f;
          dump[24576 + i] = reinterpret_cast<const float*>(vs)[i];
          dump[28672 + i] = i < G::QK_BYTES / 4 ? reinterpret_cast<const float*>(smem + G::OFF_KPH)[i] : 0.f;
          dump[32768 + i] = reinterpret_cast<const float*>(smem + G::OFF_VLO)[i];
        }
      }
      mbar_arrive(prepB);
      if (warp == 2) TF_TRACE(11, gc);
     }
    }
  } else if (warp < 12) {
    // ------------------------------------------------------------ running state + outputs
    // warp (g, sub): TMEM lanes sub*32.. (dv rows d), state columns [g*SC, (g+1)*SC),
    // output tokens [g*16, g*16+16) of each chunk.
    constexpr int SC = DKP / 2;
    const int g = (warp - 4) / 4;
    const int sub = (warp - 4) % 4;
    const int d = sub * 32 + (int)lane;
    const int col0 = g * SC;
    const int sidx = (int)threadIdx.x - 128;
    const bool leader = sidx == 0;
    const uint32_t lane_base = tbase + ((uint32_t)(sub * 32) << 16);
    float S[SC];
    auto publish = [&]() {
#pragma unroll
      for (int j = 0; j < SC / 8; ++j) {
        uint32_t hv[8], lv[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float h = tf32_hi(S[8 * j + i]);
          hv[i] = __float_as_uint(h);
          lv[i] = __float_as_uint(S[8 * j + i] - h);
        }
        tmem_st8(lane_base + T_SHI + col0 + 8 * j, hv);
        tmem_st8(lane_base + T_SLO + col0 + 8 * j, lv);
      }
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(st_full);
    };
    int gc = 0;
    for (int it = 0; it < nitems; ++it) {
      const WorkItem w = item(it);
      const int jd = w.j0 + d;
      const bool dv_ok = jd < dv;
      const float lgi = log2g[w.bh % H];
      load_table(pw_st, w, it, sidx, 256, 6);
      if (w.in_slot >= 0) {
        // balanced tail: the previous range's head published the state at lo (s_in included)
        if (leader)
          while (ld_acquire_gpu(bal.flags + w.in_slot) == 0u) __nanosleep(256);
        named_bar_sync(6, 256);
        const float* hp = bal.hst + (size_t)w.in_slot * dk * kDVT + d;
#pragma unroll
        for (int i = 0; i < SC; ++i) S[i] = (col0 + i < dk) ? __ldcg(hp + (size_t)(col0 + i) * kDVT) : 0.f;
      } else {
        // S_init = gamma^lo s_in + sum_{q: hi_q <= lo} gamma^(lo - hi_q) loc[q]  (SegArgs), 16 columns at a time
        const float w_in = gpow(lgi, (float)w.lo);
        const bool in_ok = s_in != nullptr && dv_ok;
#pragma unroll
        for (int j = 0; j < SC; j += 16) {
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const int ci = col0 + j + i;
            S[j + i] = (in_ok && ci < dk) ? w_in * __ldg(s_in + ((size_t)w.bh * dk + ci) * dv + jd) : 0.f;
          }
          for (int qi = 0; qi < sa.nloc; ++qi) {
            const float wq = seg_loc_weight(sa, qi, N, w.lo, lgi);
            if (wq < 0.f || !dv_ok) continue;
            const float* lq = sa.loc + qi * per_state + ((size_t)w.bh * dk + col0 + j) * dv + jd;
#pragma unroll
            for (int i = 0; i < 16; ++i)
              if (col0 + j + i < dk) S[j + i] = fmaf(wq, __ldg(lq + (size_t)i * dv), S[j + i]);
          }
        }
      }
      const int nch = item_chunks(w);
      if (!SO && nch > 0) publish();
      float* orow = SO ? nullptr : o + ((size_t)w.bh * N + w.lo) * dv + jd;
      for (int c = 0; c < nch; ++c, ++gc) {
        const int L = min(kC, w.hi - w.lo - c * kC);
        mbar_wait(mma_s_bar, gc & 1);
        tc_fence_after();
        if (warp == 4) TF_TRACE(0, gc);
        const float carry = pw_st[L];
#pragma unroll
        for (int j = 0; j < SC / 16; ++j) {
          float ds[16];
          tmem_ld16(lane_base + T_DS + col0 + 16 * j, ds);
          tmem_wait_ld();
          if (dumping && gc == 0)
            for (int i = 0; i < 16; ++i) dump[2048 + d * 128 + col0 + 16 * j + i] = ds[i];
#pragma unroll
          for (int i = 0; i < 16; ++i) S[16 * j + i] = fmaf(carry, S[16 * j + i], ds[i]);
        }
        tc_fence_before();
        mbar_arrive(ds_free);
        if (warp == 4) TF_TRACE(1, gc);
        if (SO) continue;
        mbar_wait(mma_o_bar, gc & 1);                 // Oi, Ox done: S hi/lo may be replaced
        tc_fence_after();
        if (warp == 4) TF_TRACE(2, gc);
        if (c != nch - 1) publish();
        if (warp == 4) TF_TRACE(3, gc);
        // ---- outputs: O[t][d] = Oi^T[d][t] + gamma^(t+1) Ox^T[d][t], tokens g*16 .. g*16+15;
        //      for each t the 32 lanes of a warp store 32 consecutive dv columns (128 B)
        float ov[16], xv[16];
        tmem_ld16(lane_base + T_OI + g * 16, ov);
        tmem_ld16(lane_base + T_OX + g * 16, xv);
        tmem_wait_ld();
        tc_fence_before();
        mbar_arrive(o_free);
        if (warp == 4) TF_TRACE(4, gc);
        if (dv_ok) {
          float* orc = orow + (size_t)(c * kC + g * 16) * dv;
#pragma unroll
          for (int i = 0; i < 16; ++i)
            if (g * 16 + i < L) __stcs(orc + (size_t)i * dv, fmaf(pw_st[g * 16 + i + 1], xv[i], ov[i]));
        }
      }
      // end state: a balanced head publishes it to its hand-off slot; otherwise state-only
      // launches write one local state per segment and full launches only the segment ending
      // the sequence (its seed already covers every earlier token)
      if (w.out_slot >= 0) {
        float* hp = bal.hst + (size_t)w.out_slot * dk * kDVT + d;
#pragma unroll
        for (int i = 0; i < SC; ++i)
          if (col0 + i < dk) hp[(size_t)(col0 + i) * kDVT] = S[i];
        __threadfence();
        named_bar_sync(7, 256);
        if (leader) st_release_gpu(bal.flags + w.out_slot, 1u);
      } else if (s_out && dv_ok && (BAL ? w.hi == N : (SO || blockIdx.z == gridDim.z - 1))) {
        float* so = s_out + (SO ? blockIdx.z * per_state : 0) + (size_t)w.bh * dk * dv + jd;
#pragma unroll
        for (int i = 0; i < SC; ++i)
          if (col0 + i < dk) so[(size_t)(col0 + i) * dv] = S[i];
      }
    }
  } else if (warp == 12) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      // L2-prefetch cursor over the work list's chunk stream, KVST chunks ahead of the loads
      struct Cursor { int it, c; WorkItem w; };
      auto settle = [&](Cursor& u) {
        while (u.it < nitems && u.c >= item_chunks(u.w)) {
          ++u.it;
          u.c = 0;
          if (u.it < nitems) u.w = item(u.it);
        }
      };
      Cursor pf{0, 0, WorkItem{}};
      if (nitems > 0) pf.w = item(0);
      settle(pf);
      for (int i = 0; i < KVST && pf.it < nitems; ++i) {
        ++pf.c;
        settle(pf);
      }
      int gc = 0;
      for (int it = 0; it < nitems; ++it) {
        const WorkItem w = item(it);
        const int nch = item_chunks(w);
        for (int c = 0; c < nch; ++c, ++gc) {
          const int sq = gc % QST, skv = gc % KVST;
          const int t0 = w.lo + c * kC;
          // warm L2 with the chunk that will reuse this K|V stage, so its load is an L2 hit
          if (TF32_L2_PREFETCH && pf.it < nitems) {
            const int tp = pf.w.lo + pf.c * kC;
#pragma unroll
            for (int kb = 0; kb < G::KB; ++kb) {
              if (!SO) tma_prefetch_l2_3d(&tm_q, kb * 32, tp, pf.w.bh);
              tma_prefetch_l2_3d(&tm_k, kb * 32, tp, pf.w.bh);
            }
#pragma unroll
            for (int nb = 0; nb < 4; ++nb) tma_prefetch_l2_3d(&tm_v, pf.w.j0 + nb * 32, tp, pf.w.bh);
            ++pf.c;
            settle(pf);
          }
          if (!SO) {
            mbar_wait(&empty_q[sq], ((gc / QST) & 1) ^ 1);
            uint8_t* qd = smem + sq * G::QK_BYTES;
            mbar_arrive_expect_tx(&full_q[sq], G::QK_BYTES);
#pragma unroll
            for (int kb = 0; kb < G::KB; ++kb) tma_load_3d(qd + kb * 4096, &tm_q, &full_q[sq], kb * 32, t0, w.bh);
          }
          mbar_wait(&empty_kv[skv], ((gc / KVST) & 1) ^ 1);
          TF_TRACE(12, gc);
          uint8_t* kd = smem + G::OFF_KV + skv * G::KV_BYTES;
          mbar_arrive_expect_tx(&full_kv[skv], G::KV_BYTES);
#pragma unroll
          for (int kb = 0; kb < G::KB; ++kb) tma_load_3d(kd + kb * 4096, &tm_k, &full_kv[skv], kb * 32, t0, w.bh);
#pragma unroll
          for (int nb = 0; nb < 4; ++nb)
            tma_load_3d(kd + G::QK_BYTES + nb * 4096, &tm_v, &full_kv[skv], w.j0 + nb * 32, t0, w.bh);
        }
      }
    }
  } else {
    // ------------------------------------------------------------ MMA issuer (whole warp)
    // per chunk: dS(c) -> Oi(c) -> MMA1(c+1) -> Ox(c); MMA1 runs ahead so the mask epilogue of
    // c+1 overlaps the state publish that Ox(c) waits for.  The tensor pipe sees one flat chunk
    // stream across the work list (only buffer/stage indices depend on the chunk).
    constexpr uint32_t id_qk = idesc_tf32(64, kC, false, false);     // P^T = K Q^T (M = 64)
    constexpr uint32_t id_vk = idesc_tf32(128, DKP, true, true);     // dS^T = V^T K'
    constexpr uint32_t id_vkp = idesc_tf32(128, DKP + kC, true, true);   // [dS^T | Oi^T] = V^T [K' | P^T]
    constexpr uint32_t id_vp = idesc_tf32(128, kC, true, true);      // Oi^T = V^T P^T
    constexpr uint32_t id_sq = idesc_tf32(128, kC, false, false);    // Ox^T = S^T(TMEM) Q^T
    const uint32_t base = smem_u32(smem);
    const uint64_t dK0 = smem_desc_sw128(base, 16, 1024);             // K-major (TMA 128B swizzle)
    const uint64_t dM0 = smem_desc_sw128_b32(base, 4096, 512);        // MN-major tf32, 32-wide blocks
    constexpr uint64_t kQK = G::QK_BYTES >> 4, kKV = G::KV_BYTES >> 4;
    const uint64_t klo_k = dK0 + (G::OFF_KLO >> 4), qlo_k0 = dK0 + (G::OFF_QLO >> 4);
    const uint64_t kv_k0 = dK0 + (G::OFF_KV >> 4), kv_m0 = dM0 + (G::OFF_KV >> 4);
    const uint64_t kph_m = dM0 + (G::OFF_KPH >> 4), kpl_m = dM0 + (G::OFF_KPL >> 4);
    const uint64_t vlo_m = dM0 + (G::OFF_VLO >> 4);
    const uint64_t ph_m = dM0 + (G::OFF_PH >> 4), pl_m = dM0 + (G::OFF_PL >> 4);
    int nchunks = 0;
    for (int it = 0; it < nitems; ++it) nchunks += item_chunks(item(it));
    // a lane-0 broadcast makes the chunk count (and every descriptor derived from the chunk
    // index) provably warp-uniform: ptxas keeps them in uniform registers instead of wrapping each
    // tcgen05.mma in a per-lane R2UR loop
    nchunks = __shfl_sync(0xffffffffu, nchunks, 0);
    auto issue_mma1 = [&](int c) {
      const uint64_t q_k = dK0 + (c % QST) * kQK, k_k = kv_k0 + (c % KVST) * kKV;
      const uint64_t qlo_k = qlo_k0 + (c & 1) * kQK;
      mbar_wait(&full_q[c % QST], (c / QST) & 1);
      mbar_wait(&full_kv[c % KVST], (c / KVST) & 1);
      mbar_wait(&prepA[c & 1], (c >> 1) & 1);
      tc_fence_after();
      // P^T = Khi Qhi + Khi Qlo + Klo Qhi
#pragma unroll
      for (int kb = 0; kb < G::KB; ++kb)
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const uint64_t off = kb * 256 + kk * 2;
          mma_tf32_ss_elect(tbase + T_P, k_k + off, q_k + off, id_qk, (kb | kk) != 0);
          mma_tf32_ss_elect(tbase + T_P, k_k + off, qlo_k + off, id_qk, 1);
          mma_tf32_ss_elect(tbase + T_P, klo_k + off, q_k + off, id_qk, 1);
        }
      mma_commit_elect(mma1_bar);
      mma_commit_elect(klo_free);
      TF_TRACE(7, c);
    };
    if (!SO && nchunks > 0) issue_mma1(0);
    for (int c = 0; c < nchunks; ++c) {
      const int sq = c % QST, skv = c % KVST;
      const uint64_t q_k = dK0 + sq * kQK;                            // raw Q (hi), K-major
      const uint64_t qlo_k = qlo_k0 + (c & 1) * kQK;
      const uint64_t v_m = kv_m0 + skv * kKV + kQK;                   // V (hi), MN-major
      TF_TRACE(13, c);
      mbar_wait(&full_kv[skv], (c / KVST) & 1);
      mbar_wait(prepB, c & 1);
      if (c > 0) mbar_wait(ds_free, (c - 1) & 1);
      const bool fuse = TF32_FUSE_DS_OI && !SO;
      if (fuse) {                                      // the fused group also writes O_intra and reads P^T
        mbar_wait(mask_bar, c & 1);
        if (c > 0) mbar_wait(o_free, (c - 1) & 1);
      }
      tc_fence_after();
      TF_TRACE(5, c);
      if (fuse) {
        // [dS^T | Oi^T] = V^T [K' | P^T]: Vhi (K'|P)hi + Vhi (K'|P)lo + Vlo (K'|P)hi -- one N = dk + 32
        // group, so V^T (hi and lo) is read from shared memory once for both products
#pragma unroll
        for (int ks = 0; ks < kC / 8; ++ks) {
          const uint64_t off = ks * 64;
          mma_tf32_ss_elect(tbase + T_DS, v_m + off, kph_m + off, id_vkp, ks != 0);
          mma_tf32_ss_elect(tbase + T_DS, v_m + off, kpl_m + off, id_vkp, 1);
          mma_tf32_ss_elect(tbase + T_DS, vlo_m + off, kph_m + off, id_vkp, 1);
        }
        mma_commit_elect(mma_s_bar);
      } else {
        // dS^T = Vhi K'hi + Vhi K'lo + Vlo K'hi   (K step = 8 token rows = 1 KiB)
#pragma unroll
        for (int ks = 0; ks < kC / 8; ++ks) {
          const uint64_t off = ks * 64;
          mma_tf32_ss_elect(tbase + T_DS, v_m + off, kph_m + off, id_vk, ks != 0);
          mma_tf32_ss_elect(tbase + T_DS, v_m + off, kpl_m + off, id_vk, 1);
          mma_tf32_ss_elect(tbase + T_DS, vlo_m + off, kph_m + off, id_vk, 1);
        }
        mma_commit_elect(mma_s_bar);
      }
      if (!SO) {
        if (!fuse) {
          mbar_wait(mask_bar, c & 1);
          if (c > 0) mbar_wait(o_free, (c - 1) & 1);
          tc_fence_after();
          // Oi^T = Vhi Phi + Vhi Plo + Vlo Phi
#pragma unroll
          for (int ks = 0; ks < kC / 8; ++ks) {
            const uint64_t off = ks * 64;
            mma_tf32_ss_elect(tbase + T_OI, v_m + off, ph_m + off, id_vp, ks != 0);
            mma_tf32_ss_elect(tbase + T_OI, v_m + off, pl_m + off, id_vp, 1);
            mma_tf32_ss_elect(tbase + T_OI, vlo_m + off, ph_m + off, id_vp, 1);
          }
        }
        mma_commit_elect(p_free);
        TF_TRACE(6, c);
        mma_commit_elect(derB_free);
        mma_commit_elect(&empty_kv[skv]);            // K (MMA1, K') and V (dS, Oi) consumed
        if (c + 1 < nchunks) issue_mma1(c + 1);
        mbar_wait(st_full, c & 1);
        tc_fence_after();
        // Ox^T = Shi Qhi + Shi Qlo + Slo Qhi   (A from TMEM: 8 columns per K step)
#pragma unroll
        for (int kb = 0; kb < G::KB; ++kb)
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const uint64_t off = kb * 256 + kk * 2;
            const uint32_t col = (kb * 4 + kk) * 8;
            mma_tf32_ts_elect(tbase + T_OX, tbase + T_SHI + col, q_k + off, id_sq, (kb | kk) != 0);
            mma_tf32_ts_elect(tbase + T_OX, tbase + T_SHI + col, qlo_k + off, id_sq, 1);
            mma_tf32_ts_elect(tbase + T_OX, tbase + T_SLO + col, q_k + off, id_sq, 1);
          }
        mma_commit_elect(mma_o_bar);
        TF_TRACE(8, c);
        mma_commit_elect(&derA_free[c & 1]);
        mma_commit_elect(&empty_q[sq]);
      } else {
        mma_commit_elect(derB_free);
        mma_commit_elect(&empty_kv[skv]);
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 13) tmem_dealloc<kTmemCols>(tbase);
}

}  // namespace v4

// [BH][N][D] fp32 viewed as a 3-D tensor (D fastest); boxes of 32 x 32, 128B swizzle.
bool make_map_f32(CUtensorMap* map, const void* base, int64_t D, int64_t N, int64_t BH,
                  CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
  auto fn = tf32_encode_fn();
  if (!fn) return false;
  cuuint64_t dims[3] = {(cuuint64_t)D, (cuuint64_t)N, (cuuint64_t)BH};
  cuuint64_t strides[2] = {(cuuint64_t)D * 4, (cuuint64_t)(N * D * 4)};
  cuuint32_t box[3] = {32, 32, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

template <int DKP, int QST, int KVST, bool SO, bool BAL = false>
cudaError_t launch_v4(const void* q, const void* k, const void* v, void* o, const float* log2g, const float* s_in,
                      float* s_out, const ShapeArgs& s, const SegArgs& sa, int nz, cudaStream_t stream,
                      const Balance& bal = Balance{}, int ctas = 0) {
  using G = v4::Cfg<DKP, QST, KVST>;
  static_assert(G::SMEM <= 227 * 1024, "shared memory budget");
  const int64_t BH = s.B * s.H;
  CUtensorMap mq, mk, mv;
  // V is only ever an MN-major operand: with TF32_V_ATOM32 the TMA writes it straight into the
  // 32-byte-granule swizzle kind::tf32 reads (no relayout pass)
  if (!make_map_f32(&mk, k, s.dk, s.N, BH) ||
      !make_map_f32(&mv, v, s.dv, s.N, BH,
                    TF32_V_ATOM32 ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B))
    return cudaErrorInvalidValue;
  mq = mk;
  if (!SO && !make_map_f32(&mq, q, s.dk, s.N, BH)) return cudaErrorInvalidValue;
  auto kern = v4::prefill_tf32_kernel<DKP, QST, KVST, SO, BAL>;
  cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, G::SMEM);
  if (err != cudaSuccess) return err;
  if constexpr (BAL && !TF32_BAL_PDL) {   // follows the memset of its flags: plain stream order
    kern<<<dim3((unsigned)ctas), v4::kThreads, G::SMEM, stream>>>(mq, mk, mv, static_cast<float*>(o), log2g, s_in,
                                                                  s_out, (int)s.H, (int)s.N, (int)s.dk, (int)s.dv,
                                                                  sa, bal, nullptr, nullptr);
  } else {
    const dim3 grid = BAL ? dim3((unsigned)ctas)
                          : dim3((unsigned)((s.dv + v4::kDVT - 1) / v4::kDVT), (unsigned)BH, (unsigned)nz);
    err = launch_pdl(kern, grid, dim3(v4::kThreads), G::SMEM, stream, mq, mk, mv, static_cast<float*>(o), log2g,
                     s_in, s_out, (int)s.H, (int)s.N, (int)s.dk, (int)s.dv, sa, bal, g_tf32_dump,
                     BAL ? nullptr : trace_buffer());
    if (err != cudaSuccess) return err;
  }
  count_launch();
  return cudaGetLastError();
}

}  // namespace

PFN_cuTensorMapEncodeTiled_v12000 tf32_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult qr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &qr) == cudaSuccess &&
        qr == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

bool tf32_supported(const ShapeArgs& s, int dtype) {
  if (dtype != LINATTN_F32) return false;
  if (s.dk < 1 || s.dk > 128 || s.dk % 4 != 0 || s.dv % 4 != 0) return false;   // TMA: 16-byte rows
  return tf32_encode_fn() != nullptr;
}

cudaError_t launch_prefill_tf32(const void* q, const void* k, const void* v, void* o, const float* log2g,
                                const float* s_in, float* s_out, const ShapeArgs& s, bool state_only,
                                const SegArgs& sa, int nz, cudaStream_t stream) {
  for (const void* p : {q, k, v, (const void*)o})
    if (p && (reinterpret_cast<uintptr_t>(p) & 15)) return cudaErrorNotSupported;
  if (!tf32_supported(s, LINATTN_F32)) return cudaErrorNotSupported;
  if (s.dk <= 32)
    return state_only ? launch_v4<32, 4, 5, true>(q, k, v, o, log2g, s_in, s_out, s, sa, nz, stream)
                      : launch_v4<32, 4, 5, false>(q, k, v, o, log2g, s_in, s_out, s, sa, nz, stream);
  if (s.dk <= 64)
    return state_only ? launch_v4<64, 4, 4, true>(q, k, v, o, log2g, s_in, s_out, s, sa, nz, stream)
                      : launch_v4<64, 4, 4, false>(q, k, v, o, log2g, s_in, s_out, s, sa, nz, stream);
  return state_only ? launch_v4<128, 3, 2, true>(q, k, v, o, log2g, s_in, s_out, s, sa, nz, stream)
                    : launch_v4<128, 3, 2, false>(q, k, v, o, log2g, s_in, s_out, s, sa, nz, stream);
}

int tf32_balance_ctas(const ShapeArgs& s, int sms) {
  // one CTA per SM over equal chunk ranges when the (b, h, 128-wide dv tile) units do not fill whole
  // waves: the kernel is tensor-pipe bound, so a partly filled last wave idles SMs outright
  const int64_t units = s.B * s.H * ((s.dv + v4::kDVT - 1) / v4::kDVT), nc = (s.N + v4::kC - 1) / v4::kC;
  if (units <= sms || units % sms == 0 || units * nc > (1LL << 31) - 1) return 0;
  // measured (B200): 149 units x 8192 tokens 1.41 -> 0.87 ms balanced; configs[1] (256 units,
  // 1.73 waves) gains nothing (1.488 both: per-chunk time rises with the number of busy SMs, so
  // the light second wave of the plain grid already runs faster), hence the margin
  const double plain = (double)((units + sms - 1) / sms) * (double)nc;
  const double bal = (double)((units * nc + sms - 1) / sms);
  return bal < 0.8 * plain ? sms : 0;
}

size_t tf32_balance_workspace_bytes(const ShapeArgs& s, int ctas) {
  return 256 * (size_t)((ctas + 1 + 63) / 64) + (size_t)ctas * s.dk * v4::kDVT * sizeof(float);
}

cudaError_t launch_prefill_tf32_balanced(const void* q, const void* k, const void* v, void* o, const float* log2g,
                                         const float* s_in, float* s_out, const ShapeArgs& s, int ctas, void* ws,
                                         cudaStream_t stream) {
  for (const void* p : {q, k, v, (const void*)o})
    if (reinterpret_cast<uintptr_t>(p) & 15) return cudaErrorNotSupported;
  if (!tf32_supported(s, LINATTN_F32)) return cudaErrorNotSupported;
  const int64_t ntiles = (s.dv + v4::kDVT - 1) / v4::kDVT;
  const int64_t units = s.B * s.H * ntiles, nc = (s.N + v4::kC - 1) / v4::kC;
  const int64_t w = (units * nc + ctas - 1) / ctas;
  if (w < nc || units * nc > (1LL << 31) - 1) return cudaErrorNotSupported;
  Balance bal;
  bal.on = 1;
  bal.units = (int)units;
  bal.nc = (int)nc;
  bal.w = (int)w;
  bal.ntiles = (int)ntiles;
  bal.chunk = v4::kC;
  bal.tile = v4::kDVT;
  bal.flags = static_cast<unsigned*>(ws);
  bal.hst = reinterpret_cast<float*>(static_cast<uint8_t*>(ws) + 256 * (size_t)((ctas + 1 + 63) / 64));
  const int used = (int)((units * nc + w - 1) / w);
  cudaError_t err = cudaMemsetAsync(ws, 0, sizeof(unsigned) * (ctas + 1), stream);
  if (err != cudaSuccess) return err;
  const SegArgs sa{};
  if (s.dk <= 32) return launch_v4<32, 4, 5, false, true>(q, k, v, o, log2g, s_in, s_out, s, sa, 1, stream, bal, used);
  if (s.dk <= 64) return launch_v4<64, 4, 4, false, true>(q, k, v, o, log2g, s_in, s_out, s, sa, 1, stream, bal, used);
  return launch_v4<128, 3, 2, false, true>(q, k, v, o, log2g, s_in, s_out, s, sa, 1, stream, bal, used);
}

}  // namespace linattn
