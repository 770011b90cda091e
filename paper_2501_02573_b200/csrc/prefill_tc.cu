// K1 (+K2, K4): tensor-core chunked prefill for sm_100a -- TMA + tcgen05 + TMEM.
//
// One CTA owns one (batch*head, 128-wide dv tile, sequence segment) unit and walks its tokens in
// chunks of C = 64 (the reference default, kernels.py:57).  The algebra is the reference
// two-level-block method (kernels.py:139-166) written TRANSPOSED so every accumulator has
// M = 128 TMEM lanes (lane = dv row) while the chunk stays at 64:
//
//   MMA1  P^T[s][t]   = sum_i K[s][i] Q[t][i]              (M=128 (64 live), N=64, K=dk)
//   epi1  P^T[s][t]  *= gamma^(t-s) for t >= s else 0      (mask built from a gamma^n table)
//   MMA2  Oi^T[d][t]  = sum_s V[s][d] P^T[s][t]             (M=128, N=64, K=64)
//         Ox^T[d][t]  = sum_i S^T[d][i] Q[t][i]             (A = bf16 S^T in TMEM)
//         S^T[d][i]  <- gamma^L S^T + sum_s gamma^(L-1-s) V[s][d] K[s][i]
//   out   O[t][d]     = Oi^T[d][t] + gamma^(t+1) Ox^T[d][t]
//
// v2:  dk <= 128 (configs[1], configs[4]) -- running state in registers of 8 state warps.
// v3:  dk = 256 (configs[2]) -- state in TMEM, lazy scalar decay normalisation, 4-CTA clusters
//      sharing Q/K by TMA multicast.
// Both take a SegArgs geometry (blockIdx.z = segment) for the sequence split.
#include <cstdlib>
#include <mutex>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "sm100.cuh"

#ifndef V3_PUB_ILP
#define V3_PUB_ILP 0
#endif
#ifndef V3_PACK_ALU
#define V3_PACK_ALU 0
#endif
#ifndef V3_PF_AHEAD
#define V3_PF_AHEAD 2     // dk = 256: L2 prefetch distance (chunks) of the Q/K ring; 0 = off
#endif
#ifndef TC_SMEM_SPACE
#define TC_SMEM_SPACE 1
#endif

namespace linattn {
namespace {

using namespace sm100;

constexpr int kC = 64;          // tokens per chunk
constexpr int kDVT = 128;       // dv rows per CTA (MMA M)
constexpr uint32_t kTmemCols = 512;
// ============================================================================================
// Pipelined variant for dk <= 128 (the configs[1] hot path).  Same algebra, organised so the
// per-chunk serial chain is short and every epilogue is a few instructions per element:
//   * the running state S lives in REGISTERS of 8 state warps (fp32); the tensor pipe only
//     produces dS_c = V^T K'_c into a TMEM scratch, so the state update never round-trips
//     through TMEM and never blocks the next chunk's MMAs;
//   * P^T and both output accumulators (Oi = V^T P^T, Ox = S^T Q^T) are double-buffered in
//     TMEM (P^T x2, Oi x2, Ox x2, dS = 512 columns) and MMA1 of chunk c+1 runs ahead;
//   * decay masks are applied as packed bf16x2 multiplies from a (gamma^k, gamma^(k+1)) table
//     (P^T and K'); the inter-chunk weight gamma^(t+1) is applied exactly in fp32 when the
//     output tile is combined;
//   * outputs leave through tcgen05.ld.16x256b -> stmatrix.trans -> TMA bulk store.
// Per-chunk critical chain: publish S_c -> {O_c, dS_c} MMAs -> state warps load dS_c ->
// publish S_{c+1}.
// Warp roles (448 threads): 0-1 P^T mask, 2-3 K' scaling, 4-11 state + outputs,
// 12 TMA producer, 13 MMA issuer / TMEM owner.
namespace v2 {

constexpr int kThreads = 448;
#ifndef V2_OT_BUFS
#define V2_OT_BUFS 1
#endif
constexpr int kOtBufs = V2_OT_BUFS;     // output staging tiles (2: a store never blocks the next chunk)
// TMEM column map: P^T | O_inter | O_intra x2 | dS | S^T (bf16 A operand) x2.  O_inter = S_c^T Q^T
// is kept apart so gamma^(t+1) is applied in fp32 in the output epilogue instead of rescaling Q
// in shared memory (a 32 KiB read-modify-write per chunk on the mask warps' path).
constexpr uint32_t T_P = 0, T_OX = 64, T_O = 128, T_DS = 256, T_ST = 384;

// SO = state-only instantiation: no Q slot in the ring, so the same shared memory holds more
// K/V stages (the state pass is bound by how many bytes each SM keeps in flight).
template <int DK, int STAGES, bool SO = false>
struct Cfg {
  static constexpr int KB = DK / 64;
  static constexpr int Q_BYTES = SO ? 0 : kC * DK * 2;
  static constexpr int K_BYTES = kC * DK * 2;
  static constexpr int V_BYTES = kC * kDVT * 2;
  static constexpr int STAGE_BYTES = Q_BYTES + K_BYTES + V_BYTES;
  static constexpr int PT_BYTES = kC * kC * 2;
  static constexpr int OT_BYTES = kC * kDVT * 2;    // one output staging tile [64 t][128 d]
  static constexpr int OFF_PT = STAGES * STAGE_BYTES;
  static constexpr int OFF_OT = OFF_PT + 2 * PT_BYTES;
  static constexpr int OT_BUFS =                               // double-buffer the output tile if it fits
      (OFF_OT + kOtBufs * OT_BYTES + 128 * 4 + 192 * 4 + 512 + 1024 <= 227 * 1024) ? kOtBufs : 1;
  static constexpr int OFF_POW = OFF_OT + OT_BUFS * OT_BYTES; // fp32 gamma^n, n = 0..64
  static constexpr int OFF_POW2 = OFF_POW + 128 * 4;          // bf16x2 (gamma^k, gamma^(k+1)), k = -64..127
  static constexpr int OFF_BAR = OFF_POW2 + 192 * 4;
  static constexpr int SMEM = OFF_BAR + 512 + 1024;
};

__device__ __forceinline__ uint32_t hmul2_bf16(uint32_t a, uint32_t b) {
  uint32_t r;
  asm("mul.rn.bf16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}

// BAL: balanced persistent work list (Balance); false = one unit per CTA from blockIdx, where
// every item field is a compile-time-known function of blockIdx (no extra live registers).
template <int DK, int STAGES, bool SO, bool BAL, bool PADK>
__global__ void __launch_bounds__(kThreads, 1)
prefill_tc_pipe_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                       const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_o,
                       const float* __restrict__ log2g, const float* __restrict__ s_in,
                       float* __restrict__ s_out, int H, int N, int dv, int dk_arg, int state_only,
                       const SegArgs sa, const Balance bal, unsigned long long* __restrict__ trace,
                       unsigned long long* __restrict__ nonfinite) {
  using G = Cfg<DK, STAGES, SO>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
#if TC_SMEM_SPACE
  // aligned by pointer arithmetic so ptxas keeps the shared address space (LDS/STS, not generic)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
#else
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
#endif
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + G::OFF_BAR);
  uint64_t* empty = full + STAGES;
  uint64_t* mma1_bar = empty + STAGES;   // P^T accumulator ready (single buffer)
  // [STAGES] stage s: P^T smem written, K' scaled (64 or 128 arrivals).  Indexed by stage, not
  // by P^T buffer: in the state pass nothing else paces the K' warps, and a barrier indexed by
  // c & 1 could complete two phases before the MMA warp observes the first (lapping).
  uint64_t* epi1_bar = mma1_bar + 2;
  uint64_t* mma_s_bar = epi1_bar + STAGES;  // dS_c ready
  uint64_t* ds_free = mma_s_bar + 1;     // dS read by the state warps            (256 arrivals)
  uint64_t* st_full = ds_free + 1;       // [2] S^T bf16 operand b published (TMEM) (256 arrivals)
  uint64_t* mma_o_bar = st_full + 2;     // [2] O accumulator b ready
  uint64_t* o_free = mma_o_bar + 2;      // [2] O_intra accumulator b drained     (256 arrivals)
  uint64_t* ox_free = o_free + 2;        // O_inter accumulator drained            (256 arrivals)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(ox_free + 1);
  // work-list header {ticket, items, range start, range end}: re-read from shared memory at each
  // item boundary so none of it stays live in registers across the chunk loops
  int* wl = reinterpret_cast<int*>(tmem_slot + 2);
  float* pw = reinterpret_cast<float*>(smem + G::OFF_POW);
  uint32_t* pw2 = reinterpret_cast<uint32_t*>(smem + G::OFF_POW2) + 64;   // pw2[k], k in [-64, 127]
  uint8_t* pt_smem = smem + G::OFF_PT;
  uint8_t* ot_smem = smem + G::OFF_OT;

  const uint32_t warp = warp_id();
  const uint32_t lane = threadIdx.x & 31;
  // PADK: dk < DK (Q/K boxes past dk are TMA zero fill); external states are [BH][dkr][dv]
  const int dkr = PADK ? dk_arg : DK;
  const size_t per_state = (size_t)gridDim.y * dkr * dv;

  if (warp == 12 && lane == 0) {
    // balanced schedule: tickets in start order, so the range before ours is already running
    if constexpr (BAL) {
      const int t = (int)atomicAdd(bal.flags + gridDim.x, 1u);
      long long r0 = 0, r1 = 0;
      wl[1] = balance_items(bal, t, r0, r1);
      wl[0] = t;
      reinterpret_cast<long long*>(wl)[1] = r0;
      reinterpret_cast<long long*>(wl)[2] = r1;
    } else {
      wl[1] = 1;
    }
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
      mbar_init(&epi1_bar[i], 128);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&mma1_bar[b], 1);
      mbar_init(&o_free[b], 256);
      mbar_init(&mma_o_bar[b], 1);
    }
    mbar_init(ox_free, 256);
    mbar_init(mma_s_bar, 1);
    mbar_init(ds_free, 256);
    mbar_init(&st_full[0], 256);
    mbar_init(&st_full[1], 256);
    fence_barrier_init();
    if (!state_only) {
      tma_prefetch_desc(&tm_q);
      tma_prefetch_desc(&tm_o);
    }
    tma_prefetch_desc(&tm_k);
    tma_prefetch_desc(&tm_v);
  }
  if (warp == 13) tmem_alloc<kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;
  if constexpr (!BAL) pdl_wait();   // everything above overlapped the previous kernel's tail
  // work list: the one unit of blockIdx (SegArgs segment blockIdx.z), or this ticket's range
  const int nitems = BAL ? wl[1] : 1;
  auto item = [&](int k) {
    if constexpr (BAL) {
      const volatile int* v = wl;
      const volatile long long* r = reinterpret_cast<const volatile long long*>(wl);
      return balance_item(bal, N, v[0], k, r[1], r[2]);
    }
    WorkItem w;
    w.bh = blockIdx.y;
    w.j0 = blockIdx.x * kDVT;
    seg_bounds(sa.seg_len, sa.sub, sa.m, blockIdx.z, N, w.lo, w.hi);  // multiples of kC except N
    w.in_slot = w.out_slot = -1;
    return w;
  };
  auto item_chunks = [&](const WorkItem& w) { return w.hi > w.lo ? (w.hi - w.lo + kC - 1) / kC : 0; };
  // debug trace of one CTA: (bh = trace[15 * 4096], dv tile 0, segment 0); trace[15 * 4096] is set by the host
  // (balanced launches: the CTA whose ticket is trace[15 * 4096]; events indexed by global chunk)
  const bool tracing = trace != nullptr &&
                       (BAL ? wl[0] == (int)trace[15 * 4096]
                            : blockIdx.x == 0 && blockIdx.z == 0 && blockIdx.y == (unsigned)trace[15 * 4096]);
  const int lin_block = blockIdx.y * gridDim.x + blockIdx.x;
  auto gtime = [] {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
  };
  if (trace != nullptr && threadIdx.x == 0 && lin_block < 4096) {
    unsigned smid;
    asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
    trace[8 * 4096 + lin_block] = gtime();
    trace[0 * 4096 + lin_block] = smid;
  }

  if (warp < 4) {
    // ------------------------------------------------------------ P^T mask / K' scaling
    int gc = 0;                                     // chunk counter over the whole work list
    for (int it = 0; it < nitems; ++it) {
     const WorkItem w = item(it);
     {
      // this role's (gamma^k, gamma^(k+1)) table for the item's head, k = -64..127
      const float lg = log2g[w.bh % H];
      if (it > 0) named_bar_sync(4, 128);           // every mask thread is done with the old table
      for (int i = (int)threadIdx.x; i < 192; i += 128) {
        const int k = i - 64;
        pw2[k] = pack_bf16x2(k >= 0 ? gpow(lg, (float)k) : 0.f, k + 1 >= 0 ? gpow(lg, (float)(k + 1)) : 0.f);
      }
      named_bar_sync(4, 128);
     }
     const int nch = item_chunks(w);
     for (int c = 0; c < nch; ++c, ++gc) {
      const int s = gc % STAGES;
      const int b = gc & 1;
      const int L = min(kC, w.hi - w.lo - c * kC);
      mbar_wait(&full[s], (gc / STAGES) & 1);
      if (!state_only) {
        mbar_wait(mma1_bar, gc & 1);                // MMA1 has consumed the unscaled K
        tc_fence_after();
      }
      if (warp < 2 && !state_only) {
        // P^T[s][t] *= gamma^(t-s) (t >= s), bf16: row s of the MN-major B operand of Oi
        const int srow = warp * 32 + lane;
        const uint32_t ta = tbase + ((warp * 32) << 16) + T_P;
        uint8_t* row = pt_smem + b * G::PT_BYTES + srow * 128;
#pragma unroll
        for (int half = 0; half < 2; ++half) {
          float p[32];
          tmem_ld32(ta + half * 32, p);
          tmem_wait_ld();
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int t0 = half * 32 + 8 * j;
            uint4 pk;
            pk.x = hmul2_bf16(pack_bf16x2(p[8 * j + 0], p[8 * j + 1]), pw2[t0 + 0 - srow]);
            pk.y = hmul2_bf16(pack_bf16x2(p[8 * j + 2], p[8 * j + 3]), pw2[t0 + 2 - srow]);
            pk.z = hmul2_bf16(pack_bf16x2(p[8 * j + 4], p[8 * j + 5]), pw2[t0 + 4 - srow]);
            pk.w = hmul2_bf16(pack_bf16x2(p[8 * j + 6], p[8 * j + 7]), pw2[t0 + 6 - srow]);
            *reinterpret_cast<uint4*>(row + (((half * 4 + j) ^ (srow & 7)) << 4)) = pk;
          }
        }
      } else if (!state_only) {
        // K'[s] = gamma^(L-1-s) K[s], zero beyond the ragged end (in place, bf16x2 multiplies)
        const int srow = (warp - 2) * 32 + lane;
        const uint32_t w2 = pw2[srow < L ? L - 1 - srow : -64];     // pw2[-64] = (0, 0)
        const uint32_t wk = (w2 & 0xFFFFu) | (w2 << 16);
        uint8_t* k_smem = smem + s * G::STAGE_BYTES + G::Q_BYTES;
        uint4 x[G::KB * 8];                       // issue every load before the first store
#pragma unroll
        for (int kb = 0; kb < G::KB; ++kb)
#pragma unroll
          for (int j = 0; j < 8; ++j)
            x[kb * 8 + j] = *reinterpret_cast<const uint4*>(k_smem + kb * 8192 + srow * 128 + ((j ^ (srow & 7)) << 4));
#pragma unroll
        for (int kb = 0; kb < G::KB; ++kb)
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            uint4 y = x[kb * 8 + j];
            y.x = hmul2_bf16(y.x, wk);
            y.y = hmul2_bf16(y.y, wk);
            y.z = hmul2_bf16(y.z, wk);
            y.w = hmul2_bf16(y.w, wk);
            *reinterpret_cast<uint4*>(k_smem + kb * 8192 + srow * 128 + ((j ^ (srow & 7)) << 4)) = y;
          }
      }
      if (state_only) {
        // state pass: no P^T, so all four warps share K' (thread -> row, 64-column block)
        const int tid = (int)warp * 32 + (int)lane;
        const int srow = tid & 63;
        const uint32_t w2 = pw2[srow < L ? L - 1 - srow : -64];
        const uint32_t wk = (w2 & 0xFFFFu) | (w2 << 16);
        uint8_t* k_smem = smem + s * G::STAGE_BYTES + G::Q_BYTES;
        for (int kb = tid >> 6; kb < G::KB; kb += 2) {
          uint4 x[8];
#pragma unroll
          for (int j = 0; j < 8; ++j)
            x[j] = *reinterpret_cast<const uint4*>(k_smem + kb * 8192 + srow * 128 + ((j ^ (srow & 7)) << 4));
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            x[j].x = hmul2_bf16(x[j].x, wk);
            x[j].y = hmul2_bf16(x[j].y, wk);
            x[j].z = hmul2_bf16(x[j].z, wk);
            x[j].w = hmul2_bf16(x[j].w, wk);
            *reinterpret_cast<uint4*>(k_smem + kb * 8192 + srow * 128 + ((j ^ (srow & 7)) << 4)) = x[j];
          }
        }
      }
      fence_proxy_async_smem();
      tc_fence_before();
      if (tracing && lane == 0 && gc < 4096) trace[(warp < 2 ? 3 : 4) * 4096 + gc] = clock64();
      mbar_arrive(&epi1_bar[s]);
     }
    }
  } else if (warp < 12) {
    // ------------------------------------------------------------ running state + outputs
    // warp (g, sub): TMEM lanes sub*32.. (dv rows d); state columns [g*SC, (g+1)*SC);
    // output rows d0 = sub*32 + g*16 .. +15 (a 16-lane half of the subpartition).
    constexpr int SC = DK / 2;
    const int g = (warp - 4) / 4;
    const int sub = (warp - 4) % 4;
    const int d = sub * 32 + lane;
    const int col0 = g * SC;
    const uint32_t ta_s = tbase + ((sub * 32) << 16) + T_DS + col0;
    const int d0 = sub * 32 + g * 16;
    const uint32_t ta_o = tbase + ((uint32_t)d0 << 16);
    const bool leader = (warp == 4 && lane == 0);
    const int sidx = (int)threadIdx.x - 128;     // 0..255 within the role
    // S (fp32 regs) -> bf16 pairs -> TMEM S^T operand buffer `buf` (row d, columns col0/2..)
    const uint32_t ta_st = tbase + ((sub * 32) << 16) + T_ST + col0 / 2;
    float S[SC];
    auto publish = [&](int buf) {
#pragma unroll
      for (int j = 0; j < SC / 32; ++j) {
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) pk[i] = pack_bf16x2(S[32 * j + 2 * i], S[32 * j + 2 * i + 1]);
        tmem_st16(ta_st + buf * (DK / 2) + 16 * j, pk);
      }
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(&st_full[buf]);
    };
    // stmatrix row address of this thread: matrix m = lane/8 of each x4 group, row lane%8
    const int mrow = lane & 7;
    const int mi = lane >> 3;                  // 0: (d0, t), 1: (d0+8, t), 2: (d0, t+8), 3: (d0+8, t+8)
    uint32_t out_bad = 0;                      // any non-finite output value seen (fused entry check)
    const int md = d0 + (mi & 1) * 8;          // 8-aligned dv row of the tile this address serves
    int gc = 0;
    for (int it = 0; it < nitems; ++it) {
      const WorkItem w = item(it);
      const int jd = w.j0 + d;
      const bool dv_ok = jd < dv;
      const float lg = log2g[w.bh % H];
      // this role's gamma^n table (n = 0..64) for the item's head; a seeded tail also waits here
      // for the previous range's published head state
      if (it > 0) named_bar_sync(3, 256);      // every state thread is done with the old table
      if (sidx <= kC) pw[sidx] = gpow(lg, (float)sidx);
      if (w.in_slot >= 0 && leader)
        while (ld_acquire_gpu(bal.flags + w.in_slot) == 0u) __nanosleep(256);
      named_bar_sync(3, 256);
      if (w.in_slot >= 0) {
        // balanced tail: the hand-off state already covers s_in and every earlier token
        const float* hp = bal.hst + ((size_t)w.in_slot * DK + col0) * kDVT + d;
#pragma unroll
        for (int i = 0; i < SC; ++i) S[i] = dv_ok ? __ldcg(hp + (size_t)i * kDVT) : 0.f;
      } else {
        // S_init = gamma^lo s_in + sum_{q: hi_q <= lo} gamma^(lo - hi_q) loc[q]  (SegArgs)
        const float w_in = gpow(lg, (float)w.lo);
#pragma unroll
        for (int j = 0; j < SC; j += 16) {
#pragma unroll
          for (int i = 0; i < 16; ++i)
            S[j + i] = (s_in && dv_ok && (!PADK || col0 + j + i < dkr)) ? w_in * s_in[((size_t)w.bh * dkr + col0 + j + i) * dv + jd] : 0.f;
          for (int qi = 0; qi < sa.nloc; ++qi) {
            const float wq = seg_loc_weight(sa, qi, N, w.lo, lg);
            if (wq < 0.f || !dv_ok) continue;
            const float* lq = sa.loc + qi * per_state + ((size_t)w.bh * dkr + col0 + j) * dv + jd;
#pragma unroll
            for (int i = 0; i < 16; ++i)
              if (!PADK || col0 + j + i < dkr) S[j + i] = fmaf(wq, lq[(size_t)i * dv], S[j + i]);
          }
        }
      }
      // end state (written after the last chunk): a balanced head publishes it to its hand-off
      // slot; otherwise state-only launches write one local state per segment and full launches
      // only the segment ending the sequence (whose seed already covers every earlier token)
#define LA_WRITE_STATE()                                                                              \
  do {                                                                                                \
    float* so = nullptr;                                                                              \
    size_t so_stride = dv;                                                                            \
    if (w.out_slot >= 0) {                                                                            \
      if (dv_ok) so = bal.hst + ((size_t)w.out_slot * DK + col0) * kDVT + d;                          \
      so_stride = kDVT;                                                                               \
    } else if (s_out && dv_ok && (BAL ? w.hi == N : (state_only || blockIdx.z == gridDim.z - 1))) { \
      so = s_out + (state_only ? blockIdx.z * per_state : 0) + ((size_t)w.bh * dkr + col0) * dv + jd; \
    }                                                                                                 \
    if (so != nullptr) { /* hand-off slots hold all DK rows, external states the dkr real ones */    \
      const int nrow = (!PADK || w.out_slot >= 0) ? SC : min(SC, dkr - col0);                         \
      _Pragma("unroll") for (int i = 0; i < SC; ++i) if (i < nrow) so[(size_t)i * so_stride] = S[i];  \
    }                                                                                                 \
    if (w.out_slot >= 0) { /* release the hand-off to the next range's tail */                       \
      __threadfence();                                                                                \
      named_bar_sync(5, 256);                                                                         \
      if (leader) st_release_gpu(bal.flags + w.out_slot, 1u);                                         \
    }                                                                                                 \
  } while (0)
      const int nch = item_chunks(w);
      if (!state_only && nch > 0) publish(gc & 1);
      for (int c = 0; c < nch; ++c, ++gc) {
        const int L = min(kC, w.hi - w.lo - c * kC);
        const int b = gc & 1;
        mbar_wait(mma_s_bar, gc & 1);
        tc_fence_after();
        const float carry = pw[L];
#pragma unroll
        for (int j = 0; j < SC / 16; ++j) {
          float ds[16];
          tmem_ld16(ta_s + 16 * j, ds);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 16; ++i) S[16 * j + i] = fmaf(carry, S[16 * j + i], ds[i]);
        }
        tc_fence_before();
        mbar_arrive(ds_free);
        if (tracing && lane == 0 && sub == 0 && g == 0 && gc < 4096) trace[6 * 4096 + gc] = clock64();
        if (state_only) continue;
        if (c != nch - 1) {
          // buffer (gc+1)&1 was last read by Ox_{gc-1}, which precedes dS_gc in the tensor pipe
          publish((gc + 1) & 1);
          if (tracing && lane == 0 && sub == 0 && g == 0 && gc < 4096) trace[7 * 4096 + gc] = clock64();
        }
        mbar_wait(&mma_o_bar[b], (gc >> 1) & 1);   // O_gc done
        tc_fence_after();
        // ---- outputs of chunk c: O = Oi + gamma^(t+1) Ox (16 lanes x 64 tokens) -> bf16 ->
        //      smem [t][d] (stmatrix.trans, 128B swizzle) -> TMA bulk store (clips N and dv)
        uint8_t* ot = ot_smem + (gc % G::OT_BUFS) * G::OT_BYTES;
        if (leader) bulk_wait_read<G::OT_BUFS - 1>();   // the store that last used this tile has read it
        named_bar_sync(1, 256);
#pragma unroll
        for (int q4 = 0; q4 < 2; ++q4) {           // tokens q4*32 .. q4*32+31
          uint32_t ro[16], rx[16];
          tmem_ld_16x256b_x4(ta_o + T_O + b * kC + q4 * 32, ro);
          tmem_ld_16x256b_x4(ta_o + T_OX + q4 * 32, rx);
          tmem_wait_ld();
          if (q4 == 1) {
            tc_fence_before();
            mbar_arrive(&o_free[b]);
            mbar_arrive(ox_free);
          }
          uint32_t pk[8];
#pragma unroll
          for (int r = 0; r < 4; ++r) {            // 8-token group r: t = q4*32 + 8r + tq + {0,1}
            // O = Oi + gamma^(t+1) Ox, in fp32 (the inter-chunk weight, reference w_t kernels.py:125)
            const int t0 = q4 * 32 + 8 * r + 2 * (lane & 3);
            const float w0 = pw[t0 + 1], w1 = pw[t0 + 2];
            pk[2 * r + 0] = pack_bf16x2(fmaf(w0, __uint_as_float(rx[4 * r + 0]), __uint_as_float(ro[4 * r + 0])),
                                        fmaf(w1, __uint_as_float(rx[4 * r + 1]), __uint_as_float(ro[4 * r + 1])));
            pk[2 * r + 1] = pack_bf16x2(fmaf(w0, __uint_as_float(rx[4 * r + 2]), __uint_as_float(ro[4 * r + 2])),
                                        fmaf(w1, __uint_as_float(rx[4 * r + 3]), __uint_as_float(ro[4 * r + 3])));
          }
          // entry-contract NaN/Inf check fused into the epilogue: every non-finite input reaches
          // some output, so a clean output proves clean inputs (bf16 exponent all ones)
#pragma unroll
          for (int i = 0; i < 8; ++i) out_bad |= __vcmpeq2(pk[i] & 0x7f807f80u, 0x7f807f80u);
#pragma unroll
          for (int rr = 0; rr < 4; rr += 2) {      // two 8-token groups per stmatrix.x4
            const int tt = q4 * 32 + rr * 8 + (mi >> 1) * 8 + mrow;     // token row this lane addresses
            const uint32_t addr = smem_u32(ot + (md / 64) * (kC * 128) + tt * 128 +
                                           ((((md % 64) >> 3) ^ (tt & 7)) << 4));
            stmatrix_x4_trans(addr, pk[2 * rr + 0], pk[2 * rr + 1], pk[2 * rr + 2], pk[2 * rr + 3]);
          }
        }
        fence_proxy_async_smem();
        named_bar_sync(2, 256);
        if (leader) {
          tma_store_3d(&tm_o, ot, w.j0, w.lo + c * kC, w.bh);
          tma_store_3d(&tm_o, ot + kC * 128, w.j0 + 64, w.lo + c * kC, w.bh);
          bulk_commit();
        }
        if (tracing && lane == 0 && sub == 0 && g == 0 && gc < 4096) trace[5 * 4096 + gc] = clock64();
      }
      LA_WRITE_STATE();
    }
    if (nonfinite != nullptr && __any_sync(0xffffffffu, out_bad != 0u) && lane == 0) atomicMin(nonfinite, 0ull);
    if (leader) bulk_wait<0>();
  } else {
    if (warp == 12) {
      // ---------------------------------------------------------- TMA producer
      if (lane == 0) {
        const uint32_t bytes = (state_only ? 0 : G::Q_BYTES) + G::K_BYTES + G::V_BYTES;
        int gc = 0;
        for (int it = 0; it < nitems; ++it) {
          const WorkItem w = item(it);
          const int nch = item_chunks(w);
          for (int c = 0; c < nch; ++c, ++gc) {
            const int s = gc % STAGES;
            const int t0 = w.lo + c * kC;
            mbar_wait(&empty[s], ((gc / STAGES) & 1) ^ 1);
            if (tracing && gc < 4096) trace[13 * 4096 + gc] = clock64();
            uint8_t* st = smem + s * G::STAGE_BYTES;
            mbar_arrive_expect_tx(&full[s], bytes);
#pragma unroll
            for (int kb = 0; kb < G::KB; ++kb) {
              if (!state_only) tma_load_3d(st + kb * 8192, &tm_q, &full[s], kb * 64, t0, w.bh);
              tma_load_3d(st + G::Q_BYTES + kb * 8192, &tm_k, &full[s], kb * 64, t0, w.bh);
            }
#pragma unroll
            for (int nb = 0; nb < kDVT / 64; ++nb)
              tma_load_3d(st + G::Q_BYTES + G::K_BYTES + nb * 8192, &tm_v, &full[s], w.j0 + nb * 64, t0, w.bh);
          }
        }
      }
    } else if (warp == 13) {
      // ---------------------------------------------------------- MMA issuer (whole warp)
      // Descriptors are built once; a K step only adds (byte offset >> 4) to the start-address
      // field (smem addresses < 256 KiB, so the 14-bit field never carries).
      constexpr uint32_t id_qk = idesc_bf16(128, kC, false, false);   // P^T = K Q^T
      constexpr uint32_t id_vp = idesc_bf16(128, kC, true, true);     // O^T  = V^T P^T
      constexpr uint32_t id_sq = idesc_bf16(128, kC, false, false);   // Ox^T = S^T(TMEM) Q^T
      constexpr uint32_t id_vk = idesc_bf16(128, DK, true, true);     // dS^T = V^T K'
      const uint32_t base_addr = smem_u32(smem);
      const uint64_t dq0 = smem_desc_sw128(base_addr, 16, 1024);                          // K-major rows
      const uint64_t dmn0 = smem_desc_sw128(base_addr, 8192, 1024);                       // MN-major
      const uint64_t dpt0 = smem_desc_sw128(smem_u32(pt_smem), 8192, 1024);
      constexpr uint64_t kStage = G::STAGE_BYTES >> 4, kQ = G::Q_BYTES >> 4, kK = G::K_BYTES >> 4;
      auto issue_mma1 = [&](int c) {
        const int s = c % STAGES;
        mbar_wait(&full[s], (c / STAGES) & 1);
        if (tracing && lane == 0 && c < 4096) trace[10 * 4096 + c] = clock64();
        tc_fence_after();
        const uint64_t dq = dq0 + s * kStage, dk = dq + kQ;
#pragma unroll
        for (int kb = 0; kb < G::KB; ++kb)
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            mma_bf16_ss_elect(tbase + T_P, dk + (kb * 512 + kk * 2), dq + (kb * 512 + kk * 2), id_qk,
                              (kb | kk) != 0);
        mma_commit_elect(mma1_bar);
        if (tracing && lane == 0 && c < 4096) trace[11 * 4096 + c] = clock64();
      };
      // the tensor pipe sees one flat chunk stream across the work list (c counts every chunk)
      int nchunks = 0;
      for (int it = 0; it < nitems; ++it) nchunks += item_chunks(item(it));
      // lane-0 broadcast: a provably warp-uniform chunk count keeps the descriptors in uniform
      // registers (otherwise ptxas wraps every tcgen05.mma of the balanced build in an R2UR loop)
      nchunks = __shfl_sync(0xffffffffu, nchunks, 0);
      if (!state_only && nchunks > 0) issue_mma1(0);
      for (int c = 0; c < nchunks; ++c) {
        const int s = c % STAGES;
        const int b = c & 1;
        const uint64_t dq = dq0 + s * kStage;                 // Q, K-major
        const uint64_t dv_mn = dmn0 + s * kStage + kQ + kK;   // V, MN-major (A of V^T x)
        const uint64_t dk_mn = dmn0 + s * kStage + kQ;        // K', MN-major (B of V^T K')
        if (state_only) mbar_wait(&full[s], (c / STAGES) & 1);
        mbar_wait(&epi1_bar[s], (c / STAGES) & 1);     // P^T_c in smem (TMEM copy free), K'_c scaled
        if (tracing && lane == 0 && c < 4096) trace[12 * 4096 + c] = clock64();
        // P^T TMEM is free again: start MMA1 of the next chunk before this chunk's dS, so its
        // mask epilogue overlaps the state chain instead of following it
        if (!state_only && c + 1 < nchunks) issue_mma1(c + 1);
        if (c > 0) mbar_wait(ds_free, (c - 1) & 1);    // state warps hold dS_{c-1}
        tc_fence_after();
        if (tracing && lane == 0 && c < 4096) trace[1 * 4096 + c] = clock64();
#pragma unroll
        for (int ks = 0; ks < kC / 16; ++ks)
          mma_bf16_ss_elect(tbase + T_DS, dv_mn + ks * 128, dk_mn + ks * 128, id_vk, ks != 0);
        mma_commit_elect(mma_s_bar);
        if (!state_only) {
          mbar_wait(&st_full[b], (c >> 1) & 1);        // S_c (bf16) published in TMEM buffer b
          if (tracing && lane == 0 && c < 4096) trace[14 * 4096 + c] = clock64();
          if (c >= 2) mbar_wait(&o_free[b], ((c >> 1) - 1) & 1);
          if (c >= 1) mbar_wait(ox_free, (c - 1) & 1);
          tc_fence_after();
          if (tracing && lane == 0 && c < 4096) trace[2 * 4096 + c] = clock64();
          const uint64_t dpt = dpt0 + b * (G::PT_BYTES >> 4);
#pragma unroll
          for (int ks = 0; ks < kC / 16; ++ks)
            mma_bf16_ss_elect(tbase + T_O + b * kC, dv_mn + ks * 128, dpt + ks * 128, id_vp, ks != 0);
#pragma unroll
          for (int kb = 0; kb < G::KB; ++kb)
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              mma_bf16_ts_elect(tbase + T_OX, tbase + T_ST + b * (DK / 2) + (kb * 4 + kk) * 8,
                                dq + (kb * 512 + kk * 2), id_sq, (kb | kk) != 0);
          mma_commit_elect(&mma_o_bar[b]);
        }
        mma_commit_elect(&empty[s]);
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (trace != nullptr && threadIdx.x == 0 && lin_block < 4096) trace[9 * 4096 + lin_block] = gtime();
  if (warp == 13) tmem_dealloc<kTmemCols>(tbase);
}

}  // namespace v2

// ============================================================================================
// dk = 256 (configs[2], RetNet-shaped heads).  The per-CTA state S^T [128 dv][256 dk] fp32 is
// 128 KiB -- half the register file -- so it lives in TMEM and the tensor pipe accumulates
// into it directly:
//   state warps   S_c (TMEM fp32) -> bf16 S_c^T operand (TMEM) ; S <- gamma^L S (in place)
//   MMA2          O^T  = V^T P^T + S_c^T Q'^T     (TS form: A = bf16 S^T from TMEM)
//                 S^T += V^T K'                    (accumulates onto the rescaled state)
// TMEM (512 cols): P^T 64 | O 64 | S fp32 256 | S^T bf16 128 -- single-buffered.  The chain
// per chunk is {state warps: ld/st 128 KiB of TMEM} -> {MMA2}; MMA1 of the next chunk and the
// mask / Q' / K' epilogue run in its shadow, outputs drain on their own warps.
// Warp roles (448 threads): 0-1 P^T mask + Q', 2-3 K', 4-7 state, 8-11 outputs,
// 12 TMA producer, 13 MMA issuer / TMEM owner.
namespace v3 {

// Warp roles (512 threads = 4 warpgroups, 128 registers): 0-1 V' scaling and P^T mask,
// 2 TMA producer, 3 MMA issuer / TMEM owner, 4-11 state (two per TMEM subpartition),
// 12-15 inter-chunk column scaling and the output drain.  Pipe order per chunk:
//   S update (V'^T K) -> O_inter = S^T Q^T (unscaled Q) -> MMA1(c+1) -> O_intra = V^T P^T.
// Between O_inter and O_intra the aux warps scale O column t by gamma^(t+1) in TMEM (fp32),
// so Q is never rescaled in shared memory (that rescale was 128 KiB of smem traffic a chunk).
// The state warps publish bf16 S_{c+1} as soon as O_inter(c) has read the operand.
constexpr int kThreads = 512;
constexpr uint32_t T_P = 0, T_O = 64, T_S = 128, T_SB = 384;

// Two TMA rings: Q+K (STAGES x 64 KiB, released after O_inter) and V (VST x 16 KiB, released
// after O_intra), so the next Q/K loads start a whole O_intra earlier than with one ring.
constexpr int VST = 3;

template <int DK, int STAGES>
struct Cfg {
  static constexpr int KB = DK / 64;
  static constexpr int Q_BYTES = kC * DK * 2;
  static constexpr int K_BYTES = kC * DK * 2;
  static constexpr int V_BYTES = kC * kDVT * 2;
  static constexpr int STAGE_BYTES = Q_BYTES + K_BYTES;
  static constexpr int PT_BYTES = kC * kC * 2;
  static constexpr int OT_BYTES = kC * kDVT * 2;
  static constexpr int OFF_V = STAGES * STAGE_BYTES;
  static constexpr int OFF_PT = OFF_V + VST * V_BYTES;
  static constexpr int OFF_VS = OFF_PT + 2 * PT_BYTES;         // V' = gamma^(L-1-s) V[s] (S update operand)
  static constexpr int OFF_OT = OFF_VS + V_BYTES;
  static constexpr int OFF_POW = OFF_OT + OT_BYTES;
  static constexpr int OFF_POW2 = OFF_POW + 128 * 4;
  static constexpr int OFF_BAR = OFF_POW2 + 192 * 4;
  static constexpr int SMEM = OFF_BAR + 512 + 1024;
};

// dst row `row`, 64-column blocks [nb0, nb0 + NB) of a SW128 bf16 tile: dst = (w, w) * src
template <int NB>
__device__ __forceinline__ void scale_row_blocks(const uint8_t* src, uint8_t* dst, int row, int nb0, uint32_t w2) {
  uint4 x[NB * 8];
#pragma unroll
  for (int kb = 0; kb < NB; ++kb)
#pragma unroll
    for (int j = 0; j < 8; ++j)
      x[kb * 8 + j] = *reinterpret_cast<const uint4*>(src + (nb0 + kb) * 8192 + row * 128 + ((j ^ (row & 7)) << 4));
#pragma unroll
  for (int kb = 0; kb < NB; ++kb)
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      uint4 y = x[kb * 8 + j];
      y.x = v2::hmul2_bf16(y.x, w2);
      y.y = v2::hmul2_bf16(y.y, w2);
      y.z = v2::hmul2_bf16(y.z, w2);
      y.w = v2::hmul2_bf16(y.w, w2);
      *reinterpret_cast<uint4*>(dst + (nb0 + kb) * 8192 + row * 128 + ((j ^ (row & 7)) << 4)) = y;
    }
}

__device__ __forceinline__ uint32_t dup_lo(uint32_t w2) { return (w2 & 0xFFFFu) | (w2 << 16); }

// fp32 pair -> bf16x2 (round to nearest even) for the state publish: F2FP (cvt.rn.bf16x2.f32), or
// with V3_PACK_ALU the same rounding on the integer pipes (F2FP showed as 14% of the issued
// instructions of this kernel)
__device__ __forceinline__ uint32_t pack_bf16x2_pub(float lo, float hi) {
#if V3_PACK_ALU
  uint32_t a = __float_as_uint(lo), b = __float_as_uint(hi);
  a += 0x7fffu + ((a >> 16) & 1u);
  b += 0x7fffu + ((b >> 16) & 1u);
  return __byte_perm(a, b, 0x7632);
#else
  return pack_bf16x2(lo, hi);
#endif
}

// Lazy decay normalisation.  gamma is a per-head SCALAR, so the state is kept as S_c = sig_c T_c:
// the update S_{c+1} = gamma^L S_c + V'^T K becomes T_{c+1} = T_c + (V'/sig_{c+1})^T K with
// sig_{c+1} = sig_c gamma^L -- the 1/sig factor rides on V' (16 KiB, already rescaled every
// chunk) and sig_c on the O_inter column scale, so the 128 KiB TMEM state is not rewritten.
// When sig would drop below kSigMin (or gamma^L itself is tiny, e.g. gamma = 0) the chunk
// renormalises: T <- sig gamma^L T in TMEM and sig = 1.  Every role walks the same sequence.
constexpr float kSigMin = 0x1p-40f;
struct Lazy {
  float sig = 1.f;      // sig_c of the chunk about to be processed
  float sig_c = 1.f;    // sig_c saved for this chunk's O_inter scale
  float vfac = 1.f;     // factor on V'_c (1 / sig_{c+1}, or 1 when renormalising)
  float rescale = 1.f;  // T_c multiplier when renormalising
  bool renorm = false;
  __device__ __forceinline__ void step(float gL) {
    sig_c = sig;
    const float sn = sig * gL;
    renorm = !(sn >= kSigMin);
    rescale = sn;
    vfac = renorm ? 1.f : 1.f / sn;
    sig = renorm ? 1.f : sn;
  }
};

// MC = CTAs per cluster sharing each Q/K tile: the dv tiles of one head (blockIdx.x = cluster
// rank).  Each CTA loads KB/MC of the 64-column Q/K boxes and multicasts them to all MC CTAs, so
// L2 -> SM traffic for Q/K drops MC-fold; a stage is refilled only once every CTA released it
// (tcgen05.commit multicast into each CTA's `empty`, arrival count MC).
// BAL: balanced persistent schedule over cluster ranges (Balance mode 0: unit = (b*h, group of MC
// dv tiles), tile = MC*128, hand-off slots per CTA = ticket*MC + cluster rank, gamma tables per
// head in global memory because three roles read them across item boundaries).
template <int DK, int STAGES, int MC, bool BAL, bool PADK>
__global__ void __launch_bounds__(kThreads, 1)
prefill_tc_tmem_state_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                             const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_o,
                             const float* __restrict__ log2g, const float* __restrict__ s_in,
                             float* __restrict__ s_out, int H, int N, int dv, int dk_arg, int state_only,
                             const SegArgs sa, const Balance bal, unsigned long long* __restrict__ trace) {
  using G = Cfg<DK, STAGES>;
  static_assert(DK % 128 == 0 && kDVT == 128, "layout: two state warps per TMEM subpartition");
  static_assert(G::KB % MC == 0, "Q/K boxes split evenly over the cluster");
  constexpr uint16_t kMask = (uint16_t)((1u << MC) - 1);
  constexpr int SCOL = DK / 2;                     // state columns per state warp
  extern __shared__ __align__(1024) uint8_t smem_raw[];
#if TC_SMEM_SPACE
  // aligned by pointer arithmetic so ptxas keeps the shared address space (LDS/STS, not generic)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
#else
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
#endif
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + G::OFF_BAR);   // Q/K ring
  uint64_t* empty = full + STAGES;
  uint64_t* vfull = empty + STAGES;        // [VST] V ring
  uint64_t* vempty = vfull + VST;
  uint64_t* pt_bar = vempty + VST;         // [STAGES] P^T smem (buffer c&1) written (64)
  uint64_t* vs_bar = pt_bar + STAGES;      // [STAGES] V' written                    (64)
  uint64_t* mma1_bar = vs_bar + STAGES;    // P^T accumulator ready
  uint64_t* st_done = mma1_bar + 1;        // S_c published (bf16) and rescaled     (256)
  uint64_t* mma_s_bar = st_done + 1;       // S_{c+1} = gamma^L S_c + V'^T K done
  uint64_t* ox_bar = mma_s_bar + 1;        // O_inter(c) done (bf16 S operand free)
  uint64_t* ox_scaled = ox_bar + 1;        // O column t scaled by gamma^(t+1)       (128)
  uint64_t* mma_o_bar = ox_scaled + 1;     // O_intra(c) done: O_c complete
  uint64_t* o_free = mma_o_bar + 1;        // O drained                              (128)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_free + 1);
  float* pw = reinterpret_cast<float*>(smem + G::OFF_POW);
  uint32_t* pw2 = reinterpret_cast<uint32_t*>(smem + G::OFF_POW2) + 64;
  uint8_t* pt_smem = smem + G::OFF_PT;
  uint8_t* vs_smem = smem + G::OFF_VS;
  uint8_t* ot_smem = smem + G::OFF_OT;

  const uint32_t warp = warp_id();
  const uint32_t lane = threadIdx.x & 31;
  // PADK: dk < DK (Q/K boxes past dk are TMA zero fill); external states are [BH][dkr][dv]
  const int dkr = PADK ? dk_arg : DK;
  const size_t per_state = (size_t)gridDim.y * dkr * dv;
  int* wl = reinterpret_cast<int*>(tmem_slot + 2);   // BAL: ticket of this cluster's range

  if (warp == 2 && lane == 0) {
    if constexpr (BAL) {
      // one ticket per cluster (start order); rank 0 takes it and parks it in global memory for
      // the other ranks, which read it after the cluster barrier below
      if (MC == 1 || cluster_ctarank() == 0) {
        const unsigned t = atomicAdd(bal.flags + gridDim.x, 1u);
        if constexpr (MC == 1) *wl = (int)t;
        else bal.flags[gridDim.x + 1 + blockIdx.x / MC] = t;
      }
    }
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], MC);
      mbar_init(&pt_bar[i], 64);
      mbar_init(&vs_bar[i], 64);
    }
    for (int i = 0; i < VST; ++i) {
      mbar_init(&vfull[i], 1);
      mbar_init(&vempty[i], 1);
    }
    mbar_init(mma1_bar, 1);
    mbar_init(st_done, 256);
    mbar_init(mma_s_bar, 1);
    mbar_init(ox_bar, 1);
    mbar_init(ox_scaled, 128);
    mbar_init(mma_o_bar, 1);
    mbar_init(o_free, 128);
    fence_barrier_init();
    if (!state_only) {
      tma_prefetch_desc(&tm_q);
      tma_prefetch_desc(&tm_o);
    }
    tma_prefetch_desc(&tm_k);
    tma_prefetch_desc(&tm_v);
  }
  if (warp == 3) tmem_alloc<kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  if constexpr (MC > 1) cluster_sync_all();   // peers' barriers exist before any multicast
  if constexpr (BAL && MC > 1) {
    if (threadIdx.x == 0) *wl = (int)__ldcg(bal.flags + gridDim.x + 1 + blockIdx.x / MC);
    __syncthreads();
  }
  if constexpr (!BAL) {
    pdl_wait();   // everything above overlapped the previous kernel's tail
    // the gamma tables read log2g, which an earlier kernel in the stream may have written
    const float lg0 = log2g[blockIdx.y % H];
    if (threadIdx.x <= kC) pw[threadIdx.x] = gpow(lg0, (float)threadIdx.x);
    if (threadIdx.x < 192) {
      const int k = (int)threadIdx.x - 64;
      const float a = k >= 0 ? gpow(lg0, (float)k) : 0.f;
      const float b = k + 1 >= 0 ? gpow(lg0, (float)(k + 1)) : 0.f;
      pw2[k] = pack_bf16x2(a, b);
    }
    __syncthreads();
  }
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;
  const uint32_t crank = MC > 1 ? cluster_ctarank() : 0;
  // work list: the unit of blockIdx (SegArgs segment blockIdx.z), or this cluster's range
  auto item = [&](int k) {
    WorkItem w;
    if constexpr (BAL) {
      const int t = *reinterpret_cast<volatile int*>(wl);
      long long a = 0, b = 0;
      balance_items(bal, t, a, b);
      w = balance_item(bal, N, t, k, a, b);
      w.j0 += (int)crank * kDVT;
      if (w.in_slot >= 0) w.in_slot = w.in_slot * MC + (int)crank;
      if (w.out_slot >= 0) w.out_slot = w.out_slot * MC + (int)crank;
    } else {
      w.bh = blockIdx.y;
      w.j0 = blockIdx.x * kDVT;
      seg_bounds(sa.seg_len, sa.sub, sa.m, blockIdx.z, N, w.lo, w.hi);
      w.in_slot = w.out_slot = -1;
    }
    return w;
  };
  int nitems = 1;
  if constexpr (BAL) {
    long long a = 0, b = 0;
    nitems = balance_items(bal, *reinterpret_cast<volatile int*>(wl), a, b);
  }
  auto tables = [&](int bh_, const float*& pwv, const uint32_t*& pw2v) {
    if constexpr (BAL) {
      const float* tb = bal.tab + (size_t)(bh_ % H) * 257;
      pwv = tb;
      pw2v = reinterpret_cast<const uint32_t*>(tb + 65) + 64;
    } else {
      pwv = pw;
      pw2v = pw2;
    }
  };
  // debug: per-chunk clock64 of CTA (0,0,0), trace[event * 4096 + chunk]
  const bool tracing = trace != nullptr && !BAL && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0;
#define V3_TRACE(ev, c) do { if (tracing && lane == 0 && (c) < 4096) trace[(ev) * 4096 + (c)] = clock64(); } while (0)

  if (warp < 2) {
    // ------------------------------------------------------------ V' and P^T mask (TMEM lanes 0-63)
    const int srow = warp * 32 + lane;
    int c = 0;                                     // chunk counter over the whole work list
    for (int it = 0; it < nitems; ++it) {
     const WorkItem w = item(it);
     const float* pwv;
     const uint32_t* pw2v;
     tables(w.bh, pwv, pw2v);
     Lazy lz;
     for (int t0 = w.lo; t0 < w.hi; t0 += kC, ++c) {
      const int s = c % STAGES;
      const int L = min(kC, w.hi - t0);
      mbar_wait(&vfull[c % VST], (c / VST) & 1);
      if (c > 0) {
        mbar_wait(mma_s_bar, (c - 1) & 1);           // S update c-1 has consumed V'
        tc_fence_after();
      }
      if (warp == 0) V3_TRACE(12, c);
      lz.step(pwv[L]);
      {   // V'[s] = gamma^(L-1-s) V[s] / sig_{c+1}, 0 past L (row srow, both 64-column blocks)
        const float wv = srow < L ? pwv[L - 1 - srow] * lz.vfac : 0.f;
        scale_row_blocks<kDVT / 64>(smem + G::OFF_V + (c % VST) * G::V_BYTES, vs_smem, srow, 0, pack_bf16x2(wv, wv));
      }
      fence_proxy_async_smem();
      mbar_arrive(&vs_bar[s]);
      if (warp == 0) V3_TRACE(7, c);
      if (state_only) continue;
      mbar_wait(mma1_bar, c & 1);
      tc_fence_after();
      if (warp == 0) V3_TRACE(11, c);
      const uint32_t ta = tbase + ((warp * 32) << 16) + T_P;
      uint8_t* row = pt_smem + (c & 1) * G::PT_BYTES + srow * 128;
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        float p[32];
        tmem_ld32(ta + half * 32, p);
        tmem_wait_ld();
        if (warp == 0 && half == 0) V3_TRACE(2, c);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int tc = half * 32 + 8 * j;
          uint4 pk;
          pk.x = v2::hmul2_bf16(pack_bf16x2(p[8 * j + 0], p[8 * j + 1]), pw2v[tc + 0 - srow]);
          pk.y = v2::hmul2_bf16(pack_bf16x2(p[8 * j + 2], p[8 * j + 3]), pw2v[tc + 2 - srow]);
          pk.z = v2::hmul2_bf16(pack_bf16x2(p[8 * j + 4], p[8 * j + 5]), pw2v[tc + 4 - srow]);
          pk.w = v2::hmul2_bf16(pack_bf16x2(p[8 * j + 6], p[8 * j + 7]), pw2v[tc + 6 - srow]);
          *reinterpret_cast<uint4*>(row + (((half * 4 + j) ^ (srow & 7)) << 4)) = pk;
        }
      }
      fence_proxy_async_smem();
      tc_fence_before();
      mbar_arrive(&pt_bar[s]);
      if (warp == 0) V3_TRACE(14, c);
      if (warp == 0) V3_TRACE(6, c);
     }
    }
  } else if (warp >= 12) {
    // ------------------------------------------------------------ V', Q' scaling and outputs
    const int sub = warp - 12;
    const int tid = threadIdx.x - 12 * 32;           // 0..127
    const int row = tid >> 1;                        // token row of the chunk
    const int part = tid & 1;                        // which half of the 64-column blocks
    const bool leader = (tid == 0);
    const int mrow = lane & 7;
    const int mi = lane >> 3;
    // O^T (TMEM, lane = dv row) -> bf16 -> smem [t][d] (stmatrix.trans, 128B swizzle) -> TMA store
    auto drain_outputs = [&](int c, int t0, const WorkItem& w) {
      mbar_wait(mma_o_bar, c & 1);
      tc_fence_after();
      if (sub == 0) V3_TRACE(13, c);
      if (leader) bulk_wait_read<0>();               // the previous store has read the tile
      named_bar_sync(1, 128);
#pragma unroll
      for (int g = 0; g < 2; ++g) {
        const int d0 = sub * 32 + g * 16;
        const int md = d0 + (mi & 1) * 8;
        const uint32_t ta_o = tbase + ((uint32_t)d0 << 16) + T_O;
#pragma unroll
        for (int q4 = 0; q4 < 2; ++q4) {
          uint32_t ro[16];
          tmem_ld_16x256b_x4(ta_o + q4 * 32, ro);
          tmem_wait_ld();
          uint32_t pk[8];
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            pk[2 * r + 0] = pack_bf16x2(__uint_as_float(ro[4 * r + 0]), __uint_as_float(ro[4 * r + 1]));
            pk[2 * r + 1] = pack_bf16x2(__uint_as_float(ro[4 * r + 2]), __uint_as_float(ro[4 * r + 3]));
          }
#pragma unroll
          for (int rr = 0; rr < 4; rr += 2) {
            const int tt = q4 * 32 + rr * 8 + (mi >> 1) * 8 + mrow;
            const uint32_t addr = smem_u32(ot_smem + (md / 64) * (kC * 128) + tt * 128 +
                                           ((((md % 64) >> 3) ^ (tt & 7)) << 4));
            stmatrix_x4_trans(addr, pk[2 * rr + 0], pk[2 * rr + 1], pk[2 * rr + 2], pk[2 * rr + 3]);
          }
        }
      }
      tc_fence_before();
      mbar_arrive(o_free);
      if (sub == 0) V3_TRACE(8, c);
      fence_proxy_async_smem();
      named_bar_sync(2, 128);
      if (leader) {
        tma_store_3d(&tm_o, ot_smem, w.j0, t0, w.bh);
        tma_store_3d(&tm_o, ot_smem + kC * 128, w.j0 + 64, t0, w.bh);
        bulk_commit();
      }
    };
    int c = 0;
    for (int it = 0; it < (state_only ? 0 : nitems); ++it) {
     const WorkItem w = item(it);
     const float* pwv;
     const uint32_t* pw2v;
     tables(w.bh, pwv, pw2v);
     Lazy lz;
     for (int t0 = w.lo; t0 < w.hi; t0 += kC, ++c) {
      const int L = min(kC, w.hi - t0);
      lz.step(pwv[L]);
      {
        // O_inter(c)[d][t] *= sig_c gamma^(t+1)  (fp32, in TMEM: lanes sub*32.., columns t)
        mbar_wait(ox_bar, c & 1);
        tc_fence_after();
        const uint32_t ta_o = tbase + ((uint32_t)(sub * 32) << 16) + T_O;
#pragma unroll
        for (int half = 0; half < 2; ++half) {
          float o[32];
          tmem_ld32(ta_o + half * 32, o);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 32; ++i) o[i] *= lz.sig_c * pwv[half * 32 + i + 1];
          tmem_st32(ta_o + half * 32, o);
        }
        tmem_wait_st();
        tc_fence_before();
        mbar_arrive(ox_scaled);
        if (sub == 0) V3_TRACE(6, c);
      }
      drain_outputs(c, t0, w);
     }
    }
    if (leader) bulk_wait<0>();
  } else if (warp >= 4) {
    // ------------------------------------------------------------ state (TMEM fp32)
    // warp (half, sub): TMEM lanes sub*32.. (dv rows), state columns [half*SCOL, +SCOL)
    const int sub = (warp - 4) % 4;
    const int col0 = ((warp - 4) / 4) * SCOL;
    const int d = sub * 32 + lane;                       // dv row within the 128-wide tile
    const uint32_t ta_s = tbase + ((sub * 32) << 16) + T_S + col0;
    const uint32_t ta_sb = tbase + ((sub * 32) << 16) + T_SB + col0 / 2;
    const bool leader = (warp == 4 && lane == 0);
    int c = 0;
    for (int it = 0; it < nitems; ++it) {
    const WorkItem w = item(it);
    const float* pwv;
    const uint32_t* pw2v;
    tables(w.bh, pwv, pw2v);
    const float lg = log2g[w.bh % H];
    const int jd = w.j0 + d;
    const bool dv_ok = jd < dv;
    const int nch = w.hi > w.lo ? (w.hi - w.lo + kC - 1) / kC : 0;
    // end state: a balanced head publishes it to its hand-off slot; otherwise state-only launches
    // write one local state per segment, full launches only the segment ending the sequence
    float* so = nullptr;
    size_t so_stride = dv;
    int srows = dkr;                                     // hand-off slots hold all DK rows
    if (BAL && w.out_slot >= 0) {
      if (dv_ok) so = bal.hst + ((size_t)w.out_slot * DK + col0) * kDVT + d;
      so_stride = kDVT;
      srows = DK;
    } else if (s_out && dv_ok && (BAL ? w.hi == N : (state_only || blockIdx.z == gridDim.z - 1))) {
      so = s_out + (state_only ? blockIdx.z * per_state : 0) + ((size_t)w.bh * dkr + col0) * dv + jd;
    }
    if (it > 0) {
      // the previous item's last S update and O_inter are done before T is re-seeded
      mbar_wait(state_only ? mma_s_bar : ox_bar, (c - 1) & 1);
      tc_fence_after();
    }
    if (BAL && w.in_slot >= 0) {
      if (leader)
        while (ld_acquire_gpu(bal.flags + w.in_slot) == 0u) __nanosleep(256);
      named_bar_sync(3, 256);
    }
    {
      // S_init = gamma^lo s_in + sum_{q: hi_q <= lo} gamma^(lo - hi_q) loc[q]  (SegArgs), or a
      // balanced tail's hand-off state (s_in and every earlier token already folded in)
      const float w_in = gpow(lg, (float)w.lo);
      for (int cb = 0; cb < SCOL / 32; ++cb) {
        float sv[32];
        if (BAL && w.in_slot >= 0) {
          const float* hp = bal.hst + ((size_t)w.in_slot * DK + col0 + cb * 32) * kDVT + d;
#pragma unroll
          for (int i = 0; i < 32; ++i) sv[i] = dv_ok ? __ldcg(hp + (size_t)i * kDVT) : 0.f;
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i)
            sv[i] = (s_in && dv_ok && (!PADK || col0 + cb * 32 + i < dkr))
                        ? w_in * s_in[((size_t)w.bh * dkr + col0 + cb * 32 + i) * dv + jd] : 0.f;
          for (int qi = 0; qi < sa.nloc; ++qi) {
            const float wq = seg_loc_weight(sa, qi, N, w.lo, lg);
            if (wq < 0.f || !dv_ok) continue;
            const float* lq = sa.loc + qi * per_state + ((size_t)w.bh * dkr + col0 + cb * 32) * dv + jd;
#pragma unroll
            for (int i = 0; i < 32; ++i)
              if (!PADK || col0 + cb * 32 + i < dkr) sv[i] = fmaf(wq, lq[(size_t)i * dv], sv[i]);
          }
        }
        if (nch == 0) {
          if (so) {
#pragma unroll
            for (int i = 0; i < 32; ++i)
              if (!PADK || col0 + cb * 32 + i < srows) so[(size_t)(cb * 32 + i) * so_stride] = sv[i];
          }
        } else {
          tmem_st32(ta_s + cb * 32, sv);
        }
      }
      tmem_wait_st();
    }
    Lazy lz;
    for (int t0 = w.lo; t0 < w.hi; t0 += kC, ++c) {
      const int L = min(kC, w.hi - t0);
      if (c > 0) {
        // S_c complete; in the full pass also O_inter(c-1) done (it follows the S update in
        // the pipe), so the bf16 operand buffer is free and S_c can be published straight away
        mbar_wait(state_only ? mma_s_bar : ox_bar, (c - 1) & 1);
        tc_fence_after();
      }
      if (warp == 4) V3_TRACE(0, c);
      lz.step(pwv[L]);
      // publish bf16 T_c for O_inter(c); rewrite T only when renormalising (T <- sig gamma^L T)
      if (!state_only || lz.renorm) {
#if V3_PUB_ILP
        // two 32-column TMEM loads in flight per wait: the publish is on the per-chunk chain
#pragma unroll 1
        for (int cb = 0; cb < SCOL / 32; cb += 2) {
          float sv[32], sw[32];
          tmem_ld32(ta_s + cb * 32, sv);
          tmem_ld32(ta_s + (cb + 1) * 32, sw);
          tmem_wait_ld();
          if (!state_only) {
            uint32_t pk[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) pk[i] = pack_bf16x2_pub(sv[2 * i], sv[2 * i + 1]);
            tmem_st16(ta_sb + cb * 16, pk);
#pragma unroll
            for (int i = 0; i < 16; ++i) pk[i] = pack_bf16x2_pub(sw[2 * i], sw[2 * i + 1]);
            tmem_st16(ta_sb + (cb + 1) * 16, pk);
          }
          if (lz.renorm) {
#pragma unroll
            for (int i = 0; i < 32; ++i) sv[i] *= lz.rescale;
            tmem_st32(ta_s + cb * 32, sv);
#pragma unroll
            for (int i = 0; i < 32; ++i) sw[i] *= lz.rescale;
            tmem_st32(ta_s + (cb + 1) * 32, sw);
          }
        }
#else
#pragma unroll 1
        for (int cb = 0; cb < SCOL / 32; ++cb) {
          float sv[32];
          tmem_ld32(ta_s + cb * 32, sv);
          tmem_wait_ld();
          if (!state_only) {
            uint32_t pk[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) pk[i] = pack_bf16x2_pub(sv[2 * i], sv[2 * i + 1]);
            tmem_st16(ta_sb + cb * 16, pk);
          }
          if (lz.renorm) {
#pragma unroll
            for (int i = 0; i < 32; ++i) sv[i] *= lz.rescale;
            tmem_st32(ta_s + cb * 32, sv);
          }
        }
#endif
        tmem_wait_st();
      }
      tc_fence_before();
      mbar_arrive(st_done);
      if (warp == 4) V3_TRACE(1, c);
    }
    // tcgen05.ld is warp-collective: the whole warp loads when any lane has a row to write (lanes
    // past dv have none when dv is not a multiple of 32)
    if (nch > 0 && __any_sync(0xffffffffu, so != nullptr)) {
      mbar_wait(mma_s_bar, (c - 1) & 1);
      tc_fence_after();
      for (int cb = 0; cb < SCOL / 32; ++cb) {
        float sv[32];
        tmem_ld32(ta_s + cb * 32, sv);
        tmem_wait_ld();
        if (so) {
#pragma unroll
          for (int i = 0; i < 32; ++i)   // S = sig T
            if (!PADK || col0 + cb * 32 + i < srows) so[(size_t)(cb * 32 + i) * so_stride] = lz.sig * sv[i];
        }
      }
    }
    if (BAL && w.out_slot >= 0) {                 // release the hand-off to the next range's tail
      __threadfence();
      named_bar_sync(4, 256);
      if (leader) st_release_gpu(bal.flags + w.out_slot, 1u);
    }
    }  // work items
  } else if (warp == 2) {
    // ------------------------------------------------------------ TMA producer
    // lane 0 streams the Q/K ring, lane 1 the V ring (independent waits)
    if (lane == 0) {
      const uint32_t bytes = (state_only ? 0 : G::Q_BYTES) + G::K_BYTES;
      int c = 0;
      for (int it = 0; it < nitems; ++it) {
       const WorkItem w = item(it);
       for (int t0 = w.lo; t0 < w.hi; t0 += kC, ++c) {
        const int s = c % STAGES;
        mbar_wait(&empty[s], ((c / STAGES) & 1) ^ 1);   // every CTA of the cluster released s
        V3_TRACE(9, c);
        uint8_t* st = smem + s * G::STAGE_BYTES;
        mbar_arrive_expect_tx(&full[s], bytes);        // the whole tile, from all MC issuers
#pragma unroll
        for (int j = 0; j < G::KB / MC; ++j) {
          const int kb = (int)crank * (G::KB / MC) + j;
          if constexpr (MC > 1) {
            if (!state_only) tma_load_3d_mc(st + kb * 8192, &tm_q, &full[s], kb * 64, t0, w.bh, kMask);
            tma_load_3d_mc(st + G::Q_BYTES + kb * 8192, &tm_k, &full[s], kb * 64, t0, w.bh, kMask);
          } else {
            if (!state_only) tma_load_3d(st + kb * 8192, &tm_q, &full[s], kb * 64, t0, w.bh);
            tma_load_3d(st + G::Q_BYTES + kb * 8192, &tm_k, &full[s], kb * 64, t0, w.bh);
          }
        }
        // The Q/K ring has only STAGES = 2 stages of 64 KiB (shared memory is full), so the load
        // of chunk c + STAGES waits for chunk c's release; warm L2 with it now so that load
        // is an L2 hit instead of a full HBM round trip on the per-chunk critical path.
        if (V3_PF_AHEAD > 0 && t0 + V3_PF_AHEAD * kC < w.hi) {
#pragma unroll
          for (int j = 0; j < G::KB / MC; ++j) {
            const int kb = (int)crank * (G::KB / MC) + j;
            if (!state_only) tma_prefetch_l2_3d(&tm_q, kb * 64, t0 + V3_PF_AHEAD * kC, w.bh);
            tma_prefetch_l2_3d(&tm_k, kb * 64, t0 + V3_PF_AHEAD * kC, w.bh);
          }
        }
       }
      }
      if constexpr (MC > 1) {   // peers' final releases have landed before this CTA may exit
        const int nchunks = c;
        for (int cc = (nchunks > STAGES ? nchunks - STAGES : 0); cc < nchunks; ++cc)
          mbar_wait(&empty[cc % STAGES], (cc / STAGES) & 1);
      }
    } else if (lane == 1) {
      int c = 0;
      for (int it = 0; it < nitems; ++it) {
       const WorkItem w = item(it);
       for (int t0 = w.lo; t0 < w.hi; t0 += kC, ++c) {
        const int s = c % VST;
        mbar_wait(&vempty[s], ((c / VST) & 1) ^ 1);
        uint8_t* st = smem + G::OFF_V + s * G::V_BYTES;
        mbar_arrive_expect_tx(&vfull[s], G::V_BYTES);
#pragma unroll
        for (int nb = 0; nb < kDVT / 64; ++nb)
          tma_load_3d(st + nb * 8192, &tm_v, &vfull[s], w.j0 + nb * 64, t0, w.bh);
        if (V3_PF_AHEAD > 0 && t0 + VST * kC < w.hi) {
#pragma unroll
          for (int nb = 0; nb < kDVT / 64; ++nb) tma_prefetch_l2_3d(&tm_v, w.j0 + nb * 64, t0 + VST * kC, w.bh);
        }
       }
      }
    }
  } else {
    // ------------------------------------------------------------ MMA issuer (warp 3)
    // pipe order per chunk: S update (the serial chain) first, then O, then MMA1 of c+1
    constexpr uint32_t id_qk = idesc_bf16(128, kC, false, false);   // P^T  = K Q^T
    constexpr uint32_t id_vp = idesc_bf16(128, kC, true, true);     // O^T  = V^T P^T
    constexpr uint32_t id_sq = idesc_bf16(128, kC, false, false);   // O^T  = S^T(TMEM) Q^T
    constexpr uint32_t id_vk = idesc_bf16(128, DK, true, true);     // S^T += V'^T K
    // descriptors built once; K steps add (byte offset >> 4) to the start-address field
    const uint32_t base_addr = smem_u32(smem);
    const uint64_t dq0 = smem_desc_sw128(base_addr, 16, 1024);
    const uint64_t dmn0 = smem_desc_sw128(base_addr, 8192, 1024);
    const uint64_t dpt0 = smem_desc_sw128(smem_u32(pt_smem), 8192, 1024);
    const uint64_t dvs = smem_desc_sw128(smem_u32(vs_smem), 8192, 1024);
    constexpr uint64_t kStage = G::STAGE_BYTES >> 4, kQ = G::Q_BYTES >> 4;
    auto issue_mma1 = [&](int c) {
      const int s = c % STAGES;
      mbar_wait(&full[s], (c / STAGES) & 1);
      tc_fence_after();
      const uint64_t dq = dq0 + s * kStage, dk = dq + kQ;
#pragma unroll
      for (int kb = 0; kb < G::KB; ++kb)
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          mma_bf16_ss_elect(tbase + T_P, dk + (kb * 512 + kk * 2), dq + (kb * 512 + kk * 2), id_qk,
                            (kb | kk) != 0);
      mma_commit_elect(mma1_bar);
      V3_TRACE(5, c);
    };
    // the tensor pipe sees one flat chunk stream across the work list
    int nchunks = 0;
    for (int it = 0; it < nitems; ++it) {
      const WorkItem w = item(it);
      nchunks += w.hi > w.lo ? (w.hi - w.lo + kC - 1) / kC : 0;
    }
    nchunks = __shfl_sync(0xffffffffu, nchunks, 0);   // warp-uniform: descriptors stay in uniform registers
    if (!state_only && nchunks > 0) issue_mma1(0);
    for (int c = 0; c < nchunks; ++c) {
      const int s = c % STAGES;
      const uint64_t dq = dq0 + s * kStage;                               // Q, K-major
      const uint64_t dk_mn = dmn0 + s * kStage + kQ;                      // K, MN-major (B of V'^T K)
      const uint64_t dv_mn = dmn0 + ((G::OFF_V + (c % VST) * G::V_BYTES) >> 4);   // V, MN-major
      V3_TRACE(10, c);
      if (state_only) mbar_wait(&full[s], (c / STAGES) & 1);   // K_c landed (MMA1 waited otherwise)
      mbar_wait(&vs_bar[s], (c / STAGES) & 1);        // V'_c written
      mbar_wait(st_done, c & 1);                      // S_c rescaled and published in TMEM
      tc_fence_after();
#pragma unroll
      for (int ks = 0; ks < kC / 16; ++ks)
        mma_bf16_ss_elect(tbase + T_S, dvs + ks * 128, dk_mn + ks * 128, id_vk, 1);
      mma_commit_elect(mma_s_bar);
      V3_TRACE(3, c);
      if (!state_only) {
        if (c > 0) {
          mbar_wait(o_free, (c - 1) & 1);             // O_{c-1} drained
          tc_fence_after();
        }
#pragma unroll
        for (int kb = 0; kb < G::KB; ++kb)
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            mma_bf16_ts_elect(tbase + T_O, tbase + T_SB + (kb * 4 + kk) * 8, dq + (kb * 512 + kk * 2), id_sq,
                              (kb | kk) != 0);
        mma_commit_elect(ox_bar);
        if constexpr (MC > 1) mma_commit_mc_elect(&empty[s], kMask);   // Q_c, K_c consumed (cluster)
        else mma_commit_elect(&empty[s]);
        mbar_wait(&pt_bar[s], (c / STAGES) & 1);      // P^T_c in smem: its TMEM copy is free
        if (c + 1 < nchunks) issue_mma1(c + 1);
        mbar_wait(ox_scaled, c & 1);                  // O_inter(c) scaled by gamma^(t+1)
        tc_fence_after();
        const uint64_t dpt = dpt0 + (c & 1) * (G::PT_BYTES >> 4);
#pragma unroll
        for (int ks = 0; ks < kC / 16; ++ks)
          mma_bf16_ss_elect(tbase + T_O, dv_mn + ks * 128, dpt + ks * 128, id_vp, 1);
        mma_commit_elect(mma_o_bar);
        V3_TRACE(4, c);
      } else {
        if constexpr (MC > 1) mma_commit_mc_elect(&empty[s], kMask);
        else mma_commit_elect(&empty[s]);
      }
      mma_commit_elect(&vempty[c % VST]);             // V_c consumed (O_intra / V')
    }
  }

  tc_fence_before();
  __syncthreads();
  if constexpr (MC > 1) cluster_sync_all();
  tc_fence_after();
  if (warp == 3) tmem_dealloc<kTmemCols>(tbase);
}

}  // namespace v3

// ---- host side ---------------------------------------------------------------------------

unsigned long long* g_trace = nullptr;  // debug: set by linattn_debug_set_trace

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// [BH][N][D] bf16 viewed as a 3-D tensor (D fastest); 64 x 64 boxes, 128B swizzle.
bool make_map(CUtensorMap* map, const void* base, int64_t D, int64_t N, int64_t BH) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[3] = {(cuuint64_t)D, (cuuint64_t)N, (cuuint64_t)BH};
  cuuint64_t strides[2] = {(cuuint64_t)D * 2, (cuuint64_t)(N * D * 2)};
  cuuint32_t box[3] = {64, 64, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box,
                  estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

template <int DK, int STAGES, bool SO = false>
cudaError_t launch_pipe(const void* q, const void* k, const void* v, void* o, const float* log2g,
                        const float* s_in, float* s_out, const ShapeArgs& s, bool state_only,
                        const SegArgs& sa, int nz, cudaStream_t stream, const Balance& bal = Balance{},
                        int ctas = 0) {
  using G = v2::Cfg<DK, STAGES, SO>;
  static_assert(G::SMEM <= 227 * 1024, "shared memory budget");
  CUtensorMap mq, mk, mv;
  const int64_t BH = s.B * s.H;
  if (!make_map(&mk, k, s.dk, s.N, BH) || !make_map(&mv, v, s.dv, s.N, BH)) return cudaErrorInvalidValue;
  if (state_only) {
    mq = mk;
  } else if (!make_map(&mq, q, s.dk, s.N, BH)) {
    return cudaErrorInvalidValue;
  }
  CUtensorMap mo = mk;
  if (!state_only && !make_map(&mo, o, s.dv, s.N, BH)) return cudaErrorInvalidValue;
  // dk < DK: the padded instantiation (the benched dk == DK kernels stay free of the row guards)
  const bool padk = s.dk != DK;
  auto kern = bal.on ? (padk ? v2::prefill_tc_pipe_kernel<DK, STAGES, SO, true, true>
                             : v2::prefill_tc_pipe_kernel<DK, STAGES, SO, true, false>)
                     : (padk ? v2::prefill_tc_pipe_kernel<DK, STAGES, SO, false, true>
                             : v2::prefill_tc_pipe_kernel<DK, STAGES, SO, false, false>);
  cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, G::SMEM);
  if (err != cudaSuccess) return err;
  const dim3 grid = bal.on ? dim3((unsigned)ctas)
                           : dim3((unsigned)((s.dv + kDVT - 1) / kDVT), (unsigned)BH, (unsigned)nz);
  // fused NaN/Inf output check (linattn_prefill_checked): full launches only
  unsigned long long* nf = state_only ? nullptr : reinterpret_cast<unsigned long long*>(nonfinite_slot());
  if (nf) mark_nonfinite_consumed();
  if (bal.on) {   // the balanced launch follows the memset of its flags: plain stream order
    kern<<<grid, v2::kThreads, G::SMEM, stream>>>(mq, mk, mv, mo, log2g, s_in, s_out,
                                                  (int)s.H, (int)s.N, (int)s.dv, (int)s.dk, state_only ? 1 : 0,
                                                  sa, bal, g_trace, nf);
  } else {
    err = launch_pdl(kern, grid, dim3(v2::kThreads), G::SMEM, stream, mq, mk, mv, mo, log2g, s_in, s_out,
                     (int)s.H, (int)s.N, (int)s.dv, (int)s.dk, state_only ? 1 : 0, sa, bal, g_trace, nf);
    if (err != cudaSuccess) return err;
  }
  count_launch();
  return cudaGetLastError();
}

template <int DK, int STAGES, int MC>
cudaError_t launch_tmem_state_mc(const CUtensorMap& mq, const CUtensorMap& mk, const CUtensorMap& mv,
                                 const CUtensorMap& mo, const float* log2g, const float* s_in, float* s_out,
                                 const ShapeArgs& s, bool state_only, const SegArgs& sa, int nz,
                                 cudaStream_t stream, const Balance& bal = Balance{}, int ctas = 0) {
  using G = v3::Cfg<DK, STAGES>;
  static_assert(G::SMEM <= 227 * 1024, "shared memory budget");
  const bool padk = s.dk != DK;
  auto kern = bal.on ? (padk ? v3::prefill_tc_tmem_state_kernel<DK, STAGES, MC, true, true>
                             : v3::prefill_tc_tmem_state_kernel<DK, STAGES, MC, true, false>)
                     : (padk ? v3::prefill_tc_tmem_state_kernel<DK, STAGES, MC, false, true>
                             : v3::prefill_tc_tmem_state_kernel<DK, STAGES, MC, false, false>);
  cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, G::SMEM);
  if (err != cudaSuccess) return err;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = bal.on ? dim3((unsigned)ctas)
                       : dim3((unsigned)((s.dv + kDVT - 1) / kDVT), (unsigned)(s.B * s.H), (unsigned)nz);
  cfg.blockDim = dim3(v3::kThreads);
  cfg.dynamicSmemBytes = G::SMEM;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = MC;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;   // see pdl_wait (plain grid only)
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = bal.on ? 1 : 2;
  err = cudaLaunchKernelEx(&cfg, kern, mq, mk, mv, mo, log2g, s_in, s_out, (int)s.H, (int)s.N, (int)s.dv, (int)s.dk,
                           state_only ? 1 : 0, sa, bal, g_trace);
  count_launch();
  if (err != cudaSuccess) return err;
  return cudaGetLastError();
}

// Co-resident clusters of the dk=256 kernel for cluster size m on the current device (cached).
template <int DK, int STAGES>
int max_active_clusters(int m) {
  static std::mutex mu;
  static int cache[64][5] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64 || m < 1 || m > 4) return 0;
  std::lock_guard<std::mutex> lock(mu);
  if (cache[dev][m] != 0) return cache[dev][m];
  using G = v3::Cfg<DK, STAGES>;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(4 * m));
  cfg.blockDim = dim3(v3::kThreads);
  cfg.dynamicSmemBytes = G::SMEM;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = m;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = 0;
  cudaError_t err = cudaErrorInvalidValue;
  if (m == 4) {
    auto kern = v3::prefill_tc_tmem_state_kernel<DK, STAGES, 4, false, false>;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, G::SMEM) == cudaSuccess)
      err = cudaOccupancyMaxActiveClusters(&n, kern, &cfg);
  } else if (m == 2) {
    auto kern = v3::prefill_tc_tmem_state_kernel<DK, STAGES, 2, false, false>;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, G::SMEM) == cudaSuccess)
      err = cudaOccupancyMaxActiveClusters(&n, kern, &cfg);
  }
  if (err != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  cache[dev][m] = n;
  return n;
}

template <int DK, int STAGES>
cudaError_t launch_tmem_state(const void* q, const void* k, const void* v, void* o, const float* log2g,
                              const float* s_in, float* s_out, const ShapeArgs& s, bool state_only,
                              const SegArgs& sa, int nz, cudaStream_t stream) {
  CUtensorMap mq, mk, mv;
  const int64_t BH = s.B * s.H;
  if (!make_map(&mk, k, s.dk, s.N, BH) || !make_map(&mv, v, s.dv, s.N, BH)) return cudaErrorInvalidValue;
  if (state_only) {
    mq = mk;
  } else if (!make_map(&mq, q, s.dk, s.N, BH)) {
    return cudaErrorInvalidValue;
  }
  CUtensorMap mo = mk;
  if (!state_only && !make_map(&mo, o, s.dv, s.N, BH)) return cudaErrorInvalidValue;
  // the dv tiles of a head share every Q/K tile: cluster them and multicast (LINATTN_NO_MULTICAST=1: off).
  // Cluster size = the one with the fewest waves of co-resident clusters (ties: the larger one):
  // GPC packing fits only 32 four-CTA clusters (128 SMs) but 74 two-CTA ones (all 148), so e.g.
  // 36 heads x 4 tiles run in one wave of pairs instead of two waves of quads.
  const int64_t tiles = (s.dv + kDVT - 1) / kDVT;
  const int64_t ctas = tiles * s.B * s.H * nz;
  static const bool no_mc = getenv("LINATTN_NO_MULTICAST") != nullptr;
  static const int force_mc = getenv("LINATTN_V3_MC") ? atoi(getenv("LINATTN_V3_MC")) : 0;   // dev A/B: 2 or 4
  int mc = 1;
  if (!no_mc && (force_mc == 2 || force_mc == 4) && tiles % force_mc == 0) {
    mc = force_mc;
  } else if (!no_mc) {
    int64_t best = -1;
    for (int m : {4, 2}) {
      if (tiles % m != 0) continue;
      const int slots = max_active_clusters<DK, STAGES>(m);
      if (slots <= 0) continue;
      const int64_t waves = (ctas / m + slots - 1) / slots;
      if (best < 0 || waves < best) {
        best = waves;
        mc = m;
      }
    }
  }
  if (mc == 4)
    return launch_tmem_state_mc<DK, STAGES, 4>(mq, mk, mv, mo, log2g, s_in, s_out, s, state_only, sa, nz, stream);
  if (mc == 2)
    return launch_tmem_state_mc<DK, STAGES, 2>(mq, mk, mv, mo, log2g, s_in, s_out, s, state_only, sa, nz, stream);
  return launch_tmem_state_mc<DK, STAGES, 1>(mq, mk, mv, mo, log2g, s_in, s_out, s, state_only, sa, nz, stream);
}

}  // namespace

void set_trace(void* buf) { g_trace = static_cast<unsigned long long*>(buf); }
unsigned long long* trace_buffer() { return g_trace; }

#ifndef V2_STAGES128
#define V2_STAGES128 4
#endif

// Any dk <= 256 and dv with 16-byte rows: the kernel for the next DK in {64, 128, 256} runs,
// its Q/K boxes past dk zero-filled by TMA (the extra state columns stay exactly zero, and the
// OOB fill costs no HBM traffic); V boxes past dv are zero-filled and output stores clipped.
int tc_bucket(int64_t dk) { return dk <= 64 ? 64 : dk <= 128 ? 128 : 256; }

bool tc_supported(const ShapeArgs& s, int dtype) {
  if (dtype != LINATTN_BF16) return false;
  if (s.dk < 1 || s.dk > 256 || s.dk % 8 != 0 || s.dv % 8 != 0) return false;
  return encode_fn() != nullptr;
}

cudaError_t launch_prefill_tc(const void* q, const void* k, const void* v, void* o,
                              const float* log2g, const float* s_in, float* s_out,
                              const ShapeArgs& s, bool state_only, const SegArgs& sa, int nz,
                              cudaStream_t stream) {
  for (const void* p : {q, k, v, (const void*)o})
    if (p && (reinterpret_cast<uintptr_t>(p) & 15)) return cudaErrorNotSupported;
  switch (tc_bucket(s.dk)) {
    case 64:
      if (state_only) return launch_pipe<64, 8, true>(q, k, v, o, log2g, s_in, s_out, s, true, sa, nz, stream);
      return launch_pipe<64, 6>(q, k, v, o, log2g, s_in, s_out, s, false, sa, nz, stream);
    case 128:
      if (state_only) return launch_pipe<128, 6, true>(q, k, v, o, log2g, s_in, s_out, s, true, sa, nz, stream);
      return launch_pipe<128, V2_STAGES128>(q, k, v, o, log2g, s_in, s_out, s, false, sa, nz, stream);
    case 256: return launch_tmem_state<256, 2>(q, k, v, o, log2g, s_in, s_out, s, state_only, sa, nz, stream);
    default: return cudaErrorNotSupported;
  }
}

namespace {
// Per-head gamma tables of the balanced dk = 256 kernel: [H][65 fp32 gamma^n | 192 bf16x2 pairs].
__global__ void gamma_tables_kernel(const float* __restrict__ log2g, float* __restrict__ tab) {
  const float lg = log2g[blockIdx.x];
  float* t = tab + (size_t)blockIdx.x * 257;
  uint32_t* t2 = reinterpret_cast<uint32_t*>(t + 65);
  for (int n = threadIdx.x; n <= kC; n += blockDim.x) t[n] = gpow(lg, (float)n);
  for (int i = threadIdx.x; i < 192; i += blockDim.x) {
    const int k = i - 64;
    t2[i] = pack_bf16x2(k >= 0 ? gpow(lg, (float)k) : 0.f, k + 1 >= 0 ? gpow(lg, (float)(k + 1)) : 0.f);
  }
}
// [ctas] hand-off flags, the ticket counter, then [ctas] per-cluster ticket slots
size_t flags_bytes(int ctas) { return 256 * (size_t)((2 * ctas + 1 + 63) / 64); }
size_t tab_bytes(const ShapeArgs& s) { return tc_bucket(s.dk) == 256 ? 256 * (size_t)((s.H * 257 * 4 + 255) / 256) : 0; }
}  // namespace

int tc_balance_ctas(const ShapeArgs& s, int sms, int env) {
  const int64_t tiles = (s.dv + kDVT - 1) / kDVT;
  if (tc_bucket(s.dk) <= 128) {
    const int64_t units = s.B * s.H * tiles, rem = units % sms;
    if (units <= sms || rem == 0) return 0;
    // a last wave more than half full already streams near the HBM roofline (each CTA is bound
    // by its own serial chunk chain, so fewer CTAs each go faster)
    return (env > 0 || 2 * rem <= sms) ? sms : 0;
  }
  if (tiles % 2 != 0) return 0;
  // dk = 256: ranges over clusters of two CTAs (74 co-resident pairs, all SMs) against the
  // plain grid's whole waves of the best cluster size (33 co-resident quads)
  const int slots2 = max_active_clusters<256, 2>(2);
  if (slots2 <= 0) return 0;
  const int64_t pairs = s.B * s.H * tiles / 2;
  if (pairs <= slots2 || pairs % slots2 == 0) return 0;
  int64_t plain = (pairs + slots2 - 1) / slots2;
  if (tiles % 4 == 0) {
    const int slots4 = max_active_clusters<256, 2>(4);
    if (slots4 > 0) plain = std::min<int64_t>(plain, (pairs / 2 + slots4 - 1) / slots4);
  }
  // measured (1 x H x 16384, dv = 512): a wave of 33 quads 0.41 ms, of 74 pairs 0.45 ms, and the
  // balanced ranges cost ~11 % over the pairs' steady state (item switches, hand-offs), so the
  // balanced launch wins when its fractional waves stay under 0.75 of the plain whole waves
  // (H = 40: 0.72 -> 0.54 ms, H = 48: 0.74 -> 0.65 ms; H = 56 and configs[2] (H = 64) stay plain)
  const double bal = (double)pairs / slots2;
  return (env > 0 || bal < 0.75 * (double)plain) ? 2 * slots2 : 0;
}

size_t balance_workspace_bytes(const ShapeArgs& s, int ctas) {
  return flags_bytes(ctas) + tab_bytes(s) + (size_t)ctas * tc_bucket(s.dk) * kDVT * sizeof(float);
}

cudaError_t launch_prefill_tc_balanced(const void* q, const void* k, const void* v, void* o,
                                       const float* log2g, const float* s_in, float* s_out,
                                       const ShapeArgs& s, int ctas, void* ws, cudaStream_t stream) {
  for (const void* p : {q, k, v, (const void*)o})
    if (reinterpret_cast<uintptr_t>(p) & 15) return cudaErrorNotSupported;
  const int DKB = tc_bucket(s.dk);
  const int mc = DKB == 256 ? 2 : 1;                       // CTAs per cluster (one range each)
  const int64_t ntiles = (s.dv + kDVT - 1) / kDVT;
  if (ntiles % mc != 0 || ctas % mc != 0) return cudaErrorNotSupported;
  const int64_t units = s.B * s.H * (ntiles / mc), nc = (s.N + kC - 1) / kC;
  const int ranges = ctas / mc;
  const int64_t w = (units * nc + ranges - 1) / ranges;
  if (!tc_supported(s, LINATTN_BF16) || w < nc || units * nc > (1LL << 31) - 1)
    return cudaErrorNotSupported;
  Balance bal;
  bal.on = 1;
  bal.units = (int)units;
  bal.nc = (int)nc;
  bal.w = (int)w;
  bal.ntiles = (int)(ntiles / mc);
  bal.tile = mc * kDVT;
  uint8_t* base = static_cast<uint8_t*>(ws);
  bal.flags = reinterpret_cast<unsigned*>(base);
  float* tab = reinterpret_cast<float*>(base + flags_bytes(ctas));
  bal.tab = tab;
  bal.hst = reinterpret_cast<float*>(base + flags_bytes(ctas) + tab_bytes(s));
  const int used = (int)((units * nc + w - 1) / w) * mc;   // CTAs whose range holds work
  cudaError_t err = cudaMemsetAsync(ws, 0, sizeof(unsigned) * (ctas + 1), stream);
  if (err != cudaSuccess) return err;
  if (DKB == 64)
    return launch_pipe<64, 6>(q, k, v, o, log2g, s_in, s_out, s, false, SegArgs{}, 1, stream, bal, used);
  if (DKB == 128)
    return launch_pipe<128, V2_STAGES128>(q, k, v, o, log2g, s_in, s_out, s, false, SegArgs{}, 1, stream, bal, used);
  gamma_tables_kernel<<<(unsigned)s.H, 64, 0, stream>>>(log2g, tab);
  count_launch();
  if ((err = cudaGetLastError()) != cudaSuccess) return err;
  CUtensorMap mq, mk, mv, mo;
  const int64_t BH = s.B * s.H;
  if (!make_map(&mk, k, s.dk, s.N, BH) || !make_map(&mv, v, s.dv, s.N, BH) || !make_map(&mq, q, s.dk, s.N, BH) ||
      !make_map(&mo, o, s.dv, s.N, BH))
    return cudaErrorInvalidValue;
  return launch_tmem_state_mc<256, 2, 2>(mq, mk, mv, mo, log2g, s_in, s_out, s, false, SegArgs{}, 1, stream, bal,
                                          used);
}

}  // namespace linattn
