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

// gamma^n for an integer count that may exceed 2^24 (exact in float only up to there): the
// exponent n * log2(gamma) is formed in double before the float exp2.
__device__ __forceinline__ float gpow_n(float log2g, long long n) {
  return n == 0 ? 1.f : exp2f((float)((double)log2g * (double)n));
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

// Programmatic dependent launch: a kernel launched with launch_pdl may start while the previous
// kernel in the stream drains (its prologue overlaps that tail); pdl_wait() must precede every
// access to memory an earlier kernel in the stream writes or reads.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                       Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// ---- internal launchers (return cudaError_t of the launch) -------------------
struct ShapeArgs {
  int64_t B, H, N, dk, dv;
};

// Sequence-segment geometry of one launch (sequence split inside a device, and the local
// half of multi-GPU sequence parallelism).  blockIdx.z = p * m + r walks segment p
// (tokens [p*seg_len, (p+1)*seg_len) clipped at N), sub-segment r of `sub` tokens.
// `loc` optionally holds the LOCAL end states (from a zero state) of the sub-segments of an
// earlier state-only launch with geometry (loc_seg_len, loc_sub, loc_m); a segment starting
// at token lo is seeded with
//     S_init = gamma^lo * s_in + sum_{q : hi_q <= lo} gamma^(lo - hi_q) * loc[q]
// which is the reference recursion cross term (kernels.py:185-189) applied across segments.
//
// Inclusive mode (loc_incl = 1): loc[q] is instead the prefix state at token min(N, (q+1)*loc_seg_len)
// from a zero state (linattn_segment_prefix), so a segment starting at lo > 0 reads the single
// entry ending at lo with weight 1 -- one 64 KiB state per CTA instead of every earlier entry.
struct SegArgs {
  int seg_len = 0x7fffffff, sub = 0x7fffffff, m = 1;
  const float* loc = nullptr;
  int loc_seg_len = 0, loc_sub = 0, loc_m = 1, nloc = 0, loc_incl = 0;
};

__host__ __device__ __forceinline__ void seg_bounds(int seg_len, int sub, int m, int z, int N, int& lo,
                                                    int& hi) {
  const int p = z / m, r = z % m;
  const long long base = (long long)p * seg_len;
  const long long a = base + (long long)r * sub;
  const long long b = base + (long long)min((long long)(r + 1) * sub, (long long)seg_len);
  lo = (int)min(a, (long long)N);
  hi = (int)min(b, (long long)N);
}

// Weight of loc entry q for a segment starting at `lo`: gamma^(lo - hi_q) if the entry lies
// entirely before lo, else 0 (returned as a negative flag).
__device__ __forceinline__ float seg_loc_weight(const SegArgs& sa, int q, int N, int lo, float lg) {
  if (sa.loc_incl) {
    const long long end = min((long long)(q + 1) * sa.loc_seg_len, (long long)N);
    return (lo > 0 && end == lo) ? 1.f : -1.f;
  }
  int qlo, qhi;
  seg_bounds(sa.loc_seg_len, sa.loc_sub, sa.loc_m, q, N, qlo, qhi);
  if (qhi > lo || qhi <= qlo) return -1.f;
  return gpow(lg, (float)(lo - qhi));
}

// Balanced persistent schedule (tensor-core kernel, dk <= 128, units >= CTAs): the units x nc
// chunks of the launch are cut into equal contiguous ranges of w >= nc chunks, one per CTA in
// ticket order.  A range ends with the HEAD of one sequence and starts with the TAIL of another;
// the CTA runs the head first and publishes its end state (hst slot t, flags[t]), then whole
// sequences, then its tail seeded from slot t-1 -- by then the previous CTA has long finished
// that head, so the hand-off never stalls and every SM streams until the end (no tail wave).
struct Balance {
  int on = 0;
  int units = 0, nc = 0, w = 0, ntiles = 1;
  int chunk = 64, tile = 128;    // tokens per chunk, dv columns per unit
  float* hst = nullptr;          // [grid][dk][tile] fp32 hand-off states
  const float* tab = nullptr;    // dk = 256 kernel: per-head gamma tables [H][65 fp32 + 192 bf16x2]
  unsigned* flags = nullptr;     // [grid] published flags, then the ticket counter (zeroed per launch)
};

struct WorkItem {
  int bh, j0, lo, hi;            // unit (batch*head, dv tile) and its token range
  int in_slot, out_slot;         // hand-off slot to seed from / publish to, -1 = none
};

__host__ __device__ __forceinline__ int balance_items(const Balance& P, int t, long long& start, long long& end) {
  const long long total = (long long)P.units * P.nc;
  start = (long long)t * P.w;
  if (start >= total) return 0;
  end = start + P.w < total ? start + P.w : total;
  const int us = (int)(start / P.nc), cs = (int)(start % P.nc);
  const int ue = (int)(end / P.nc), ce = (int)(end % P.nc);
  return (ce != 0) + (ue - (cs ? us + 1 : us)) + (cs != 0);
}

__host__ __device__ __forceinline__ WorkItem balance_item(const Balance& P, int N, int t, int k, long long start,
                                                          long long end) {
  const int us = (int)(start / P.nc), cs = (int)(start % P.nc);
  const int ue = (int)(end / P.nc), ce = (int)(end % P.nc);
  const int f0 = cs ? us + 1 : us;
  WorkItem w;
  int u;
  w.in_slot = -1;
  w.out_slot = -1;
  if (ce != 0 && k == 0) {                    // head of unit ue: publish its end state
    u = ue;
    w.lo = 0;
    w.hi = ce * P.chunk;
    w.out_slot = t;
  } else {
    const int kk = k - (ce != 0);
    if (kk < ue - f0) {                       // whole sequence
      u = f0 + kk;
      w.lo = 0;
      w.hi = N;
    } else {                                  // tail of unit us, seeded by the previous range's head
      u = us;
      w.lo = cs * P.chunk;
      w.hi = N;
      w.in_slot = t - 1;
    }
  }
  w.bh = u / P.ntiles;
  w.j0 = (u % P.ntiles) * P.tile;
  return w;
}

// `nz` = number of (sub-)segments in the launch (grid.z).  In state-only mode s_out receives
// one local end state per z ([nz][B*H][dk][dv]); otherwise only the last segment writes s_out.
cudaError_t launch_prefill_simt(const void* q, const void* k, const void* v, void* o,
                                const float* log2g, const float* s_in, float* s_out,
                                const ShapeArgs& s, int dtype, bool state_only,
                                const SegArgs& sa, int nz, cudaStream_t stream);

// Balanced persistent FFMA prefill (chunk 32, 64-wide dv tiles): slots = resident CTAs on the
// device for this shape (0 = not applicable); `ws` holds simt_balance_workspace_bytes bytes.
int simt_balance_slots(const void* q, const void* k, const void* v, const ShapeArgs& s, int dtype);
size_t simt_balance_workspace_bytes(const ShapeArgs& s, int slots);
cudaError_t launch_prefill_simt_balanced(const void* q, const void* k, const void* v, void* o,
                                         const float* log2g, const float* s_in, float* s_out,
                                         const ShapeArgs& s, int dtype, int slots, void* ws,
                                         cudaStream_t stream);

// 3xTF32 tensor-core prefill (fp32 parity mode): fp32, dk <= 128, dk and dv multiples of 4,
// 16-byte aligned tensors; cudaErrorNotSupported otherwise.  Same SegArgs / nz contract.
bool tf32_supported(const ShapeArgs& s, int dtype);
cudaError_t launch_prefill_tf32(const void* q, const void* k, const void* v, void* o, const float* log2g,
                                const float* s_in, float* s_out, const ShapeArgs& s, bool state_only,
                                const SegArgs& sa, int nz, cudaStream_t stream);

// Balanced persistent 3xTF32 prefill (one CTA per SM over equal chunk ranges with head -> tail
// state hand-off): grid for this shape or 0 (keep the plain grid); workspace bytes; launcher.
int tf32_balance_ctas(const ShapeArgs& s, int sms);
size_t tf32_balance_workspace_bytes(const ShapeArgs& s, int ctas);
cudaError_t launch_prefill_tf32_balanced(const void* q, const void* k, const void* v, void* o, const float* log2g,
                                         const float* s_in, float* s_out, const ShapeArgs& s, int ctas, void* ws,
                                         cudaStream_t stream);

// Returns cudaErrorNotSupported when the shape is outside the TC kernel's envelope.
cudaError_t launch_prefill_tc(const void* q, const void* k, const void* v, void* o,
                              const float* log2g, const float* s_in, float* s_out,
                              const ShapeArgs& s, bool state_only, const SegArgs& sa, int nz,
                              cudaStream_t stream);

// Inclusive prefixes incl[p] = state at min(N, (p+1)*seg_len) for p < nseg, from the local states
// `sa.loc` of a state-only launch (geometry in sa.loc_*): one running scan per element.
cudaError_t launch_segment_prefix(const SegArgs& sa, float* incl, int64_t seg_len, int64_t nseg,
                                  const float* log2g, const ShapeArgs& s, cudaStream_t stream);

// State at token position `pos` from segment-local states (elementwise over [B*H][dk][dv]):
//   out = gamma^pos * s_in + sum_{q : hi_q <= pos} gamma^(pos - hi_q) * loc[q]
cudaError_t launch_state_at(const float* loc, const float* s_in, float* out, const SegArgs& sa,
                            int64_t pos, const float* log2g, const ShapeArgs& s, cudaStream_t stream);
bool tc_supported(const ShapeArgs& s, int dtype);

// Balanced persistent tensor-core prefill (Balance mode 0): dk in {64, 128} (one CTA per SM) or
// dk = 256 (two-CTA clusters).  tc_balance_ctas = grid of a balanced launch for this shape, 0 when
// the plain grid is kept (env: LINATTN_BALANCE, -1 auto / 1 whenever the units do not fill whole
// waves).  `ws` holds balance_workspace_bytes(s, ctas) bytes (flags are zeroed on the stream).
int tc_balance_ctas(const ShapeArgs& s, int sms, int env);
size_t balance_workspace_bytes(const ShapeArgs& s, int ctas);
cudaError_t launch_prefill_tc_balanced(const void* q, const void* k, const void* v, void* o,
                                       const float* log2g, const float* s_in, float* s_out,
                                       const ShapeArgs& s, int ctas, void* ws, cudaStream_t stream);
void set_trace(void* buf);  // debug only: per-chunk clock64 trace of CTA (0,0), nullptr = off
unsigned long long* trace_buffer();   // the buffer set_trace installed (nullptr = off)

// Whole-sequence row recurrence in one launch (reference _row_based_slice, kernels.py:93-106).
cudaError_t launch_recurrent(const void* q, const void* k, const void* v, void* o, const float* log2g,
                             const float* s_in, float* s_out, const ShapeArgs& s, int dtype,
                             cudaStream_t stream);

cudaError_t launch_decode_step(const void* q, const void* k, const void* v, void* o,
                               float* state, const float* log2g, const ShapeArgs& s,
                               int dtype, cudaStream_t stream);

cudaError_t launch_prefix_combine(const float* gathered, float* s_in, const int64_t* seg_lens,
                                  int P, int rank, const float* log2g, const ShapeArgs& s,
                                  cudaStream_t stream);

// Lowers *first_bad (device int64, caller-initialised to INT64_MAX) to the smallest flat index of a
// NaN/Inf element among the n elements of x (f32 or bf16): one coalesced read.
cudaError_t launch_nonfinite(const void* x, int64_t n, int dtype, int64_t* first_bad, cudaStream_t stream);

void count_launch();

// Fused entry-contract check (linattn_prefill_checked): a thread-local device int64 slot that a
// full prefill launch lowers to 0 when it writes a non-finite output (kernels that fuse the check
// mark it consumed; for the others the C side scans the output into the slot afterwards).
int64_t* nonfinite_slot();
void mark_nonfinite_consumed();

}  // namespace linattn
