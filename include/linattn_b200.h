/*
 * linattn_b200.h -- C ABI of the B200 (sm_100a) decayed causal linear-attention path.
 *
 *   O = (Q K^T (.) M_gamma) V,   M_gamma[i, j] = gamma^(i - j) for i >= j, else 0,
 *   one gamma per head; gamma^0 == 1 even for gamma == 0.
 *
 * Reference being replaced (paths relative to /root/reference/pkg/src/linattn):
 *   linattn_prefill       <- run_method(...) over the CPU blocking routes
 *                            _block_based_slice (kernels.py:109-136) and
 *                            _two_level_block_slice (kernels.py:139-166), driven by the
 *                            batch x head loop of run_method (kernels.py:257-281)
 *   linattn_decode_step   <- one iteration of _row_based_slice (kernels.py:100-104)
 *   linattn_state_pass    <- the decayed block carry u <- gamma^L u + (w_rev c)^T v
 *                            (kernels.py:127-128), i.e. the recursion factor
 *                            (w2 (.) C1)^T V1 (kernels.py:187-188)
 *   linattn_prefix_combine<- the recursion cross-term weights (kernels.py:185-189)
 *                            applied across sequence segments (new: SP prefix)
 *
 * The reference's slice kernels take one (N, r) slice; this ABI takes whole
 * (B, H, N, .) tensors at run_method granularity.
 *
 * Conventions
 *   - q, k: [B, H, N, dk]; v, o: [B, H, N, dv]; contiguous, row-major, DEVICE pointers.
 *     (reference names: q = B, k = C, dk = rank r, dv = dim d; tensor.py:62-94)
 *   - states (s_in, s_out, state): [B, H, dk, dv] fp32, device pointers, nullable where noted.
 *   - log2g: [H] fp32 DEVICE pointer, log2(gamma_h) computed in f64 on the host
 *     (-inf for gamma == 0, 0 for gamma == 1 or for the binary mask decay=False).
 *   - dtype: LINATTN_F32 or LINATTN_BF16, for q/k/v/o alike.
 *   - stream: a cudaStream_t passed as void* (0 = legacy default stream).
 *   - all calls are stream-ordered and asynchronous; no implicit synchronisation.
 *   - calls are reentrant; the only process state is per-device kernel attributes
 *     (set once) and a thread-local error string.
 *
 * Status codes map onto the reference exception classes (errors.py:4-29):
 *   ESHAPE -> ShapeError, EPARAM -> ParameterError, EDTYPE/EUNSUPPORTED -> UsageError,
 *   ECUDA -> LinAttnError.
 */
#ifndef LINATTN_B200_H
#define LINATTN_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LINATTN_ABI_VERSION 4

#if defined(__GNUC__)
#define LINATTN_API __attribute__((visibility("default")))
#else
#define LINATTN_API
#endif

typedef enum {
  LINATTN_OK = 0,
  LINATTN_ESHAPE = 1,
  LINATTN_EPARAM = 2,
  LINATTN_EDTYPE = 3,
  LINATTN_EUNSUPPORTED = 4,
  LINATTN_ECUDA = 5,
  LINATTN_ENOMEM = 6   /* device memory exhausted (the reference's ResourceError) */
} linattn_status;

typedef enum { LINATTN_F32 = 0, LINATTN_BF16 = 1 } linattn_dtype;

/* Kernel family selector for linattn_prefill / linattn_state_pass. */
typedef enum {
  LINATTN_KERNEL_AUTO = 0, /* bf16 -> TC, f32 -> TF32 when the shape/alignment allows, else SIMT */
  LINATTN_KERNEL_TC = 1,   /* tcgen05 + TMA chunked kernel: bf16, dk <= 256, dk and dv multiples of 8;
                              EUNSUPPORTED otherwise */
  LINATTN_KERNEL_SIMT = 2, /* fp32-FFMA chunked kernel (f32 or bf16; any dk, dv) */
  LINATTN_KERNEL_TF32 = 3  /* tcgen05 kind::tf32 3xTF32 chunked kernel, the f32 parity mode on the
                              tensor cores (f32, dk <= 128, dk and dv multiples of 4) */
} linattn_kernel;

/* Chunked prefill.  Optional s_in seeds the recurrence (nullptr = zero state, the
 * reference behaviour, kernels.py:114/144); optional s_out receives the end state
 * S_N = sum_j gamma^(N-1-j) k_j^T v_j (+ gamma^N s_in). */
LINATTN_API int linattn_prefill(const void* q, const void* k, const void* v, void* o,
                    const float* log2g, const float* s_in, float* s_out,
                    int64_t B, int64_t H, int64_t N, int64_t dk, int64_t dv,
                    int dtype, int kernel, void* stream);

/* Segment end state from K and V only (no Q, no O): s_out = sum_t gamma^(N-1-t) k_t^T v_t. */
LINATTN_API int linattn_state_pass(const void* k, const void* v, float* s_out, const float* log2g,
                       int64_t B, int64_t H, int64_t N, int64_t dk, int64_t dv,
                       int dtype, int kernel, void* stream);

/* Exclusive gamma-weighted prefix of gathered segment end states (sequence parallelism):
 *   gathered: [P, B, H, dk, dv] fp32 (device); seg_lens: [P] (HOST array);
 *   s_in = sum_{q < rank} gamma^(sum_{q < m < rank} L_m) * gathered[q]. */
LINATTN_API int linattn_prefix_combine(const float* gathered, float* s_in, const int64_t* seg_lens,
                           int P, int rank, const float* log2g,
                           int64_t B, int64_t H, int64_t dk, int64_t dv, void* stream);

/* One recurrent decode step for a batch of single tokens:
 *   q, k: [B, H, dk]; v, o: [B, H, dv]; state: [B, H, dk, dv] fp32 updated in place:
 *   S <- gamma S + k^T v ;  o = q S   (update first, then read: kernels.py:100-104). */
LINATTN_API int linattn_decode_step(const void* q, const void* k, const void* v, void* o, float* state,
                        const float* log2g, int64_t B, int64_t H, int64_t dk, int64_t dv,
                        int dtype, void* stream);

/* ---- Sequence segments (split inside one device; local half of multi-GPU sequence parallel) ----
 * Segment p covers tokens [p*seg_len, (p+1)*seg_len) clipped at N; with a sub-split m it is cut
 * into m sub-segments of sub = roundup(ceil(seg_len/m), 64) tokens, indexed z = p*m + r.
 * Tensor-core segments must be multiples of 64 tokens (only the last one may be ragged).
 * The algebra is the reference recursion cross term (kernels.py:185-189) applied across
 * segments: the state at token lo is gamma^lo*s_in + sum_{z: hi_z <= lo} gamma^(lo-hi_z)*loc[z].
 * linattn_prefill (AUTO/TC) applies this split itself when B*H*ceil(dv/128) leaves SMs idle,
 * with a workspace from a library-owned stream-ordered pool. */

/* Plan linattn_prefill would use: plan = {seg_len, nseg, m, sub}; nseg == 1 means no split. */
LINATTN_API int linattn_seq_plan(int64_t B, int64_t H, int64_t N, int64_t dk, int64_t dv, int dtype,
                                 int kernel, int64_t* plan);

/* Local end states (each from a zero state) of the first nseg segments, m sub-segments each:
 * loc_out [nseg*m][B][H][dk][dv] fp32 (device).  Replaces, per sub-segment, the decayed carry
 * u <- gamma^L u + (w_rev c)^T v of the reference blocking routes (kernels.py:125-128). */
LINATTN_API int linattn_state_pass_segmented(const void* k, const void* v, float* loc_out,
                                             const float* log2g, int64_t B, int64_t H, int64_t N,
                                             int64_t dk, int64_t dv, int dtype, int kernel,
                                             int64_t seg_len, int64_t m, int64_t nseg, void* stream);

/* Inclusive prefixes: incl[p] = state at token min(N, (p+1)*seg_len), p < nseg, accumulated from a
 * zero state over the local states of linattn_state_pass_segmented (geometry loc_seg_len, loc_m;
 * seg_len a multiple of loc_seg_len).  incl: [nseg][B][H][dk][dv] fp32.  With nseg = ceil(N/seg_len)
 * the last entry is the end state of the whole sequence (the per-rank state that sequence
 * parallelism all-gathers). */
LINATTN_API int linattn_segment_prefix(const float* loc, int64_t loc_seg_len, int64_t loc_m, int64_t nloc,
                                       float* incl, int64_t seg_len, int64_t nseg, const float* log2g,
                                       int64_t B, int64_t H, int64_t N, int64_t dk, int64_t dv,
                                       void* stream);

/* Prefill with every segment of seg_len tokens running in parallel, each seeded from s_in
 * (nullable; the state before token 0) and the nloc states `loc`: either local states produced by
 * linattn_state_pass_segmented with geometry (loc_seg_len, loc_m) (loc_inclusive = 0), or
 * inclusive prefixes from linattn_segment_prefix (loc_inclusive = 1, loc_m = 1, each segment
 * reads only the entry ending at its first token).  The caller guarantees loc covers every token
 * before the last segment.  s_out (nullable) receives the end state. */
LINATTN_API int linattn_prefill_segmented(const void* q, const void* k, const void* v, void* o,
                                          const float* log2g, const float* s_in, float* s_out,
                                          const float* loc, int64_t loc_seg_len, int64_t loc_m,
                                          int64_t nloc, int loc_inclusive, int64_t B, int64_t H,
                                          int64_t N, int64_t dk, int64_t dv, int dtype, int kernel,
                                          int64_t seg_len, void* stream);

/* out = gamma^pos * s_in + sum_{z: hi_z <= pos} gamma^(pos - hi_z) * loc[z]   ([B,H,dk,dv] fp32);
 * with pos == N this is the end state of the whole sequence from its segment-local states. */
LINATTN_API int linattn_state_at(const float* loc, int64_t loc_seg_len, int64_t loc_m, int64_t nloc,
                                 const float* s_in, float* out, int64_t pos, const float* log2g,
                                 int64_t B, int64_t H, int64_t N, int64_t dk, int64_t dv, void* stream);

/* The reference row-based route for a whole sequence in one launch (_row_based_slice,
 * kernels.py:93-106): for t = 0..N-1, S <- gamma S + k_t^T v_t, o_t = q_t S, with the fp32 state
 * in registers; s_in / s_out (nullable) seed / receive S.  Needs dk <= 256, dk and dv rows that are
 * multiples of 16 bytes and 16-byte aligned q, k, v (tokens are staged with cp.async). */
LINATTN_API int linattn_recurrent(const void* q, const void* k, const void* v, void* o, const float* log2g,
                                  const float* s_in, float* s_out, int64_t B, int64_t H, int64_t N,
                                  int64_t dk, int64_t dv, int dtype, void* stream);

/* Kernel family LINATTN_KERNEL_AUTO resolves to for this shape/dtype (TC or SIMT). */
LINATTN_API int linattn_prefill_kernel(int64_t dk, int64_t dv, int dtype);

/* linattn_prefill plus the entry contract's NaN/Inf check on the way (reference check_finite,
 * tensor.py:20-25): *nonfinite (DEVICE int64, caller-initialised to INT64_MAX) is lowered below
 * INT64_MAX if the output holds a NaN/Inf.  Every non-finite input element reaches some output (a
 * NaN/Inf times a zero mask weight is NaN), so a clean output proves clean inputs; the caller then
 * scans the inputs (linattn_nonfinite_index) only to name the offending entry.  The bf16 tensor-core
 * kernel checks its outputs in its epilogue (no extra memory traffic); other kernels are followed by
 * one scan of the output. */
LINATTN_API int linattn_prefill_checked(const void* q, const void* k, const void* v, void* o,
                                        const float* log2g, const float* s_in, float* s_out,
                                        int64_t B, int64_t H, int64_t N, int64_t dk, int64_t dv,
                                        int dtype, int kernel, int64_t* nonfinite, void* stream);

/* Finiteness scan of the entry contract (reference check_finite, tensor.py:20-25), one HBM pass:
 * atomically lowers *first_bad (DEVICE int64, initialised by the caller to INT64_MAX) to the
 * smallest flat index of a NaN/Inf among the n elements of x (dtype f32 or bf16).  Scanning q, k
 * and v into three slots needs a single synchronisation to read the verdicts back. */
LINATTN_API int linattn_nonfinite_index(const void* x, int64_t n, int dtype, int64_t* first_bad, void* stream);

/* Return the library's cached split/balance workspace memory (stream-ordered pools, one per
 * device) to the driver; up to 256 MiB per device is otherwise kept mapped between calls. */
LINATTN_API int linattn_release_workspace(void);

/* Thread-local message for the last non-OK status returned on this thread. */
LINATTN_API const char* linattn_last_error(void);

/* LINATTN_ABI_VERSION of the loaded library. */
LINATTN_API int linattn_abi_version(void);

/* Number of kernels this library launched on this thread since load (evidence counter). */
LINATTN_API int64_t linattn_launch_count(void);

#ifdef __cplusplus
}
#endif

#endif /* LINATTN_B200_H */
