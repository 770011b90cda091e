// extern "C" boundary of liblinattn_b200.so (declared in include/linattn_b200.h).
// Host-side validation mirrors the reference's typed errors (tensor.py:97-123,
// errors.py:4-29); every entry point is stream-ordered and never synchronises.
#include <cstdio>
#include <cstdarg>
#include <atomic>
#include <string>

#include "common.cuh"

namespace linattn {

static thread_local std::string g_last_error;
static thread_local int64_t g_launches = 0;

void count_launch() { ++g_launches; }

static int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

static int cuda_status(cudaError_t err, const char* what) {
  if (err == cudaSuccess) return LINATTN_OK;
  if (err == cudaErrorNotSupported)
    return fail(LINATTN_EUNSUPPORTED, "%s: shape/dtype outside this kernel's envelope", what);
  return fail(LINATTN_ECUDA, "%s: CUDA error %d (%s)", what, (int)err, cudaGetErrorString(err));
}

static int check_dims(const ShapeArgs& s, bool need_n) {
  if (s.B < 1) return fail(LINATTN_ESHAPE, "batch extent must be >= 1, got %lld", (long long)s.B);
  if (s.H < 1) return fail(LINATTN_ESHAPE, "heads extent must be >= 1, got %lld", (long long)s.H);
  if (need_n && s.N < 1)
    return fail(LINATTN_ESHAPE, "seqlen extent must be >= 1, got %lld", (long long)s.N);
  if (s.dk < 1) return fail(LINATTN_ESHAPE, "rank extent must be >= 1, got %lld", (long long)s.dk);
  if (s.dv < 1) return fail(LINATTN_ESHAPE, "dim extent must be >= 1, got %lld", (long long)s.dv);
  if (s.N > (1LL << 31) - 1 || s.B * s.H > (1LL << 31) - 1)
    return fail(LINATTN_ESHAPE, "extent too large for 32-bit indexing");
  return LINATTN_OK;
}

static int check_dtype(int dtype) {
  if (dtype != LINATTN_F32 && dtype != LINATTN_BF16)
    return fail(LINATTN_EDTYPE, "unsupported dtype code %d (expected f32=0 or bf16=1)", dtype);
  return LINATTN_OK;
}

}  // namespace linattn

using namespace linattn;

extern "C" {

int linattn_prefill(const void* q, const void* k, const void* v, void* o, const float* log2g,
                    const float* s_in, float* s_out, int64_t B, int64_t H, int64_t N, int64_t dk,
                    int64_t dv, int dtype, int kernel, void* stream) {
  ShapeArgs s{B, H, N, dk, dv};
  if (int e = check_dims(s, true)) return e;
  if (int e = check_dtype(dtype)) return e;
  if (!q || !k || !v || !o || !log2g) return fail(LINATTN_EPARAM, "null tensor pointer");
  cudaStream_t st = (cudaStream_t)stream;
  const bool tc_ok = tc_supported(s, dtype);
  if (kernel == LINATTN_KERNEL_TC && !tc_ok)
    return fail(LINATTN_EUNSUPPORTED,
                "tensor-core prefill needs bf16, dk in {64,128,256} and dv %% 64 == 0 "
                "(got dtype=%d dk=%lld dv=%lld)", dtype, (long long)dk, (long long)dv);
  if (kernel != LINATTN_KERNEL_AUTO && kernel != LINATTN_KERNEL_TC && kernel != LINATTN_KERNEL_SIMT)
    return fail(LINATTN_EPARAM, "unknown kernel selector %d", kernel);
  if (kernel != LINATTN_KERNEL_SIMT && tc_ok)
    return cuda_status(launch_prefill_tc(q, k, v, o, log2g, s_in, s_out, s, false, st), "prefill_tc");
  return cuda_status(launch_prefill_simt(q, k, v, o, log2g, s_in, s_out, s, dtype, false, st),
                     "prefill_simt");
}

int linattn_state_pass(const void* k, const void* v, float* s_out, const float* log2g, int64_t B,
                       int64_t H, int64_t N, int64_t dk, int64_t dv, int dtype, int kernel,
                       void* stream) {
  ShapeArgs s{B, H, N, dk, dv};
  if (int e = check_dims(s, true)) return e;
  if (int e = check_dtype(dtype)) return e;
  if (!k || !v || !s_out || !log2g) return fail(LINATTN_EPARAM, "null tensor pointer");
  cudaStream_t st = (cudaStream_t)stream;
  const bool tc_ok = tc_supported(s, dtype);
  if (kernel == LINATTN_KERNEL_TC && !tc_ok)
    return fail(LINATTN_EUNSUPPORTED, "tensor-core state pass needs bf16 and a supported shape");
  if (kernel != LINATTN_KERNEL_SIMT && tc_ok)
    return cuda_status(launch_prefill_tc(nullptr, k, v, nullptr, log2g, nullptr, s_out, s, true, st),
                       "state_pass_tc");
  return cuda_status(launch_prefill_simt(nullptr, k, v, nullptr, log2g, nullptr, s_out, s, dtype,
                                         true, st), "state_pass_simt");
}

int linattn_prefix_combine(const float* gathered, float* s_in, const int64_t* seg_lens, int P,
                           int rank, const float* log2g, int64_t B, int64_t H, int64_t dk,
                           int64_t dv, void* stream) {
  ShapeArgs s{B, H, 1, dk, dv};
  if (int e = check_dims(s, false)) return e;
  if (P < 1 || P > 64) return fail(LINATTN_EPARAM, "segment count must be in [1, 64], got %d", P);
  if (rank < 0 || rank >= P) return fail(LINATTN_EPARAM, "rank %d outside [0, %d)", rank, P);
  if (!gathered || !s_in || !seg_lens || !log2g) return fail(LINATTN_EPARAM, "null pointer");
  for (int p = 0; p < P; ++p)
    if (seg_lens[p] < 0) return fail(LINATTN_EPARAM, "segment %d has negative length", p);
  return cuda_status(launch_prefix_combine(gathered, s_in, seg_lens, P, rank, log2g, s,
                                           (cudaStream_t)stream), "prefix_combine");
}

int linattn_decode_step(const void* q, const void* k, const void* v, void* o, float* state,
                        const float* log2g, int64_t B, int64_t H, int64_t dk, int64_t dv,
                        int dtype, void* stream) {
  ShapeArgs s{B, H, 1, dk, dv};
  if (int e = check_dims(s, false)) return e;
  if (int e = check_dtype(dtype)) return e;
  if (!q || !k || !v || !o || !state || !log2g) return fail(LINATTN_EPARAM, "null tensor pointer");
  return cuda_status(launch_decode_step(q, k, v, o, state, log2g, s, dtype, (cudaStream_t)stream),
                     "decode_step");
}

int linattn_prefill_kernel(int64_t dk, int64_t dv, int dtype) {
  ShapeArgs s{1, 1, 1, dk, dv};
  return tc_supported(s, dtype) ? LINATTN_KERNEL_TC : LINATTN_KERNEL_SIMT;
}

// Debug hook (not part of the public header): record per-chunk clock64 timestamps of
// CTA (0,0) of subsequent tensor-core launches into a device buffer of 16 x 4096 u64.
__attribute__((visibility("default"))) void linattn_debug_set_trace(void* dev_buf) { set_trace(dev_buf); }

const char* linattn_last_error(void) { return g_last_error.c_str(); }

int linattn_abi_version(void) { return LINATTN_ABI_VERSION; }

int64_t linattn_launch_count(void) { return g_launches; }

}  // extern "C"
