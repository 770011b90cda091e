// Front-door helpers: the finiteness scan of the entry contract (reference check_finite,
// tensor.py:20-25) as one HBM-bound pass per tensor, and workspace-pool trimming.
//
// linattn_nonfinite_index atomically lowers *first_bad (device int64) to the smallest flat index
// of a NaN/Inf element, so the caller scans q, k and v into three slots and reads them back with a
// single synchronisation (the reference raises DataError naming that index).
#include <cstdint>

#include "common.cuh"

namespace linattn {
namespace {

constexpr int kFinThreads = 256;

template <int EB>  // element bytes: 4 (f32) or 2 (bf16)
__device__ __forceinline__ bool bad_bits(uint32_t w) {
  if constexpr (EB == 4) return (w & 0x7f800000u) == 0x7f800000u;
  return (w & 0x7f80u) == 0x7f80u;
}

template <int EB>
__global__ void __launch_bounds__(kFinThreads)
nonfinite_kernel(const uint8_t* __restrict__ x, int64_t n, int64_t head, unsigned long long* __restrict__ first_bad) {
  constexpr int EV = 16 / EB;                     // elements per 16-byte vector
  const int64_t nvec = (n - head) / EV;
  const uint4* body = reinterpret_cast<const uint4*>(x + head * EB);
  unsigned long long best = ~0ull;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  // body: 8 independent 16-byte loads in flight per thread per iteration; the exponent test is
  // branch-free (per word for fp32, per 16-bit half via __vcmpeq2 for bf16) and only a vector that
  // holds a NaN/Inf takes the slow path that finds its first element
  constexpr int U = 8;
  for (int64_t i = tid; i < nvec; i += U * stride) {
    uint4 r[U];
#pragma unroll
    for (int u = 0; u < U; ++u) r[u] = i + u * stride < nvec ? __ldcs(body + i + u * stride) : make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t w[4] = {r[u].x, r[u].y, r[u].z, r[u].w};
      uint32_t any = 0;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if constexpr (EB == 4) any |= (uint32_t)bad_bits<4>(w[j]);
        else any |= __vcmpeq2(w[j] & 0x7f807f80u, 0x7f807f80u);
      }
      if (any) {
        const int64_t e0 = head + (i + u * stride) * EV;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if constexpr (EB == 4) {
            if (bad_bits<4>(w[j])) best = min(best, (unsigned long long)(e0 + j));
          } else {
            if (bad_bits<2>(w[j] & 0xffffu)) best = min(best, (unsigned long long)(e0 + 2 * j));
            if (bad_bits<2>(w[j] >> 16)) best = min(best, (unsigned long long)(e0 + 2 * j + 1));
          }
        }
      }
    }
  }
  // unaligned head and ragged tail, element by element
  const int64_t tail0 = head + nvec * EV;
  for (int64_t e = tid; e < head + (n - tail0); e += stride) {
    const int64_t idx = e < head ? e : tail0 + (e - head);
    uint32_t w = EB == 4 ? *reinterpret_cast<const uint32_t*>(x + idx * 4)
                         : (uint32_t)*reinterpret_cast<const uint16_t*>(x + idx * 2);
    if (bad_bits<EB>(w)) best = min(best, (unsigned long long)idx);
  }
  if (__any_sync(0xffffffffu, best != ~0ull)) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) best = min(best, __shfl_xor_sync(0xffffffffu, best, o));
    if ((threadIdx.x & 31) == 0 && best != ~0ull) atomicMin(first_bad, best);
  }
}

}  // namespace

cudaError_t launch_nonfinite(const void* x, int64_t n, int dtype, int64_t* first_bad, cudaStream_t stream) {
  const int eb = dtype == LINATTN_BF16 ? 2 : 4;
  const uintptr_t addr = reinterpret_cast<uintptr_t>(x);
  int64_t head = addr % 16 ? (int64_t)((16 - addr % 16) / eb) : 0;
  if (head > n) head = n;
  int sms = 148, dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t vec = (n - head) / (16 / eb);
  int64_t blocks = (vec / 8 + kFinThreads - 1) / kFinThreads;
  blocks = blocks < 1 ? 1 : blocks;
  if (blocks > 8LL * sms) blocks = 8LL * sms;      // grid-stride: 8 resident CTAs per SM
  auto* fb = reinterpret_cast<unsigned long long*>(first_bad);
  if (eb == 4)
    nonfinite_kernel<4><<<(unsigned)blocks, kFinThreads, 0, stream>>>(static_cast<const uint8_t*>(x), n, head, fb);
  else
    nonfinite_kernel<2><<<(unsigned)blocks, kFinThreads, 0, stream>>>(static_cast<const uint8_t*>(x), n, head, fb);
  count_launch();
  return cudaGetLastError();
}

}  // namespace linattn
