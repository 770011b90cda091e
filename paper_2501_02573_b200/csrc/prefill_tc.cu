// K1: tensor-core chunked prefill (tcgen05 + TMA).  Placeholder until the kernel lands.
#include "common.cuh"

namespace linattn {

bool tc_supported(const ShapeArgs&, int) { return false; }

cudaError_t launch_prefill_tc(const void*, const void*, const void*, void*, const float*,
                              const float*, float*, const ShapeArgs&, bool, cudaStream_t) {
  return cudaErrorNotSupported;
}

}  // namespace linattn
