// prefill.cu -- placeholder until the tcgen05 GEMM lands.
#include "paro_internal.h"

namespace paro {

bool prefill_supported(int64_t, int64_t, int64_t) { return false; }

cudaError_t launch_prefill_gemm(const void*, int64_t, const uint8_t*, const uint8_t*, const uint8_t*, const float*,
                                void*, int, int64_t, int64_t, int, cudaStream_t) {
  return cudaErrorNotSupported;
}

}  // namespace paro
