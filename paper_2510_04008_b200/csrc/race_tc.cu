// race_tc.cu -- sm_100a tcgen05/TMA fast path (placeholder until implemented).
#include "race_internal.h"

namespace race {
bool tc_supported(const Geo&) { return false; }
cudaError_t tc_aggregate(const Geo&, const void*, const void*, const float*, float*, cudaStream_t) {
  return cudaErrorNotSupported;
}
cudaError_t tc_readout(const Geo&, const void*, const float*, const float*, void*, float*, cudaStream_t) {
  return cudaErrorNotSupported;
}
}  // namespace race
