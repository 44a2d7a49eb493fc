// sm_100a tensor-core backward (placeholder until the tcgen05 kernel lands).
#include "internal.h"

namespace sppo {
cudaError_t launch_bwd_sm100(const BwdParams&, const KvWindow&, const KvGradWindow&, const void*, const TmaSlots&,
                             int32_t, int32_t, cudaStream_t) {
  return cudaErrorNotSupported;
}
}  // namespace sppo
