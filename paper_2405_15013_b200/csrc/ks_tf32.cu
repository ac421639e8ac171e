// tcgen05 TF32 KS kernel (placeholder until built).
#include "ks_internal.h"

namespace ks {
bool tf32_supports(const ks_handle_s&, const KsCall&) { return false; }
cudaError_t tf32_launch(const ks_handle_s&, const KsCall&) { return cudaErrorNotSupported; }
}  // namespace ks
