// Register-tiled FP32 KS kernel for larger b, c (placeholder until built).
#include "ks_internal.h"

namespace ks {
bool ffma_supports(const ks_handle_s&, const KsCall&) { return false; }
cudaError_t ffma_launch(const ks_handle_s&, const KsCall&) { return cudaErrorNotSupported; }
}  // namespace ks
