// attn_bwd.cu -- K3 backward (placeholder until the tcgen05 backward lands).
#include "radial_internal.h"

namespace radial_detail {

size_t bwd_workspace_bytes(uint32_t heads, uint64_t n, uint32_t D) {
    (void)D;
    return static_cast<size_t>(heads) * n * sizeof(float) + 256;
}

int launch_bwd(const void*, const void*, const void*, const void*, const float*, const void*, void*,
               void*, void*, uint32_t, uint64_t, uint32_t, float, const radial_layout*, void*,
               cudaStream_t) {
    return fail(RADIAL_ERR_INVALID, "attn_bwd: not built in this version");
}

}  // namespace radial_detail
