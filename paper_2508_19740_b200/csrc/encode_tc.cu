// K2 — tcgen05 bulk key encoder (placeholder until the UMMA path lands).
#include "spl_launch.cuh"

namespace spl {
spl_status encode_tc_launch(spl_ctx* ctx, const spl_hasher*, const float*, uint32_t, uint32_t,
                            uint32_t*, cudaStream_t) {
    return fail(ctx, SPL_E_STATE, "encode: SPL_ENCODE_TC not available in this build");
}
}  // namespace spl
