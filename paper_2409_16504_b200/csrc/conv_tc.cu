// tcgen05 gather-GEMM for the P2ENet sparse convolutions (work in progress:
// the SIMT path in net.cu is used until this lands).
#include "common.cuh"

namespace sfb {

bool conv_tc_supported(const NetLayer &) { return false; }
void prepare_tc_weights(sfb_ctx *, NetLayer &) {}
void conv_layer_tc(sfb_ctx *, const NetLayer &, const float *, int, const int32_t *, int64_t, int,
                   float *, int) {
    throw Error(SFB_ERR_STATE, "tcgen05 conv path not built");
}

}  // namespace sfb
