// tcgen05 implicit-GEMM 3x3 conv (sm_100a). Placeholder: filled in by the tensor-core milestone.
#include "net.cuh"

namespace regen {

bool conv_tc_supported(const SRNet*, const ConvDesc&) { return false; }
regen_status conv_tc_prepare(SRNet* net) {
  net->use_tc = false;
  return REGEN_OK;
}
regen_status conv_tc_launch(const SRNet*, const ConvDesc&, const void*, void*, const void*, const int32_t*, int,
                            const int32_t*, int, int, cudaStream_t) {
  set_error("tcgen05 conv not built");
  return REGEN_E_UNSUPPORTED;
}

}  // namespace regen
