// tcx 2:4 sparse GEMM (tcgen05.mma.sp) — built in the next step.
#include "tcx_internal.h"
namespace tcx {
tcx_status launch_gemm_sp24(const GemmArgs&, const DevInfo&, cudaStream_t) {
  return set_error(TCX_ERR_UNSUPPORTED, "tcx_gemm_sp24: not built yet");
}
}  // namespace tcx
