// tcx_probe — built in the next step.
#include "tcx_internal.h"
namespace tcx {
tcx_status run_probe(const DevInfo&, const tcx_probe_config*, tcx_probe_result*) {
  return set_error(TCX_ERR_UNSUPPORTED, "tcx_probe: not built yet");
}
tcx_status launch_tiles_tc05(tcx_dtype, int, int64_t, const void*, const void*, const void*, void*, cudaStream_t) {
  return set_error(TCX_ERR_UNSUPPORTED, "tcx_mma_tiles_tc05: not built yet");
}
}  // namespace tcx
