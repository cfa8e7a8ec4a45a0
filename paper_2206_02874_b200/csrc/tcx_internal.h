// tcx internal host-side helpers shared by the C-ABI front end and kernel launchers.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <atomic>
#include <cstdint>
#include <cstdio>
#include <cstdarg>
#include "../../include/tcx.h"

namespace tcx {

extern std::atomic<uint64_t> g_launches;
inline void count_launch(uint64_t n = 1) { g_launches.fetch_add(n, std::memory_order_relaxed); }

tcx_status set_error(tcx_status s, const char* fmt, ...);
inline tcx_status ok() { return TCX_OK; }

struct DevInfo { int device; int sm_count; int cc_major; int cc_minor; int max_smem_optin; };
tcx_status current_device(DevInfo* out);
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device), not per launch
cudaError_t ensure_max_smem(const void* kern, int bytes, int device);   // validates sm_100

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda needed)
tcx_status make_tmap_2d(CUtensorMap* map, CUtensorMapDataType dt, const void* base,
                        uint64_t inner, uint64_t outer, uint64_t row_stride_bytes,
                        uint32_t box_inner, uint32_t box_outer, CUtensorMapSwizzle swz);

#define TCX_CUDA_TRY(expr)                                                                 \
  do {                                                                                     \
    cudaError_t _e = (expr);                                                               \
    if (_e != cudaSuccess)                                                                 \
      return ::tcx::set_error(TCX_ERR_CUDA, "%s: %s (%s:%d)", #expr, cudaGetErrorString(_e), \
                              __FILE__, __LINE__);                                         \
  } while (0)

// ---- launchers (validated arguments) ----
tcx_status launch_tiles(tcx_dtype ab, tcx_dtype cd, int k, int64_t count, const void* A, const void* B,
                        const void* C, void* D, cudaStream_t s);
tcx_status launch_tiles_tc05(tcx_dtype ab, int k, int64_t count, const void* A, const void* B,
                             const void* C, void* D, cudaStream_t s);

tcx_status launch_chain(tcx_dtype ab, int n_steps, int64_t count, const void* A0, const void* Bs, float* Ds,
                        cudaStream_t s);

struct GemmArgs {
  tcx_dtype ab;
  tcx_dtype cd;
  int64_t M, N, K;
  const void* A; int64_t lda;
  const void* B; int64_t ldb;
  const void* C; int64_t ldc;
  void* D; int64_t ldd;
  const void* meta_hw;   // sparse only
  int cta_group;
  int max_ctas;
  int group_m;    // 0 = default
  int tile_n;     // dense: 256 / 512 / 0 = auto
  int pairs_m = 1;  // dense, CTA pair: multicast cluster shape in pairs
  int pairs_n = 1;
  bool pairs_auto = true;   // dense: the caller left pairs_m / pairs_n at 0 (library choice)
  int fault = 0;    // debug builds only (TCX_WATCHDOG): 1 = the dense producer drops one TMA load
  uint64_t* trace = nullptr;   // debug builds only: tile timeline (tcx_debug_trace)
  int64_t trace_cap = 0;
};
tcx_status launch_gemm_dense(const GemmArgs& a, const DevInfo& dev, cudaStream_t s);
tcx_status launch_gemm_sp24(const GemmArgs& a, const DevInfo& dev, cudaStream_t s);
tcx_status launch_fill_c(const GemmArgs& a, cudaStream_t s);   // K == 0: D = C (or 0)

tcx_status launch_sp24_compress(int esize, bool pair, int64_t M, int64_t K, const void* A, int64_t lda,
                                void* vals, uint32_t* meta, int64_t* d_bad, cudaStream_t s);
tcx_status launch_sp24_pack(tcx_dtype ab, int64_t M, int64_t K, const uint32_t* meta, void* hw, int64_t* d_bad,
                            cudaStream_t s);
tcx_status launch_round_tf32(const float* in, float* out, int64_t n, cudaStream_t s);
tcx_status run_probe(const DevInfo& dev, const tcx_probe_config* cfg, tcx_probe_result* out);
tcx_status launch_sm_clock_stamp(long long* out, int max_sms, int sm_count, cudaStream_t s);
tcx_status run_probe_mem(const DevInfo& dev, const tcx_probe_config* cfg, tcx_probe_result* out);
tcx_status launch_ldmatrix_dump(int n, int trans, const void* src, const int* row_elem, uint32_t* out, cudaStream_t s);

}  // namespace tcx
