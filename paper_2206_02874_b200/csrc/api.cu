// tcx C-ABI front end: argument validation, dispatch, tensor-map creation, error strings.
// Declarations and contracts: include/tcx.h.
#include <cstring>
#include <mutex>
#include <unordered_map>
#include "tcx_internal.h"

namespace tcx {

std::atomic<uint64_t> g_launches{0};
static thread_local char t_err[512] = "";

tcx_status set_error(tcx_status s, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(t_err, sizeof(t_err), fmt, ap);
  va_end(ap);
  return s;
}

static std::mutex g_dev_mu;
static DevInfo g_dev_cache[64];
static bool g_dev_valid[64];

tcx_status current_device(DevInfo* out) {
  int dev = -1;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return set_error(TCX_ERR_NO_DEVICE, "cudaGetDevice: %s", cudaGetErrorString(e));
  if (dev < 0 || dev >= 64) return set_error(TCX_ERR_NO_DEVICE, "device id %d", dev);
  std::lock_guard<std::mutex> lk(g_dev_mu);
  if (!g_dev_valid[dev]) {
    DevInfo d{};
    d.device = dev;
    TCX_CUDA_TRY(cudaDeviceGetAttribute(&d.sm_count, cudaDevAttrMultiProcessorCount, dev));
    TCX_CUDA_TRY(cudaDeviceGetAttribute(&d.cc_major, cudaDevAttrComputeCapabilityMajor, dev));
    TCX_CUDA_TRY(cudaDeviceGetAttribute(&d.cc_minor, cudaDevAttrComputeCapabilityMinor, dev));
    TCX_CUDA_TRY(cudaDeviceGetAttribute(&d.max_smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    g_dev_cache[dev] = d;
    g_dev_valid[dev] = true;
  }
  *out = g_dev_cache[dev];
  if (out->cc_major != 10 || out->cc_minor != 0)
    return set_error(TCX_ERR_ARCH, "device %d is sm_%d%d; libtcx is built for sm_100a only", dev, out->cc_major, out->cc_minor);
  return TCX_OK;
}

cudaError_t ensure_max_smem(const void* kern, int bytes, int device) {
  static std::mutex mu;
  static std::unordered_map<const void*, uint64_t> done;       // kernel -> bitmask of devices
  const uint64_t bit = 1ull << (device & 63);
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = done.find(kern);
    if (it != done.end() && (it->second & bit)) return cudaSuccess;
  }
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) {
    std::lock_guard<std::mutex> lk(mu);
    done[kern] |= bit;
  }
  return e;
}

typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_encodeTiled get_encode() {
  static PFN_encodeTiled fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_encodeTiled)p;
  });
  return fn;
}

// A descriptor is a pure function of its arguments, so repeated calls on the same buffers (a
// serving loop, a graph capture, the bench) reuse the last encodings: a per-thread direct-mapped
// cache keyed on every argument (a GEMM call encodes 4 maps; this cuts the C ABI's host cost).
namespace {
struct TmapKey {
  const void* base; uint64_t inner, outer, stride; uint32_t box_inner, box_outer; int dt, swz;
  bool operator==(const TmapKey& o) const {
    return base == o.base && inner == o.inner && outer == o.outer && stride == o.stride && box_inner == o.box_inner &&
           box_outer == o.box_outer && dt == o.dt && swz == o.swz;
  }
};
struct TmapEntry { TmapKey key; CUtensorMap map; bool valid; };
constexpr int TMAP_CACHE = 64;
thread_local TmapEntry g_tmap_cache[TMAP_CACHE];
inline int tmap_slot(const TmapKey& k) {
  uint64_t h = (uint64_t)(uintptr_t)k.base * 0x9E3779B97F4A7C15ull;
  h ^= (k.inner * 31 + k.outer) * 0xC2B2AE3D27D4EB4Full;
  h ^= (k.stride + ((uint64_t)k.box_inner << 32) + ((uint64_t)k.box_outer << 48) + ((uint64_t)k.dt << 8) + k.swz) *
       0x165667B19E3779F9ull;
  return (int)((h >> 40) % TMAP_CACHE);
}
}  // namespace

tcx_status make_tmap_2d(CUtensorMap* map, CUtensorMapDataType dt, const void* base, uint64_t inner, uint64_t outer,
                        uint64_t row_stride_bytes, uint32_t box_inner, uint32_t box_outer, CUtensorMapSwizzle swz) {
  const TmapKey key{base, inner, outer, row_stride_bytes, box_inner, box_outer, (int)dt, (int)swz};
  TmapEntry& slot = g_tmap_cache[tmap_slot(key)];
  if (slot.valid && slot.key == key) {
    *map = slot.map;
    return TCX_OK;
  }
  PFN_encodeTiled enc = get_encode();
  if (!enc) return set_error(TCX_ERR_CUDA, "cuTensorMapEncodeTiled entry point unavailable");
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {row_stride_bytes};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, dt, 2, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return set_error(TCX_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d): dims %llu x %llu stride %llu box %u x %u", (int)r,
                     (unsigned long long)inner, (unsigned long long)outer, (unsigned long long)row_stride_bytes, box_inner,
                     box_outer);
  slot.key = key;
  slot.map = *map;
  slot.valid = true;
  return TCX_OK;
}

static int esize_of(tcx_dtype t) {
  switch (t) {
    case TCX_F16: case TCX_BF16: return 2;
    case TCX_TF32: case TCX_F32: case TCX_S32: return 4;
    case TCX_S8: return 1;
  }
  return 0;
}

static bool aligned16(const void* p) { return ((uintptr_t)p & 15u) == 0; }

static tcx_status check_gemm_common(const char* fn, tcx_dtype ab, tcx_dtype cd, int64_t M, int64_t N, int64_t K,
                                    const void* A, int64_t lda, const void* B, int64_t ldb, const void* C, int64_t ldc,
                                    void* D, int64_t ldd, int64_t a_cols) {
  if (M < 0 || N < 0 || K < 0) return set_error(TCX_ERR_INVALID_VALUE, "%s: negative size", fn);
  if (M == 0 || N == 0) return TCX_OK;
  const int es = esize_of(ab);
  if (!D || (K > 0 && (!A || !B))) return set_error(TCX_ERR_INVALID_VALUE, "%s: NULL operand", fn);
  if (lda < a_cols || ldb < K || ldd < N || (C && ldc < N))
    return set_error(TCX_ERR_INVALID_VALUE, "%s: leading dimension smaller than the row length", fn);
  if ((A && !aligned16(A)) || (B && !aligned16(B)) || (C && !aligned16(C)) || !aligned16(D))
    return set_error(TCX_ERR_MISALIGNED, "%s: device pointers must be 16-byte aligned", fn);
  const int cs = cd == TCX_F16 ? 2 : 4;
  if ((lda * es) % 16 || (ldb * es) % 16 || (C && (ldc * cs) % 16) || (ldd * cs) % 16)
    return set_error(TCX_ERR_MISALIGNED, "%s: lda*esize, ldb*esize, ldc*csize, ldd*csize must be multiples of 16 bytes", fn);
  if ((K * es) % 16) return set_error(TCX_ERR_MISALIGNED, "%s: K*esize must be a multiple of 16 bytes", fn);
  if (M > (1ll << 31) - 1 || N > (1ll << 31) - 1 || K > (1ll << 31) - 1)
    return set_error(TCX_ERR_UNSUPPORTED, "%s: dimension >= 2^31", fn);
  return TCX_OK;
}

}  // namespace tcx

using namespace tcx;

#if TCX_WATCHDOG
static uint64_t* g_trace = nullptr;   // tcx_debug_trace (debug library only)
static int64_t g_trace_cap = 0;
#endif

extern "C" {

const char* tcx_status_string(tcx_status s) {
  switch (s) {
    case TCX_OK: return "TCX_OK";
    case TCX_ERR_INVALID_VALUE: return "TCX_ERR_INVALID_VALUE";
    case TCX_ERR_UNSUPPORTED: return "TCX_ERR_UNSUPPORTED";
    case TCX_ERR_MISALIGNED: return "TCX_ERR_MISALIGNED";
    case TCX_ERR_BAD_SPARSITY: return "TCX_ERR_BAD_SPARSITY";
    case TCX_ERR_NO_DEVICE: return "TCX_ERR_NO_DEVICE";
    case TCX_ERR_ARCH: return "TCX_ERR_ARCH";
    case TCX_ERR_CUDA: return "TCX_ERR_CUDA";
  }
  return "TCX_ERR_UNKNOWN";
}

const char* tcx_last_error(void) { return t_err; }
const char* tcx_version(void) { return "tcx 0.1 (sm_100a)"; }

tcx_status tcx_debug_trace(void* d_buf, int64_t capacity) {
#if TCX_WATCHDOG
  if (capacity < 0 || (d_buf && ((uintptr_t)d_buf & 7)))
    return set_error(TCX_ERR_INVALID_VALUE, "tcx_debug_trace: bad buffer / capacity");
  g_trace = (uint64_t*)d_buf;
  g_trace_cap = d_buf ? capacity : 0;
  return TCX_OK;
#else
  (void)d_buf; (void)capacity;
  return set_error(TCX_ERR_UNSUPPORTED, "tcx_debug_trace: only in the debug library (libtcx_debug.so)");
#endif
}
uint64_t tcx_launch_count(void) { return g_launches.load(); }

tcx_status tcx_sm_clock_stamp(int64_t* d_out, int max_sms, void* stream) {
  if (!d_out || max_sms < 1) return set_error(TCX_ERR_INVALID_VALUE, "tcx_sm_clock_stamp: NULL buffer / max_sms < 1");
  if (((uintptr_t)d_out & 7u) != 0) return set_error(TCX_ERR_MISALIGNED, "tcx_sm_clock_stamp: buffer alignment");
  DevInfo dev;
  tcx_status st = current_device(&dev);
  if (st != TCX_OK) return st;
  return launch_sm_clock_stamp((long long*)d_out, max_sms, dev.sm_count, (cudaStream_t)stream);
}

tcx_status tcx_mma_tiles(tcx_dtype ab, tcx_dtype cd, int m, int n, int k, int64_t count, const void* A, const void* B,
                         const void* C, void* D, void* stream) {
  const bool fp = (ab == TCX_F16 || ab == TCX_BF16) && cd == TCX_F32 && m == 16 && n == 8 && (k == 16 || k == 8);
  const bool hh = ab == TCX_F16 && cd == TCX_F16 && m == 16 && n == 8 && (k == 16 || k == 8);
  const bool tf = ab == TCX_TF32 && cd == TCX_F32 && m == 16 && n == 8 && (k == 8 || k == 16);
  const bool i8 = ab == TCX_S8 && cd == TCX_S32 && m == 16 && n == 8 && k == 32;
  if (!(fp || hh || tf || i8))
    return set_error(TCX_ERR_UNSUPPORTED, "tcx_mma_tiles: (ab=%d, cd=%d, m%dn%dk%d) not supported", ab, cd, m, n, k);
  if (count < 0) return set_error(TCX_ERR_INVALID_VALUE, "tcx_mma_tiles: count < 0");
  if (count == 0) return TCX_OK;
  if (!A || !B || !D) return set_error(TCX_ERR_INVALID_VALUE, "tcx_mma_tiles: NULL operand");
  if (!aligned16(A) || !aligned16(B) || !aligned16(D) || (C && !aligned16(C)))
    return set_error(TCX_ERR_MISALIGNED, "tcx_mma_tiles: pointers must be 16-byte aligned");
  DevInfo dev;
  tcx_status st = current_device(&dev);
  if (st != TCX_OK) return st;
  return launch_tiles(ab, cd, k, count, A, B, C, D, (cudaStream_t)stream);
}

tcx_status tcx_mma_chain(tcx_dtype ab, int n_steps, int64_t count, const void* A0, const void* Bs, float* Ds,
                         void* stream) {
  if (ab != TCX_F16 && ab != TCX_BF16 && ab != TCX_TF32)
    return set_error(TCX_ERR_UNSUPPORTED, "tcx_mma_chain: ab %d (F16, BF16 or TF32)", (int)ab);
  if (count < 0 || n_steps < 0) return set_error(TCX_ERR_INVALID_VALUE, "tcx_mma_chain: count/n_steps < 0");
  if (count == 0 || n_steps == 0) return TCX_OK;
  if (!A0 || !Bs || !Ds) return set_error(TCX_ERR_INVALID_VALUE, "tcx_mma_chain: NULL operand");
  if (!aligned16(A0) || !aligned16(Bs) || !aligned16(Ds))
    return set_error(TCX_ERR_MISALIGNED, "tcx_mma_chain: pointers must be 16-byte aligned");
  DevInfo dev;
  tcx_status st = current_device(&dev);
  if (st != TCX_OK) return st;
  return launch_chain(ab, n_steps, count, A0, Bs, Ds, (cudaStream_t)stream);
}

tcx_status tcx_ldmatrix_dump(int num, int trans, const void* src, const int32_t* row_elem, uint32_t* out,
                             void* stream) {
  if (!src || !row_elem || !out) return set_error(TCX_ERR_INVALID_VALUE, "tcx_ldmatrix_dump: NULL pointer");
  DevInfo dev;
  tcx_status st = current_device(&dev);
  if (st != TCX_OK) return st;
  return launch_ldmatrix_dump(num, trans, src, row_elem, out, (cudaStream_t)stream);
}

tcx_status tcx_mma_tiles_tc05(tcx_dtype ab, tcx_dtype cd, int m, int n, int k, int64_t count, const void* A,
                              const void* B, const void* C, void* D, void* stream) {
  const bool fp = (ab == TCX_F16 || ab == TCX_BF16) && cd == TCX_F32 && m == 16 && n == 8 && k == 16;
  const bool tf = ab == TCX_TF32 && cd == TCX_F32 && m == 16 && n == 8 && (k == 8 || k == 16);
  if (!(fp || tf))
    return set_error(TCX_ERR_UNSUPPORTED, "tcx_mma_tiles_tc05: (ab=%d, cd=%d, m%dn%dk%d) not supported", ab, cd, m, n, k);
  if (count < 0) return set_error(TCX_ERR_INVALID_VALUE, "tcx_mma_tiles_tc05: count < 0");
  if (count == 0) return TCX_OK;
  if (!A || !B || !D) return set_error(TCX_ERR_INVALID_VALUE, "tcx_mma_tiles_tc05: NULL operand");
  DevInfo dev;
  tcx_status st = current_device(&dev);
  if (st != TCX_OK) return st;
  return launch_tiles_tc05(ab, k, count, A, B, C, D, (cudaStream_t)stream);
}

tcx_status tcx_gemm_ex(tcx_dtype ab, tcx_dtype cd, int64_t M, int64_t N, int64_t K, const void* A, int64_t lda,
                       const void* B, int64_t ldb, const void* C, int64_t ldc, void* D, int64_t ldd,
                       const tcx_gemm_opts* opts, void* stream) {
  const bool ok = ((ab == TCX_F16 || ab == TCX_BF16 || ab == TCX_TF32) && cd == TCX_F32) || (ab == TCX_S8 && cd == TCX_S32) ||
                  (ab == TCX_F16 && cd == TCX_F16);
  if (!ok) return set_error(TCX_ERR_UNSUPPORTED, "tcx_gemm: (ab=%d, cd=%d) not supported", ab, cd);
  tcx_status st = check_gemm_common("tcx_gemm", ab, cd, M, N, K, A, lda, B, ldb, C, ldc, D, ldd, K);
  if (st != TCX_OK || M == 0 || N == 0) return st;
  // every argument check precedes the device query (host-testable without a GPU)
  GemmArgs g{ab, cd, M, N, K, A, lda, B, ldb, C, ldc, D, ldd, nullptr, 2, 0, 0, 0};
  if (opts) {
    if (opts->cta_group != 0 && opts->cta_group != 1 && opts->cta_group != 2)
      return set_error(TCX_ERR_INVALID_VALUE, "tcx_gemm: cta_group must be 0, 1 or 2");
    if (opts->cta_group) g.cta_group = opts->cta_group;
    g.max_ctas = opts->max_ctas;
    g.group_m = opts->group_m;
    const int tn = opts->tile_n;
    if (!(tn == 0 || tn == 128 || tn == 160 || tn == 192 || tn == 224 || tn == 256 || tn == 512))
      return set_error(TCX_ERR_INVALID_VALUE, "tcx_gemm: tile_n must be 0, 128, 160, 192, 224, 256 or 512");
    g.tile_n = tn;
    const int pm = opts->pairs_m ? opts->pairs_m : 1, pn = opts->pairs_n ? opts->pairs_n : 1;
    if (pm < 1 || pm > 2 || pn < 1 || pn > 2)
      return set_error(TCX_ERR_INVALID_VALUE, "tcx_gemm: pairs_m and pairs_n must be 0, 1 or 2");
    if ((pm > 1 || pn > 1) && (g.cta_group != 2 || (g.tile_n != 0 && g.tile_n != 256)))
      return set_error(TCX_ERR_INVALID_VALUE, "tcx_gemm: multicast clusters need cta_group 2 and the 256-wide tile");
    if (tn != 0 && tn < 256 && g.cta_group != 2)
      return set_error(TCX_ERR_UNSUPPORTED, "tcx_gemm: tile_n < 256 (narrow pair tiles) needs cta_group 2");
    if (g.tile_n == 512 && (g.cta_group != 2 || cd == TCX_F16))
      return set_error(TCX_ERR_UNSUPPORTED, "tcx_gemm: tile_n 512 (the 256 x 512 pair tile) needs cta_group 2 and a "
                       "32-bit accumulator");
    g.pairs_m = pm;
    g.pairs_n = pn;
    g.pairs_auto = opts->pairs_m == 0 && opts->pairs_n == 0 && opts->cta_group != 1 && (g.tile_n == 0 || g.tile_n == 256);
#if TCX_WATCHDOG
    g.fault = opts->reserved[0];   // fault injection exists only in the debug library
#endif
  }
  DevInfo dev;
  st = current_device(&dev);
  if (st != TCX_OK) return st;
#if TCX_WATCHDOG
  g.trace = g_trace;
  g.trace_cap = g_trace_cap;
#endif
  if (K == 0) return launch_fill_c(g, (cudaStream_t)stream);
  return launch_gemm_dense(g, dev, (cudaStream_t)stream);
}

tcx_status tcx_gemm(tcx_dtype ab, tcx_dtype cd, int64_t M, int64_t N, int64_t K, const void* A, int64_t lda,
                    const void* B, int64_t ldb, const void* C, int64_t ldc, void* D, int64_t ldd, void* stream) {
  return tcx_gemm_ex(ab, cd, M, N, K, A, lda, B, ldb, C, ldc, D, ldd, nullptr, stream);
}

tcx_status tcx_sp24_compress(tcx_dtype ab, int64_t M, int64_t K, const void* A_dense, int64_t lda, void* A_vals,
                             uint32_t* meta_canon, int64_t* d_first_bad, void* stream) {
  const int es = esize_of(ab);
  if (!(ab == TCX_F16 || ab == TCX_BF16 || ab == TCX_S8 || ab == TCX_TF32))
    return set_error(TCX_ERR_UNSUPPORTED, "tcx_sp24_compress: ab=%d", ab);
  if (M < 0 || K < 0 || K % 32) return set_error(TCX_ERR_INVALID_VALUE, "tcx_sp24_compress: K must be a multiple of 32");
  if (lda < K) return set_error(TCX_ERR_INVALID_VALUE, "tcx_sp24_compress: lda < K");
  if (!d_first_bad) return set_error(TCX_ERR_INVALID_VALUE, "tcx_sp24_compress: d_first_bad is NULL");
  if (M > 0 && K > 0 && (!A_dense || !A_vals || !meta_canon))
    return set_error(TCX_ERR_INVALID_VALUE, "tcx_sp24_compress: NULL operand");
  if (((uintptr_t)d_first_bad & 7u) != 0) return set_error(TCX_ERR_MISALIGNED, "tcx_sp24_compress: d_first_bad alignment");
  DevInfo dev;
  tcx_status st = current_device(&dev);
  if (st != TCX_OK) return st;
  return launch_sp24_compress(es, ab == TCX_TF32, M, K, A_dense, lda, A_vals, meta_canon, d_first_bad,
                              (cudaStream_t)stream);
}

size_t tcx_sp24_meta_hw_bytes(tcx_dtype ab, int64_t M, int64_t K) {
  if (!(ab == TCX_F16 || ab == TCX_BF16 || ab == TCX_S8 || ab == TCX_TF32) || M < 0 || K < 0) return 0;
  return (size_t)(M * K / (ab == TCX_TF32 ? 4 : 8));
}

tcx_status tcx_sp24_pack_meta(tcx_dtype ab, int64_t M, int64_t K, const uint32_t* meta_canon, void* meta_hw,
                              int64_t* d_first_bad, void* stream) {
  if (!(ab == TCX_F16 || ab == TCX_BF16 || ab == TCX_S8 || ab == TCX_TF32))
    return set_error(TCX_ERR_UNSUPPORTED, "tcx_sp24_pack_meta: ab=%d", ab);
  if (M < 0 || K < 0 || M % 128 || K % (ab == TCX_TF32 ? 64 : 128))
    return set_error(TCX_ERR_UNSUPPORTED, "tcx_sp24_pack_meta: M %% 128 and K %% %d must be 0", ab == TCX_TF32 ? 64 : 128);
  if (!d_first_bad) return set_error(TCX_ERR_INVALID_VALUE, "tcx_sp24_pack_meta: d_first_bad is NULL");
  if (M > 0 && K > 0 && (!meta_canon || !meta_hw)) return set_error(TCX_ERR_INVALID_VALUE, "tcx_sp24_pack_meta: NULL operand");
  DevInfo dev;
  tcx_status st = current_device(&dev);
  if (st != TCX_OK) return st;
  return launch_sp24_pack(ab, M, K, meta_canon, meta_hw, d_first_bad, (cudaStream_t)stream);
}

tcx_status tcx_gemm_sp24(tcx_dtype ab, tcx_dtype cd, int64_t M, int64_t N, int64_t K, const void* A_vals,
                         int64_t lda_vals, const void* meta_hw, const void* B, int64_t ldb, const void* C, int64_t ldc,
                         void* D, int64_t ldd, void* stream) {
  return tcx_gemm_sp24_ex(ab, cd, M, N, K, A_vals, lda_vals, meta_hw, B, ldb, C, ldc, D, ldd, nullptr, stream);
}

tcx_status tcx_gemm_sp24_ex(tcx_dtype ab, tcx_dtype cd, int64_t M, int64_t N, int64_t K, const void* A_vals,
                            int64_t lda_vals, const void* meta_hw, const void* B, int64_t ldb, const void* C,
                            int64_t ldc, void* D, int64_t ldd, const tcx_gemm_opts* opts, void* stream) {
  if (!(((ab == TCX_F16 || ab == TCX_BF16 || ab == TCX_TF32) && cd == TCX_F32) || (ab == TCX_S8 && cd == TCX_S32)))
    return set_error(TCX_ERR_UNSUPPORTED, "tcx_gemm_sp24: (ab=%d, cd=%d) not supported", ab, cd);
  if (M < 0 || N < 0 || K < 0) return set_error(TCX_ERR_INVALID_VALUE, "tcx_gemm_sp24: negative size");
  if (M == 0 || N == 0) return TCX_OK;
  const int64_t kstage = ab == TCX_S8 ? 256 : ab == TCX_TF32 ? 64 : 128;
  if (M % 128 || K % kstage || N % 16 || K == 0)
    return set_error(TCX_ERR_UNSUPPORTED, "tcx_gemm_sp24: requires M %% 128 == 0, K %% %d == 0, N %% 16 == 0",
                     (int)kstage);
  tcx_status st = check_gemm_common("tcx_gemm_sp24", ab, cd, M, N, K, A_vals, lda_vals, B, ldb, C, ldc, D, ldd, K / 2);
  if (st != TCX_OK) return st;
  if (!meta_hw || !aligned16(meta_hw)) return set_error(TCX_ERR_MISALIGNED, "tcx_gemm_sp24: meta_hw NULL or misaligned");
  GemmArgs g{ab, cd, M, N, K, A_vals, lda_vals, B, ldb, C, ldc, D, ldd, meta_hw, 2, 0, 0, 0};
  if (opts) {
    if (opts->cta_group != 0 && opts->cta_group != 1 && opts->cta_group != 2)
      return set_error(TCX_ERR_INVALID_VALUE, "tcx_gemm_sp24: cta_group must be 0, 1 or 2");
    if (opts->cta_group) g.cta_group = opts->cta_group;
    g.max_ctas = opts->max_ctas;
    g.group_m = opts->group_m;
    if (opts->tile_n != 0 && opts->tile_n != 256 && opts->tile_n != 512)
      return set_error(TCX_ERR_INVALID_VALUE, "tcx_gemm_sp24: tile_n (tile height) must be 0, 256 or 512");
    g.tile_n = opts->tile_n;
    const int pm = opts->pairs_m ? opts->pairs_m : 1, pn = opts->pairs_n ? opts->pairs_n : 1;
    if (pm < 1 || pm > 2 || pn < 1 || pn > 2)
      return set_error(TCX_ERR_INVALID_VALUE, "tcx_gemm_sp24: pairs_m and pairs_n must be 0, 1 or 2");
    if ((pm > 1 || pn > 1) && g.cta_group != 2)
      return set_error(TCX_ERR_INVALID_VALUE, "tcx_gemm_sp24: multicast groups need cta_group 2");
    if (g.tile_n == 512 && (g.cta_group != 2 || ab == TCX_S8 || M % 512))
      return set_error(TCX_ERR_UNSUPPORTED, "tcx_gemm_sp24: tile_n 512 (the 512 x 240 pair tile) needs cta_group 2, "
                       "F16/BF16/TF32 and M %% 512 == 0");
    g.pairs_m = pm;
    g.pairs_n = pn;
#if TCX_WATCHDOG
    g.fault = opts->reserved[0];   // debug library: energy-decomposition knobs (gemm_sp24.cu)
#endif
  }
  if (g.cta_group == 2 && M % 256)
    return set_error(TCX_ERR_UNSUPPORTED, "tcx_gemm_sp24: the CTA-pair kernel needs M %% 256 == 0 (use cta_group=1)");
#if TCX_WATCHDOG
  g.trace = g_trace;
  g.trace_cap = g_trace_cap;
#endif
  DevInfo dev;
  st = current_device(&dev);
  if (st != TCX_OK) return st;
  return launch_gemm_sp24(g, dev, (cudaStream_t)stream);
}

tcx_status tcx_round_tf32(const float* in, float* out, int64_t n, void* stream) {
  if (n < 0) return set_error(TCX_ERR_INVALID_VALUE, "tcx_round_tf32: n < 0");
  if (n == 0) return TCX_OK;
  if (!in || !out) return set_error(TCX_ERR_INVALID_VALUE, "tcx_round_tf32: NULL pointer");
  DevInfo dev;
  tcx_status st = current_device(&dev);
  if (st != TCX_OK) return st;
  return launch_round_tf32(in, out, n, (cudaStream_t)stream);
}

tcx_status tcx_probe(int device, const tcx_probe_config* cfg, tcx_probe_result* out) {
  if (!cfg || !out) return set_error(TCX_ERR_INVALID_VALUE, "tcx_probe: NULL cfg/out");
  int prev = -1;
  TCX_CUDA_TRY(cudaGetDevice(&prev));
  if (device >= 0 && device != prev) TCX_CUDA_TRY(cudaSetDevice(device));
  DevInfo dev;
  tcx_status st = current_device(&dev);
  if (st == TCX_OK) st = run_probe(dev, cfg, out);
  if (device >= 0 && device != prev) cudaSetDevice(prev);
  return st;
}

}  // extern "C"
