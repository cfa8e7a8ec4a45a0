// tcx dense GEMM on sm_100a:  D = A x B + C   ("row.col" operands PAPER.md:313-317)
//
// Persistent, warp-specialised tcgen05 kernel:
//   warp 0      TMA producer: A (128 x BK) and B (BN_LOAD x BK) K-major tiles -> 128B-swizzled smem
//   warp 1      MMA issuer (leader CTA only): tcgen05.mma kind::{f16,tf32,i8} into TMEM
//   warp 2      TMEM allocator (512 columns = two 128 x 256 FP32/S32 accumulators)
//   warps 4..7  epilogue: tcgen05.ld 32x32b -> (+C) -> vectorised global stores
// CG = 2 runs a CTA pair (cluster of 2, tcgen05 cta_group::2, UMMA M = 256): each CTA loads its
// 128 rows of A and half (128 rows) of the N x K B tile; the leader issues the MMAs.
// BK is one 128-byte swizzle row for every kind (64 f16/bf16, 32 tf32, 128 s8), and every
// UMMA consumes 32 bytes of K (UMMA_K = 16 / 8 / 32).
#include "tcx_internal.h"
#include "ptx.cuh"

namespace tcx {
namespace {

constexpr int BM = 128;            // rows per CTA (UMMA M = BM * CG)
constexpr int BN = 256;            // UMMA N
constexpr int KBYTES = 128;        // K bytes per stage (one SW128 row)
constexpr int UMMA_KBYTES = 32;    // K bytes per tcgen05.mma
constexpr int EPI_WARPS = 4;
constexpr int NUM_THREADS = 256;
constexpr int GROUP_M = 8;         // default raster: GROUP_M cluster-tile rows share B tiles in L2

template <int CG>
struct Cfg {
  static constexpr int BN_LOAD = BN / CG;                        // B rows loaded per CTA
  static constexpr int A_BYTES = BM * KBYTES;                    // 16 KiB
  static constexpr int B_BYTES = BN_LOAD * KBYTES;               // 32 or 16 KiB
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = CG == 1 ? 4 : 6;
  static constexpr int SMEM_DATA = STAGES * STAGE_BYTES;
  static constexpr int SMEM_TOTAL = SMEM_DATA + 1024 /*barriers*/ + 1024 /*align slack*/;
};

template <int KIND> struct KindT;
template <> struct KindT<KIND_F16> { static constexpr int ESIZE = 2; };
template <> struct KindT<KIND_TF32> { static constexpr int ESIZE = 4; };
template <> struct KindT<KIND_I8> { static constexpr int ESIZE = 1; };

// instruction descriptor (kind::f16 / tf32 / i8), K-major A and B, dense
__host__ __device__ constexpr uint32_t make_idesc(int kind, int a_fmt, int M, int N) {
  // c_format [4,6): F32 = 1, S32 = 2;  a_format [7,10), b_format [10,13);
  // N >> 3 at [17,23), M >> 4 at [24,29)
  return ((kind == KIND_I8 ? 2u : 1u) << 4) | ((uint32_t)a_fmt << 7) | ((uint32_t)a_fmt << 10) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

struct Smem {
  uint64_t full[8];
  uint64_t empty[8];
  uint64_t tmem_full[2];
  uint64_t tmem_empty[2];
  uint32_t tmem_base;
};

__device__ __forceinline__ void tile_coords(int64_t tile, int64_t m_tiles, int64_t n_tiles, int group_m,
                                            int64_t& mt, int64_t& nt) {
  // grouped raster: group_m m-tiles x all n-tiles, m fastest inside a group
  int64_t per_group = (int64_t)group_m * n_tiles;
  int64_t g = tile / per_group;
  int64_t first_m = g * group_m;
  int64_t gm = m_tiles - first_m < group_m ? m_tiles - first_m : group_m;
  int64_t r = tile - g * per_group;
  mt = first_m + r % gm;
  nt = r / gm;
}

template <int CG, int KIND>
__global__ void __launch_bounds__(NUM_THREADS, 1)
gemm_dense_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                  int64_t M, int64_t N, int64_t K, const void* __restrict__ Cptr, int64_t ldc,
                  void* __restrict__ Dptr, int64_t ldd, uint32_t idesc, int group_m) {
  using C_ = Cfg<CG>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  Smem* sm = (Smem*)(smem + C_::SMEM_DATA);

  const int warp = threadIdx.x / 32;
  const uint32_t rank = CG == 2 ? cluster_ctarank() : 0;
  const bool leader = rank == 0;

  const int64_t m_tiles = (M + BM * CG - 1) / (BM * CG);
  const int64_t n_tiles = (N + BN - 1) / BN;
  const int64_t num_tiles = m_tiles * n_tiles;
  const int64_t k_blocks = (K * KindT<KIND>::ESIZE + KBYTES - 1) / KBYTES;
  const int64_t cluster_id = blockIdx.x / CG;
  const int64_t num_clusters = gridDim.x / CG;

  if (threadIdx.x == 0) {
    for (int s = 0; s < C_::STAGES; ++s) { mbar_init(&sm->full[s], 1); mbar_init(&sm->empty[s], 1); }
    for (int a = 0; a < 2; ++a) { mbar_init(&sm->tmem_full[a], 1); mbar_init(&sm->tmem_empty[a], EPI_WARPS * CG); }
    fence_mbar_init();
  }
  if (warp == 0 && elect_one()) { tma_prefetch(&tmA); tma_prefetch(&tmB); }
  if (warp == 2) { tmem_alloc<CG>(&sm->tmem_base, 512); tmem_relinquish<CG>(); }
  tc05_fence_before();
  if constexpr (CG == 2) cluster_sync(); else __syncthreads();
  tc05_fence_after();
  const uint32_t tmem_base = sm->tmem_base;

  if (warp == 0) {
    // ================= TMA producer =================
    if (elect_one()) {
      int stage = 0; uint32_t phase = 0;
      const uint32_t full0_cluster = CG == 2 ? mapa(smem_u32(&sm->full[0]), 0) : 0;
      for (int64_t tile = cluster_id; tile < num_tiles; tile += num_clusters) {
        int64_t mt, nt;
        tile_coords(tile, m_tiles, n_tiles, group_m, mt, nt);
        const int arow = (int)(mt * BM * CG + rank * BM);
        const int brow = (int)(nt * BN + rank * C_::BN_LOAD);
        for (int64_t kb = 0; kb < k_blocks; ++kb) {
          mbar_wait(&sm->empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * C_::STAGE_BYTES;
          uint8_t* sb = sa + C_::A_BYTES;
          const int kx = (int)(kb * (KBYTES / KindT<KIND>::ESIZE));
          if constexpr (CG == 1) {
            mbar_arrive_expect_tx(&sm->full[stage], C_::STAGE_BYTES);
            tma_load_2d(sa, &tmA, &sm->full[stage], kx, arow);
            tma_load_2d(sb, &tmB, &sm->full[stage], kx, brow);
          } else {
            if (leader) mbar_arrive_expect_tx(&sm->full[stage], 2 * C_::STAGE_BYTES);
            const uint32_t bar = full0_cluster + stage * 8;
            tma_load_2d_cg2(sa, &tmA, bar, kx, arow);
            tma_load_2d_cg2(sb, &tmB, bar, kx, brow);
          }
          if (++stage == C_::STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ================= MMA issuer (leader CTA) =================
    if (leader) {
      int stage = 0; uint32_t phase = 0;
      int acc = 0; uint32_t acc_phase = 0;
      for (int64_t tile = cluster_id; tile < num_tiles; tile += num_clusters) {
        mbar_wait(&sm->tmem_empty[acc], acc_phase ^ 1);
        tc05_fence_after();
        const uint32_t tmem_d = tmem_base + acc * BN;
        for (int64_t kb = 0; kb < k_blocks; ++kb) {
          mbar_wait(&sm->full[stage], phase);
          tc05_fence_after();
          if (elect_one()) {
            const uint32_t sa = smem_u32(smem + stage * C_::STAGE_BYTES);
            const uint32_t sb = sa + C_::A_BYTES;
#pragma unroll
            for (int k = 0; k < KBYTES / UMMA_KBYTES; ++k) {
              const uint64_t ad = sdesc(sa + k * UMMA_KBYTES, 16, 1024, 2);
              const uint64_t bd = sdesc(sb + k * UMMA_KBYTES, 16, 1024, 2);
              umma<CG, KIND>(tmem_d, ad, bd, idesc, (kb | k) ? 1u : 0u);
            }
            tc05_commit<CG>(&sm->empty[stage]);                   // frees the smem slot
            if (kb == k_blocks - 1) tc05_commit<CG>(&sm->tmem_full[acc]);   // accumulator ready
          }
          __syncwarp();
          if (++stage == C_::STAGES) { stage = 0; phase ^= 1; }
        }
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else if (warp >= 4) {
    // ================= epilogue =================
    const int e = warp - 4;                       // TMEM lanes 32e .. 32e+31
    const int lane = threadIdx.x & 31;
    int acc = 0; uint32_t acc_phase = 0;
    const uint32_t tmem_empty_cluster = CG == 2 ? mapa(smem_u32(&sm->tmem_empty[0]), 0) : smem_u32(&sm->tmem_empty[0]);
    for (int64_t tile = cluster_id; tile < num_tiles; tile += num_clusters) {
      int64_t mt, nt;
      tile_coords(tile, m_tiles, n_tiles, group_m, mt, nt);
      const int64_t row = mt * BM * CG + rank * BM + e * 32 + lane;
      const int64_t col0 = nt * BN;
      mbar_wait(&sm->tmem_full[acc], acc_phase);
      tc05_fence_after();
      const bool row_ok = row < M;
#pragma unroll 1
      for (int ch = 0; ch < BN / 32; ++ch) {
        const int64_t c0 = col0 + ch * 32;
        uint32_t v[32];
        tmem_ld_32x32b_x32(tmem_base + acc * BN + ch * 32 + ((uint32_t)(e * 32) << 16), v);
        uint32_t cv[32];
        const bool full_chunk = c0 + 32 <= N;
        if (Cptr != nullptr && row_ok && c0 < N) {
          const uint32_t* crow = (const uint32_t*)Cptr + row * ldc + c0;
          if (full_chunk) {
#pragma unroll
            for (int j = 0; j < 32; j += 4) {
              uint4 t = __ldg((const uint4*)(crow + j));
              cv[j] = t.x; cv[j + 1] = t.y; cv[j + 2] = t.z; cv[j + 3] = t.w;
            }
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j) cv[j] = (c0 + j < N) ? crow[j] : 0u;
          }
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j) cv[j] = 0u;
        }
        tmem_ld_wait();
        if (ch == BN / 32 - 1) {
          // accumulator fully read: hand the TMEM buffer back to the MMA warp
          tc05_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_cluster(tmem_empty_cluster + acc * 8);
        }
        uint32_t out[32];
        if constexpr (KIND == KIND_I8) {
#pragma unroll
          for (int j = 0; j < 32; ++j) out[j] = v[j] + cv[j];          // wrap mod 2^32
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j) out[j] = __float_as_uint(__fadd_rn(__uint_as_float(v[j]), __uint_as_float(cv[j])));
          if (Cptr == nullptr) {
#pragma unroll
            for (int j = 0; j < 32; ++j) out[j] = v[j];                  // no C: D = acc exactly
          }
        }
        if (row_ok && c0 < N) {
          uint32_t* drow = (uint32_t*)Dptr + row * ldd + c0;
          if (full_chunk) {
#pragma unroll
            for (int j = 0; j < 32; j += 4)
              *(uint4*)(drow + j) = make_uint4(out[j], out[j + 1], out[j + 2], out[j + 3]);
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j) if (c0 + j < N) drow[j] = out[j];
          }
        }
      }
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
  }

  tc05_fence_before();
  if constexpr (CG == 2) cluster_sync(); else __syncthreads();
  if (warp == 2) { tc05_fence_after(); tmem_dealloc<CG>(tmem_base, 512); }
}

__global__ void fill_c_kernel(const uint32_t* C, int64_t ldc, uint32_t* D, int64_t ldd, int64_t M, int64_t N) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t total = M * N;
  for (; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = i / N, c = i % N;
    D[r * ldd + c] = C ? C[r * ldc + c] : 0u;
  }
}

template <int CG, int KIND>
tcx_status launch_t(const GemmArgs& a, const DevInfo& dev, cudaStream_t s, CUtensorMapDataType dt, int a_fmt) {
  using C_ = Cfg<CG>;
  constexpr int ES = KindT<KIND>::ESIZE;
  CUtensorMap tA, tB;
  tcx_status st = make_tmap_2d(&tA, dt, a.A, (uint64_t)a.K, (uint64_t)a.M, (uint64_t)(a.lda * ES),
                               KBYTES / ES, BM, CU_TENSOR_MAP_SWIZZLE_128B);
  if (st != TCX_OK) return st;
  st = make_tmap_2d(&tB, dt, a.B, (uint64_t)a.K, (uint64_t)a.N, (uint64_t)(a.ldb * ES),
                    KBYTES / ES, C_::BN_LOAD, CU_TENSOR_MAP_SWIZZLE_128B);
  if (st != TCX_OK) return st;
  auto kern = gemm_dense_kernel<CG, KIND>;
  TCX_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C_::SMEM_TOTAL));
  const int64_t m_tiles = (a.M + BM * CG - 1) / (BM * CG);
  const int64_t n_tiles = (a.N + BN - 1) / BN;
  int64_t clusters = m_tiles * n_tiles;
  int64_t max_clusters = dev.sm_count / CG;
  if (a.max_ctas > 0 && a.max_ctas / CG < max_clusters) max_clusters = a.max_ctas / CG > 0 ? a.max_ctas / CG : 1;
  if (clusters > max_clusters) clusters = max_clusters;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(clusters * CG));
  cfg.blockDim = dim3(NUM_THREADS);
  cfg.dynamicSmemBytes = C_::SMEM_TOTAL;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CG; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr; cfg.numAttrs = 1;
  const uint32_t idesc = make_idesc(KIND, a_fmt, BM * CG, BN);
  TCX_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, tA, tB, (int64_t)a.M, (int64_t)a.N, (int64_t)a.K, a.C,
                                  (int64_t)a.ldc, a.D, (int64_t)a.ldd, idesc,
                                  a.group_m > 0 ? a.group_m : GROUP_M));
  count_launch();
  return TCX_OK;
}

}  // namespace

tcx_status launch_fill_c(const GemmArgs& a, cudaStream_t s) {
  int64_t total = a.M * a.N;
  int blocks = (int)((total + 255) / 256 < 4096 ? (total + 255) / 256 : 4096);
  if (blocks < 1) blocks = 1;
  fill_c_kernel<<<blocks, 256, 0, s>>>((const uint32_t*)a.C, a.ldc, (uint32_t*)a.D, a.ldd, a.M, a.N);
  TCX_CUDA_TRY(cudaGetLastError());
  count_launch();
  return TCX_OK;
}

tcx_status launch_gemm_dense(const GemmArgs& a, const DevInfo& dev, cudaStream_t s) {
  const int cg = a.cta_group == 1 ? 1 : 2;
  switch (a.ab) {
    case TCX_F16:
      return cg == 1 ? launch_t<1, KIND_F16>(a, dev, s, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 0)
                     : launch_t<2, KIND_F16>(a, dev, s, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 0);
    case TCX_BF16:
      return cg == 1 ? launch_t<1, KIND_F16>(a, dev, s, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 1)
                     : launch_t<2, KIND_F16>(a, dev, s, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 1);
    case TCX_TF32:
      return cg == 1 ? launch_t<1, KIND_TF32>(a, dev, s, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2)
                     : launch_t<2, KIND_TF32>(a, dev, s, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2);
    case TCX_S8:
      return cg == 1 ? launch_t<1, KIND_I8>(a, dev, s, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1)
                     : launch_t<2, KIND_I8>(a, dev, s, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1);
    default:
      return set_error(TCX_ERR_UNSUPPORTED, "tcx_gemm: unsupported ab type %d", (int)a.ab);
  }
}

}  // namespace tcx
