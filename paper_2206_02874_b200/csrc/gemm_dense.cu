// tcx dense GEMM on sm_100a:  D = A x B + C   ("row.col" operands PAPER.md:313-317)
//
// Persistent, warp-specialised tcgen05 kernel:
//   warp 0      TMA producer: A (128 x BK) and B (BN_LOAD x BK) K-major tiles -> 128B-swizzled smem
//   warp 1      MMA issuer (leader CTA only): tcgen05.mma kind::{f16,tf32,i8} into TMEM
//   warp 2      TMEM allocator (512 columns = two 128 x 256 FP32/S32 accumulators)
//   warps 4..7  epilogue: tcgen05.ld 32x32b -> (+C via TMA) -> swizzled smem -> TMA store
// CG = 2 runs a CTA pair (cluster of 2, tcgen05 cta_group::2, UMMA M = 256): each CTA loads its
// 128 rows of A and half (128 rows) of the N x K B tile; the leader issues the MMAs.
// NH = 2 ("wide" tile, 256 x 512 per pair): every k-step issues two N = 256 MMAs that share the
// A operand, so each stage moves 48 KiB per CTA for 2x the work of a 32 KiB NH = 1 stage — 25%
// less L2->SM operand traffic per FLOP (the power-capped B200 turns that into clock); the two
// halves fill all 512 TMEM columns, so the accumulator is single-buffered and the epilogue drains
// half 0 first (its own empty barrier) so the next tile's half-0 MMAs can start early.
// PM x PN > 1 (CG = 2, NH = 1): a group of PM x PN CTA pairs (CL = 2 PM PN consecutive CTAs)
// computes a (256 PM) x (256 PN) block of adjacent pair tiles.  The pairs of a row need the same A
// rows and the pairs of a column the same B rows, so when the group is one cluster each CTA
// TMA-loads only a 1/PN slice of its A half and a 1/PM slice of its B half and multicasts it to the
// CTAs that share it (same pair rank): L2->SM operand reads drop by (1/PN + 1/PM)/2 with the
// 256 x 256 double-buffered accumulator kept, and every pair's commit of a smem slot arrives at
// every CTA of the cluster (empty barriers count PM x PN arrivals).  Clusters of 4 / 8 CTAs must
// sit inside one GPC and B200's GPCs fit fewer of them than 148 SMs (33 x 4, 15 x 8), so the
// launch asks for CL-CTA clusters as the *preferred* shape over plain pairs: a group the hardware
// could not place as one cluster runs as independent pairs (%cluster_nctarank == 2) on the same
// tiles, loading every slice itself — every SM works, and the groups that did form multicast.
// BK is one 128-byte swizzle row for every kind (64 f16/bf16, 32 tf32, 128 s8), and every
// UMMA consumes 32 bytes of K (UMMA_K = 16 / 8 / 32).
#include <cstdio>
#include <cstdlib>
#include "tcx_internal.h"
#include "ptx.cuh"

namespace tcx {
namespace {

constexpr int BM = 128;            // rows per CTA (UMMA M = BM * CG)
constexpr int BN_FULL = 256;       // UMMA N of the default tile (narrower N: wave-quantisation choice)
constexpr int KBYTES = 128;        // K bytes per stage (one SW128 row)
constexpr int UMMA_KBYTES = 32;    // K bytes per tcgen05.mma
constexpr int EPI_WARPS = 4;
constexpr int NUM_THREADS = 256;
constexpr int GROUP_M = 8;         // default raster: GROUP_M cluster-tile rows share B tiles in L2

template <int CG, int NH, int BN_ = BN_FULL>
struct Cfg {
  static constexpr int BN = BN_;                                 // UMMA N (one N-half)
  static_assert(BN % 32 == 0 && BN >= 128 && BN <= 256 && (NH == 1 || BN == 256), "tile width");
  static constexpr int ACC_COLS = NH * 256;                      // TMEM column stride between accumulators
  static constexpr int TILE_M = BM * CG;                         // output rows per tile
  static constexpr int TILE_N = BN * NH;                         // output columns per tile
  static constexpr int BN_LOAD = BN / CG;                        // B rows per CTA per N-half
  static constexpr int HALF_BYTES = BN_LOAD * KBYTES;            // one N-half of B in smem
  static constexpr int A_BYTES = BM * KBYTES;                    // 16 KiB
  static constexpr int B_BYTES = NH * HALF_BYTES;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
#ifndef TCX_DENSE_STAGES          // experiment knobs (tools/build_variant.py); defaults are the product's
#define TCX_DENSE_STAGES 6
#endif
#ifndef TCX_DENSE_NBE
#define TCX_DENSE_NBE 2
#endif
#ifndef TCX_WIDE_STAGES
#define TCX_WIDE_STAGES 3
#endif
#ifndef TCX_WIDE_NBE
#define TCX_WIDE_NBE 4
#endif
  static constexpr int STAGES = NH == 2 ? TCX_WIDE_STAGES : (CG == 1 ? 4 : TCX_DENSE_STAGES);
  // epilogue staging buffers per warp (4 KiB each) and how far ahead C is loaded: the wide tile's
  // single accumulator puts the epilogue on the critical path, so it trades a ring stage for depth
  static constexpr int NBE = NH == 2 ? TCX_WIDE_NBE : (CG == 1 ? 2 : TCX_DENSE_NBE);
  static constexpr int C_AHEAD = NBE == 2 ? 2 : NBE - 1;
  static constexpr int NBUF = 2 / NH;                            // TMEM accumulator buffers
  static constexpr int SMEM_DATA = STAGES * STAGE_BYTES;
  static constexpr int STG_BYTES = EPI_WARPS * NBE * 4096;       // epilogue: NBE x 4 KiB per warp
  static constexpr int SMEM_TOTAL = SMEM_DATA + STG_BYTES + 1024 /*barriers*/ + 1024 /*align slack*/;
  static_assert(NH == 1 || CG == 2, "wide tiles need the CTA pair");
  static_assert(SMEM_TOTAL <= 232448, "smem budget");
};

// FP16 inputs with an FP16 accumulator (idesc c_format F16; the f16.f16.f16.f16 MMA of PAPER.md:428-429
// at GEMM scale): C and D are FP16, and C is the MMA's own C operand — preloaded into the tensor-memory
// accumulator by the epilogue warps (tcgen05.st) before the tile's first MMA (enable_input_d = 1).
constexpr int KIND_F16ACC = 3;
template <int KIND> struct KindT;
template <> struct KindT<KIND_F16> { static constexpr int ESIZE = 2; };
template <> struct KindT<KIND_F16ACC> { static constexpr int ESIZE = 2; };
template <> struct KindT<KIND_TF32> { static constexpr int ESIZE = 4; };
template <> struct KindT<KIND_I8> { static constexpr int ESIZE = 1; };

// instruction descriptor (kind::f16 / tf32 / i8), K-major A and B, dense
__host__ __device__ constexpr uint32_t make_idesc(int kind, int a_fmt, int M, int N) {
  // c_format [4,6): F16 = 0, F32 = 1, S32 = 2;  a_format [7,10), b_format [10,13);
  // N >> 3 at [17,23), M >> 4 at [24,29)
  return ((kind == KIND_I8 ? 2u : kind == KIND_F16ACC ? 0u : 1u) << 4) | ((uint32_t)a_fmt << 7) | ((uint32_t)a_fmt << 10) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

struct Smem {
  uint64_t full[8];
  uint64_t empty[8];
  uint64_t tmem_full[2];
  uint64_t tmem_empty[2];      // NH = 1: per buffer; NH = 2: per N-half of the single buffer
  uint64_t cbar[EPI_WARPS][4]; // epilogue: C chunk landed in staging buffer b of warp e
  uint64_t cring[EPI_WARPS];   // epilogue, last tile: all of warp e's C chunks landed in the idle ring
  uint32_t tmem_base;
};

__device__ __forceinline__ void tile_coords(int64_t tile, int64_t m_tiles, int64_t n_tiles, int group,
                                            int64_t& mt, int64_t& nt) {
  // grouped raster.  group > 0: `group` m-tiles x all n-tiles per group, m fastest inside a group
  // (the group's A rows stay in L2 while B streams past); group < 0: |group| n-tiles x all m-tiles,
  // n fastest (B's columns stay while A streams) — the cheaper one re-reads the smaller operand
  const bool by_m = group > 0;
  const int64_t g_tiles = by_m ? group : -group;
  const int64_t major = by_m ? m_tiles : n_tiles, minor = by_m ? n_tiles : m_tiles;
  const int64_t per_group = g_tiles * minor;
  const int64_t g = tile / per_group;
  const int64_t first = g * g_tiles;
  const int64_t gm = major - first < g_tiles ? major - first : g_tiles;
  const int64_t r = tile - g * per_group;
  const int64_t a = first + r % gm;
  // serpentine: odd groups sweep the minor dimension backwards, so a group starts on the operand
  // tiles the previous group read last (still in L2)
  const int64_t b = (g & 1) ? minor - 1 - r / gm : r / gm;
  mt = by_m ? a : b;
  nt = by_m ? b : a;
}

#if TCX_WATCHDOG
// debug library, energy decomposition (knob "no operand loads"): fill the operand ring once with
// pseudo-random FP16/BF16 values of N(0,1)-like magnitude (random sign, exponent 2^-4 .. 2^1, random
// fraction) and valid 2:4 metadata nibbles, so the MMAs of a load-free run toggle like real data
__device__ __forceinline__ uint32_t dbg_hash(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}
__device__ __forceinline__ uint32_t dbg_half(uint32_t h, bool bf16) {
  const uint32_t sign = (h >> 31) & 1u, e = 11u + (h >> 28 & 7u) % 6u;     // f16 exponent field 11..16
  if (!bf16) return (sign << 15) | (e << 10) | (h & 0x3FFu);
  return (sign << 15) | ((e - 15u + 127u) << 7) | (h & 0x7Fu);
}
__device__ void dbg_fill_ring(uint8_t* base, int bytes, int meta_off, int meta_bytes, int stage_bytes, bool bf16) {
  static const uint8_t nib[6] = {0x4, 0x8, 0xC, 0x9, 0xD, 0xE};
  for (int i = threadIdx.x * 4; i < bytes; i += blockDim.x * 4) {
    const uint32_t h = dbg_hash((uint32_t)i * 2654435761u + blockIdx.x * 97u);
    const int in_stage = i % stage_bytes;
    uint32_t w;
    if (meta_bytes > 0 && in_stage >= meta_off && in_stage < meta_off + meta_bytes) {
      w = 0;
      for (int j = 0; j < 8; ++j) w |= (uint32_t)nib[(h >> (4 * j)) % 6u] << (4 * j);
    } else {
      w = dbg_half(h, bf16) | (dbg_half(dbg_hash(h), bf16) << 16);
    }
    *(uint32_t*)(base + i) = w;
  }
}
#endif

template <int CG, int KIND, int NH, int PM, int PN, int BNT>
__global__ void __launch_bounds__(NUM_THREADS, 1)
gemm_dense_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                  const __grid_constant__ CUtensorMap tmC, const __grid_constant__ CUtensorMap tmD,
                  int64_t M, int64_t N, int64_t K, int has_c, uint32_t idesc, int group_m, int look, int fault,
                  uint64_t* trace, int64_t trace_cap) {
  using C_ = Cfg<CG, NH, BNT>;
  constexpr int BN = BNT;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  Smem* sm = (Smem*)(smem + C_::SMEM_DATA + C_::STG_BYTES);
  // `fault` (debug library only, 0 in the product): 1 = drop one TMA load (watchdog test); energy
  // decomposition bits as in gemm_sp24.cu: 2 = no MMAs, 4 = no operand loads, 8 = no epilogue traffic
#if !TCX_WATCHDOG
  fault = 0;
#endif
  const bool k_nomma = fault & 2, k_noload = fault & 4, k_noepi = fault & 8;
  if (k_noepi && KIND != KIND_F16ACC) has_c = 0;

  constexpr int P = PM * PN;                 // CTA pairs per cluster
  constexpr int CL = CG * P;                 // CTAs per cluster
  static_assert(P == 1 || (CG == 2 && NH == 1), "multicast clusters: CTA pairs, 256-wide tile");
  const int warp = threadIdx.x / 32;
  const uint32_t crank = CG > 1 ? cluster_ctarank() : 0;
  const bool mc = P > 1 && cluster_nctarank() == (uint32_t)CL;    // this group formed one cluster
  const uint32_t rank = crank % CG;          // rank inside the CTA pair
  const uint32_t pair = (blockIdx.x % CL) / CG;                   // pair slot inside the group
  const int pm = (int)(pair % PM), pn = (int)(pair / PM);
  const uint32_t lead_rank = mc ? pair * CG : 0;                  // this pair's leader CTA (cluster rank)
  const bool leader = rank == 0;
  if (P > 1 && crank != (mc ? blockIdx.x % CL : blockIdx.x % CG)) __trap();   // cluster = aligned CTA block

  const int64_t m_tiles = (M + C_::TILE_M - 1) / C_::TILE_M;
  const int64_t n_tiles = (N + C_::TILE_N - 1) / C_::TILE_N;
  const int64_t sm_tiles = (m_tiles + PM - 1) / PM;     // cluster tiles (PM x PN pair tiles each)
  const int64_t sn_tiles = (n_tiles + PN - 1) / PN;
  const int64_t num_tiles = sm_tiles * sn_tiles;
  const int64_t k_blocks = (K * KindT<KIND>::ESIZE + KBYTES - 1) / KBYTES;
  const int64_t cluster_id = blockIdx.x / CL;
  const int64_t num_clusters = gridDim.x / CL;
  // this pair's tile of cluster tile `tile` (a pair past the M / N edge computes on TMA zero fill
  // and its stores are clipped: it still feeds its multicast slices to the other pairs)
  auto pair_tile = [&](int64_t tile, int64_t& mt, int64_t& nt) {
    int64_t smt, snt;
    tile_coords(tile, sm_tiles, sn_tiles, group_m, smt, snt);
    mt = smt * PM + pm;
    nt = snt * PN + pn;
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < C_::STAGES; ++s) { mbar_init(&sm->full[s], 1); mbar_init(&sm->empty[s], mc ? P : 1); }
    for (int a = 0; a < 2; ++a) { mbar_init(&sm->tmem_full[a], 1); mbar_init(&sm->tmem_empty[a], EPI_WARPS * CG); }
    for (int w = 0; w < EPI_WARPS; ++w) {
      for (int b = 0; b < 4; ++b) mbar_init(&sm->cbar[w][b], 1); mbar_init(&sm->cring[w], 1);
    }
    fence_mbar_init();
  }
  if (warp == 0 && elect_one()) { tma_prefetch(&tmA); tma_prefetch(&tmB); tma_prefetch(&tmC); tma_prefetch(&tmD); }
  if (warp == 2) { tmem_alloc<CG>(&sm->tmem_base, 512); tmem_relinquish<CG>(); }
  tc05_fence_before();
  if constexpr (CG > 1) cluster_sync(); else __syncthreads();
  tc05_fence_after();
  const uint32_t tmem_base = sm->tmem_base;
  // PDL: the setup above (barriers, TMEM allocation, descriptor prefetch) overlapped the previous
  // grid's tail; no global memory is touched before its completion
  pdl_wait();
  pdl_trigger();
#if TCX_WATCHDOG
  if (k_noload && KIND == KIND_F16) {
    dbg_fill_ring(smem, C_::SMEM_DATA, 0, 0, C_::STAGE_BYTES, true);
    fence_proxy_async_smem();
    __syncthreads();
  }
#endif

  if (warp == 0) {
    // ================= TMA producer =================
    if (elect_one()) {
      int stage = 0; uint32_t phase = 0;
      const uint32_t full0_cluster = CG == 2 ? mapa(smem_u32(&sm->full[0]), lead_rank) : 0;
      constexpr int A_ROWS = BM / PN, B_ROWS = C_::BN_LOAD / PM;       // rows this CTA loads
      uint16_t mask_a = 0, mask_b = 0;                                   // CTAs sharing them
      for (int j = 0; j < PN; ++j) mask_a |= (uint16_t)(1u << ((pm + PM * j) * CG + rank));
      for (int i = 0; i < PM; ++i) mask_b |= (uint16_t)(1u << ((i + PM * pn) * CG + rank));
      for (int64_t tile = cluster_id; tile < num_tiles; tile += num_clusters) {
        int64_t mt, nt;
        pair_tile(tile, mt, nt);
        const int arow = (int)(mt * C_::TILE_M + rank * BM);               // + j * A_ROWS for slice j
        const int brow = (int)(nt * C_::TILE_N + rank * C_::BN_LOAD);      // + h * BN for N-half h
        // wide tile: segments (N-half 0, k-blocks [0, L)), (N-half 1, [0, L)), (both halves, [L, KB))
        // — the first L k-blocks are loaded once per half (A twice), see the MMA warp
        const int64_t L = NH == 2 ? (look < k_blocks ? look : k_blocks) : 0;
        for (int64_t i = 0; i < k_blocks + L; ++i) {
          const int64_t kb = i < 2 * L ? (i < L ? i : i - L) : i - L;
          const uint32_t hmask = i < L ? 1u : i < 2 * L ? 2u : 3u;   // N-halves this slot carries
          mbar_wait(&sm->empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * C_::STAGE_BYTES;
          uint8_t* sb = sa + C_::A_BYTES;
          const int kx = (int)(kb * (KBYTES / KindT<KIND>::ESIZE));
          if (k_noload) {                       // debug: the slot is "filled" without moving a byte
            if (CG == 1 || leader) mbar_arrive_expect_tx(&sm->full[stage], 0);
            if (++stage == C_::STAGES) { stage = 0; phase ^= 1; }
            continue;
          }
          if constexpr (CG == 1) {
            mbar_arrive_expect_tx(&sm->full[stage], C_::STAGE_BYTES);
            tma_load_2d<HINT_AB>(sa, &tmA, &sm->full[stage], kx, arow, l2_policy_a());
            tma_load_2d<HINT_AB>(sb, &tmB, &sm->full[stage], kx, brow, l2_policy_b());
          } else {
            if (leader)
              mbar_arrive_expect_tx(&sm->full[stage], NH == 2 && hmask != 3u ? 2 * (C_::A_BYTES + C_::HALF_BYTES)
                                                                              : 2 * C_::STAGE_BYTES);
            const uint32_t bar = full0_cluster + stage * 8;
#if TCX_WATCHDOG
            // fault injection (debug library): the first A load is never issued, its barrier never
            // completes, and the MMA warp's bounded wait traps
            if ((fault & 1) && tile == cluster_id && kb == 0) {
              if (++stage == C_::STAGES) { stage = 0; phase ^= 1; }
              continue;
            }
#else
            (void)fault; (void)trace; (void)trace_cap;
#endif
            if (PN > 1 && mc) {
              tma_load_2d_cg2_mc<HINT_AB>(sa + pn * A_ROWS * KBYTES, &tmA, bar, kx, arow + pn * A_ROWS, mask_a, l2_policy_a());
            } else {
#pragma unroll
              for (int j = 0; j < PN; ++j) tma_load_2d_cg2<HINT_AB>(sa + j * A_ROWS * KBYTES, &tmA, bar, kx, arow + j * A_ROWS, l2_policy_a());
            }
            if (PM > 1 && mc) {
              tma_load_2d_cg2_mc<HINT_AB>(sb + pm * B_ROWS * KBYTES, &tmB, bar, kx, brow + pm * B_ROWS, mask_b, l2_policy_b());
            } else {
#pragma unroll
              for (int h = 0; h < NH; ++h)
#pragma unroll
                for (int r = 0; r < PM; ++r)
                  if ((hmask >> h) & 1u)
                    tma_load_2d_cg2<HINT_AB>(sb + h * C_::HALF_BYTES + r * B_ROWS * KBYTES, &tmB, bar, kx, brow + h * BN + r * B_ROWS, l2_policy_b());
            }
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
      // FP16 accumulate with C: the accumulator holds C (preloaded) from the first MMA on
      const bool acc16_c = KIND == KIND_F16ACC && has_c;
      auto issue = [&](int st, int h, int64_t kb, uint32_t tmem_d) {
        if (k_nomma) return;
        const uint32_t sa = smem_u32(smem + st * C_::STAGE_BYTES);
        const uint32_t sb = sa + C_::A_BYTES + h * C_::HALF_BYTES;              // N-half h's B rows
#pragma unroll
        for (int k = 0; k < KBYTES / UMMA_KBYTES; ++k)
          umma<CG, KIND == KIND_F16ACC ? KIND_F16 : KIND>(tmem_d + h * BN, sdesc(sa + k * UMMA_KBYTES, 16, 1024, 2),
                                                          sdesc(sb + k * UMMA_KBYTES, 16, 1024, 2), idesc,
                                                          (acc16_c || (kb | k)) ? 1u : 0u);
      };
      // a slot's commit reaches every CTA that fed it (P > 1: the whole cluster); the accumulator's
      // reaches both CTAs of this pair
      auto commit_slot = [&](uint64_t* bar) {
        if (P > 1 && mc) tc05_commit_mc(bar, (uint16_t)((1u << CL) - 1)); else tc05_commit<CG>(bar);
      };
      auto commit_acc = [&](uint64_t* bar) {
        if (P > 1 && mc) tc05_commit_mc(bar, (uint16_t)(3u << lead_rank)); else tc05_commit<CG>(bar);
      };
      for (int64_t tile = cluster_id; tile < num_tiles; tile += num_clusters) {
        const uint32_t tmem_d = tmem_base + acc * C_::ACC_COLS;
        int64_t kb0 = 0;
        if constexpr (NH == 1) {
          // FP16 accumulate: every use of a buffer (the first included) waits for the epilogue's
          // arrival, which also means "C preloaded"
          mbar_wait(&sm->tmem_empty[acc], KIND == KIND_F16ACC ? acc_phase : acc_phase ^ 1);
          tc05_fence_after();
        } else {
          // single-buffered wide accumulator: the epilogue drains N-half 0 first, so the next tile
          // starts on N-half 0 alone for its first L k-blocks while half 1 is still being read out,
          // then runs half 1's first L k-blocks (the producer loads those slots again, A re-read from
          // L2), then both halves share each slot.  Every accumulator half still receives its
          // k-blocks in ascending order: D is bit-identical to the narrow tile's.
          const int64_t L = look < k_blocks ? look : k_blocks;
#pragma unroll 1
          for (int h = 0; h < 2; ++h) {
            mbar_wait(&sm->tmem_empty[h], acc_phase ^ 1);
            tc05_fence_after();
#pragma unroll 1
            for (int64_t kb = 0; kb < L; ++kb) {
              mbar_wait(&sm->full[stage], phase);
              tc05_fence_after();
              if (elect_one()) {
                issue(stage, h, kb, tmem_d);
                tc05_commit<CG>(&sm->empty[stage]);
                if (h == 1 && kb == k_blocks - 1) tc05_commit<CG>(&sm->tmem_full[acc]);
#if TCX_WATCHDOG
                if (trace && tile < trace_cap && h == 0 && kb == 0) {   // debug timeline: first MMA
                  trace[4 * tile] = ((uint64_t)(cluster_id * P + pair) << 32) | (uint64_t)tile;
                  trace[4 * tile + 1] = globaltimer_ns();
                }
#endif
              }
              __syncwarp();
              if (++stage == C_::STAGES) { stage = 0; phase ^= 1; }
            }
          }
          kb0 = L;
        }
        for (int64_t kb = kb0; kb < k_blocks; ++kb) {
          mbar_wait(&sm->full[stage], phase);
          tc05_fence_after();
          if (elect_one()) {
#pragma unroll
            if constexpr (NH == 2 && KIND != KIND_F16ACC) {
              // both N-halves read the same A: per k-step the half-0 MMA fills the A-operand collector
              // and the half-1 MMA reuses it (A read from smem once per pair of MMAs); each
              // accumulator still sees its k-steps in ascending order, so the result is unchanged
              if (!k_nomma) {
                const uint32_t sa = smem_u32(smem + stage * C_::STAGE_BYTES);
                const uint32_t sb0 = sa + C_::A_BYTES, sb1 = sb0 + C_::HALF_BYTES;
#pragma unroll
                for (int k = 0; k < KBYTES / UMMA_KBYTES; ++k) {
                  const uint64_t ad = sdesc(sa + k * UMMA_KBYTES, 16, 1024, 2);
                  const uint32_t en = (kb | k) ? 1u : 0u;
                  umma_c<CG, KIND, COLL_FILL>(tmem_d, ad, sdesc(sb0 + k * UMMA_KBYTES, 16, 1024, 2), idesc, en);
                  umma_c<CG, KIND, COLL_LASTUSE>(tmem_d + BN, ad, sdesc(sb1 + k * UMMA_KBYTES, 16, 1024, 2), idesc, en);
                }
              }
            } else {
#pragma unroll
              for (int h = 0; h < NH; ++h) issue(stage, h, kb, tmem_d);
            }
            commit_slot(&sm->empty[stage]);                       // frees the smem slot
            if (kb == k_blocks - 1) commit_acc(&sm->tmem_full[acc]);   // accumulator ready
#if TCX_WATCHDOG
            if (trace && tile < trace_cap) {                      // debug tile timeline
              if (kb == kb0 && (NH == 1 || kb0 == 0)) {
                trace[4 * tile] = ((uint64_t)(cluster_id * P + pair) << 32) | (uint64_t)tile;
                trace[4 * tile + 1] = globaltimer_ns();
              }
              if (kb == k_blocks - 1) trace[4 * tile + 2] = globaltimer_ns();
            }
#endif
          }
          __syncwarp();
          if (++stage == C_::STAGES) { stage = 0; phase ^= 1; }
        }
        if (++acc == C_::NBUF) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else if (warp >= 4 && KIND == KIND_F16ACC) {
    // ================= epilogue, FP16 accumulate =================
    // D: tcgen05.ld (FP16 in the low half of each 32-bit column) -> packed f16x2 -> 64B-swizzled
    // 2 KiB staging -> TMA store of the 32 x 32 FP16 box.  Then the drained buffer is refilled with
    // the C of the tile that will use it next (two tiles ahead): TMA load of 32 x 32 FP16 boxes ->
    // unpacked to one value per column -> tcgen05.st; the arrival on tmem_empty means "free + C".
    const int e = warp - 4;
    const int lane = threadIdx.x & 31;
    constexpr int CH = BN / 32;
    uint8_t* stg = smem + C_::SMEM_DATA + e * C_::NBE * 4096;
    uint64_t* cbar = &sm->cbar[e][0];
    uint32_t cph = 0u;                            // bit b: phase of cbar[b] (a register, not a local array)
    const uint32_t tmem_empty_cluster = CG == 2 ? mapa(smem_u32(&sm->tmem_empty[0]), lead_rank) : smem_u32(&sm->tmem_empty[0]);
    const int64_t my_tiles = cluster_id < num_tiles ? (num_tiles - 1 - cluster_id) / num_clusters + 1 : 0;
    const uint32_t lane_off = (uint32_t)(e * 32) << 16;
    // origins of the (at most two) tiles the epilogue addresses at a time — this one and the next —
    // cached, so the raster's 64-bit divisions (~800 cycles) run once per tile, not once per chunk
    int64_t oa_it = -1, ob_it = -1;
    int oa_x = 0, oa_y = 0, ob_x = 0, ob_y = 0;
    auto origin = [&](int64_t it, int& x, int& y) {
      if (it == oa_it) { x = oa_x; y = oa_y; return; }
      if (it == ob_it) { x = ob_x; y = ob_y; return; }
      int64_t mt, nt;
      pair_tile(cluster_id + it * num_clusters, mt, nt);
      x = (int)(nt * C_::TILE_N);
      y = (int)(mt * C_::TILE_M + rank * BM + e * 32);
      if (oa_it < ob_it) { oa_it = it; oa_x = x; oa_y = y; } else { ob_it = it; ob_x = x; ob_y = y; }
    };
    auto coords = [&](int64_t it, int ch, int& x, int& y) {
      origin(it, x, y);
      x += ch * 32;
    };
    auto preload_c = [&](int64_t it, int buf) {
      if (lane == 0) bulk_wait_read<0>();       // staging no longer read by earlier D stores
      __syncwarp();
      auto load = [&](int ch) {
        if (lane == 0) {
          int x, y; coords(it, ch, x, y);
          mbar_arrive_expect_tx(&cbar[ch & 1], 2048);
          tma_load_2d<HINT_C>(stg + (ch & 1) * 2048, &tmC, &cbar[ch & 1], x, y, l2_evict_first());
        }
      };
      load(0);
      load(1);
#pragma unroll 1
      for (int ch = 0; ch < CH; ++ch) {
        const int b = ch & 1;
        mbar_wait(&cbar[b], (cph >> b) & 1u);
        cph ^= 1u << b;
        const uint32_t rowa = smem_u32(stg) + b * 2048 + lane * 64;
        uint32_t r[32];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint4 w = lds128(rowa + ((j ^ ((lane >> 1) & 3)) * 16));   // SW64
          const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
          for (int i = 0; i < 4; ++i) { r[8 * j + 2 * i] = ws[i] & 0xFFFFu; r[8 * j + 2 * i + 1] = ws[i] >> 16; }
        }
        tmem_st_32x32b_x32(tmem_base + buf * C_::ACC_COLS + ch * 32 + lane_off, r);
        __syncwarp();                             // every lane has read buffer b
        if (ch + 2 < CH) load(ch + 2);
      }
      tmem_st_wait();
    };
    for (int t = 0; t < 2; ++t) {                 // buffers 0 and 1 start free (+ C of tiles 0, 1)
      if (has_c && t < my_tiles) preload_c(t, t);
      tc05_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(tmem_empty_cluster + t * 8);
    }
    int acc = 0; uint32_t acc_phase = 0;
    int64_t nstore = 0;
    for (int64_t it = 0; it < my_tiles; ++it) {
      mbar_wait(&sm->tmem_full[acc], acc_phase);
      tc05_fence_after();
#pragma unroll 1
      for (int ch = 0; ch < CH; ++ch, ++nstore) {
        const int b = (int)(nstore & 1);
        uint32_t v[32];
        tmem_ld_32x32b_x32(tmem_base + acc * C_::ACC_COLS + ch * 32 + lane_off, v);
        if (lane == 0 && nstore >= 2) bulk_wait_read<1>();   // store nstore-2 has read buffer b
        __syncwarp();
        tmem_ld_wait();
        const uint32_t rowa = smem_u32(stg) + b * 2048 + lane * 64;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint4 w = make_uint4((v[8 * j] & 0xFFFFu) | (v[8 * j + 1] << 16), (v[8 * j + 2] & 0xFFFFu) | (v[8 * j + 3] << 16),
                                     (v[8 * j + 4] & 0xFFFFu) | (v[8 * j + 5] << 16), (v[8 * j + 6] & 0xFFFFu) | (v[8 * j + 7] << 16));
          sts128(rowa + ((j ^ ((lane >> 1) & 3)) * 16), w);
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          int x, y; coords(it, ch, x, y);
          tma_store_2d<HINT_D>(&tmD, stg + b * 2048, x, y, l2_evict_first());
          bulk_commit();
        }
      }
      if (has_c && it + 2 < my_tiles) { preload_c(it + 2, acc); nstore = 0; }
      tc05_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(tmem_empty_cluster + acc * 8);
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
    if (lane == 0) bulk_wait<0>();
  } else if (warp >= 4) {
    // ================= epilogue =================
    // Per 32-column chunk: tcgen05.ld (thread = row) -> (+ C chunk, TMA-loaded into a 128B-swizzled
    // 4 KiB staging buffer) -> result written back into that buffer -> one TMA store of the 32 x 32
    // box (full-line, coalesced HBM writes; TMA clips rows >= M / columns >= N).  Two buffers per
    // warp alternate, the C chunk two ahead loading while this one is stored.
    const int e = warp - 4;                       // TMEM lanes 32e .. 32e+31
    const int lane = threadIdx.x & 31;
    constexpr int CH = NH * BN / 32;              // 32-column chunks per tile (over both halves)
    uint8_t* stg = smem + C_::SMEM_DATA + e * C_::NBE * 4096;
    uint64_t* cbar = &sm->cbar[e][0];
    uint32_t cph = 0u;                            // bit b: phase of cbar[b] (a register, not a local array)
    const uint32_t tmem_empty_cluster = CG == 2 ? mapa(smem_u32(&sm->tmem_empty[0]), lead_rank) : smem_u32(&sm->tmem_empty[0]);
    const int64_t my_tiles = cluster_id < num_tiles ? (num_tiles - 1 - cluster_id) / num_clusters + 1 : 0;
    const int64_t nq = my_tiles * CH;
    // The CTA's last tile: once its accumulator is full every MMA has finished reading the operand
    // ring and no load will refill it, so the epilogue stages the whole tile there (warp e: CH
    // chunks of 4 KiB) — all C chunks are loaded at once and no chunk waits for an earlier store to
    // free its buffer.  The exposed tail of every launch (and all of a one-tile problem) shrinks.
    // (multicast groups too: the pairs of a group run the same cluster tiles, so by the time this
    // pair's last accumulator is full no peer has a load left to land in this CTA's ring)
#ifndef TCX_RING_LAST_MC
#define TCX_RING_LAST_MC 1
#endif
    constexpr bool RING_LAST = NH == 1 && (P == 1 || TCX_RING_LAST_MC) && EPI_WARPS * CH * 4096 <= C_::SMEM_DATA;
    const int64_t q_last0 = (my_tiles - 1) * CH;             // first chunk of the last tile
    // origins of the (at most two) tiles the epilogue addresses at a time — this one and the next —
    // cached, so the raster's 64-bit divisions (~800 cycles) run once per tile, not once per chunk
    int64_t oa_it = -1, ob_it = -1;
    int oa_x = 0, oa_y = 0, ob_x = 0, ob_y = 0;
    auto origin = [&](int64_t it, int& x, int& y) {
      if (it == oa_it) { x = oa_x; y = oa_y; return; }
      if (it == ob_it) { x = ob_x; y = ob_y; return; }
      int64_t mt, nt;
      pair_tile(cluster_id + it * num_clusters, mt, nt);
      x = (int)(nt * C_::TILE_N);
      y = (int)(mt * C_::TILE_M + rank * BM + e * 32);
      if (oa_it < ob_it) { oa_it = it; oa_x = x; oa_y = y; } else { ob_it = it; ob_x = x; ob_y = y; }
    };
    auto coords = [&](int64_t q, int& x, int& y) {
      origin(q / CH, x, y);
      x += (int)(q % CH) * 32;
    };
    auto load_c = [&](int64_t q) {
      if (has_c && lane == 0 && q < nq && !(RING_LAST && q >= q_last0)) {
        int x, y; coords(q, x, y);
        const int bq = (int)(q % C_::NBE);
        mbar_arrive_expect_tx(&cbar[bq], 4096);
        tma_load_2d<HINT_C>(stg + bq * 4096, &tmC, &cbar[bq], x, y, l2_evict_first());
      }
    };
    // single-buffered (wide) tiles: the epilogue is on the critical path, so each tile's C is
    // L2-prefetched a tile ahead and its chunk loads hit L2 (double-buffered tiles hide the latency
    // — except the first tile's, prefetched while the mainloop starts: small problems are one tile)
    auto prefetch_c_tile = [&](int64_t it) {
      if ((NH == 2 || it == 0) && has_c && lane == 0 && it < my_tiles)
        for (int ch = 0; ch < CH; ++ch) { int x, y; coords(it * CH + ch, x, y); tma_prefetch_2d<HINT_C>(&tmC, x, y, l2_evict_first()); }
    };
    prefetch_c_tile(0);
    for (int c = 0; c < C_::C_AHEAD; ++c) load_c(c);
    int acc = 0; uint32_t acc_phase = 0;
    const uint32_t lane_off = (uint32_t)(e * 32) << 16;
#if TCX_WATCHDOG
    // debug chunk-phase stamps (clock64): cluster 0, CTA rank 0, lane 0 of each epilogue warp e,
    // first CHUNK_TILES tiles, 8 per chunk, after the tile timeline (trace_cap >= num_tiles + ...)
    constexpr int CHUNK_TILES = 6;
    uint64_t* const cst = (trace && cluster_id == 0 && rank == 0 && lane == 0 &&
                           trace_cap >= num_tiles + 8 * CHUNK_TILES * CH)
                              ? trace + 4 * num_tiles + e * CHUNK_TILES * CH * 8 : nullptr;
#define TCX_STAMP(it_, ch_, k_) do { if (cst && (it_) < CHUNK_TILES) cst[((it_) * CH + (ch_)) * 8 + (k_)] = clock64(); } while (0)
#else
#define TCX_STAMP(it_, ch_, k_) do { } while (0)
#endif
    for (int64_t it = 0; it < my_tiles; ++it) {
      prefetch_c_tile(it + 1);
      TCX_STAMP(it, 0, 7);
      mbar_wait(&sm->tmem_full[acc], acc_phase);
      TCX_STAMP(it, 1, 7);
      tc05_fence_after();
      const bool ring = RING_LAST && it == my_tiles - 1;
      uint8_t* const ring_stg = smem + e * CH * 4096;
      if (ring && has_c) {                        // every C chunk of the tile, into the idle ring
        if (lane == 0) {
          mbar_arrive_expect_tx(&sm->cring[e], CH * 4096);
          for (int ch = 0; ch < CH; ++ch) {
            int x, y; coords(it * CH + ch, x, y);
            tma_load_2d<HINT_C>(ring_stg + ch * 4096, &tmC, &sm->cring[e], x, y, l2_evict_first());
          }
        }
        __syncwarp();
      }
      uint32_t v[32], vn[32];
      tmem_ld_32x32b_x32(tmem_base + acc * C_::ACC_COLS + lane_off, vn);   // chunk 0
      if (ring && has_c) mbar_wait(&sm->cring[e], 0);
#pragma unroll 1
      for (int ch = 0; ch < CH; ++ch) {
        const int64_t q = it * CH + ch;
        const int b = (int)(q % C_::NBE);
        const int h = ch / (BN / 32);
        TCX_STAMP(it, ch, 0);
        tmem_ld_wait();                           // chunk ch has landed in vn
        TCX_STAMP(it, ch, 1);
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = vn[j];
        if (ch + 1 < CH) {                        // read the next chunk while this one is stored
          const int hn = (ch + 1) / (BN / 32);
          tmem_ld_32x32b_x32(tmem_base + acc * C_::ACC_COLS + hn * BN + ((ch + 1) % (BN / 32)) * 32 + lane_off, vn);
        }
        if (ring) {
          // own buffer per chunk in the ring; C (if any) already landed
        } else if (has_c) {
          mbar_wait(&cbar[b], (cph >> b) & 1u);
          cph ^= 1u << b;
        } else if (q >= C_::NBE) {
          if (lane == 0) bulk_wait_read<C_::NBE - 1>();   // the store of chunk q-NBE has read buffer b
          __syncwarp();
        }
        TCX_STAMP(it, ch, 2);
        if (ch % (BN / 32) == BN / 32 - 1 && (NH == 2 || ch == CH - 1)) {
          // this part of the accumulator is read: hand it back to the MMA warp
          // (NH = 1: the whole buffer `acc`; NH = 2: N-half h of the single buffer)
          tc05_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_cluster(tmem_empty_cluster + (NH == 2 ? h : acc) * 8);
        }
        uint8_t* const buf = ring ? ring_stg + ch * 4096 : stg + b * 4096;
        const uint32_t rowa = smem_u32(buf) + lane * 128;      // this thread's row of the box
        uint4 cv[8];                                           // all C loads first: 8 in flight
        if (has_c) {
#pragma unroll
          for (int j = 0; j < 8; ++j) cv[j] = lds128(rowa + ((j ^ (lane & 7)) * 16));
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const uint32_t pa = rowa + ((j ^ (lane & 7)) * 16);  // SW128: chunk j at j ^ (row % 8)
          uint4 o = make_uint4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
          if (has_c) {
            const uint4 c = cv[j];
            if constexpr (KIND == KIND_I8) {                   // S32: wrap mod 2^32
              o.x += c.x; o.y += c.y; o.z += c.z; o.w += c.w;
            } else {                                          // FP32: one RNE add
              o.x = __float_as_uint(__fadd_rn(__uint_as_float(o.x), __uint_as_float(c.x)));
              o.y = __float_as_uint(__fadd_rn(__uint_as_float(o.y), __uint_as_float(c.y)));
              o.z = __float_as_uint(__fadd_rn(__uint_as_float(o.z), __uint_as_float(c.z)));
              o.w = __float_as_uint(__fadd_rn(__uint_as_float(o.w), __uint_as_float(c.w)));
            }
          }
          sts128(pa, o);
        }
        TCX_STAMP(it, ch, 3);
        if (ring) continue;                       // the last tile's stores leave together, below
        fence_proxy_async_smem();
        __syncwarp();
        TCX_STAMP(it, ch, 4);
        if (lane == 0 && !k_noepi) {
          int x, y; coords(q, x, y);
          tma_store_2d<HINT_D>(&tmD, buf, x, y, l2_evict_first());
          bulk_commit();
          TCX_STAMP(it, ch, 5);
          // the buffer of chunk q + C_AHEAD was last read by the store of chunk q + C_AHEAD - NBE
          if (!ring && has_c && q + C_::C_AHEAD < nq && !(RING_LAST && q + C_::C_AHEAD >= q_last0))
            bulk_wait_read<C_::NBE - C_::C_AHEAD>();
        }
        TCX_STAMP(it, ch, 6);
        load_c(q + C_::C_AHEAD);
      }
      if (ring) {
        // every chunk of the last tile has its own ring buffer: one proxy fence, then the CH TMA
        // stores back to back (no per-chunk fence / store-issue round trip on the exposed tail)
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0 && !k_noepi) {
          for (int ch = 0; ch < CH; ++ch) {
            int x, y; coords(it * CH + ch, x, y);
            tma_store_2d<HINT_D>(&tmD, ring_stg + ch * 4096, x, y, l2_evict_first());
          }
          bulk_commit();
        }
      }
#if TCX_WATCHDOG
      if (trace && e == 0 && lane == 0 && rank == 0) {
        const int64_t tile = cluster_id + it * num_clusters;
        if (tile < trace_cap) trace[4 * tile + 3] = globaltimer_ns();
      }
#endif
      if (++acc == C_::NBUF) { acc = 0; acc_phase ^= 1; }
    }
    if (lane == 0) bulk_wait<0>();                            // stores complete before exit
#undef TCX_STAMP
  }

  tc05_fence_before();
  if constexpr (CG > 1) cluster_sync(); else __syncthreads();
  if (warp == 2) { tc05_fence_after(); tmem_dealloc<CG>(tmem_base, 512); }
}

template <typename T>
__global__ void fill_c_kernel(const T* C, int64_t ldc, T* D, int64_t ldd, int64_t M, int64_t N) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t total = M * N;
  for (; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = i / N, c = i % N;
    D[r * ldd + c] = C ? C[r * ldc + c] : (T)0;
  }
}

// wide tile: k-blocks of N-half 0 the next tile runs ahead while half 1 drains.  A/B on C3
// (gpurun_out r02 wide-lookahead study): L = 0 / 4 / 8 / 16 / 32 -> 1474 / 1470 / 1473 /
// 1469 / 1427 TFLOP/s; the inter-tile MMA gap falls 15.4 -> 8.2 us at L = 16 but the half-only
// k-blocks run slower (tile 91.8 -> 97.6 us), so the wide tile stays an option, not the default
#ifndef TCX_WIDE_LOOK
#define TCX_WIDE_LOOK 8
#endif
static int wide_look() { return TCX_WIDE_LOOK; }

template <int CG, int KIND, int NH, int PM = 1, int PN = 1, int BNT = BN_FULL>
tcx_status launch_t(const GemmArgs& a, const DevInfo& dev, cudaStream_t s, CUtensorMapDataType dt, int a_fmt) {
  using C_ = Cfg<CG, NH, BNT>;
  constexpr int ES = KindT<KIND>::ESIZE;
  constexpr int CL = CG * PM * PN;
  CUtensorMap tA, tB;
  tcx_status st = make_tmap_2d(&tA, dt, a.A, (uint64_t)a.K, (uint64_t)a.M, (uint64_t)(a.lda * ES),
                               KBYTES / ES, BM / PN, CU_TENSOR_MAP_SWIZZLE_128B);
  if (st != TCX_OK) return st;
  st = make_tmap_2d(&tB, dt, a.B, (uint64_t)a.K, (uint64_t)a.N, (uint64_t)(a.ldb * ES),
                    KBYTES / ES, C_::BN_LOAD / PM, CU_TENSOR_MAP_SWIZZLE_128B);
  if (st != TCX_OK) return st;
  // C and D: 32 x 32 boxes of 4-byte elements (128-byte rows) through 128B-swizzled staging
  // (FP16 accumulate: 32 x 32 boxes of FP16, 64-byte rows, 64B-swizzled)
  constexpr bool H = KIND == KIND_F16ACC;
  const CUtensorMapDataType cdt = H ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
  const CUtensorMapSwizzle csw = H ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B;
  const int ces = H ? 2 : 4;
  CUtensorMap tC, tD;
  st = make_tmap_2d(&tD, cdt, a.D, (uint64_t)a.N, (uint64_t)a.M, (uint64_t)(a.ldd * ces), 32, 32, csw);
  if (st != TCX_OK) return st;
  if (a.C) {
    st = make_tmap_2d(&tC, cdt, a.C, (uint64_t)a.N, (uint64_t)a.M, (uint64_t)(a.ldc * ces), 32, 32, csw);
    if (st != TCX_OK) return st;
  } else {
    tC = tD;                                                  // unused (has_c = 0)
  }
  auto kern = gemm_dense_kernel<CG, KIND, NH, PM, PN, BNT>;
  TCX_CUDA_TRY(ensure_max_smem((const void*)kern, C_::SMEM_TOTAL, dev.device));
  const int64_t m_tiles = (a.M + C_::TILE_M - 1) / C_::TILE_M;
  const int64_t n_tiles = (a.N + C_::TILE_N - 1) / C_::TILE_N;
  int64_t clusters = ((m_tiles + PM - 1) / PM) * ((n_tiles + PN - 1) / PN);
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(NUM_THREADS);
  cfg.dynamicSmemBytes = C_::SMEM_TOTAL;
  cfg.stream = s;
  cudaLaunchAttribute attr[3];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = CG; attr[1].val.clusterDim.y = 1; attr[1].val.clusterDim.z = 1;
  attr[2].id = cudaLaunchAttributePreferredClusterDimension;       // CL-CTA groups where a GPC has room
  attr[2].val.preferredClusterDim.x = CL; attr[2].val.preferredClusterDim.y = 1; attr[2].val.preferredClusterDim.z = 1;
  cfg.attrs = attr; cfg.numAttrs = CL > CG ? 3 : 2;
  int64_t max_clusters = dev.sm_count / CL;                        // CTA groups (persistent)
  if (a.max_ctas > 0 && a.max_ctas / CL < max_clusters) max_clusters = a.max_ctas / CL > 0 ? a.max_ctas / CL : 1;
  if (clusters > max_clusters) clusters = max_clusters;
  cfg.gridDim = dim3((unsigned)(clusters * CL));
#if TCX_WATCHDOG
  if (getenv("TCX_DEBUG_LAUNCH"))   // debug library: print the launch shape
    fprintf(stderr, "tcx_gemm: grid %u CTAs, cluster %d (pairs %dx%d), tile %dx%d, %lld cluster tiles\n", cfg.gridDim.x, CL,
            PM, PN, C_::TILE_M, C_::TILE_N, (long long)(((m_tiles + PM - 1) / PM) * ((n_tiles + PN - 1) / PN)));
#endif
  const uint32_t idesc = make_idesc(KIND, a_fmt, BM * CG, C_::BN);
  TCX_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, tA, tB, tC, tD, (int64_t)a.M, (int64_t)a.N, (int64_t)a.K,
                                  a.C ? 1 : 0, idesc, a.group_m != 0 ? a.group_m : GROUP_M, wide_look(), a.fault, a.trace,
                                  a.trace_cap));
  count_launch();
  return TCX_OK;
}

}  // namespace

tcx_status launch_fill_c(const GemmArgs& a, cudaStream_t s) {
  int64_t total = a.M * a.N;
  int blocks = (int)((total + 255) / 256 < 4096 ? (total + 255) / 256 : 4096);
  if (blocks < 1) blocks = 1;
  if (a.cd == TCX_F16)
    fill_c_kernel<uint16_t><<<blocks, 256, 0, s>>>((const uint16_t*)a.C, a.ldc, (uint16_t*)a.D, a.ldd, a.M, a.N);
  else
    fill_c_kernel<uint32_t><<<blocks, 256, 0, s>>>((const uint32_t*)a.C, a.ldc, (uint32_t*)a.D, a.ldd, a.M, a.N);
  TCX_CUDA_TRY(cudaGetLastError());
  count_launch();
  return TCX_OK;
}

// Library choice of the multicast group (the caller left pairs at 0): 1 x 2 — two CTA pairs of a row
// share A by TMA multicast — once the problem has at least two waves of pair tiles and two tile
// columns.  At the power cap it cuts L2 reads ~15% and measured +0.8-1.0% on C3 (BF16 and TF32)
// and C4 in the bench's burst conditions, equal sustained; smaller problems keep
// plain pairs (fewer, coupled groups would cost more than they save).
static bool auto_pairs_1x2(const GemmArgs& a, const DevInfo& dev) {
  if (!a.pairs_auto || a.cta_group != 2 || a.tile_n == 512) return false;
  const int64_t m_tiles = (a.M + 255) / 256, n_tiles = (a.N + 255) / 256;
  return n_tiles >= 2 && m_tiles * n_tiles >= 2 * (int64_t)(dev.sm_count / 2);
}

// Wave quantisation (CTA pair, library choice of the tile width): P pairs run a call of T tiles in
// ceil(T / P) waves, each one tile-time long, and a tile's time is proportional to its width (its
// K loop is the same).  So the call costs ~ ceil(T(w) / P) * w for UMMA N = w: when T(256) fills
// its last wave poorly (a row-sharded rank's small M, e.g. C3 / 8 ranks = 1024 rows: 128 tiles on
// 74 pairs, 2 waves 86% full), a narrower tile that fills it (224: 148 tiles, exactly 2 waves)
// finishes sooner (measured +4.1% on 1024 x 8192 x 8192 and +4.4% on 2048 x 8192 x 8192 BF16,
// unchanged on the full configs).  A narrower width is taken only when it is >= 5% cheaper by this
// count.  Returns the width (256 = the default tile).
static int wave_tile_width(const GemmArgs& a, const DevInfo& dev) {
  if (a.tile_n != 0) return a.tile_n == 512 ? 256 : a.tile_n;   // caller's choice
  if (a.cta_group != 2 || !a.pairs_auto) return 256;
  int64_t pairs = dev.sm_count / 2;
  if (a.max_ctas > 0 && a.max_ctas / 2 < pairs) pairs = a.max_ctas / 2 > 0 ? a.max_ctas / 2 : 1;
  const int64_t mt = (a.M + 255) / 256;
  // a narrower tile also runs fewer FLOP/s: per-width throughput relative to 256 on full waves
  // (C3 BF16 8192^3, tools/wave_study.py: 224 0.979, 192 0.944, 160 0.879, 128 0.806), so a tile
  // costs width / rate
  auto cost = [&](int w, int rate_permille) {
    const int64_t t = mt * ((a.N + w - 1) / w);
    return (t + pairs - 1) / pairs * w * 1000 / rate_permille;
  };
  const int64_t c256 = cost(256, 1000);
  int best = 256; int64_t bc = c256;
  const int widths[4] = {224, 192, 160, 128}, rates[4] = {979, 944, 879, 806};
  for (int i = 0; i < 4; ++i) {
    const int64_t c = cost(widths[i], rates[i]);
    if (c < bc && 20 * c <= 19 * c256) { best = widths[i]; bc = c; }
  }
  return best;
}

template <int KIND>
tcx_status launch_narrow(int w, const GemmArgs& a, const DevInfo& dev, cudaStream_t s, CUtensorMapDataType dt, int a_fmt) {
  switch (w) {
    case 224: return launch_t<2, KIND, 1, 1, 1, 224>(a, dev, s, dt, a_fmt);
    case 192: return launch_t<2, KIND, 1, 1, 1, 192>(a, dev, s, dt, a_fmt);
    case 160: return launch_t<2, KIND, 1, 1, 1, 160>(a, dev, s, dt, a_fmt);
    default: return launch_t<2, KIND, 1, 1, 1, 128>(a, dev, s, dt, a_fmt);
  }
}

// Long K loops (library choice): the 256 x 512 pair tile moves 25% fewer operand bytes per FLOP but
// its single accumulator exposes a drain of fixed length per tile, so it wins once a tile's K loop
// is long enough for the drain to be a small share — K >= 16384 BF16/FP16 MMA-equivalents (TF32
// runs at half the rate: K >= 8192; INT8 at twice: K >= 32768) — and when its tiles fill the waves
// within 3% of the 256-wide tiles' fill.  Burst A/B (profiles/r02_studies/dense_wide_long_k/):
// BF16 16384^3 +4.3%, 8192 x 8192 x 32768 +4.0%, 8192 x 8192 x 16384 +1.1%; TF32 16384^3 +8.0%,
// 8192^3 +0.5%; INT8 16384 x 16384 x 32768 +6.8%; at K_eff = 8192 (C3 BF16, C4) the default wins.
template <int KIND>
static bool auto_wide(const GemmArgs& a, const DevInfo& dev) {
  if (a.tile_n != 0 || !a.pairs_auto || a.cta_group != 2 || KIND == KIND_F16ACC) return false;
  const int64_t k_eff = KIND == KIND_TF32 ? 2 * a.K : KIND == KIND_I8 ? a.K / 2 : a.K;
  if (k_eff < 16384) return false;
  int64_t pairs = dev.sm_count / 2;
  if (a.max_ctas > 0 && a.max_ctas / 2 < pairs) pairs = a.max_ctas / 2 > 0 ? a.max_ctas / 2 : 1;
  const int64_t mt = (a.M + 255) / 256;
  auto fill = [&](int64_t t) { return (double)t / (double)(((t + pairs - 1) / pairs) * pairs); };
  return fill(mt * ((a.N + 511) / 512)) >= 0.97 * fill(mt * ((a.N + 255) / 256));
}

template <int KIND>
tcx_status launch_kind(const GemmArgs& a, const DevInfo& dev, cudaStream_t s, CUtensorMapDataType dt, int a_fmt) {
  if (a.cta_group == 1) return launch_t<1, KIND, 1>(a, dev, s, dt, a_fmt);
  const int w = wave_tile_width(a, dev);
  if (w != 256) return launch_narrow<KIND>(w, a, dev, s, dt, a_fmt);
  if (auto_wide<KIND>(a, dev)) return launch_t<2, KIND, 2>(a, dev, s, dt, a_fmt);
  if (auto_pairs_1x2(a, dev)) return launch_t<2, KIND, 1, 1, 2>(a, dev, s, dt, a_fmt);
  // 256 x 512 pair tiles only when asked: they cut L2->SM operand traffic by 25% (and run at a
  // higher clock under the power cap), but the single-buffered accumulator exposes the epilogue,
  // whose FP32 C read + D write bursts from all CTAs at once (profiles/r01_dense_tile_study.txt);
  // the double-buffered 256 x 256 tile is faster for this API's FP32 C/D.
  if (a.tile_n == 512) return launch_t<2, KIND, 2>(a, dev, s, dt, a_fmt);
  if (a.pairs_m == 2 && a.pairs_n == 2) return launch_t<2, KIND, 1, 2, 2>(a, dev, s, dt, a_fmt);
  if (a.pairs_m == 2) return launch_t<2, KIND, 1, 2, 1>(a, dev, s, dt, a_fmt);
  if (a.pairs_n == 2) return launch_t<2, KIND, 1, 1, 2>(a, dev, s, dt, a_fmt);
  return launch_t<2, KIND, 1>(a, dev, s, dt, a_fmt);
}

tcx_status launch_gemm_dense(const GemmArgs& a, const DevInfo& dev, cudaStream_t s) {
  if (a.cd == TCX_F16) {   // FP16 accumulate (F16 inputs only; validated by the front end)
    constexpr CUtensorMapDataType h = CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
    if (a.cta_group == 1) return launch_t<1, KIND_F16ACC, 1>(a, dev, s, h, 0);
    const int w = wave_tile_width(a, dev);
    if (w != 256) return launch_narrow<KIND_F16ACC>(w, a, dev, s, h, 0);
    if (auto_pairs_1x2(a, dev)) return launch_t<2, KIND_F16ACC, 1, 1, 2>(a, dev, s, h, 0);
    if (a.pairs_m == 2 && a.pairs_n == 2) return launch_t<2, KIND_F16ACC, 1, 2, 2>(a, dev, s, h, 0);
    if (a.pairs_m == 2) return launch_t<2, KIND_F16ACC, 1, 2, 1>(a, dev, s, h, 0);
    if (a.pairs_n == 2) return launch_t<2, KIND_F16ACC, 1, 1, 2>(a, dev, s, h, 0);
    return launch_t<2, KIND_F16ACC, 1>(a, dev, s, h, 0);
  }
  switch (a.ab) {
    case TCX_F16: return launch_kind<KIND_F16>(a, dev, s, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 0);
    case TCX_BF16: return launch_kind<KIND_F16>(a, dev, s, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 1);
    case TCX_TF32: return launch_kind<KIND_TF32>(a, dev, s, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2);
    case TCX_S8: return launch_kind<KIND_I8>(a, dev, s, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1);
    default:
      return set_error(TCX_ERR_UNSUPPORTED, "tcx_gemm: unsupported ab type %d", (int)a.ab);
  }
}

}  // namespace tcx
