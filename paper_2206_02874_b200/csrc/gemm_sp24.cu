// tcx 2:4 structured-sparse GEMM on sm_100a (the paper's mma.sp, at GEMM scale):
//     D = expand(sA, e) x B + C
// sA: M x K/2 kept values (K-major), e: hardware metadata image (sp24.cu), B: N x K, C/D: M x N FP32.
//
// Same warp-specialised persistent structure as gemm_dense.cu; per 128-logical-K stage each CTA
// TMA-loads 128 rows of sA (128 B/row, SW128), its half of the B tile (two SW128 64-element
// boxes) and one 2 KiB metadata atom; the MMA thread copies the atom smem -> TMEM with
// tcgen05.cp 128x128b, then issues 4 x tcgen05.mma.sp.kind::f16 (logical K = 32 each).
// TMEM: two 240-column FP32 accumulators (cols 0 and 256) + a 4-slot metadata ring (cols 496..511),
// so the epilogue of tile t overlaps the MMAs of tile t+1 (UMMA N = 240: 2 x 240 + 16 <= 512).
// KIND_I8 (2:4 on bytes, S32 accumulate, wrap): a stage is 256 logical K (sA 128 B/row, B two
// 128-byte boxes, metadata two 2 KiB atoms copied by two 128x128b tcgen05.cp into 8 columns), and
// each of the 4 tcgen05.mma.sp.kind::i8 (logical K = 64) reads 2 metadata columns; the ring is
// 4 x 8 columns at 480..511 and the accumulators sit at 0 and 240.
// KIND_TF32 (hardware 1:2 sparsity, logical K = 16 per MMA): a stage is 64 logical K (32 kept TF32 =
// 128 B of sA per row), B two 32-element boxes, one metadata atom; layout as kind::f16 over 2K.
// "The hardware selector determines which values should participate ... on the fly":
// the MMA skips the zero products; throughput doubles at the same latency.
#include <cstdlib>
#include "tcx_internal.h"
#include "ptx.cuh"

namespace tcx {
namespace {

constexpr int BM = 128;
constexpr int BN = 240;            // UMMA N
constexpr int NUM_THREADS = 256;
constexpr int EPI_WARPS = 4;
constexpr int GROUP_M = 8;            // default raster group (cluster-tile rows sweeping N together)
// epilogue staging buffers per warp: the C chunk two ahead goes into the buffer the store before
// last read, so issuing it waits only for that older store, not for the one just issued
constexpr int STG_BUFS = 3;
constexpr int C_AHEAD = 2;
// MW = 1 ("M-wide", CTA pair tile 512 x 240): two M-halves share each stage's B (30 of the 48 KiB a
// stage moves), so a stage carries 66 KiB for twice the work — 31% fewer operand bytes per FLOP
// into each SM, whose TMA ingress the 2:4 stream otherwise saturates.  Both halves'
// accumulators fill TMEM (2 x 240 columns + the metadata ring), so the accumulator is
// single-buffered: per-half empty barriers and a half-0 lookahead as in gemm_dense.cu's wide tile.
// PM x PN > 1 (CTA pair, MW = 0): groups of PM x PN pairs launched as preferred clusters, as in
// gemm_dense.cu.  In a formed cluster the pairs of a column share B — each loads one of the stage's
// two 64-element K boxes of B and multicasts it — and the pairs of a row share sA (a 1/PN row
// slice each); metadata atoms are per pair.  A group the hardware did not place as one cluster
// runs as independent pairs on the same tiles.
template <int CG, int KIND, int MW = 0>
struct SpCfg {
  static constexpr int MH = MW ? 2 : 1;                    // M-halves per tile (accumulators)
  static constexpr int ES = KIND == KIND_I8 ? 1 : KIND == KIND_TF32 ? 4 : 2;   // element bytes
  static constexpr int KL = 256 / ES;                      // logical K per stage (= 128 B of kept A)
  static constexpr int BOX = 128 / ES;                     // elements per 128-byte SW128 box row
  // 2 KiB metadata atoms per stage and M-half (one atom = 128 rows x 128 logical 8/16-bit K; a TF32
  // element counts as two 16-bit halves, so a 64-logical-K TF32 stage is one atom)
  static constexpr int META_ATOMS = KIND == KIND_TF32 ? 1 : KL / 128;
  static constexpr int META_BYTES = 2048 * META_ATOMS * MH;
  static constexpr int META_COLS = 4 * META_ATOMS * MH;    // TMEM columns per stage
  static constexpr int BN_LOAD = BN / CG;
  static constexpr int A_HALF = BM * 128;                  // 128 bytes of kept values per row
  static constexpr int A_BYTES = A_HALF * MH;
  static constexpr int B_HALF = BN_LOAD * 128;             // one SW128 box (128 bytes of K per row)
  static constexpr int B_BYTES = 2 * B_HALF;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES + META_BYTES;
  static constexpr int STAGES = CG == 1 ? 2 : (MW ? 3 : 4);
  static constexpr int TILE_M = BM * CG * MH;
  static constexpr int SMEM_DATA = STAGES * STAGE_BYTES;
  static constexpr int STG_BYTES = EPI_WARPS * STG_BUFS * 2048;   // epilogue: 3 x 2 KiB (32 rows x 16 cols) per warp
  static constexpr int SMEM_TOTAL = SMEM_DATA + STG_BYTES + 1024 + 1024;
  static constexpr int META_COL = 512 - STAGES * META_COLS;    // metadata ring at the top of TMEM
  // accumulator columns: MW -> M-half h at h * BN (one buffer); else buffer b at b * ACC_STRIDE
  static constexpr int ACC_STRIDE = MW ? BN : (KIND == KIND_I8 ? BN : 256);
  static_assert(B_HALF % 1024 == 0, "SW128 atoms need 1 KiB alignment");
  static_assert(ACC_STRIDE + BN <= META_COL, "TMEM budget");
  static_assert(!MW || (CG == 2 && KIND != KIND_I8), "M-wide sparse tiles: CTA pair, f16/bf16/tf32");
  static_assert(SMEM_TOTAL <= 232448, "smem budget");
};

struct Smem {
  uint64_t full[8];
  uint64_t empty[8];
  uint64_t tmem_full[2];
  uint64_t tmem_empty[2];
  uint64_t cbar[EPI_WARPS][STG_BUFS]; // epilogue: C chunk landed in staging buffer b of warp e
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

template <int CG, int KIND, int MW, int PM, int PN>
__global__ void __launch_bounds__(NUM_THREADS, 1)
gemm_sp24_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                 const __grid_constant__ CUtensorMap tmE, const __grid_constant__ CUtensorMap tmC,
                 const __grid_constant__ CUtensorMap tmD, int64_t M, int64_t N, int64_t K, int has_c, uint32_t idesc,
                 int group_m, uint64_t* trace, int64_t trace_cap, int knobs) {
  // knobs (debug library only, 0 in the product): energy decomposition of the pipeline —
  // 2 = no MMAs (the MMA warp still waits and commits), 4 = no operand TMA loads (the producer only
  // arrives), 8 = no epilogue global traffic (TMEM is still drained; C not loaded, D not stored)
#if !TCX_WATCHDOG
  knobs = 0;
#endif
  const bool k_nomma = knobs & 2, k_noload = knobs & 4, k_noepi = knobs & 8;
  if (k_noepi) has_c = 0;
  using C_ = SpCfg<CG, KIND, MW>;
  constexpr int KL = C_::KL;
  constexpr int MH = C_::MH;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  Smem* sm = (Smem*)(smem + C_::SMEM_DATA + C_::STG_BYTES);

  constexpr int P = PM * PN;                 // CTA pairs per group
  constexpr int CL = CG * P;                 // CTAs per group
  static_assert(P == 1 || CG == 2, "multicast groups: CTA pairs");
  static_assert(PM <= 2, "B is shared as its two K boxes");
  const int warp = threadIdx.x / 32;
  const uint32_t crank = CG > 1 ? cluster_ctarank() : 0;
  const bool mc = P > 1 && cluster_nctarank() == (uint32_t)CL;    // this group formed one cluster
  const uint32_t rank = crank % CG;
  const uint32_t pair = (blockIdx.x % CL) / CG;
  const int pm = (int)(pair % PM), pn = (int)(pair / PM);
  const uint32_t lead_rank = mc ? pair * CG : 0;
  const bool leader = rank == 0;
  if (P > 1 && crank != (mc ? blockIdx.x % CL : blockIdx.x % CG)) __trap();
  const int64_t m_tiles = M / C_::TILE_M;
  const int64_t n_tiles = (N + BN - 1) / BN;
  const int64_t sm_tiles = (m_tiles + PM - 1) / PM;
  const int64_t sn_tiles = (n_tiles + PN - 1) / PN;
  const int64_t num_tiles = sm_tiles * sn_tiles;
  const int64_t k_blocks = K / KL;
  const int64_t cluster_id = blockIdx.x / CL;
  const int64_t num_clusters = gridDim.x / CL;
  auto pair_tile = [&](int64_t tile, int64_t& mt, int64_t& nt) {
    int64_t smt, snt;
    tile_coords(tile, sm_tiles, sn_tiles, group_m, smt, snt);
    mt = smt * PM + pm;
    nt = snt * PN + pn;
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < C_::STAGES; ++s) { mbar_init(&sm->full[s], 1); mbar_init(&sm->empty[s], mc ? P : 1); }
    for (int a = 0; a < 2; ++a) { mbar_init(&sm->tmem_full[a], 1); mbar_init(&sm->tmem_empty[a], EPI_WARPS * CG); }
    for (int w = 0; w < EPI_WARPS; ++w)
      for (int b = 0; b < STG_BUFS; ++b) mbar_init(&sm->cbar[w][b], 1);
    fence_mbar_init();
  }
  if (warp == 0 && elect_one()) { tma_prefetch(&tmA); tma_prefetch(&tmB); tma_prefetch(&tmE); tma_prefetch(&tmC); tma_prefetch(&tmD); }
  if (warp == 2) { tmem_alloc<CG>(&sm->tmem_base, 512); tmem_relinquish<CG>(); }
  tc05_fence_before();
  if constexpr (CG == 2) cluster_sync(); else __syncthreads();
  tc05_fence_after();
  const uint32_t tmem_base = sm->tmem_base;
  // PDL: the setup above (barriers, TMEM allocation, descriptor prefetch) overlapped the previous
  // grid's tail; no global memory is touched before its completion
  pdl_wait();
  pdl_trigger();
#if TCX_WATCHDOG
  if (k_noload && KIND != KIND_I8) {
    dbg_fill_ring(smem, C_::SMEM_DATA, C_::A_BYTES + C_::B_BYTES, C_::META_BYTES, C_::STAGE_BYTES, false);
    fence_proxy_async_smem();
    __syncthreads();
  }
#endif

  if (warp == 0) {
    if (elect_one()) {
      int stage = 0; uint32_t phase = 0;
      const uint32_t full0_cluster = CG == 2 ? mapa(smem_u32(&sm->full[0]), lead_rank) : 0;
      constexpr int A_ROWS = BM / PN;
      uint16_t mask_a = 0, mask_b = 0;
      for (int j = 0; j < PN; ++j) mask_a |= (uint16_t)(1u << ((pm + PM * j) * CG + rank));
      for (int i = 0; i < PM; ++i) mask_b |= (uint16_t)(1u << ((i + PM * pn) * CG + rank));
      for (int64_t tile = cluster_id; tile < num_tiles; tile += num_clusters) {
        int64_t mt, nt;
        pair_tile(tile, mt, nt);
        const int64_t mrow = mt * C_::TILE_M + rank * BM;            // + h * BM * CG for M-half h
        const int brow = (int)(nt * BN + rank * C_::BN_LOAD);
        for (int64_t kb = 0; kb < k_blocks; ++kb) {
          mbar_wait(&sm->empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * C_::STAGE_BYTES;
          uint8_t* sb = sa + C_::A_BYTES;
          uint8_t* se = sb + C_::B_BYTES;
          const int ka = (int)(kb * (KL / 2));     // kept-value column
          const int kx = (int)(kb * KL);           // logical column of B
          if (k_noload) {                       // debug: the slot is "filled" without moving a byte
            if (CG == 1 || leader) mbar_arrive_expect_tx(&sm->full[stage], 0);
            if (++stage == C_::STAGES) { stage = 0; phase ^= 1; }
            continue;
          }
          if constexpr (CG == 1) {
            mbar_arrive_expect_tx(&sm->full[stage], C_::STAGE_BYTES);
          } else {
            if (leader) mbar_arrive_expect_tx(&sm->full[stage], 2 * C_::STAGE_BYTES);
          }
          const uint32_t bar = CG == 2 ? full0_cluster + stage * 8 : smem_u32(&sm->full[stage]);
          auto load = [&](void* dst, const CUtensorMap* m, int x, int y) {
            const uint64_t pol = m == &tmB ? l2_policy_b() : l2_policy_a();
            if constexpr (CG == 1) tma_load_2d<HINT_AB>(dst, m, &sm->full[stage], x, y, pol);
            else tma_load_2d_cg2<HINT_AB>(dst, m, bar, x, y, pol);
          };
#pragma unroll
          for (int h = 0; h < MH; ++h) {
            const int64_t mrow_h = mrow + h * BM * CG;
            if (PN > 1 && mc) {
              tma_load_2d_cg2_mc<HINT_AB>(sa + h * C_::A_HALF + pn * A_ROWS * 128, &tmA, bar, ka, (int)mrow_h + pn * A_ROWS, mask_a, l2_policy_a());
            } else {
#pragma unroll
              for (int j = 0; j < PN; ++j) load(sa + h * C_::A_HALF + j * A_ROWS * 128, &tmA, ka, (int)mrow_h + j * A_ROWS);
            }
            load(se + h * 2048 * C_::META_ATOMS, &tmE, 0, (int)(((mrow_h / 128) * k_blocks + kb) * 16 * C_::META_ATOMS));
          }
          if (PM > 1 && mc) {
            tma_load_2d_cg2_mc<HINT_AB>(sb + pm * C_::B_HALF, &tmB, bar, kx + pm * C_::BOX, brow, mask_b, l2_policy_b());
          } else {
            load(sb, &tmB, kx, brow);
            load(sb + C_::B_HALF, &tmB, kx + C_::BOX, brow);
          }
          if (++stage == C_::STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (leader) {
      int stage = 0; uint32_t phase = 0;
      int acc = 0; uint32_t acc_phase = 0;
      // stage `st`, M-half h: metadata atoms -> TMEM (in order before the MMAs), then 4 sparse MMAs
      auto issue = [&](int st, int h, int64_t kb, uint32_t tmem_d) {
        if (k_nomma) return;
        const uint32_t sa = smem_u32(smem + st * C_::STAGE_BYTES) + h * C_::A_HALF;
        const uint32_t sb = smem_u32(smem + st * C_::STAGE_BYTES) + C_::A_BYTES;
        const uint32_t se = sb + C_::B_BYTES + h * 2048 * C_::META_ATOMS;
        const uint32_t tmeta = tmem_base + C_::META_COL + st * C_::META_COLS + h * 4 * C_::META_ATOMS;
#pragma unroll
        for (int a = 0; a < C_::META_ATOMS; ++a) tc05_cp_128x128b<CG>(tmeta + 4 * a, sdesc(se + 2048 * a, 128, 128, 0));
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          // MMA j: 32 bytes of kept A (K/2 logical), 64 bytes of B (one half of a SW128 box row)
          const uint64_t ad = sdesc(sa + j * 32, 16, 1024, 2);
          const uint64_t bd = sdesc(sb + (j >> 1) * C_::B_HALF + (j & 1) * 64, 16, 1024, 2);
          if constexpr (KIND == KIND_I8) {
            const uint32_t e = tmeta + 2 * j;          // 2 columns per MMA, selector 0
            umma_sp<CG, KIND_I8>(tmem_d, ad, bd, e, idesc, (kb | j) ? 1u : 0u);
          } else {
            const uint32_t e = tmeta + j;              // low address bit -> sparse selector
            umma_sp<CG, KIND>(tmem_d, ad, bd, e & ~1u, idesc | (e & 1u), (kb | j) ? 1u : 0u);
          }
        }
      };
      auto commit_slot = [&](uint64_t* bar) {
        if (P > 1 && mc) tc05_commit_mc(bar, (uint16_t)((1u << CL) - 1)); else tc05_commit<CG>(bar);
      };
      auto commit_acc = [&](uint64_t* bar) {
        if (P > 1 && mc) tc05_commit_mc(bar, (uint16_t)(3u << lead_rank)); else tc05_commit<CG>(bar);
      };
      for (int64_t tile = cluster_id; tile < num_tiles; tile += num_clusters) {
        int64_t kb0 = 0;
        if constexpr (!MW) {
          if constexpr (CG == 2) mbar_wait_cluster(&sm->tmem_empty[acc], acc_phase ^ 1);
          else mbar_wait(&sm->tmem_empty[acc], acc_phase ^ 1);
          tc05_fence_after();
        } else {
          // single buffer: half 0 for the first L resident stages while half 1 still drains
          const int64_t L = k_blocks < C_::STAGES ? k_blocks : C_::STAGES;
          const int st0 = stage;
          mbar_wait_cluster(&sm->tmem_empty[0], acc_phase ^ 1);
          tc05_fence_after();
          for (int64_t kb = 0; kb < L; ++kb) {
            mbar_wait(&sm->full[stage], phase);
            tc05_fence_after();
#if TCX_WATCHDOG
            if (kb == 0 && trace && tile < trace_cap && elect_one()) {   // debug tile timeline
              trace[4 * tile] = ((uint64_t)cluster_id << 32) | (uint64_t)tile;
              trace[4 * tile + 1] = globaltimer_ns();
            }
            __syncwarp();
#endif
            if (elect_one()) issue(stage, 0, kb, tmem_base);
            __syncwarp();
            if (++stage == C_::STAGES) { stage = 0; phase ^= 1; }
          }
          mbar_wait_cluster(&sm->tmem_empty[1], acc_phase ^ 1);
          tc05_fence_after();
          int st = st0;
          for (int64_t kb = 0; kb < L; ++kb) {
            if (elect_one()) {
              issue(st, 1, kb, tmem_base + BN);
              commit_slot(&sm->empty[st]);                       // every CTA that fed the slot
              if (kb == k_blocks - 1) commit_acc(&sm->tmem_full[0]);
            }
            __syncwarp();
            if (++st == C_::STAGES) st = 0;
          }
          kb0 = L;
        }
        const uint32_t tmem_d = tmem_base + acc * C_::ACC_STRIDE;
        for (int64_t kb = kb0; kb < k_blocks; ++kb) {
          mbar_wait(&sm->full[stage], phase);
          tc05_fence_after();
          if (elect_one()) {
#pragma unroll
            for (int h = 0; h < MH; ++h) issue(stage, h, kb, MW ? tmem_base + h * BN : tmem_d);
            commit_slot(&sm->empty[stage]);
            if (kb == k_blocks - 1) commit_acc(&sm->tmem_full[acc]);
#if TCX_WATCHDOG
            if (trace && tile < trace_cap) {                      // debug tile timeline
              if (!MW && kb == 0) {
                trace[4 * tile] = ((uint64_t)cluster_id << 32) | (uint64_t)tile;
                trace[4 * tile + 1] = globaltimer_ns();
              }
              if (kb == k_blocks - 1) trace[4 * tile + 2] = globaltimer_ns();
            }
#else
            (void)trace; (void)trace_cap;
#endif
          }
          __syncwarp();
          if (++stage == C_::STAGES) { stage = 0; phase ^= 1; }
        }
        if (MW) { acc_phase ^= 1; }
        else if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else if (warp >= 4) {
    // per 16-column chunk: tcgen05.ld (thread = row) -> (+ C chunk TMA-loaded into a 64B-swizzled
    // 2 KiB staging buffer) -> result back into the buffer -> one TMA store of the 32 x 16 box
    // (coalesced full-line HBM writes, TMA clips rows >= M / columns >= N).  STG_BUFS buffers per
    // warp rotate, the C chunk C_AHEAD ahead loading while this one is stored.
    const int e = warp - 4;
    const int lane = threadIdx.x & 31;
    constexpr int HCH = BN / 16;                 // chunks per accumulator (M-half)
    constexpr int CH = HCH * MH;                 // chunks per tile
    uint8_t* stg = smem + C_::SMEM_DATA + e * STG_BUFS * 2048;
    uint64_t* cbar = &sm->cbar[e][0];
    uint32_t cph = 0u;                            // bit b: phase of cbar[b] (a register, not a local array)
    const uint32_t tmem_empty_cluster = CG == 2 ? mapa(smem_u32(&sm->tmem_empty[0]), lead_rank) : smem_u32(&sm->tmem_empty[0]);
    const int64_t my_tiles = cluster_id < num_tiles ? (num_tiles - 1 - cluster_id) / num_clusters + 1 : 0;
    const int64_t nq = my_tiles * CH;
    // origins of the (at most two) tiles the epilogue addresses at a time — this one and the next —
    // cached, so the raster's 64-bit divisions (~800 cycles) run once per tile, not once per chunk
    int64_t oa_it = -1, ob_it = -1;
    int oa_x = 0, oa_y = 0, ob_x = 0, ob_y = 0;
    auto origin = [&](int64_t it, int& x, int& y) {
      if (it == oa_it) { x = oa_x; y = oa_y; return; }
      if (it == ob_it) { x = ob_x; y = ob_y; return; }
      int64_t mt, nt;
      pair_tile(cluster_id + it * num_clusters, mt, nt);
      x = (int)(nt * BN);
      y = (int)(mt * C_::TILE_M + rank * BM + e * 32);
      if (oa_it < ob_it) { oa_it = it; oa_x = x; oa_y = y; } else { ob_it = it; ob_x = x; ob_y = y; }
    };
    auto coords = [&](int64_t q, int& x, int& y) {
      origin(q / CH, x, y);
      const int ch = (int)(q % CH);
      y += (ch / HCH) * BM * CG;
      x += (ch % HCH) * 16;
    };
    auto load_c = [&](int64_t q) {
      if (has_c && lane == 0 && q < nq) {
        int x, y; coords(q, x, y);
        const int bq = (int)(q % STG_BUFS);
        mbar_arrive_expect_tx(&cbar[bq], 2048);
        tma_load_2d<HINT_C>(stg + bq * 2048, &tmC, &cbar[bq], x, y, l2_evict_first());
      }
    };
    // single-buffered (wide) tiles: the epilogue is on the critical path, so each tile's C is
    // L2-prefetched a tile ahead and its chunk loads hit L2 (double-buffered tiles hide the latency)
    auto prefetch_c_tile = [&](int64_t it) {
      if (MW && has_c && lane == 0 && it < my_tiles)
        for (int ch = 0; ch < CH; ++ch) { int x, y; coords(it * CH + ch, x, y); tma_prefetch_2d<HINT_C>(&tmC, x, y, l2_evict_first()); }
    };
    prefetch_c_tile(0);
    load_c(0);
    load_c(1);
    int acc = 0; uint32_t acc_phase = 0;
    const uint32_t lane_off = (uint32_t)(e * 32) << 16;
    for (int64_t it = 0; it < my_tiles; ++it) {
      prefetch_c_tile(it + 1);
      mbar_wait(&sm->tmem_full[acc], acc_phase);
      tc05_fence_after();
      uint32_t v[16], vn[16];
      // chunk ch lives at column (M-half) * BN + (ch % HCH) * 16 (MW) or acc * ACC_STRIDE + ch * 16
      auto tcol = [&](int ch) { return tmem_base + (MW ? (ch / HCH) * BN : acc * C_::ACC_STRIDE) + (ch % HCH) * 16 + lane_off; };
      tmem_ld_32x32b_x16(tcol(0), vn);
#pragma unroll 1
      for (int ch = 0; ch < CH; ++ch) {
        const int64_t q = it * CH + ch;
        const int b = (int)(q % STG_BUFS);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = vn[j];
        if (ch + 1 < CH) tmem_ld_32x32b_x16(tcol(ch + 1), vn);
        if (ch % HCH == HCH - 1) {
          // accumulator part read: MW -> M-half ch / HCH of the single buffer; else buffer `acc`
          tc05_fence_before();
          __syncwarp();
#if TCX_WATCHDOG
          // debug knob 16 (drain-cost experiment): hold the accumulator ~4 us longer before releasing it
          if ((knobs & 16) && lane == 0) { const uint64_t t0 = globaltimer_ns(); while (globaltimer_ns() - t0 < 4000) {} }
#endif
          if (lane == 0) mbar_arrive_cluster(tmem_empty_cluster + (MW ? ch / HCH : acc) * 8);
        }
        if (has_c) {
          mbar_wait(&cbar[b], (cph >> b) & 1u);
          cph ^= 1u << b;
        } else if (q >= STG_BUFS) {
          if (lane == 0) bulk_wait_read<STG_BUFS - 1>();   // the store of chunk q - STG_BUFS has read buffer b
          __syncwarp();
        }
        const uint32_t rowa = smem_u32(stg) + b * 2048 + lane * 64;   // this thread's row of the box
        uint4 cv[4];                                           // all C loads first: 4 in flight
        if (has_c) {
#pragma unroll
          for (int j = 0; j < 4; ++j) cv[j] = lds128(rowa + ((j ^ ((lane >> 1) & 3)) * 16));
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint32_t pa = rowa + ((j ^ ((lane >> 1) & 3)) * 16);   // SW64: chunk j at j ^ ((row/2) % 4)
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
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0 && !k_noepi) {
          int x, y; coords(q, x, y);
          tma_store_2d<HINT_D>(&tmD, stg + b * 2048, x, y, l2_evict_first());
          bulk_commit();
          // the buffer of chunk q + C_AHEAD was last read by the store of chunk q + C_AHEAD - STG_BUFS
          if (has_c && q + C_AHEAD < nq) bulk_wait_read<STG_BUFS - C_AHEAD>();
        }
        load_c(q + C_AHEAD);
      }
#if TCX_WATCHDOG
      if (trace && e == 0 && lane == 0 && rank == 0) {
        const int64_t tile = cluster_id + it * num_clusters;
        if (tile < trace_cap) trace[4 * tile + 3] = globaltimer_ns();
      }
#endif
      if (MW) { acc_phase ^= 1; }
      else if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
    if (lane == 0) bulk_wait<0>();
  }

  tc05_fence_before();
  if constexpr (CG == 2) cluster_sync(); else __syncthreads();
  if (warp == 2) { tc05_fence_after(); tmem_dealloc<CG>(tmem_base, 512); }
}

template <int CG, int KIND, int MW = 0, int PM = 1, int PN = 1>
tcx_status launch_sp(const GemmArgs& a, const DevInfo& dev, cudaStream_t s) {
  constexpr int CL = CG * PM * PN;
  using C_ = SpCfg<CG, KIND, MW>;
  if (a.M % C_::TILE_M) return set_error(TCX_ERR_UNSUPPORTED, "tcx_gemm_sp24: M %% %d != 0", C_::TILE_M);
  const CUtensorMapDataType dt = KIND == KIND_I8 ? CU_TENSOR_MAP_DATA_TYPE_UINT8
                                 : KIND == KIND_TF32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                 : a.ab == TCX_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
  CUtensorMap tA, tB, tE;
  tcx_status st = make_tmap_2d(&tA, dt, a.A, (uint64_t)(a.K / 2), (uint64_t)a.M, (uint64_t)(a.lda * C_::ES), C_::BOX, BM / PN,
                               CU_TENSOR_MAP_SWIZZLE_128B);
  if (st != TCX_OK) return st;
  st = make_tmap_2d(&tB, dt, a.B, (uint64_t)a.K, (uint64_t)a.N, (uint64_t)(a.ldb * C_::ES), C_::BOX, C_::BN_LOAD,
                    CU_TENSOR_MAP_SWIZZLE_128B);
  if (st != TCX_OK) return st;
  const uint64_t meta_rows = (uint64_t)(a.M * a.K * (KIND == KIND_TF32 ? 2 : 1) / 8) / 128;
  st = make_tmap_2d(&tE, CU_TENSOR_MAP_DATA_TYPE_UINT8, a.meta_hw, 128, meta_rows, 128, 128, 16 * C_::META_ATOMS,
                    CU_TENSOR_MAP_SWIZZLE_NONE);
  if (st != TCX_OK) return st;
  // C and D: 32-row x 16-column boxes of 4-byte elements (64-byte rows), 64B-swizzled staging
  CUtensorMap tC, tD;
  st = make_tmap_2d(&tD, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, a.D, (uint64_t)a.N, (uint64_t)a.M, (uint64_t)(a.ldd * 4),
                    16, 32, CU_TENSOR_MAP_SWIZZLE_64B);
  if (st != TCX_OK) return st;
  if (a.C) {
    st = make_tmap_2d(&tC, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, a.C, (uint64_t)a.N, (uint64_t)a.M, (uint64_t)(a.ldc * 4),
                      16, 32, CU_TENSOR_MAP_SWIZZLE_64B);
    if (st != TCX_OK) return st;
  } else {
    tC = tD;
  }
  auto kern = gemm_sp24_kernel<CG, KIND, MW, PM, PN>;
  TCX_CUDA_TRY(ensure_max_smem((const void*)kern, C_::SMEM_TOTAL, dev.device));
  const int64_t m_tiles = a.M / C_::TILE_M, n_tiles = (a.N + BN - 1) / BN;
  int64_t clusters = ((m_tiles + PM - 1) / PM) * ((n_tiles + PN - 1) / PN);
  int64_t max_clusters = dev.sm_count / CL;
  if (a.max_ctas > 0 && a.max_ctas / CL < max_clusters) max_clusters = a.max_ctas / CL > 0 ? a.max_ctas / CL : 1;
  if (clusters > max_clusters) clusters = max_clusters;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(clusters * CL));
  cfg.blockDim = dim3(NUM_THREADS);
  cfg.dynamicSmemBytes = C_::SMEM_TOTAL;
  cfg.stream = s;
  cudaLaunchAttribute attr[3];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;     // PDL (see pdl_wait in the kernel)
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = CG; attr[1].val.clusterDim.y = 1; attr[1].val.clusterDim.z = 1;
  attr[2].id = cudaLaunchAttributePreferredClusterDimension;
  attr[2].val.preferredClusterDim.x = CL; attr[2].val.preferredClusterDim.y = 1; attr[2].val.preferredClusterDim.z = 1;
  cfg.attrs = attr; cfg.numAttrs = CL > CG ? 3 : 2;
  // idesc: sparse flag [2], c format [4,6) (F32 = 1, S32 = 2), a/b format [7,10)/[10,13)
  // (f16 0, bf16 1; s8 signed 1), N>>3 [17,23), M>>4 [24,29); saturate [3] = 0 (wrap)
  const uint32_t fmt = KIND == KIND_TF32 ? 2u : (KIND == KIND_I8 || a.ab == TCX_BF16) ? 1u : 0u;
  const uint32_t cfmt = KIND == KIND_I8 ? 2u : 1u;
  const uint32_t idesc = (1u << 2) | (cfmt << 4) | (fmt << 7) | (fmt << 10) | ((uint32_t)(BN >> 3) << 17) |
                         ((uint32_t)((BM * CG) >> 4) << 24);
  TCX_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, tA, tB, tE, tC, tD, (int64_t)a.M, (int64_t)a.N, (int64_t)a.K,
                                  a.C ? 1 : 0, idesc, a.group_m != 0 ? a.group_m : GROUP_M, a.trace, a.trace_cap,
                                  a.fault));
  count_launch();
  return TCX_OK;
}

template <int KIND>
tcx_status launch_sp_kind(const GemmArgs& a, const DevInfo& dev, cudaStream_t s) {
  if (a.cta_group == 1) return launch_sp<1, KIND>(a, dev, s);
  // tile_m = 512 (opts.tile_n field reused as the sparse tile height): the 512 x 240 M-wide pair
  // tile (F16/BF16/TF32, M % 512 == 0, no multicast group) is the default when each tile's K loop
  // is long — K >= 16384 for F16/BF16, K >= 8192 for TF32 (half the MMA rate) — so its
  // single-buffer drain is a small share of the tile, and when its tiles fill the SMs' waves about
  // as well as the 256-row tiles do: its 31% fewer operand bytes per FLOP then win at the power cap
  // (burst A/B over 8 shapes, profiles/r02_studies/sparse_tile_height/: K = 16384 F16 +3-4% incl.
  // C5, TF32 8192^3 +3.2%, 16384^3 +13%; K = 8192 F16 the 256-row tile +5-8%).  tile_n = 256 /
  // 512 forces either.
  if constexpr (KIND != KIND_I8) {
    const bool grouped = a.pairs_m > 1 || a.pairs_n > 1;
    const int64_t k_time = a.K * (KIND == KIND_TF32 ? 2 : 1);      // the K loop in F16-MMA units
    int64_t pairs = dev.sm_count / 2;
    if (a.max_ctas > 0 && a.max_ctas / 2 < pairs) pairs = a.max_ctas / 2 > 0 ? a.max_ctas / 2 : 1;
    const int64_t nt = (a.N + 239) / 240;
    auto fill = [&](int64_t tiles) { return (double)tiles / (double)(((tiles + pairs - 1) / pairs) * pairs); };
    const bool long_call = k_time >= 16384 && fill((a.M / 512) * nt) >= 0.97 * fill(((a.M + 255) / 256) * nt);
    if (a.M % 512 == 0 && (a.tile_n == 512 || (a.tile_n == 0 && !grouped && long_call))) {
      // M-wide tile, optionally in multicast groups of pairs: pairs_m pairs of a column share B
      // (1024 x 240 per group), pairs_n pairs of a row share sA and metadata rows (512 x 480)
      if (a.pairs_m == 2 && a.pairs_n == 2) return launch_sp<2, KIND, 1, 2, 2>(a, dev, s);
      if (a.pairs_m == 2) return launch_sp<2, KIND, 1, 2, 1>(a, dev, s);
      if (a.pairs_n == 2) return launch_sp<2, KIND, 1, 1, 2>(a, dev, s);
      return launch_sp<2, KIND, 1>(a, dev, s);
    }
  }
  if (a.pairs_m == 2 && a.pairs_n == 2) return launch_sp<2, KIND, 0, 2, 2>(a, dev, s);
  if (a.pairs_m == 2) return launch_sp<2, KIND, 0, 2, 1>(a, dev, s);
  if (a.pairs_n == 2) return launch_sp<2, KIND, 0, 1, 2>(a, dev, s);
  return launch_sp<2, KIND>(a, dev, s);
}

}  // namespace

tcx_status launch_gemm_sp24(const GemmArgs& a, const DevInfo& dev, cudaStream_t s) {
  if (a.ab == TCX_S8) return launch_sp_kind<KIND_I8>(a, dev, s);
  if (a.ab == TCX_TF32) return launch_sp_kind<KIND_TF32>(a, dev, s);
  return launch_sp_kind<KIND_F16>(a, dev, s);
}

}  // namespace tcx
