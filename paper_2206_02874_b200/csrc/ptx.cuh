// tcx — thin inline-PTX wrappers for sm_100a (tcgen05 / TMEM / TMA / mbarrier / clusters).
// Product code.  Shares nothing with oracle/.
#pragma once
#include <cstdint>
#include <cuda.h>

#ifndef TCX_WATCHDOG
#define TCX_WATCHDOG 0
#endif

namespace tcx {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// 16-byte shared-window accesses by 32-bit address: LDS.128 / STS.128.  A dereference of the
// aligned extern-shared pointer compiles to generic LD/ST.E.128 (64-bit address arithmetic, the
// generic-window check) because the alignment cast loses the address space.  volatile + memory
// clobber keep them ordered with the mbarrier waits and proxy fences around them.
__device__ __forceinline__ uint4 lds128(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void sts128(uint32_t a, uint4 v) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" :: "r"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}


__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred P;\n\t"
      "elect.sync _|P, 0xffffffff;\n\t"
      "selp.u32 %0, 1, 0, P;\n\t}"
      : "=r"(pred));
  return pred != 0;
}

// ------------------------------------------------------------------ clusters
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r;
}
__device__ __forceinline__ uint32_t cluster_nctarank() {
  uint32_t r; asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r)); return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// map a shared::cta address of this CTA to the same offset in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa(uint32_t addr, uint32_t rank) {
  uint32_t r; asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank)); return r;
}

// ------------------------------------------------------------------ mbarrier
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;"
               :: "r"(smem_u32(bar)), "r"(bytes) : "memory");
}
// arrive on a barrier given by its shared::cluster address (may live in the peer CTA)
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" :: "r"(cluster_addr) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint32_t addr, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, P;\n\t}"
      : "=r"(ok) : "r"(addr), "r"(parity) : "memory");
  return ok != 0;
}
__device__ __forceinline__ bool mbar_try_wait_cluster(uint32_t addr, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P;\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, P;\n\t}"
      : "=r"(ok) : "r"(addr), "r"(parity) : "memory");
  return ok != 0;
}
// Debug builds (libtcx_debug.so, -DTCX_WATCHDOG=1) bound every barrier wait: a phase that does not
// complete within TCX_WATCHDOG_NS of wall time (globaltimer) traps, so a pipeline bug becomes a
// launch error returned through the C-ABI instead of a hung GPU.
#ifndef TCX_WATCHDOG_NS
#define TCX_WATCHDOG_NS 4000000000ull
#endif
__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t a = smem_u32(bar);
#if TCX_WATCHDOG
  const uint64_t t0 = globaltimer_ns();
#endif
  while (!mbar_try_wait(a, parity)) {
#if TCX_WATCHDOG
    if (globaltimer_ns() - t0 > TCX_WATCHDOG_NS) __trap();
#endif
  }
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  uint32_t a = smem_u32(bar);
#if TCX_WATCHDOG
  const uint64_t t0 = globaltimer_ns();
#endif
  while (!mbar_try_wait_cluster(a, parity)) {
#if TCX_WATCHDOG
    if (globaltimer_ns() - t0 > TCX_WATCHDOG_NS) __trap();
#endif
  }
}

// ------------------------------------------------------------------ fences
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tc05_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc05_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// ------------------------------------------------------------------ programmatic dependent launch
// launch_dependents: the next grid in the stream may begin launching (its CTAs take SMs as this
// grid's CTAs exit); wait: block until the previous grid has completed and its memory is visible.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// ------------------------------------------------------------------ TMA
__device__ __forceinline__ void tma_prefetch(const CUtensorMap* m) {
  asm volatile("prefetch.tensormap [%0];" :: "l"(reinterpret_cast<uint64_t>(m)) : "memory");
}
// L2 eviction priority of a TMA transfer (`.L2::cache_hint` + a createpolicy operand): the operand
// tiles a raster group re-reads stay (evict_last), the C/D streams touched once leave first
// (evict_first).  H = false issues the plain form; `pol` is then ignored.
#ifndef TCX_L2HINT
#define TCX_L2HINT 0      // bit 0: C loads/prefetches evict_first, bit 1: D stores evict_first,
#endif                    // bit 2: A/B loads evict_last, bit 3: A/B loads evict_normal (explicit),
                          // bit 4: B loads evict_first, bit 5: A (+ sparse metadata) loads evict_last
constexpr bool HINT_C = (TCX_L2HINT & 1) != 0;
constexpr bool HINT_D = (TCX_L2HINT & 2) != 0;
constexpr bool HINT_AB = (TCX_L2HINT & 60) != 0;
__device__ __forceinline__ uint64_t l2_evict_first() {
  uint64_t p; asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p)); return p;
}
__device__ __forceinline__ uint64_t l2_evict_last() {
  uint64_t p; asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p)); return p;
}
__device__ __forceinline__ uint64_t l2_evict_normal() {
  uint64_t p; asm("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p)); return p;
}
__device__ __forceinline__ uint64_t l2_policy_a() { return (TCX_L2HINT & 36) ? l2_evict_last() : l2_evict_normal(); }
__device__ __forceinline__ uint64_t l2_policy_b() {
  return (TCX_L2HINT & 16) ? l2_evict_first() : (TCX_L2HINT & 4) ? l2_evict_last() : l2_evict_normal();
}

// 2D tile load into this CTA's smem, completion on this CTA's barrier
template <bool H = false>
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* m, uint64_t* bar, int x, int y,
                                            uint64_t pol = 0) {
  if constexpr (H)
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%3, %4}], [%2], %5;"
        :: "r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(x), "r"(y), "l"(pol)
        : "memory");
  else
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
        :: "r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(x), "r"(y)
        : "memory");
}
// 2D tile load for a CTA pair: data lands in this CTA's smem, complete_tx goes to the
// barrier at `bar_cluster` (a shared::cluster address, normally the leader CTA's barrier)
template <bool H = false>
__device__ __forceinline__ void tma_load_2d_cg2(void* dst, const CUtensorMap* m, uint32_t bar_cluster, int x, int y,
                                                uint64_t pol = 0) {
  if constexpr (H)
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%3, %4}], [%2], %5;"
        :: "r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(m)), "r"(bar_cluster), "r"(x), "r"(y), "l"(pol)
        : "memory");
  else
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
        :: "r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(m)), "r"(bar_cluster), "r"(x), "r"(y)
        : "memory");
}
// the same, multicast: the box lands at this smem offset in every CTA of `mask`; each destination's
// complete_tx goes to the barrier at the same offset in the CTA of the destination's pair that
// `bar_cluster` names (the pair leader)
template <bool H = false>
__device__ __forceinline__ void tma_load_2d_cg2_mc(void* dst, const CUtensorMap* m, uint32_t bar_cluster, int x, int y,
                                                   uint16_t mask, uint64_t pol = 0) {
  if constexpr (H)
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
        ".L2::cache_hint [%0], [%1, {%3, %4}], [%2], %5, %6;"
        :: "r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(m)), "r"(bar_cluster), "r"(x), "r"(y), "h"(mask),
           "l"(pol)
        : "memory");
  else
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
        " [%0], [%1, {%3, %4}], [%2], %5;"
        :: "r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(m)), "r"(bar_cluster), "r"(x), "r"(y), "h"(mask)
        : "memory");
}
// multicast to the CTAs of `mask` (no CTA pair): each destination's complete_tx goes to the barrier
// at the same offset in that destination CTA
__device__ __forceinline__ void tma_load_2d_mc(void* dst, const CUtensorMap* m, uint64_t* bar, int x, int y,
                                               uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1, {%3, %4}], [%2], %5;"
      :: "r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(x), "r"(y), "h"(mask)
      : "memory");
}
// L2 prefetch of a 2D tile (no smem, no barrier): warms L2 so a later load of the same box hits
template <bool H = false>
__device__ __forceinline__ void tma_prefetch_2d(const CUtensorMap* m, int x, int y, uint64_t pol = 0) {
  if constexpr (H)
    asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile.L2::cache_hint [%0, {%1, %2}], %3;"
                 :: "l"(reinterpret_cast<uint64_t>(m)), "r"(x), "r"(y), "l"(pol) : "memory");
  else
    asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];"
                 :: "l"(reinterpret_cast<uint64_t>(m)), "r"(x), "r"(y) : "memory");
}
template <bool H = false>
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* m, const void* src, int x, int y, uint64_t pol = 0) {
  if constexpr (H)
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%2, %3}], [%1], %4;"
                 :: "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(src)), "r"(x), "r"(y), "l"(pol) : "memory");
  else
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];"
                 :: "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(src)), "r"(x), "r"(y) : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" :: "n"(N) : "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait() {
  asm volatile("cp.async.bulk.wait_group %0;" :: "n"(N) : "memory");
}

// ------------------------------------------------------------------ TMEM
template <int CG>
__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {
  if constexpr (CG == 1)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" :: "r"(smem_u32(dst_smem)), "r"(ncols) : "memory");
  else
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" :: "r"(smem_u32(dst_smem)), "r"(ncols) : "memory");
}
template <int CG>
__device__ __forceinline__ void tmem_relinquish() {
  if constexpr (CG == 1) asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  else asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
template <int CG>
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  if constexpr (CG == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(taddr), "r"(ncols) : "memory");
  else asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" :: "r"(taddr), "r"(ncols) : "memory");
}

// tcgen05.commit: arrive (once) on an mbarrier when all prior tcgen05 ops of this thread finish
template <int CG>
__device__ __forceinline__ void tc05_commit(uint64_t* bar) {
  if constexpr (CG == 1)
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(smem_u32(bar)) : "memory");
  else
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                 :: "r"(smem_u32(bar)), "h"((uint16_t)0x3) : "memory");
}
// CTA-pair commit arriving on the barrier at this offset in every CTA of `mask`
__device__ __forceinline__ void tc05_commit_mc(uint64_t* bar, uint16_t mask) {
  asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
               :: "r"(smem_u32(bar)), "h"(mask) : "memory");
}

// ------------------------------------------------------------------ UMMA descriptors
// shared-memory matrix descriptor (sm_100): start>>4 [0,14), LBO>>4 [16,30), SBO>>4 [32,46),
// version=1 [46,48), base offset [49,52), lbo mode [52], layout [61,64) (SW128 = 2, none = 0)
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46) | ((uint64_t)(layout & 7u) << 61);
}

// kinds
enum : int { KIND_F16 = 0, KIND_TF32 = 1, KIND_I8 = 2 };

template <int CG, int KIND>
__device__ __forceinline__ void umma(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t accumulate) {
#define TCX_UMMA(CGS, KS)                                                                  \
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"                           \
               "tcgen05.mma.cta_group::" CGS ".kind::" KS " [%0], %1, %2, %3, p;\n\t}"     \
               :: "r"(tmem_d), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate) : "memory")
  if constexpr (CG == 1) {
    if constexpr (KIND == KIND_F16) TCX_UMMA("1", "f16");
    else if constexpr (KIND == KIND_TF32) TCX_UMMA("1", "tf32");
    else TCX_UMMA("1", "i8");
  } else {
    if constexpr (KIND == KIND_F16) TCX_UMMA("2", "f16");
    else if constexpr (KIND == KIND_TF32) TCX_UMMA("2", "tf32");
    else TCX_UMMA("2", "i8");
  }
#undef TCX_UMMA
}

// sparse: metadata operand is a TMEM address
template <int CG, int KIND>
__device__ __forceinline__ void umma_sp(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t tmem_e,
                                        uint32_t idesc, uint32_t accumulate) {
#define TCX_UMMA_SP(CGS, KS)                                                                     \
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %5, 0;\n\t"                                 \
               "tcgen05.mma.sp.cta_group::" CGS ".kind::" KS " [%0], %1, %2, [%3], %4, p;\n\t}"   \
               :: "r"(tmem_d), "l"(adesc), "l"(bdesc), "r"(tmem_e), "r"(idesc), "r"(accumulate) : "memory")
  if constexpr (CG == 1) {
    if constexpr (KIND == KIND_F16) TCX_UMMA_SP("1", "f16");
    else if constexpr (KIND == KIND_TF32) TCX_UMMA_SP("1", "tf32");
    else TCX_UMMA_SP("1", "i8");
  } else {
    if constexpr (KIND == KIND_F16) TCX_UMMA_SP("2", "f16");
    else if constexpr (KIND == KIND_TF32) TCX_UMMA_SP("2", "tf32");
    else TCX_UMMA_SP("2", "i8");
  }
#undef TCX_UMMA_SP
}

// A-operand collector usage (tcgen05.mma .collector::a::*): FILL keeps this MMA's A in the collector
// buffer, USE / LASTUSE read it from there instead of shared memory (LASTUSE releases it) — two MMAs
// that share A (different B / accumulator) read A from smem once
enum : int { COLL_NONE = 0, COLL_FILL = 1, COLL_USE = 2, COLL_LASTUSE = 3 };
template <int CG, int KIND, int COLL>
__device__ __forceinline__ void umma_c(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t accumulate) {
  if constexpr (COLL == COLL_NONE) { umma<CG, KIND>(tmem_d, adesc, bdesc, idesc, accumulate); return; }
#define TCX_UMMA_C(CGS, KS, CS)                                                                       \
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"                                   \
               "tcgen05.mma.cta_group::" CGS ".kind::" KS ".collector::a::" CS " [%0], %1, %2, %3, p;\n\t}" \
               :: "r"(tmem_d), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate) : "memory")
#define TCX_UMMA_C_K(CGS, CS)                                     \
  if constexpr (KIND == KIND_F16) TCX_UMMA_C(CGS, "f16", CS);      \
  else if constexpr (KIND == KIND_TF32) TCX_UMMA_C(CGS, "tf32", CS); \
  else TCX_UMMA_C(CGS, "i8", CS);
  if constexpr (CG == 1) {
    if constexpr (COLL == COLL_FILL) { TCX_UMMA_C_K("1", "fill") }
    else if constexpr (COLL == COLL_USE) { TCX_UMMA_C_K("1", "use") }
    else { TCX_UMMA_C_K("1", "lastuse") }
  } else {
    if constexpr (COLL == COLL_FILL) { TCX_UMMA_C_K("2", "fill") }
    else if constexpr (COLL == COLL_USE) { TCX_UMMA_C_K("2", "use") }
    else { TCX_UMMA_C_K("2", "lastuse") }
  }
#undef TCX_UMMA_C_K
#undef TCX_UMMA_C
}
template <int CG, int KIND, int COLL>
__device__ __forceinline__ void umma_sp_c(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t tmem_e, uint32_t idesc,
                                          uint32_t accumulate) {
  if constexpr (COLL == COLL_NONE) { umma_sp<CG, KIND>(tmem_d, adesc, bdesc, tmem_e, idesc, accumulate); return; }
#define TCX_UMMA_SPC(CGS, KS, CS)                                                                          \
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %5, 0;\n\t"                                        \
               "tcgen05.mma.sp.cta_group::" CGS ".kind::" KS ".collector::a::" CS " [%0], %1, %2, [%3], %4, p;\n\t}" \
               :: "r"(tmem_d), "l"(adesc), "l"(bdesc), "r"(tmem_e), "r"(idesc), "r"(accumulate) : "memory")
#define TCX_UMMA_SPC_K(CGS, CS)                                       \
  if constexpr (KIND == KIND_F16) TCX_UMMA_SPC(CGS, "f16", CS);        \
  else if constexpr (KIND == KIND_TF32) TCX_UMMA_SPC(CGS, "tf32", CS); \
  else TCX_UMMA_SPC(CGS, "i8", CS);
  if constexpr (CG == 1) {
    if constexpr (COLL == COLL_FILL) { TCX_UMMA_SPC_K("1", "fill") }
    else if constexpr (COLL == COLL_USE) { TCX_UMMA_SPC_K("1", "use") }
    else { TCX_UMMA_SPC_K("1", "lastuse") }
  } else {
    if constexpr (COLL == COLL_FILL) { TCX_UMMA_SPC_K("2", "fill") }
    else if constexpr (COLL == COLL_USE) { TCX_UMMA_SPC_K("2", "use") }
    else { TCX_UMMA_SPC_K("2", "lastuse") }
  }
#undef TCX_UMMA_SPC_K
#undef TCX_UMMA_SPC
}

// smem -> TMEM copy, 128 lanes x 128 bits
template <int CG>
__device__ __forceinline__ void tc05_cp_128x128b(uint32_t tmem_addr, uint64_t sdesc_) {
  if constexpr (CG == 1) asm volatile("tcgen05.cp.cta_group::1.128x128b [%0], %1;" :: "r"(tmem_addr), "l"(sdesc_) : "memory");
  else asm volatile("tcgen05.cp.cta_group::2.128x128b [%0], %1;" :: "r"(tmem_addr), "l"(sdesc_) : "memory");
}

// TMEM -> registers: 32 lanes (one per thread) x 32 consecutive 32-bit columns
__device__ __forceinline__ void tmem_ld_32x32b_x32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
// TMEM -> registers: 32 lanes x 16 consecutive 32-bit columns
__device__ __forceinline__ void tmem_ld_32x32b_x16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// registers -> TMEM: 32 lanes x 8 columns
__device__ __forceinline__ void tmem_st_32x32b_x8(uint32_t taddr, const uint32_t (&r)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
               :: "r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
               : "memory");
}
// registers -> TMEM: 32 lanes x 32 columns
__device__ __forceinline__ void tmem_st_32x32b_x32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
      :: "r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
         "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]),
         "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]),
         "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }


}  // namespace tcx
