// tcx_probe — the paper's clock-counter microbenchmark on sm_100a (Fig.
// code-benchmark):
//   each issuer runs ITERS iterations of ILP independent MMAs, every slot a dependency chain across
//   iterations (D_i feeds the next C_i), with a warp sync at the end of each iteration;
//   latency = cycles / ITERS; throughput = issuers*ILP*m*n*k / latency.
// Kinds:
//   MMA_SYNC / MMA_SP_SYNC: the paper's own warp-level instructions (mma.sync / mma.sp), every shape
//     of Tables A100-mma and A100-mmasp.
//   TC05 / TC05_SP: tcgen05.mma(.sp) issued by one thread per CTA; an "iteration" is ILP MMAs then
//     tcgen05.commit -> mbarrier wait (the analogue of the paper's per-iteration sync).
// Also here: tcx_mma_tiles_tc05, the numeric-probe tile batch through tcgen05 with C preloaded into
// tensor memory (8 tiles packed block-diagonally into one M=128,N=64 MMA).
#include <algorithm>
#include <vector>
#include "tcx_internal.h"
#include "ptx.cuh"

namespace tcx {
namespace {

__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t;
}

// ------------------------------------------------------------------ mma.sync instruction table
#define MMA4_4_2(NAME, PTX)                                                                       \
  struct NAME { using CT = float; static constexpr int NA = 4, NB = 2, NC = 4;                    \
    __device__ static void mma(CT* c, const uint32_t* a, const uint32_t* b, uint32_t) {           \
      asm volatile(PTX " {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"                   \
                   : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])                               \
                   : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1])); } };
#define MMA4_2_1(NAME, PTX)                                                                       \
  struct NAME { using CT = float; static constexpr int NA = 2, NB = 1, NC = 4;                    \
    __device__ static void mma(CT* c, const uint32_t* a, const uint32_t* b, uint32_t) {           \
      asm volatile(PTX " {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"                            \
                   : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3]) : "r"(a[0]), "r"(a[1]), "r"(b[0])); } };
#define MMAI4_4_2(NAME, PTX)                                                                      \
  struct NAME { using CT = uint32_t; static constexpr int NA = 4, NB = 2, NC = 4;                 \
    __device__ static void mma(CT* c, const uint32_t* a, const uint32_t* b, uint32_t) {           \
      asm volatile(PTX " {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"                   \
                   : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])                               \
                   : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1])); } };
#define MMAI4_2_1(NAME, PTX)                                                                      \
  struct NAME { using CT = uint32_t; static constexpr int NA = 2, NB = 1, NC = 4;                 \
    __device__ static void mma(CT* c, const uint32_t* a, const uint32_t* b, uint32_t) {           \
      asm volatile(PTX " {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"                            \
                   : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3]) : "r"(a[0]), "r"(a[1]), "r"(b[0])); } };
#define MMAH2_4_2(NAME, PTX)                                                                      \
  struct NAME { using CT = uint32_t; static constexpr int NA = 4, NB = 2, NC = 2;                 \
    __device__ static void mma(CT* c, const uint32_t* a, const uint32_t* b, uint32_t) {           \
      asm volatile(PTX " {%0,%1}, {%2,%3,%4,%5}, {%6,%7}, {%0,%1};"                               \
                   : "+r"(c[0]), "+r"(c[1]) : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1])); } };
#define MMAH2_2_1(NAME, PTX)                                                                      \
  struct NAME { using CT = uint32_t; static constexpr int NA = 2, NB = 1, NC = 2;                 \
    __device__ static void mma(CT* c, const uint32_t* a, const uint32_t* b, uint32_t) {           \
      asm volatile(PTX " {%0,%1}, {%2,%3}, {%4}, {%0,%1};" : "+r"(c[0]), "+r"(c[1]) : "r"(a[0]), "r"(a[1]), "r"(b[0])); } };
#define MMAI2_1_1(NAME, PTX)                                                                      \
  struct NAME { using CT = uint32_t; static constexpr int NA = 1, NB = 1, NC = 2;                 \
    __device__ static void mma(CT* c, const uint32_t* a, const uint32_t* b, uint32_t) {           \
      asm volatile(PTX " {%0,%1}, {%2}, {%3}, {%0,%1};" : "+r"(c[0]), "+r"(c[1]) : "r"(a[0]), "r"(b[0])); } };
#define SP4_4_4(NAME, PTX, CTY, CON)                                                              \
  struct NAME { using CT = CTY; static constexpr int NA = 4, NB = 4, NC = 4;                      \
    __device__ static void mma(CT* c, const uint32_t* a, const uint32_t* b, uint32_t e) {         \
      asm volatile(PTX " {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9,%10,%11}, {%0,%1,%2,%3}, %12, 0x0;" \
                   : CON(c[0]), CON(c[1]), CON(c[2]), CON(c[3])                                   \
                   : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]), "r"(b[2]), "r"(b[3]), "r"(e)); } };
#define SP4_2_2(NAME, PTX, CTY, CON)                                                              \
  struct NAME { using CT = CTY; static constexpr int NA = 2, NB = 2, NC = 4;                      \
    __device__ static void mma(CT* c, const uint32_t* a, const uint32_t* b, uint32_t e) {         \
      asm volatile(PTX " {%0,%1,%2,%3}, {%4,%5}, {%6,%7}, {%0,%1,%2,%3}, %8, 0x0;"                \
                   : CON(c[0]), CON(c[1]), CON(c[2]), CON(c[3])                                   \
                   : "r"(a[0]), "r"(a[1]), "r"(b[0]), "r"(b[1]), "r"(e)); } };
#define FCON(x) "+f"(x)
#define ICON(x) "+r"(x)

MMA4_4_2(F16F32_16816, "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32")
MMA4_2_1(F16F32_1688, "mma.sync.aligned.m16n8k8.row.col.f32.f16.f16.f32")
MMAH2_4_2(F16F16_16816, "mma.sync.aligned.m16n8k16.row.col.f16.f16.f16.f16")
MMAH2_2_1(F16F16_1688, "mma.sync.aligned.m16n8k8.row.col.f16.f16.f16.f16")
MMA4_4_2(BF16F32_16816, "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32")
MMA4_2_1(BF16F32_1688, "mma.sync.aligned.m16n8k8.row.col.f32.bf16.bf16.f32")
MMA4_4_2(TF32_1688, "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32")
MMA4_2_1(TF32_1684, "mma.sync.aligned.m16n8k4.row.col.f32.tf32.tf32.f32")
MMAI2_1_1(S8_8816, "mma.sync.aligned.m8n8k16.row.col.s32.s8.s8.s32")
MMAI4_4_2(S8_16832, "mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32")
MMAI4_2_1(S8_16816, "mma.sync.aligned.m16n8k16.row.col.s32.s8.s8.s32")
SP4_4_4(SP_F16_16832, "mma.sp::ordered_metadata.sync.aligned.m16n8k32.row.col.f32.f16.f16.f32", float, FCON)
SP4_2_2(SP_F16_16816, "mma.sp::ordered_metadata.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32", float, FCON)
SP4_4_4(SP_BF16_16832, "mma.sp::ordered_metadata.sync.aligned.m16n8k32.row.col.f32.bf16.bf16.f32", float, FCON)
SP4_2_2(SP_BF16_16816, "mma.sp::ordered_metadata.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32", float, FCON)
SP4_4_4(SP_TF32_16816, "mma.sp::ordered_metadata.sync.aligned.m16n8k16.row.col.f32.tf32.tf32.f32", float, FCON)
SP4_2_2(SP_TF32_1688, "mma.sp::ordered_metadata.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32", float, FCON)
SP4_4_4(SP_S8_16864, "mma.sp::ordered_metadata.sync.aligned.m16n8k64.row.col.s32.s8.s8.s32", uint32_t, ICON)
SP4_2_2(SP_S8_16832, "mma.sp::ordered_metadata.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32", uint32_t, ICON)

template <class I, int ILP>
__global__ void probe_mma_kernel(int iters, long long* __restrict__ cycles, long long* __restrict__ ns,
                                 uint32_t* __restrict__ sink, uint32_t aval, uint32_t meta) {
  typename I::CT c[ILP][I::NC];
  uint32_t a[I::NA], b[I::NB];
#pragma unroll
  for (int i = 0; i < I::NA; ++i) a[i] = aval ^ (threadIdx.x & 1u);
#pragma unroll
  for (int i = 0; i < I::NB; ++i) b[i] = aval;
#pragma unroll
  for (int s = 0; s < ILP; ++s)
#pragma unroll
    for (int j = 0; j < I::NC; ++j) c[s][j] = 0;
  // warm-up (instruction cache, first-issue effects)
  for (int it = 0; it < 4; ++it) {
#pragma unroll
    for (int s = 0; s < ILP; ++s) I::mma(c[s], a, b, meta);
    __syncwarp();
  }
  __syncthreads();
  const long long t0 = clock64();
  const uint64_t g0 = globaltimer();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int s = 0; s < ILP; ++s) I::mma(c[s], a, b, meta);
    __syncwarp();
  }
  const long long t1 = clock64();
  const uint64_t g1 = globaltimer();
  uint32_t x = 0;
#pragma unroll
  for (int s = 0; s < ILP; ++s)
#pragma unroll
    for (int j = 0; j < I::NC; ++j) {
      typename I::CT v = c[s][j];
      x ^= *reinterpret_cast<uint32_t*>(&v);
    }
  const int w = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  if ((threadIdx.x & 31) == 0) {
    cycles[w] = t1 - t0;
    ns[w] = (long long)(g1 - g0);
  }
  if (x == 0x9E3779B9u) sink[0] = x;   // practically never; keeps the chains alive
}

template <class I>
tcx_status launch_probe_mma(int ilp, int grid, int warps, int iters, long long* cyc, long long* ns, uint32_t* sink,
                            uint32_t aval, uint32_t meta) {
  switch (ilp) {
#define CASE(n) case n: probe_mma_kernel<I, n><<<grid, warps * 32>>>(iters, cyc, ns, sink, aval, meta); break;
    CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8)
#undef CASE
    default: return set_error(TCX_ERR_UNSUPPORTED, "tcx_probe: mma.sync ILP must be 1..8");
  }
  TCX_CUDA_TRY(cudaGetLastError());
  count_launch();
  return TCX_OK;
}

// ------------------------------------------------------------------ tcgen05 probe
// The paper's method re-cast for the asynchronous, single-thread-issued tcgen05.mma
// (SURVEY §8(a6)): one elected thread per issuing CTA (pair) is the "warp"; up to two issuing CTAs
// share an SM (`issuers`, each with 512 / issuers TMEM columns) — the analogue of #warps per SM;
// ILP = MMAs issued per iteration, rotating over n_acc independent accumulators (n_acc = 1: one
// dependent chain into one accumulator, the GEMM mainloop pattern).  Modes:
//   SYNC    every iteration ends with tcgen05.commit -> mbarrier wait (the paper's per-iteration
//           sync); ILP 1 gives the completion latency (MMA + commit round trip)
//   STREAM  ITERS x ILP MMAs back to back, one commit + wait at the end: the pipe's issue-limited rate
//   COMMIT  ITERS x (commit -> wait) with no MMA: the commit round trip alone (latency split)
// Operands (optional) are copied from global into the 128B-swizzled smem tiles the MMAs read; the
// accumulators of one issuer (the first active one to finish) can be read back (acc_out) so a test can check the MMA count exactly.
// issuers = 2 launches two CTAs per SM on every SM (the smem request caps residency at two); %smid of
// every CTA is recorded so the co-residency is checked, not assumed.
struct Tc05ProbeArgs {
  int mode, iters, ilp, n_acc, acc_cols, alloc_cols, a_bytes, b_bytes, n_rows;
  uint32_t idesc;
  const uint8_t* a_op;
  const uint8_t* b_op;
  long long* cycles;
  long long* ns;
  int* smid_out;
  uint32_t* acc_out;
  int* claim;        // the first active issuer to finish writes acc_out (zeroed per launch)
  long long* g0;     // per issuer: %globaltimer at the start / end of the timed region
  long long* g1;
};
constexpr int TC05_WARMUP = 2;
constexpr int TC05_META_COLS = 8;
constexpr int TC05_STAGES = 4;                  // rotating modes: stage buffers of A (16 KiB) + B (32 KiB)
constexpr int TC05_STAGE_BYTES = 16384 + 32768;

template <int CG, int KIND, bool SPARSE>
__global__ void __launch_bounds__(128, 1)
probe_tc05_kernel(const Tc05ProbeArgs p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sa = smem;                 // 128 rows x 128 B (SW128) per stage
  uint8_t* sb = smem + 16384;         // up to 256 rows x 128 B (SW128) per stage
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base_s;
  const int warp = threadIdx.x / 32;
  const uint32_t rank = CG == 2 ? cluster_ctarank() : 0;
  if (threadIdx.x == 0) {
    int sm; asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
    p.smid_out[blockIdx.x] = sm;                  // co-residency (issuers per SM) is checked, not assumed
  }
  // operands: this CTA's A rows (rank * 128 ..) and B rows (rank * n_rows ..), SW128 placement.  The
  // rotating modes read TC05_STAGES stage buffers at every k-offset of the 128-byte row (like a GEMM
  // ring): each row's operand bytes are replicated into every slot, so every MMA still computes the
  // same A.B and the accumulator check holds
  const bool rot = p.mode >= 3;
  const int nst = rot ? TC05_STAGES : 1;
  for (int i = threadIdx.x; i < nst * TC05_STAGE_BYTES / 16; i += blockDim.x) ((uint4*)smem)[i] = make_uint4(0, 0, 0, 0);
  __syncthreads();
  for (int st = 0; st < nst; ++st) {
    uint8_t* sa_s = sa + st * TC05_STAGE_BYTES;
    uint8_t* sb_s = sb + st * TC05_STAGE_BYTES;
    if (p.a_op) {
      const int ch = p.a_bytes / 16, rep = rot ? 128 / p.a_bytes : 1;
      for (int i = threadIdx.x; i < 128 * ch * rep; i += blockDim.x) {
        const int r = i / (ch * rep), c = i % (ch * rep);
        *(uint4*)(sa_s + r * 128 + ((c ^ (r % 8)) * 16)) =
            *(const uint4*)(p.a_op + ((int64_t)rank * 128 + r) * p.a_bytes + (c % ch) * 16);
      }
    }
    if (p.b_op) {
      const int ch = p.b_bytes / 16, rep = rot ? 128 / p.b_bytes : 1;
      for (int i = threadIdx.x; i < p.n_rows * ch * rep; i += blockDim.x) {
        const int r = i / (ch * rep), c = i % (ch * rep);
        *(uint4*)(sb_s + r * 128 + ((c ^ (r % 8)) * 16)) =
            *(const uint4*)(p.b_op + ((int64_t)rank * p.n_rows + r) * p.b_bytes + (c % ch) * 16);
      }
    }
  }
  fence_proxy_async_smem();
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (warp == 0) {
    if (p.alloc_cols == 512) tmem_alloc<CG>(&tmem_base_s, 512); else tmem_alloc<CG>(&tmem_base_s, 256);
    tmem_relinquish<CG>();
  }
  tc05_fence_before();
  if constexpr (CG == 2) cluster_sync(); else __syncthreads();
  tc05_fence_after();
  const uint32_t tbase = tmem_base_s;
  const uint32_t tmeta = tbase + p.alloc_cols - TC05_META_COLS;
  if constexpr (SPARSE) {
    // metadata: every 4-group keeps positions (0, 1) (nibble 0x4) in the metadata columns of every
    // lane (TF32: the first element of every aligned pair)
    uint32_t r8[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r8[j] = 0x44444444u;
    tmem_st_32x32b_x8(tmeta + ((uint32_t)(warp * 32) << 16), r8);
    tmem_st_wait();
  }
  tc05_fence_before();
  if constexpr (CG == 2) cluster_sync(); else __syncthreads();
  tc05_fence_after();
  // the issuer: warp 0 of the leader CTA runs the loop converged (warp-uniform addresses live in
  // uniform registers) and one elected lane issues each iteration's MMAs, as the GEMMs' MMA warp does
  if (rank == 0 && warp == 0) {
    const uint64_t ad = sdesc(smem_u32(sa), 16, 1024, 2);
    const uint64_t bd = sdesc(smem_u32(sb), 16, 1024, 2);
    const int ilp = p.ilp, n_acc = p.n_acc;
    const uint32_t acc_step = (uint32_t)p.acc_cols;
    uint32_t phase = 0;
    // rotating modes: MMA slot -> (stage, k-offset) of the operand ring.  The descriptors are
    // advanced incrementally (start-address field in 16-byte units) so the issue loop stays a few
    // uniform-register adds per MMA, as in a GEMM mainloop
    const uint32_t a_adv = (uint32_t)p.a_bytes >> 4, b_adv = (uint32_t)p.b_bytes >> 4;
    const int a_steps = 128 / p.a_bytes, b_steps = 128 / p.b_bytes;
    constexpr uint32_t STAGE_ADV = TC05_STAGE_BYTES >> 4;
    int j = 0, jb = 0, stg = 0;
    uint64_t ra = ad, rb = bd;                       // current slot's descriptors
    auto advance = [&]() {
      if (++jb == b_steps) jb = 0;
      if (++j == a_steps) { j = 0; jb = 0; if (++stg == TC05_STAGES) stg = 0; }
      ra = ad + (uint64_t)(stg * STAGE_ADV + j * a_adv);
      rb = bd + (uint64_t)(stg * STAGE_ADV + jb * b_adv);
    };
    auto mma_iter = [&](uint32_t first) {
      if (elect_one()) {
        uint32_t d = tbase;
        int a = 0;
        if (p.mode == 4) {
          // pairs sharing A through the collector: (acc 0, A fill, B of slot s), (acc 1, A lastuse,
          // B of slot s + 1) — the N-wide tile's pattern; n_acc = 2
          for (int i = 0; i + 1 < ilp; i += 2) {
            const uint64_t a_d = ra, b0 = rb;
            advance();
            const uint64_t b1 = rb;
            advance();
            const uint32_t acc = first && i == 0 ? 0u : 1u;
            if constexpr (SPARSE) {
              umma_sp_c<CG, KIND, COLL_FILL>(tbase, a_d, b0, tmeta, p.idesc, acc);
              umma_sp_c<CG, KIND, COLL_LASTUSE>(tbase + acc_step, a_d, b1, tmeta, p.idesc, acc);
            } else {
              umma_c<CG, KIND, COLL_FILL>(tbase, a_d, b0, p.idesc, acc);
              umma_c<CG, KIND, COLL_LASTUSE>(tbase + acc_step, a_d, b1, p.idesc, acc);
            }
          }
        } else {
          for (int i = 0; i < ilp; ++i) {
            const uint32_t acc = (first && i < n_acc) ? 0u : 1u;   // first use of an accumulator: D = A.B
            const uint64_t a_d = p.mode == 3 ? ra : ad, b_d = p.mode == 3 ? rb : bd;
            if (p.mode == 3) advance();
            if constexpr (SPARSE) umma_sp<CG, KIND>(d, a_d, b_d, tmeta, p.idesc, acc);
            else umma<CG, KIND>(d, a_d, b_d, p.idesc, acc);
            d += acc_step;
            if (++a == n_acc) { a = 0; d = tbase; }
          }
        }
      }
      __syncwarp();
    };
    auto commit_wait = [&]() {
      if (elect_one()) {
        if constexpr (CG == 1)
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(smem_u32(&bar)) : "memory");
        else
          asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                       :: "r"(smem_u32(&bar)), "h"((uint16_t)1) : "memory");
      }
      __syncwarp();
      mbar_wait(&bar, phase);
      phase ^= 1;
      tc05_fence_after();
    };
    const bool mmas = p.mode != 2;
    const bool stream = p.mode == 1 || p.mode >= 3;
    for (int it = 0; it < TC05_WARMUP; ++it) {
      if (mmas) mma_iter(it == 0);
      commit_wait();
    }
    const long long t0 = clock64();
    const uint64_t g0 = globaltimer();
    if (stream) {
      for (int it = 0; it < p.iters; ++it) mma_iter(0);
      commit_wait();
    } else {
      for (int it = 0; it < p.iters; ++it) {
        if (mmas) mma_iter(0);
        commit_wait();
      }
    }
    const long long t1 = clock64();
    const uint64_t g1 = globaltimer();
    if (threadIdx.x == 0) {
      p.cycles[blockIdx.x / CG] = t1 - t0;
      p.ns[blockIdx.x / CG] = (long long)(g1 - g0);
      p.g0[blockIdx.x / CG] = (long long)g0;
      p.g1[blockIdx.x / CG] = (long long)g1;
    }
  }
  __shared__ int writer_s;
  if (threadIdx.x == 0 && rank == 0) {
    const int w = p.acc_out ? (atomicCAS(p.claim, 0, 1) == 0) : 0;
    writer_s = w;
    if constexpr (CG == 2) asm volatile("st.shared::cluster.u32 [%0], %1;" :: "r"(mapa(smem_u32(&writer_s), 1)), "r"(w) : "memory");
  }
  tc05_fence_before();
  if constexpr (CG == 2) cluster_sync(); else __syncthreads();
  tc05_fence_after();
  if (writer_s) {
    // issuer 0's accumulators: acc_out[a][rank * 128 + lane row][col], 32-bit words
    const int lane = threadIdx.x & 31;
    const int row = (int)rank * 128 + warp * 32 + lane;
    const int rows = 128 * CG;
    for (int a = 0; a < p.n_acc; ++a)
      for (int c0 = 0; c0 < p.acc_cols; c0 += 16) {
        uint32_t v[16];
        tmem_ld_32x32b_x16(tbase + a * p.acc_cols + c0 + ((uint32_t)(warp * 32) << 16), v);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 16; ++j) p.acc_out[((int64_t)a * rows + row) * p.acc_cols + c0 + j] = v[j];
      }
  }
  tc05_fence_before();
  if constexpr (CG == 2) cluster_sync(); else __syncthreads();
  if (warp == 0) {
    tc05_fence_after();
    if (p.alloc_cols == 512) tmem_dealloc<CG>(tbase, 512); else tmem_dealloc<CG>(tbase, 256);
  }
}

template <int CG, int KIND, bool SPARSE>
tcx_status launch_probe_tc05(int grid_ctas, int issuers, const Tc05ProbeArgs& a) {
  auto kern = probe_tc05_kernel<CG, KIND, SPARSE>;
  // 49 KiB of operands; two issuers per SM: request enough smem that at most two CTAs fit an SM
  const int smem = a.mode >= 3 ? TC05_STAGES * TC05_STAGE_BYTES + 1024 : issuers == 2 ? 100 * 1024 : TC05_STAGE_BYTES + 1024;
  TCX_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid_ctas);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CG; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr; cfg.numAttrs = 1;
  TCX_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, a));
  count_launch();
  return TCX_OK;
}

// device scratch freed on every exit path (the probe returns early on errors)
struct DevBuf {
  void* p = nullptr;
  ~DevBuf() { if (p) cudaFree(p); }
  cudaError_t alloc(size_t n) { return cudaMalloc(&p, n); }
};

double median(std::vector<double> v) {
  std::sort(v.begin(), v.end());
  if (v.empty()) return 0;
  return v.size() % 2 ? v[v.size() / 2] : 0.5 * (v[v.size() / 2 - 1] + v[v.size() / 2]);
}

// ------------------------------------------------------------------ numeric-probe tiles via tcgen05
// 8 tiles per MMA: A (128 x K) = 8 stacked 16 x K tiles; B (64 x K) = 8 concatenated 8 x K tiles;
// D (128 x 64) initialised in TMEM with C_t on the diagonal blocks (rows 16t.., cols 8t..) and
// zeros elsewhere; only the diagonal blocks are read back.  One CTA of 128 threads per group.
template <int KIND, int KT>   // KIND_F16 (f16/bf16, KT = 16) or KIND_TF32 (KT = 8 or 16)
__global__ void __launch_bounds__(128, 1)
tiles_tc05_kernel(const uint8_t* __restrict__ A, const uint8_t* __restrict__ B, const float* __restrict__ C,
                  float* __restrict__ D, int64_t count, uint32_t idesc) {
  constexpr int ES = KIND == KIND_F16 ? 2 : 4;
  constexpr int ROWB = KT * ES;              // bytes of K per row (32 or 64)
  __shared__ __align__(1024) uint8_t sa[128 * 128];
  __shared__ __align__(1024) uint8_t sb[64 * 128];
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base_s;
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  const int r = threadIdx.x;                 // TMEM lane / A row
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (warp == 0) { tmem_alloc<1>(&tmem_base_s, 64); tmem_relinquish<1>(); }
  for (int i = threadIdx.x; i < 128 * 128 / 16; i += 128) ((uint4*)sa)[i] = make_uint4(0, 0, 0, 0);
  for (int i = threadIdx.x; i < 64 * 128 / 16; i += 128) ((uint4*)sb)[i] = make_uint4(0, 0, 0, 0);
  tc05_fence_before();
  __syncthreads();
  tc05_fence_after();
  const uint32_t tbase = tmem_base_s;
  uint32_t phase = 0;
  const int64_t groups = (count + 7) / 8;
  for (int64_t g = blockIdx.x; g < groups; g += gridDim.x) {
    const int t = r / 16;                    // tile within the group owned by this row
    const int64_t tile = g * 8 + t;
    const bool valid = tile < count;
    // A row r = row (r % 16) of tile t; 128B-swizzled placement (16-byte chunk c -> c ^ (r % 8))
    for (int c = 0; c < ROWB / 16; ++c) {
      uint4 v = valid ? *(const uint4*)(A + ((tile * 16 + (r % 16)) * KT) * ES + c * 16) : make_uint4(0, 0, 0, 0);
      *(uint4*)(sa + r * 128 + ((c ^ (r % 8)) * 16)) = v;
    }
    if (r < 64) {                            // B row r = n-row (r % 8) of tile r / 8
      const int64_t bt = g * 8 + r / 8;
      for (int c = 0; c < ROWB / 16; ++c) {
        uint4 v = bt < count ? *(const uint4*)(B + ((bt * 8 + (r % 8)) * KT) * ES + c * 16) : make_uint4(0, 0, 0, 0);
        *(uint4*)(sb + r * 128 + ((c ^ (r % 8)) * 16)) = v;
      }
    }
    // C preload: row r gets C_t[r % 16][0..7] in columns 8t..8t+7, zeros elsewhere (64 columns)
    for (int cb = 0; cb < 8; ++cb) {
      uint32_t v8[8];
#pragma unroll
      for (int j = 0; j < 8; ++j)
        v8[j] = (cb == t && valid && C) ? __float_as_uint(C[(tile * 16 + (r % 16)) * 8 + j]) : 0u;
      tmem_st_32x32b_x8(tbase + cb * 8 + ((uint32_t)(warp * 32) << 16), v8);
    }
    tmem_st_wait();
    fence_proxy_async_smem();
    tc05_fence_before();
    __syncthreads();
    tc05_fence_after();
    if (threadIdx.x == 0) {
#pragma unroll
      for (int k = 0; k < ROWB / 32; ++k)
        umma<1, KIND>(tbase, sdesc(smem_u32(sa) + k * 32, 16, 1024, 2), sdesc(smem_u32(sb) + k * 32, 16, 1024, 2), idesc, 1u);
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(smem_u32(&bar)) : "memory");
    }
    mbar_wait(&bar, phase);
    phase ^= 1;
    tc05_fence_after();
    // warp w holds rows 32w..32w+31 = tiles 2w and 2w+1 -> columns 16w .. 16w+15
    uint32_t v[16];
    tmem_ld_32x32b_x16(tbase + warp * 16 + ((uint32_t)(warp * 32) << 16), v);
    tmem_ld_wait();
    if (valid) {
      const int off = (t & 1) * 8;
      float* Dr = D + (tile * 16 + (r % 16)) * 8;
#pragma unroll
      for (int j = 0; j < 8; ++j) Dr[j] = __uint_as_float(v[off + j]);
    }
    tc05_fence_before();
    __syncthreads();                          // smem / TMEM reuse by the next group
    tc05_fence_after();
    (void)lane;
  }
  tc05_fence_before();
  __syncthreads();
  if (warp == 0) { tc05_fence_after(); tmem_dealloc<1>(tbase, 64); }
}

}  // namespace

tcx_status launch_tiles_tc05(tcx_dtype ab, int k, int64_t count, const void* A, const void* B, const void* C, void* D,
                             cudaStream_t s) {
  const int64_t groups = (count + 7) / 8;
  const int grid = (int)std::min<int64_t>(groups, 148 * 4);
  // idesc: F32 accum, M = 128, N = 64, K-major
  if (ab == TCX_F16 || ab == TCX_BF16) {
    const uint32_t f = ab == TCX_BF16 ? 1u : 0u;
    const uint32_t idesc = (1u << 4) | (f << 7) | (f << 10) | ((64u >> 3) << 17) | ((128u >> 4) << 24);
    tiles_tc05_kernel<KIND_F16, 16><<<grid, 128, 0, s>>>((const uint8_t*)A, (const uint8_t*)B, (const float*)C, (float*)D,
                                                         count, idesc);
  } else {
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((64u >> 3) << 17) | ((128u >> 4) << 24);
    if (k == 8)
      tiles_tc05_kernel<KIND_TF32, 8><<<grid, 128, 0, s>>>((const uint8_t*)A, (const uint8_t*)B, (const float*)C, (float*)D,
                                                           count, idesc);
    else
      tiles_tc05_kernel<KIND_TF32, 16><<<grid, 128, 0, s>>>((const uint8_t*)A, (const uint8_t*)B, (const float*)C, (float*)D,
                                                            count, idesc);
  }
  TCX_CUDA_TRY(cudaGetLastError());
  count_launch();
  return TCX_OK;
}

tcx_status run_probe(const DevInfo& dev, const tcx_probe_config* cfg, tcx_probe_result* out) {
  *out = tcx_probe_result{};
  const int iters = cfg->iters > 0 ? cfg->iters : 1024;
  const int reps = cfg->repeats > 0 ? cfg->repeats : 5;
  const int nsm = cfg->num_sms > 0 ? std::min(cfg->num_sms, dev.sm_count) : 1;
  const int ilp = cfg->ilp > 0 ? cfg->ilp : 1;
  const int nslots = 148 * 32;
  DevBuf b_cyc, b_ns, b_sink;
  TCX_CUDA_TRY(b_cyc.alloc(nslots * sizeof(long long)));
  TCX_CUDA_TRY(b_ns.alloc(nslots * sizeof(long long)));
  TCX_CUDA_TRY(b_sink.alloc(16));
  long long* d_cyc = (long long*)b_cyc.p;
  long long* d_ns = (long long*)b_ns.p;
  uint32_t* d_sink = (uint32_t*)b_sink.p;
  std::vector<double> per_iter, per_ns;
  tcx_status st = TCX_OK;
  double issuers_per_sm = 1, mnk = 0;
  const int ab = cfg->ab, cd = cfg->cd, m = cfg->m, n = cfg->n, k = cfg->k;

  if (cfg->kind == TCX_PROBE_MMA_SYNC || cfg->kind == TCX_PROBE_MMA_SP_SYNC) {
    const int warps = cfg->warps > 0 ? cfg->warps : 1;
    if (warps > 32) { st = set_error(TCX_ERR_INVALID_VALUE, "tcx_probe: warps <= 32"); goto done; }
    issuers_per_sm = warps;
    mnk = (double)m * n * k;
    const bool sp = cfg->kind == TCX_PROBE_MMA_SP_SYNC;
    // operand bit patterns: 1.0 (f16 / bf16 / tf32) or 0x01 bytes (s8)
    uint32_t aval = 0x3C003C00u;
    if (ab == TCX_BF16) aval = 0x3F803F80u;
    if (ab == TCX_TF32) aval = 0x3F800000u;
    if (ab == TCX_S8) aval = 0x01010101u;
    const uint32_t meta = 0x44444444u;
    for (int rep = 0; rep < reps && st == TCX_OK; ++rep) {
#define P(T) st = launch_probe_mma<T>(ilp, nsm, warps, iters, d_cyc, d_ns, d_sink, aval, meta)
      if (!sp) {
        if ((ab == TCX_F16) && cd == TCX_F32 && m == 16 && n == 8 && k == 16) P(F16F32_16816);
        else if (ab == TCX_F16 && cd == TCX_F32 && m == 16 && n == 8 && k == 8) P(F16F32_1688);
        else if (ab == TCX_F16 && cd == TCX_F16 && m == 16 && n == 8 && k == 16) P(F16F16_16816);
        else if (ab == TCX_F16 && cd == TCX_F16 && m == 16 && n == 8 && k == 8) P(F16F16_1688);
        else if (ab == TCX_BF16 && cd == TCX_F32 && m == 16 && n == 8 && k == 16) P(BF16F32_16816);
        else if (ab == TCX_BF16 && cd == TCX_F32 && m == 16 && n == 8 && k == 8) P(BF16F32_1688);
        else if (ab == TCX_TF32 && m == 16 && n == 8 && k == 8) P(TF32_1688);
        else if (ab == TCX_TF32 && m == 16 && n == 8 && k == 4) P(TF32_1684);
        else if (ab == TCX_S8 && m == 8 && n == 8 && k == 16) P(S8_8816);
        else if (ab == TCX_S8 && m == 16 && n == 8 && k == 32) P(S8_16832);
        else if (ab == TCX_S8 && m == 16 && n == 8 && k == 16) P(S8_16816);
        else st = set_error(TCX_ERR_UNSUPPORTED, "tcx_probe: mma.sync shape not in the paper's table");
      } else {
        if (ab == TCX_F16 && m == 16 && n == 8 && k == 32) P(SP_F16_16832);
        else if (ab == TCX_F16 && m == 16 && n == 8 && k == 16) P(SP_F16_16816);
        else if (ab == TCX_BF16 && m == 16 && n == 8 && k == 32) P(SP_BF16_16832);
        else if (ab == TCX_BF16 && m == 16 && n == 8 && k == 16) P(SP_BF16_16816);
        else if (ab == TCX_TF32 && m == 16 && n == 8 && k == 16) P(SP_TF32_16816);
        else if (ab == TCX_TF32 && m == 16 && n == 8 && k == 8) P(SP_TF32_1688);
        else if (ab == TCX_S8 && m == 16 && n == 8 && k == 64) P(SP_S8_16864);
        else if (ab == TCX_S8 && m == 16 && n == 8 && k == 32) P(SP_S8_16832);
        else st = set_error(TCX_ERR_UNSUPPORTED, "tcx_probe: mma.sp shape not in the paper's table");
      }
#undef P
      if (st != TCX_OK) break;
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { st = set_error(TCX_ERR_CUDA, "probe kernel: %s", cudaGetErrorString(e)); break; }
      std::vector<long long> cyc(nsm * warps), nsv(nsm * warps);
      cudaMemcpy(cyc.data(), d_cyc, cyc.size() * sizeof(long long), cudaMemcpyDeviceToHost);
      cudaMemcpy(nsv.data(), d_ns, nsv.size() * sizeof(long long), cudaMemcpyDeviceToHost);
      // per CTA: the slowest warp sets the iteration time; across CTAs: median
      std::vector<double> cta_c, cta_n;
      for (int b = 0; b < nsm; ++b) {
        long long mc = 0, mn = 0;
        for (int w = 0; w < warps; ++w) { mc = std::max(mc, cyc[b * warps + w]); mn = std::max(mn, nsv[b * warps + w]); }
        cta_c.push_back((double)mc); cta_n.push_back((double)mn);
      }
      per_iter.push_back(median(cta_c) / iters);
      per_ns.push_back(median(cta_n) / iters);
    }
  } else if (cfg->kind == TCX_PROBE_TC05 || cfg->kind == TCX_PROBE_TC05_SP) {
    const bool sp = cfg->kind == TCX_PROBE_TC05_SP;
    const int cg = cfg->cta_group == 2 ? 2 : 1;
    const int issuers = cfg->issuers > 0 ? cfg->issuers : 1;
    const int mode = cfg->mode;
    int kind;
    uint32_t fmt;
    const int kbytes = sp ? 64 : 32;           // logical K bytes of one MMA (B operand row bytes)
    if (ab == TCX_F16 || ab == TCX_BF16) { kind = KIND_F16; fmt = ab == TCX_BF16 ? 1 : 0; }
    else if (ab == TCX_TF32) { kind = KIND_TF32; fmt = 2; }
    else if (ab == TCX_S8) { kind = KIND_I8; fmt = 1; }
    else { st = set_error(TCX_ERR_UNSUPPORTED, "tcx_probe: tcgen05 kind"); goto done; }
    const int esz = ab == TCX_S8 ? 1 : (ab == TCX_TF32 ? 4 : 2);
    const int kexp = kbytes / esz;
    if (k != kexp) { st = set_error(TCX_ERR_UNSUPPORTED, "tcx_probe: tcgen05 K must be %d for this kind", kexp); goto done; }
    if (issuers != 1 && issuers != 2) { st = set_error(TCX_ERR_INVALID_VALUE, "tcx_probe: issuers must be 1 or 2"); goto done; }
    if (mode < 0 || mode > 4) { st = set_error(TCX_ERR_INVALID_VALUE, "tcx_probe: tcgen05 mode must be 0 .. 4"); goto done; }
    if (mode >= 3 && issuers != 1) { st = set_error(TCX_ERR_UNSUPPORTED, "tcx_probe: rotating modes need issuers = 1"); goto done; }
    if (mode == 4 && (cfg->n_acc != 2 || ilp % 2)) {
      st = set_error(TCX_ERR_INVALID_VALUE, "tcx_probe: STREAM_AREUSE needs n_acc = 2 and an even ILP"); goto done;
    }
    const bool mok = cg == 1 ? (m == 64 || m == 128) : (m == 128 || m == 256);
    const bool nok = n >= 16 && n <= 256 && n % 16 == 0;
    if (!mok || !nok) { st = set_error(TCX_ERR_UNSUPPORTED, "tcx_probe: tcgen05 M/N"); goto done; }
    const int alloc_cols = 512 / issuers;
    const int avail = alloc_cols - (sp ? TC05_META_COLS : 0);
    const int max_acc = avail / n;
    if (max_acc < 1) { st = set_error(TCX_ERR_UNSUPPORTED, "tcx_probe: N = %d does not fit %d TMEM columns", n, avail); goto done; }
    const int n_acc = cfg->n_acc > 0 ? cfg->n_acc : std::min(ilp, max_acc);
    if (n_acc > max_acc || n_acc > ilp) {
      st = set_error(TCX_ERR_INVALID_VALUE, "tcx_probe: n_acc %d must be <= ilp (%d) and <= %d", n_acc, ilp, max_acc); goto done;
    }
    if ((cfg->acc_out || cfg->a_op || cfg->b_op) && m != 128 * cg) {
      st = set_error(TCX_ERR_UNSUPPORTED, "tcx_probe: operands / acc_out need M = 128 per CTA"); goto done;
    }
    const uint32_t cfmt = ab == TCX_S8 ? 2u : 1u;
    const uint32_t idesc = (sp ? (1u << 2) : 0u) | (cfmt << 4) | (fmt << 7) | (fmt << 10) | ((uint32_t)(n >> 3) << 17) |
                           ((uint32_t)(m >> 4) << 24);
    // issuers = 1: num_sms CTAs (pairs), one per SM; issuers = 2: two CTAs on every SM of the chip
    // (the smem request caps residency at two; num_sms is not used — which SM a CTA lands on cannot
    // be chosen, and gating by %smid lets the scheduler refill vacated SMs)
    const int grid = issuers == 1 ? std::max(1, nsm / cg) * cg : dev.sm_count * 2;
    const int nclusters = grid / cg;
    DevBuf b_smid, b_t;
    TCX_CUDA_TRY(b_smid.alloc((grid + 1) * sizeof(int)));
    TCX_CUDA_TRY(b_t.alloc(4 * nclusters * sizeof(long long)));   // cycles, ns, g0, g1 per issuer
    int* d_smid = (int*)b_smid.p;
    long long* d_t = (long long*)b_t.p;
    Tc05ProbeArgs pa{mode, iters, ilp, n_acc, n, alloc_cols, 32, kbytes, n / cg, idesc,
                     (const uint8_t*)cfg->a_op, (const uint8_t*)cfg->b_op, d_t, d_t + nclusters,
                     d_smid, (uint32_t*)cfg->acc_out, d_smid + grid, d_t + 2 * nclusters, d_t + 3 * nclusters};
    std::vector<int> smid(grid);
    std::vector<double> rate;               // FMA per clk per SM over the union of the issuers' timed regions
    int used = 0, mx = 0;
    for (int rep = 0; rep < reps && st == TCX_OK; ++rep) {
      TCX_CUDA_TRY(cudaMemset(pa.cycles, 0xff, nclusters * sizeof(long long)));
      TCX_CUDA_TRY(cudaMemset(pa.claim, 0, sizeof(int)));
#define T(CGV, KV, SPV) st = launch_probe_tc05<CGV, KV, SPV>(grid, issuers, pa)
      if (cg == 1) {
        if (kind == KIND_F16) { if (sp) T(1, KIND_F16, true); else T(1, KIND_F16, false); }
        else if (kind == KIND_TF32) { if (sp) T(1, KIND_TF32, true); else T(1, KIND_TF32, false); }
        else { if (sp) T(1, KIND_I8, true); else T(1, KIND_I8, false); }
      } else {
        if (kind == KIND_F16) { if (sp) T(2, KIND_F16, true); else T(2, KIND_F16, false); }
        else if (kind == KIND_TF32) { if (sp) T(2, KIND_TF32, true); else T(2, KIND_TF32, false); }
        else { if (sp) T(2, KIND_I8, true); else T(2, KIND_I8, false); }
      }
#undef T
      if (st != TCX_OK) break;
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { st = set_error(TCX_ERR_CUDA, "probe kernel: %s", cudaGetErrorString(e)); break; }
      std::vector<long long> t(4 * nclusters);
      cudaMemcpy(t.data(), d_t, t.size() * sizeof(long long), cudaMemcpyDeviceToHost);
      cudaMemcpy(smid.data(), d_smid, grid * sizeof(int), cudaMemcpyDeviceToHost);
      std::vector<double> c2, n2, ghz;
      long long gmin = 0, gmax = 0;
      int active = 0;
      for (int c = 0; c < nclusters; ++c) {
        if (t[c] < 0) continue;                                 // gated issuer
        c2.push_back((double)t[c]); n2.push_back((double)t[nclusters + c]);
        if (t[nclusters + c] > 0) ghz.push_back((double)t[c] / (double)t[nclusters + c]);
        const long long a = t[2 * nclusters + c], b = t[3 * nclusters + c];
        if (active++ == 0) { gmin = a; gmax = b; } else { gmin = std::min(gmin, a); gmax = std::max(gmax, b); }
      }
      // latency: the median issuer's cycles per iteration (the paper's per-warp clock counters)
      per_iter.push_back(median(c2) / iters);
      per_ns.push_back(median(n2) / iters);
      std::vector<int> per_sm(4096, 0);
      used = 0; mx = 0;
      for (int c = 0; c < grid; ++c)
        if (smid[c] >= 0 && smid[c] < 4096) { if (per_sm[smid[c]]++ == 0) ++used; mx = std::max(mx, per_sm[smid[c]]); }
      // throughput: every active issuer's MMAs over the union of their timed regions (global timer,
      // converted with the measured SM clock), per SM used
      const double span_cyc = (double)(gmax - gmin) * median(ghz);
      if (used > 0 && span_cyc > 0)
        rate.push_back((double)active * iters * (mode == 2 ? 0 : ilp) * m * n * k / ((double)used * span_cyc));
    }
    if (st == TCX_OK) {
      out->sms_used = used;
      out->max_issuers_per_sm = mx;
      out->mmas_per_issuer = mode == 2 ? 0 : (int64_t)iters * ilp;
      out->warmup_iters = TC05_WARMUP;
      out->n_acc = n_acc;
    }
    if (st == TCX_OK && !per_iter.empty()) {
      const double med = median(per_iter);
      out->cycles_per_iter_min = *std::min_element(per_iter.begin(), per_iter.end());
      out->cycles_per_iter_median = med;
      out->latency_cycles = med;
      out->ns_per_iter = median(per_ns);
      out->sm_mhz = out->ns_per_iter > 0 ? med / out->ns_per_iter * 1000.0 : 0;
      out->fma_per_clk_per_sm = rate.empty() ? 0.0 : median(rate);
      out->iters = iters;
    }
    goto done;
  } else if (cfg->kind == TCX_PROBE_LDMATRIX || cfg->kind == TCX_PROBE_LDSHARED || cfg->kind == TCX_PROBE_TMEM_LD ||
             cfg->kind == TCX_PROBE_TMA_LOAD || cfg->kind == TCX_PROBE_TC05_CP ||
             cfg->kind == TCX_PROBE_TMA_MULTICAST || cfg->kind == TCX_PROBE_DSMEM) {
    st = run_probe_mem(dev, cfg, out);
    goto done;
  } else {
    st = set_error(TCX_ERR_INVALID_VALUE, "tcx_probe: unknown kind %d", cfg->kind);
  }

  if (st == TCX_OK && !per_iter.empty()) {
    const double med = median(per_iter);
    out->cycles_per_iter_min = *std::min_element(per_iter.begin(), per_iter.end());
    out->cycles_per_iter_median = med;
    out->latency_cycles = med;
    const double nsi = median(per_ns);
    out->ns_per_iter = nsi;
    out->sm_mhz = nsi > 0 ? med / nsi * 1000.0 : 0;
    if (cfg->kind == TCX_PROBE_MMA_SYNC || cfg->kind == TCX_PROBE_MMA_SP_SYNC)
      out->fma_per_clk_per_sm = issuers_per_sm * ilp * mnk / med;
    else
      out->fma_per_clk_per_sm = issuers_per_sm * mnk / med;
    out->iters = iters;
    uint32_t sink = 0;
    cudaMemcpy(&sink, d_sink, 4, cudaMemcpyDeviceToHost);
    out->sink = sink;
  }
done:
  return st;
}

}  // namespace tcx

// ------------------------------------------------------------------ SM clock stamps (tcx_sm_clock_stamp)
namespace tcx {
namespace {
__global__ void sm_clock_stamp_kernel(long long* out, int max_sms) {
  int sm; asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
  const long long c = clock64();
  const uint64_t g = globaltimer();
  if (sm < max_sms) {
    // one record per SM; a second CTA on the same SM overwrites it with its own consistent pair
    out[2 * sm] = c;
    out[2 * sm + 1] = (long long)g;
  }
}
}  // namespace

tcx_status launch_sm_clock_stamp(long long* out, int max_sms, int sm_count, cudaStream_t s) {
  sm_clock_stamp_kernel<<<sm_count, 32, 0, s>>>(out, max_sms);
  TCX_CUDA_TRY(cudaGetLastError());
  return TCX_OK;
}
}  // namespace tcx
