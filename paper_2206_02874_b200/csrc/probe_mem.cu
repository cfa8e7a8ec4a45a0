// tcx data-movement probes: the paper's §VII microbenchmarks of the step
// BEFORE the MMA re-measured on sm_100a with the same clock-counter method as
// tcx_probe: each warp runs ITERS iterations of ILP independent loads, each slot
// a dependency chain across iterations (the next address depends on the loaded value through a
// runtime mask of 0), with a warp sync per iteration.
//   LDMATRIX  ldmatrix.sync.aligned.m8n8.x{1,2,4}[.trans].shared.b16: N x 128 bytes per warp
//             (Table ldmatrix-ld.shared; Table ldmatrix-summary)
//   LDSHARED  ld.shared.u32 / .u64 with an n-way bank conflict (Table ldshared-latency,
//             PAPER.md:783-793): lane l reads byte offset l * 4 * ways
//   TMEM_LD   B200's staging path out of the tensor core: tcgen05.ld.sync.aligned.32x32b.x{N}
//             (+ tcgen05.wait::ld), 32 lanes x N x 4 bytes per warp — the epilogue's read of the
//             accumulator (not in the paper: B200-specific)
//   TMA_LOAD  the GEMMs' operand staging: ILP cp.async.bulk.tensor.2d boxes (m rows x n bytes) in
//             flight per mbarrier wait, from an L2-resident 16 MiB buffer
//   TC05_CP   the sparse path's metadata staging: ILP tcgen05.cp.128x128b (2 KiB) per commit
// Throughput is bytes/clk/SM.  Also: tcx_ldmatrix_dump, the functional check
// that ldmatrix delivers exactly the fragments its definition names.
#include <algorithm>
#include <vector>
#include "tcx_internal.h"
#include "ptx.cuh"

namespace tcx {
namespace {

__device__ __forceinline__ uint64_t gtimer() {
  uint64_t t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t;
}

template <int N, int TRANS>
__device__ __forceinline__ void ldsm(uint32_t (&r)[4], uint32_t addr) {
  if constexpr (N == 1 && !TRANS) asm volatile("ldmatrix.sync.aligned.m8n8.x1.shared.b16 {%0}, [%1];" : "=r"(r[0]) : "r"(addr));
  if constexpr (N == 2 && !TRANS) asm volatile("ldmatrix.sync.aligned.m8n8.x2.shared.b16 {%0,%1}, [%2];" : "=r"(r[0]), "=r"(r[1]) : "r"(addr));
  if constexpr (N == 4 && !TRANS)
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(addr));
  if constexpr (N == 1 && TRANS) asm volatile("ldmatrix.sync.aligned.m8n8.x1.trans.shared.b16 {%0}, [%1];" : "=r"(r[0]) : "r"(addr));
  if constexpr (N == 2 && TRANS)
    asm volatile("ldmatrix.sync.aligned.m8n8.x2.trans.shared.b16 {%0,%1}, [%2];" : "=r"(r[0]), "=r"(r[1]) : "r"(addr));
  if constexpr (N == 4 && TRANS)
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(addr));
}

constexpr int SMEM_PROBE = 40960;   // 8 ILP slots x up to 4 KiB + slack

// ---------------------------------------------------------------- ldmatrix
template <int N, int TRANS, int ILP>
__global__ void probe_ldsm_kernel(int iters, uint32_t mask, long long* cycles, long long* ns, uint32_t* sink) {
  __shared__ __align__(1024) uint8_t buf[SMEM_PROBE];
  for (int i = threadIdx.x; i < SMEM_PROBE / 16; i += blockDim.x) ((uint4*)buf)[i] = make_uint4(0, 0, 0, 0);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  // slot s: 4 matrices x 8 rows x 16 B = 512 contiguous bytes (conflict-free rows); row address of
  // lane l = matrix l/8, row l%8 (lanes beyond 8N are ignored by the instruction)
  uint32_t addr[ILP];
#pragma unroll
  for (int s = 0; s < ILP; ++s) addr[s] = smem_u32(buf) + s * 512 + lane * 16;
  uint32_t acc = 0;
  uint32_t r[4] = {0, 0, 0, 0};
  long long t0 = 0; uint64_t g0 = 0;
  for (int it = -4; it < iters; ++it) {
#pragma unroll
    for (int s = 0; s < ILP; ++s) {
      ldsm<N, TRANS>(r, addr[s]);
      addr[s] += r[0] & mask;              // the next load depends on this one
      acc ^= r[0];
    }
    __syncwarp();
    if (it == -1) { t0 = clock64(); g0 = gtimer(); }
  }
  const long long t1 = clock64();
  const uint64_t g1 = gtimer();
  if (lane == 0) {
    cycles[blockIdx.x * 32 + threadIdx.x / 32] = t1 - t0;
    ns[blockIdx.x * 32 + threadIdx.x / 32] = (long long)(g1 - g0);
  }
  if (acc == 0x9E3779B9u) sink[0] = acc;
}

// ---------------------------------------------------------------- ld.shared with n-way conflicts
template <int BYTES, int ILP>
__global__ void probe_lds_kernel(int iters, int ways, uint32_t mask, long long* cycles, long long* ns, uint32_t* sink) {
  __shared__ __align__(1024) uint8_t buf[SMEM_PROBE];
  for (int i = threadIdx.x; i < SMEM_PROBE / 16; i += blockDim.x) ((uint4*)buf)[i] = make_uint4(0, 0, 0, 0);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  uint32_t addr[ILP];
#pragma unroll
  for (int s = 0; s < ILP; ++s) addr[s] = smem_u32(buf) + s * 4096 + lane * 4 * ways;
  uint32_t acc = 0;
  long long t0 = 0; uint64_t g0 = 0;
  for (int it = -4; it < iters; ++it) {
#pragma unroll
    for (int s = 0; s < ILP; ++s) {
      uint32_t v;
      if constexpr (BYTES == 4) {
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr[s]));
      } else {
        uint64_t w;
        asm volatile("ld.shared.u64 %0, [%1];" : "=l"(w) : "r"(addr[s]));
        v = (uint32_t)w ^ (uint32_t)(w >> 32);
      }
      addr[s] += v & mask;
      acc ^= v;
    }
    __syncwarp();
    if (it == -1) { t0 = clock64(); g0 = gtimer(); }
  }
  const long long t1 = clock64();
  const uint64_t g1 = gtimer();
  if (lane == 0) {
    cycles[blockIdx.x * 32 + threadIdx.x / 32] = t1 - t0;
    ns[blockIdx.x * 32 + threadIdx.x / 32] = (long long)(g1 - g0);
  }
  if (acc == 0x9E3779B9u) sink[0] = acc;
}

// ---------------------------------------------------------------- tcgen05.ld (TMEM -> registers)
template <int N>
__device__ __forceinline__ uint32_t tmem_ld_n(uint32_t taddr) {
  uint32_t x = 0;
  if constexpr (N == 1) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(x) : "r"(taddr));
  } else if constexpr (N == 2) {
    uint32_t y; asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0,%1}, [%2];" : "=r"(x), "=r"(y) : "r"(taddr)); x ^= y;
  } else if constexpr (N == 4) {
    uint32_t r[4];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(taddr));
    x = r[0] ^ r[1] ^ r[2] ^ r[3];
  } else if constexpr (N == 8) {
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]) : "r"(taddr));
#pragma unroll
    for (int i = 0; i < 8; ++i) x ^= r[i];
  } else if constexpr (N == 16) {
    uint32_t r[16];
    tmem_ld_32x32b_x16(taddr, r);
#pragma unroll
    for (int i = 0; i < 16; ++i) x ^= r[i];
  } else {
    uint32_t r[32];
    tmem_ld_32x32b_x32(taddr, r);
#pragma unroll
    for (int i = 0; i < 32; ++i) x ^= r[i];
  }
  return x;
}

template <int N>
__global__ void __launch_bounds__(512, 1) probe_tmem_ld_kernel(int iters, int ilp, uint32_t mask, long long* cycles,
                                                               long long* ns, uint32_t* sink) {
  __shared__ uint32_t tbase_s;
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  if (warp == 0) { tmem_alloc<1>(&tbase_s, 512); tmem_relinquish<1>(); }
  tc05_fence_before();
  __syncthreads();
  tc05_fence_after();
  const uint32_t lane_base = (uint32_t)((warp % 4) * 32) << 16;    // warp w owns lanes 32(w%4)..
  const uint32_t col0 = (uint32_t)((warp / 4) * 128);              // 4 warp groups x 128 columns
  uint32_t off = 0, acc = 0;
  long long t0 = 0; uint64_t g0 = 0;
  for (int it = -4; it < iters; ++it) {
    for (int s = 0; s < ilp; ++s) acc ^= tmem_ld_n<N>(tbase_s + lane_base + col0 + ((s * N + off) & 127));
    tmem_ld_wait();
    off = acc & mask;                                              // next loads depend on these
    __syncwarp();
    if (it == -1) { t0 = clock64(); g0 = gtimer(); }
  }
  const long long t1 = clock64();
  const uint64_t g1 = gtimer();
  if (lane == 0) {
    cycles[blockIdx.x * 32 + warp] = t1 - t0;
    ns[blockIdx.x * 32 + warp] = (long long)(g1 - g0);
  }
  if (acc == 0x9E3779B9u) sink[0] = acc;
  tc05_fence_before();
  __syncthreads();
  if (warp == 0) { tc05_fence_after(); tmem_dealloc<1>(tbase_s, 512); }
}

// ---------------------------------------------------------------- TMA 2D loads (global -> smem)
// B200's operand staging: one thread issues ILP cp.async.bulk.tensor.2d loads of a
// (box_rows x box_bytes) box into distinct smem slots, then waits on the mbarrier (the iteration's
// sync).  The source is a 16 MiB buffer (L2-resident after the warm-up): L2-hit latency/bandwidth.
__global__ void __launch_bounds__(32, 1) probe_tma_kernel(const __grid_constant__ CUtensorMap tm, int iters, int ilp,
                                                          int box_rows, uint32_t box_bytes, int rows_total,
                                                          long long* cycles, long long* ns) {
  extern __shared__ uint8_t dyn[];
  uint8_t* buf = (uint8_t*)(((uintptr_t)dyn + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  __syncwarp();
  if (threadIdx.x != 0) return;
  uint32_t phase = 0;
  long long t0 = 0; uint64_t g0 = 0;
  int y = (blockIdx.x * 97) % (rows_total - box_rows);
  for (int it = -4; it < iters; ++it) {
    if (it == 0) { t0 = clock64(); g0 = gtimer(); }
    mbar_arrive_expect_tx(&bar, (uint32_t)ilp * box_bytes);
    for (int s = 0; s < ilp; ++s) {
      tma_load_2d(buf + s * box_bytes, &tm, &bar, 0, y);
      y += box_rows;
      if (y + box_rows > rows_total) y = 0;
    }
    mbar_wait(&bar, phase);
    phase ^= 1;
  }
  const long long t1 = clock64();
  const uint64_t g1 = gtimer();
  cycles[blockIdx.x * 32] = t1 - t0;
  ns[blockIdx.x * 32] = (long long)(g1 - g0);
}

// ---------------------------------------------------------------- TMA multicast (clusters)
// every CTA of a cluster needs the same ilp boxes per iteration.  mc: box s is issued once, by the
// CTA of cluster rank s % cs, multicast to all cs CTAs; else every CTA loads every box itself.
// Each CTA's barrier expects ilp boxes either way (delivered bytes per CTA are equal).
__global__ void __launch_bounds__(32, 1) probe_tma_mc_kernel(const __grid_constant__ CUtensorMap tm, int iters, int ilp,
                                                             int box_rows, uint32_t box_bytes, int rows_total, int mc,
                                                             long long* cycles, long long* ns) {
  extern __shared__ uint8_t dyn[];
  uint8_t* buf = (uint8_t*)(((uintptr_t)dyn + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  const uint32_t cs = cluster_nctarank(), r = cluster_ctarank();
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  cluster_sync();                                   // every barrier armed before any multicast lands
  if (threadIdx.x == 0) {
    const uint16_t mask = (uint16_t)((1u << cs) - 1);
    uint32_t phase = 0;
    long long t0 = 0; uint64_t g0 = 0;
    int y = (int)((blockIdx.x / cs) * 97) % (rows_total - box_rows);   // the same boxes per cluster
    for (int it = -4; it < iters; ++it) {
      if (it == 0) { t0 = clock64(); g0 = gtimer(); }
      mbar_arrive_expect_tx(&bar, (uint32_t)ilp * box_bytes);
      for (int s = 0; s < ilp; ++s) {
        if (!mc) tma_load_2d(buf + s * box_bytes, &tm, &bar, 0, y);
        else if ((uint32_t)s % cs == r) tma_load_2d_mc(buf + s * box_bytes, &tm, &bar, 0, y, mask);
        y += box_rows;
        if (y + box_rows > rows_total) y = 0;
      }
      mbar_wait(&bar, phase);
      phase ^= 1;
    }
    const long long t1 = clock64();
    const uint64_t g1 = gtimer();
    cycles[blockIdx.x * 32] = t1 - t0;
    ns[blockIdx.x * 32] = (long long)(g1 - g0);
  }
  cluster_sync();                                   // no CTA leaves while peers still write into it
}

// ---------------------------------------------------------------- distributed shared memory
// SM-to-SM operand forwarding inside a cluster: every CTA bulk-copies ILP boxes of its own shared
// memory into the next CTA's (cp.async.bulk.shared::cluster.shared::cta, complete_tx on the
// destination's mbarrier), waits for its predecessor's boxes, then the cluster syncs (flow
// control).  The payload is pseudo-random (toggling like real operands).  Throughput = bytes
// received per clk per SM — the alternative to re-reading a shared operand from L2.
__global__ void __launch_bounds__(32, 1) probe_dsmem_kernel(int iters, int ilp, uint32_t box_bytes, long long* cycles,
                                                            long long* ns) {
  extern __shared__ uint8_t dyn[];
  uint8_t* base = (uint8_t*)(((uintptr_t)dyn + 127) & ~(uintptr_t)127);
  uint8_t* src = base;
  uint8_t* dst = base + (size_t)ilp * box_bytes;
  __shared__ uint64_t bar;
  const uint32_t cs = cluster_nctarank(), r = cluster_ctarank();
  for (uint32_t i = threadIdx.x; i < ilp * box_bytes / 4; i += 32) {
    uint32_t x = i * 2654435761u + blockIdx.x * 40503u;
    x ^= x >> 15; x *= 0x2c1b3c6dU; x ^= x >> 12;
    ((uint32_t*)src)[i] = x;
  }
  fence_proxy_async_smem();
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  cluster_sync();
  if (threadIdx.x == 0) {
    const uint32_t peer = (r + 1) % cs;
    const uint32_t dst_peer = mapa(smem_u32(dst), peer), bar_peer = mapa(smem_u32(&bar), peer);
    uint32_t phase = 0;
    long long t0 = 0; uint64_t g0 = 0;
    for (int it = -4; it < iters; ++it) {
      if (it == 0) { t0 = clock64(); g0 = gtimer(); }
      mbar_arrive_expect_tx(&bar, (uint32_t)ilp * box_bytes);
      for (int s2 = 0; s2 < ilp; ++s2)
        asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     :: "r"(dst_peer + s2 * box_bytes), "r"(smem_u32(src + s2 * box_bytes)), "r"(box_bytes), "r"(bar_peer)
                     : "memory");
      mbar_wait(&bar, phase);
      phase ^= 1;
      asm volatile("barrier.cluster.arrive.release;\n\tbarrier.cluster.wait.acquire;" ::: "memory");
    }
    const long long t1 = clock64();
    const uint64_t g1 = gtimer();
    cycles[blockIdx.x * 32] = t1 - t0;
    ns[blockIdx.x * 32] = (long long)(g1 - g0);
  } else {
    for (int it = -4; it < iters; ++it) asm volatile("barrier.cluster.arrive.release;\n\tbarrier.cluster.wait.acquire;" ::: "memory");
  }
  cluster_sync();
}

__global__ void fill_random_kernel(uint32_t* p, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint32_t x = (uint32_t)i * 2654435761u + 0x9E3779B9u;
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
    p[i] = x;
  }
}

// ---------------------------------------------------------------- tcgen05.cp (smem -> TMEM)
// the sparse path's metadata staging: ILP tcgen05.cp.cta_group::1.128x128b (2 KiB each) into
// distinct TMEM columns, then tcgen05.commit -> mbarrier wait.
__global__ void __launch_bounds__(128, 1) probe_tc05_cp_kernel(int iters, int ilp, long long* cycles, long long* ns) {
  __shared__ __align__(1024) uint8_t src[16 * 2048];
  __shared__ uint64_t bar;
  __shared__ uint32_t tb;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 16 * 2048 / 16; i += blockDim.x) ((uint4*)src)[i] = make_uint4(i, 0, 0, 0);
  fence_proxy_async_smem();
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (warp == 0) { tmem_alloc<1>(&tb, 512); tmem_relinquish<1>(); }
  tc05_fence_before();
  __syncthreads();
  tc05_fence_after();
  if (threadIdx.x == 0) {
    uint32_t phase = 0;
    long long t0 = 0; uint64_t g0 = 0;
    for (int it = -4; it < iters; ++it) {
      if (it == 0) { t0 = clock64(); g0 = gtimer(); }
      for (int s = 0; s < ilp; ++s)
        tc05_cp_128x128b<1>(tb + (uint32_t)((s * 4) & 511), sdesc(smem_u32(src) + (s & 15) * 2048, 128, 128, 0));
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(smem_u32(&bar)) : "memory");
      mbar_wait(&bar, phase);
      phase ^= 1;
      tc05_fence_after();
    }
    const long long t1 = clock64();
    const uint64_t g1 = gtimer();
    cycles[blockIdx.x * 32] = t1 - t0;
    ns[blockIdx.x * 32] = (long long)(g1 - g0);
  }
  tc05_fence_before();
  __syncthreads();
  if (warp == 0) { tc05_fence_after(); tmem_dealloc<1>(tb, 512); }
}

// ---------------------------------------------------------------- functional ldmatrix dump
// src: 512 b16 elements (4 matrices x 8 rows x 16 B, row-major), row_elem[l] = element offset of
// the row lane l addresses; out[l * N + j] = register j of lane l.
template <int N, int TRANS>
__global__ void ldsm_dump_kernel(const uint16_t* __restrict__ src, const int* __restrict__ row_elem, uint32_t* out) {
  __shared__ __align__(128) uint16_t buf[1024];
  for (int i = threadIdx.x; i < 1024; i += 32) buf[i] = i < 512 ? src[i] : 0;
  __syncwarp();
  uint32_t r[4];
  ldsm<N, TRANS>(r, smem_u32(buf) + 2u * (uint32_t)row_elem[threadIdx.x]);
#pragma unroll
  for (int j = 0; j < N; ++j) out[threadIdx.x * N + j] = r[j];
}

double med(std::vector<double> v) {
  std::sort(v.begin(), v.end());
  if (v.empty()) return 0;
  return v.size() % 2 ? v[v.size() / 2] : 0.5 * (v[v.size() / 2 - 1] + v[v.size() / 2]);
}

}  // namespace

tcx_status launch_ldmatrix_dump(int n, int trans, const void* src, const int* row_elem, uint32_t* out, cudaStream_t s) {
#define D(NN, TT) ldsm_dump_kernel<NN, TT><<<1, 32, 0, s>>>((const uint16_t*)src, row_elem, out)
  if (n == 1) { if (trans) D(1, 1); else D(1, 0); }
  else if (n == 2) { if (trans) D(2, 1); else D(2, 0); }
  else if (n == 4) { if (trans) D(4, 1); else D(4, 0); }
  else return set_error(TCX_ERR_UNSUPPORTED, "tcx_ldmatrix_dump: num must be 1, 2 or 4");
#undef D
  TCX_CUDA_TRY(cudaGetLastError());
  count_launch();
  return TCX_OK;
}

// data-movement kinds of tcx_probe; result throughput (fma_per_clk_per_sm) is bytes/clk/SM here
tcx_status run_probe_mem(const DevInfo& dev, const tcx_probe_config* cfg, tcx_probe_result* out) {
  const int iters = cfg->iters > 0 ? cfg->iters : 1024;
  const int reps = cfg->repeats > 0 ? cfg->repeats : 5;
  const int nsm = cfg->num_sms > 0 ? std::min(cfg->num_sms, dev.sm_count) : 1;
  const int ilp = cfg->ilp > 0 ? cfg->ilp : 1;
  const int warps = cfg->warps > 0 ? cfg->warps : 1;
  if (warps > 32 || ilp > 8) return set_error(TCX_ERR_INVALID_VALUE, "tcx_probe: warps <= 32, ilp <= 8");
  long long *d_cyc = nullptr, *d_ns = nullptr;
  uint32_t* d_sink = nullptr;
  TCX_CUDA_TRY(cudaMalloc(&d_cyc, 148 * 32 * sizeof(long long)));
  TCX_CUDA_TRY(cudaMalloc(&d_ns, 148 * 32 * sizeof(long long)));
  TCX_CUDA_TRY(cudaMalloc(&d_sink, 16));
  tcx_status st = TCX_OK;
  double bytes_per_warp_iter = 0;
  int warps_eff = warps;              // timing slots per CTA (1 for the single-thread TMA / cp probes)
  int launched = nsm;                 // CTAs actually timed (the multicast probe rounds to clusters)
  void* tma_src = nullptr;
  std::vector<double> per_iter, per_ns;
  for (int rep = 0; rep < reps && st == TCX_OK; ++rep) {
    cudaError_t le = cudaSuccess;
    if (cfg->kind == TCX_PROBE_LDMATRIX) {
      const int n = cfg->m, tr = cfg->n ? 1 : 0;
      bytes_per_warp_iter = 128.0 * n * ilp;
#define L(NN, TT, II) probe_ldsm_kernel<NN, TT, II><<<nsm, warps * 32>>>(iters, 0u, d_cyc, d_ns, d_sink)
#define LI(NN, TT) switch (ilp) { case 1: L(NN, TT, 1); break; case 2: L(NN, TT, 2); break; case 3: L(NN, TT, 3); break; \
      case 4: L(NN, TT, 4); break; case 5: L(NN, TT, 5); break; case 6: L(NN, TT, 6); break; case 7: L(NN, TT, 7); break; \
      default: L(NN, TT, 8); }
      if (n == 1) { if (tr) { LI(1, 1) } else { LI(1, 0) } }
      else if (n == 2) { if (tr) { LI(2, 1) } else { LI(2, 0) } }
      else if (n == 4) { if (tr) { LI(4, 1) } else { LI(4, 0) } }
      else { st = set_error(TCX_ERR_UNSUPPORTED, "tcx_probe: ldmatrix .x1/.x2/.x4 (m = 1, 2, 4)"); break; }
#undef LI
#undef L
    } else if (cfg->kind == TCX_PROBE_LDSHARED) {
      const int bytes = cfg->m, ways = cfg->n > 0 ? cfg->n : 1;
      if (!(bytes == 4 || bytes == 8) || ways > 32 || (ways & (ways - 1)) || (bytes == 8 && ways < 2)) {
        st = set_error(TCX_ERR_UNSUPPORTED, "tcx_probe: ld.shared u32 (ways 1..32) / u64 (ways 2..32), power of 2");
        break;
      }
      bytes_per_warp_iter = 32.0 * bytes * ilp;
#define S(BB, II) probe_lds_kernel<BB, II><<<nsm, warps * 32>>>(iters, ways, 0u, d_cyc, d_ns, d_sink)
#define SI(BB) switch (ilp) { case 1: S(BB, 1); break; case 2: S(BB, 2); break; case 3: S(BB, 3); break; \
      case 4: S(BB, 4); break; case 5: S(BB, 5); break; case 6: S(BB, 6); break; case 7: S(BB, 7); break; default: S(BB, 8); }
      if (bytes == 4) { SI(4) } else { SI(8) }
#undef SI
#undef S
    } else if (cfg->kind == TCX_PROBE_TMEM_LD) {
      const int n = cfg->m;
      if (warps > 16) { st = set_error(TCX_ERR_INVALID_VALUE, "tcx_probe: tcgen05.ld warps <= 16"); break; }
      bytes_per_warp_iter = 32.0 * 4 * n * ilp;
#define T(NN) probe_tmem_ld_kernel<NN><<<nsm, warps * 32>>>(iters, ilp, 0u, d_cyc, d_ns, d_sink)
      if (n == 1) T(1); else if (n == 2) T(2); else if (n == 4) T(4); else if (n == 8) T(8);
      else if (n == 16) T(16); else if (n == 32) T(32);
      else { st = set_error(TCX_ERR_UNSUPPORTED, "tcx_probe: tcgen05.ld 32x32b.x{1,2,4,8,16,32}"); break; }
#undef T
    } else if (cfg->kind == TCX_PROBE_TMA_LOAD) {
      // box = m rows x n bytes (n in {16..256}, multiple of 16), u8 tensor of 4096 rows x 4096 B
      const int rows = cfg->m > 0 ? cfg->m : 128, inner = cfg->n > 0 ? cfg->n : 128;
      if (rows > 256 || inner > 256 || inner % 16 || rows * inner * ilp > 200 * 1024) {
        st = set_error(TCX_ERR_UNSUPPORTED, "tcx_probe: TMA box m <= 256 rows, n <= 256 bytes (x16), ilp*box <= 200 KiB");
        break;
      }
      if (!tma_src) {
        if (cudaMalloc(&tma_src, 4096u * 4096u) != cudaSuccess) { st = set_error(TCX_ERR_CUDA, "probe: cudaMalloc"); break; }
        if (cfg->mode & 1) fill_random_kernel<<<592, 256>>>((uint32_t*)tma_src, 4096u * 4096u / 4);
        else cudaMemset(tma_src, 1, 4096u * 4096u);
      }
      CUtensorMap tm;
      st = make_tmap_2d(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, tma_src, 4096, 4096, 4096, (uint32_t)inner, (uint32_t)rows,
                        CU_TENSOR_MAP_SWIZZLE_NONE);
      if (st != TCX_OK) break;
      const int smem = rows * inner * ilp + 1024;
      cudaFuncSetAttribute(probe_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      bytes_per_warp_iter = (double)rows * inner * ilp;
      probe_tma_kernel<<<nsm, 32, smem>>>(tm, iters, ilp, rows, (uint32_t)(rows * inner), 4096, d_cyc, d_ns);
      warps_eff = 1;
    } else if (cfg->kind == TCX_PROBE_TMA_MULTICAST) {
      const int rows = cfg->m > 0 ? cfg->m : 128, inner = cfg->n > 0 ? cfg->n : 128;
      const int cs = cfg->cta_group > 0 ? cfg->cta_group : 1;
      if (rows > 256 || inner > 256 || inner % 16 || rows * inner * ilp > 200 * 1024 || cs > 8 || (cs & (cs - 1)) ||
          (cfg->k && ilp % cs)) {
        st = set_error(TCX_ERR_UNSUPPORTED, "tcx_probe: TMA multicast box m <= 256, n <= 256 (x16), "
                                            "ilp*box <= 200 KiB, cluster 1/2/4/8, ilp %% cluster == 0");
        break;
      }
      if (!tma_src) {
        if (cudaMalloc(&tma_src, 4096u * 4096u) != cudaSuccess) { st = set_error(TCX_ERR_CUDA, "probe: cudaMalloc"); break; }
        if (cfg->mode & 1) fill_random_kernel<<<592, 256>>>((uint32_t*)tma_src, 4096u * 4096u / 4);
        else cudaMemset(tma_src, 1, 4096u * 4096u);
      }
      CUtensorMap tm;
      st = make_tmap_2d(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, tma_src, 4096, 4096, 4096, (uint32_t)inner, (uint32_t)rows,
                        CU_TENSOR_MAP_SWIZZLE_NONE);
      if (st != TCX_OK) break;
      const int smem = rows * inner * ilp + 1024;
      cudaFuncSetAttribute(probe_tma_mc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      cudaLaunchConfig_t lc = {};
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
      lc.blockDim = dim3(32);
      lc.dynamicSmemBytes = smem;
      lc.attrs = at; lc.numAttrs = 1;
      // co-resident clusters only, so every measured CTA loads while all others do
      int ncl = nsm / cs > 0 ? nsm / cs : 1;
      lc.gridDim = dim3((unsigned)(ncl * cs));
      int fit = 0;
      if (cudaOccupancyMaxActiveClusters(&fit, probe_tma_mc_kernel, &lc) == cudaSuccess && fit > 0 && fit < ncl) ncl = fit;
      lc.gridDim = dim3((unsigned)(ncl * cs));
      launched = ncl * cs;
      bytes_per_warp_iter = (double)rows * inner * ilp;
      le = cudaLaunchKernelEx(&lc, probe_tma_mc_kernel, tm, iters, ilp, rows, (uint32_t)(rows * inner), 4096,
                              cfg->k ? 1 : 0, d_cyc, d_ns);
      if (le != cudaSuccess) { st = set_error(TCX_ERR_CUDA, "probe multicast launch: %s", cudaGetErrorString(le)); break; }
      warps_eff = 1;
    } else if (cfg->kind == TCX_PROBE_DSMEM) {
      // cluster of cta_group (2..8) CTAs, ilp boxes of n bytes (multiple of 16) forwarded per iteration
      const int cs = cfg->cta_group >= 2 ? cfg->cta_group : 2;
      const int box = cfg->n > 0 ? cfg->n : 16384;
      if (cs > 8 || box % 16 || 2 * box * ilp > 200 * 1024) {
        st = set_error(TCX_ERR_UNSUPPORTED, "tcx_probe: DSMEM cluster 2..8, n %% 16 == 0, 2*ilp*n <= 200 KiB");
        break;
      }
      const int smem = 2 * box * ilp + 128;
      cudaFuncSetAttribute(probe_dsmem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      cudaLaunchConfig_t lc = {};
      launched = std::max(cs, (nsm / cs) * cs);
      lc.gridDim = dim3(launched);
      lc.blockDim = dim3(32);
      lc.dynamicSmemBytes = smem;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
      lc.attrs = at; lc.numAttrs = 1;
      bytes_per_warp_iter = (double)box * ilp;
      cudaError_t le2 = cudaLaunchKernelEx(&lc, probe_dsmem_kernel, iters, ilp, (uint32_t)box, d_cyc, d_ns);
      if (le2 != cudaSuccess) { st = set_error(TCX_ERR_CUDA, "probe DSMEM launch: %s", cudaGetErrorString(le2)); break; }
      warps_eff = 1;
    } else if (cfg->kind == TCX_PROBE_TC05_CP) {
      bytes_per_warp_iter = 2048.0 * ilp;
      probe_tc05_cp_kernel<<<nsm, 128>>>(iters, ilp, d_cyc, d_ns);
      warps_eff = 1;
    } else {
      st = set_error(TCX_ERR_INVALID_VALUE, "tcx_probe: unknown kind %d", cfg->kind);
      break;
    }
    le = cudaGetLastError();
    if (le == cudaSuccess) le = cudaDeviceSynchronize();
    if (le != cudaSuccess) { st = set_error(TCX_ERR_CUDA, "probe kernel: %s", cudaGetErrorString(le)); break; }
    count_launch();
    std::vector<long long> cyc(nsm * 32), nsv(nsm * 32);
    cudaMemcpy(cyc.data(), d_cyc, cyc.size() * sizeof(long long), cudaMemcpyDeviceToHost);
    cudaMemcpy(nsv.data(), d_ns, nsv.size() * sizeof(long long), cudaMemcpyDeviceToHost);
    std::vector<double> c2, n2;
    for (int b = 0; b < launched; ++b)
      for (int w = 0; w < warps_eff; ++w) { c2.push_back((double)cyc[b * 32 + w]); n2.push_back((double)nsv[b * 32 + w]); }
    per_iter.push_back(*std::max_element(c2.begin(), c2.end()) / iters);   // the slowest warp bounds the SM
    per_ns.push_back(*std::max_element(n2.begin(), n2.end()) / iters);
  }
  if (st == TCX_OK && !per_iter.empty()) {
    const double m = med(per_iter);
    out->cycles_per_iter_min = *std::min_element(per_iter.begin(), per_iter.end());
    out->cycles_per_iter_median = m;
    out->latency_cycles = m;
    const double nsi = med(per_ns);
    out->ns_per_iter = nsi;
    out->sm_mhz = nsi > 0 ? m / nsi * 1000.0 : 0;
    out->fma_per_clk_per_sm = warps_eff * bytes_per_warp_iter / m;      // bytes/clk/SM
    out->iters = iters;
    uint32_t sink = 0;
    cudaMemcpy(&sink, d_sink, 4, cudaMemcpyDeviceToHost);
    out->sink = sink;
  }
  cudaFree(d_cyc);
  cudaFree(d_ns);
  cudaFree(d_sink);
  if (tma_src) cudaFree(tma_src);
  return st;
}

}  // namespace tcx
