// Scratch experiment (not part of libtcx): how does tcgen05.mma kind::f16 with an F16 accumulator
// (idesc c_format = 0) lay D out in tensor memory, and how is a tcgen05.st-preloaded C read?
// One CTA, M = 128, N = 16, K = 16.  A[m][k] = (k == m % 16), B[n][k] = n + 1 + 16*k (so D[m][n] =
// B[n][m % 16] = n + 1 + 16*(m%16)), C preload = 0.5 (f16 0x3800) in the low half, 0 high half.
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>
#include "../../paper_2206_02874_b200/csrc/ptx.cuh"
using namespace tcx;

__global__ void k(uint32_t* out, int preload, uint32_t preload_word) {
  __shared__ __align__(1024) uint8_t sa[128 * 128];
  __shared__ __align__(1024) uint8_t sb[16 * 128];
  __shared__ uint64_t bar;
  __shared__ uint32_t tb;
  const int r = threadIdx.x, warp = r / 32;
  if (r == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (warp == 0) { tmem_alloc<1>(&tb, 32); tmem_relinquish<1>(); }
  // A: 128 rows x 16 f16 (32 B used of a 128 B SW128 row); swizzle 16B chunk c -> c ^ (r % 8)
  for (int c = 0; c < 8; ++c) {
    __half h[8];
    for (int j = 0; j < 8; ++j) { int kk = c * 8 + j; h[j] = __float2half(kk < 16 && kk == r % 16 ? 1.f : 0.f); }
    *(uint4*)(sa + r * 128 + ((c ^ (r % 8)) * 16)) = *(uint4*)h;
  }
  if (r < 16) {
    for (int c = 0; c < 8; ++c) {
      __half h[8];
      for (int j = 0; j < 8; ++j) { int kk = c * 8 + j; h[j] = __float2half(kk < 16 ? (float)(r + 1 + 16 * kk) : 0.f); }
      *(uint4*)(sb + r * 128 + ((c ^ (r % 8)) * 16)) = *(uint4*)h;
    }
  }
  tc05_fence_before();
  __syncthreads();
  tc05_fence_after();
  const uint32_t tbase = tb;
  if (preload) {
    uint32_t v8[8];
    for (int j = 0; j < 8; ++j) v8[j] = preload_word;
    tmem_st_32x32b_x8(tbase + ((uint32_t)(warp * 32) << 16), v8);
    tmem_st_32x32b_x8(tbase + 8 + ((uint32_t)(warp * 32) << 16), v8);
    tmem_st_32x32b_x8(tbase + 16 + ((uint32_t)(warp * 32) << 16), v8);
    tmem_st_32x32b_x8(tbase + 24 + ((uint32_t)(warp * 32) << 16), v8);
    tmem_st_wait();
  }
  fence_proxy_async_smem();
  tc05_fence_before();
  __syncthreads();
  tc05_fence_after();
  if (r == 0) {
    // idesc: c_format F16 = 0 at [4,6), a/b f16 = 0, N>>3 at 17, M>>4 at 24
    const uint32_t idesc = (0u << 4) | ((16u >> 3) << 17) | ((128u >> 4) << 24);
    umma<1, KIND_F16>(tbase, sdesc(smem_u32(sa), 16, 1024, 2), sdesc(smem_u32(sb), 16, 1024, 2), idesc, preload ? 1u : 0u);
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(smem_u32(&bar)) : "memory");
  }
  mbar_wait(&bar, 0);
  tc05_fence_after();
  uint32_t v[32];
  tmem_ld_32x32b_x32(tbase + ((uint32_t)(warp * 32) << 16), v);
  tmem_ld_wait();
  for (int j = 0; j < 32; ++j) out[r * 32 + j] = v[j];
  tc05_fence_before();
  __syncthreads();
  if (warp == 0) { tc05_fence_after(); tmem_dealloc<1>(tbase, 32); }
}

int main() {
  uint32_t* d; cudaMalloc(&d, 128 * 32 * 4);
  uint32_t h[128 * 32];
  for (int pre = 0; pre < 3; ++pre) {
    uint32_t word = pre == 1 ? 0x00003800u : 0x38003800u;
    cudaMemset(d, 0xAB, 128 * 32 * 4);
    k<<<1, 128>>>(d, pre > 0, word);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("== preload %d word %08x\n", pre, pre ? word : 0);
    for (int r : {0, 1, 5, 17, 64, 127}) {
      printf("row %3d:", r);
      for (int j = 0; j < 20; ++j) printf(" %08x", h[r * 32 + j]);
      printf("\n");
    }
  }
  return 0;
}
