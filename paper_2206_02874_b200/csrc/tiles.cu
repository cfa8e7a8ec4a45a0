// tcx_mma_tiles: a batch of independent tiles, ONE tensor-core MMA per tile — the paper's
// own warp-level instruction (mma.sync) at batch scale:
//     D_t = A_t x B_t + C_t   (C_t is the MMA's C operand, as in the probes)
// f16/bf16 m16n8k16 -> HMMA.16816.F32(.BF16); tf32 m16n8k8 (k16 = 2 chained) -> HMMA.1688.F32.TF32;
// s8 m16n8k32 -> IMMA.16832.S8.S8.
// HBM-bound (1792 B per 4096 FLOP tile): each warp streams tiles; the next tile's fragments are
// loaded before the current MMA issues (two tiles in flight per warp).
// Layouts: A_t m x k row-major, B_t n x k (n-major "col"), C_t/D_t m x n row-major.
#include "tcx_internal.h"

namespace tcx {
namespace {

constexpr int WARPS = 8;

template <int AB>  // 0 f16, 1 bf16
__device__ __forceinline__ void mma_16816(float (&d)[4], const uint32_t (&a)[4], const uint32_t (&b)[2]) {
  if constexpr (AB == 0)
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                 : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
                 : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
  else
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                 : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
                 : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}
__device__ __forceinline__ void mma_1688_tf32(float (&d)[4], const uint32_t (&a)[4], const uint32_t (&b)[2]) {
  asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
               : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
               : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}
__device__ __forceinline__ void mma_16832_s8(int (&d)[4], const uint32_t (&a)[4], const uint32_t (&b)[2]) {
  asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
               : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
               : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

// fragment loaders (PTX ISA mma fragment layouts; g = lane/4, t = lane%4)
struct Frag16 {   // f16/bf16 m16n8k16: A 16x16 (2-byte), B 8x16
  uint32_t a[4], b[2];
  uint2 c0, c1;   // C rows g and g+8, cols 2t..2t+1 (fp32 bits)
};
__device__ __forceinline__ void load16(Frag16& f, const uint16_t* A, const uint16_t* B, const float* C, int g, int t) {
  const uint32_t* A32 = (const uint32_t*)A;   // row r, k pair j -> A32[r*8 + j]
  f.a[0] = __ldg(A32 + g * 8 + t);
  f.a[1] = __ldg(A32 + (g + 8) * 8 + t);
  f.a[2] = __ldg(A32 + g * 8 + t + 4);
  f.a[3] = __ldg(A32 + (g + 8) * 8 + t + 4);
  const uint32_t* B32 = (const uint32_t*)B;   // n row g, k pair t
  f.b[0] = __ldg(B32 + g * 8 + t);
  f.b[1] = __ldg(B32 + g * 8 + t + 4);
  if (C) {
    f.c0 = __ldg((const uint2*)(C + g * 8 + 2 * t));
    f.c1 = __ldg((const uint2*)(C + (g + 8) * 8 + 2 * t));
  } else {
    f.c0 = make_uint2(0, 0); f.c1 = make_uint2(0, 0);
  }
}

template <int AB>
__global__ void __launch_bounds__(WARPS * 32) tiles16_kernel(const uint16_t* __restrict__ A, const uint16_t* __restrict__ B,
                                                              const float* __restrict__ C, float* __restrict__ D, int64_t count) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  int64_t tile = warp;
  if (tile >= count) return;
  Frag16 cur;
  load16(cur, A + tile * 256, B + tile * 128, C ? C + tile * 128 : nullptr, g, t);
  while (tile < count) {
    const int64_t nxt = tile + nwarps;
    Frag16 nf;
    if (nxt < count) load16(nf, A + nxt * 256, B + nxt * 128, C ? C + nxt * 128 : nullptr, g, t);
    float d[4] = {__uint_as_float(cur.c0.x), __uint_as_float(cur.c0.y), __uint_as_float(cur.c1.x), __uint_as_float(cur.c1.y)};
    mma_16816<AB>(d, cur.a, cur.b);
    float* Dt = D + tile * 128;
    *(float2*)(Dt + g * 8 + 2 * t) = make_float2(d[0], d[1]);
    *(float2*)(Dt + (g + 8) * 8 + 2 * t) = make_float2(d[2], d[3]);
    tile = nxt;
    if (tile < count) cur = nf;
  }
}

// tf32: A_t 16 x K (K = 8 or 16) fp32, B_t 8 x K; K/8 chained m16n8k8 MMAs (D of one = C of next)
template <int KT>
__global__ void __launch_bounds__(WARPS * 32) tiles_tf32_kernel(const uint32_t* __restrict__ A, const uint32_t* __restrict__ B,
                                                                 const float* __restrict__ C, float* __restrict__ D, int64_t count) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t tile = warp; tile < count; tile += nwarps) {
    const uint32_t* At = A + tile * 16 * KT;
    const uint32_t* Bt = B + tile * 8 * KT;
    float d[4] = {0.f, 0.f, 0.f, 0.f};
    if (C) {
      const float* Ct = C + tile * 128;
      float2 x = __ldg((const float2*)(Ct + g * 8 + 2 * t)), y = __ldg((const float2*)(Ct + (g + 8) * 8 + 2 * t));
      d[0] = x.x; d[1] = x.y; d[2] = y.x; d[3] = y.y;
    }
#pragma unroll
    for (int k0 = 0; k0 < KT; k0 += 8) {
      uint32_t a[4], b[2];
      a[0] = __ldg(At + g * KT + k0 + t);
      a[1] = __ldg(At + (g + 8) * KT + k0 + t);
      a[2] = __ldg(At + g * KT + k0 + t + 4);
      a[3] = __ldg(At + (g + 8) * KT + k0 + t + 4);
      b[0] = __ldg(Bt + g * KT + k0 + t);
      b[1] = __ldg(Bt + g * KT + k0 + t + 4);
      mma_1688_tf32(d, a, b);
    }
    float* Dt = D + tile * 128;
    *(float2*)(Dt + g * 8 + 2 * t) = make_float2(d[0], d[1]);
    *(float2*)(Dt + (g + 8) * 8 + 2 * t) = make_float2(d[2], d[3]);
  }
}

// s8: A_t 16 x 32 int8, B_t 8 x 32, C/D int32 16 x 8
__global__ void __launch_bounds__(WARPS * 32) tiles_s8_kernel(const int8_t* __restrict__ A, const int8_t* __restrict__ B,
                                                               const int* __restrict__ C, int* __restrict__ D, int64_t count) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t tile = warp; tile < count; tile += nwarps) {
    const uint32_t* A32 = (const uint32_t*)(A + tile * 512);   // row r, k quad j -> A32[r*8 + j]
    const uint32_t* B32 = (const uint32_t*)(B + tile * 256);
    uint32_t a[4], b[2];
    a[0] = __ldg(A32 + g * 8 + t);
    a[1] = __ldg(A32 + (g + 8) * 8 + t);
    a[2] = __ldg(A32 + g * 8 + t + 4);
    a[3] = __ldg(A32 + (g + 8) * 8 + t + 4);
    b[0] = __ldg(B32 + g * 8 + t);
    b[1] = __ldg(B32 + g * 8 + t + 4);
    int d[4] = {0, 0, 0, 0};
    if (C) {
      const int* Ct = C + tile * 128;
      int2 x = __ldg((const int2*)(Ct + g * 8 + 2 * t)), y = __ldg((const int2*)(Ct + (g + 8) * 8 + 2 * t));
      d[0] = x.x; d[1] = x.y; d[2] = y.x; d[3] = y.y;
    }
    mma_16832_s8(d, a, b);
    int* Dt = D + tile * 128;
    *(int2*)(Dt + g * 8 + 2 * t) = make_int2(d[0], d[1]);
    *(int2*)(Dt + (g + 8) * 8 + 2 * t) = make_int2(d[2], d[3]);
  }
}

int grid_for(int64_t count) {
  int64_t warps = count;
  int64_t blocks = (warps + WARPS - 1) / WARPS;
  const int64_t cap = 148 * 16;   // persistent-ish: 16 CTAs of 8 warps per SM at most
  return (int)(blocks < cap ? blocks : cap);
}

}  // namespace

tcx_status launch_tiles(tcx_dtype ab, int k, int64_t count, const void* A, const void* B,
                        const void* C, void* D, cudaStream_t s) {
  const int grid = grid_for(count);
  switch (ab) {
    case TCX_F16:
      tiles16_kernel<0><<<grid, WARPS * 32, 0, s>>>((const uint16_t*)A, (const uint16_t*)B, (const float*)C, (float*)D, count);
      break;
    case TCX_BF16:
      tiles16_kernel<1><<<grid, WARPS * 32, 0, s>>>((const uint16_t*)A, (const uint16_t*)B, (const float*)C, (float*)D, count);
      break;
    case TCX_TF32:
      if (k == 8) tiles_tf32_kernel<8><<<grid, WARPS * 32, 0, s>>>((const uint32_t*)A, (const uint32_t*)B, (const float*)C, (float*)D, count);
      else tiles_tf32_kernel<16><<<grid, WARPS * 32, 0, s>>>((const uint32_t*)A, (const uint32_t*)B, (const float*)C, (float*)D, count);
      break;
    case TCX_S8:
      tiles_s8_kernel<<<grid, WARPS * 32, 0, s>>>((const int8_t*)A, (const int8_t*)B, (const int*)C, (int*)D, count);
      break;
    default:
      return set_error(TCX_ERR_UNSUPPORTED, "tcx_mma_tiles: ab %d", (int)ab);
  }
  TCX_CUDA_TRY(cudaGetLastError());
  count_launch();
  return TCX_OK;
}

}  // namespace tcx
