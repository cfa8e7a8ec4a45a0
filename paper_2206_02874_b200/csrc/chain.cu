// tcx_mma_chain: the paper's chain matrix multiplication (§VIII-B, Fig.
// code-chain-matmul): for each chain, D_1 = A_1 x B_1, and for i > 1  A_i = cvt(D_{i-1}),
// D_i = A_i x B_i, with m16n8k8 MMAs ("we choose mma instructions with shape m16b8k8", read as
// m16n8k8, DESIGN.md R-C6) — A_i is 16 x 8, B_i is 8 x 8 ("col": stored n x k), D_i is 16 x 8 FP32.
// cvt = round-to-nearest-even of the FP32 result into the input format (FP16 overflow -> inf,
// the range loss the paper reports for FP16 at N >= 10).
//
// One warp per chain; A_i never leaves registers: for f16/bf16 the D fragment of m16n8k8
// (rows g, g+8; cols 2t, 2t+1) IS the A fragment of the next MMA (rows g, g+8; k 2t, 2t+1), so the
// conversion is a register-local cvt.rn.{f16,bf16}x2.f32.  For tf32 the A fragment holds
// (g, t), (g+8, t), (g, t+4), (g+8, t+4): gathered from the quad with warp shuffles.
// Every D_i is written (count x n_steps x 16 x 8 FP32) so each step can be checked.
#include "tcx_internal.h"

namespace tcx {
namespace {

constexpr int WARPS = 8;

__device__ __forceinline__ uint32_t tf32_rne(float x) {   // FP32 -> TF32, RNE (DESIGN.md R-C1)
  uint32_t u = __float_as_uint(x);
  if ((u & 0x7F800000u) == 0x7F800000u) return u;        // inf / nan unchanged
  u += 0xFFFu + ((u >> 13) & 1u);
  return u & 0xFFFFE000u;
}

template <int AB>   // 0 f16, 1 bf16, 2 tf32
__device__ __forceinline__ void mma_k8(float (&d)[4], const uint32_t* a, const uint32_t* b) {
  if constexpr (AB == 0)
    asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                 : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3]) : "r"(a[0]), "r"(a[1]), "r"(b[0]));
  else if constexpr (AB == 1)
    asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                 : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3]) : "r"(a[0]), "r"(a[1]), "r"(b[0]));
  else
    asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                 : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
                 : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

template <int AB>
__global__ void __launch_bounds__(WARPS * 32) chain_kernel(const void* __restrict__ A0, const void* __restrict__ Bs,
                                                            float* __restrict__ Ds, int n_steps, int64_t count) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int64_t chain = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (chain >= count) return;
  uint32_t a[4];
  if constexpr (AB == 2) {           // tf32: A 16 x 8 fp32 words
    const uint32_t* At = (const uint32_t*)A0 + chain * 128;
    a[0] = __ldg(At + g * 8 + t); a[1] = __ldg(At + (g + 8) * 8 + t);
    a[2] = __ldg(At + g * 8 + t + 4); a[3] = __ldg(At + (g + 8) * 8 + t + 4);
  } else {                           // 16-bit: A 16 x 8 = 4 words per row
    const uint32_t* At = (const uint32_t*)A0 + chain * 64;
    a[0] = __ldg(At + g * 4 + t); a[1] = __ldg(At + (g + 8) * 4 + t);
  }
  for (int i = 0; i < n_steps; ++i) {
    uint32_t b[2];
    if constexpr (AB == 2) {
      const uint32_t* Bt = (const uint32_t*)Bs + (chain * n_steps + i) * 64;     // 8 x 8 fp32
      b[0] = __ldg(Bt + g * 8 + t); b[1] = __ldg(Bt + g * 8 + t + 4);
    } else {
      const uint32_t* Bt = (const uint32_t*)Bs + (chain * n_steps + i) * 32;     // 8 x 8 16-bit
      b[0] = __ldg(Bt + g * 4 + t);
    }
    float d[4] = {0.f, 0.f, 0.f, 0.f};
    mma_k8<AB>(d, a, b);
    float* Dt = Ds + (chain * n_steps + i) * 128;
    *(float2*)(Dt + g * 8 + 2 * t) = make_float2(d[0], d[1]);
    *(float2*)(Dt + (g + 8) * 8 + 2 * t) = make_float2(d[2], d[3]);
    // A_{i+1} = cvt(D_i)
    if constexpr (AB == 0) {
      asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(a[0]) : "f"(d[1]), "f"(d[0]));
      asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(a[1]) : "f"(d[3]), "f"(d[2]));
    } else if constexpr (AB == 1) {
      asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(a[0]) : "f"(d[1]), "f"(d[0]));
      asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(a[1]) : "f"(d[3]), "f"(d[2]));
    } else {
      // element (row, col c) of D sits in lane 4*(row%8) + c/2, slot c%2 (+2 for row + 8)
      const int src0 = (lane & ~3) | (t >> 1), src1 = (lane & ~3) | (2 + (t >> 1));
      const float x0 = __shfl_sync(0xffffffffu, d[0], src0), x1 = __shfl_sync(0xffffffffu, d[1], src0);
      const float y0 = __shfl_sync(0xffffffffu, d[2], src0), y1 = __shfl_sync(0xffffffffu, d[3], src0);
      const float u0 = __shfl_sync(0xffffffffu, d[0], src1), u1 = __shfl_sync(0xffffffffu, d[1], src1);
      const float v0 = __shfl_sync(0xffffffffu, d[2], src1), v1 = __shfl_sync(0xffffffffu, d[3], src1);
      const bool odd = t & 1;
      a[0] = tf32_rne(odd ? x1 : x0);    // (g, t)
      a[1] = tf32_rne(odd ? y1 : y0);    // (g + 8, t)
      a[2] = tf32_rne(odd ? u1 : u0);    // (g, t + 4)
      a[3] = tf32_rne(odd ? v1 : v0);    // (g + 8, t + 4)
    }
  }
}

}  // namespace

tcx_status launch_chain(tcx_dtype ab, int n_steps, int64_t count, const void* A0, const void* Bs, float* Ds,
                        cudaStream_t s) {
  const int64_t blocks64 = (count + WARPS - 1) / WARPS;
  const unsigned blocks = (unsigned)blocks64;
  switch (ab) {
    case TCX_F16: chain_kernel<0><<<blocks, WARPS * 32, 0, s>>>(A0, Bs, Ds, n_steps, count); break;
    case TCX_BF16: chain_kernel<1><<<blocks, WARPS * 32, 0, s>>>(A0, Bs, Ds, n_steps, count); break;
    case TCX_TF32: chain_kernel<2><<<blocks, WARPS * 32, 0, s>>>(A0, Bs, Ds, n_steps, count); break;
    default: return set_error(TCX_ERR_UNSUPPORTED, "tcx_mma_chain: ab %d", (int)ab);
  }
  TCX_CUDA_TRY(cudaGetLastError());
  count_launch();
  return TCX_OK;
}

}  // namespace tcx
