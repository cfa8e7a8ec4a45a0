// tcx 2:4 operand preparation ("programmers need to first compress the sparse
// matrix A into the non-zeros matrix (denoted as sA) with the index metadata"), and TF32 rounding.
//
// Canonical metadata: u32 words, K/32 per row; group g = nibble at bits 4*(g%8) of word g/8,
// nibble = i0 | i1 << 2, i0 < i1 (include/tcx.h).
//
// Hardware metadata image (tcx_sp24_pack_meta) for kind::f16 tcgen05.mma.sp: per 128-row x
// 128-logical-K block a 2048-byte atom, atoms ordered [row block][k block].  One 128x128b
// tcgen05.cp moves an atom to tensor memory; lane L = (m % 8) + 8*k1 + 16*(m / 16) of column j
// then holds, for MMA j (logical k 32j .. 32j+31 of the block), 16 bits for row m with m/8 even
// and 16 bits for row m + 8, k1 selecting the half [32j + 16*k1, +16).  In 16-bit units:
//     u16 index = (m % 8)*8 + ((m / 8) % 2) + (m / 16)*128 + k1*64 + 2*j
// and each 16-bit unit is exactly one half of a canonical word (4 nibbles, lowest group first).
// Verified bit-exactly on B200 by the one-hot layout probes in tests/test_gpu_sparse.py.
//
// kind::tf32 (hardware 1:2 sparsity): the kind::f16 image over K_f16 = 2K (sp24_pack_tf32_kernel).
//
// Hardware metadata image for kind::i8 (2:4 on bytes, logical K = 64 per tcgen05.mma.sp): tensor
// lane = row and each 32-bit column holds one canonical word (32 logical K; nibble g at bits 4g),
// an MMA reading 2 consecutive columns.  Image: per 128-row x 128-logical-K block a 2048-byte atom
// (row r: the 4 canonical words of the block, 16 bytes), atoms ordered [row block][k block]; one
// 128x128b tcgen05.cp moves an atom (4 columns).  Same verification (one-hot probes, bit-exact
// integer GEMMs in tests/test_gpu_sparse_i8.py).
#include "tcx_internal.h"

namespace tcx {
namespace {

template <int ES>
__device__ __forceinline__ bool nz(const uint8_t* p) {
  if constexpr (ES == 1) return *(const int8_t*)p != 0;
  else if constexpr (ES == 2) return ((*(const uint16_t*)p) & 0x7FFFu) != 0;
  else return ((*(const uint32_t*)p) & 0x7FFFFFFFu) != 0;
}

// one thread per (row, word): 8 groups of 4 = 32 dense elements.
// PAIR (TF32, hardware 1:2 sparsity; DESIGN.md R-C12): each aligned pair keeps its nonzero (or,
// if both are zero, its lower element); a pair with two nonzeros is a violation.
template <int ES, bool PAIR = false>
__global__ void sp24_compress_kernel(int64_t M, int64_t K, const uint8_t* __restrict__ A, int64_t lda,
                                     uint8_t* __restrict__ vals, uint32_t* __restrict__ meta,
                                     unsigned long long* __restrict__ bad) {
  const int64_t W = K / 32;
  const int64_t G = K / 4;
  int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (id >= M * W) return;
  const int64_t r = id / W, w = id % W;
  const uint8_t* src = A + (r * lda + w * 32) * ES;
  uint8_t* dst = vals + (r * (K / 2) + w * 16) * ES;
  uint32_t word = 0;
#pragma unroll
  for (int gi = 0; gi < 8; ++gi) {
    int i0, i1;
    if constexpr (PAIR) {
      const bool z0 = nz<ES>(src + (gi * 4) * ES), z1 = nz<ES>(src + (gi * 4 + 1) * ES);
      const bool z2 = nz<ES>(src + (gi * 4 + 2) * ES), z3 = nz<ES>(src + (gi * 4 + 3) * ES);
      if ((z0 && z1) || (z2 && z3)) atomicMin(bad, (unsigned long long)(r * G + w * 8 + gi));
      i0 = (z1 && !z0) ? 1 : 0;
      i1 = (z3 && !z2) ? 3 : 2;
    } else {
      int idx[4]; int n = 0;
#pragma unroll
      for (int p = 0; p < 4; ++p) if (nz<ES>(src + (gi * 4 + p) * ES)) { if (n < 4) idx[n] = p; ++n; }
      if (n > 2) {
        atomicMin(bad, (unsigned long long)(r * G + w * 8 + gi));
        n = 2; // keep going deterministically; output is discarded by the caller
      }
      // pad with the lowest free indices
      for (int p = 0; p < 4 && n < 2; ++p) {
        bool used = false;
        for (int q = 0; q < n; ++q) used |= (idx[q] == p);
        if (!used) idx[n++] = p;
      }
      i0 = idx[0] < idx[1] ? idx[0] : idx[1];
      i1 = idx[0] < idx[1] ? idx[1] : idx[0];
    }
#pragma unroll
    for (int b = 0; b < ES; ++b) {
      dst[(gi * 2) * ES + b] = src[(gi * 4 + i0) * ES + b];
      dst[(gi * 2 + 1) * ES + b] = src[(gi * 4 + i1) * ES + b];
    }
    word |= (uint32_t)(i0 | (i1 << 2)) << (4 * gi);
  }
  meta[r * W + w] = word;
}

// place canonical kind::f16 word w (logical K 32w .. 32w+31) of row r into the image (K = image K)
__device__ __forceinline__ void put_f16_word(uint16_t* hw, int64_t K, int64_t r, int64_t w, uint32_t word) {
  const int64_t mb = r / 128, m = r % 128;
  const int64_t kb = w / 4, j = w % 4;
  uint16_t* atom = hw + (mb * (K / 128) + kb) * 1024;
  const int64_t base = (m % 8) * 8 + ((m / 8) % 2) + (m / 16) * 128 + 2 * j;
  atom[base] = (uint16_t)(word & 0xFFFFu);
  atom[base + 64] = (uint16_t)(word >> 16);
}

__global__ void sp24_pack_kernel(int64_t M, int64_t K, const uint32_t* __restrict__ meta, uint16_t* __restrict__ hw,
                                 unsigned long long* __restrict__ bad) {
  const int64_t W = K / 32;
  int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (id >= M * W) return;
  const int64_t r = id / W, w = id % W;
  const uint32_t word = meta[id];
#pragma unroll
  for (int gi = 0; gi < 8; ++gi) {
    uint32_t nib = (word >> (4 * gi)) & 0xFu;
    if ((nib & 3u) >= (nib >> 2)) { atomicMin(bad, (unsigned long long)(r * (K / 4) + w * 8 + gi)); break; }
  }
  put_f16_word(hw, K, r, w, word);
}

// TF32 (kind::tf32 .sp, hardware 1:2): a TF32 element is two 16-bit halves to the tensor core, so
// the metadata is the kind::f16 image over K_f16 = 2K, each kept TF32 element becoming the 16-bit
// nibble that keeps its two halves: pair element 0 -> halves {0,1} = 0x4, element 1 -> {2,3} = 0xE.
// Canonical TF32 nibble (i0 | i1 << 2) must have i0 in {0,1}, i1 in {2,3}, else a violation.
__global__ void sp24_pack_tf32_kernel(int64_t M, int64_t K, const uint32_t* __restrict__ meta, uint16_t* __restrict__ hw,
                                      unsigned long long* __restrict__ bad) {
  const int64_t W = K / 32;
  int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (id >= M * W) return;
  const int64_t r = id / W, w = id % W;
  const uint32_t word = meta[id];
  uint32_t h16[2] = {0u, 0u};
#pragma unroll
  for (int gi = 0; gi < 8; ++gi) {
    const uint32_t nib = (word >> (4 * gi)) & 0xFu, i0 = nib & 3u, i1 = nib >> 2;
    if (i0 > 1u || i1 < 2u) { atomicMin(bad, (unsigned long long)(r * (K / 4) + w * 8 + gi)); break; }
    const uint32_t lo = i0 == 0u ? 0x4u : 0xEu, hi = i1 == 2u ? 0x4u : 0xEu;
    h16[gi / 4] |= (lo | (hi << 4)) << (8 * (gi % 4));
  }
  put_f16_word(hw, 2 * K, r, 2 * w, h16[0]);
  put_f16_word(hw, 2 * K, r, 2 * w + 1, h16[1]);
}

__global__ void sp24_pack_i8_kernel(int64_t M, int64_t K, const uint32_t* __restrict__ meta, uint32_t* __restrict__ hw,
                                    unsigned long long* __restrict__ bad) {
  const int64_t W = K / 32;
  int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (id >= M * W) return;
  const int64_t r = id / W, w = id % W;
  const uint32_t word = meta[id];
#pragma unroll
  for (int gi = 0; gi < 8; ++gi) {
    uint32_t nib = (word >> (4 * gi)) & 0xFu;
    if ((nib & 3u) >= (nib >> 2)) { atomicMin(bad, (unsigned long long)(r * (K / 4) + w * 8 + gi)); break; }
  }
  const int64_t mb = r / 128, m = r % 128;
  const int64_t kb = w / 4, j = w % 4;
  hw[(mb * (K / 128) + kb) * 512 + m * 4 + j] = word;
}

__global__ void bad_init_kernel(unsigned long long* bad) { *bad = ~0ull; }
__global__ void bad_final_kernel(unsigned long long* bad, int64_t G) {
  unsigned long long v = *bad;
  int64_t* out = (int64_t*)bad;
  if (v == ~0ull) { out[0] = -1; out[1] = -1; }
  else { out[0] = (int64_t)(v / (unsigned long long)G); out[1] = (int64_t)(v % (unsigned long long)G); }
}

__global__ void round_tf32_kernel(const uint32_t* __restrict__ in, uint32_t* __restrict__ out, int64_t n) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (; i < n; i += stride) {
    uint32_t u = in[i];
    if ((u & 0x7F800000u) != 0x7F800000u) u = (u + 0xFFFu + ((u >> 13) & 1u)) & 0xFFFFE000u;
    out[i] = u;
  }
}

int blocks_for(int64_t n, int tpb) {
  int64_t b = (n + tpb - 1) / tpb;
  return (int)(b < 1 ? 1 : (b > (1ll << 30) ? (1ll << 30) : b));
}

}  // namespace

tcx_status launch_sp24_compress(int esize, bool pair, int64_t M, int64_t K, const void* A, int64_t lda,
                                void* vals, uint32_t* meta, int64_t* d_bad, cudaStream_t s) {
  unsigned long long* bad = (unsigned long long*)d_bad;
  bad_init_kernel<<<1, 1, 0, s>>>(bad);
  const int64_t n = M * (K / 32);
  if (n > 0) {
    const int b = blocks_for(n, 256);
    if (esize == 2) sp24_compress_kernel<2><<<b, 256, 0, s>>>(M, K, (const uint8_t*)A, lda, (uint8_t*)vals, meta, bad);
    else if (esize == 1) sp24_compress_kernel<1><<<b, 256, 0, s>>>(M, K, (const uint8_t*)A, lda, (uint8_t*)vals, meta, bad);
    else if (pair) sp24_compress_kernel<4, true><<<b, 256, 0, s>>>(M, K, (const uint8_t*)A, lda, (uint8_t*)vals, meta, bad);
    else sp24_compress_kernel<4><<<b, 256, 0, s>>>(M, K, (const uint8_t*)A, lda, (uint8_t*)vals, meta, bad);
  }
  bad_final_kernel<<<1, 1, 0, s>>>(bad, K / 4 > 0 ? K / 4 : 1);
  TCX_CUDA_TRY(cudaGetLastError());
  count_launch(n > 0 ? 3 : 2);
  return TCX_OK;
}

tcx_status launch_sp24_pack(tcx_dtype ab, int64_t M, int64_t K, const uint32_t* meta, void* hw, int64_t* d_bad,
                            cudaStream_t s) {
  unsigned long long* bad = (unsigned long long*)d_bad;
  bad_init_kernel<<<1, 1, 0, s>>>(bad);
  const int64_t n = M * (K / 32);
  if (n > 0) {
    if (ab == TCX_S8) sp24_pack_i8_kernel<<<blocks_for(n, 256), 256, 0, s>>>(M, K, meta, (uint32_t*)hw, bad);
    else if (ab == TCX_TF32) sp24_pack_tf32_kernel<<<blocks_for(n, 256), 256, 0, s>>>(M, K, meta, (uint16_t*)hw, bad);
    else sp24_pack_kernel<<<blocks_for(n, 256), 256, 0, s>>>(M, K, meta, (uint16_t*)hw, bad);
  }
  bad_final_kernel<<<1, 1, 0, s>>>(bad, K / 4 > 0 ? K / 4 : 1);
  TCX_CUDA_TRY(cudaGetLastError());
  count_launch(n > 0 ? 3 : 2);
  return TCX_OK;
}

tcx_status launch_round_tf32(const float* in, float* out, int64_t n, cudaStream_t s) {
  if (n == 0) return TCX_OK;
  int b = blocks_for(n, 256);
  if (b > 148 * 32) b = 148 * 32;
  round_tf32_kernel<<<b, 256, 0, s>>>((const uint32_t*)in, (uint32_t*)out, n);
  TCX_CUDA_TRY(cudaGetLastError());
  count_launch();
  return TCX_OK;
}

}  // namespace tcx
