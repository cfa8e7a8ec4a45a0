"""tcx ORACLE — plain, slow, obviously-correct CPU implementation of the hot path.

TEST INFRASTRUCTURE.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The product package
(``paper_2206_02874_b200``) never imports it, and the two share no code: the C sources
here (``tcxref.c``, ``models.c``) are compiled into their own ``libtcxref.so``.

Definitions (cited in the C sources):
  * ``D = A x B + C`` (§II-A); "row.col": A is m x k row-major, B is stored
    n x k.
  * FP16/BF16/TF32 -> FP32: every product exact, the sum exact, ONE RNE rounding to FP32.
  * FP16 -> FP16 (C/D FP16, the mma f16.f16.f16.f16 variant): the same exact
    sum rounded ONCE to FP16.
  * INT8 -> INT32: exact int64 sum, two's-complement wrap to 32 bits.
  * 2:4 sparse: expand(sA, meta) then dense.

Every function is pinned by ``tests/test_oracle_*.py`` against brute-force rational
arithmetic, closed forms, SPEC worked examples and the paper's zero-error cells.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libtcxref.so")
_SRCS = [os.path.join(_HERE, "tcxref.c"), os.path.join(_HERE, "models.c")]

# format ids (oracle-local; deliberately not imported from the product header)
F16, BF16, TF32, F32, S8, S32 = 0, 1, 2, 3, 4, 5
_NP = {F16: np.uint16, BF16: np.uint16, TF32: np.uint32, F32: np.uint32, S8: np.int8, S32: np.int32}


def build(force: bool = False) -> str:
    """Compile libtcxref.so with gcc (-O2, no fast-math, no FMA contraction)."""
    newest = max(os.path.getmtime(s) for s in _SRCS)
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < newest:
        cmd = ["gcc", "-O2", "-std=gnu11", "-fPIC", "-shared", "-ffp-contract=off",
               "-fno-fast-math", "-pthread", "-o", _LIB_PATH] + _SRCS + ["-lm"]
        subprocess.check_call(cmd)
    return _LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB_PATH)
        vp, i64, u32, i32, dbl = ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint32, ctypes.c_int, ctypes.c_double
        L.tcxref_quantize.argtypes = [dbl, i32, i32]; L.tcxref_quantize.restype = u32
        L.tcxref_decode.argtypes = [i32, u32]; L.tcxref_decode.restype = dbl
        L.tcxref_dot_fp.argtypes = [i32, i64, vp, vp, u32, ctypes.POINTER(dbl)]; L.tcxref_dot_fp.restype = u32
        L.tcxref_dot_fp2.argtypes = [i32, i64, vp, vp, i32, u32, i32, i32, ctypes.POINTER(dbl)]
        L.tcxref_dot_fp2.restype = u32
        L.tcxref_dot_s8.argtypes = [i64, vp, vp, ctypes.c_int32]; L.tcxref_dot_s8.restype = ctypes.c_int32
        L.tcxref_sum_round.argtypes = [i32, vp, vp, vp, i32, i32]; L.tcxref_sum_round.restype = u32
        L.tcxref_gemm_samples.argtypes = [i32, i64, vp, i64, vp, i64, vp, i64, i64, vp, vp, vp, vp, i32]
        L.tcxref_gemm_samples.restype = i32
        L.tcxref_gemm_samples2.argtypes = [i32, i32, i64, vp, i64, vp, i64, vp, i64, i64, vp, vp, vp, vp, i32]
        L.tcxref_gemm_samples2.restype = i32
        L.tcxref_sp24_expand.argtypes = [i32, i64, i64, vp, i64, vp, vp, i64]; L.tcxref_sp24_expand.restype = i64
        L.tcxref_sp24_compress.argtypes = [i32, i64, i64, vp, i64, vp, i64, vp]; L.tcxref_sp24_compress.restype = i64
        L.tcxref_sp12_compress.argtypes = [i64, i64, vp, i64, vp, i64, vp]; L.tcxref_sp12_compress.restype = i64
        L.tcxref_tiles.argtypes = [i32, i32, i32, i32, i64, vp, vp, vp, vp, vp]; L.tcxref_tiles.restype = i32
        L.tcxref_tiles2.argtypes = [i32, i32, i32, i32, i32, i64, vp, vp, vp, vp, vp]; L.tcxref_tiles2.restype = i32
        L.tcxref_model_dot.argtypes = [i32, i32, vp, vp, u32, i32, i32, i32, i32, i32, i32]
        L.tcxref_model_dot.restype = u32
        L.tcxref_model_batch.argtypes = [i32, ctypes.c_long, i32, vp, vp, vp, i32, i32, i32, i32, i32, i32, i32, vp, i32]
        L.tcxref_model_batch.restype = i32
        L.tcxref_model_batch2.argtypes = [i32, ctypes.c_long, i32, vp, vp, vp, i32, i32, i32, i32, i32, i32, i32, i32,
                                          vp, i32]
        L.tcxref_model_batch2.restype = i32
        L.tcxref_model_batch3.argtypes = [i32, ctypes.c_long, i32, vp, vp, vp, i32, i32, i32, i32, i32, i32, i32, i32,
                                          i32, vp, i32]
        L.tcxref_model_batch3.restype = i32
        L.tcxref_seq32.argtypes = [i32, vp, vp, ctypes.c_float, i32]; L.tcxref_seq32.restype = ctypes.c_float
        L.tcxref_quantize_f32_bits.argtypes = [i32, i64, vp, vp]; L.tcxref_quantize_f32_bits.restype = None
        L.tcxref_chain_fp32.argtypes = [i64, i32, vp, vp, vp]; L.tcxref_chain_fp32.restype = None
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


# ---------------------------------------------------------------------------- formats
def quantize(x: float, fmt: int, rz: bool = False) -> int:
    """SPEC.md:38-46 quantize(x, fmt, NearestEven|TowardZero) -> stored bits."""
    return int(lib().tcxref_quantize(float(x), fmt, int(rz)))


def decode(fmt: int, bits: int) -> float:
    return float(lib().tcxref_decode(fmt, int(bits) & 0xFFFFFFFF))


def quantize_array(x: np.ndarray, fmt: int) -> np.ndarray:
    L = lib()
    flat = np.asarray(x, dtype=np.float64).ravel()
    out = np.fromiter((L.tcxref_quantize(float(v), fmt, 0) for v in flat), dtype=np.uint32, count=flat.size)
    return out.astype(_NP[fmt]).reshape(np.shape(x))


# ---------------------------------------------------------------------------- dots
def dot_fp(ab: int, a_bits: np.ndarray, b_bits: np.ndarray, c_bits: int = 0, c_fmt: int = F32,
           out_fmt: int = F32, rz: bool = False):
    """One FP output element: R_out(c + sum a_k b_k) computed exactly and rounded once (RNE, or
    toward zero if rz) into out_fmt (FP32, or FP16 for the FP16-accumulate variant); c is given
    in c_fmt.  Returns (bits, sum|ab|+|c|)."""
    a = _c(a_bits, _NP[ab]); b = _c(b_bits, _NP[ab])
    absv = ctypes.c_double(0.0)
    r = lib().tcxref_dot_fp2(ab, a.size, _p(a), _p(b), c_fmt, int(c_bits) & 0xFFFFFFFF, out_fmt, int(rz),
                             ctypes.byref(absv))
    return int(r), absv.value


def dot_s8(a: np.ndarray, b: np.ndarray, c: int = 0) -> int:
    a = _c(a, np.int8); b = _c(b, np.int8)
    return int(lib().tcxref_dot_s8(a.size, _p(a), _p(b), int(c)))


def sum_round(signs, mants, exps, out_fmt=F32, rz=False) -> int:
    s = _c(signs, np.int32); m = _c(mants, np.uint64); e = _c(exps, np.int32)
    return int(lib().tcxref_sum_round(len(s), _p(s), _p(m), _p(e), out_fmt, int(rz)))


def gemm_samples(ab: int, A: np.ndarray, B: np.ndarray, C, rows, cols, nthreads: int | None = None, cd: int = F32):
    """D[rows[s], cols[s]] for A (M x K), B (N x K, 'col'), C (M x N or None).

    Returns (out, abs) where out is uint32 bits (FP32 bits, or int32 bits for S8; cd = F16: C is
    FP16 and out holds RNE_fp16 bits of the exact value) and abs is the float64 bound magnitude
    sum_k|a b| + |c| (FP only)."""
    A = np.ascontiguousarray(A); B = np.ascontiguousarray(B)
    assert A.dtype == _NP[ab] and B.dtype == _NP[ab], (A.dtype, B.dtype)
    M, K = A.shape
    N, K2 = B.shape
    assert K == K2
    rows = _c(rows, np.int64); cols = _c(cols, np.int64)
    n = rows.size
    out = np.zeros(n, dtype=np.uint32)
    absv = np.zeros(n, dtype=np.float64)
    Cc = None
    if C is not None:
        Cc = np.ascontiguousarray(C)
        assert Cc.shape == (M, N) and Cc.itemsize == (2 if cd == F16 else 4)
    nt = nthreads or len(os.sched_getaffinity(0))
    rc = lib().tcxref_gemm_samples2(ab, cd, K, _p(A), K, _p(B), K, _p(Cc) if Cc is not None else None,
                                    N, n, _p(rows), _p(cols), _p(out), _p(absv), nt)
    assert rc == 0
    return out, absv


def gemm_full(ab: int, A, B, C=None, nthreads=None):
    M = A.shape[0]; N = B.shape[0]
    ii, jj = np.meshgrid(np.arange(M), np.arange(N), indexing="ij")
    out, absv = gemm_samples(ab, A, B, C, ii.ravel(), jj.ravel(), nthreads)
    return out.reshape(M, N), absv.reshape(M, N)


def tiles(ab: int, m: int, n: int, k: int, A, B, C, cd: int = F32):
    """Batch of independent tiles: D_t = A_t B_t + C_t (layouts as tcx_mma_tiles).
    cd = F32 (C/D FP32 bits, INT32 for S8) or F16 (C given as uint16 FP16 bits; D returned as
    FP16 bits in uint32, = RNE_fp16 of the exact value)."""
    A = np.ascontiguousarray(A); B = np.ascontiguousarray(B)
    count = A.size // (m * k)
    Cc = np.ascontiguousarray(C) if C is not None else None
    if Cc is not None:
        assert Cc.itemsize == (2 if cd == F16 else 4)
    D = np.zeros(count * m * n, dtype=np.uint32)
    absv = np.zeros(count * m * n, dtype=np.float64)
    lib().tcxref_tiles2(ab, cd, m, n, k, count, _p(A), _p(B), _p(Cc) if Cc is not None else None, _p(D), _p(absv))
    return D.reshape(count, m, n), absv.reshape(count, m, n)


# ---------------------------------------------------------------------------- 2:4 sparse
def sp24_expand(vals: np.ndarray, meta: np.ndarray, K: int) -> np.ndarray:
    vals = np.ascontiguousarray(vals); meta = _c(meta, np.uint32)
    M = vals.shape[0]
    dense = np.zeros((M, K), dtype=vals.dtype)
    bad = lib().tcxref_sp24_expand(vals.itemsize, M, K, _p(vals), vals.shape[1], _p(meta), _p(dense), K)
    if bad >= 0:
        raise ValueError(f"bad metadata nibble at row {bad // (K // 4)}, group {bad % (K // 4)}")
    return dense


def sp24_compress(dense: np.ndarray):
    dense = np.ascontiguousarray(dense)
    M, K = dense.shape
    vals = np.zeros((M, K // 2), dtype=dense.dtype)
    meta = np.zeros((M, K // 32), dtype=np.uint32)
    bad = lib().tcxref_sp24_compress(dense.itemsize, M, K, _p(dense), K, _p(vals), K // 2, _p(meta))
    return vals, meta, int(bad)


def sp12_compress(dense: np.ndarray):
    """TF32 1:2 compress (FP32-container bits, M x K): one kept element per aligned pair; returns
    (vals M x K/2, canonical meta M x K/32, first violation row*G+group or -1)."""
    dense = _c(dense, np.uint32)
    M, K = dense.shape
    vals = np.zeros((M, K // 2), dtype=np.uint32)
    meta = np.zeros((M, K // 32), dtype=np.uint32)
    bad = lib().tcxref_sp12_compress(M, K, _p(dense), K, _p(vals), K // 2, _p(meta))
    return vals, meta, int(bad)


# ---------------------------------------------------------------------------- probe models
def model_dot(ab: int, a_bits, b_bits, c_bits: int, Ki: int, g: int, p: int, rz: bool,
              floor_mode: bool = False, c_after: bool = False) -> int:
    a = _c(a_bits, _NP[ab]); b = _c(b_bits, _NP[ab])
    return int(lib().tcxref_model_dot(ab, a.size, _p(a), _p(b), int(c_bits) & 0xFFFFFFFF, Ki, g, p,
                                      int(rz), int(floor_mode), int(c_after)))


def seq32(a: np.ndarray, b: np.ndarray, c: float, c_last: bool = False) -> float:
    a = _c(a, np.float32); b = _c(b, np.float32)
    return float(lib().tcxref_seq32(a.size, _p(a), _p(b), float(c), int(c_last)))


def model_batch(ab: int, a_rows, b_rows, c_bits, Ki: int, g: int, p: int, rz: bool, floor_mode=False,
                c_after=False, emode=0, nthreads=None, acc_fmt: int = F32, win_fmt: int | None = None) -> np.ndarray:
    """model_dot over n rows at once (n x K element bits for a and b, n FP32 bits for c).
    emode 3: as 2 with the accumulator's exponent read from its exponent field (a subnormal c
    counts as emin, like a subnormal input).
    emode 0: align on the actual leading bit of the largest addend; 1: on exponent sums
    (product nominal leading exponent = e_a + e_b + 1, subnormal inputs at emin).
    acc_fmt: the accumulator's format (c in and D out): FP32, or FP16 for the FP16-accumulate
    variant (truncation window and every block rounding then use FP16's 11-bit significand).
    win_fmt: the format whose significand sets the truncation window (default acc_fmt); FP32 with
    acc_fmt = FP16 aligns like the FP32 datapath and rounds once into FP16."""
    a = _c(a_rows, _NP[ab]); b = _c(b_rows, _NP[ab]); c = _c(c_bits, np.uint32)
    n, K = a.shape
    out = np.zeros(n, dtype=np.uint32)
    nt = nthreads or len(os.sched_getaffinity(0))
    rc = lib().tcxref_model_batch3(ab, n, K, _p(a), _p(b), _p(c), Ki, g, p, int(rz), int(floor_mode), int(c_after),
                                   int(emode), acc_fmt, acc_fmt if win_fmt is None else win_fmt, _p(out), nt)
    assert rc == 0
    return out


# ---------------------------------------------------------------------------- chain matmul
def quantize_f32_bits(bits32: np.ndarray, fmt: int) -> np.ndarray:
    """FP32 bits -> fmt bits (RNE), elementwise: the chain's D_{i-1} -> A_i conversion."""
    x = _c(bits32, np.uint32)
    out = np.zeros(x.size, dtype=np.uint32)
    lib().tcxref_quantize_f32_bits(fmt, x.size, _p(x), _p(out))
    return out.astype(_NP[fmt] if fmt != S8 else np.uint32).reshape(np.shape(bits32))


def chain_fp32(A0: np.ndarray, Bs: np.ndarray) -> np.ndarray:
    """The paper's CPU FP32 chain: A0 (count,16,8) float32, Bs
    (count,n_steps,8,8) float32 stored n x k; returns every D_i (count,n_steps,16,8) float32."""
    A0 = _c(A0, np.float32); Bs = _c(Bs, np.float32)
    count, n_steps = Bs.shape[0], Bs.shape[1]
    Ds = np.zeros((count, n_steps, 16, 8), dtype=np.float32)
    lib().tcxref_chain_fp32(count, n_steps, _p(A0), _p(Bs), _p(Ds))
    return Ds


# ---------------------------------------------------------------------------- ldmatrix (NEXT-3)
def ldmatrix(num: int, trans: bool, smem_u16: np.ndarray, row_elem: np.ndarray) -> np.ndarray:
    """The fragments one warp receives from ldmatrix.sync.aligned.m8n8.x{num}[.trans].shared.b16
    (Fig. func_ldmatrix: "it loads N x 128 bytes per warp ... each thread stores
    N x 4 bytes"; "If N = 4, then every thread will provide a valid p ... (e.g. T0 - T7 for N = 1)").
    Matrix j (j < num) is 8 rows x 8 b16 elements; its row r starts at element row_elem[8j + r].
    Lane l's register j holds two b16 (first in the low half):
      non-trans: M_j[l // 4][2 (l % 4)], M_j[l // 4][2 (l % 4) + 1]
      trans:     M_j[2 (l % 4)][l // 4], M_j[2 (l % 4) + 1][l // 4]
    (the register layout the paper says matches the mma operand arrangement).
    Plain Python loops (32 lanes x num registers).  Returns (32, num) uint32."""
    smem = np.asarray(smem_u16, dtype=np.uint16)
    out = np.zeros((32, num), dtype=np.uint32)
    for j in range(num):
        M = [[int(smem[int(row_elem[8 * j + r]) + c]) for c in range(8)] for r in range(8)]
        for l in range(32):
            g, t = l // 4, l % 4
            lo, hi = (M[g][2 * t], M[g][2 * t + 1]) if not trans else (M[2 * t][g], M[2 * t + 1][g])
            out[l, j] = lo | (hi << 16)
    return out


# ---------------------------------------------------------------------------- TF32 input conversion
def tf32_convert(bits32: np.ndarray, mode: str) -> np.ndarray:
    """How FP32 storage may become a TF32 operand (SURVEY §8(c) reading C1: the paper never says;
    C2's raw-input sub-class observes it).  Element-wise on FP32 bits, finite inputs:
      "rz"  drop the low 13 significand bits (truncation toward zero);
      "rne" round to nearest, ties to even (quantize(x, TF32));
      "rna" round to nearest, ties away from zero (add half a TF32 ulp to the magnitude, then drop
            the low 13 bits: PTX cvt.rna.tf32.f32);
      "fp32" keep every bit (the tensor core reads FP32)."""
    b = np.asarray(bits32, dtype=np.uint32)
    if mode == "fp32":
        return b.copy()
    if mode == "rz":
        return b & np.uint32(0xFFFFE000)
    if mode == "rna":
        return (b + np.uint32(0x1000)) & np.uint32(0xFFFFE000)     # sign bit untouched for finite values
    if mode == "rne":
        return quantize_f32_bits(b, TF32).astype(np.uint32)
    raise ValueError(mode)
