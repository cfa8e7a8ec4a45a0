"""paper_2206_02874_b200 — Python binding of libtcx.so (the B200 tensor-core MMA library).

Argument marshalling only: every step of the hot path runs in the CUDA kernels behind the
C ABI declared in include/tcx.h.  torch supplies device memory and streams.  There is no
CPU fallback: if libtcx.so is missing or a call fails, an exception is raised.

Functions (same names as the C ABI, minus the ``tcx_`` prefix):
  mma_tiles(A, B, C, D=None)            batch of m16n8k16 / m16n8k8|16 (tf32) / m16n8k32 (s8) tiles
  mma_tiles_tc05(A, B, C, D=None)       the same tiles through tcgen05 (C preloaded in TMEM)
  mma_chain(A0, Bs)                     the paper's chain matmul: D_i = cvt(D_{i-1}) x B_i (m16n8k8)
  gemm(A, B, C=None, D=None, ...)       dense D = A @ B^T-stored + C   (B is N x K, "col")
  sp24_compress(A_dense)                -> (vals, meta_canon)
  sp24_pack_meta(meta_canon, M, K)      -> meta_hw
  gemm_sp24(vals, meta_hw, B, C, D, K)  2:4 sparse D = expand(vals, meta) x B + C
  round_tf32(x)                         FP32 -> TF32 RNE (FP32 storage)
  probe(config dict)                    clock-counter latency/throughput
"""
from __future__ import annotations

import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# TCX_LIB_PATH selects another build of the same library (A/B experiments); never a fallback
LIB_PATH = os.environ.get("TCX_LIB_PATH", os.path.join(_HERE, "libtcx.so"))

F16, BF16, TF32, F32, S8, S32 = 0, 1, 2, 3, 4, 5
_STATUS = {0: "TCX_OK", 1: "TCX_ERR_INVALID_VALUE", 2: "TCX_ERR_UNSUPPORTED", 3: "TCX_ERR_MISALIGNED",
           4: "TCX_ERR_BAD_SPARSITY", 5: "TCX_ERR_NO_DEVICE", 6: "TCX_ERR_ARCH", 7: "TCX_ERR_CUDA"}

EXPORTS = ["tcx_mma_tiles", "tcx_mma_tiles_tc05", "tcx_mma_chain", "tcx_gemm", "tcx_gemm_ex", "tcx_sp24_compress",
           "tcx_sp24_meta_hw_bytes", "tcx_sp24_pack_meta", "tcx_gemm_sp24", "tcx_gemm_sp24_ex", "tcx_round_tf32",
           "tcx_probe", "tcx_ldmatrix_dump",
           "tcx_status_string", "tcx_last_error", "tcx_version", "tcx_launch_count", "tcx_debug_trace",
           "tcx_sm_clock_stamp"]


class TcxError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{_STATUS.get(status, status)}: {msg}")
        self.status = status


class GemmOpts(ctypes.Structure):
    _fields_ = [("cta_group", ctypes.c_int), ("max_ctas", ctypes.c_int), ("group_m", ctypes.c_int),
                ("tile_n", ctypes.c_int), ("pairs_m", ctypes.c_int), ("pairs_n", ctypes.c_int),
                ("reserved", ctypes.c_int * 2)]


class ProbeConfig(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int) for n in ("kind", "ab", "cd", "m", "n", "k", "cta_group", "warps", "ilp",
                                             "iters", "repeats", "num_sms", "issuers", "n_acc", "mode")] + \
               [("a_op", ctypes.c_void_p), ("b_op", ctypes.c_void_p), ("acc_out", ctypes.c_void_p)]


class ProbeResult(ctypes.Structure):
    _fields_ = [("cycles_per_iter_min", ctypes.c_double), ("cycles_per_iter_median", ctypes.c_double),
                ("latency_cycles", ctypes.c_double), ("fma_per_clk_per_sm", ctypes.c_double),
                ("sm_mhz", ctypes.c_double), ("ns_per_iter", ctypes.c_double), ("iters", ctypes.c_int64),
                ("sink", ctypes.c_uint32), ("mmas_per_issuer", ctypes.c_int64), ("warmup_iters", ctypes.c_int32),
                ("n_acc", ctypes.c_int32), ("sms_used", ctypes.c_int32), ("max_issuers_per_sm", ctypes.c_int32)]


_lib = None


def lib():
    """Load libtcx.so (fails loudly if it is missing: there is no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libtcx.so not found at {LIB_PATH}; run `python -m paper_2206_02874_b200.build`")
    L = ctypes.CDLL(LIB_PATH)
    vp, i64, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
    L.tcx_mma_tiles.argtypes = [i32, i32, i32, i32, i32, i64, vp, vp, vp, vp, vp]
    L.tcx_mma_tiles_tc05.argtypes = [i32, i32, i32, i32, i32, i64, vp, vp, vp, vp, vp]
    L.tcx_mma_chain.argtypes = [i32, i32, i64, vp, vp, vp, vp]
    L.tcx_gemm.argtypes = [i32, i32, i64, i64, i64, vp, i64, vp, i64, vp, i64, vp, i64, vp]
    L.tcx_gemm_ex.argtypes = [i32, i32, i64, i64, i64, vp, i64, vp, i64, vp, i64, vp, i64, ctypes.POINTER(GemmOpts), vp]
    L.tcx_sp24_compress.argtypes = [i32, i64, i64, vp, i64, vp, vp, vp, vp]
    L.tcx_sp24_meta_hw_bytes.argtypes = [i32, i64, i64]
    L.tcx_sp24_meta_hw_bytes.restype = ctypes.c_size_t
    L.tcx_sp24_pack_meta.argtypes = [i32, i64, i64, vp, vp, vp, vp]
    L.tcx_gemm_sp24.argtypes = [i32, i32, i64, i64, i64, vp, i64, vp, vp, i64, vp, i64, vp, i64, vp]
    L.tcx_gemm_sp24_ex.argtypes = [i32, i32, i64, i64, i64, vp, i64, vp, vp, i64, vp, i64, vp, i64,
                                   ctypes.POINTER(GemmOpts), vp]
    L.tcx_round_tf32.argtypes = [vp, vp, i64, vp]
    L.tcx_probe.argtypes = [i32, ctypes.POINTER(ProbeConfig), ctypes.POINTER(ProbeResult)]
    L.tcx_ldmatrix_dump.argtypes = [i32, i32, vp, vp, vp, vp]
    L.tcx_status_string.restype = ctypes.c_char_p
    L.tcx_last_error.restype = ctypes.c_char_p
    L.tcx_version.restype = ctypes.c_char_p
    L.tcx_launch_count.restype = ctypes.c_uint64
    L.tcx_debug_trace.argtypes = [vp, i64]
    L.tcx_sm_clock_stamp.argtypes = [vp, i32, vp]
    for f in ("tcx_mma_tiles", "tcx_mma_tiles_tc05", "tcx_mma_chain", "tcx_gemm", "tcx_gemm_ex", "tcx_sp24_compress",
              "tcx_sp24_pack_meta", "tcx_gemm_sp24", "tcx_gemm_sp24_ex", "tcx_round_tf32", "tcx_probe", "tcx_ldmatrix_dump",
              "tcx_debug_trace", "tcx_sm_clock_stamp"):
        getattr(L, f).restype = ctypes.c_int
    _lib = L
    return L


def _check(st):
    if st != 0:
        raise TcxError(st, lib().tcx_last_error().decode())


def _ptr(t):
    return None if t is None else t.data_ptr()          # argtypes are c_void_p: plain ints marshal directly


_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)


def _stream(t=None):
    """the caller's current stream on t's device, as the void* the C ABI takes"""
    dev = t.device if t is not None else torch.device("cuda", torch.cuda.current_device())
    if _raw_stream is not None:
        return _raw_stream(dev.index if dev.index is not None else torch.cuda.current_device())
    return torch.cuda.current_stream(dev).cuda_stream


def launch_count() -> int:
    return int(lib().tcx_launch_count())


def sm_clock_stamp(buf):
    """stamp (clock64, globaltimer) per SM into buf (int64 CUDA tensor of 2 * n_sm) in stream order"""
    _dev_check(buf)
    _need(buf.dtype == torch.int64 and buf.is_contiguous() and buf.numel() >= 2, "sm_clock_stamp: int64 buffer")
    _check(lib().tcx_sm_clock_stamp(_ptr(buf), buf.numel() // 2, _stream(buf)))


def sm_mhz_between(s0, s1):
    """median over SMs of dclock64 / dglobaltimer between two stamp buffers (MHz); None if no SM has both"""
    a = s0.view(-1, 2).cpu().double()
    b = s1.view(-1, 2).cpu().double()
    dc, dn = b[:, 0] - a[:, 0], b[:, 1] - a[:, 1]
    ok = (dn > 0) & (dc > 0) & (a[:, 1] > 0)
    if not bool(ok.any()):
        return None
    return float((dc[ok] / dn[ok]).median()) * 1000.0


_TORCH_AB = {torch.float16: F16, torch.bfloat16: BF16, torch.int8: S8}


def ab_code(t: torch.Tensor, tf32: bool = False) -> int:
    if t.dtype == torch.float32:
        if not tf32:
            raise TypeError("float32 operands are TF32 inputs: pass tf32=True (values must be TF32-representable)")
        return TF32
    return _TORCH_AB[t.dtype]


def _dev_check(*ts):
    ts = [t for t in ts if t is not None]
    for t in ts:
        if not t.is_cuda:
            raise ValueError("tcx operates on CUDA tensors only (no CPU fallback)")
    if len({t.device for t in ts}) > 1:
        raise ValueError("tcx: all tensors of a call must be on one CUDA device")


_CD_TORCH = {F32: torch.float32, S32: torch.int32, F16: torch.float16}


def _need(cond, msg):
    if not cond:
        raise ValueError(msg)


def _rows_ok(name, t, shape, dtype):
    """t is a 2-D (or N-D) tensor of `shape` and `dtype` whose innermost stride is 1 (rows may be
    padded: the C ABI takes the row stride); raised before any pointer reaches the library, so a
    mismatched buffer can never be read or written out of bounds by the TMA engine"""
    _need(t.dim() == len(shape), f"{name}: expected {len(shape)}-D, got shape {tuple(t.shape)}")
    _need(tuple(t.shape) == tuple(shape), f"{name}: expected shape {tuple(shape)}, got {tuple(t.shape)}")
    _need(t.dtype == dtype, f"{name}: expected dtype {dtype}, got {t.dtype}")
    _need(t.numel() == 0 or t.stride(-1) == 1, f"{name}: the innermost dimension must be contiguous (stride 1)")
    if t.dim() > 2:
        _need(t.is_contiguous(), f"{name}: must be contiguous")


def _mat(name, t, rows, cols, dtype):
    """the per-call check of a 2-D operand (shape, dtype, unit inner stride), cheap on the accepting
    path (a GEMM call's host cost is part of every small call's latency); returns the row stride.
    Any mismatch is re-checked by _rows_ok, which raises the precise error."""
    sh = t.shape
    if len(sh) != 2 or sh[0] != rows or sh[1] != cols or t.dtype != dtype:
        _rows_ok(name, t, (rows, cols), dtype)
    st = t.stride()
    if st[1] != 1 and rows and cols:
        _rows_ok(name, t, (rows, cols), dtype)
    return st[0]


def _tile3(name, t, count, m, n, dtype):
    """the per-call check of a contiguous (count, m, n) tile array; mismatches re-checked by _rows_ok"""
    sh = t.shape
    if len(sh) != 3 or sh[0] != count or sh[1] != m or sh[2] != n or t.dtype != dtype or not t.is_contiguous():
        _rows_ok(name, t, (count, m, n), dtype)


def _device_of(*ts):
    """the one CUDA device index all given tensors live on (None entries skipped); raises otherwise"""
    d = -2
    for t in ts:
        if t is not None:
            g = t.get_device()
            if g < 0:
                raise ValueError("tcx operates on CUDA tensors only (no CPU fallback)")
            if d != g:
                if d != -2:
                    raise ValueError("tcx: all tensors of a call must be on one CUDA device")
                d = g
    return d


def _stream_of(dev_index):
    if _raw_stream is not None:
        return _raw_stream(dev_index)
    return torch.cuda.current_stream(dev_index).cuda_stream


# ---------------------------------------------------------------------------------------- tiles
def mma_tiles(A, B, C=None, D=None, tf32=False, tc05=False, f16_acc=False):
    """D_t = A_t B_t + C_t for A (count, 16, k), B (count, 8, k), C/D (count, 16, 8).
    f16_acc: C/D are FP16 (the f16.f16.f16.f16 MMA); C, if given, must be float16."""
    ab = ab_code(A, tf32)
    _need(A.dim() == 3, f"A: expected (count, 16, k), got shape {tuple(A.shape)}")
    count, m, k = A.shape
    n = 8
    cd = S32 if ab == S8 else (F16 if f16_acc else F32)
    if C is not None and cd == F16 and C.dtype != torch.float16:
        raise ValueError("f16_acc: C must be float16")
    _tile3("A", A, count, m, k, A.dtype)
    _tile3("B", B, count, n, k, A.dtype)
    if C is not None:
        _tile3("C", C, count, m, n, _CD_TORCH[cd])
    if D is not None:
        _tile3("D", D, count, m, n, _CD_TORCH[cd])
    dev = _device_of(A, B, C, D)
    if D is None:
        D = torch.empty((count, m, n), dtype=_CD_TORCH[cd], device=A.device)
    L = _lib or lib()
    fn = L.tcx_mma_tiles_tc05 if tc05 else L.tcx_mma_tiles
    st = fn(ab, cd, m, n, k, count, A.data_ptr(), B.data_ptr(), _ptr(C), D.data_ptr(), _stream_of(dev))
    if st:
        _check(st)
    return D


def mma_tiles_tc05(A, B, C=None, D=None, tf32=False):
    return mma_tiles(A, B, C, D, tf32=tf32, tc05=True)


def mma_chain(A0, Bs, tf32=False, Ds=None):
    """The paper's chain matmul: A0 (count, 16, 8), Bs (count, n_steps, 8, 8)
    stored n x k; returns Ds (count, n_steps, 16, 8) FP32 — D_i = cvt(D_{i-1}) x B_i."""
    _dev_check(A0, Bs, Ds)
    ab = ab_code(A0, tf32)
    count, n_steps = Bs.shape[0], Bs.shape[1]
    if tuple(A0.shape) != (count, 16, 8) or tuple(Bs.shape[2:]) != (8, 8) or Bs.dtype != A0.dtype:
        raise ValueError("mma_chain: A0 (count, 16, 8), Bs (count, n_steps, 8, 8) of one dtype")
    if Ds is None:
        Ds = torch.empty((count, n_steps, 16, 8), dtype=torch.float32, device=A0.device)
    _check(lib().tcx_mma_chain(ab, n_steps, count, _ptr(A0), _ptr(Bs), _ptr(Ds), _stream(A0)))
    return Ds


# ---------------------------------------------------------------------------------------- GEMM
def gemm(A, B, C=None, D=None, tf32=False, cta_group=0, max_ctas=0, group_m=0, tile_n=0, f16_acc=False, pairs=(0, 0),
         _fault=0):
    """Dense D = A x B + C with A (M, K), B stored (N, K) ("row.col"), C/D (M, N).
    f16_acc: FP16 inputs with an FP16 accumulator (C, D float16; C is the MMA's C operand).
    pairs = (pairs_m, pairs_n): TMA-multicast cluster of CTA pairs (tcx_gemm_opts)."""
    ab = ab_code(A, tf32)
    _need(A.dim() == 2 and B.dim() == 2, "gemm: A (M, K) and B (N, K) must be 2-D")
    M, K = A.shape
    N = B.shape[0]
    cd = S32 if ab == S8 else (F16 if f16_acc else F32)
    if cd == F16 and C is not None and C.dtype != torch.float16:
        raise ValueError("f16_acc: C must be float16")
    cdt = _CD_TORCH[cd]
    lda = _mat("A", A, M, K, A.dtype)
    ldb = _mat("B", B, N, K, A.dtype)
    ldc = _mat("C", C, M, N, cdt) if C is not None else N
    ldd = _mat("D", D, M, N, cdt) if D is not None else N
    dev = _device_of(A, B, C, D)
    if D is None:
        D = torch.empty((M, N), dtype=cdt, device=A.device)
    L = _lib or lib()
    if not (cta_group or max_ctas or group_m or tile_n or pairs[0] or pairs[1] or _fault):
        st = L.tcx_gemm(ab, cd, M, N, K, A.data_ptr(), lda, B.data_ptr(), ldb, _ptr(C), ldc, D.data_ptr(), ldd,
                        _stream_of(dev))
    else:
        opts = GemmOpts(cta_group, max_ctas, group_m, tile_n, pairs[0], pairs[1], (ctypes.c_int * 2)(_fault, 0))
        st = L.tcx_gemm_ex(ab, cd, M, N, K, A.data_ptr(), lda, B.data_ptr(), ldb, _ptr(C), ldc, D.data_ptr(), ldd,
                           ctypes.byref(opts), _stream_of(dev))
    if st:
        _check(st)
    return D


def debug_trace(buf=None):
    """debug library only: record a per-tile timeline of later tcx_gemm launches into `buf`
    (int64 CUDA tensor of 4 * capacity; None = off).  See include/tcx.h tcx_debug_trace."""
    if buf is None:
        _check(lib().tcx_debug_trace(None, 0))
    else:
        _dev_check(buf)
        _check(lib().tcx_debug_trace(_ptr(buf), buf.numel() // 4))


# ---------------------------------------------------------------------------------------- sparse
def sp24_compress(A_dense, tf32=False):
    """dense (M, K) 2:4 matrix -> (vals (M, K/2), meta_canon (M, K/32) int32).
    Raises ValueError naming the first (row, group) with more than 2 nonzeros.  tf32=True (FP32
    storage): the hardware's 1:2 rule — one element kept per aligned pair."""
    ab = ab_code(A_dense, tf32)
    _need(A_dense.dim() == 2, "sp24_compress: A must be 2-D")
    M, K = A_dense.shape
    _rows_ok("A", A_dense, (M, K), A_dense.dtype)
    _dev_check(A_dense)
    vals = torch.empty((M, K // 2), dtype=A_dense.dtype, device=A_dense.device)
    meta = torch.empty((M, K // 32), dtype=torch.int32, device=A_dense.device)
    bad = torch.empty(2, dtype=torch.int64, device=A_dense.device)
    _check(lib().tcx_sp24_compress(ab, M, K, _ptr(A_dense), A_dense.stride(0), _ptr(vals), _ptr(meta),
                                   _ptr(bad), _stream(A_dense)))
    r, g = bad.tolist()
    if r >= 0:
        raise ValueError(f"2:4 violation at row {r}, group {g}")
    return vals, meta


def sp24_meta_hw_bytes(M, K, ab=F16):
    return int(lib().tcx_sp24_meta_hw_bytes(ab, M, K))


def sp24_pack_meta(meta_canon, M, K, ab=F16, check=True):
    _rows_ok("meta_canon", meta_canon, (M, K // 32), torch.int32)
    _need(meta_canon.is_contiguous(), "meta_canon must be contiguous")
    _dev_check(meta_canon)
    nbytes = sp24_meta_hw_bytes(M, K, ab)
    hw = torch.empty(nbytes, dtype=torch.uint8, device=meta_canon.device)
    bad = torch.empty(2, dtype=torch.int64, device=meta_canon.device)
    _check(lib().tcx_sp24_pack_meta(ab, M, K, _ptr(meta_canon), _ptr(hw), _ptr(bad), _stream(meta_canon)))
    if check:
        r, g = bad.tolist()
        if r >= 0:
            raise ValueError(f"bad metadata nibble at row {r}, group {g}")
    return hw


def gemm_sp24(vals, meta_hw, B, C=None, D=None, cta_group=0, max_ctas=0, group_m=0, tf32=False, tile_m=0, pairs=(0, 0),
              _knobs=0):
    """D = expand(vals, meta) x B + C; vals (M, K/2), B (N, K).  FP16/BF16 -> FP32, INT8 -> INT32
    (meta_hw packed with the same ab: sp24_pack_meta(meta, M, K, ab=S8) for int8)."""
    ab = ab_code(vals, tf32)
    _need(vals.dim() == 2 and B.dim() == 2, "gemm_sp24: vals (M, K/2) and B (N, K) must be 2-D")
    M = vals.shape[0]
    N, K = B.shape
    cd = S32 if ab == S8 else F32
    _rows_ok("vals", vals, (M, K // 2), vals.dtype)
    _need(2 * vals.shape[1] == K, f"gemm_sp24: vals has {vals.shape[1]} kept columns, B's K = {K} needs {K // 2}")
    _rows_ok("B", B, (N, K), vals.dtype)
    _need(meta_hw.dtype == torch.uint8 and meta_hw.is_contiguous(), "gemm_sp24: meta_hw must be a contiguous uint8 "
          "tensor from sp24_pack_meta")
    _need(meta_hw.numel() == sp24_meta_hw_bytes(M, K, ab),
          f"gemm_sp24: meta_hw has {meta_hw.numel()} bytes, ({M}, {K}) needs {sp24_meta_hw_bytes(M, K, ab)}")
    cdt = _CD_TORCH[cd]
    ldc = _mat("C", C, M, N, cdt) if C is not None else N
    ldd = _mat("D", D, M, N, cdt) if D is not None else N
    dev = _device_of(vals, meta_hw, B, C, D)
    if D is None:
        D = torch.empty((M, N), dtype=cdt, device=vals.device)
    opts = GemmOpts(cta_group, max_ctas, group_m, int(tile_m), pairs[0], pairs[1], (ctypes.c_int * 2)(_knobs, 0))
    st = (_lib or lib()).tcx_gemm_sp24_ex(ab, cd, M, N, K, vals.data_ptr(), vals.stride(0), meta_hw.data_ptr(),
                                          B.data_ptr(), B.stride(0), _ptr(C), ldc, D.data_ptr(), ldd,
                                          ctypes.byref(opts), _stream_of(dev))
    if st:
        _check(st)
    return D


def round_tf32(x, out=None):
    _need(x.dtype == torch.float32 and x.is_contiguous(), "round_tf32: x must be a contiguous float32 tensor")
    if out is not None:
        _need(out.dtype == torch.float32 and out.is_contiguous() and out.numel() == x.numel(),
              "round_tf32: out must be a contiguous float32 tensor of x's size")
    _dev_check(x, out)
    if out is None:
        out = torch.empty_like(x)
    _check(lib().tcx_round_tf32(_ptr(x), _ptr(out), x.numel(), _stream(x)))
    return out


# ---------------------------------------------------------------------------------------- probe
PROBE_KINDS = {"mma_sync": 0, "mma_sp_sync": 1, "tc05": 2, "tc05_sp": 3, "ldmatrix": 4, "ld_shared": 5,
               "tmem_ld": 6, "tma_load": 7, "tc05_cp": 8, "tma_multicast": 9, "dsmem": 10}
TC05_MODES = {"sync": 0, "stream": 1, "commit": 2, "stream_rot": 3, "stream_areuse": 4}


def probe(kind="mma_sync", ab=F16, cd=F32, m=16, n=8, k=16, cta_group=1, warps=1, ilp=1, iters=1024,
          repeats=5, num_sms=1, device=-1, issuers=0, n_acc=0, mode="sync", a_op=None, b_op=None, acc_out=None):
    """tcx_probe (include/tcx.h).  tcgen05 kinds: issuers per SM, n_acc accumulators, mode in
    {"sync", "stream", "commit"}; a_op / b_op / acc_out: optional CUDA tensors (operands and issuer 0's
    accumulators, layouts in tcx.h)."""
    for t in (a_op, b_op, acc_out):
        if t is not None and (not t.is_cuda or not t.is_contiguous()):
            raise ValueError("probe: a_op / b_op / acc_out must be contiguous CUDA tensors")
    cfg = ProbeConfig(PROBE_KINDS[kind] if isinstance(kind, str) else kind, ab, cd, m, n, k, cta_group, warps, ilp,
                      iters, repeats, num_sms, issuers, n_acc, TC05_MODES[mode] if isinstance(mode, str) else mode,
                      _ptr(a_op), _ptr(b_op), _ptr(acc_out))
    res = ProbeResult()
    _check(lib().tcx_probe(device, ctypes.byref(cfg), ctypes.byref(res)))
    return {f: getattr(res, f) for f, _ in ProbeResult._fields_}


def ldmatrix_dump(num, trans, src_u16, row_elem):
    """one warp's ldmatrix.x{num}[.trans] fragments: src (512,) 16-bit tensor on the GPU, row_elem
    (32,) int32 element offsets; returns (32, num) int32 (register j of lane l)."""
    _dev_check(src_u16, row_elem)
    out = torch.empty((32, num), dtype=torch.int32, device=src_u16.device)
    _check(lib().tcx_ldmatrix_dump(num, int(trans), _ptr(src_u16), _ptr(row_elem), _ptr(out), _stream(src_u16)))
    return out
