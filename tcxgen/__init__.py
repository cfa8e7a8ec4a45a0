"""tcxgen — seeded synthetic input generators shared by tests, bench and the oracle checks.

This module holds NONE of the method's arithmetic (no products, sums, MMA, 2:4 expansion):
it only draws random numbers and rounds reals into the stated input formats.  Both the
CUDA path (via device tensors) and the oracle (via host copies of the very same bytes)
consume its output, so no input ever comes from the CUDA path.

Generator (pinned; deterministic regardless of device or chunking):
  * counter-based SplitMix64: z = seed*0x9E3779B97F4A7C15 + (stream << 48) + index, then the
    standard SplitMix64 finaliser (precedent: SPEC.md:425-426 pins SplitMix64 + Box-Muller);
  * uniform [0,1) = (z >> 11) * 2^-53;
  * N(0,1) = Box-Muller cosine branch from draws 2i, 2i+1 (float64);
  * reals are float64, rounded RNE to FP32 and then RNE to the target format
    (FP16 / BF16 / TF32-in-FP32).  The paper uses N(0,1) with one shared seed
    (PAPER.md:900); its generator is unpublished.
  * int8 = top byte of z; int32 in [-2^20, 2^20] = (z >> 32) mod (2^21 + 1) - 2^20;
    2:4 pair = (z >> 32) mod 6 over {(0,1),(0,2),(0,3),(1,2),(1,3),(2,3)}.
Streams: A=1, B=2, C=3, positions=4, sparse values=5, probe classes=16+class.

Works on CPU or CUDA torch tensors (torch is plumbing here, as in the product).
"""
from __future__ import annotations

import math

import torch

GOLDEN = 0x9E3779B97F4A7C15
M1 = 0xBF58476D1CE4E5B9
M2 = 0x94D049BB133111EB
STREAM_A, STREAM_B, STREAM_C, STREAM_POS, STREAM_SPVAL = 1, 2, 3, 4, 5
PAIRS = ((0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3))


def _s64(x: int) -> int:
    x &= (1 << 64) - 1
    return x - (1 << 64) if x >= (1 << 63) else x


def _srl(z: torch.Tensor, s: int) -> torch.Tensor:
    """logical right shift of a uint64 held in int64"""
    return (z >> s) & ((1 << (64 - s)) - 1)


def splitmix_ref(seed: int, stream: int, index: int) -> int:
    """pure-Python SplitMix64 (the definition the torch version is tested against)"""
    m = (1 << 64) - 1
    z = (seed * GOLDEN + (stream << 48) + index) & m
    z = ((z ^ (z >> 30)) * M1) & m
    z = ((z ^ (z >> 27)) * M2) & m
    return z ^ (z >> 31)


def splitmix(seed: int, stream: int, idx: torch.Tensor) -> torch.Tensor:
    """uint64 words (as int64 bit patterns) for counters idx (int64 tensor)."""
    base = _s64(seed * GOLDEN + (stream << 48))
    z = idx + base
    z = (z ^ _srl(z, 30)) * _s64(M1)
    z = (z ^ _srl(z, 27)) * _s64(M2)
    return z ^ _srl(z, 31)


def _chunks(n: int, chunk: int = 1 << 24):
    for s in range(0, n, chunk):
        yield s, min(n, s + chunk)


def uniform01(seed, stream, start, n, device="cpu") -> torch.Tensor:
    idx = torch.arange(start, start + n, dtype=torch.int64, device=device)
    z = splitmix(seed, stream, idx)
    return _srl(z, 11).to(torch.float64) * (2.0 ** -53)


def normal(seed, stream, start, n, device="cpu") -> torch.Tensor:
    """N(0,1) in float64: Box-Muller cosine branch on draws (2i, 2i+1)."""
    idx = torch.arange(2 * start, 2 * (start + n), dtype=torch.int64, device=device)
    z = splitmix(seed, stream, idx)
    u = _srl(z, 11).to(torch.float64) * (2.0 ** -53)
    u1, u2 = u[0::2], u[1::2]
    return torch.sqrt(-2.0 * torch.log1p(-u1)) * torch.cos((2.0 * math.pi) * u2)


def round_tf32_bits(x32: torch.Tensor) -> torch.Tensor:
    """FP32 -> TF32 round-to-nearest-even, stored in FP32 (low 13 bits zero).
    NaN/inf untouched; a carry out of max-finite becomes inf."""
    u = x32.view(torch.int32).to(torch.int64) & 0xFFFFFFFF
    expall = (u & 0x7F800000) == 0x7F800000
    r = (u + 0xFFF + ((u >> 13) & 1)) & 0xFFFFE000
    r = torch.where(expall, u, r)
    r = torch.where(r >= (1 << 31), r - (1 << 32), r)
    return r.to(torch.int32).view(torch.float32)


def to_format(x64: torch.Tensor, fmt: str) -> torch.Tensor:
    """float64 reals -> stored format: 'f16' | 'bf16' | 'tf32' (FP32 storage) | 'f32'."""
    x32 = x64.to(torch.float32)
    if fmt == "f32":
        return x32
    if fmt == "tf32":
        return round_tf32_bits(x32)
    if fmt == "f16":
        return x32.to(torch.float16)
    if fmt == "bf16":
        return x32.to(torch.bfloat16)
    raise ValueError(fmt)


def _fill(out_flat: torch.Tensor, fn, chunk=1 << 24):
    n = out_flat.numel()
    for s, e in _chunks(n, chunk):
        out_flat[s:e] = fn(s, e - s)
    return out_flat


def normal_matrix(shape, fmt, seed, stream, device="cpu", redraw_zero=False) -> torch.Tensor:
    """matrix of N(0,1) rounded to fmt; element (i, j) uses counter i*cols + j.
    redraw_zero: values that round to +-0 are replaced by a draw from stream+64 at the
    same counter (repeated until nonzero) — the C5 "exactly 2 nonzeros" rule."""
    n = int(math.prod(shape))
    dt = {"f16": torch.float16, "bf16": torch.bfloat16, "tf32": torch.float32, "f32": torch.float32}[fmt]
    out = torch.empty(n, dtype=dt, device=device)

    def fn(s, m):
        v = to_format(normal(seed, stream, s, m, device), fmt)
        if redraw_zero:
            k = 1
            while True:
                z = v == 0
                if not bool(z.any()):
                    break
                alt = to_format(normal(seed, stream + 64 * k, s, m, device), fmt)
                v = torch.where(z, alt, v)
                k += 1
        return v
    _fill(out, fn)
    return out.view(*shape)


def uniform_matrix(shape, fmt, seed, stream, lo=-1.0, hi=1.0, device="cpu") -> torch.Tensor:
    """reals uniform in [lo, hi) then RNE to fmt ([-1,1) then RNE; +-1 reachable)."""
    n = int(math.prod(shape))
    dt = {"f16": torch.float16, "bf16": torch.bfloat16, "tf32": torch.float32, "f32": torch.float32}[fmt]
    out = torch.empty(n, dtype=dt, device=device)
    _fill(out, lambda s, m: to_format(lo + (hi - lo) * uniform01(seed, stream, s, m, device), fmt))
    return out.view(*shape)


def int8_matrix(shape, seed, stream, device="cpu") -> torch.Tensor:
    """uniform int8 in [-128, 127] (inclusive): top byte of z."""
    n = int(math.prod(shape))
    out = torch.empty(n, dtype=torch.int8, device=device)

    def fn(s, m):
        z = splitmix(seed, stream, torch.arange(s, s + m, dtype=torch.int64, device=device))
        return (_srl(z, 56) - 128).to(torch.int8)   # top byte, re-centred (a bijection of the byte)
    _fill(out, fn)
    return out.view(*shape)


def int32_matrix(shape, seed, stream, lo=-(1 << 20), hi=(1 << 20), device="cpu") -> torch.Tensor:
    """uniform int32 in [lo, hi] inclusive: (z >> 32) mod (hi-lo+1) + lo."""
    n = int(math.prod(shape))
    out = torch.empty(n, dtype=torch.int32, device=device)

    def fn(s, m):
        z = splitmix(seed, stream, torch.arange(s, s + m, dtype=torch.int64, device=device))
        return (torch.remainder(_srl(z, 32), hi - lo + 1) + lo).to(torch.int32)
    _fill(out, fn)
    return out.view(*shape)


def sp24_pairs(M, K, seed, stream=STREAM_POS, device="cpu") -> torch.Tensor:
    """index of the kept pair (0..5 into PAIRS) for every (row, group): shape (M, K/4) uint8."""
    n = M * (K // 4)
    out = torch.empty(n, dtype=torch.uint8, device=device)

    def fn(s, m):
        z = splitmix(seed, stream, torch.arange(s, s + m, dtype=torch.int64, device=device))
        return torch.remainder(_srl(z, 32), 6).to(torch.uint8)
    _fill(out, fn)
    return out.view(M, K // 4)


def sp24_canonical_meta(pairs: torch.Tensor) -> torch.Tensor:
    """canonical metadata words (M, K/32) int32 from pair indices: nibble = i0 | i1 << 2 at
    bits 4*(g%8) of word g/8.  Bit packing only."""
    nib_table = torch.tensor([i0 | (i1 << 2) for i0, i1 in PAIRS], dtype=torch.int64, device=pairs.device)
    nib = nib_table[pairs.long()]                               # (M, G)
    M, G = nib.shape
    nib = nib.view(M, G // 8, 8)
    shifts = (4 * torch.arange(8, device=pairs.device, dtype=torch.int64)).view(1, 1, 8)
    words = (nib << shifts).sum(dim=2)                          # < 2^32
    words = torch.where(words >= (1 << 31), words - (1 << 32), words)
    return words.to(torch.int32)


def sp24_problem(M, K, seed, fmt="f16", device="cpu"):
    """C5-style 2:4 operand: (vals (M, K/2), canonical meta (M, K/32) int32).
    positions uniform over the 6 pairs; values N(0,1) with zero-redraw (never +-0)."""
    pairs = sp24_pairs(M, K, seed, STREAM_POS, device)
    vals = normal_matrix((M, K // 2), fmt, seed, STREAM_SPVAL, device, redraw_zero=True)
    return vals, sp24_canonical_meta(pairs)


def sp24_problem_i8(M, K, seed, device="cpu"):
    """INT8 2:4 operand (NEXT-1 at C4's shape): pairs uniform over the 6, kept values uniform in
    [-128, 127] without 0 (so every group has exactly 2 nonzeros)."""
    pairs = sp24_pairs(M, K, seed, STREAM_POS, device)
    v = int32_matrix((M, K // 2), seed, STREAM_SPVAL, -128, 126, device)
    v = torch.where(v >= 0, v + 1, v)
    return v.to(torch.int8), sp24_canonical_meta(pairs)


def sp12_problem_tf32(M, K, seed, device="cpu"):
    """TF32 1:2 operand (hardware TF32 sparsity, DESIGN.md R-C12): in every aligned pair one element
    kept, position uniform; values N(0,1) rounded to TF32, never 0.  Canonical nibble per group of 4:
    i0 in {0,1}, i1 in {2,3}.  Returns (vals (M, K/2) float32, meta (M, K/32) int32)."""
    n = M * (K // 4)
    pat = torch.empty(n, dtype=torch.uint8, device=device)

    def fn(s, m):
        z = splitmix(seed, STREAM_POS, torch.arange(s, s + m, dtype=torch.int64, device=device))
        return torch.remainder(_srl(z, 32), 4).to(torch.uint8)
    _fill(pat, fn)
    # pattern p -> (i0, i1) = (p & 1, 2 + (p >> 1)) -> index into PAIRS
    to_pair = torch.tensor([PAIRS.index((p & 1, 2 + (p >> 1))) for p in range(4)], dtype=torch.uint8, device=device)
    pairs = to_pair[pat.long()].view(M, K // 4)
    vals = normal_matrix((M, K // 2), "tf32", seed, STREAM_SPVAL, device, redraw_zero=True)
    return vals, sp24_canonical_meta(pairs)


# ----------------------------------------------------------------------------------------------
# Config 2: crafted numeric-probe tiles (SURVEY §8(d) "The eight C2 crafted classes").
# Each tile is m16n8k16 (TF32: k16 = two chained k8); only d00 is probed, the paper's placement
# (PAPER.md:900): values in row 0 of A, column 0 of B ("n-row" 0 of the stored B) and c00,
# everything else zero.  Random numbers only; the MMA arithmetic lives elsewhere.
# ----------------------------------------------------------------------------------------------
CLASSES = ("SPREAD", "CANCEL", "BIGC", "LADDER", "TIES", "SUBNORMAL", "PAPER3_init_low", "PAPER3_init_FP32")
PROBE_TYPES = ("mul", "inner", "accum", "accum_c32")


def _u(seed, stream, n, k=1):
    return uniform01(seed, stream, 0, n * k).view(n, k).double()


def probe_classes(fmt, n_per_class=8192, seed=0):
    """returns dict: A (T,16,16), B (T,8,16), C (T,16,8) [stored formats], cls (T,), ptype (T,),
    a32/b32/c32 (T,16)/(T,16)/(T,): the FP32 values the paper's CPU baseline would use."""
    import numpy as np
    K = 16
    T = n_per_class * len(CLASSES)
    a = torch.zeros(T, K, dtype=torch.float64)
    b = torch.zeros(T, K, dtype=torch.float64)
    c = torch.zeros(T, dtype=torch.float64)
    a32 = torch.zeros(T, K, dtype=torch.float64)      # CPU-baseline inputs for PAPER3_init_FP32
    b32 = torch.zeros(T, K, dtype=torch.float64)
    c32 = torch.zeros(T, dtype=torch.float64)
    ptype = torch.full((T,), -1, dtype=torch.int64)
    cls = torch.arange(T) // n_per_class
    emin = {"f16": -14, "bf16": -126, "tf32": -126}[fmt]
    fbits = {"f16": 10, "bf16": 7, "tf32": 10}[fmt]
    n = n_per_class

    def sig(u):                                        # random significand in [1, 2) with fbits bits
        return 1.0 + torch.floor(u * (1 << fbits)) / (1 << fbits)

    def sgn(u):
        return torch.where(u < 0.5, -1.0, 1.0).double()

    def split(e, ua, ub, us):                          # product exponent e -> a, b with normal exponents
        ea = torch.floor(e / 2.0)
        eb = e - ea
        ea = torch.clamp(ea, min=emin)
        eb = e - ea
        return sgn(us) * sig(ua) * torch.pow(2.0, ea), sig(ub) * torch.pow(2.0, eb)

    for ci, name in enumerate(CLASSES):
        s = slice(ci * n, (ci + 1) * n)
        st = 16 + ci
        U = _u(seed, st, n, 8 * K)
        if name == "SPREAD":
            e = torch.floor(U[:, 0:K] * 41) - 30                  # product exponents in [-30, 10]
            a[s], b[s] = split(e, U[:, K:2 * K], U[:, 2 * K:3 * K], U[:, 3 * K:4 * K])
        elif name == "CANCEL":
            e = torch.floor(U[:, 0:K] * 8) - 4
            x, y = split(e, U[:, K:2 * K], U[:, 2 * K:3 * K], U[:, 3 * K:4 * K])
            x[:, 1::2] = -x[:, 0::2]
            y[:, 1::2] = y[:, 0::2]
            er = -(10 + torch.floor(U[:, 4 * K] * 21))            # residual 2^-10 .. 2^-30
            rx, ry = split(er.unsqueeze(1), U[:, 5 * K:5 * K + 1], U[:, 5 * K + 1:5 * K + 2], U[:, 5 * K + 2:5 * K + 3])
            x[:, 14:15], y[:, 14:15] = rx, ry
            x[:, 15], y[:, 15] = 0.0, 0.0
            a[s], b[s] = x, y
            c[s] = (normal(seed, st + 64, 0, n).double()).to(torch.float32).double()
        elif name == "BIGC":
            m = torch.floor(U[:, 6 * K] * (1 << 23))
            c[s] = sgn(U[:, 6 * K + 1]) * (2.0 ** 24) * (1 + m * 2.0 ** -23)
            e = torch.floor(U[:, 0:K] * 33) - 30                  # products 2^-30 .. 2^2
            a[s], b[s] = split(e, U[:, K:2 * K], U[:, 2 * K:3 * K], U[:, 3 * K:4 * K])
        elif name == "LADDER":
            j = torch.floor(U[:, 0] * 11)                         # 16 equal products 2^-j, j = 0..10
            ea = -torch.floor(j / 2)
            a[s] = torch.pow(2.0, ea).unsqueeze(1).expand(n, K)
            b[s] = torch.pow(2.0, -j - ea).unsqueeze(1).expand(n, K)
            c[s] = 2.0 ** 24
        elif name == "TIES":
            t = torch.floor(U[:, 0] * (1 << 20))
            c[s] = sgn(U[:, 1]) * (2.0 ** 24 + 2 * t)             # ulp(c) = 2: a product of +-1 is a tie
            v = torch.floor(U[:, 2] * 3)
            x = torch.zeros(n, K, dtype=torch.float64)
            y = torch.zeros(n, K, dtype=torch.float64)
            pm = sgn(U[:, 3])
            x[:, 0] = pm                                          # exact tie
            y[:, 0] = 1.0
            sel = v == 1                                          # tie made of two halves
            x[sel, 0] = pm[sel] * 0.5
            x[sel, 1] = pm[sel] * 0.5
            y[sel, 1] = 1.0
            sel = v == 2                                          # just above/below the tie
            j = 12 + torch.floor(U[:, 4] * 10)
            x[sel, 1] = (sgn(U[:, 5]) * torch.pow(2.0, -j))[sel]
            y[sel, 1] = 1.0
            a[s], b[s] = x, y
        elif name == "SUBNORMAL":
            if fmt == "f16":                                      # FP16 subnormal inputs (2^-24 .. 2^-15)
                ea = -(15 + torch.floor(U[:, 0:K] * 10))
                x = sgn(U[:, K:2 * K]) * torch.floor(1 + U[:, 2 * K:3 * K] * 1023) * 2.0 ** -24
                x = torch.where(U[:, 3 * K:4 * K] < 0.5, x, sgn(U[:, K:2 * K]) * torch.pow(2.0, ea))
                y = sig(U[:, 4 * K:5 * K]) * torch.pow(2.0, torch.floor(U[:, 5 * K:6 * K] * 20) - 10)
            else:                                                 # products below 2^-126: FP32-subnormal results
                e = -(127 + torch.floor(U[:, 0:K] * 22))          # 2^-127 .. 2^-148
                x, y = split(e, U[:, K:2 * K], U[:, 2 * K:3 * K], U[:, 3 * K:4 * K])
            a[s], b[s] = x, y
            c[s] = torch.where(U[:, 7 * K] < 0.5, 0.0, sgn(U[:, 7 * K + 1]) * 2.0 ** -140 * torch.floor(1 + U[:, 7 * K + 2] * 7))
        else:  # PAPER3: a0b0 / a0b0 + a1b1 / a0b0 + c0 (c0 low-format or FP32), N(0,1), one seed
            z = normal(seed, 16 + 6, 0, 5 * n).view(n, 5).double()   # the same draws for both inits
            z32 = z.to(torch.float32).double()
            pt = torch.arange(n) % 4
            x = torch.zeros(n, K, dtype=torch.float64)
            y = torch.zeros(n, K, dtype=torch.float64)
            cc = torch.zeros(n, dtype=torch.float64)
            x[:, 0], y[:, 0] = z32[:, 0], z32[:, 1]
            inner = pt == 1
            x[inner, 1], y[inner, 1] = z32[inner, 2], z32[inner, 3]
            acc = pt >= 2
            cc[acc] = z32[acc, 4]
            a32[s], b32[s], c32[s] = x, y, cc
            a[s], b[s] = x, y
            if name == "PAPER3_init_low":                     # created in low precision: baseline = same values
                a[s] = to_format(x, fmt).double()
                b[s] = to_format(y, fmt).double()
                a32[s], b32[s] = a[s], b[s]
                clow = torch.where(pt == 2, to_format(cc, fmt).double(), cc)    # accum: c0 low; accum_c32: FP32
                c[s] = clow
                c32[s] = clow
            else:
                c[s] = cc
            ptype[s] = pt
    A = torch.zeros(T, 16, K, dtype=torch.float64)
    B = torch.zeros(T, 8, K, dtype=torch.float64)
    A[:, 0, :] = a
    B[:, 0, :] = b
    C = torch.zeros(T, 16, 8, dtype=torch.float32)
    C[:, 0, 0] = c.to(torch.float32)
    return {"A": to_format(A, fmt), "B": to_format(B, fmt), "C": C, "cls": cls, "ptype": ptype,
            "a32": a32.to(torch.float32), "b32": b32.to(torch.float32), "c32": c32.to(torch.float32), "K": K}


# ----------------------------------------------------------------------------------------------
# FP16-accumulate numeric probe: the mma f16.f16.f16.f16 variant
# probed like Table FP16-FP16-numeric-profiling.  The
# crafted classes of configs[1] rescaled to FP16's range (c = 2^11 is where ulp(c) = 2, as 2^24 is
# for FP32); d00 only, values in row 0 of A / column 0 of B / c00.
# ----------------------------------------------------------------------------------------------
CLASSES_F16ACC = ("SPREAD16", "CANCEL16", "BIGC16", "LADDER16", "TIES16", "PAPER3_init_FP16", "PAPER3_init_FP32")


def probe_classes_f16acc(n_per_class=8192, seed=0):
    """returns dict: A (T,16,16) f16, B (T,8,16) f16, C (T,16,8) f16, cls, ptype (PROBE_TYPES index,
    -1 for crafted), a32/b32/c32: the FP32 values of the paper's CPU baseline."""
    K = 16
    T = n_per_class * len(CLASSES_F16ACC)
    a = torch.zeros(T, K, dtype=torch.float64)
    b = torch.zeros(T, K, dtype=torch.float64)
    c = torch.zeros(T, dtype=torch.float64)
    a32 = torch.zeros(T, K, dtype=torch.float64)
    b32 = torch.zeros(T, K, dtype=torch.float64)
    c32 = torch.zeros(T, dtype=torch.float64)
    ptype = torch.full((T,), -1, dtype=torch.int64)
    cls = torch.arange(T) // n_per_class
    n = n_per_class

    def sig(u):
        return 1.0 + torch.floor(u * 1024) / 1024

    def sgn(u):
        return torch.where(u < 0.5, -1.0, 1.0).double()

    def split(e, ua, ub, us):
        ea = torch.clamp(torch.floor(e / 2.0), min=-14)
        eb = e - ea
        return sgn(us) * sig(ua) * torch.pow(2.0, ea), sig(ub) * torch.pow(2.0, eb)

    for ci, name in enumerate(CLASSES_F16ACC):
        s = slice(ci * n, (ci + 1) * n)
        st = 48 + ci
        U = _u(seed, st, n, 8 * K)
        if name == "SPREAD16":
            e = torch.floor(U[:, 0:K] * 19) - 14                   # product exponents in [-14, 4]
            a[s], b[s] = split(e, U[:, K:2 * K], U[:, 2 * K:3 * K], U[:, 3 * K:4 * K])
        elif name == "CANCEL16":
            e = torch.floor(U[:, 0:K] * 6) - 3
            x, y = split(e, U[:, K:2 * K], U[:, 2 * K:3 * K], U[:, 3 * K:4 * K])
            x[:, 1::2] = -x[:, 0::2]
            y[:, 1::2] = y[:, 0::2]
            er = -(4 + torch.floor(U[:, 4 * K] * 11))              # residual 2^-4 .. 2^-14
            rx, ry = split(er.unsqueeze(1), U[:, 5 * K:5 * K + 1], U[:, 5 * K + 1:5 * K + 2], U[:, 5 * K + 2:5 * K + 3])
            x[:, 14:15], y[:, 14:15] = rx, ry
            x[:, 15], y[:, 15] = 0.0, 0.0
            a[s], b[s] = x, y
            c[s] = to_format(normal(seed, st + 64, 0, n).double(), "f16").double()
        elif name == "BIGC16":
            m = torch.floor(U[:, 6 * K] * 1024)
            c[s] = sgn(U[:, 6 * K + 1]) * 2048.0 * (1 + m / 1024)  # [2^11, 2^12): ulp 2
            e = torch.floor(U[:, 0:K] * 11) - 9                    # products 2^-9 .. 2^1
            a[s], b[s] = split(e, U[:, K:2 * K], U[:, 2 * K:3 * K], U[:, 3 * K:4 * K])
        elif name == "LADDER16":
            j = torch.floor(U[:, 0] * 11)                          # 16 equal products 2^-j
            ea = -torch.floor(j / 2)
            a[s] = torch.pow(2.0, ea).unsqueeze(1).expand(n, K)
            b[s] = torch.pow(2.0, -j - ea).unsqueeze(1).expand(n, K)
            c[s] = 2048.0
        elif name == "TIES16":
            t = torch.floor(U[:, 0] * 512)
            c[s] = sgn(U[:, 1]) * (2048.0 + 2 * t)                 # ulp(c) = 2: a product of +-1 is a tie
            v = torch.floor(U[:, 2] * 3)
            x = torch.zeros(n, K, dtype=torch.float64)
            y = torch.zeros(n, K, dtype=torch.float64)
            pm = sgn(U[:, 3])
            x[:, 0] = pm
            y[:, 0] = 1.0
            sel = v == 1
            x[sel, 0] = pm[sel] * 0.5
            x[sel, 1] = pm[sel] * 0.5
            y[sel, 1] = 1.0
            sel = v == 2
            j = 4 + torch.floor(U[:, 4] * 8)                       # 2^-4 .. 2^-11 nudges
            x[sel, 1] = (sgn(U[:, 5]) * torch.pow(2.0, -j))[sel]
            y[sel, 1] = 1.0
            a[s], b[s] = x, y
        else:   # the paper's three probes, N(0,1), c0 FP16 (init_FP16) or converted at copy (init_FP32)
            z = normal(seed, 48 + 5, 0, 5 * n).view(n, 5).double()
            z32 = z.to(torch.float32).double()
            pt = torch.arange(n) % 3
            x = torch.zeros(n, K, dtype=torch.float64)
            y = torch.zeros(n, K, dtype=torch.float64)
            cc = torch.zeros(n, dtype=torch.float64)
            x[:, 0], y[:, 0] = z32[:, 0], z32[:, 1]
            inner = pt == 1
            x[inner, 1], y[inner, 1] = z32[inner, 2], z32[inner, 3]
            acc = pt == 2
            cc[acc] = z32[acc, 4]
            ptype[s] = pt
            if name == "PAPER3_init_FP16":
                x = to_format(x, "f16").double()
                y = to_format(y, "f16").double()
                cc = to_format(cc, "f16").double()
            a32[s], b32[s], c32[s] = x, y, cc
            a[s], b[s], c[s] = x, y, cc
    A = torch.zeros(T, 16, K, dtype=torch.float16)
    B = torch.zeros(T, 8, K, dtype=torch.float16)
    C = torch.zeros(T, 16, 8, dtype=torch.float16)
    A[:, 0, :] = to_format(a, "f16")
    B[:, 0, :] = to_format(b, "f16")
    C[:, 0, 0] = to_format(c, "f16")
    return {"A": A, "B": B, "C": C, "cls": cls, "ptype": ptype, "a32": a32.float(), "b32": b32.float(),
            "c32": c32.float(), "K": K}


# ----------------------------------------------------------------------------------------------
# Chain matrix multiplication: "All values are randomly
# generated by normal distribution with mu = 0 and sigma = 1" (Fig. chain-result caption).
# init "low": values created in the low-precision type, so the CPU FP32 baseline uses the same
# values; init "fp32": values created in FP32 and converted when copied to the GPU.
# ----------------------------------------------------------------------------------------------
CHAIN_STREAM = 96


def chain_problem(fmt, count, n_steps, init="low", seed=0):
    """returns (A0_gpu, Bs_gpu) in fmt's storage (TF32 in FP32) and (A0_cpu, Bs_cpu) float32:
    A0 (count, 16, 8), Bs (count, n_steps, 8, 8) stored n x k."""
    a = normal(seed, CHAIN_STREAM, 0, count * 128).view(count, 16, 8).to(torch.float32)
    b = normal(seed, CHAIN_STREAM + 1, 0, count * n_steps * 64).view(count, n_steps, 8, 8).to(torch.float32)
    a_low, b_low = to_format(a.double(), fmt), to_format(b.double(), fmt)
    if init == "low":
        return a_low, b_low, a_low.to(torch.float32), b_low.to(torch.float32)
    if init == "fp32":
        return a_low, b_low, a, b
    raise ValueError(init)
