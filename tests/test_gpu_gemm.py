"""tcx_gemm (tcgen05 dense) vs the oracle: small shapes whole-matrix, ragged tails, both CTA
modes, every kind; BASELINE configs[2] (C3 BF16/TF32 8192^3) and configs[3] (C4 INT8 16384^3)
at full size on >= 65,536 sampled outputs + full-coverage properties."""
import numpy as np
import pytest
import torch

import oracle as O
import tcxgen
import paper_2206_02874_b200 as tcx
from parity import host_bits, fp_bound_check, gemm_sample_coords, check_gemm_samples, TORCH2ORACLE, model_predict

pytestmark = pytest.mark.gpu
DEV = "cuda"


def _problem(M, N, K, fmt, seed=0, with_c=True):
    if fmt == "s8":
        A = tcxgen.int8_matrix((M, K), seed, tcxgen.STREAM_A, DEV)
        B = tcxgen.int8_matrix((N, K), seed, tcxgen.STREAM_B, DEV)
        C = tcxgen.int32_matrix((M, N), seed, tcxgen.STREAM_C, device=DEV) if with_c else None
        return A, B, C
    A = tcxgen.normal_matrix((M, K), fmt, seed, tcxgen.STREAM_A, DEV)
    B = tcxgen.normal_matrix((N, K), fmt, seed, tcxgen.STREAM_B, DEV)
    C = tcxgen.normal_matrix((M, N), "f32", seed, tcxgen.STREAM_C, DEV) if with_c else None
    return A, B, C


def _full_check(fmt, A, B, C, D):
    M, K = A.shape
    N = B.shape[0]
    ii, jj = np.meshgrid(np.arange(M), np.arange(N), indexing="ij")
    ab = TORCH2ORACLE[A.dtype]
    return check_gemm_samples(ab, A, B, C, D, ii.ravel(), jj.ravel(), K, f"gemm {fmt} {M}x{N}x{K}")


SMALL = [(256, 256, 128), (128, 256, 64), (512, 512, 512), (200, 136, 72), (264, 520, 40), (1, 4, 8), (384, 16, 1024)]


@pytest.mark.parametrize("cg", [1, 2])
@pytest.mark.parametrize("fmt", ["bf16", "f16", "tf32", "s8"])
@pytest.mark.parametrize("shape", SMALL)
def test_gemm_small_whole_matrix(fmt, cg, shape):
    M, N, K = shape
    if fmt == "s8":
        K = max(16, (K + 15) // 16 * 16)
    A, B, C = _problem(M, N, K, fmt, seed=M + N + K)
    D = tcx.gemm(A, B, C, tf32=(fmt == "tf32"), cta_group=cg)
    torch.cuda.synchronize()
    _full_check(fmt, A, B, C, D)


@pytest.mark.parametrize("cg", [1, 2])
@pytest.mark.parametrize("fmt", ["bf16", "tf32"])
def test_gemm_integer_valued_bit_exact(fmt, cg):
    """|a|,|b| <= 8 integers: exact sums -> bit-exact on every path (pins indexing/layout)."""
    M, N, K = 512, 768, 320
    dt = {"bf16": torch.bfloat16, "tf32": torch.float32}[fmt]
    A = tcxgen.int32_matrix((M, K), 1, 1, -8, 8, DEV).to(dt)
    B = tcxgen.int32_matrix((N, K), 1, 2, -8, 8, DEV).to(dt)
    C = tcxgen.int32_matrix((M, N), 1, 3, -1000, 1000, DEV).to(torch.float32)
    D = tcx.gemm(A, B, C, tf32=(fmt == "tf32"), cta_group=cg)
    ref = (A.double() @ B.double().T + C.double())
    torch.cuda.synchronize()
    assert torch.equal(D.double(), ref)


WIDE = [(256, 512, 128), (512, 1024, 256), (200, 600, 72), (264, 520, 40), (768, 1536, 1024), (256, 16, 64)]


@pytest.mark.parametrize("tile_n", [512])
@pytest.mark.parametrize("fmt", ["bf16", "tf32", "s8"])
@pytest.mark.parametrize("shape", WIDE)
def test_gemm_wide_tile_whole_matrix(fmt, shape, tile_n):
    """the 256 x 512 pair tile (tile_n = 512; two N-halves share A), incl. ragged M/N/K and an N
    smaller than one half."""
    M, N, K = shape
    if fmt == "s8":
        K = max(16, (K + 15) // 16 * 16)
    A, B, C = _problem(M, N, K, fmt, seed=M + 3 * N + K)
    D = tcx.gemm(A, B, C, tf32=(fmt == "tf32"), tile_n=tile_n)
    torch.cuda.synchronize()
    _full_check(fmt, A, B, C, D)


@pytest.mark.parametrize("fmt", ["bf16", "s8"])
def test_gemm_wide_equals_narrow_and_persistent(fmt):
    """wide and narrow tiles run the same MMA sequence per output element: bit-identical D; and
    the single-buffered wide accumulator survives many tiles per CTA pair (max_ctas = 2)."""
    M, N, K = 1024, 2048, 768
    A, B, C = _problem(M, N, K, fmt, seed=17)
    Dn = tcx.gemm(A, B, C, tile_n=256)
    Dw = tcx.gemm(A, B, C, tile_n=512)
    Dp = tcx.gemm(A, B, C, tile_n=512, max_ctas=2)
    torch.cuda.synchronize()
    assert torch.equal(Dn.view(torch.int32), Dw.view(torch.int32))
    assert torch.equal(Dw.view(torch.int32), Dp.view(torch.int32))


NARROW = [(256, 512, 128), (200, 600, 72), (264, 520, 40), (512, 1000, 320), (256, 96, 64)]


@pytest.mark.parametrize("width", [224, 192, 160, 128])
@pytest.mark.parametrize("fmt", ["bf16", "tf32", "s8"])
@pytest.mark.parametrize("shape", NARROW)
def test_gemm_narrow_tile_whole_matrix(fmt, shape, width):
    """the narrower pair tiles (tile_n = 224 / 192 / 160 / 128: UMMA N = width, the wave-quantisation
    choice): whole matrix against the oracle, incl. ragged M/N/K, N not a multiple of the width and
    N smaller than one tile."""
    M, N, K = shape
    if fmt == "s8":
        K = max(16, (K + 15) // 16 * 16)
    A, B, C = _problem(M, N, K, fmt, seed=M + 5 * N + K + width)
    D = tcx.gemm(A, B, C, tf32=(fmt == "tf32"), tile_n=width)
    torch.cuda.synchronize()
    _full_check(fmt, A, B, C, D)


@pytest.mark.parametrize("fmt", ["bf16", "s8", "f16acc"])
def test_gemm_narrow_equals_default_and_persistent(fmt):
    """every width runs the same per-element MMA sequence: D bit-identical to the 256-wide tile's,
    also with many tiles per CTA pair (max_ctas = 2) and for the FP16-accumulate kind; and the
    library's own choice (tile_n = 0) for a row-sharded-rank shape (1024 x 8192: 224 wide) too."""
    M, N, K = 1024, 8192 if fmt == "bf16" else 2048, 256
    if fmt == "f16acc":
        A, B, _ = _problem(M, N, K, "f16", seed=23)
        C = tcxgen.normal_matrix((M, N), "f16", 23, tcxgen.STREAM_C, DEV)
        run = lambda **kw: tcx.gemm(A, B, C, f16_acc=True, **kw)
    else:
        A, B, C = _problem(M, N, K, fmt, seed=23)
        run = lambda **kw: tcx.gemm(A, B, C, **kw)
    ref = run(tile_n=256, pairs=(1, 1))
    outs = [run(tile_n=w) for w in (224, 192, 160, 128)] + [run(tile_n=224, max_ctas=2), run()]
    torch.cuda.synchronize()
    r = ref.view(torch.int16 if fmt == "f16acc" else torch.int32)
    for o in outs:
        assert torch.equal(o.view(r.dtype), r)


@pytest.mark.parametrize("fmt,K", [("bf16", 16384), ("tf32", 8192), ("s8", 32768)])
def test_gemm_long_k_default_wide_tile(fmt, K):
    """long K loops take the 256 x 512 tile by default (K_eff >= 16384): with few pairs (max_ctas = 8)
    each pair runs several wide tiles back to back through the half-0 lookahead; D equals the
    256-wide tile's bit for bit, and sampled outputs match the oracle (bound / bit-exact INT8)."""
    M, N = 1024, 2048
    A, B, C = _problem(M, N, K, fmt, seed=K + 5)
    Dd = tcx.gemm(A, B, C, tf32=(fmt == "tf32"), max_ctas=8)
    Dn = tcx.gemm(A, B, C, tf32=(fmt == "tf32"), max_ctas=8, tile_n=256, pairs=(1, 1))
    torch.cuda.synchronize()
    assert torch.equal(Dd.view(torch.int32), Dn.view(torch.int32))
    rows, cols = gemm_sample_coords(M, N, 256, 512, nsamp=4096)
    check_gemm_samples(TORCH2ORACLE[A.dtype], A, B, C, Dd, rows, cols, K, f"long-K {fmt}")


@pytest.mark.parametrize("fmt,K", [("bf16", 16384), ("tf32", 8192)])
def test_gemm_long_k_wide_full_waves(fmt, K):
    """>= 2 full waves of long-K wide tiles (the default there): bit-identical to the plain 256-wide
    tile, oracle on samples incl. every tile corner."""
    M, N = 4096, 8192
    A, B, C = _problem(M, N, K, fmt, seed=K + 11)
    Dd = tcx.gemm(A, B, C, tf32=(fmt == "tf32"))
    Dn = tcx.gemm(A, B, C, tf32=(fmt == "tf32"), tile_n=256, pairs=(1, 1))
    torch.cuda.synchronize()
    assert torch.equal(Dd.view(torch.int32), Dn.view(torch.int32))
    rows, cols = gemm_sample_coords(M, N, 256, 512, nsamp=8192)
    check_gemm_samples(TORCH2ORACLE[A.dtype], A, B, C, Dd, rows, cols, K, f"long-K waves {fmt}")


def test_gemm_tall_m_large_coordinates():
    """maximum-size edge: ~2^20 rows (TMA row coordinates past 2^20, D > 2^33 bytes, far past any
    32-bit byte offset), ragged M and N: sampled outputs incl. the last rows / columns vs the oracle."""
    M, N, K = (1 << 20) + 200, 2048 + 8, 64
    A, B, C = _problem(M, N, K, "bf16", seed=101, with_c=False)
    D = tcx.gemm(A, B, None)
    torch.cuda.synchronize()
    rng = np.random.default_rng(3)
    rows = np.concatenate([rng.integers(0, M, 4096), np.arange(M - 300, M)])
    cols = np.concatenate([rng.integers(0, N, 4096), rng.integers(N - 40, N, 300)])
    check_gemm_samples(TORCH2ORACLE[A.dtype], A, B, None, D, rows, cols, K, "tall M")
    del A, B, D


def test_gemm_same_base_pointer_new_shape():
    """the C ABI caches tensor-map descriptors keyed on every argument: views sharing a base pointer
    with other rows / columns / strides must not reuse a stale descriptor (each result vs the oracle)"""
    A, B, C = _problem(512, 512, 128, "bf16", seed=41)
    for M, N in [(512, 512), (256, 512), (512, 256), (256, 128), (512, 512)]:
        D = tcx.gemm(A[:M], B[:N], C[:M, :N].contiguous())
        torch.cuda.synchronize()
        _full_check("bf16", A[:M], B[:N], C[:M, :N].contiguous(), D)
    Ap = torch.zeros(512, 192, dtype=torch.bfloat16, device=DEV)
    Ap[:, :128] = A                                   # same data, padded rows (row stride 192)
    D = tcx.gemm(Ap[:, :128], B, C)
    torch.cuda.synchronize()
    _full_check("bf16", A, B, C, D)


@pytest.mark.parametrize("cg", [1, 2])
def test_gemm_persistent_many_tiles_per_cta(cg):
    """few CTAs, many tiles each: exercises the smem ring and TMEM double-buffer phases."""
    M, N, K = 1024, 1280, 1024
    A, B, C = _problem(M, N, K, "bf16", seed=3)
    D = tcx.gemm(A, B, C, cta_group=cg, max_ctas=2 * cg)
    D2 = tcx.gemm(A, B, C, cta_group=cg)
    torch.cuda.synchronize()
    assert torch.equal(D.view(torch.int32), D2.view(torch.int32))   # same per-element arithmetic
    rows, cols = gemm_sample_coords(M, N, 128 * cg, 256, nsamp=8192)
    check_gemm_samples(O.BF16, A, B, C, D, rows, cols, K, "persistent")


def test_gemm_no_c_k0_and_errors():
    A, B, _ = _problem(256, 256, 64, "bf16", seed=4, with_c=False)
    D = tcx.gemm(A, B, None)
    torch.cuda.synchronize()
    _full_check("bf16", A, B, None, D)
    # K == 0: D = C
    C = torch.randn(64, 32, device=DEV)
    D0 = tcx.gemm(A[:64, :0], B[:32, :0], C)
    torch.cuda.synchronize()
    assert torch.equal(D0, C)
    # misaligned K (K*2 % 16 != 0) is rejected, not computed
    A2 = torch.zeros(64, 12, dtype=torch.bfloat16, device=DEV)
    B2 = torch.zeros(64, 12, dtype=torch.bfloat16, device=DEV)
    with pytest.raises(tcx.TcxError):
        tcx.gemm(A2, B2)


def test_gemm_determinism_and_cta_modes_agree():
    A, B, C = _problem(1024, 1024, 2048, "bf16", seed=6)
    D1 = tcx.gemm(A, B, C, cta_group=1)
    D2 = tcx.gemm(A, B, C, cta_group=2)
    D3 = tcx.gemm(A, B, C, cta_group=2)
    torch.cuda.synchronize()
    assert torch.equal(D2.view(torch.int32), D3.view(torch.int32))
    # both modes are inside the bound; they need not be bitwise equal
    rows, cols = gemm_sample_coords(1024, 1024, 256, 256, nsamp=4096)
    check_gemm_samples(O.BF16, A, B, C, D1, rows, cols, 2048, "cg1")


def _float64_full_coverage(A, B, C, D, K):
    """every output vs float64 A.B (a library routine used as a check, not the oracle):
    |D - ref64| <= (K+2) 2^-23 (|A||B| + |C|) + K 2^-52 (|A||B|) for all M*N outputs."""
    Ad, Bd = A.double(), B.double()
    ref = Ad @ Bd.T
    mag = Ad.abs() @ Bd.abs().T
    if C is not None:
        ref += C.double()
        mag += C.double().abs()
    err = (D.double() - ref).abs()
    bound = (K + 2) * 2.0 ** -23 * mag + K * 2.0 ** -52 * mag
    bad = int((err > bound).sum())
    assert bad == 0, f"{bad} outputs exceed the bound"
    return float((err / (2.0 ** -23 * mag).clamp_min(1e-300)).max())


@pytest.mark.parametrize("fmt", ["bf16", "tf32"])
def test_config3_full_size(fmt):
    """BASELINE configs[2]: M=N=K=8192, A,B N(0,1) (BF16, or FP32 rounded to TF32), C FP32 zeros."""
    M = N = K = 8192
    A, B, _ = _problem(M, N, K, fmt, seed=0, with_c=False)
    C = torch.zeros(M, N, dtype=torch.float32, device=DEV)
    D = tcx.gemm(A, B, C, tf32=(fmt == "tf32"))
    torch.cuda.synchronize()
    rows, cols = gemm_sample_coords(M, N, 256, 256, nsamp=65536)
    norm = check_gemm_samples(TORCH2ORACLE[A.dtype], A, B, C, D, rows, cols, K, f"C3 {fmt}")
    assert norm < K + 2
    _float64_full_coverage(A, B, C, D, K)
    # bit for bit: 4096 sampled outputs against the observed instruction model chained over K
    # (Ki = 16 BF16 / 8 TF32 per tcgen05.mma; DESIGN.md §7 finding 3b)
    r, c = rows[:4096], cols[:4096]
    Ah, Bh = host_bits(A), host_bits(B)
    pred = model_predict(TORCH2ORACLE[A.dtype], Ah[r], Bh[c], np.zeros(r.size, np.float32), Ki=8 if fmt == "tf32" else 16)
    got = host_bits(D)[r, c]
    assert np.array_equal(pred, got), int((pred != got).sum())


def test_config4_full_size_int8_bit_exact():
    """BASELINE configs[3]: INT8 16384^3, C int32 U[-2^20, 2^20]: bit-exact; Freivalds mod 2^32
    on all outputs."""
    M = N = K = 16384
    A, B, C = _problem(M, N, K, "s8", seed=0)
    D = tcx.gemm(A, B, C)
    torch.cuda.synchronize()
    rows, cols = gemm_sample_coords(M, N, 256, 256, nsamp=65536)
    check_gemm_samples(O.S8, A, B, C, D, rows, cols, K, "C4")
    # Freivalds, exact mod 2^32: float64 products are exact here (|D r| < 2^52, |A (B r)| < 2^49)
    g = torch.Generator(device=DEV).manual_seed(1)
    Dd, Ad, Bd, Cd = D.double(), A.double(), B.double(), C.double()
    for _ in range(8):
        r = torch.randint(0, 128, (N, 1), device=DEV, generator=g).double()
        lhs = (Dd @ r).long()
        rhs = (Ad @ (Bd.T @ r) + Cd @ r).long()   # D = A B^T (B stored N x K)
        assert torch.equal((lhs - rhs) & 0xFFFFFFFF, torch.zeros_like(lhs))


@pytest.mark.parametrize("fmt", ["bf16", "s8"])
def test_gemm_in_place_d_aliases_c(fmt):
    """D may alias C (include/tcx.h): every C chunk is read before the D chunk at the same place is
    written (TMA-store epilogue), so in-place equals out-of-place bit for bit."""
    M, N, K = 512, 768, 256
    A, B, C = _problem(M, N, K, fmt, seed=31)
    D = tcx.gemm(A, B, C)
    C2 = C.clone()
    tcx.gemm(A, B, C2, C2)
    torch.cuda.synchronize()
    assert torch.equal(D.view(torch.int32), C2.view(torch.int32))


def test_gemm_bad_tile_n_rejected():
    A, B, C = _problem(256, 256, 64, "bf16", seed=1)
    with pytest.raises(tcx.TcxError):
        tcx.gemm(A, B, C, tile_n=384)


MC_SHAPES = [(256, 256, 128), (512, 512, 512), (200, 600, 72), (264, 520, 40), (768, 1280, 1024), (1, 4, 8),
             (1300, 260, 192)]


@pytest.mark.parametrize("pairs", [(1, 2), (2, 1), (2, 2)])
@pytest.mark.parametrize("fmt", ["bf16", "tf32", "s8"])
@pytest.mark.parametrize("shape", MC_SHAPES)
def test_gemm_multicast_cluster_whole_matrix(fmt, shape, pairs):
    """TMA-multicast clusters of CTA pairs (tcx_gemm_opts.pairs_m/pairs_n): ragged M/N/K, shapes whose
    pair-tile count is odd (a pair past the edge computes on zero fill and feeds the others)."""
    M, N, K = shape
    if fmt == "s8":
        K = max(16, (K + 15) // 16 * 16)
    A, B, C = _problem(M, N, K, fmt, seed=M + 5 * N + K)
    D = tcx.gemm(A, B, C, tf32=(fmt == "tf32"), pairs=pairs)
    torch.cuda.synchronize()
    _full_check(fmt, A, B, C, D)


@pytest.mark.parametrize("fmt", ["bf16", "s8", "f16acc"])
def test_gemm_multicast_equals_default_and_persistent(fmt):
    """a multicast cluster changes who loads which operand rows, not the MMA sequence: D is bit-
    identical to the default pair kernel's, also with few clusters looping over many tiles."""
    M, N, K = 1536, 2304, 1024
    if fmt == "f16acc":
        A, B, _ = _problem(M, N, K, "f16", seed=23, with_c=False)
        C = tcxgen.normal_matrix((M, N), "f16", 23, tcxgen.STREAM_C, DEV)
        kw = dict(f16_acc=True)
        view = torch.int16
    else:
        A, B, C = _problem(M, N, K, fmt, seed=23)
        kw = {}
        view = torch.int32
    ref = tcx.gemm(A, B, C, **kw)
    for pairs in [(1, 2), (2, 1), (2, 2)]:
        for max_ctas in (0, 8, 16):
            D = tcx.gemm(A, B, C, pairs=pairs, max_ctas=max_ctas, **kw)
            torch.cuda.synchronize()
            assert torch.equal(ref.view(view), D.view(view)), (pairs, max_ctas)


def test_gemm_multicast_config3_full_size():
    """BASELINE configs[2] through the 2 x 2 multicast cluster: sampled oracle parity + full-coverage bound."""
    M = N = K = 8192
    A, B, _ = _problem(M, N, K, "bf16", seed=0, with_c=False)
    C = torch.zeros(M, N, dtype=torch.float32, device=DEV)
    D = tcx.gemm(A, B, C, pairs=(2, 2))
    torch.cuda.synchronize()
    rows, cols = gemm_sample_coords(M, N, 256, 256, nsamp=65536)
    check_gemm_samples(O.BF16, A, B, C, D, rows, cols, K, "C3 mc22")
    _float64_full_coverage(A, B, C, D, K)


def test_gemm_bad_pairs_rejected():
    A, B, C = _problem(256, 256, 64, "bf16", seed=1)
    for kw in (dict(pairs=(3, 1)), dict(pairs=(2, 1), cta_group=1), dict(pairs=(1, 2), tile_n=512)):
        with pytest.raises(tcx.TcxError):
            tcx.gemm(A, B, C, **kw)


@pytest.mark.parametrize("group_m", [-1, -3, -8, 5])
def test_gemm_raster_orders_bit_identical(group_m):
    """the raster (group_m > 0: M-groups sweeping N; < 0: N-groups sweeping M) only reorders tiles:
    D is bit-identical to the default, also with a persistent grid of few CTAs."""
    M, N, K = 1300, 1800, 320
    A, B, C = _problem(M, N, K, "bf16", seed=29)
    ref = tcx.gemm(A, B, C)
    D = tcx.gemm(A, B, C, group_m=group_m)
    Dp = tcx.gemm(A, B, C, group_m=group_m, max_ctas=6)
    torch.cuda.synchronize()
    assert torch.equal(ref.view(torch.int32), D.view(torch.int32))
    assert torch.equal(ref.view(torch.int32), Dp.view(torch.int32))
