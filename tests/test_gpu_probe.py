"""tcx_probe (clock-counter latency/throughput) and the tcgen05 numeric-probe
tile path (tcx_mma_tiles_tc05) on B200.

The tcgen05 rows are checked for what they claim, not by re-deriving the probe's
own formula: every timed run below also reads issuer 0's accumulators back and compares them
bit for bit with the oracle's chain of the same MMAs — accumulator a received
(warmup + ITERS) x |{i < ILP : i % n_acc == a}| MMAs of the probe operands, which is ONE dot
product of that many repeated K-blocks (oracle.gemm_samples on the K-tiled operands).  Operands
are in {-1, 0, 1}, so every partial sum is an integer below 2^24 and the FP32 chain is exact
whatever the hardware's accumulation order: a missing or extra MMA changes the result."""
import numpy as np
import pytest
import torch

import oracle as O
import tcxgen
import paper_2206_02874_b200 as tcx
from parity import host_bits, fp_bound_check

pytestmark = pytest.mark.gpu
DEV = "cuda"
NSM = 148


def test_completion_latency_and_identity():
    r = tcx.probe("mma_sync", tcx.F16, tcx.F32, 16, 8, 16, warps=1, ilp=1, iters=2048, repeats=3)
    lat = r["latency_cycles"]
    assert 5 < lat < 200, r
    assert 300 < r["sm_mhz"] < 2200


def test_throughput_grows_with_warps_and_ilp():
    lo = tcx.probe("mma_sync", tcx.BF16, tcx.F32, 16, 8, 16, warps=1, ilp=1, iters=1024)["fma_per_clk_per_sm"]
    hi = tcx.probe("mma_sync", tcx.BF16, tcx.F32, 16, 8, 16, warps=8, ilp=4, iters=1024)["fma_per_clk_per_sm"]
    assert hi > 2 * lo


@pytest.mark.parametrize("ab,m,n,k", [(tcx.F16, 16, 8, 8), (tcx.TF32, 16, 8, 8), (tcx.TF32, 16, 8, 4),
                                      (tcx.S8, 8, 8, 16), (tcx.S8, 16, 8, 32), (tcx.S8, 16, 8, 16)])
def test_every_dense_shape_runs(ab, m, n, k):
    cd = tcx.S32 if ab == tcx.S8 else tcx.F32
    r = tcx.probe("mma_sync", ab, cd, m, n, k, warps=4, ilp=2, iters=256, repeats=2)
    assert r["latency_cycles"] > 0


@pytest.mark.parametrize("ab,k", [(tcx.F16, 32), (tcx.F16, 16), (tcx.BF16, 32), (tcx.TF32, 16), (tcx.TF32, 8),
                                  (tcx.S8, 64), (tcx.S8, 32)])
def test_every_sparse_shape_runs(ab, k):
    cd = tcx.S32 if ab == tcx.S8 else tcx.F32
    r = tcx.probe("mma_sp_sync", ab, cd, 16, 8, k, warps=4, ilp=2, iters=256, repeats=2)
    assert r["latency_cycles"] > 0


# ------------------------------------------------------------------------------- tcgen05 rows
_OFMT = {tcx.F16: O.F16, tcx.BF16: O.BF16, tcx.TF32: O.TF32, tcx.S8: O.S8}
_TDT = {tcx.F16: torch.float16, tcx.BF16: torch.bfloat16, tcx.TF32: torch.float32, tcx.S8: torch.int8}
_ES = {tcx.F16: 2, tcx.BF16: 2, tcx.TF32: 4, tcx.S8: 1}


def _operands(ab, rows_a, n, sparse, seed):
    """A: rows_a x 32 bytes (kept values if sparse), B: n x (64 if sparse else 32) bytes, values in
    {-1, 0, 1} (kept A values nonzero)."""
    es = _ES[ab]
    ka = 32 // es
    kb = (64 if sparse else 32) // es
    a = tcxgen.int32_matrix((rows_a, ka), seed, 1, -1, 1, DEV)
    if sparse:
        a = torch.where(a == 0, torch.ones_like(a), a)
    b = tcxgen.int32_matrix((n, kb), seed, 2, -1, 1, DEV)
    return a.to(_TDT[ab]).contiguous(), b.to(_TDT[ab]).contiguous()


def _mma_counts(r, ilp, iters):
    n_acc = r["n_acc"]
    per_iter = [len([i for i in range(ilp) if i % n_acc == a]) for a in range(n_acc)]
    return [(r["warmup_iters"] + iters) * p for p in per_iter]


def _check_accumulators(ab, sparse, a_op, b_op, acc, counts, nsamp=192, seed=0):
    """every accumulator equals the oracle's chain of counts[a] MMAs (sampled elements, bitwise)"""
    A = host_bits(a_op)
    B = host_bits(b_op)
    K1 = B.shape[1]                                          # logical K of one MMA
    if sparse:
        words = K1 // 32 if K1 >= 32 else 1
        # metadata: every 4-group keeps (0, 1) -> nibble 0x4; TF32 1:2 in 16-bit halves is (0, 2) in
        # canonical TF32 groups -> 0x8 (the first element of each aligned pair)
        nib = 0x88888888 if ab == tcx.TF32 else 0x44444444
        meta = np.full((A.shape[0], max(1, K1 // 32)), nib, dtype=np.uint32)
        Kpad = max(K1, 32)
        Ap = np.zeros((A.shape[0], Kpad // 2), dtype=A.dtype); Ap[:, :A.shape[1]] = A
        A = O.sp24_expand(Ap, meta, Kpad)[:, :K1]
        del words
    rng = np.random.default_rng(seed)
    got = host_bits(acc)                                     # (n_acc, rows, n) uint32
    for a, cnt in enumerate(counts):
        rows = rng.integers(0, A.shape[0], nsamp)
        cols = rng.integers(0, B.shape[0], nsamp)
        ref, _ = O.gemm_samples(_OFMT[ab], np.tile(A, (1, cnt)), np.tile(B, (1, cnt)), None, rows, cols)
        g = got[a][rows, cols]
        bad = np.nonzero(g != ref)[0]
        assert bad.size == 0, (f"accumulator {a} ({cnt} MMAs): {bad.size} of {nsamp} sampled elements differ; "
                               f"first ({rows[bad[0]]}, {cols[bad[0]]}) got {g[bad[0]]:#x} oracle {ref[bad[0]]:#x}")


def _tc05(kind, ab, m, n, cg, mode, ilp, iters, n_acc=0, issuers=1, num_sms=1, readback=True, seed=0, repeats=3):
    sparse = kind == "tc05_sp"
    k = (64 if sparse else 32) // _ES[ab]
    cd = tcx.S32 if ab == tcx.S8 else tcx.F32
    a_op = b_op = acc = None
    if readback:
        a_op, b_op = _operands(ab, m, n, sparse, seed)
        nacc = n_acc or min(ilp, ((512 // issuers) - (8 if sparse else 0)) // n)
        acc = torch.zeros((nacc, m, n), dtype=torch.int32, device=DEV)
    r = tcx.probe(kind, ab, cd, m, n, k, cta_group=cg, ilp=ilp, iters=iters, repeats=repeats, num_sms=num_sms,
                  issuers=issuers, n_acc=n_acc, mode=mode, a_op=a_op, b_op=b_op, acc_out=acc)
    torch.cuda.synchronize()
    if readback:
        assert r["n_acc"] == acc.shape[0]
        _check_accumulators(ab, sparse, a_op, b_op, acc, _mma_counts(r, ilp, iters), seed=seed)
    return r


NOMINAL = {tcx.F16: 4096, tcx.BF16: 4096, tcx.TF32: 2048, tcx.S8: 8192}      # dense FMA/clk/SM


@pytest.mark.parametrize("ab", [tcx.BF16, tcx.F16, tcx.TF32, tcx.S8])
def test_tc05_stream_chain_rate_and_count(ab):
    """one dependent chain (n_acc = 1) of m256n256 MMAs per CTA pair on every SM, no wait until the
    end: the tensor pipe's own rate, >= 95% of the nominal per-SM peak, and the accumulators prove
    that every counted MMA ran."""
    r = _tc05("tc05", ab, 256, 256, 2, "stream", ilp=16, iters=256, n_acc=1, num_sms=NSM)
    assert r["mmas_per_issuer"] == 16 * 256
    assert r["fma_per_clk_per_sm"] >= 0.95 * NOMINAL[ab], r


@pytest.mark.parametrize("ab", [tcx.F16, tcx.BF16, tcx.TF32, tcx.S8])
def test_tc05_sparse_stream_rate_and_count(ab):
    """2:4 (TF32 1:2) tcgen05.mma.sp: dense-equivalent rate well above the dense pipe's, exact count"""
    r = _tc05("tc05_sp", ab, 256, 240, 2, "stream", ilp=16, iters=256, n_acc=1, num_sms=NSM)
    assert r["fma_per_clk_per_sm"] >= 1.6 * NOMINAL[ab], r


@pytest.mark.parametrize("kind,ab,n", [("tc05", tcx.BF16, 256), ("tc05_sp", tcx.F16, 240), ("tc05", tcx.S8, 256)])
@pytest.mark.parametrize("mode", ["stream_rot", "stream_areuse"])
def test_tc05_rotating_operands_count(kind, ab, n, mode):
    """a GEMM-like smem read pattern (4-stage ring, every k-offset) and A shared by two MMAs through
    the collector (fill / lastuse): the same MMA count and result, at the pipe's rate"""
    n_acc = 2 if mode == "stream_areuse" else 1
    r = _tc05(kind, ab, 256, n, 2, mode, ilp=16, iters=128, n_acc=n_acc, num_sms=NSM)
    lo = (1.6 if kind == "tc05_sp" else 0.95) * NOMINAL[ab]
    assert r["fma_per_clk_per_sm"] >= lo, r


@pytest.mark.parametrize("cg,m", [(1, 128), (2, 256)])
def test_tc05_sync_mode_count_and_ilp(cg, m):
    """the paper's per-iteration sync: ILP MMAs over n_acc accumulators, commit + wait each
    iteration; every accumulator's count checked (uneven rotation: ilp % n_acc != 0)"""
    r = _tc05("tc05", tcx.BF16, m, 128, cg, "sync", ilp=5, iters=64, n_acc=3)
    assert r["n_acc"] == 3 and r["mmas_per_issuer"] == 5 * 64


def test_tc05_latency_split():
    """completion latency (ILP 1, SYNC) = MMA + commit round trip; COMMIT mode measures the round
    trip alone, so the MMA part is their difference (both positive)"""
    lat = _tc05("tc05", tcx.BF16, 128, 256, 1, "sync", ilp=1, iters=512, readback=False)["latency_cycles"]
    com = _tc05("tc05", tcx.BF16, 128, 256, 1, "commit", ilp=1, iters=512, readback=False)["latency_cycles"]
    assert 0 < com < lat < 5000, (com, lat)


def test_tc05_two_issuers_per_sm():
    """issuers = 2: two CTAs share every SM (each with 256 TMEM columns), verified by %smid"""
    r = _tc05("tc05", tcx.BF16, 128, 256, 1, "stream", ilp=8, iters=128, n_acc=1, issuers=2, num_sms=NSM)
    assert r["max_issuers_per_sm"] == 2 and r["sms_used"] == NSM, r
    # two streams per SM share the one tensor pipe: the per-SM rate stays at the pipe's
    assert 0.9 * 4096 <= r["fma_per_clk_per_sm"] <= 1.02 * 4096, r
    p2 = _tc05("tc05", tcx.BF16, 256, 256, 2, "sync", ilp=4, iters=64, n_acc=1, issuers=2, num_sms=NSM)
    assert p2["max_issuers_per_sm"] == 2 and p2["sms_used"] == NSM, p2


def test_tc05_argument_errors():
    with pytest.raises(tcx.TcxError):
        tcx.probe("tc05", tcx.BF16, tcx.F32, 128, 256, 16, ilp=2, n_acc=3)          # n_acc > ilp
    with pytest.raises(tcx.TcxError):
        tcx.probe("tc05", tcx.BF16, tcx.F32, 128, 256, 16, ilp=2, issuers=3)
    with pytest.raises(tcx.TcxError):
        tcx.probe("tc05", tcx.BF16, tcx.F32, 128, 256, 16, ilp=2, mode=7)


def _tiles(count, fmt, seed, k=16):
    A = tcxgen.uniform_matrix((count, 16, k), fmt, seed, tcxgen.STREAM_A, device=DEV)
    B = tcxgen.uniform_matrix((count, 8, k), fmt, seed, tcxgen.STREAM_B, device=DEV)
    C = tcxgen.uniform_matrix((count, 16, 8), "f32", seed, tcxgen.STREAM_C, device=DEV)
    return A, B, C


@pytest.mark.parametrize("fmt,k", [("f16", 16), ("bf16", 16), ("tf32", 8), ("tf32", 16)])
@pytest.mark.parametrize("count", [1, 9, 1000])
def test_tiles_tc05_vs_oracle(fmt, k, count):
    A, B, C = _tiles(count, fmt, count + k, k)
    D = tcx.mma_tiles_tc05(A, B, C, tf32=(fmt == "tf32"))
    torch.cuda.synchronize()
    of = {"f16": O.F16, "bf16": O.BF16, "tf32": O.TF32}[fmt]
    ref, absv = O.tiles(of, 16, 8, k, host_bits(A), host_bits(B), host_bits(C))
    fp_bound_check(host_bits(D).reshape(ref.shape), ref, absv, k, f"tc05 tiles {fmt}")


def test_tiles_tc05_integer_bit_exact():
    count = 512
    A = tcxgen.int32_matrix((count, 16, 16), 2, 1, -8, 8, DEV).to(torch.float16)
    B = tcxgen.int32_matrix((count, 8, 16), 2, 2, -8, 8, DEV).to(torch.float16)
    C = tcxgen.int32_matrix((count, 16, 8), 2, 3, -999, 999, DEV).to(torch.float32)
    D = tcx.mma_tiles_tc05(A, B, C)
    torch.cuda.synchronize()
    ref, _ = O.tiles(O.F16, 16, 8, 16, host_bits(A), host_bits(B), host_bits(C))
    assert np.array_equal(host_bits(D).reshape(ref.shape), ref)
