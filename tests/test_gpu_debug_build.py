"""The debug library (libtcx_debug.so: every mbarrier wait bounded by a globaltimer watchdog, plus
a fault-injection hook) — SURVEY §5 "race detection / failure detection": a pipeline bug must end
as an error returned to the caller, never as a hung GPU.  Each case runs in a subprocess with
TCX_LIB_PATH naming the debug build (a trapped kernel poisons its CUDA context)."""
import os
import subprocess
import sys
import textwrap

import numpy as np
import pytest
import torch

import tcxgen
import paper_2206_02874_b200 as tcx

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DEBUG_LIB = os.path.join(ROOT, "paper_2206_02874_b200", "libtcx_debug.so")


def _run(code, tmp_path, timeout=120):
    if not os.path.exists(DEBUG_LIB):
        from paper_2206_02874_b200 import build as b
        b.build(debug=True)
    env = dict(os.environ, TCX_LIB_PATH=DEBUG_LIB, PYTHONPATH=ROOT)
    script = tmp_path / "case.py"
    script.write_text(textwrap.dedent(code))
    return subprocess.run([sys.executable, str(script)], env=env, capture_output=True, text=True, timeout=timeout,
                          cwd=str(tmp_path))


PROBLEM = """
import numpy as np, torch
import tcxgen, paper_2206_02874_b200 as tcx
assert tcx.LIB_PATH.endswith("libtcx_debug.so"), tcx.LIB_PATH
dev = "cuda"
A = tcxgen.normal_matrix((512, 320), "bf16", 5, tcxgen.STREAM_A, dev)
B = tcxgen.normal_matrix((768, 320), "bf16", 5, tcxgen.STREAM_B, dev)
C = tcxgen.normal_matrix((512, 768), "f32", 5, tcxgen.STREAM_C, dev)
"""


def test_debug_library_matches_product(tmp_path):
    """the watchdog changes no arithmetic: dense (default and multicast groups), sparse and tile
    results from the debug build are bit-identical to the product build's."""
    code = PROBLEM + """
vals, meta = tcxgen.sp24_problem(512, 256, 6, "f16", dev)
Bs = tcxgen.normal_matrix((480, 256), "f16", 6, tcxgen.STREAM_B, dev)
hw = tcx.sp24_pack_meta(meta, 512, 256)
At = tcxgen.uniform_matrix((64, 16, 16), "f16", 0, 1, device=dev)
Bt = tcxgen.uniform_matrix((64, 8, 16), "f16", 0, 2, device=dev)
out = {"d": tcx.gemm(A, B, C), "d22": tcx.gemm(A, B, C, pairs=(2, 2)), "s": tcx.gemm_sp24(vals, hw, Bs, None),
       "t": tcx.mma_tiles(At, Bt, None)}
torch.cuda.synchronize()
np.savez("out.npz", **{k: v.cpu().view(torch.int32).numpy() for k, v in out.items()})
print("OK")
"""
    r = _run(code, tmp_path)
    assert r.returncode == 0 and "OK" in r.stdout, r.stderr[-2000:]
    got = np.load(tmp_path / "out.npz")
    dev = "cuda"
    A = tcxgen.normal_matrix((512, 320), "bf16", 5, tcxgen.STREAM_A, dev)
    B = tcxgen.normal_matrix((768, 320), "bf16", 5, tcxgen.STREAM_B, dev)
    C = tcxgen.normal_matrix((512, 768), "f32", 5, tcxgen.STREAM_C, dev)
    vals, meta = tcxgen.sp24_problem(512, 256, 6, "f16", dev)
    Bs = tcxgen.normal_matrix((480, 256), "f16", 6, tcxgen.STREAM_B, dev)
    hw = tcx.sp24_pack_meta(meta, 512, 256)
    At = tcxgen.uniform_matrix((64, 16, 16), "f16", 0, 1, device=dev)
    Bt = tcxgen.uniform_matrix((64, 8, 16), "f16", 0, 2, device=dev)
    ref = {"d": tcx.gemm(A, B, C), "d22": tcx.gemm(A, B, C), "s": tcx.gemm_sp24(vals, hw, Bs, None),
           "t": tcx.mma_tiles(At, Bt, None)}
    torch.cuda.synchronize()
    for k, v in ref.items():
        assert np.array_equal(got[k], v.cpu().view(torch.int32).numpy()), k


def test_watchdog_turns_a_stalled_pipeline_into_an_error(tmp_path):
    """fault injection: the producer drops one TMA load, so a full barrier never completes; the
    MMA warp's bounded wait traps and the caller gets a CUDA error (not a hang)."""
    code = PROBLEM + """
import time
t0 = time.time()
try:
    D = tcx.gemm(A, B, C, _fault=1)
    torch.cuda.synchronize()
    print("NO_ERROR")
except Exception as e:
    print("TRAPPED", round(time.time() - t0, 1), type(e).__name__, str(e).splitlines()[0][:200])
"""
    r = _run(code, tmp_path, timeout=90)
    assert "TRAPPED" in r.stdout, (r.stdout[-1000:], r.stderr[-2000:])
    secs = float(r.stdout.split("TRAPPED")[1].split()[0])
    assert secs < 60


def test_product_library_ignores_the_fault_hook():
    """the product build has no fault injection: reserved[0] = 1 computes normally."""
    A = tcxgen.normal_matrix((256, 128), "bf16", 1, tcxgen.STREAM_A, "cuda")
    B = tcxgen.normal_matrix((256, 128), "bf16", 1, tcxgen.STREAM_B, "cuda")
    D1 = tcx.gemm(A, B, None, _fault=1)
    D0 = tcx.gemm(A, B, None)
    torch.cuda.synchronize()
    assert torch.equal(D0, D1)


def test_tile_trace_records_every_tile(tmp_path):
    """tcx_debug_trace: one record per cluster tile, start <= MMA end <= epilogue end, each pair's
    tiles in raster order; the product library refuses the call."""
    code = PROBLEM + """
M, N, K = 1024, 1536, 512
A = tcxgen.normal_matrix((M, K), "bf16", 8, tcxgen.STREAM_A, dev)
B = tcxgen.normal_matrix((N, K), "bf16", 8, tcxgen.STREAM_B, dev)
T = (M // 256) * (N // 256)
buf = torch.zeros(4 * T, dtype=torch.int64, device=dev)
tcx.debug_trace(buf)
D = tcx.gemm(A, B, None, max_ctas=8)
torch.cuda.synchronize()
tcx.debug_trace(None)
np.save("trace.npy", buf.view(T, 4).cpu().numpy())
print("OK")
"""
    r = _run(code, tmp_path)
    assert r.returncode == 0 and "OK" in r.stdout, r.stderr[-2000:]
    t = np.load(tmp_path / "trace.npy").astype(np.int64)
    assert np.array_equal(t[:, 0] & 0xFFFFFFFF, np.arange(len(t)))
    assert np.all(t[:, 1] > 0) and np.all(t[:, 1] <= t[:, 2]) and np.all(t[:, 2] <= t[:, 3])
    pair = t[:, 0] >> 32
    assert set(pair.tolist()) == set(range(4))                    # max_ctas = 8: four pairs
    for p in range(4):
        s = t[pair == p, 1]
        assert np.all(np.diff(s) > 0)                             # a pair's tiles run in order
    with pytest.raises(tcx.TcxError):
        tcx.debug_trace(torch.zeros(8, dtype=torch.int64, device="cuda"))


def test_wave_aware_width_choice(tmp_path):
    """the library's tile-width choice (gemm_dense.cu wave_tile_width), observed through the debug
    tile timeline: 1024 x 8192 (C3's rows per GPU at 8 ranks) runs 4 x 37 = 148 tiles of 256 x 224
    (2 full waves on 74 pairs) instead of 4 x 32 = 128 256-wide tiles; forcing tile_n = 256 gives
    128; 8192 x 8192 keeps the 256-wide tile (1024 tiles of the 1 x 2 groups: 512 cluster tiles)."""
    code = PROBLEM + """
def tiles_run(M, N, **kw):
    A = tcxgen.normal_matrix((M, 64), "bf16", 9, tcxgen.STREAM_A, dev)
    B = tcxgen.normal_matrix((N, 64), "bf16", 9, tcxgen.STREAM_B, dev)
    buf = torch.zeros(4 * 2048, dtype=torch.int64, device=dev)
    tcx.debug_trace(buf)
    tcx.gemm(A, B, None, **kw)
    torch.cuda.synchronize()
    tcx.debug_trace(None)
    r = buf.view(-1, 4).cpu()
    ok = ((r[:, 0] & 0xFFFFFFFF) == torch.arange(len(r))) & (r[:, 1] > 0)   # tile records (chunk stamps follow)
    return int(ok.int().cumprod(0).sum())
print("TILES", tiles_run(1024, 8192), tiles_run(1024, 8192, tile_n=256), tiles_run(8192, 8192))
"""
    r = _run(code, tmp_path)
    assert r.returncode == 0 and "TILES" in r.stdout, r.stderr[-2000:]
    got = [int(x) for x in r.stdout.split("TILES")[1].split()]
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    if sms == 148:
        assert got == [148, 128, 512], got
    else:                                            # another part: the choice only has to be consistent
        assert got[1] == 128 and got[0] >= 128, got


def test_dense_default_tile_choices(tmp_path):
    """the library's dense tile choices (gemm_dense.cu), read from the debug build's launch report:
    C3 (BF16 8192^3) runs 256 x 256 tiles in 1 x 2 multicast groups; a long K loop (BF16 K = 16384,
    TF32 K = 8192) the 256 x 512 tile; a row-sharded rank (1024 x 8192) the 256 x 224 tile."""
    code = PROBLEM + """
def run(fmt, M, N, K):
    A = tcxgen.normal_matrix((M, K), fmt, 9, tcxgen.STREAM_A, dev)
    B = tcxgen.normal_matrix((N, K), fmt, 9, tcxgen.STREAM_B, dev)
    tcx.gemm(A, B, None, tf32=(fmt == "tf32"))
    torch.cuda.synchronize()
run("bf16", 8192, 8192, 8192)
run("bf16", 8192, 8192, 16384)
run("tf32", 8192, 8192, 8192)
run("bf16", 1024, 8192, 8192)
print("OK")
"""
    env_keep = os.environ.get("TCX_DEBUG_LAUNCH")
    os.environ["TCX_DEBUG_LAUNCH"] = "1"
    try:
        r = _run(code, tmp_path)
    finally:
        if env_keep is None:
            del os.environ["TCX_DEBUG_LAUNCH"]
        else:
            os.environ["TCX_DEBUG_LAUNCH"] = env_keep
    assert r.returncode == 0 and "OK" in r.stdout, r.stderr[-2000:]
    lines = [ln for ln in r.stderr.splitlines() if ln.startswith("tcx_gemm:")]
    assert len(lines) == 4, r.stderr[-2000:]
    if torch.cuda.get_device_properties(0).multi_processor_count == 148:
        assert "pairs 1x2), tile 256x256" in lines[0], lines[0]
        assert "tile 256x512" in lines[1] and "tile 256x512" in lines[2], lines[1:3]
        assert "tile 256x224" in lines[3], lines[3]


def test_sparse_tile_trace(tmp_path):
    """tcx_debug_trace on the 2:4 kernel (narrow and M-wide tiles): every tile recorded, in order."""
    code = """
import numpy as np, torch
import tcxgen, paper_2206_02874_b200 as tcx
dev = "cuda"
M, N, K = 1024, 960, 512
vals, meta = tcxgen.sp24_problem(M, K, 4, "f16", dev)
B = tcxgen.normal_matrix((N, K), "f16", 4, tcxgen.STREAM_B, dev)
hw = tcx.sp24_pack_meta(meta, M, K)
out = {}
for tm in (0, 512):
    T = (M // (512 if tm else 256)) * (N // 240)
    buf = torch.zeros(4 * T, dtype=torch.int64, device=dev)
    tcx.debug_trace(buf)
    tcx.gemm_sp24(vals, hw, B, None, tile_m=tm or 256, max_ctas=4)
    torch.cuda.synchronize()
    tcx.debug_trace(None)
    out[str(tm)] = buf.view(T, 4).cpu().numpy()
np.savez("tr.npz", **out)
print("OK")
"""
    r = _run(code, tmp_path)
    assert r.returncode == 0 and "OK" in r.stdout, r.stderr[-2000:]
    z = np.load(tmp_path / "tr.npz")
    for k in z.files:
        t = z[k].astype(np.int64)
        assert np.array_equal(t[:, 0] & 0xFFFFFFFF, np.arange(len(t))), k
        assert np.all(t[:, 1] > 0) and np.all(t[:, 1] <= t[:, 2]) and np.all(t[:, 2] <= t[:, 3]), k


def test_chunk_phase_stamps(tmp_path):
    """With a buffer past the tile records, the dense epilogue stamps its chunk phases (tcx.h):
    for each epilogue warp, tiles it ran and chunks 0..CH-1, the seven phase stamps are in
    order, chunks follow one another, and the tile's accumulator-full wait brackets chunk 0."""
    code = PROBLEM + """
M, N, K = 2048, 1024, 256
A = tcxgen.normal_matrix((M, K), "bf16", 9, tcxgen.STREAM_A, dev)
B = tcxgen.normal_matrix((N, K), "bf16", 9, tcxgen.STREAM_B, dev)
C = tcxgen.normal_matrix((M, N), "f32", 9, tcxgen.STREAM_C, dev)
T, CH = (M // 256) * (N // 256), 8
buf = torch.zeros(4 * (T + 48 * CH), dtype=torch.int64, device=dev)
tcx.debug_trace(buf)
D = tcx.gemm(A, B, C, max_ctas=2)              # one pair: cluster 0 runs all T tiles
torch.cuda.synchronize()
tcx.debug_trace(None)
assert torch.equal(D, tcx.gemm(A, B, C))
np.save("st.npy", buf[4 * T:].view(4, 6, CH, 8).cpu().numpy())
print("OK")
"""
    r = _run(code, tmp_path)
    assert r.returncode == 0 and "OK" in r.stdout, r.stderr[-2000:]
    st = np.load(tmp_path / "st.npy").astype(np.int64)          # [warp, tile, chunk, phase]
    for e in range(4):
        for t in range(6):
            s = st[e, t]
            assert np.all(s[:, :7] > 0), (e, t)
            assert np.all(np.diff(s[:, :7], axis=1) >= 0), (e, t)              # phases in order
            assert np.all(s[1:, 0] >= s[:-1, 6]), (e, t)                       # chunks in order
            assert s[0, 7] <= s[1, 7] <= s[0, 0], (e, t)                       # full-wait, then chunk 0
            if t:
                assert st[e, t, 0, 7] >= st[e, t - 1, -1, 6], (e, t)           # tiles in order
