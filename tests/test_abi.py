"""The C-ABI library builds, loads and exports every symbol include/tcx.h declares (no GPU calls)."""
import ctypes
import os
import re
import subprocess

import paper_2206_02874_b200 as tcx

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "tcx.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(tcx_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = _declared()
    for n in ["tcx_mma_tiles", "tcx_gemm", "tcx_gemm_sp24", "tcx_probe", "tcx_sp24_compress",
              "tcx_sp24_pack_meta", "tcx_round_tf32", "tcx_status_string", "tcx_last_error"]:
        assert n in names


def test_library_exports_every_declared_symbol():
    from paper_2206_02874_b200 import build
    build.build()
    L = ctypes.CDLL(tcx.LIB_PATH)
    for n in _declared():
        assert hasattr(L, n), n
    out = subprocess.run(["nm", "-D", "--defined-only", tcx.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (tcx_\w+)", out))
    assert set(_declared()) <= exported
    assert set(tcx.EXPORTS) <= exported


def test_debug_library_exports_the_same_boundary():
    """libtcx_debug.so (watchdog-bounded waits) is the same ABI; built here like the product."""
    from paper_2206_02874_b200 import build
    path = build.build(debug=True)
    out = subprocess.run(["nm", "-D", "--defined-only", path], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (tcx_\w+)", out))
    assert set(_declared()) <= exported
    assert path != tcx.LIB_PATH


def test_host_only_calls_without_gpu():
    L = tcx.lib()
    assert L.tcx_status_string(2) == b"TCX_ERR_UNSUPPORTED"
    assert L.tcx_version().startswith(b"tcx")
    # pure-host size query and argument validation return before any device work
    assert tcx.sp24_meta_hw_bytes(256, 1024) == 256 * 1024 // 8
    st = L.tcx_mma_tiles(0, 3, 16, 8, 4, 1, None, None, None, None, None)    # bad shape
    assert st == 2
    assert L.tcx_mma_chain(4, 3, 1, None, None, None, None) == 2              # S8 chain: unsupported
    assert L.tcx_mma_chain(0, 3, 0, None, None, None, None) == 0              # count 0: no-op
    st = L.tcx_gemm(4, 3, 16, 16, 16, None, 16, None, 16, None, 16, None, 16, None)   # s8 -> f32 unsupported
    assert st == 2


def test_product_does_not_reference_oracle():
    """the product package never imports or links the oracle"""
    pkg = os.path.join(ROOT, "paper_2206_02874_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dp, f)).read()
                assert "import oracle" not in txt and "tcxref" not in txt and "from oracle" not in txt, f
