"""SASS evidence: the built libtcx.so contains the instructions each kernel claims.

`cuobjdump -sass` of the product library, split per kernel instance (no GPU needed):
  * every GEMM instance (dense and 2:4) issues tcgen05 MMAs (UTCHMMA / UTCIMMA), loads operands
    with TMA (UTMALDG), drains TMEM with tcgen05.ld (LDTM) and stores D with TMA (UTMASTG); the
    cta_group::2 instances (first template argument 2) issue the .2CTA forms, the cta_group::1 ones
    do not; multicast instances (PM or PN > 1) issue UTMALDG.*.MULTICAST; no GEMM instance falls
    back to warp-level mma.sync (HMMA.* / IMMA.*);
  * the 2:4 GEMM moves its metadata into TMEM with tcgen05.cp (UTCCP);
  * the mma.sync paths the paper measures (tile batch, chain) are HMMA.16816 / HMMA.1688 /
    IMMA.16832, the tcgen05 tile batch is UTCHMMA/UTCIMMA + LDTM/STTM.
"""
import collections
import os
import re
import shutil
import subprocess

import pytest

import paper_2206_02874_b200 as tcx

CUOBJDUMP = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
OPS = re.compile(r"\b((?:UTC|UTMA)\w+(?:\.\w+)*|LDTM\S*|STTM\S*|[HI]MMA\.\S*)")


@pytest.fixture(scope="module")
def kernels():
    if not os.path.exists(CUOBJDUMP):
        pytest.skip("cuobjdump not available")
    from paper_2206_02874_b200 import build
    build.build()
    sass = subprocess.run([CUOBJDUMP, "-sass", tcx.LIB_PATH], capture_output=True, text=True,
                          check=True).stdout
    parts = re.split(r"\n\s*Function : (\S+)\n", sass)
    mangled = parts[1::2]
    names = subprocess.run(["c++filt"], input="\n".join(mangled), capture_output=True, text=True,
                           check=True).stdout.splitlines()
    fam = collections.defaultdict(list)
    for name, body in zip(names, parts[2::2]):
        m = re.search(r"(\w+_kernel)(?:<([^>]*)>)?\(", name)
        assert m, name
        targs = [x.strip() for x in m.group(2).split(",")] if m.group(2) else []
        fam[m.group(1)].append((name, targs, set(OPS.findall(body))))
    return fam


def _has(ops, prefix):
    return any(o == prefix or o.startswith(prefix + ".") for o in ops)


@pytest.mark.parametrize("kernel", ["gemm_dense_kernel", "gemm_sp24_kernel"])
def test_gemm_kernels_are_tcgen05_tma(kernels, kernel):
    insts = kernels[kernel]
    assert len(insts) >= 8, f"{kernel}: only {len(insts)} instances"
    seen_cg = set()
    for name, targs, ops in insts:
        cg, pm, pn = int(targs[0]), int(targs[3]), int(targs[4])
        seen_cg.add(cg)
        mma = [o for o in ops if o.startswith(("UTCHMMA", "UTCIMMA"))]
        assert mma, f"no tcgen05.mma in {name}"
        assert not any(o.startswith(("HMMA.", "IMMA.")) for o in ops), f"mma.sync in {name}"
        for need in ("UTMALDG", "UTMASTG"):
            assert any(o.startswith(need) for o in ops), f"no {need} in {name}"
        assert any(o.startswith("LDTM") for o in ops), f"no tcgen05.ld in {name}"
        if cg == 2:
            assert all(".2CTA" in o for o in mma), f"cta_group::1 MMA in 2-CTA {name}: {mma}"
            assert "UTMALDG.2D.2CTA" in ops, name
        else:
            assert not any(".2CTA" in o for o in mma), f"2CTA MMA in 1-CTA {name}"
        if pm * pn > 1:
            assert any("MULTICAST" in o and o.startswith("UTMALDG") for o in ops), \
                f"no multicast TMA load in {name}"
        if kernel == "gemm_sp24_kernel":
            assert any(o.startswith("UTCCP") for o in ops), f"no tcgen05.cp (metadata) in {name}"
    assert seen_cg == {1, 2}, seen_cg


def test_gemm_dense_covers_every_kind(kernels):
    mma = set()
    for _, _, ops in kernels["gemm_dense_kernel"]:
        mma |= {o for o in ops if o.startswith(("UTCHMMA", "UTCIMMA"))}
    assert _has(mma, "UTCHMMA") and _has(mma, "UTCIMMA"), mma     # f16/bf16/tf32 and i8 kinds


def test_mma_sync_paths_use_the_papers_shapes(kernels):
    """The paper's measured instructions (PAPER.md Tables: m16n8k16 f16/bf16, m16n8k8 tf32,
    m16n8k32 s8) are what the mma.sync tile batch and the chain matmul compile to."""
    t16 = set().union(*(ops for _, _, ops in kernels["tiles16_kernel"]))
    assert {"HMMA.16816.F32", "HMMA.16816.F32.BF16"} <= t16, t16
    tf = set().union(*(ops for _, _, ops in kernels["tiles_tf32_kernel"]))
    assert any(o.startswith("HMMA.1688.F32.TF32") for o in tf), tf
    s8 = set().union(*(ops for _, _, ops in kernels["tiles_s8_kernel"]))
    assert any(o.startswith("IMMA.16832.S8.S8") for o in s8), s8
    ch = set().union(*(ops for _, _, ops in kernels["chain_kernel"]))
    assert {"HMMA.1688.F32", "HMMA.1688.F32.BF16", "HMMA.1688.F32.TF32"} <= ch, ch


def test_tcgen05_tile_batch_and_probes(kernels):
    for name, _, ops in kernels["tiles_tc05_kernel"]:
        assert any(o.startswith(("UTCHMMA", "UTCIMMA")) for o in ops), name
        assert any(o.startswith("LDTM") for o in ops) and any(o.startswith("STTM") for o in ops), name
    mc = set().union(*(ops for _, _, ops in kernels["probe_tma_mc_kernel"]))
    assert any("MULTICAST" in o for o in mc), mc
    cp = set().union(*(ops for _, _, ops in kernels["probe_tc05_cp_kernel"]))
    assert any(o.startswith("UTCCP") for o in cp), cp
