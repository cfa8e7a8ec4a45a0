"""Data-movement probes (the paper's §VII) on B200.

Parity: ldmatrix.x{1,2,4}[.trans] fragments bit-exact against the instruction's definition
(oracle.ldmatrix) for random data and random (permuted, conflict-bearing) row addresses.
Probes (clock-counter method): properties that hold whatever the numbers —
more bytes per instruction never lowers latency, conflicts never speed ld.shared up, throughput
rises with warps x ILP — and the sweep is written to $TCX_REPORT_DIR/data_movement_report.json
with the paper's A100 table values beside it as context."""
import json
import os

import numpy as np
import pytest
import torch

import oracle as O
import paper_2206_02874_b200 as tcx

pytestmark = pytest.mark.gpu
DEV = "cuda"


@pytest.mark.parametrize("num", [1, 2, 4])
@pytest.mark.parametrize("trans", [False, True])
def test_ldmatrix_fragments_vs_definition(num, trans):
    rng = np.random.default_rng(10 * num + trans)
    for trial in range(8):
        smem = rng.integers(0, 1 << 16, 512, dtype=np.uint32).astype(np.uint16)
        rows = rng.permutation(64)[:32]                       # any 16-byte-aligned rows of the 1 KiB image
        row_elem = (rows * 8).astype(np.int32)
        got = tcx.ldmatrix_dump(num, trans, torch.from_numpy(smem.view(np.int16)).to(DEV),
                                torch.from_numpy(row_elem).to(DEV))
        torch.cuda.synchronize()
        want = O.ldmatrix(num, trans, np.concatenate([smem, np.zeros(512, np.uint16)]), row_elem)
        assert np.array_equal(got.cpu().numpy().view(np.uint32), want), (num, trans, trial)


def _p(kind, **kw):
    kw.setdefault("iters", 512)
    kw.setdefault("repeats", 3)
    return tcx.probe(kind, **kw)


def test_ldmatrix_latency_and_throughput_properties():
    lat = {n: _p("ldmatrix", m=n)["latency_cycles"] for n in (1, 2, 4)}
    assert lat[1] <= lat[2] + 1 and lat[2] <= lat[4] + 1
    one = _p("ldmatrix", m=4, warps=1, ilp=1)["fma_per_clk_per_sm"]
    many = _p("ldmatrix", m=4, warps=8, ilp=4)["fma_per_clk_per_sm"]
    assert many > 1.5 * one


def test_ld_shared_conflict_latency_grows():
    lat = [_p("ld_shared", m=4, n=w)["latency_cycles"] for w in (1, 2, 4, 8, 16, 32)]
    assert all(b >= a - 0.5 for a, b in zip(lat, lat[1:]))
    assert lat[-1] > lat[0] + 8


def test_tmem_ld_runs_and_scales():
    a = _p("tmem_ld", m=32, warps=4, ilp=1)
    b = _p("tmem_ld", m=32, warps=16, ilp=2)
    assert a["latency_cycles"] > 0 and b["fma_per_clk_per_sm"] >= a["fma_per_clk_per_sm"]


def test_tma_and_tc05_cp_probes():
    """B200's staging path: TMA 2D box loads from L2 and tcgen05.cp smem->TMEM;
    more boxes in flight per wait raise bytes/clk/SM (latency is amortised)."""
    t1 = _p("tma_load", m=128, n=128, ilp=1, num_sms=148)
    t8 = _p("tma_load", m=128, n=128, ilp=8, num_sms=148)
    assert t1["latency_cycles"] > 100 and t8["fma_per_clk_per_sm"] > 2 * t1["fma_per_clk_per_sm"]
    c1 = _p("tc05_cp", ilp=1)
    c8 = _p("tc05_cp", ilp=8)
    assert c1["latency_cycles"] > 0 and c8["fma_per_clk_per_sm"] > c1["fma_per_clk_per_sm"]


def test_tma_multicast_probe():
    """clusters whose CTAs all need the same boxes: multicast (each box fetched once, delivered to
    every CTA) and unicast (every CTA fetches every box) deliver the same bytes per CTA.  Both must
    complete every wait (a lost multicast signal would hang) and deliver at a sane rate; which one
    is faster is a measurement (DESIGN.md §7 data movement), not asserted."""
    for cs in (2, 4, 8):
        uc = _p("tma_multicast", m=128, n=128, ilp=8, cta_group=cs, k=0, num_sms=148)
        mc = _p("tma_multicast", m=128, n=128, ilp=8, cta_group=cs, k=1, num_sms=148)
        assert uc["latency_cycles"] > 0 and mc["latency_cycles"] > 0
        assert uc["fma_per_clk_per_sm"] > 10 and mc["fma_per_clk_per_sm"] > 10, (cs, uc, mc)
    with pytest.raises(tcx.TcxError):
        _p("tma_multicast", m=128, n=128, ilp=6, cta_group=4, k=1)      # ilp must split over the cluster


def test_dsmem_forwarding_probe():
    """SM-to-SM bulk copies inside clusters of 2 and 4 CTAs complete every wait (a lost complete_tx
    would hang) at a positive rate; how it compares with TMA from L2 is a measurement"""
    for cs in (2, 4):
        r = _p("dsmem", n=16384, ilp=4, cta_group=cs, num_sms=148, iters=256)
        assert r["latency_cycles"] > 0 and r["fma_per_clk_per_sm"] > 1, (cs, r)
    with pytest.raises(tcx.TcxError):
        _p("dsmem", n=16384 + 8, ilp=2, cta_group=2)                  # box must be a multiple of 16 B


def test_data_movement_sweep_report():
    rep = {"units": {"latency": "cycles per iteration (clock64)", "throughput": "bytes/clk/SM"},
           "paper_A100_context": {
               "ldmatrix.x1": {"completion": 23.1, "(4,5)": [26.8, 95.4], "(8,4)": [32.1, 127.7]},
               "ldmatrix.x2": {"completion": 25.1, "(4,4)": [32.1, 127.8], "(8,2)": [32.1, 127.7]},
               "ldmatrix.x4": {"completion": 29.3, "(4,2)": [32.2, 127.3], "(8,1)": [32.6, 125.9]},
               "ld.shared.u32": {"1-way": 23.0, "2-way": 25.0, "4-way": 29.0, "8-way": 37.0},
               "ld.shared.u64": {"2-way": 25.1, "4-way": 29.1, "8-way": 37.0},
               "source": "PAPER.md:766-777, 783-793 (A100, context only)"},
           "ldmatrix": {}, "ld_shared": {}, "tmem_ld": {}}
    for n in (1, 2, 4):
        for tr in (0, 1):
            key = f"x{n}{'.trans' if tr else ''}"
            rows = {"completion": _p("ldmatrix", m=n, n=tr)["latency_cycles"]}
            for w in (1, 2, 4, 8, 16):
                for ilp in (1, 2, 4, 8):
                    r = _p("ldmatrix", m=n, n=tr, warps=w, ilp=ilp, repeats=2)
                    rows[f"({w},{ilp})"] = [round(r["latency_cycles"], 2), round(r["fma_per_clk_per_sm"], 2)]
            rep["ldmatrix"][key] = rows
    for b, ways in ((4, (1, 2, 4, 8, 16, 32)), (8, (2, 4, 8, 16, 32))):
        rep["ld_shared"][f"u{8 * b}"] = {f"{w}-way": round(_p("ld_shared", m=b, n=w)["latency_cycles"], 2) for w in ways}
    for n in (1, 2, 4, 8, 16, 32):
        rows = {"completion": round(_p("tmem_ld", m=n)["latency_cycles"], 2)}
        for w in (4, 8, 16):
            for ilp in (1, 2, 4):
                r = _p("tmem_ld", m=n, warps=w, ilp=ilp, repeats=2)
                rows[f"({w},{ilp})"] = [round(r["latency_cycles"], 2), round(r["fma_per_clk_per_sm"], 2)]
        rep["tmem_ld"][f"32x32b.x{n}"] = rows
    rep["tma_load"] = {}
    for rows, inner in ((128, 128), (256, 128), (64, 128), (128, 256)):
        row = {}
        for ilp in (1, 2, 4, 8):
            if rows * inner * ilp > 200 * 1024:
                continue
            for nsm in (1, 148):
                r = _p("tma_load", m=rows, n=inner, ilp=ilp, num_sms=nsm, repeats=2)
                row[f"ilp{ilp}_sms{nsm}"] = [round(r["latency_cycles"], 1), round(r["fma_per_clk_per_sm"], 2)]
        rep["tma_load"][f"box{rows}x{inner}B"] = row
    rep["tc05_cp_128x128b"] = {f"ilp{ilp}": [round(r["latency_cycles"], 1), round(r["fma_per_clk_per_sm"], 2)]
                                for ilp in (1, 2, 4, 8) for r in [_p("tc05_cp", ilp=ilp, repeats=2)]}
    rep["tma_multicast"] = {}
    for cs in (1, 2, 4, 8):
        for mcast in ((0, 1) if cs > 1 else (0,)):
            for nsm in (cs, 148):
                r = _p("tma_multicast", m=128, n=128, ilp=8, cta_group=cs, k=mcast, num_sms=nsm, repeats=2)
                rep["tma_multicast"][f"cluster{cs}_{'mc' if mcast else 'uc'}_sms{nsm}"] = [
                    round(r["latency_cycles"], 1), round(r["fma_per_clk_per_sm"], 2)]
    out = os.environ.get("TCX_REPORT_DIR", "gpurun_out")
    os.makedirs(out, exist_ok=True)
    with open(os.path.join(out, "data_movement_report.json"), "w") as f:
        json.dump(rep, f, indent=1)
    # the smem read port: ldmatrix throughput saturates near a fixed bytes/clk/SM figure
    best = max(v[1] for k, v in rep["ldmatrix"]["x4"].items() if k.startswith("("))
    assert best > 60
