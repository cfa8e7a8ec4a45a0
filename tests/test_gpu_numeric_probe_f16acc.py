"""FP16-accumulate numeric probe: the mma f16.f16.f16.f16 variant (C and D
FP16), probed the way Table FP16-FP16-numeric-profiling does.

Seven classes x 8192 tiles (tcxgen.probe_classes_f16acc): the configs[1] crafted classes rescaled to
FP16's range, plus the paper's three probes (mul / inner / accum) with FP16 and FP32 init.  d00 of
every tile is classified bit-exactly against
  * exact_RNE16 (the oracle: one rounding of the exact value into FP16) and exact_RZ16;
  * the model family M(g, p, R, t, o, e) with an FP16 accumulator (oracle/models.c, acc_fmt = F16:
    truncation window and every block rounding at FP16's 11-bit significand);
  * two-stage models: an FP32-accumulator model (incl. the one observed for FP16 -> FP32,
    DESIGN.md §7) followed by one conversion FP32 -> FP16 (RNE or RZ);
  * single-rounding models M16w32: the FP32 datapath's truncation window, one rounding into FP16;
so "computation in high precision, converted only at the end" is tested, not assumed.
Gate: every output of every tile within the FP16 bar of the oracle (tests/parity.py).
Report: numeric_probe_f16acc_report.json in $TCX_REPORT_DIR (default gpurun_out/)."""
import json
import os

import numpy as np
import pytest
import torch

import oracle as O
import tcxgen
import paper_2206_02874_b200 as tcx
from parity import host_bits, fp16_bound_check

pytestmark = pytest.mark.gpu
DEV = "cuda"


def _f16(bits):
    return np.asarray(bits).astype(np.uint16).view(np.float16).astype(np.float64)


def _f32_to_f16_bits(bits32, rz):
    return np.array([O.quantize(float(v), O.F16, rz) for v in np.asarray(bits32, np.uint32).view(np.float32)],
                    dtype=np.uint32)


def models():
    ms = [("exact_RNE16", dict(g=16, p=-1, rz=False)), ("exact_RZ16", dict(g=16, p=-1, rz=True))]
    for em in (0, 2):
        for g in (16, 8, 1):
            for p in range(0, 14):
                for rz in (True, False):
                    for fl in (False, True):
                        for ca in (False, True):
                            nm = (f"M16(g={g},p={p},{'RZ' if rz else 'RNE'},{'floor' if fl else 'tz'},"
                                  f"{'c_after' if ca else 'c_in'},{('lead', 'esum', 'esum2')[em]})")
                            ms.append((nm, dict(g=g, p=p, rz=rz, floor_mode=fl, c_after=ca, emode=em)))
    return ms


# aligned like the FP32 datapath (window p bits below FP32's significand), rounded ONCE into FP16:
# the single-rounding alternative to the two-stage models (oracle.model_batch win_fmt = FP32)
FP32_WINDOW = [(f"M16w32(g=16,p={p},{'RZ' if rz else 'RNE'},tz,{'c_after' if ca else 'c_in'},{('lead', 'esum', 'esum2')[em]})",
                dict(g=16, p=p, rz=rz, c_after=ca, emode=em))
               for em in (0, 2) for p in range(0, 9) for rz in (True, False) for ca in (False, True)]

TWO_STAGE = [("exact32_RNE", dict(g=16, p=-1, rz=False, emode=0))] + [
    (f"M32(g=16,p={p},{'RZ' if rz else 'RNE'},tz,{'c_after' if ca else 'c_in'},esum2)",
     dict(g=16, p=p, rz=rz, c_after=ca, emode=2))
    for p in (3, 4, 5, 6, 8, 10, 13) for rz in (True, False) for ca in (False, True)]


def test_numeric_probe_fp16_accumulate():
    n_per = 8192
    d = tcxgen.probe_classes_f16acc(n_per, seed=0)
    A, B, C = d["A"].to(DEV), d["B"].to(DEV), d["C"].to(DEV)
    D = tcx.mma_tiles(A, B, C, f16_acc=True)
    torch.cuda.synchronize()
    K = d["K"]
    ref, absv = O.tiles(O.F16, 16, 8, K, host_bits(A), host_bits(B), host_bits(C), cd=O.F16)
    got_all = host_bits(D).reshape(ref.shape).astype(np.uint32)
    max_ulp = fp16_bound_check(got_all, ref, absv, K, "f16acc probe")       # the gate

    a_rows, b_rows = host_bits(A[:, 0, :]), host_bits(B[:, 0, :])
    c16 = host_bits(C[:, 0, 0]).astype(np.uint32)
    c32 = np.array([O.quantize(float(v), O.F32) for v in _f16(c16)], dtype=np.uint32)   # exact widening
    cls = d["cls"].numpy()
    gv = got_all[:, 0, 0]
    outs = {nm: O.model_batch(O.F16, a_rows, b_rows, c16, Ki=16, acc_fmt=O.F16, **kw) for nm, kw in models()}
    assert np.array_equal(outs["exact_RNE16"], ref[:, 0, 0])       # the model family's special case
    for nm, kw in FP32_WINDOW:
        outs[nm] = O.model_batch(O.F16, a_rows, b_rows, c16, Ki=16, acc_fmt=O.F16, win_fmt=O.F32, **kw)
    for nm, kw in TWO_STAGE:
        m32 = O.model_batch(O.F16, a_rows, b_rows, c32, Ki=16, **kw)
        outs[nm + "->RNE16"] = _f32_to_f16_bits(m32, False)
        outs[nm + "->RZ16"] = _f32_to_f16_bits(m32, True)
    crafted = cls < 5
    rep = {"tiles": int(A.shape[0]), "classes": list(tcxgen.CLASSES_F16ACC), "max_err_fp16_ulps": max_ulp,
           "all_100pct_models": [nm for nm, o in outs.items() if np.array_equal(o, gv)],
           "crafted_100pct_models": [nm for nm, o in outs.items() if np.array_equal(o[crafted], gv[crafted])]}
    rep["observed"] = rep["all_100pct_models"][0] if rep["all_100pct_models"] else None
    per = {}
    for ci, cname in enumerate(tcxgen.CLASSES_F16ACC):
        sel = cls == ci
        full = [nm for nm, o in outs.items() if np.array_equal(o[sel], gv[sel])]
        per[cname] = {"n_models_100pct": len(full), "first": full[:8],
                      "exact_RNE16": float((outs["exact_RNE16"][sel] == gv[sel]).mean()),
                      "exact_RZ16": float((outs["exact_RZ16"][sel] == gv[sel]).mean())}
    rep["per_class"] = per
    allm = {nm: {cn: float((o[cls == ci] == gv[cls == ci]).mean()) for ci, cn in enumerate(tcxgen.CLASSES_F16ACC)}
            for nm, o in outs.items()}
    best = sorted(allm, key=lambda nm: -float((outs[nm] == gv).mean()))[:6]
    rep["best_models"] = {nm: {"overall": float((outs[nm] == gv).mean()), "per_class": allm[nm]} for nm in best}
    # the paper's table: mean |err| vs CPU FP32 and vs CPU FP32 converted to FP16
    pt = d["ptype"].numpy()
    a32, b32, cc32 = d["a32"].numpy(), d["b32"].numpy(), d["c32"].numpy()
    tables = {}
    gvals = _f16(gv)
    for ci in (5, 6):
        for ptn, pname in enumerate(("mul", "inner", "accum")):
            idx = np.nonzero((cls == ci) & (pt == ptn))[0]
            cpu32 = np.array([O.seq32(a32[i], b32[i], float(cc32[i]), c_last=True) for i in idx])
            cpu16 = cpu32.astype(np.float32).astype(np.float16).astype(np.float64)
            tables[f"{tcxgen.CLASSES_F16ACC[ci]}/{pname}"] = {
                "CPU_FP32": float(np.mean(np.abs(gvals[idx] - cpu32))),
                "CPU_FP32cvtFP16": float(np.mean(np.abs(gvals[idx] - cpu16))), "n": int(idx.size)}
    rep["paper_table"] = tables
    out_dir = os.environ.get("TCX_REPORT_DIR", "gpurun_out")
    os.makedirs(out_dir, exist_ok=True)
    with open(os.path.join(out_dir, "numeric_probe_f16acc_report.json"), "w") as f:
        json.dump(rep, f, indent=1)
    # PAPER.md:975-977 (init_FP16 vs CPU_FP32cvtFP16 = 0.00) is a claim about A100: on B200 it is
    # reported (paper_table), not asserted; the gate above is the FP16 bar.
    assert all(v["n"] > 0 for v in tables.values())
