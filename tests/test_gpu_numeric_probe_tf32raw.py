"""TF32 raw-input sub-class of configs[1] (SURVEY §8(c) reading C1): what does B200 do with FP32
storage whose low 13 significand bits are NOT zero when it is fed to a TF32 MMA?  The paper keeps
TF32 in a 32-bit register and never says.  The API requires TF32-representable
inputs; this probe deliberately violates that to OBSERVE the hardware.

Each tile is the paper's multiplication probe: a0 in row 0 of A, b0 in column 0
of B, everything else 0, so d00 = conv(a0) * conv(b0) exactly (a TF32 x TF32 product fits FP32;
a full-FP32 product is then rounded by the accumulator).  The inputs are random FP32 values with
random low bits, including exact TF32 ties; d00 is classified against the conversions
oracle.tf32_convert names: RZ (truncate), RNE, RNA (cvt.rna) and full FP32.
Report: tf32_raw_input_report.json in $TCX_REPORT_DIR."""
import json
import os

import numpy as np
import pytest
import torch

import oracle as O
import paper_2206_02874_b200 as tcx
from parity import host_bits

pytestmark = pytest.mark.gpu
DEV = "cuda"


def _inputs(n, seed=0):
    rng = np.random.default_rng(seed)
    a = (rng.standard_normal(n) * 2.0 ** rng.integers(-8, 8, n)).astype(np.float32).view(np.uint32)
    b = (rng.standard_normal(n) * 2.0 ** rng.integers(-8, 8, n)).astype(np.float32).view(np.uint32)
    # a quarter of the a's sit exactly on a TF32 tie (low 13 bits = 0x1000), so RNE and RNA differ
    tie = rng.random(n) < 0.25
    a[tie] = (a[tie] & np.uint32(0xFFFFE000)) | np.uint32(0x1000)
    return a, b


def _oracle_d00(a_bits, b_bits, mode):
    ca = O.tf32_convert(a_bits, mode).view(np.float32).astype(np.float64)
    cb = O.tf32_convert(b_bits, mode).view(np.float32).astype(np.float64)
    return (ca * cb).astype(np.float32)        # one product: exact in float64, one RNE to FP32


@pytest.mark.parametrize("path", ["mma.sync", "tcgen05"])
def test_tf32_raw_fp32_inputs(path):
    n = 8192
    a, b = _inputs(n)
    A = np.zeros((n, 16, 8), np.uint32)
    B = np.zeros((n, 8, 8), np.uint32)
    A[:, 0, 0] = a
    B[:, 0, 0] = b
    At = torch.from_numpy(A.view(np.float32)).to(DEV)
    Bt = torch.from_numpy(B.view(np.float32)).to(DEV)
    D = (tcx.mma_tiles if path == "mma.sync" else tcx.mma_tiles_tc05)(At, Bt, None, tf32=True)
    torch.cuda.synchronize()
    got = host_bits(D)[:, 0, 0].view(np.float32)
    rep = {"path": path, "n": n, "match": {}}
    for mode in ("rz", "rne", "rna", "fp32"):
        rep["match"][mode] = float(np.mean(_oracle_d00(a, b, mode) == got))
    full = [m for m, v in rep["match"].items() if v == 1.0]
    rep["observed"] = full
    out = os.environ.get("TCX_REPORT_DIR", "gpurun_out")
    os.makedirs(out, exist_ok=True)
    fn = os.path.join(out, "tf32_raw_input_report.json")
    prev = json.load(open(fn)) if os.path.exists(fn) else {}
    prev[path] = rep
    with open(fn, "w") as f:
        json.dump(prev, f, indent=1)
    # whatever the hardware does, it must be one of the named conversions on every element
    assert full, f"no conversion model matches all elements: {rep['match']}"
