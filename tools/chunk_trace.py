#!/usr/bin/env python
"""Where the dense epilogue's time goes, per 32-column chunk (debug library chunk-phase stamps,
gemm_dense.cu TCX_STAMP: cluster 0, CTA 0, lane 0 of each epilogue warp, first 6 tiles; SM clock64):
TCX_LIB_PATH=.../libtcx_debug.so python tools/chunk_trace.py c3|c4|c3tf32 [wide] [noc]
Phases: tmem_ld_wait (k0->k1), C wait or store-buffer wait (k1->k2), C smem loads + adds + smem
writes (k2->k3), fence.proxy.async + syncwarp (k3->k4), TMA store issue + commit (k4->k5),
wait for the store to read the buffer (k5->k6), next C load issue (k6 -> next k0).
Tile level: the tmem_full wait (slot 7 of chunks 0 / 1)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402

NT = 6


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
    wide = "wide" in sys.argv[2:]
    noc = "noc" in sys.argv[2:]
    torch.cuda.set_device(0)
    w = bench.Work(cfg, 0, 1, torch.device("cuda", 0))
    tcx = w.tcx
    M, N, K = w.shape
    tn = 512 if wide else 256
    T = ((M + 255) // 256) * ((N + tn - 1) // tn)
    CH = tn // 32
    step = lambda: tcx.gemm(w.A, w.B, None if noc else w.C, w.D, tf32=getattr(w, "tf32", False), tile_n=tn)
    buf = torch.zeros(4 * (T + 8 * NT * CH), dtype=torch.int64, device="cuda")
    for _ in range(3):
        step()
    tcx.debug_trace(buf)
    step()
    torch.cuda.synchronize()
    tcx.debug_trace(None)
    names = ["tmem_ld_wait", "c_or_buffer_wait", "smem_math", "fence_syncwarp", "store_issue", "store_read_wait"]
    for e in range(4):                               # epilogue warp e = warp 4 + e, on SM sub-partition e
        o = 4 * T + e * NT * CH * 8
        st = buf[o:o + NT * CH * 8].view(NT, CH, 8).cpu().numpy().astype(np.int64)
        ph = {n: np.diff(st[1:, :, :7], axis=2)[..., i] for i, n in enumerate(names)}   # tiles 1..NT-1
        nxt = st[1:, 1:, 0] - st[1:, :-1, 6]
        rep = {"cfg": cfg, "wide": wide, "no_c": noc, "warp": 4 + e, "chunks_per_tile": CH,
               "cycles_median": {n: float(np.median(v)) for n, v in ph.items()},
               "cycles_p90": {n: float(np.percentile(v, 90)) for n, v in ph.items()}}
        rep["cycles_median"]["c_load_issue"] = float(np.median(nxt))
        chunk = st[1:, 1:, 0] - st[1:, :-1, 0]
        rep["chunk_period_cycles"] = {"median": float(np.median(chunk)), "p90": float(np.percentile(chunk, 90))}
        rep["tile_drain_cycles"] = [int(st[t, CH - 1, 6] - st[t, 1, 7]) for t in range(1, NT)]
        rep["tmem_full_wait_cycles"] = [int(st[t, 1, 7] - st[t, 0, 7]) for t in range(1, NT)]
        rep["per_chunk_tile1"] = [[int(x) for x in np.diff(st[1, c, :7])] for c in range(CH)]
        print(json.dumps(rep), flush=True)


if __name__ == "__main__":
    main()
