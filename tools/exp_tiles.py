#!/usr/bin/env python
"""Tile-batch (tcx_mma_tiles) launch sweep: µs per launch and GB/s vs batch size, one CUDA graph of
`copies` launches over distinct batch copies (total > L2, so reads are cold).
usage: TCX_TILES_IMPL=<n> python tools/exp_tiles.py [fmt]"""
import hashlib
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2206_02874_b200 as tcx  # noqa: E402
import tcxgen as g  # noqa: E402


def main():
    fmt = sys.argv[1] if len(sys.argv) > 1 else "f16"
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(0)
    out = {"impl": os.environ.get("TCX_TILES_IMPL", "0"), "fmt": fmt}
    for count, copies in ((1, 64), (4096, 64), (65536, 8), (524288, 2)):
        As = [g.uniform_matrix((count, 16, 16), fmt, i, g.STREAM_A, device=dev) for i in range(copies)]
        Bs = [g.uniform_matrix((count, 8, 16), fmt, i, g.STREAM_B, device=dev) for i in range(copies)]
        Cs = [g.uniform_matrix((count, 16, 8), "f32", i, g.STREAM_C, device=dev) for i in range(copies)]
        Ds = [torch.empty(count, 16, 8, device=dev) for _ in range(copies)]
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            for j in range(copies):
                tcx.mma_tiles(As[j], Bs[j], Cs[j], Ds[j])
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        if count == 4096:
            out["d_sha"] = hashlib.sha1(Ds[0].cpu().numpy().tobytes()).hexdigest()[:16]
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            for j in range(copies):
                tcx.mma_tiles(As[j], Bs[j], Cs[j], Ds[j])
        for _ in range(3):
            graph.replay()
        torch.cuda.synchronize()
        reps = 20
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            graph.replay()
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / (reps * copies)
        out[f"n{count}"] = {"us_per_launch": round(us, 3), "GBps": round(1792 * count / us / 1e3, 1)}
        del As, Bs, Cs, Ds, graph
        torch.cuda.empty_cache()
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
