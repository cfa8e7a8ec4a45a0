#!/usr/bin/env python
"""Tile timeline of one dense GEMM launch through the debug library (tcx_debug_trace):
TCX_LIB_PATH=.../libtcx_debug.so python tools/trace_gemm.py c3|c3tf32|c4 [group_m]
Prints per-launch statistics: tile MMA durations, epilogue lag, and — for the L2 reuse question —
the spread of K-progress start times among the tiles that read the same B tile (same n) or the
same A tile (same m) while they run concurrently."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402


def tile_coords(t, m_tiles, n_tiles, g):
    by_m = g > 0
    gt = g if by_m else -g
    major, minor = (m_tiles, n_tiles) if by_m else (n_tiles, m_tiles)
    per = gt * minor
    grp = t // per
    first = grp * gt
    gm = np.minimum(major - first, gt)
    r = t - grp * per
    a = first + r % gm
    b = np.where(grp & 1, minor - 1 - r // gm, r // gm)          # serpentine (gemm_dense.cu)
    return (a, b) if by_m else (b, a)


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
    g = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    wide = "wide" in sys.argv[3:]                            # c5: the 512 x 240 M-wide tile
    noc = "noc" in sys.argv[3:]                              # D = A B (no C): the epilogue's C path off
    torch.cuda.set_device(0)
    w = bench.Work(cfg, 0, 1, torch.device("cuda", 0))
    tcx = w.tcx
    M, N, K = w.shape
    if cfg.startswith("c5"):
        m_tiles, n_tiles = M // (512 if wide else 256), (N + 239) // 240
        step = lambda: tcx.gemm_sp24(w.vals, w.meta_hw, w.B, None if noc else w.C, w.D, group_m=g, tile_m=512 if wide else 256)
    else:
        tn = 512 if wide else 256                            # dense: the 256 x 512 pair tile
        m_tiles, n_tiles = (M + 255) // 256, (N + tn - 1) // tn
        step = lambda: tcx.gemm(w.A, w.B, None if noc else w.C, w.D, tf32=getattr(w, "tf32", False), group_m=g, tile_n=tn)
    T = m_tiles * n_tiles
    buf = torch.zeros(4 * T, dtype=torch.int64, device="cuda")
    for _ in range(3):
        step()
    tcx.debug_trace(buf)
    step()
    torch.cuda.synchronize()
    tcx.debug_trace(None)
    r = buf.view(T, 4).cpu().numpy().astype(np.int64)
    t0 = r[:, 1].min()
    start, mend, eend = (r[:, 1] - t0) / 1e3, (r[:, 2] - t0) / 1e3, (r[:, 3] - t0) / 1e3   # us
    pair = r[:, 0] >> 32
    tiles = np.arange(T)
    mt, nt = tile_coords(tiles, m_tiles, n_tiles, g)
    dur = mend - start
    # concurrent sharers: tiles with the same n (B tile) whose MMA intervals overlap
    def spread(key):
        out = []
        for v in np.unique(key):
            idx = np.where(key == v)[0]
            s = np.sort(start[idx])
            # split into concurrency clusters: consecutive starts closer than one tile duration
            cl = [[s[0]]]
            for x in s[1:]:
                (cl[-1].append(x) if x - cl[-1][0] < 0.5 * np.median(dur) else cl.append([x]))
            out += [c[-1] - c[0] for c in cl if len(c) > 1]
        return np.array(out)
    sb, sa = spread(nt), spread(mt)
    rep = {"cfg": cfg, "group_m": g, "tiles": int(T), "pairs": int(len(np.unique(pair))), "kernel_us": float(eend.max()),
           "tile_mma_us": {"median": float(np.median(dur)), "p10": float(np.percentile(dur, 10)),
                           "p90": float(np.percentile(dur, 90))},
           "epilogue_lag_us_median": float(np.median(eend - mend)),
           "B_sharers_start_spread_us": {"median": float(np.median(sb)), "p90": float(np.percentile(sb, 90)),
                                         "max": float(sb.max())} if len(sb) else None,
           "A_sharers_start_spread_us": {"median": float(np.median(sa)), "p90": float(np.percentile(sa, 90)),
                                         "max": float(sa.max())} if len(sa) else None,
           "last_tile_end_spread_us": float(np.ptp([eend[pair == p].max() for p in np.unique(pair)]))}
    # MMA idle between a pair's consecutive tiles (next first MMA - this tile's last commit)
    gaps = []
    for p in np.unique(pair):
        idx = np.where(pair == p)[0]
        idx = idx[np.argsort(start[idx])]
        gaps += list(start[idx[1:]] - mend[idx[:-1]])
    gaps = np.array(gaps)
    rep["inter_tile_mma_gap_us"] = {"median": float(np.median(gaps)), "p90": float(np.percentile(gaps, 90))} if gaps.size else None
    rep["mma_busy_fraction"] = float(dur.sum() / (dur.sum() + gaps.sum())) if gaps.size else None
    rep["wide"] = wide
    rep["no_c"] = noc
    print(json.dumps(rep))
    np.save(os.path.join(os.environ.get("TCX_REPORT_DIR", "gpurun_out"), f"trace_{cfg}_g{g}{'_wide' if wide else ''}.npy"), r)


if __name__ == "__main__":
    main()
