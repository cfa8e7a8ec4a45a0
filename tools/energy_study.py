#!/usr/bin/env python
"""Energy per launch of GEMM variants on the power-capped B200 (NVML total-energy counter).

At the 1000 W board cap a long GEMM's throughput is (P_cap - P_static) / (energy per FLOP), so the
lever is joules, not tensor-pipe occupancy.  For each variant: warm up, then launch back to back for
~SECONDS, reading nvmlDeviceGetTotalEnergyConsumption (mJ) and CUDA events around the run; report
J/launch, mean W, ms, TFLOP/s, pJ per (dense-equivalent) FLOP and the NVML SM clock.
python tools/energy_study.py OUT.jsonl variant[,variant...] [seconds] [rounds]
variants: c5, c5_noC, c5_t256, c5_pm2, c5_k4k, c5_k4k_noC, c3, c3_noC, c3_w512, c3_cublas, c4, c4_noC,
          probe_sp, probe_bf16 (pure MMA, smem-resident operands, all SMs), idle"""
import json
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2206_02874_b200 as tcx  # noqa: E402
import tcxgen as g  # noqa: E402


class Nvml:
    def __init__(self):
        import pynvml
        pynvml.nvmlInit()
        self.nv = pynvml
        self.h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())

    def energy_mj(self):
        return self.nv.nvmlDeviceGetTotalEnergyConsumption(self.h)

    def sample(self):
        return (self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM),
                int(self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)))


WORK = {}


def work(cfg):
    if cfg not in WORK:
        WORK.clear()
        torch.cuda.empty_cache()
        WORK[cfg] = bench.Work(cfg, 0, 1, torch.device("cuda", 0))
    return WORK[cfg]


def variant(name):
    """-> (step callable, dense-equivalent FLOPs per step)"""
    if name.startswith("c5"):
        if "k4k" in name:
            key = "c5k4k"
            if key not in WORK:
                WORK.clear(); torch.cuda.empty_cache()
                import types
                M, N, K = 65536, 16384, 4096
                vals, meta = g.sp24_problem(M, K, 0, "f16", "cuda")
                WORK[key] = types.SimpleNamespace(vals=vals, meta_hw=tcx.sp24_pack_meta(meta, M, K),
                                                  B=g.normal_matrix((N, K), "f16", 0, g.STREAM_B, "cuda"),
                                                  C=torch.zeros(M, N, device="cuda"), D=torch.empty(M, N, device="cuda"),
                                                  flops=2.0 * M * N * K)
            w = WORK[key]
        else:
            w = work("c5")
        C = None if name.endswith("noC") else w.C
        kw = {}
        if "t256" in name:
            kw["tile_m"] = 256
        if "pm2" in name and "mw" not in name:
            kw["tile_m"] = 256
            kw["pairs"] = (2, 1)
        for tag, pr in (("mwpm2", (2, 1)), ("mwpn2", (1, 2)), ("mw22", (2, 2))):   # M-wide tile in multicast groups
            if tag in name:
                kw["tile_m"] = 512
                kw["pairs"] = pr
        for tag, pr in (("t256pn2", (1, 2)), ("t256p22", (2, 2))):                 # 256-row tile in groups
            if tag in name:
                kw["tile_m"] = 256
                kw["pairs"] = pr
        # debug library (TCX_LIB_PATH=libtcx_debug.so) decomposition knobs: _nomma, _noload, _noepi
        kn = (2 if "_nomma" in name else 0) | (4 if "_noload" in name else 0) | (8 if "_noepi" in name else 0) | \
             (16 if "_slowdrain" in name else 0)
        if kn:
            kw["_knobs"] = kn
        import re
        mg = re.search(r"_g(m?)(\d+)", name)            # raster: _g16 = group_m 16, _gm8 = group_m -8
        if mg:
            kw["group_m"] = -int(mg.group(2)) if mg.group(1) else int(mg.group(2))
        return (lambda: tcx.gemm_sp24(w.vals, w.meta_hw, w.B, C, w.D, **kw)), w.flops
    if name.startswith("c3") or name.startswith("c4"):
        w = work(name[:2])
        C = None if "noC" in name else w.C
        if name == "c3_cublas":
            out = torch.empty(8192, 8192, dtype=torch.bfloat16, device="cuda")
            return (lambda: torch.matmul(w.A, w.B.t(), out=out)), w.flops
        kw = {"tile_n": 512} if "w512" in name else {}
        for tag, pr in (("_p12", (1, 2)), ("_p21", (2, 1)), ("_p22", (2, 2))):      # multicast clusters
            if tag in name:
                kw["pairs"] = pr
        kn = (2 if "_nomma" in name else 0) | (4 if "_noload" in name else 0) | (8 if "_noepi" in name else 0)
        if kn:                                    # debug library decomposition knobs
            kw["_fault"] = kn
        return (lambda: tcx.gemm(w.A, w.B, C, w.D, **kw)), w.flops
    if name.startswith("probe"):
        # probe_{sp,bf16}[_rot|_areuse]: pure MMA streams on every SM (smem-resident operands); _rot reads
        # a 4-stage ring at every k-offset (a GEMM's smem read pattern), _areuse shares A via the collector
        # suffix _n: operands drawn N(0,1) (the GEMM configs' data) instead of {-1, 0, 1}
        sp = name.startswith("probe_sp")
        base = name[:-2] if name.endswith("_n") else name
        mode = "stream_areuse" if base.endswith("_areuse") else "stream_rot" if base.endswith("_rot") else "stream"
        ab = tcx.F16 if sp else tcx.BF16
        n, k = (240, 32) if sp else (256, 16)
        iters = 4096
        es = 2
        fmt = "f16" if sp else "bf16"
        if name.endswith("_n"):
            a_op = g.normal_matrix((256, 32 // es), fmt, 1, 1, "cuda", redraw_zero=sp)
            b_op = g.normal_matrix((n, (64 if sp else 32) // es), fmt, 1, 2, "cuda")
        else:
            a_op = g.int32_matrix((256, 32 // es), 1, 1, -1, 1, "cuda").to(torch.float16 if sp else torch.bfloat16)
            b_op = g.int32_matrix((n, (64 if sp else 32) // es), 1, 2, -1, 1, "cuda").to(a_op.dtype)
        fl = 2.0 * 74 * iters * 16 * 256 * n * k
        return (lambda: tcx.probe("tc05_sp" if sp else "tc05", ab, tcx.F32, 256, n, k, cta_group=2, ilp=16,
                                  iters=iters, repeats=1, num_sms=148, n_acc=2 if mode == "stream_areuse" else 1,
                                  mode=mode, a_op=a_op, b_op=b_op)), fl
    if name == "tma_l2":
        # L2 -> SM operand staging alone: every SM streams 8 x 16 KiB TMA boxes per wait from an
        # L2-resident 16 MiB source (tcx_probe TMA_LOAD); "flops" here = bytes delivered
        iters = 20000
        return (lambda: tcx.probe("tma_load", tcx.S8, tcx.S32, 128, 128, 0, ilp=8, iters=iters, repeats=1,
                                  num_sms=148)), float(148 * (iters + 4) * 8 * 128 * 128)
    if name == "tma_l2_rand":
        # as tma_l2, the L2-resident source filled with pseudo-random bytes (toggles like operands)
        iters = 20000
        return (lambda: tcx.probe("tma_load", tcx.S8, tcx.S32, 128, 128, 0, ilp=8, iters=iters, repeats=1,
                                  num_sms=148, mode=1)), float(148 * (iters + 4) * 8 * 128 * 128)
    if name.startswith("dsmem"):
        # SM-to-SM forwarding inside clusters of 2 (dsmem2) or 4 (dsmem4): 4 x 16 KiB random boxes
        cs = int(name[5:])
        iters = 20000
        return (lambda: tcx.probe("dsmem", tcx.S8, tcx.S32, 0, 16384, 0, cta_group=cs, ilp=4, iters=iters, repeats=1,
                                  num_sms=148)), float((148 // cs) * cs * (iters + 4) * 4 * 16384)
    if name == "dram_copy":
        # HBM alone: a 2 GiB random buffer copied (read + write bytes), far beyond L2
        if "dram" not in WORK:
            WORK.clear(); torch.cuda.empty_cache()
            a = torch.randint(-2 ** 31, 2 ** 31 - 1, (1 << 29,), dtype=torch.int32, device="cuda")
            WORK["dram"] = (a, torch.empty_like(a))
        a, b = WORK["dram"]
        return (lambda: b.copy_(a)), float(2 * a.numel() * 4)
    if name == "idle":
        return (lambda: time.sleep(0.05)), 0.0
    raise ValueError(name)


def measure(name, seconds, nv):
    step, flops = variant(name)
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    time.sleep(0.3)
    samples = []
    stop = threading.Event()

    def sampler():
        while not stop.is_set():
            samples.append(nv.sample())
            time.sleep(0.02)
    th = threading.Thread(target=sampler, daemon=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    th.start()
    j0 = nv.energy_mj()
    t0 = time.time()
    e0.record()
    n = 0
    while time.time() - t0 < seconds:
        step()
        n += 1
        if n % 4 == 0:
            torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    t1 = time.time()
    j1 = nv.energy_mj()
    stop.set()
    th.join()
    ms = e0.elapsed_time(e1) / n
    joules = (j1 - j0) / 1000.0
    s = samples[len(samples) // 4:] or samples
    mhz = sorted(x[0] for x in s)
    return {"variant": name, "launches": n, "ms": round(ms, 4), "wall_s": round(t1 - t0, 3),
            "J_per_launch": round(joules / n, 4), "W": round(joules / (t1 - t0), 1),
            "tflops": round(flops / (ms * 1e-3) / 1e12, 1) if flops else None,
            "pJ_per_flop": round(joules / n / flops * 1e12, 4) if flops else None,
            "note": "data-movement variant: 'tflops' and 'pJ_per_flop' are per BYTE moved"
            if name in ("tma_l2", "tma_l2_rand", "dram_copy") or name.startswith("dsmem") else None,
            "sm_mhz_median": mhz[len(mhz) // 2] if mhz else None,
            "power_cap_frac": round(sum(1 for x in s if x[1] & 4) / max(1, len(s)), 2)}


def main():
    out = open(sys.argv[1], "a")
    names = sys.argv[2].split(",")
    seconds = float(sys.argv[3]) if len(sys.argv) > 3 else 1.5
    rounds = int(sys.argv[4]) if len(sys.argv) > 4 else 1
    torch.cuda.set_device(0)
    nv = Nvml()
    for r in range(rounds):
        order = names if r % 2 == 0 else names[::-1]
        for nm in order:
            d = measure(nm, seconds, nv)
            d["round"] = r
            print(json.dumps(d), flush=True)
            out.write(json.dumps(d) + "\n")
            out.flush()


if __name__ == "__main__":
    main()
