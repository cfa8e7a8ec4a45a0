#!/usr/bin/env python
"""tcx benchmark — BASELINE.json metric: dense & 2:4-sparse MMA TFLOP/s (INT8 TOPS) per B200,
% of tensor-core peak.

A step is one call of the hot path on its config's synthetic input, resident in HBM:
  c3     (default) dense BF16 GEMM M=N=K=8192, C FP32 zeros (real buffer), FP32 D  (configs[2])
  c3tf32 the same shape with TF32 inputs                                             (configs[2])
  c4     INT8 GEMM M=N=K=16384, C int32 U[-2^20,2^20], INT32 D                        (configs[3])
  c5     2:4 sparse FP16 GEMM M=65536, N=K=16384, C FP32 zeros                        (configs[4])
  c1     4096 m16n8k16 FP16 tiles (HBM-bound; GB/s)                                   (configs[0])
At N=1 the default run also measures c3tf32 / c4 / c5 / c1 on rank 0 ("also" key).
Multi-GPU (torchrun): rows of A, C, D are sharded across ranks — by default weak scaling (each
rank one config-sized row block of an N-times taller problem, per-GPU work fixed); --scaling strong
splits the config itself.  B is replicated by one NCCL broadcast before timing; time = max over ranks.

--impl reference times the CPU oracle (oracle/, exact Kulisch accumulation) on a bounded sample
of the same workload, on the host cores (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np
import torch

L2_BYTES = 126 * 1024 * 1024


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return {"bf16": d["bf16_tflops"], "bf16_sustained": d.get("bf16_tflops_sustained"), "hbm": d["hbm_gbs"],
                "source": "measured (MEASURED_PEAKS.json)"}
    return {"bf16": 1590.0, "bf16_sustained": 1400.0, "hbm": 6650.0, "source": "fallback (B200_PROFILING.md)"}


# nominal dense ratios vs bf16 (B200_PROFILING.md nominal table: tf32 1.1 vs 2.25; int8 = fp8 rate 4.5;
# 2:4 sparse doubles the dense rate): peak for kind = measured bf16 peak x ratio
CFG_SHAPES = {"c3": (8192, 8192, 8192), "c3tf32": (8192, 8192, 8192), "c3f16acc": (8192, 8192, 8192),
              "c4": (16384, 16384, 16384), "c4sp": (16384, 16384, 16384), "c3sptf32": (8192, 8192, 8192),
              "c5": (65536, 16384, 16384), "c1": (4096,)}
KIND_RATIO = {"bf16": 1.0, "f16": 1.0, "f16acc": 1.0, "tf32": 0.5, "s8": 2.0, "sp16": 2.0, "sp8": 4.0, "sptf32": 1.0}
# SURVEY §8(d)'s two extra denominators: the datasheet dense BF16 peak (2.25 PFLOP/s) x the same
# ratio, and the clock-normalised peak 148 SMs x 4096 dense BF16 FMA/clk/SM x ratio x 2 x the SM clock
# NVML saw during the timed region
DATASHEET_BF16_TFLOPS = 2250.0
BF16_FMA_PER_CLK_SM = 4096


class ClockSampler:
    """nvidia-smi style clocks + throttle reasons sampled via NVML during the timed region."""

    def __init__(self, index):
        self.samples = []
        self.on = False
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover
            log("nvml unavailable:", e)

    def _run(self):
        nv = self.nv
        while self.on:
            try:
                mhz = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                try:
                    pw = nv.nvmlDeviceGetPowerUsage(self.h) / 1000.0
                except Exception:
                    pw = None
                self.samples.append((time.time(), mhz, rs, pw))
            except Exception:
                pass
            time.sleep(0.005)

    def start(self):
        if self.ok:
            self.on = True
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()

    def stop(self):
        if self.ok and self.on:
            self.on = False
            self.t.join()

    def summary(self, t0, t1):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        nv = self.nv
        inside = [s for s in self.samples if t0 <= s[0] <= t1] or self.samples[-3:]
        names = {getattr(nv, "nvmlClocksEventReasonGpuIdle", 1): "gpu_idle",
                 getattr(nv, "nvmlClocksEventReasonApplicationsClocksSetting", 2): "applications_clocks_setting",
                 getattr(nv, "nvmlClocksEventReasonSwPowerCap", 4): "sw_power_cap",
                 getattr(nv, "nvmlClocksEventReasonHwSlowdown", 8): "hw_slowdown",
                 getattr(nv, "nvmlClocksEventReasonSyncBoost", 16): "sync_boost",
                 getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 32): "sw_thermal_slowdown",
                 getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 64): "hw_thermal_slowdown",
                 getattr(nv, "nvmlClocksEventReasonHwPowerBrakeSlowdown", 128): "hw_power_brake_slowdown"}
        rs = set()
        for _, _, r, _ in inside:
            for bit, nm in names.items():
                if r & bit:
                    rs.add(nm)
        mhz = [s[1] for s in inside]
        pw = [s[3] for s in inside if s[3] is not None]
        return {"sm_mhz": statistics.median(mhz) if mhz else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(rs), "samples": len(inside),
                "power_w_median": round(statistics.median(pw), 1) if pw else None}


def sparse_mwide(M, N, K, tf32=False, sm_count=148):
    """the sparse tile height the library picks by default (gemm_sp24.cu launch_sp_kind): the 512 x 240
    M-wide tile when M % 512 == 0, the K loop is long (K >= 16384, TF32 K >= 8192) and its tiles fill
    the waves within 3% of the 256-row tiles' fill"""
    pairs = sm_count // 2
    nt = (N + 239) // 240

    def fill(t):
        return t / (((t + pairs - 1) // pairs) * pairs)
    return M % 512 == 0 and K * (2 if tf32 else 1) >= 16384 and fill((M // 512) * nt) >= 0.97 * fill(((M + 255) // 256) * nt)


def dense_kernel_name(kind, M, N, K=8192, sm_count=148):
    """the dense kernel instance the library picks by default (gemm_dense.cu): the wave-aware narrow
    width when 256-wide tiles fill the waves poorly, the 256 x 512 tile for long K loops (K_eff >=
    16384 with a wave fill within 3%), else 1 x 2 multicast groups once there are >= 2 waves of
    256 x 256 pair tiles over >= 2 tile columns"""
    pairs = sm_count // 2
    mt = (M + 255) // 256

    def waves_cost(w, rate):
        t = mt * ((N + w - 1) // w)
        return ((t + pairs - 1) // pairs) * w * 1000 // rate

    c256 = waves_cost(256, 1000)
    best, bc = 256, c256
    for w, rate in ((224, 979), (192, 944), (160, 879), (128, 806)):
        c = waves_cost(w, rate)
        if c < bc and 20 * c <= 19 * c256:
            best, bc = w, c
    if best != 256:
        return f"gemm_dense_kernel<2,{kind},1,1,1,{best}> (256x{best} tile)"

    def fill(t):
        return t / (((t + pairs - 1) // pairs) * pairs)
    k_eff = 2 * K if kind == 1 else K // 2 if kind == 2 else K
    if kind != "f16acc" and k_eff >= 16384 and fill(mt * ((N + 511) // 512)) >= 0.97 * fill(mt * ((N + 255) // 256)):
        return f"gemm_dense_kernel<2,{kind},2,1,1,256> (256x512 tile)"
    n_tiles = (N + 255) // 256
    groups = n_tiles >= 2 and mt * n_tiles >= 2 * pairs
    return f"gemm_dense_kernel<2,{kind},1,1,{2 if groups else 1},256>" + (" (1x2 groups)" if groups else "")


# ----------------------------------------------------------------------------------- workloads
class Work:
    """one config on this rank: inputs resident in HBM, step() launches the hot path once."""

    def __init__(self, cfg, rank, world, dev, seed=0, scaling="strong"):
        import tcxgen
        import paper_2206_02874_b200 as tcx
        self.tcx, self.cfg, self.dev = tcx, cfg, dev
        self.rank, self.world = rank, world
        # weak scaling (N > 1): every rank owns a full config-sized row block of an N-times taller
        # problem (its rows drawn with seed + 1000 * rank); strong: the config itself split by rows
        self.weak = scaling == "weak" and world > 1
        from paper_2206_02874_b200.dist import shard_plan
        self._plan = lambda M: shard_plan(M, world, rank, "weak" if self.weak else "strong", seed)
        rs = self._plan(0)[2]                        # this rank's row seed
        g = tcxgen
        if cfg in ("c3", "c3tf32"):
            M = N = K = 8192
            fmt = "bf16" if cfg == "c3" else "tf32"
            self.kind = fmt
            self.shape = (M, N, K)
            m0, m1 = self._rows(M)
            self.A = g.normal_matrix((M, K), fmt, rs, g.STREAM_A, dev)[m0:m1].contiguous()
            self.B = self._bcast(lambda: g.normal_matrix((N, K), fmt, seed, g.STREAM_B, dev))
            self.C = torch.zeros(m1 - m0, N, dtype=torch.float32, device=dev)
            self.D = torch.empty(m1 - m0, N, dtype=torch.float32, device=dev)
            self.flops = 2.0 * (m1 - m0) * N * K
            self.alg_bytes = self.A.numel() * self.A.element_size() + self.B.numel() * self.B.element_size() + 8 * (m1 - m0) * N
            self.tf32 = fmt == "tf32"
            self.kernel = dense_kernel_name(0 if fmt == "bf16" else 1, m1 - m0, N, K)
            self.step = lambda: tcx.gemm(self.A, self.B, self.C, self.D, tf32=self.tf32)
            self.unit, self.bound = "TFLOP/s", "tensor"
        elif cfg == "c3f16acc":              # NEXT-2: FP16 inputs, FP16 accumulator, FP16 C/D at C3's shape
            M = N = K = 8192
            self.kind = "f16acc"
            self.shape = (M, N, K)
            m0, m1 = self._rows(M)
            self.A = g.normal_matrix((M, K), "f16", rs, g.STREAM_A, dev)[m0:m1].contiguous()
            self.B = self._bcast(lambda: g.normal_matrix((N, K), "f16", seed, g.STREAM_B, dev))
            self.C = torch.zeros(m1 - m0, N, dtype=torch.float16, device=dev)
            self.D = torch.empty(m1 - m0, N, dtype=torch.float16, device=dev)
            self.flops = 2.0 * (m1 - m0) * N * K
            self.alg_bytes = 2 * (self.A.numel() + self.B.numel()) + 4 * (m1 - m0) * N
            self.kernel = dense_kernel_name("f16acc", m1 - m0, N, K)
            self.step = lambda: tcx.gemm(self.A, self.B, self.C, self.D, f16_acc=True)
            self.unit, self.bound = "TFLOP/s", "tensor"
        elif cfg == "c4":
            M = N = K = 16384
            self.kind = "s8"
            self.shape = (M, N, K)
            m0, m1 = self._rows(M)
            self.A = g.int8_matrix((M, K), rs, g.STREAM_A, dev)[m0:m1].contiguous()
            self.B = self._bcast(lambda: g.int8_matrix((N, K), seed, g.STREAM_B, dev))
            self.C = g.int32_matrix((M, N), rs, g.STREAM_C, device=dev)[m0:m1].contiguous()
            self.D = torch.empty(m1 - m0, N, dtype=torch.int32, device=dev)
            self.flops = 2.0 * (m1 - m0) * N * K
            self.alg_bytes = self.A.numel() + self.B.numel() + 8 * (m1 - m0) * N
            self.kernel = dense_kernel_name(2, m1 - m0, N, K)
            self.step = lambda: tcx.gemm(self.A, self.B, self.C, self.D)
            self.unit, self.bound = "TOPS", "tensor"
        elif cfg in ("c5", "c5s"):       # c5s: an 8192-row slice of C5 (profiling only)
            M, N, K = (65536 if cfg == "c5" else 8192), 16384, 16384
            self.kind = "sp16"
            self.shape = (M, N, K)
            m0, m1 = self._rows(M)
            vals, meta = g.sp24_problem(M, K, rs, "f16", dev)
            self.vals = vals[m0:m1].contiguous()
            meta = meta[m0:m1].contiguous()
            del vals
            self.meta_hw = tcx.sp24_pack_meta(meta, m1 - m0, K)
            del meta
            self.B = self._bcast(lambda: g.normal_matrix((N, K), "f16", seed, g.STREAM_B, dev))
            self.C = torch.zeros(m1 - m0, N, dtype=torch.float32, device=dev)
            self.D = torch.empty(m1 - m0, N, dtype=torch.float32, device=dev)
            # dense-equivalent FLOPs 2MNK (NVIDIA's sparse convention: peak = 2x dense); the effective
            # (kept-product) rate is half of it and is reported beside it (DESIGN.md R-C13)
            self.flops = 2.0 * (m1 - m0) * N * K
            self.alg_bytes = self.vals.numel() * 2 + self.meta_hw.numel() + self.B.numel() * 2 + 8 * (m1 - m0) * N
            mw = sparse_mwide(m1 - m0, N, K)                               # gemm_sp24.cu's M-wide default
            self.kernel = "gemm_sp24_kernel<2,f16,M-wide 512x240>" if mw else "gemm_sp24_kernel<2,f16,256x240>"
            self.step = lambda: tcx.gemm_sp24(self.vals, self.meta_hw, self.B, self.C, self.D)
            self.unit, self.bound = "TFLOP/s", "tensor"
        elif cfg in ("c4sp", "c3sptf32"):   # NEXT-1: INT8 2:4 at C4's shape, TF32 1:2 at C3's shape
            M = N = K = 16384 if cfg == "c4sp" else 8192
            self.kind = "sp8" if cfg == "c4sp" else "sptf32"
            self.shape = (M, N, K)
            m0, m1 = self._rows(M)
            if cfg == "c4sp":
                vals, meta = g.sp24_problem_i8(M, K, rs, dev)
                self.B = self._bcast(lambda: g.int8_matrix((N, K), seed, g.STREAM_B, dev))
                self.C = g.int32_matrix((M, N), rs, g.STREAM_C, device=dev)[m0:m1].contiguous()
                self.D = torch.empty(m1 - m0, N, dtype=torch.int32, device=dev)
                ab, esize = tcx.S8, 1
            else:
                vals, meta = g.sp12_problem_tf32(M, K, rs, dev)
                self.B = self._bcast(lambda: g.normal_matrix((N, K), "tf32", seed, g.STREAM_B, dev))
                self.C = torch.zeros(m1 - m0, N, dtype=torch.float32, device=dev)
                self.D = torch.empty(m1 - m0, N, dtype=torch.float32, device=dev)
                ab, esize = tcx.TF32, 4
            self.vals = vals[m0:m1].contiguous()
            self.meta_hw = tcx.sp24_pack_meta(meta[m0:m1].contiguous(), m1 - m0, K, ab=ab)
            del vals, meta
            self.flops = 2.0 * (m1 - m0) * N * K          # dense-equivalent (DESIGN.md R-C13)
            self.alg_bytes = (self.vals.numel() * esize + self.meta_hw.numel() + self.B.numel() * esize
                              + 8 * (m1 - m0) * N)
            self.kernel = ("gemm_sp24_kernel<2,i8>" if cfg == "c4sp" else
                           "gemm_sp24_kernel<2,tf32,M-wide 512x240>" if sparse_mwide(m1 - m0, N, K, True)
                           else "gemm_sp24_kernel<2,tf32,256x240>")
            tf = cfg == "c3sptf32"
            self.step = lambda: tcx.gemm_sp24(self.vals, self.meta_hw, self.B, self.C, self.D, tf32=tf)
            self.unit, self.bound = ("TOPS" if cfg == "c4sp" else "TFLOP/s"), "tensor"
        elif cfg == "c1":
            count = 4096
            self.kind = "f16"
            self.shape = (count,)
            copies = 64                                 # 64 x 7 MiB = 470 MB >> L2: reads are cold
            self.As = [g.uniform_matrix((count, 16, 16), "f16", seed + i, g.STREAM_A, device=dev) for i in range(copies)]
            self.Bs = [g.uniform_matrix((count, 8, 16), "f16", seed + i, g.STREAM_B, device=dev) for i in range(copies)]
            self.Cs = [g.uniform_matrix((count, 16, 8), "f32", seed + i, g.STREAM_C, device=dev) for i in range(copies)]
            self.Ds = [torch.empty(count, 16, 8, device=dev) for _ in range(copies)]
            # one step = one CUDA-graph replay of 64 tcx_mma_tiles calls over the 64 copies (the
            # kernel is ~2 us; the graph removes host launch overhead from the device timing)
            self.flops = 4096.0 * count * copies
            self.alg_bytes = 1792 * count * copies
            self.kernel = "tiles16_kernel<0>"
            self.launches_per_step = copies
            torch.cuda.synchronize()
            s = torch.cuda.Stream()
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):
                for j in range(copies):            # warm (module load) outside capture
                    tcx.mma_tiles(self.As[j], self.Bs[j], self.Cs[j], self.Ds[j])
            torch.cuda.current_stream().wait_stream(s)
            torch.cuda.synchronize()
            self.graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(self.graph):
                for j in range(copies):
                    tcx.mma_tiles(self.As[j], self.Bs[j], self.Cs[j], self.Ds[j])
            self.step = self.graph.replay
            self.unit, self.bound = "GB/s", "hbm"
        else:
            raise ValueError(cfg)

    def _rows(self, M):
        m0, m1, _, _ = self._plan(M)
        return m0, m1

    def _bcast(self, make):
        import torch.distributed as dist
        if self.world == 1:
            return make()
        from paper_2206_02874_b200.dist import broadcast_replicated
        t = make()               # every rank allocates B; rank 0's copy is the one broadcast
        if self.rank != 0:
            t.zero_()
        broadcast_replicated(t, src=0)    # one-time NCCL broadcast over NVLink (not timed)
        return t

    def metric_value(self, seconds_per_step):
        if self.unit == "GB/s":
            return self.alg_bytes / seconds_per_step / 1e9
        return self.flops / seconds_per_step / 1e12

    # host-buffer end-to-end step through the public API: H2D of inputs, the call, D2H of D
    def e2e_setup(self):
        """host (pinned) copies of the step's inputs and result; two device slots so that step i's
        H2D, step i-1's GEMM and step i-2's D2H run concurrently on three streams (the copy
        engines and the SMs overlap; every step still moves all its bytes inside the timed region)."""
        if self.cfg == "c1":
            ins = [self.As[0], self.Bs[0], self.Cs[0]]
            out = self.Ds[0]
            self.e2e_op = lambda d: self.tcx.mma_tiles(d[0], d[1], d[2], d[3])
        elif hasattr(self, "vals"):                     # sparse configs
            ins = [self.vals, self.meta_hw, self.B, self.C]
            out = self.D
            tf = self.cfg == "c3sptf32"
            self.e2e_op = lambda d: self.tcx.gemm_sp24(d[0], d[1], d[2], d[3], d[4], tf32=tf)
        else:
            ins = [self.A, self.B, self.C]
            out = self.D
            tf = getattr(self, "tf32", False)
            h = self.cfg == "c3f16acc"
            self.e2e_op = lambda d: self.tcx.gemm(d[0], d[1], d[2], d[3], tf32=tf, f16_acc=h)
        self.h_ins = [t.cpu().pin_memory() for t in ins]
        self.hD = torch.empty_like(out, device="cpu").pin_memory()
        self.slots = [[torch.empty_like(t) for t in ins] + [torch.empty_like(out)] for _ in range(2)]
        self.s_in, self.s_cmp, self.s_out = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
        self.ev_in = [torch.cuda.Event() for _ in range(2)]
        self.ev_cmp = [torch.cuda.Event() for _ in range(2)]
        self.ev_out = [torch.cuda.Event() for _ in range(2)]
        for k in range(2):                              # slots start free
            self.ev_cmp[k].record(self.s_cmp)
            self.ev_out[k].record(self.s_out)
        self.h2d = sum(t.numel() * t.element_size() for t in self.h_ins)
        self.d2h = self.hD.numel() * self.hD.element_size()

    def e2e_step(self, i):
        k = i % 2
        d = self.slots[k]
        self.s_in.wait_event(self.ev_cmp[k])           # the GEMM of step i-2 is done reading slot k
        with torch.cuda.stream(self.s_in):
            for dst, src in zip(d, self.h_ins):
                dst.copy_(src, non_blocking=True)
            self.ev_in[k].record(self.s_in)
        self.s_cmp.wait_event(self.ev_in[k])
        self.s_cmp.wait_event(self.ev_out[k])          # slot k's D was read back (step i-2)
        with torch.cuda.stream(self.s_cmp):
            self.e2e_op(d)
            self.ev_cmp[k].record(self.s_cmp)
        self.s_out.wait_event(self.ev_cmp[k])
        with torch.cuda.stream(self.s_out):
            self.hD.copy_(d[-1], non_blocking=True)
            self.ev_out[k].record(self.s_out)


def time_steps(work, steps, warmup, dist_on, sampler=None):
    """W untimed warm-ups, then EXACTLY `steps` steps between barrier+sync; CUDA events on the
    launching (current) stream; returns (ms_per_step on this rank, launches, t0, t1)."""
    import paper_2206_02874_b200 as tcx
    for _ in range(warmup):
        work.step()
    torch.cuda.synchronize()
    if dist_on:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    st0 = torch.zeros(2 * 256, dtype=torch.int64, device=work.dev)
    st1 = torch.zeros(2 * 256, dtype=torch.int64, device=work.dev)
    n0 = tcx.launch_count()
    t0 = time.time()
    tcx.sm_clock_stamp(st0)                 # per-SM (clock64, globaltimer) just before / after the region
    e0.record(stream)
    for _ in range(steps):
        work.step()
    e1.record(stream)
    tcx.sm_clock_stamp(st1)
    torch.cuda.synchronize()
    t1 = time.time()
    if dist_on:
        torch.distributed.barrier()
    launches = tcx.launch_count() - n0 + steps * getattr(work, "launches_per_step", 0)   # graph replays launch without the host counter
    work.sm_mhz_eff = tcx.sm_mhz_between(st0, st1)
    return e0.elapsed_time(e1) / steps, launches, t0, t1


def e2e_copy_bound(work, reps=5):
    """the e2e step's floor on this box: the same H2D of every input and D2H of the result, both
    directions at once on the e2e streams, with no GEMM (PCIe Gen5 x16 full duplex)"""
    cur = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(cur)
    for _ in range(reps):
        work.s_in.wait_stream(cur)
        work.s_out.wait_stream(cur)
        with torch.cuda.stream(work.s_in):
            for dst, src in zip(work.slots[0], work.h_ins):
                dst.copy_(src, non_blocking=True)
        with torch.cuda.stream(work.s_out):
            work.hD.copy_(work.slots[1][-1], non_blocking=True)
        cur.wait_stream(work.s_in)
        cur.wait_stream(work.s_out)
    e1.record(cur)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def time_e2e(work, steps, warmup):
    """end-to-end through the public API: every step's H2D of its inputs (pinned host memory), the
    call, and the D2H of its result, pipelined over three streams; CUDA events from the first H2D
    to the last D2H."""
    work.e2e_setup()
    for i in range(max(1, warmup)):
        work.e2e_step(i)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(work.s_in)
    for i in range(steps):
        work.e2e_step(i)
    e1.record(work.s_out)                               # after the last D2H, which follows every step
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


def sustained(work, seconds, sampler, fn=None):
    """SURVEY §8(d)'s sustained figure: back-to-back steps for `seconds` (the board settles at its
    power cap), timed in chunks of CUDA events; returns the median chunk's metric value and the NVML
    clock record of the run.  `fn` replaces work.step (the cuBLAS anchor)."""
    step = fn or work.step
    chunk = 50
    vals = []
    sampler.samples = []
    sampler.start()
    t0 = time.time()
    while time.time() - t0 < seconds:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(chunk):
            step()
        e1.record()
        e1.synchronize()
        vals.append(work.metric_value(e0.elapsed_time(e1) / chunk * 1e-3))
    t1 = time.time()
    sampler.stop()
    return {"value": round(float(np.median(vals)), 2), "seconds": round(t1 - t0, 2), "chunks": len(vals),
            "steps_per_chunk": chunk, "clocks": sampler.summary(t0, t1)}


def best_of(work, n=10):
    """SURVEY §8(d)'s burst figure: the fastest of n individually event-timed steps (after warm-up)."""
    best = float("inf")
    for _ in range(n):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        work.step()
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return round(work.metric_value(best * 1e-3), 2)


def library_anchor(work, steps):
    """the same-run library rate for this config's dtype and shape (cuBLAS through torch, no C):
    bf16 torch.matmul, TF32 torch.matmul with allow_tf32 on the same TF32-representable FP32
    operands, INT8 torch._int_mm (INT32 out).  A measured peak of that dtype on this box, beside
    the bf16-peak x nominal-ratio denominator (the ratio alone let fracs pass 1)."""
    A, Bt = work.A, work.B.t()
    if work.kind == "s8":
        fn = lambda: torch._int_mm(A, Bt)
    elif work.kind == "tf32":
        def fn():
            prev = torch.backends.cuda.matmul.allow_tf32
            torch.backends.cuda.matmul.allow_tf32 = True
            try:
                return torch.matmul(A, Bt)
            finally:
                torch.backends.cuda.matmul.allow_tf32 = prev
    else:
        fn = lambda: torch.matmul(A, Bt)
    try:
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        best = float("inf")
        for _ in range(max(3, steps)):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            e1.synchronize()
            best = min(best, e0.elapsed_time(e1))
        return round(work.flops / (best * 1e-3) / 1e12, 1)
    except Exception as e:   # a library without this dtype / shape: say so, never substitute
        log("anchor unavailable:", e)
        return None


def same_work_anchor(work, steps):
    """C3 context: cuBLAS doing exactly this config's work — BF16 inputs, the FP32 C read and FP32 D
    written (torch.addmm(C, A, B^T, out_dtype=float32)) — best of n; torch.matmul's BF16-out line
    (the MEASURED_PEAKS method) skips the C read and writes half the D bytes."""
    Bt = work.B.t()
    out = torch.empty_like(work.D)
    try:
        fn = lambda: torch.addmm(work.C, work.A, Bt, out_dtype=torch.float32, out=out)
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        best = float("inf")
        for _ in range(max(3, steps)):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            e1.synchronize()
            best = min(best, e0.elapsed_time(e1))
        return round(work.flops / (best * 1e-3) / 1e12, 1), fn
    except Exception as e:
        log("same-work anchor unavailable:", e)
        return None, None


# tcx_probe operands per kind: (probe kind, ab code name, generator fmt or None = int8, UMMA N)
_POWER_KINDS = {"bf16": ("tc05", "BF16", "bf16", 256), "tf32": ("tc05", "TF32", "tf32", 256),
                "s8": ("tc05", "S8", None, 256), "sp16": ("tc05_sp", "F16", "f16", 240),
                "sp8": ("tc05_sp", "S8", None, 240), "sptf32": ("tc05_sp", "TF32", "tf32", 240)}


def power_roofline(kind, seconds=2.0):
    """The tensor cores alone at the board's power cap: tcx_probe STREAM_ROT on
    every SM — CTA-pair MMAs of this config's kind (bench KIND_RATIO names: bf16, tf32, s8, sp16, sp8,
    sptf32) on N(0,1) operands (INT8: uniform) read from a 4-stage smem ring, no operand loads, no
    epilogue — back to back for ~`seconds`; returns the median call's dense-equivalent TFLOP/s (TOPS).
    No GEMM of that kind can exceed it at the cap: it is the power roofline."""
    import tcxgen as g
    import paper_2206_02874_b200 as tcx
    pkind, abn, fmt, n = _POWER_KINDS[kind]
    sp = pkind == "tc05_sp"
    ab = getattr(tcx, abn)
    es = {"BF16": 2, "F16": 2, "TF32": 4, "S8": 1}[abn]
    ka, kb = 32 // es, (64 if sp else 32) // es          # A: 32 bytes of K (kept values), B: one UMMA K
    if fmt:
        a = g.normal_matrix((256, ka), fmt, 1, 1, "cuda", redraw_zero=sp)
        b = g.normal_matrix((n, kb), fmt, 1, 2, "cuda")
    else:
        a = g.int8_matrix((256, ka), 1, 1, "cuda")
        b = g.int8_matrix((n, kb), 1, 2, "cuda")
    cd = tcx.S32 if abn == "S8" else tcx.F32
    call = lambda it: tcx.probe(pkind, ab, cd, 256, n, kb, cta_group=2, ilp=16, iters=it,
                                repeats=1, num_sms=148, n_acc=1, mode="stream_rot", a_op=a, b_op=b)
    r = call(512)
    iters = int(min(2_000_000, max(512, 0.25 / max(r["ns_per_iter"] * 1e-9, 1e-9))))   # ~0.25 s per call
    vals = []
    t0 = time.time()
    while time.time() - t0 < seconds:
        r = call(iters)
        vals.append(2.0 * r["fma_per_clk_per_sm"] * 148 * r["sm_mhz"] * 1e6 / 1e12)
    vals.sort()
    return round(vals[len(vals) // 2], 1)


def cusparselt_anchor(work, steps=5):
    """C5 context: cuSPARSELt (torch._cslt_sparse_mm) on the same 2:4 operand; FP16 output and no C
    (its FP32 output is refused for FP16 inputs), i.e. less work than the config — best of n."""
    import tcxgen as g
    if not (getattr(torch.backends, "cusparselt", None) and torch.backends.cusparselt.is_available()):
        return None
    try:
        M, N, K = work.shape
        vals = work.vals
        pairs = g.sp24_pairs(M, K, 0, g.STREAM_POS, work.dev).long()
        P = torch.tensor(g.PAIRS, device=work.dev)[pairs]
        cols = (torch.arange(K // 4, device=work.dev) * 4).view(1, -1)
        dense = torch.zeros(M, K, dtype=vals.dtype, device=work.dev)
        dense.scatter_(1, cols + P[..., 0], vals[:, 0::2])
        dense.scatter_(1, cols + P[..., 1], vals[:, 1::2])
        del pairs, P
        comp = torch._cslt_compress(dense)
        del dense
        Bd = work.B.t()
        fn = lambda: torch._cslt_sparse_mm(comp, Bd)
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        best = float("inf")
        for _ in range(steps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            e1.synchronize()
            best = min(best, e0.elapsed_time(e1))
        del comp
        torch.cuda.empty_cache()
        return round(work.flops / (best * 1e-3) / 1e12, 1)
    except Exception as e:
        log("cuSPARSELt anchor unavailable:", e)
        return None


def tiles_steady_state(tcx, dev, count=524288, reps=10):
    """C1's kernel at steady state: one launch over 524,288 m16n8k16 FP16 tiles (940 MB > L2),
    CUDA events over `reps` launches; the C1 line itself is a 7 MB launch bound by launch latency."""
    import tcxgen as g
    A = g.uniform_matrix((count, 16, 16), "f16", 1, g.STREAM_A, device=dev)
    B = g.uniform_matrix((count, 8, 16), "f16", 1, g.STREAM_B, device=dev)
    C = g.uniform_matrix((count, 16, 8), "f32", 1, g.STREAM_C, device=dev)
    D = torch.empty(count, 16, 8, device=dev)
    for _ in range(3):
        tcx.mma_tiles(A, B, C, D)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        tcx.mma_tiles(A, B, C, D)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / reps
    gbs = 1792.0 * count / (us * 1e-6) / 1e9
    return {"tiles": count, "us_per_launch": round(us, 2), "GB/s": round(gbs, 1),
            "frac_of_hbm": round(gbs / peaks()["hbm"], 4)}


def roofline(work, ms, pk, clocks=None, anchor=None):
    src = None
    if work.bound == "hbm":
        ach = work.alg_bytes / (ms * 1e-3) / 1e9
        peak = pk["hbm"]
        unit = "GB/s"
    else:
        ach = work.flops / (ms * 1e-3) / 1e12
        peak = pk["bf16"] * KIND_RATIO[work.kind]
        unit = "TFLOP/s"
        if KIND_RATIO[work.kind] != 1.0:
            # a derived denominator (MEASURED_PEAKS bf16 x nominal ratio) is not a rate this dtype was
            # seen to reach: the primary peak is the HIGHEST rate measured for this dtype on this box —
            # the derived one, the same-run library kernel (best of n) or the power-capped MMA-only
            # probe of this kind — so no fraction rests on a ratio the hardware beats (bf16 keeps
            # MEASURED_PEAKS' own number, as the contract names it)
            if anchor and anchor > peak:
                peak, src = anchor, "same-run library anchor (best of n, this dtype and shape)"
            # (apply_power_roofline adds the power-capped MMA-only probe of this kind as a candidate)
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        traffic = json.load(open(tp)).get(work.cfg)
    extra = {}
    capped = bool(clocks) and "sw_power_cap" in (clocks.get("reasons") or [])
    if work.bound == "tensor" and pk.get("bf16_sustained") and capped:
        # the run sat at the power cap: the measured sustained (power-capped, back to back for 4 s)
        # figure is the matching denominator; `frac` stays against the burst peak
        ps = pk["bf16_sustained"] * KIND_RATIO[work.kind]
        extra = {"peak_sustained": round(ps, 2), "frac_sustained": round(ach / ps, 4)}
    if work.bound == "tensor":
        r = KIND_RATIO[work.kind]
        den = {"datasheet": {"peak": DATASHEET_BF16_TFLOPS * r, "frac": round(ach / (DATASHEET_BF16_TFLOPS * r), 4)}}
        # the clock-normalised peak: the average SM clock over the timed region itself, from per-SM
        # clock64 / globaltimer stamps bracketing it (tcx_sm_clock_stamp), else the NVML median
        mhz_eff = getattr(work, "sm_mhz_eff", None)
        mhz = mhz_eff or (clocks or {}).get("sm_mhz")
        if mhz:
            cn = 148 * BF16_FMA_PER_CLK_SM * r * 2 * mhz * 1e6 / 1e12
            den["clock_normalised"] = {"peak": round(cn, 1), "sm_mhz": round(mhz, 1), "frac": round(ach / cn, 4),
                                       "clock_source": "in-run SM clock stamps" if mhz_eff else "NVML samples"}
        if anchor:
            den["same_run_library"] = {"peak": anchor, "frac": round(ach / anchor, 4)}
        extra["denominators"] = den
    if src is None:
        src = pk["source"] + (" x nominal %s/bf16 ratio %.1f" % (work.kind, KIND_RATIO[work.kind])
                              if work.bound == "tensor" and KIND_RATIO[work.kind] != 1.0 else "")
    return {"bound": work.bound, "achieved": round(ach, 2), "peak": round(peak, 2), "unit": unit,
            "frac": round(ach / peak, 4), **extra, "traffic": traffic, "kernel": work.kernel,
            "peak_source": src}


def apply_power_roofline(rl, power, kind):
    """Add the power-capped MMA-only denominator (power_roofline(kind)) to a roofline dict; for a kind
    whose primary peak is derived (KIND_RATIO != 1) it is also a candidate for the primary: the
    highest rate measured for the dtype on this box is the denominator."""
    ach = rl["achieved"]
    rl.setdefault("denominators", {})["power_capped_mma_only"] = {
        "peak": power, "frac": round(ach / power, 4),
        "what": f"tcx_probe STREAM_ROT: {kind} CTA-pair MMAs alone on all SMs, N(0,1) operands "
                "(INT8 uniform), no loads or epilogue, at the 1000 W cap (~2 s)"}
    if KIND_RATIO[kind] != 1.0 and power > rl["peak"]:
        rl["peak"], rl["frac"] = round(power, 2), round(ach / power, 4)
        rl["peak_source"] = "power-capped MMA-only probe of this kind (tcx_probe STREAM_ROT, this run)"
    return rl


# ----------------------------------------------------------------------------------- oracle baseline
def oracle_sample(cfg, seconds=12.0, seed=0):
    """time the CPU oracle (as it stands) on a bounded sample of the config; returns dict."""
    import oracle as O
    import tcxgen as g
    cores = len(os.sched_getaffinity(0))
    rng = np.random.default_rng(seed)
    wall0 = time.perf_counter()          # wall-clock cap: counter-based row generation is not timed
    if cfg in ("c3", "c3tf32", "c4"):
        M = N = K = 16384 if cfg == "c4" else 8192
        fmt = {"c3": "bf16", "c3tf32": "tf32", "c4": "s8"}[cfg]
        ab = {"bf16": O.BF16, "tf32": O.TF32, "s8": O.S8}[fmt]
        # a sample of R rows x S cols of the same synthetic matrices (counter-based generator; INT8's
        # exact dot is cheap, so a bigger block keeps generation from dominating the wall time)
        R, S = (64, 64) if cfg == "c4" else (16, 16)

        def rows_of(stream, idx, n_cols):
            out = []
            for r in idx:   # the exact row r of the synthetic matrix, by counters
                if fmt == "s8":
                    out.append(_counter_row_int8(seed, stream, int(r), n_cols))
                else:
                    out.append(_counter_row_fp(seed, stream, int(r), n_cols, fmt))
            return np.stack(out)

        t_total = 0.0
        outputs = 0
        while t_total < seconds and time.perf_counter() - wall0 < 2.5 * seconds + 2:
            ri = rng.integers(0, M, R); ci = rng.integers(0, N, S)
            Ah = rows_of(g.STREAM_A, ri, K)
            Bh = rows_of(g.STREAM_B, ci, K)
            Ch = None
            if cfg == "c4":
                Ch = np.stack([_counter_row_int32(seed, g.STREAM_C, int(r), N)[ci] for r in ri]).astype(np.int32)
            rr, cc = np.meshgrid(np.arange(R), np.arange(S), indexing="ij")
            t0 = time.perf_counter()
            O.gemm_samples(ab, Ah, Bh, Ch.view(np.uint32) if Ch is not None else None, rr.ravel(), cc.ravel(), cores)
            t_total += time.perf_counter() - t0
            outputs += R * S
        ops = 2.0 * K * outputs
        return {"value": ops / t_total / 1e12, "unit": "TOPS" if cfg == "c4" else "TFLOP/s", "cores": cores,
                "kind": "oracle", "sample": f"{outputs} sampled outputs of the {M}x{N}x{K} {fmt} GEMM "
                f"({outputs * K:.3g} exact MACs) in {t_total:.1f} s", "seconds": t_total}
    if cfg == "c5":
        M, N, K = 65536, 16384, 16384
        R, S = 8, 16
        t_total, outputs = 0.0, 0
        while t_total < seconds and time.perf_counter() - wall0 < 2.5 * seconds + 2:
            ri = rng.integers(0, M, R); ci = rng.integers(0, N, S)
            vals = np.stack([_counter_row_fp(seed, g.STREAM_SPVAL, int(r), K // 2, "f16", redraw=True) for r in ri])
            meta = np.stack([_counter_meta_row(seed, int(r), K) for r in ri])
            Bh = np.stack([_counter_row_fp(seed, g.STREAM_B, int(c), K, "f16") for c in ci])
            t0 = time.perf_counter()
            dense = O.sp24_expand(vals, meta, K)
            rr, cc = np.meshgrid(np.arange(R), np.arange(S), indexing="ij")
            O.gemm_samples(O.F16, dense, Bh, None, rr.ravel(), cc.ravel(), cores)
            t_total += time.perf_counter() - t0
            outputs += R * S
        return {"value": 2.0 * (K // 2) * outputs / t_total / 1e12, "unit": "TFLOP/s", "cores": cores, "kind": "oracle",
                "sample": f"{outputs} sampled outputs of the {M}x{N}x{K} 2:4 FP16 GEMM in {t_total:.1f} s",
                "seconds": t_total}
    if cfg == "c3f16acc":                        # FP16 A, B, FP16 C = 0, FP16 accumulator: exact, one RNE16
        M = N = K = 8192
        R, S = 16, 16
        t_total, outputs = 0.0, 0
        while t_total < seconds and time.perf_counter() - wall0 < 2.5 * seconds + 2:
            ri = rng.integers(0, M, R); ci = rng.integers(0, N, S)
            Ah = np.stack([_counter_row_fp(seed, g.STREAM_A, int(r), K, "f16") for r in ri])
            Bh = np.stack([_counter_row_fp(seed, g.STREAM_B, int(c), K, "f16") for c in ci])
            rr, cc = np.meshgrid(np.arange(R), np.arange(S), indexing="ij")
            t0 = time.perf_counter()
            O.gemm_samples(O.F16, Ah, Bh, np.zeros((R, S), np.uint16), rr.ravel(), cc.ravel(), cores, cd=O.F16)
            t_total += time.perf_counter() - t0
            outputs += R * S
        return {"value": 2.0 * K * outputs / t_total / 1e12, "unit": "TFLOP/s", "cores": cores, "kind": "oracle",
                "sample": f"{outputs} sampled outputs of the {M}x{N}x{K} FP16-accumulate GEMM in {t_total:.1f} s",
                "seconds": t_total}
    if cfg in ("c4sp", "c3sptf32"):             # INT8 2:4 (C4's shape) / TF32 1:2 (C3's shape): expand, then dense
        i8 = cfg == "c4sp"
        M = N = K = 16384 if i8 else 8192
        R, S = (32, 64) if i8 else (16, 16)
        t_total, outputs = 0.0, 0
        while t_total < seconds and time.perf_counter() - wall0 < 2.5 * seconds + 2:
            ri = rng.integers(0, M, R); ci = rng.integers(0, N, S)
            if i8:
                v = np.stack([_counter_row_int32(seed, g.STREAM_SPVAL, int(r), K // 2, -128, 126) for r in ri])
                vals = np.where(v >= 0, v + 1, v).astype(np.int8)
                meta = np.stack([_counter_meta_row(seed, int(r), K) for r in ri])
                Bh = np.stack([_counter_row_int8(seed, g.STREAM_B, int(c), K) for c in ci])
                Ch = np.stack([_counter_row_int32(seed, g.STREAM_C, int(r), N)[ci] for r in ri]).astype(np.int32)
            else:
                vals = np.stack([_counter_row_fp(seed, g.STREAM_SPVAL, int(r), K // 2, "tf32", redraw=True) for r in ri])
                meta = np.stack([_counter_meta_row_sp12(seed, int(r), K) for r in ri])
                Bh = np.stack([_counter_row_fp(seed, g.STREAM_B, int(c), K, "tf32") for c in ci])
                Ch = None
            rr, cc = np.meshgrid(np.arange(R), np.arange(S), indexing="ij")
            t0 = time.perf_counter()
            dense = O.sp24_expand(vals, meta, K)
            O.gemm_samples(O.S8 if i8 else O.TF32, dense, Bh, Ch.view(np.uint32) if Ch is not None else None,
                           rr.ravel(), cc.ravel(), cores)
            t_total += time.perf_counter() - t0
            outputs += R * S
        return {"value": 2.0 * (K // 2) * outputs / t_total / 1e12, "unit": "TOPS" if i8 else "TFLOP/s", "cores": cores,
                "kind": "oracle", "sample": f"{outputs} sampled outputs of the {M}x{N}x{K} "
                f"{'INT8 2:4' if i8 else 'TF32 1:2'} sparse GEMM in {t_total:.1f} s", "seconds": t_total}
    if cfg == "c1":
        count = 4096
        A = g.uniform_matrix((count, 16, 16), "f16", seed, g.STREAM_A)
        B = g.uniform_matrix((count, 8, 16), "f16", seed, g.STREAM_B)
        C = g.uniform_matrix((count, 16, 8), "f32", seed, g.STREAM_C)
        hb = lambda t: t.view(torch.int16).numpy().view(np.uint16)
        t0 = time.perf_counter()
        n = 0
        while time.perf_counter() - t0 < seconds:
            O.tiles(O.F16, 16, 8, 16, hb(A), hb(B), C.view(torch.int32).numpy().view(np.uint32))
            n += 1
        dt = time.perf_counter() - t0
        return {"value": 1792 * count * n / dt / 1e9, "unit": "GB/s", "cores": 1, "kind": "oracle",
                "sample": f"{n} whole C1 batches (4096 tiles) in {dt:.1f} s", "seconds": dt}
    raise ValueError(cfg)


def _counter_row_fp(seed, stream, r, n, fmt, redraw=False):
    import tcxgen as g
    v = g.to_format(g.normal(seed, stream, r * n, n), fmt)
    if redraw:
        k = 1
        while bool((v == 0).any()):
            alt = g.to_format(g.normal(seed, stream + 64 * k, r * n, n), fmt)
            v = torch.where(v == 0, alt, v)
            k += 1
    return v.view(torch.int32 if fmt == "tf32" else torch.int16).numpy().view(np.uint32 if fmt == "tf32" else np.uint16)


def _counter_row_int8(seed, stream, r, n):
    import tcxgen as g
    z = g.splitmix(seed, stream, torch.arange(r * n, (r + 1) * n, dtype=torch.int64))
    return (g._srl(z, 56) - 128).to(torch.int8).numpy()


def _counter_row_int32(seed, stream, r, n, lo=-(1 << 20), hi=1 << 20):
    import tcxgen as g
    z = g.splitmix(seed, stream, torch.arange(r * n, (r + 1) * n, dtype=torch.int64))
    return (torch.remainder(g._srl(z, 32), hi - lo + 1) + lo).to(torch.int32).numpy()


def _counter_meta_row_sp12(seed, r, K):
    """row r of tcxgen.sp12_problem_tf32's canonical metadata (pattern (z >> 32) mod 4 per group)"""
    import tcxgen as g
    G = K // 4
    z = g.splitmix(seed, g.STREAM_POS, torch.arange(r * G, (r + 1) * G, dtype=torch.int64))
    pat = torch.remainder(g._srl(z, 32), 4)
    to_pair = torch.tensor([g.PAIRS.index((p & 1, 2 + (p >> 1))) for p in range(4)], dtype=torch.uint8)
    return g.sp24_canonical_meta(to_pair[pat].view(1, G))[0].numpy().view(np.uint32)


def _counter_meta_row(seed, r, K):
    import tcxgen as g
    G = K // 4
    z = g.splitmix(seed, g.STREAM_POS, torch.arange(r * G, (r + 1) * G, dtype=torch.int64))
    pairs = torch.remainder(g._srl(z, 32), 6).to(torch.uint8).view(1, G)
    return g.sp24_canonical_meta(pairs)[0].numpy().view(np.uint32)


# ----------------------------------------------------------------------------------- multi-GPU
def time_broadcast(t, dev, reps=3):
    """the row-sharding layer's one data-path collective: NCCL broadcast of the
    replicated operand B from rank 0, CUDA events on the current stream, max over ranks."""
    import torch.distributed as dist
    from paper_2206_02874_b200.dist import broadcast_replicated, max_over_ranks
    broadcast_replicated(t, src=0)
    torch.cuda.synchronize()
    best = float("inf")
    for _ in range(reps):
        dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        broadcast_replicated(t, src=0)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, max_over_ranks(e0.elapsed_time(e1), dev))
    nbytes = t.numel() * t.element_size()
    return {"bytes": nbytes, "ms": round(best, 4), "algbw_GBs": round(nbytes / (best * 1e-3) / 1e9, 1)}


def multi_gpu_extras(work, args, world, rank, dev, pk):
    """N > 1: the broadcast of the headline config's B (bus rate and an end-to-end figure including
    it), then strong-scaling lines for C4 and C5 — the configs north_star shards — each
    rank its rows, max-over-ranks device time, whole-job value."""
    from paper_2206_02874_b200.dist import max_over_ranks
    out = {"broadcast": time_broadcast(work.B, dev)}
    if work.bound == "tensor":
        gemm_ms = max_over_ranks(time_steps(work, 3, 1, True)[0], dev)
        tot = torch.tensor([work.flops], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(tot)
        out["with_broadcast"] = {"value": round(float(tot.item()) / ((gemm_ms + out["broadcast"]["ms"]) * 1e-3) / 1e12, 2),
                                 "unit": work.unit, "note": "one GEMM step plus the one-time broadcast of B"}
    if args.no_extras:
        return out
    for extra in ("c4", "c5"):
        if extra == args.config:
            continue
        try:
            w2 = Work(extra, rank, world, dev, scaling=args.scaling)
            ms2, l2, _, _ = time_steps(w2, max(5, min(args.steps, 10)), 3, True)
            ms2 = max_over_ranks(ms2, dev)
            tot = torch.tensor([w2.flops], device=dev, dtype=torch.float64)
            torch.distributed.all_reduce(tot)
            out[extra] = {"value": round(float(tot.item()) / (ms2 * 1e-3) / 1e12, 3), "unit": w2.unit,
                          "ms_per_step": round(ms2, 5), "rows_per_rank": int(w2.D.shape[0]),
                          "scaling": "weak" if w2.weak else "strong",
                          "broadcast": time_broadcast(w2.B, dev), "gpu_launches_rank0": l2}
            del w2
            torch.cuda.empty_cache()
        except Exception as e:  # report, never hide
            out[extra] = {"error": f"{type(e).__name__}: {e}"}
    return out


# ----------------------------------------------------------------------------------- main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="tcx", choices=["tcx", "reference"])
    ap.add_argument("--scaling", choices=["weak", "strong"], default="strong",
                    help="N > 1: strong = the config split by rows (default: the SCALE ratio is then "
                         "T1 / (N T_N)); weak = every rank a full config-sized row block")
    ap.add_argument("--sustained-s", type=float, default=4.0, help="seconds of the back-to-back sustained run (0 = skip)")
    ap.add_argument("--config", default="c3", choices=["c3", "c3tf32", "c4", "c5", "c1", "c4sp", "c3sptf32", "c3f16acc"])
    ap.add_argument("--no-extras", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        log("warmup raised to 3 (timing rule)")
        args.warmup = 3

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    cfg_names = {"c3": "dense BF16 GEMM M=N=K=8192 (configs[2])", "c3tf32": "dense TF32 GEMM M=N=K=8192 (configs[2])",
                 "c4": "INT8 GEMM M=N=K=16384 (configs[3])", "c5": "2:4 sparse FP16 GEMM M=65536 N=K=16384 (configs[4])",
                 "c1": "4096 m16n8k16 FP16 tiles (configs[0])",
                 "c4sp": "INT8 2:4 sparse GEMM M=N=K=16384 (NEXT-1 at configs[3]'s shape)",
                 "c3f16acc": "FP16 GEMM with FP16 accumulator M=N=K=8192 (NEXT-2 at configs[2]'s shape)",
                 "c3sptf32": "TF32 1:2 sparse GEMM M=N=K=8192 (NEXT-1 at configs[2]'s shape)"}
    metric = "dense & 2:4-sparse MMA TFLOP/s (INT8 TOPS) per B200, % of tensor-core peak"

    if args.impl == "reference":
        if rank != 0:
            return
        cb = oracle_sample(args.config, seconds=10.0)
        line = {"impl": "reference", "metric": metric, "value": cb["value"], "unit": cb["unit"], "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": None, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None,
                "dtype": {"c3": "bf16", "c3tf32": "tf32", "c4": "s8", "c5": "f16", "c1": "f16", "c4sp": "s8",
                          "c3sptf32": "tf32", "c3f16acc": "f16"}[args.config],
                "data": "synthetic (seeded SplitMix64 / Box-Muller, tcxgen)",
                "config": {"workload": cfg_names[args.config], "shape": list(CFG_SHAPES[args.config]),
                           "parallelism": "single GPU" if args.gpus == 1 else f"row-shard x{args.gpus} (rank 0 times the oracle)",
                           "l2": "inputs+outputs per step > 126 MiB L2 (no reuse across steps)" if args.config != "c1"
                           else "64 rotating batch copies (470 MB) > L2"},
                "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
                "e2e": {"value": cb["value"], "unit": cb["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    dist_on = world > 1
    torch.cuda.set_device(local)                 # before the NCCL group: its barriers use this GPU
    dev = torch.device("cuda", local)
    if dist_on:
        import torch.distributed as dist
        dist.init_process_group("nccl", init_method="env://", device_id=dev)
    import paper_2206_02874_b200 as tcx
    tcx.lib()
    pk = peaks()

    work = Work(args.config, rank, world, dev, scaling=args.scaling)
    torch.cuda.synchronize()
    time.sleep(1.0)                       # start from an idle board, as every "also" config does
    sampler = ClockSampler(local)
    sampler.start()
    ms, launches, t0, t1 = time_steps(work, args.steps, args.warmup, dist_on)
    sampler.stop()
    clocks = sampler.summary(t0, t1)
    if getattr(work, "sm_mhz_eff", None):
        clocks["sm_mhz_in_run"] = round(work.sm_mhz_eff, 1)
    if dist_on:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    # whole-job work: every rank's own FLOPs / bytes summed (uneven shards included), not world x
    # this rank's
    total_flops, total_bytes = work.flops, work.alg_bytes
    if dist_on:
        t = torch.tensor([work.flops, work.alg_bytes], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.SUM)
        total_flops, total_bytes = float(t[0].item()), float(t[1].item())
    value = (total_bytes / (ms * 1e-3) / 1e9) if work.unit == "GB/s" else total_flops / (ms * 1e-3) / 1e12

    e2e = None
    if not args.no_e2e:
        e2e_ms = time_e2e(work, max(3, min(args.steps, 50)), 2)
        if dist_on:
            t = torch.tensor([e2e_ms], device=dev, dtype=torch.float64)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            e2e_ms = float(t.item())
        ev = (total_bytes / (e2e_ms * 1e-3) / 1e9) if work.unit == "GB/s" else total_flops / (e2e_ms * 1e-3) / 1e12
        io = torch.tensor([work.h2d, work.d2h], device=dev, dtype=torch.float64)
        if dist_on:
            torch.distributed.all_reduce(io, op=torch.distributed.ReduceOp.SUM)
        e2e = {"value": round(ev, 3), "unit": work.unit, "h2d_bytes_per_step": int(io[0].item()),
               "d2h_bytes_per_step": int(io[1].item()), "ms_per_step": round(e2e_ms, 4)}
        cb_ms = e2e_copy_bound(work)
        e2e["copy_bound"] = {"ms_per_step": round(cb_ms, 4), "frac": round(cb_ms / e2e_ms, 4),
                             "what": "the step's H2D + D2H alone, both directions at once, no GEMM (this rank)"}

    line = {"metric": metric, "value": round(value, 3), "unit": work.unit, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms, 5), "higher_is_better": True,
            "scaling": "weak" if work.weak else "strong",
            "vs_baseline": None,
            "dtype": {"c3": "bf16", "c3tf32": "tf32", "c4": "s8", "c5": "f16", "c1": "f16", "c4sp": "s8",
                      "c3sptf32": "tf32", "c3f16acc": "f16"}[args.config],
            "data": "synthetic (seeded SplitMix64 / Box-Muller, tcxgen; generated on device)",
            "config": {"workload": cfg_names[args.config], "shape": list(work.shape),
                       "parallelism": (f"row-shard x{world} ({'weak: each rank one config-sized row block, rows seeded per rank' if work.weak else 'strong: the config split by rows'})"
                                       if world > 1 else "single GPU"),
                       "l2": "inputs+outputs per step > 126 MiB L2 (no reuse across steps)" if args.config != "c1"
                       else "64 rotating batch copies (470 MB) > L2"},
            "roofline": None, "clocks": clocks, "gpu_launches": launches,
            "e2e": e2e}
    anchor = same_work = same_work_fn = None
    if rank == 0 and world == 1 and not args.no_extras and args.config in ("c3", "c3tf32", "c4"):
        anchor = library_anchor(work, args.steps)
        if args.config == "c3":
            same_work, same_work_fn = same_work_anchor(work, args.steps)
    line["roofline"] = roofline(work, ms, pk, clocks, anchor)
    if same_work:
        line["roofline"]["denominators"]["same_run_library_same_work"] = {
            "peak": same_work, "frac": round(line["roofline"]["achieved"] / same_work, 4),
            "what": "cuBLAS torch.addmm(C, A, B^T, out_dtype=float32): the same BF16 in / FP32 C in / FP32 D out"}
    if dist_on:
        line["multi_gpu"] = multi_gpu_extras(work, args, world, rank, dev, pk)
    if rank == 0 and world == 1 and not args.no_extras and args.config == "c3":
        line["context"] = {"tcx_best_of_10_steps": best_of(work),
                           "torch_matmul_bf16_tflops_same_run": anchor,
                           "torch_addmm_fp32_out_same_work_tflops": same_work,
                           "note": "cuBLAS via torch.matmul(A, B^T) on the same bf16 A, B, bf16 output (no C), and via "
                                   "torch.addmm(C, A, B^T, out_dtype=float32) doing this step's exact work: context only, "
                                   "not part of the step"}
        also = {}
        power_kinds = {}
        # lightest first: the launch-bound C1 is clock-sensitive and the power-capped 2:4 runs leave
        # the board hot (C1 measured after C5 ran at ~850 MHz)
        for extra in ("c1", "c3tf32", "c3f16acc", "c4", "c3sptf32", "c4sp", "c5"):
            try:
                w2 = Work(extra, 0, 1, dev)
                # every config starts from the same idle board (as tools/ab_burst.py A/Bs do): the
                # previous config's power-capped run and this one's input generation leave the clock
                # in a history-dependent state for tens of ms
                torch.cuda.synchronize()
                time.sleep(1.0)
                sampler.samples = []
                sampler.start()
                ms2, l2, u0, u1 = time_steps(w2, max(5, min(args.steps, 20)), 3, False)
                sampler.stop()
                v2 = w2.metric_value(ms2 * 1e-3)
                ck2 = sampler.summary(u0, u1)
                if getattr(w2, "sm_mhz_eff", None):
                    ck2["sm_mhz_in_run"] = round(w2.sm_mhz_eff, 1)
                anc = library_anchor(w2, 5) if extra in ("c3tf32", "c4") else None
                also[extra] = {"workload": cfg_names[extra], "value": round(v2, 3), "unit": w2.unit,
                               "ms_per_step": round(ms2, 5), "roofline": roofline(w2, ms2, pk, ck2, anc),
                               "gpu_launches": l2, "clocks": ck2}
                if w2.bound == "tensor" and w2.kind in _POWER_KINDS and w2.kind != "bf16":
                    power_kinds[extra] = w2.kind
                if extra == "c1":
                    also[extra]["steady_state"] = tiles_steady_state(w2.tcx, dev)
                if extra == "c5":
                    also[extra]["context"] = {"cusparselt_f16_out_no_c_tflops": cusparselt_anchor(w2),
                                              "note": "cuSPARSELt on the same 2:4 operand, FP16 D, no C (less work): context"}
                del w2
                torch.cuda.empty_cache()
                if not args.no_cpu_baseline:       # the oracle on the host cores, a bounded sample of this config
                    cb2 = oracle_sample(extra, seconds=3.0)
                    also[extra]["cpu_baseline"] = {k: (round(cb2[k], 9) if isinstance(cb2[k], float) else cb2[k])
                                                   for k in ("value", "unit", "cores", "kind", "sample")}
                torch.cuda.empty_cache()
            except Exception as e:  # report, never hide
                also[extra] = {"error": f"{type(e).__name__}: {e}"}
        line["also"] = also
        # after every extra's timed run (each leaves the board at its power cap): the power rooflines,
        # the headline's bf16 one and one per other tensor kind
        for extra, kind in power_kinds.items():
            try:
                apply_power_roofline(also[extra]["roofline"], power_roofline(kind), kind)
            except Exception as e:  # report, never hide
                also[extra]["roofline"]["power_roofline_error"] = f"{type(e).__name__}: {e}"
        try:
            apply_power_roofline(line["roofline"], power_roofline("bf16"), "bf16")
        except Exception as e:  # report, never hide
            line["roofline"]["denominators"]["power_capped_mma_only"] = {"error": f"{type(e).__name__}: {e}"}
        if args.sustained_s > 0:
            # 4 s back to back at the power cap, ours and the cuBLAS anchor, beside the burst value
            # (after the extras: it leaves the board hot, and the launch-bound C1 is clock-sensitive)
            Bt = work.B.t()
            line["sustained"] = {"tcx": sustained(work, args.sustained_s, sampler),
                                 "torch_matmul_bf16": sustained(work, args.sustained_s, sampler,
                                                                fn=lambda: torch.matmul(work.A, Bt)),
                                 "note": "median of 50-step chunks over the run; MEASURED_PEAKS bf16_tflops_sustained "
                                         "is the same method on torch.matmul (BF16 out, no C)"}
            if same_work_fn is not None:
                line["sustained"]["torch_addmm_fp32_out_same_work"] = sustained(work, args.sustained_s, sampler,
                                                                                fn=same_work_fn)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cb = oracle_sample(args.config, seconds=10.0)
        line["cpu_baseline"] = {k: (round(cb[k], 6) if isinstance(cb[k], float) else cb[k])
                                for k in ("value", "unit", "cores", "kind", "sample")}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist_on:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
