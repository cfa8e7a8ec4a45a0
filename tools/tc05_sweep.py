#!/usr/bin/env python
"""tcgen05 half of the paper's microbenchmark method on B200, through tcx_probe.

For each tcgen05 kind / shape (dense kind::{f16,tf32,i8}, sparse .sp):
  * completion latency: SYNC mode, ILP 1, one issuer on one SM; the commit round trip alone (COMMIT
    mode) and their difference (the MMA's own latency);
  * the (issuers per SM, ILP) grid in SYNC mode (commit + wait per iteration, the paper's sync),
    issuers in {1, 2} (2 CTAs per SM, 256 TMEM columns each), ILP in {1, 2, 4, 8, 16, 32};
  * STREAM mode (no wait until the end): one dependent chain (n_acc = 1) and n_acc = 2, one SM and
    all 148 SMs — the pipe's own rate;
  * power ceiling (--power): STREAM on all SMs for ~2 s per kind with NVML sampling, giving the
    sustained clock / power of pure tensor-core work (no HBM, no L2 traffic).
Writes JSON lines to argv[1] (and a table to stdout)."""
import json
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2206_02874_b200 as tcx  # noqa: E402

F16, BF16, TF32, F32, S8, S32 = tcx.F16, tcx.BF16, tcx.TF32, tcx.F32, tcx.S8, tcx.S32
ES = {F16: 2, BF16: 2, TF32: 4, S8: 1}
NAME = {F16: "f16", BF16: "bf16", TF32: "tf32", S8: "i8"}
NOMINAL = {F16: 4096, BF16: 4096, TF32: 2048, S8: 8192}


def shapes():
    for sp in (False, True):
        for ab in (BF16, TF32, S8) + ((F16,) if sp else ()):
            n = 240 if sp else 256
            for cg, m in ((1, 128), (2, 256)):
                yield sp, ab, cg, m, n


def run(sp, ab, cg, m, n, **kw):
    k = (64 if sp else 32) // ES[ab]
    cd = S32 if ab == S8 else F32
    return tcx.probe("tc05_sp" if sp else "tc05", ab, cd, m, n, k, cta_group=cg, **kw)


class Sampler:
    def __init__(self):
        import pynvml
        pynvml.nvmlInit()
        self.nv = pynvml
        self.h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
        self.s = []
        self.stop_ev = threading.Event()

    def _run(self):
        while not self.stop_ev.is_set():
            try:
                self.s.append((self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM),
                               self.nv.nvmlDeviceGetPowerUsage(self.h) / 1000.0,
                               int(self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h))))
            except Exception:
                pass
            time.sleep(0.02)

    def __enter__(self):
        self.t = threading.Thread(target=self._run, daemon=True)
        self.t.start()
        return self

    def __exit__(self, *a):
        self.stop_ev.set()
        self.t.join()

    def summary(self):
        s = self.s[len(self.s) // 4:] or self.s       # drop the ramp
        mhz = sorted(x[0] for x in s)
        pw = sorted(x[1] for x in s)
        return {"sm_mhz_median": mhz[len(mhz) // 2] if mhz else None, "power_w_median": pw[len(pw) // 2] if pw else None,
                "power_cap_samples": sum(1 for x in s if x[2] & 4), "samples": len(s)}


def main():
    out = open(sys.argv[1], "w") if len(sys.argv) > 1 else None
    power = "--power" in sys.argv
    quick = "--quick" in sys.argv

    def emit(d):
        print(json.dumps(d), flush=True)
        if out:
            out.write(json.dumps(d) + "\n")
            out.flush()

    for sp, ab, cg, m, n in shapes():
        lab = f"{'sp ' if sp else ''}{NAME[ab]} cg{cg} m{m}n{n}"
        if not power:
            comp = run(sp, ab, cg, m, n, mode="sync", ilp=1, iters=1024, repeats=5)
            com = run(sp, ab, cg, m, n, mode="commit", ilp=1, iters=1024, repeats=5)
            row = {"instr": lab, "completion_latency": round(comp["latency_cycles"], 1),
                   "commit_round_trip": round(com["latency_cycles"], 1),
                   "mma_latency": round(comp["latency_cycles"] - com["latency_cycles"], 1),
                   "sm_mhz": round(comp["sm_mhz"])}
            grid = []
            for issuers in (1, 2):
                for ilp in ((1, 4, 16) if quick else (1, 2, 4, 8, 16, 32)):
                    try:
                        r = run(sp, ab, cg, m, n, mode="sync", ilp=ilp, iters=256, repeats=3, issuers=issuers,
                                num_sms=1)
                    except tcx.TcxError as e:
                        grid.append({"issuers": issuers, "ilp": ilp, "error": str(e)[:80]})
                        continue
                    grid.append({"issuers": issuers, "ilp": ilp, "n_acc": r["n_acc"],
                                 "cyc_per_iter": round(r["latency_cycles"], 1),
                                 "fma_clk_sm": round(r["fma_per_clk_per_sm"], 1)})
            row["sync_grid"] = grid
            st = []
            for nsm in (1, 148):
                for n_acc in (1, 2):
                    try:
                        r = run(sp, ab, cg, m, n, mode="stream", ilp=16, iters=512, repeats=3, n_acc=n_acc,
                                num_sms=nsm)
                    except tcx.TcxError as e:
                        st.append({"num_sms": nsm, "n_acc": n_acc, "error": str(e)[:80]})
                        continue
                    st.append({"num_sms": nsm, "n_acc": n_acc, "fma_clk_sm": round(r["fma_per_clk_per_sm"], 1),
                               "frac_nominal": round(r["fma_per_clk_per_sm"] / NOMINAL[ab], 4),
                               "sm_mhz": round(r["sm_mhz"])})
            row["stream"] = st
            emit(row)
        elif cg == 2:
            # power ceiling: pure MMA on every SM for ~2 s, operands N(0,1) (int8: uniform) in a 4-stage
            # smem ring read at every k-offset (STREAM_ROT), as a GEMM mainloop reads them
            import tcxgen
            es = ES[ab]
            fmt = {F16: "f16", BF16: "bf16", TF32: "tf32"}.get(ab)
            ka, kb = 32 // es, (64 if sp else 32) // es
            if fmt:
                a_op = tcxgen.normal_matrix((m, ka), fmt, 1, 1, "cuda", redraw_zero=sp)
                b_op = tcxgen.normal_matrix((n, kb), fmt, 1, 2, "cuda")
            else:
                a_op = tcxgen.int8_matrix((m, ka), 1, 1, "cuda")
                b_op = tcxgen.int8_matrix((n, kb), 1, 2, "cuda")
            prun = (lambda sp_, ab_, cg_, m_, n_, **kw:
                   tcx.probe("tc05_sp" if sp_ else "tc05", ab_, S32 if ab_ == S8 else F32, m_, n_, (64 if sp_ else 32) // ES[ab_],
                             cta_group=cg_, a_op=a_op, b_op=b_op, **{**kw, "mode": "stream_rot"}))
            r = prun(sp, ab, cg, m, n, mode="stream", ilp=16, iters=512, repeats=1, n_acc=1, num_sms=148)
            per_call_s = r["ns_per_iter"] * 512 * 1e-9
            iters = int(min(2_000_000, max(512, 0.5 / max(per_call_s / 512, 1e-9))))
            with Sampler() as smp:
                t0 = time.time()
                rs = []
                while time.time() - t0 < 2.0:
                    rs.append(prun(sp, ab, cg, m, n, mode="stream", ilp=16, iters=iters, repeats=1, n_acc=1,
                                   num_sms=148))
            fma = sorted(x["fma_per_clk_per_sm"] for x in rs)[len(rs) // 2]
            mhz = sorted(x["sm_mhz"] for x in rs)[len(rs) // 2]
            emit({"power_ceiling": lab, "fma_clk_sm": round(fma, 1), "probe_mhz": round(mhz),
                  "tflops_dense_equiv": round(2 * fma * 148 * mhz * 1e6 / 1e12, 1), "calls": len(rs),
                  **smp.summary()})


if __name__ == "__main__":
    main()
