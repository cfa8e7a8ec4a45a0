mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 300 python -m pytest tests/test_gpu_sparse.py -q -x -k "half_k" > gpurun_out/t_hk.log 2>&1; echo t=$?
cat > /tmp/hk.py <<'PY'
import sys, json, time
sys.path.insert(0, '.')
import torch, bench
torch.cuda.set_device(0)
w = bench.Work("c5", 0, 1, torch.device("cuda", 0))
tcx = w.tcx
var = {"base": dict(), "hk": dict(stage_k=64), "mw": dict(tile_m=512), "mwhk": dict(tile_m=512, stage_k=64)}
ref = None
for rnd in range(3):
    for name, kw in var.items():
        step = lambda: tcx.gemm_sp24(w.vals, w.meta_hw, w.B, w.C, w.D, **kw)
        for _ in range(3): step()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10): step()
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        same = None
        if ref is None: ref = w.D.clone()
        else: same = bool(torch.equal(ref.view(torch.int32), w.D.view(torch.int32)))
        print(json.dumps({"round": rnd, "variant": name, "ms": round(ms, 4), "tflops": round(w.flops / ms / 1e9, 1), "bit_identical": same}), flush=True)
PY
timeout 900 python /tmp/hk.py > gpurun_out/hk_time.jsonl 2>&1; echo e=$?
M=gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read.sum
cat > /tmp/hk1.py <<'PY'
import sys; sys.path.insert(0, '.')
import torch, bench
torch.cuda.set_device(0)
w = bench.Work("c5", 0, 1, torch.device("cuda", 0))
kw = {"base": {}, "hk": {"stage_k": 64}, "mw": {"tile_m": 512}, "mwhk": {"tile_m": 512, "stage_k": 64}}[sys.argv[1]]
for _ in range(3): w.tcx.gemm_sp24(w.vals, w.meta_hw, w.B, w.C, w.D, **kw)
torch.cuda.synchronize()
PY
for v in base hk mw mwhk; do
  timeout 300 ncu --metrics $M --clock-control none -k regex:gemm_sp24 -s 2 -c 1 --csv --log-file gpurun_out/hk_ncu_$v.csv python /tmp/hk1.py $v > /dev/null 2>&1; echo $v=$?
done
