mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
python - <<'PY' > gpurun_out/exp17_tc05.txt 2>&1
import paper_2206_02874_b200 as tcx
for nacc in (1, 2):
    for cg, m in ((1, 128), (2, 256)):
        for ilp in (32, 128, 256):
            r = tcx.probe("tc05", ab=tcx.BF16, cd=tcx.F32, m=m, n=256, k=16, cta_group=cg, ilp=ilp, warps=nacc, iters=64, repeats=3, num_sms=148)
            print("nacc%d bf16 m%d n256 cg%d ilp%d" % (nacc, m, cg, ilp), round(r["fma_per_clk_per_sm"], 1), round(r["latency_cycles"], 1), round(r["sm_mhz"], 0))
for nacc in (1, 2):
    r = tcx.probe("tc05_sp", ab=tcx.F16, cd=tcx.F32, m=256, n=256, k=32, cta_group=2, ilp=256, warps=nacc, iters=64, repeats=3, num_sms=148)
    print("nacc%d sp f16 m256 n256 cg2 ilp256" % nacc, round(r["fma_per_clk_per_sm"], 1), round(r["latency_cycles"], 1))
PY
timeout 900 python -m pytest tests/test_gpu_data_movement.py tests/test_gpu_probe.py tests/test_gpu_tiles.py -q -x > gpurun_out/t_dm2.log 2>&1; echo dm=$?
