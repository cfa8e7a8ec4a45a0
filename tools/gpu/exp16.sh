mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
for w in 8 4 16 32; do TCX_TILES_WARPS=$w timeout 300 python tools/exp_tiles.py f16 >> gpurun_out/exp16_tiles.jsonl 2>>gpurun_out/exp16.err; done
python - <<'PY' > gpurun_out/exp16_tc05.txt 2>&1
import paper_2206_02874_b200 as tcx
for cg, m in ((1, 128), (2, 256)):
    for ilp in (1, 8, 32, 64, 128, 256):
        r = tcx.probe("tc05", ab=tcx.BF16, cd=tcx.F32, m=m, n=256, k=16, cta_group=cg, ilp=ilp, iters=64, repeats=3, num_sms=148 if cg == 2 else 148)
        print("bf16 m%d n256 cg%d ilp%d" % (m, cg, ilp), round(r["fma_per_clk_per_sm"], 1), round(r["latency_cycles"], 1), round(r["sm_mhz"], 0))
for ilp in (32, 128, 256):
    r = tcx.probe("tc05_sp", ab=tcx.F16, cd=tcx.F32, m=256, n=256, k=32, cta_group=2, ilp=ilp, iters=64, repeats=3, num_sms=148)
    print("sp f16 m256 n256 cg2 ilp%d" % ilp, round(r["fma_per_clk_per_sm"], 1), round(r["latency_cycles"], 1), round(r["sm_mhz"], 0))
PY
echo done
