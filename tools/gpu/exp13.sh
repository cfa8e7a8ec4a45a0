mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
for pf in 1 0; do
TCX_EPI_PREFETCH=$pf timeout 400 python tools/exp_gemm.py c5 30 g8c2 g8c2 > gpurun_out/exp13_c5_pf$pf.jsonl 2>&1
TCX_EPI_PREFETCH=$pf timeout 400 python tools/exp_gemm.py c3 200 g8c2 g8c2 > gpurun_out/exp13_c3_pf$pf.jsonl 2>&1
TCX_EPI_PREFETCH=$pf timeout 400 python tools/exp_gemm.py c4 60 g8c2 g8c2 > gpurun_out/exp13_c4_pf$pf.jsonl 2>&1
done
