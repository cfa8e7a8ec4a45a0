mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
for r in 1 2; do
timeout 300 python tools/exp_gemm.py c5 20 g8c2 > gpurun_out/exp15_normal_$r.jsonl 2>&1
TCX_SP_CP_SKIP=1 timeout 300 python tools/exp_gemm.py c5 20 g8c2 > gpurun_out/exp15_skip_$r.jsonl 2>&1
done
python tools/prof_kernels.py c5s 2 > /dev/null 2>&1 && TCX_SP_CP_SKIP=1 timeout 300 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:gemm_sp24 -s 1 -c 1 --csv --log-file gpurun_out/exp15_ncu_skip.csv python tools/prof_kernels.py c5s 2 > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:gemm_sp24 -s 1 -c 1 --csv --log-file gpurun_out/exp15_ncu_normal.csv python tools/prof_kernels.py c5s 2 > /dev/null 2>&1
