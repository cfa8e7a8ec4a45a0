mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 900 python tools/exp_gemm.py c5 20 g8c2 g8c2w g8c2 g8c2w g8c2 g8c2w > gpurun_out/exp20_c5.jsonl 2>&1; echo e=$?
timeout 300 python tools/exp_anchor.py 50 > gpurun_out/exp20_anchor.jsonl 2>&1; echo a=$?
timeout 600 python tools/exp_gemm.py c5 1 g8c2w > /dev/null 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum --clock-control none -k regex:gemm_sp24 -s 3 -c 1 --csv --log-file gpurun_out/exp20_ncu.csv python tools/exp_gemm.py c5 1 g8c2w > /dev/null 2>&1; echo n=$?
