mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 900 python -m pytest tests/test_gpu_tiles.py tests/test_gpu_gemm.py tests/test_gpu_sparse.py -q -x > gpurun_out/exp4_tests.log 2>&1; echo tests=$?
timeout 400 python tools/exp_gemm.py c5 40 g8p0c2 g8p2c2 g8p4c2 g8p8c2 g8p16c2 g16p8c2 g8p0c2 > gpurun_out/exp4_c5.jsonl 2>&1
timeout 300 python tools/exp_gemm.py c3 200 g8p0c2 g8p2c2 g8p4c2 g8p8c2 g16p4c2 g8p0c2 > gpurun_out/exp4_c3.jsonl 2>&1
timeout 300 python tools/exp_gemm.py c4 60 g8p0c2 g8p2c2 g8p4c2 g8p8c2 g8p0c2 > gpurun_out/exp4_c4.jsonl 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg \
  --clock-control none -k regex:gemm_sp24 -s 3 -c 1 --csv --log-file gpurun_out/exp4_ncu_p0.csv python tools/exp_gemm.py c5 1 g8p0c2 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg \
  --clock-control none -k regex:gemm_sp24 -s 3 -c 1 --csv --log-file gpurun_out/exp4_ncu_p8.csv python tools/exp_gemm.py c5 1 g8p8c2 > /dev/null 2>&1
echo done
