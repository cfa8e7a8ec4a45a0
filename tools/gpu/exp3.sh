mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
V="g8h0c2 g8h5c2 g4h5c2 g8h20c2 g12h20c2 g8h4c2 g8h13c2 g16h20c2"
timeout 300 python tools/exp_gemm.py c5 2 $V > gpurun_out/exp3_plain.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg \
  --clock-control none -k regex:gemm_sp24 --csv --log-file gpurun_out/exp3_c5_ncu.csv python tools/exp_gemm.py c5 1 $V > gpurun_out/exp3_ncu.log 2>&1
echo ncu=$?
timeout 300 python tools/exp_gemm.py c5 40 $V g8h0c2 > gpurun_out/exp3_timed.log 2>&1
