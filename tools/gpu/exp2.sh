mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
for i in 0 1 2 3; do TCX_TILES_IMPL=$i timeout 300 python tools/exp_tiles.py f16 >> gpurun_out/exp2_tiles.jsonl 2>>gpurun_out/exp2_tiles.err; done
TCX_TILES_IMPL=1 timeout 600 python -m pytest tests/test_gpu_tiles.py -q -x > gpurun_out/exp2_tiles_tests.log 2>&1; echo tiles_tests=$?
timeout 300 python tools/exp_gemm.py c5 2 g8h0c2 g8h8c2 g12h8c2 g8h1c2 > gpurun_out/exp2_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg \
  --clock-control none -k regex:gemm_sp24 --csv --log-file gpurun_out/exp2_c5_ncu.csv python tools/exp_gemm.py c5 2 g8h0c2 g8h8c2 g12h8c2 g8h1c2 > gpurun_out/exp2_ncu.log 2>&1
echo ncu=$?
