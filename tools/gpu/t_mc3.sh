mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 600 python -m pytest tests/test_gpu_sparse.py tests/test_gpu_sparse_i8.py tests/test_gpu_sparse_tf32.py -q -x -k "multicast" > gpurun_out/t_mc3.log 2>&1; echo t=$?
timeout 600 python tools/exp_gemm.py c5 10 g8c2 g8c2p21 g8c2p12 g8c2p22 g8c2 g8c2p21 g8c2p22 > gpurun_out/exp_mc_c5.log 2>&1; echo e=$?
M=gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read.sum,launch__grid_size,sm__throughput.avg.pct_of_peak_sustained_elapsed
for v in g8c2 g8c2p21 g8c2p22; do
  timeout 300 ncu --metrics $M --clock-control none -k regex:gemm_sp24 -s 3 -c 1 --csv --log-file gpurun_out/exp24_ncu_$v.csv python tools/exp_gemm.py c5 1 $v > /dev/null 2>&1; echo $v=$?
done
