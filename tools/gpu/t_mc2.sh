mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 600 python -m pytest tests/test_gpu_gemm.py -q -x -k "multicast or pairs" > gpurun_out/t_mc.log 2>&1; echo t=$?
timeout 300 python tools/exp_gemm.py c3 50 g8c2 g8c2p12 g8c2p21 g8c2p22 g4c2p12 g16c2p12 g8c2 g8c2p12 > gpurun_out/exp_mc_c3.log 2>&1; echo e=$?
timeout 300 python tools/exp_gemm.py c4 20 g8c2 g8c2p12 g8c2p21 g8c2p22 g8c2 g8c2p12 > gpurun_out/exp_mc_c4.log 2>&1; echo e4=$?
M=gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_bytes.sum,launch__grid_size,sm__throughput.avg.pct_of_peak_sustained_elapsed
for v in narrow mc12 mc21 mc22; do
  TCX_DEBUG_LAUNCH=1 timeout 300 python tools/exp_one.py $v 3 > gpurun_out/exp23_$v.log 2>&1 && \
  timeout 300 ncu --metrics $M --clock-control none -k regex:gemm_dense -s 2 -c 1 --csv --log-file gpurun_out/exp23_ncu_$v.csv python tools/exp_one.py $v 3 > /dev/null 2>&1; echo $v=$?
done
