mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
AB=$PWD/paper_2206_02874_b200/libtcx_ab.so
timeout 600 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_sparse.py -q -x -k "raster or persistent or small_whole or multicast" > gpurun_out/t_snake.log 2>&1; echo t=$?
M=gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum
for cfg in c3 c3tf32 c4 c5; do
  K=regex:gemm_dense; [ $cfg = c5 ] && K=regex:gemm_sp24
  TCX_LIB_PATH=$AB timeout 300 ncu --metrics $M --clock-control none -k $K -s 1 -c 1 --csv --log-file gpurun_out/sn_base_$cfg.csv python tools/prof_kernels.py $cfg 2 > /dev/null 2>&1
  timeout 300 ncu --metrics $M --clock-control none -k $K -s 1 -c 1 --csv --log-file gpurun_out/sn_snake_$cfg.csv python tools/prof_kernels.py $cfg 2 > /dev/null 2>&1; echo $cfg=$?
done
for i in 1 2 3; do
  TCX_LIB_PATH=$AB timeout 300 python tools/exp_gemm.py c3 50 g8c2 | sed 's/g8c2/base/' >> gpurun_out/sn_time.jsonl
  timeout 300 python tools/exp_gemm.py c3 50 g8c2 | sed 's/g8c2/snake/' >> gpurun_out/sn_time.jsonl
done
for i in 1 2; do
  TCX_LIB_PATH=$AB timeout 300 python tools/exp_gemm.py c4 20 g8c2 | sed 's/g8c2/base/' >> gpurun_out/sn_time.jsonl
  timeout 300 python tools/exp_gemm.py c4 20 g8c2 | sed 's/g8c2/snake/' >> gpurun_out/sn_time.jsonl
done; echo e=$?
