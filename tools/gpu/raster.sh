mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 600 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_sparse.py -q -x -k "raster" > gpurun_out/t_raster.log 2>&1; echo t=$?
M=gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum
for v in g8c2 g4c2 g16c2 g2c2 g-8c2 g-4c2 g-16c2; do
  timeout 300 ncu --metrics $M --clock-control none -k regex:gemm_dense -s 3 -c 1 --csv --log-file gpurun_out/ras_c4_$v.csv python tools/exp_gemm.py c4 1 $v > /dev/null 2>&1; echo c4$v=$?
done
for v in g8c2 g-8c2 g-4c2 g-16c2 g-32c2; do
  timeout 300 ncu --metrics $M --clock-control none -k regex:gemm_sp24 -s 3 -c 1 --csv --log-file gpurun_out/ras_c5_$v.csv python tools/exp_gemm.py c5 1 $v > /dev/null 2>&1; echo c5$v=$?
done
for v in g8c2 g-8c2 g4c2 g-4c2; do
  timeout 300 ncu --metrics $M --clock-control none -k regex:gemm_dense -s 3 -c 1 --csv --log-file gpurun_out/ras_c3_$v.csv python tools/exp_gemm.py c3 1 $v > /dev/null 2>&1; echo c3$v=$?
done
timeout 600 python tools/exp_gemm.py c5 10 g8c2 g-8c2 g-16c2 g8c2 g-8c2 g-16c2 > gpurun_out/ras_c5_time.jsonl 2>&1
timeout 600 python tools/exp_gemm.py c4 20 g8c2 g-8c2 g16c2 g8c2 g-8c2 g16c2 > gpurun_out/ras_c4_time.jsonl 2>&1; echo e=$?
