mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
M=gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read.sum
for cfg in c3 c4; do
for v in g8c2 g12c2 g16c2 g24c2 g32c2; do
  timeout 300 ncu --metrics $M --clock-control none -k regex:gemm_dense -s 3 -c 1 --csv --log-file gpurun_out/r2_${cfg}_$v.csv python tools/exp_gemm.py $cfg 1 $v > /dev/null 2>&1; echo $cfg$v=$?
done; done
for v in g8c2 g16c2 g4c2; do
  timeout 300 ncu --metrics $M --clock-control none -k regex:gemm_sp24 -s 3 -c 1 --csv --log-file gpurun_out/r2_c5_$v.csv python tools/exp_gemm.py c5 1 $v > /dev/null 2>&1; echo c5$v=$?
done
for i in 1 2; do timeout 300 python tools/exp_gemm.py c3 100 g8c2 g16c2 g24c2 >> gpurun_out/r2_time.jsonl 2>&1; done
for i in 1 2; do timeout 300 python tools/exp_gemm.py c4 30 g8c2 g16c2 g24c2 >> gpurun_out/r2_time.jsonl 2>&1; done
