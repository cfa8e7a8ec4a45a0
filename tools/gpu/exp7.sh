mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
M=gpu__time_duration.sum,sm__cycles_elapsed.avg,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_write.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed,lts__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__throughput.avg.pct_of_peak_sustained_elapsed
for v in cublas narrow_noC wide_noC narrow wide; do
  python tools/exp_one.py $v 3 > /dev/null 2>&1 && \
  timeout 300 ncu --metrics $M --clock-control none -k regex:"gemm|nvjet" -s 2 -c 1 --csv --log-file gpurun_out/exp7_$v.csv python tools/exp_one.py $v 3 > /dev/null 2>&1
  echo $v=$?
done
