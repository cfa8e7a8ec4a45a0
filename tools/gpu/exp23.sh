mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
M=gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_bytes.sum,launch__grid_size,launch__cluster_dim_x,launch__occupancy_cluster_pct,sm__throughput.avg.pct_of_peak_sustained_elapsed
for v in narrow mc12 mc21 mc22; do
  TCX_DEBUG_LAUNCH=1 timeout 300 python tools/exp_one.py $v 3 > gpurun_out/exp23_$v.log 2>&1 && \
  timeout 300 ncu --metrics $M --clock-control none -k regex:gemm_dense -s 2 -c 1 --csv --log-file gpurun_out/exp23_ncu_$v.csv python tools/exp_one.py $v 3 > /dev/null 2>&1; echo $v=$?
done
