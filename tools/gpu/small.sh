mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
DBG=$PWD/paper_2206_02874_b200/libtcx_debug.so
for s in "256 64" "512 512" "1024 1024"; do
  set -- $s
  timeout 120 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:gemm_dense -s 5 -c 1 --csv --log-file gpurun_out/small_ncu_$1.csv python tools/small_gemm.py $1 $2 > /dev/null 2>&1
  TCX_LIB_PATH=$DBG timeout 120 python tools/small_gemm.py $1 $2 trace >> gpurun_out/small_trace.txt 2>&1
done; echo ok
