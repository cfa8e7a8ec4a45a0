mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 600 python -m pytest tests/test_gpu_debug_build.py -q -x > gpurun_out/t_debug.log 2>&1; echo t=$?
DBG=$PWD/paper_2206_02874_b200/libtcx_debug.so
for cfg in c3 c3tf32 c4; do
  for g in 8 4 16; do
    TCX_LIB_PATH=$DBG timeout 300 python tools/trace_gemm.py $cfg $g >> gpurun_out/trace.jsonl 2>&1
  done
done; echo e=$?
