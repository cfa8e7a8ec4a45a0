# dense epilogue: wide tile: 3 stages + 4 epilogue buffers (C 3 ahead) (new) vs 4 stages + 2 buffers (libtcx_ab.so)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
AB=$PWD/paper_2206_02874_b200/libtcx_ab.so
DBG=$PWD/paper_2206_02874_b200/libtcx_debug.so
DBGAB=$PWD/paper_2206_02874_b200/libtcx_debug_ab.so
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_gemm_model.py tests/test_gpu_debug_build.py tests/test_gpu_fuzz.py tests/test_gpu_gemm_f16acc.py tests/test_gpu_streams_graphs.py tests/test_gpu_dist.py tests/test_gpu_chain.py -q -x > gpurun_out/t_nbe.log 2>&1; echo t=$?
tail -2 gpurun_out/t_nbe.log
for a in "c3 wide" "c3"; do
  TCX_LIB_PATH=$DBG timeout 300 python tools/chunk_trace.py $a >> gpurun_out/chunk_trace5.jsonl 2>&1
done
for a in "c3 8 wide" "c3 8 x" "c4 8 wide"; do
  TCX_LIB_PATH=$DBGAB timeout 300 python tools/trace_gemm.py $a | sed 's/^{/{"lib": "old",/' >> gpurun_out/trace_nbe.jsonl 2>&1
  TCX_LIB_PATH=$DBG timeout 300 python tools/trace_gemm.py $a | sed 's/^{/{"lib": "new",/' >> gpurun_out/trace_nbe.jsonl 2>&1
done
for i in 1 2 3; do
  for cfg in c3 c4 c3tf32; do
    TCX_LIB_PATH=$AB timeout 600 python tools/exp_gemm.py $cfg 30 g8c2 g8c2w | sed 's/"variant": "/"variant": "old_/' >> gpurun_out/nbe_time.jsonl 2>&1
    timeout 600 python tools/exp_gemm.py $cfg 30 g8c2 g8c2w | sed 's/"variant": "/"variant": "new_/' >> gpurun_out/nbe_time.jsonl 2>&1
  done
done; echo e=$?
