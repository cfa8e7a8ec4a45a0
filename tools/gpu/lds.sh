# epilogue smem via LDS/STS.128 (new) vs generic LD/ST.E.128 (libtcx_ab.so)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
AB=$PWD/paper_2206_02874_b200/libtcx_ab.so
DBG=$PWD/paper_2206_02874_b200/libtcx_debug.so
DBGAB=$PWD/paper_2206_02874_b200/libtcx_debug_ab.so
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_sparse.py tests/test_gpu_sparse_i8.py tests/test_gpu_sparse_tf32.py tests/test_gpu_gemm_model.py tests/test_gpu_debug_build.py tests/test_gpu_fuzz.py tests/test_gpu_gemm_f16acc.py tests/test_gpu_streams_graphs.py -q -x > gpurun_out/t_lds.log 2>&1; echo t=$?
tail -2 gpurun_out/t_lds.log
for a in "c3 wide" "c3 wide noc" "c3"; do
  TCX_LIB_PATH=$DBG timeout 300 python tools/chunk_trace.py $a >> gpurun_out/chunk_trace3.jsonl 2>&1
done
for a in "c5 8 wide" "c3 8 wide" "c3 8 x"; do
  TCX_LIB_PATH=$DBGAB timeout 300 python tools/trace_gemm.py $a | sed 's/^{/{"lib": "old",/' >> gpurun_out/trace_lds.jsonl 2>&1
  TCX_LIB_PATH=$DBG timeout 300 python tools/trace_gemm.py $a | sed 's/^{/{"lib": "new",/' >> gpurun_out/trace_lds.jsonl 2>&1
done
for i in 1 2; do
  for cfg in c3 c4 c3tf32 c3f16acc; do
    TCX_LIB_PATH=$AB timeout 600 python tools/exp_gemm.py $cfg 30 g8c2 g8c2w | sed 's/"variant": "/"variant": "old_/' >> gpurun_out/lds_time.jsonl 2>&1
    timeout 600 python tools/exp_gemm.py $cfg 30 g8c2 g8c2w | sed 's/"variant": "/"variant": "new_/' >> gpurun_out/lds_time.jsonl 2>&1
  done
  for cfg in c4sp c3sptf32; do
    TCX_LIB_PATH=$AB timeout 600 python tools/exp_gemm.py $cfg 30 g8c2 | sed 's/"variant": "/"variant": "old_/' >> gpurun_out/lds_time.jsonl 2>&1
    timeout 600 python tools/exp_gemm.py $cfg 30 g8c2 | sed 's/"variant": "/"variant": "new_/' >> gpurun_out/lds_time.jsonl 2>&1
  done
  TCX_LIB_PATH=$AB timeout 600 python tools/exp_gemm.py c5 15 g8c2w g8c2 | sed 's/"variant": "/"variant": "old_/' >> gpurun_out/lds_time.jsonl 2>&1
  timeout 600 python tools/exp_gemm.py c5 15 g8c2w g8c2 | sed 's/"variant": "/"variant": "new_/' >> gpurun_out/lds_time.jsonl 2>&1
done; echo e=$?
