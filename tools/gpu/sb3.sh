mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
AB=$PWD/paper_2206_02874_b200/libtcx_ab.so
ABD=$PWD/paper_2206_02874_b200/libtcx_abdbg.so
DBG=$PWD/paper_2206_02874_b200/libtcx_debug.so
timeout 900 python -m pytest tests/test_gpu_sparse.py tests/test_gpu_sparse_i8.py tests/test_gpu_sparse_tf32.py tests/test_gpu_fuzz.py -q -x > gpurun_out/t_sb3.log 2>&1; echo t=$?
TCX_LIB_PATH=$ABD timeout 300 python tools/trace_gemm.py c5 8 wide | sed 's/^{/{"lib": "old", /' >> gpurun_out/sb3_trace.jsonl 2>&1
TCX_LIB_PATH=$DBG timeout 300 python tools/trace_gemm.py c5 8 wide | sed 's/^{/{"lib": "new", /' >> gpurun_out/sb3_trace.jsonl 2>&1
for i in 1 2 3 4; do
  TCX_LIB_PATH=$AB timeout 600 python tools/exp_gemm.py c5 30 g8c2w | sed 's/"variant": "/"variant": "old_/' >> gpurun_out/sb3_time.jsonl 2>&1
  timeout 600 python tools/exp_gemm.py c5 30 g8c2w | sed 's/"variant": "/"variant": "new_/' >> gpurun_out/sb3_time.jsonl 2>&1
done; echo e=$?
