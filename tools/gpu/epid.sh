# sparse epilogue with direct D stores (new) vs TMA-store epilogue (libtcx_ab.so / libtcx_debug_ab.so)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
AB=$PWD/paper_2206_02874_b200/libtcx_ab.so
DBG=$PWD/paper_2206_02874_b200/libtcx_debug.so
DBGAB=$PWD/paper_2206_02874_b200/libtcx_debug_ab.so
timeout 900 python -m pytest tests/test_gpu_sparse.py tests/test_gpu_sparse_i8.py tests/test_gpu_sparse_tf32.py tests/test_gpu_gemm_model.py tests/test_gpu_debug_build.py tests/test_gpu_fuzz.py tests/test_gpu_streams_graphs.py -q -x > gpurun_out/t_epid.log 2>&1; echo t=$?
tail -3 gpurun_out/t_epid.log
TCX_LIB_PATH=$DBGAB timeout 300 python tools/trace_gemm.py c5 8 wide | sed 's/^{/{"lib": "old",/' >> gpurun_out/trace_epid.jsonl 2>&1
TCX_LIB_PATH=$DBG timeout 300 python tools/trace_gemm.py c5 8 wide | sed 's/^{/{"lib": "new",/' >> gpurun_out/trace_epid.jsonl 2>&1
TCX_LIB_PATH=$DBGAB timeout 300 python tools/trace_gemm.py c5 8 | sed 's/^{/{"lib": "old",/' >> gpurun_out/trace_epid.jsonl 2>&1
TCX_LIB_PATH=$DBG timeout 300 python tools/trace_gemm.py c5 8 | sed 's/^{/{"lib": "new",/' >> gpurun_out/trace_epid.jsonl 2>&1
for i in 1 2 3; do
  TCX_LIB_PATH=$AB timeout 600 python tools/exp_gemm.py c5 20 g8c2w g8c2 | sed 's/"variant": "/"variant": "old_/' >> gpurun_out/epid_time.jsonl 2>&1
  timeout 600 python tools/exp_gemm.py c5 20 g8c2w g8c2 | sed 's/"variant": "/"variant": "new_/' >> gpurun_out/epid_time.jsonl 2>&1
done
for cfg in c4sp c3sptf32; do for i in 1 2; do
  TCX_LIB_PATH=$AB timeout 600 python tools/exp_gemm.py $cfg 30 g8c2 | sed 's/"variant": "/"variant": "old_/' >> gpurun_out/epid_time.jsonl 2>&1
  timeout 600 python tools/exp_gemm.py $cfg 30 g8c2 | sed 's/"variant": "/"variant": "new_/' >> gpurun_out/epid_time.jsonl 2>&1
done; done; echo e=$?
