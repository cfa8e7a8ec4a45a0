mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_gemm_f16acc.py tests/test_gpu_sparse.py tests/test_gpu_sparse_i8.py tests/test_gpu_sparse_tf32.py tests/test_gpu_gemm_model.py tests/test_gpu_fuzz.py tests/test_gpu_streams_graphs.py -q -x > gpurun_out/t_origin.log 2>&1; echo t=$?
DBG=$PWD/paper_2206_02874_b200/libtcx_debug.so
TCX_LIB_PATH=$DBG timeout 300 python tools/trace_gemm.py c5 8 > gpurun_out/trace5.jsonl 2>&1
TCX_LIB_PATH=$DBG timeout 300 python tools/trace_gemm.py c5 8 wide >> gpurun_out/trace5.jsonl 2>&1
TCX_LIB_PATH=$DBG timeout 300 python tools/trace_gemm.py c3 8 >> gpurun_out/trace5.jsonl 2>&1
TCX_LIB_PATH=$DBG timeout 300 python tools/trace_gemm.py c3 8 wide >> gpurun_out/trace5.jsonl 2>&1
timeout 600 python tools/size_sweep.py > gpurun_out/size_sweep4.jsonl 2>&1
for i in 1 2; do timeout 600 python tools/exp_gemm.py c5 20 g8c2 g8c2w >> gpurun_out/origin_c5.jsonl 2>&1; done
for i in 1 2; do timeout 600 python tools/exp_gemm.py c3 50 g8c2 g8c2w >> gpurun_out/origin_c3.jsonl 2>&1; done; echo e=$?
