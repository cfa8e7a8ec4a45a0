mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
DBG=$PWD/paper_2206_02874_b200/libtcx_debug.so
TCX_LIB_PATH=$DBG timeout 300 python tools/trace_gemm.py c5 8 >> gpurun_out/trace2.jsonl 2>&1
TCX_LIB_PATH=$DBG timeout 300 python tools/trace_gemm.py c5 8 wide >> gpurun_out/trace2.jsonl 2>&1
TCX_LIB_PATH=$DBG timeout 300 python tools/trace_gemm.py c3 8 >> gpurun_out/trace2.jsonl 2>&1
timeout 600 python -m pytest tests/test_gpu_sparse.py tests/test_gpu_debug_build.py -q -x -k "m_wide or small or debug or trace" > gpurun_out/t_tr2.log 2>&1; echo t=$?
