mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
DBG=$PWD/paper_2206_02874_b200/libtcx_debug.so
TCX_LIB_PATH=$DBG timeout 300 python tools/trace_gemm.py c3 8 >> gpurun_out/trace4.jsonl 2>&1
TCX_LIB_PATH=$DBG timeout 300 python tools/trace_gemm.py c3 8 wide >> gpurun_out/trace4.jsonl 2>&1
TCX_LIB_PATH=$DBG timeout 300 python tools/trace_gemm.py c4 8 wide >> gpurun_out/trace4.jsonl 2>&1
