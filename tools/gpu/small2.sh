mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
DBG=$PWD/paper_2206_02874_b200/libtcx_debug.so
TCX_LIB_PATH=$DBG timeout 120 python tools/small_gemm_marks.py 256 64 > gpurun_out/small_marks.txt 2>&1
TCX_LIB_PATH=$DBG timeout 120 python tools/small_gemm_marks.py 256 1024 >> gpurun_out/small_marks.txt 2>&1; echo ok
