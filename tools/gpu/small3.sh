mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
TCX_LIB_PATH=$PWD/paper_2206_02874_b200/libtcx_debug.so timeout 120 python tools/small_gemm_cyc.py > gpurun_out/small_cyc.txt 2>&1; echo ok
