# epilogue drain with and without the C path (debug-library tile trace)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
DBG=$PWD/paper_2206_02874_b200/libtcx_debug.so
for a in "c5 8 wide" "c5 8 wide noc" "c3 8 wide" "c3 8 wide noc" "c3 8 x" "c3 8 x noc"; do
  TCX_LIB_PATH=$DBG timeout 300 python tools/trace_gemm.py $a >> gpurun_out/trace_noc.jsonl 2>&1
done; echo e=$?
