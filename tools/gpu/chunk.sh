# dense epilogue chunk-phase breakdown (debug library), per epilogue warp
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
DBG=$PWD/paper_2206_02874_b200/libtcx_debug.so
timeout 300 python -m pytest tests/test_gpu_debug_build.py -q -x > gpurun_out/t_chunk.log 2>&1; echo t=$?
for a in "c3 wide" "c3 wide noc" "c3"; do
  TCX_LIB_PATH=$DBG timeout 300 python tools/chunk_trace.py $a >> gpurun_out/chunk_trace2.jsonl 2>&1
done; echo e=$?
