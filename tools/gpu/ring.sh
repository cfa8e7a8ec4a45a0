mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_gemm_model.py tests/test_gpu_fuzz.py tests/test_gpu_streams_graphs.py tests/test_gpu_dist.py tests/test_gpu_debug_build.py -q -x > gpurun_out/t_ring.log 2>&1; echo t=$?
timeout 300 python tools/host_overhead.py > gpurun_out/host_overhead3.json 2>&1
timeout 600 python tools/size_sweep.py > gpurun_out/size_sweep3.jsonl 2>&1; echo s=$?
DBG=$PWD/paper_2206_02874_b200/libtcx_debug.so
for s in "256 64" "1024 1024"; do set -- $s; TCX_LIB_PATH=$DBG timeout 120 python tools/small_gemm.py $1 $2 trace >> gpurun_out/small_trace2.txt 2>&1; done
timeout 300 python tools/exp_gemm.py c3 50 g8c2 g8c2 g8c2 > gpurun_out/ring_c3.jsonl 2>&1
timeout 300 python tools/exp_gemm.py c4 20 g8c2 g8c2 > gpurun_out/ring_c4.jsonl 2>&1; echo e=$?
