mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 300 python tools/host_overhead.py > gpurun_out/host_overhead2.json 2>&1; echo h=$?
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_tiles.py tests/test_gpu_streams_graphs.py tests/test_gpu_fuzz.py tests/test_gpu_chain.py -q -x > gpurun_out/t_host2.log 2>&1; echo t=$?
timeout 600 python tools/size_sweep.py > gpurun_out/size_sweep2.jsonl 2>&1; echo s=$?
