mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_dist.py -q -x > gpurun_out/t_dense.log 2>&1; echo gemm=$?
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
