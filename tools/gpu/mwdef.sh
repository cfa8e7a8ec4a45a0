mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 1200 python -m pytest tests/test_gpu_sparse.py tests/test_gpu_sparse_i8.py tests/test_gpu_sparse_tf32.py tests/test_gpu_gemm_model.py tests/test_gpu_fuzz.py tests/test_gpu_debug_build.py -q -x > gpurun_out/t_mwdef.log 2>&1; echo t=$?
timeout 600 python bench.py --config c5 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo b=$?
