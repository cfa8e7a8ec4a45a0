mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 900 python -m pytest tests/test_gpu_debug_build.py tests/test_gpu_sparse.py tests/test_gpu_sparse_i8.py tests/test_gpu_sparse_tf32.py -q -x > gpurun_out/t_dbg2.log 2>&1; echo t=$?
