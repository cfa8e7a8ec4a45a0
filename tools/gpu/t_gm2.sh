mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 1500 python -m pytest tests/test_gpu_gemm_model.py tests/test_gpu_gemm.py tests/test_gpu_sparse.py -q -x -k "model or config3 or config5" > gpurun_out/t_gm2.log 2>&1; echo t=$?
