mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 900 python -m pytest tests/test_gpu_gemm_f16acc.py -q -x > gpurun_out/t_f16g.log 2>&1; echo f16g=$?
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_sparse.py -q -x > gpurun_out/t_f16g2.log 2>&1; echo reg=$?
