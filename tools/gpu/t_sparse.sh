mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 900 python -m pytest tests/test_gpu_sparse.py tests/test_gpu_sparse_i8.py tests/test_gpu_sparse_tf32.py -q -x > gpurun_out/t_sparse.log 2>&1; echo sparse=$?
timeout 400 python tools/exp_gemm.py c5 30 g8c2 g8c2 > gpurun_out/exp12_c5.jsonl 2>&1; echo c5=$?
