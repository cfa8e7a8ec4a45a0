mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 600 python -m pytest tests/test_gpu_sparse.py tests/test_gpu_sparse_tf32.py -q -x -k "wide" > gpurun_out/t_spmw.log 2>&1; echo t=$?
timeout 600 python tools/exp_gemm.py c5 20 g8c2 g8c2w g8c2 g8c2w > gpurun_out/exp18_c5.jsonl 2>&1; echo e=$?
timeout 600 python -m pytest tests/test_gpu_sparse.py tests/test_gpu_sparse_i8.py tests/test_gpu_sparse_tf32.py -q -x > gpurun_out/t_spall.log 2>&1; echo all=$?
