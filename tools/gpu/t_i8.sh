mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 900 python -m pytest tests/test_gpu_sparse_i8.py -q -x -k "one_hot" > gpurun_out/t_i8.log 2>&1; echo onehot=$?
timeout 900 python -m pytest tests/test_gpu_sparse_i8.py tests/test_gpu_sparse.py -q > gpurun_out/t_i8_all.log 2>&1; echo tests=$?
