mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 600 python -m pytest tests/test_gpu_sparse_i8.py tests/test_gpu_sparse_tf32.py -q -x -k "multicast" > gpurun_out/t_mc3.log 2>&1; echo t=$?
timeout 600 python -m pytest tests/test_gpu_tiles.py -q -x > gpurun_out/t_tiles.log 2>&1; echo tt=$?
for i in 1 2 3; do timeout 300 python tools/exp_tiles.py f16 >> gpurun_out/exp_tiles_pf.jsonl 2>&1; done; echo e=$?
