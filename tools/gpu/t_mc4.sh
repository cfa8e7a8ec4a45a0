mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 600 python -m pytest tests/test_gpu_sparse.py tests/test_gpu_sparse_i8.py tests/test_gpu_sparse_tf32.py -q -x -k "multicast" > gpurun_out/t_mc3.log 2>&1; echo t=$?
timeout 600 python tools/exp_gemm.py c3 1500 g8c2 g8c2p12 g8c2p21 g8c2 g8c2p12 g8c2p21 g8c2 g8c2p12 g8c2p21 > gpurun_out/exp_mc_c3_long.log 2>&1; echo e=$?
timeout 600 python tools/exp_gemm.py c4 300 g8c2 g8c2p12 g8c2p21 g8c2 g8c2p12 g8c2p21 > gpurun_out/exp_mc_c4_long.log 2>&1; echo e4=$?
