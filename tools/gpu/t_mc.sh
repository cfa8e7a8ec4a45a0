mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 120 python -m pytest tests/test_gpu_gemm.py -q -x -k "multicast_cluster_whole_matrix and bf16 and 256-256-128" > gpurun_out/t_mc0.log 2>&1; echo t0=$?
timeout 600 python -m pytest tests/test_gpu_gemm.py -q -x -k "multicast or pairs" > gpurun_out/t_mc.log 2>&1; echo t=$?
timeout 300 python tools/exp_gemm.py c3 50 g8c2 g8c2p12 g8c2p21 g8c2p22 g4c2p22 g16c2p22 g8c2 > gpurun_out/exp_mc_c3.log 2>&1; echo e=$?
timeout 300 python tools/exp_gemm.py c4 20 g8c2 g8c2p12 g8c2p21 g8c2p22 g4c2p22 > gpurun_out/exp_mc_c4.log 2>&1; echo e4=$?
