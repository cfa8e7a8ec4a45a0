mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_gemm_f16acc.py tests/test_gpu_sparse.py -q -x -k "in_place or tile_n" > gpurun_out/t_inplace.log 2>&1; echo t=$?
