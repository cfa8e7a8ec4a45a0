mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 1500 python -m pytest tests/test_gpu_gemm_model.py -v > gpurun_out/t_gm3.log 2>&1; echo t=$?
