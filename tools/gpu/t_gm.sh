mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 1200 python -m pytest tests/test_gpu_gemm_model.py -q > gpurun_out/t_gm.log 2>&1; echo t=$?
