mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 900 python -m pytest tests/test_gpu_fuzz.py -q > gpurun_out/t_fuzz.log 2>&1; echo t=$?
