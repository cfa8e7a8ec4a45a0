mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 900 python -m pytest tests/test_gpu_numeric_probe_f16acc.py -q -x > gpurun_out/t_f16w.log 2>&1; echo t=$?
