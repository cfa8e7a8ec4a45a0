mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 900 python -m pytest tests/test_gpu_data_movement.py -q -x > gpurun_out/t_dm3.log 2>&1; echo t2=$?
