mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 600 python -m pytest tests/test_gpu_streams_graphs.py -q > gpurun_out/t_sg.log 2>&1; echo t=$?
