mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 900 python -m pytest tests/test_gpu_chain.py -v -k "instruction_model" > gpurun_out/t_ch.log 2>&1; echo t=$?
