mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 900 python -m pytest tests/test_gpu_sparse_tf32.py -q -x > gpurun_out/t_tf32sp.log 2>&1; echo tests=$?
