mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 900 python -m pytest tests/test_gpu_gemm.py -q -x -k "wide" > gpurun_out/t_wide.log 2>&1; echo wide=$?
timeout 900 python -m pytest tests/test_gpu_gemm.py -q -x > gpurun_out/t_gemm.log 2>&1; echo gemm=$?
timeout 300 python tools/exp_anchor.py 50 > gpurun_out/exp6_anchor.jsonl 2>&1; echo anchor=$?
