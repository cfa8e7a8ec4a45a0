mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 300 python -m pytest tests/test_gpu_gemm.py -q -x -k wide > gpurun_out/exp11_t.log 2>&1; echo t=$?
timeout 300 python tools/exp_anchor.py 50 > gpurun_out/exp11.jsonl 2>&1; echo a=$?
