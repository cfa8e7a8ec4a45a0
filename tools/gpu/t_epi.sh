mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 600 python -m pytest tests/test_gpu_gemm.py -q -x -k "small_whole and bf16 and shape0" > gpurun_out/t_epi0.log 2>&1; echo first=$?
timeout 900 python -m pytest tests/test_gpu_gemm.py -q -x > gpurun_out/t_epi.log 2>&1; echo gemm=$?
timeout 300 python tools/exp_anchor.py 50 > gpurun_out/exp8_anchor.jsonl 2>&1; echo anchor=$?
