mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
for o in 0 1; do TCX_WIDE_ORDER=$o timeout 300 python tools/exp_anchor.py 50 > gpurun_out/exp10_o$o.jsonl 2>&1; done
TCX_WIDE_ORDER=1 timeout 300 python -m pytest tests/test_gpu_gemm.py -q -x -k wide > gpurun_out/exp10_t.log 2>&1; echo t=$?
