mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
for st in 0 1 2; do
TCX_STAGGER=$st timeout 600 python tools/exp_gemm.py c5 20 g8c2w g8c2 g8c2w > gpurun_out/exp21_c5_s$st.jsonl 2>&1
TCX_STAGGER=$st timeout 300 python tools/exp_anchor.py 30 > gpurun_out/exp21_c3_s$st.jsonl 2>&1
done
TCX_STAGGER=1 timeout 600 python -m pytest tests/test_gpu_sparse.py tests/test_gpu_gemm.py -q -x -k "wide" > gpurun_out/exp21_t.log 2>&1; echo t=$?
