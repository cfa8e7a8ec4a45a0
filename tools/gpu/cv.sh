mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
AB=$PWD/paper_2206_02874_b200/libtcx_ab.so
ABD=$PWD/paper_2206_02874_b200/libtcx_abdbg.so
DBG=$PWD/paper_2206_02874_b200/libtcx_debug.so
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_sparse.py tests/test_gpu_fuzz.py tests/test_gpu_gemm_model.py -q -x > gpurun_out/t_cv.log 2>&1; echo t=$?
for c in "c5 8" "c3 8"; do set -- $c
  TCX_LIB_PATH=$ABD timeout 300 python tools/trace_gemm.py $1 $2 $([ $1 = c5 ] && echo wide) | sed 's/^{/{"lib": "old", /' >> gpurun_out/cv_trace.jsonl 2>&1
  TCX_LIB_PATH=$DBG timeout 300 python tools/trace_gemm.py $1 $2 $([ $1 = c5 ] && echo wide) | sed 's/^{/{"lib": "new", /' >> gpurun_out/cv_trace.jsonl 2>&1
done
for i in 1 2 3; do
  TCX_LIB_PATH=$AB timeout 600 python tools/exp_gemm.py c5 20 g8c2w | sed 's/"variant": "/"variant": "old_/' >> gpurun_out/cv_time.jsonl 2>&1
  timeout 600 python tools/exp_gemm.py c5 20 g8c2w | sed 's/"variant": "/"variant": "new_/' >> gpurun_out/cv_time.jsonl 2>&1
  TCX_LIB_PATH=$AB timeout 600 python tools/exp_gemm.py c3 50 g8c2 | sed 's/"variant": "/"variant": "old_/' >> gpurun_out/cv_time.jsonl 2>&1
  timeout 600 python tools/exp_gemm.py c3 50 g8c2 | sed 's/"variant": "/"variant": "new_/' >> gpurun_out/cv_time.jsonl 2>&1
done; echo e=$?
