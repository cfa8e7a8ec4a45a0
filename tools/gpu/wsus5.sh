# wide tile with 5 epilogue buffers (C 4 ahead): tests, burst and sustained vs narrow
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_gemm_model.py tests/test_gpu_fuzz.py tests/test_gpu_debug_build.py tests/test_gpu_gemm_f16acc.py -q -x > gpurun_out/t_w5.log 2>&1; echo t=$?; tail -1 gpurun_out/t_w5.log
for i in 1 2; do
  timeout 600 python tools/exp_gemm.py c3 30 g8c2 g8c2w >> gpurun_out/w5_burst.jsonl 2>&1
  timeout 600 python tools/exp_gemm.py c3tf32 30 g8c2 g8c2w >> gpurun_out/w5_burst.jsonl 2>&1
  timeout 600 python tools/exp_gemm.py c3 5500 g8c2 g8c2w >> gpurun_out/w5_sus.jsonl 2>&1
  timeout 600 python tools/exp_gemm.py c3 5500 g8c2w g8c2 >> gpurun_out/w5_sus.jsonl 2>&1
  timeout 600 python tools/exp_gemm.py c4 1400 g8c2 g8c2w >> gpurun_out/w5_sus.jsonl 2>&1
  timeout 600 python tools/exp_gemm.py c4 1400 g8c2w g8c2 >> gpurun_out/w5_sus.jsonl 2>&1
done; echo e=$?
