# sustained (~4 s per variant, power-capped) narrow vs wide dense tile, order alternated
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
for i in 1 2; do
  timeout 600 python tools/exp_gemm.py c3 5500 g8c2 g8c2w >> gpurun_out/wsus.jsonl 2>&1
  timeout 600 python tools/exp_gemm.py c3 5500 g8c2w g8c2 >> gpurun_out/wsus.jsonl 2>&1
  timeout 600 python tools/exp_gemm.py c4 1400 g8c2 g8c2w >> gpurun_out/wsus.jsonl 2>&1
  timeout 600 python tools/exp_gemm.py c4 1400 g8c2w g8c2 >> gpurun_out/wsus.jsonl 2>&1
done; echo e=$?
