mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
for i in 1 2 3; do timeout 600 python tools/exp_gemm.py c4 80 g8c2 g8c2w >> gpurun_out/c4w.jsonl 2>&1; done
for i in 1 2; do timeout 600 python tools/exp_gemm.py c3 600 g8c2 g8c2w >> gpurun_out/c3w.jsonl 2>&1; done; echo e=$?
