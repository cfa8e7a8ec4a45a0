mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
for i in 1 2 3 4; do timeout 600 python tools/exp_gemm.py c5 40 g8c2 g8c2w >> gpurun_out/c5mw.jsonl 2>&1; done; echo e=$?
for i in 1 2; do timeout 600 python tools/exp_gemm.py c5 40 g8c2w g8c2 >> gpurun_out/c5mw.jsonl 2>&1; done; echo e2=$?
