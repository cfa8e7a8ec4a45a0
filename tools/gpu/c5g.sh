mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
for i in 1 2 3; do timeout 600 python tools/exp_gemm.py c5 10 g8c2 g16c2 g12c2 >> gpurun_out/c5g_time.jsonl 2>&1; done; echo e=$?
