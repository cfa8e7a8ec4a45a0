# INT8 2:4 (c4sp): 2 x 1 multicast group vs default, order alternated
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
for i in 1 2 3 4; do
  timeout 600 python tools/exp_gemm.py c4sp 60 g8c2 g8c2p21 >> gpurun_out/spmc2.jsonl 2>&1
  timeout 600 python tools/exp_gemm.py c4sp 60 g8c2p21 g8c2 >> gpurun_out/spmc2.jsonl 2>&1
done; echo e=$?
