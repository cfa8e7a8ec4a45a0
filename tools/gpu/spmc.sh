# multicast groups of CTA pairs on the INT8 2:4 and TF32 1:2 sparse configs
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
for i in 1 2 3; do
  timeout 600 python tools/exp_gemm.py c4sp 30 g8c2 g8c2p12 g8c2p21 g8c2p22 g-8c2 g4c2 g16c2 >> gpurun_out/spmc.jsonl 2>&1
  timeout 600 python tools/exp_gemm.py c3sptf32 40 g8c2 g8c2p12 g8c2p21 g8c2p22 g8c2w g4c2 g16c2 >> gpurun_out/spmc.jsonl 2>&1
done; echo e=$?
