# raster group for the M-wide sparse tile (C5)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
for i in 1 2 3; do timeout 600 python tools/exp_gemm.py c5 20 g8c2w g4c2w g16c2w g-4c2w g2c2w g8c2w >> gpurun_out/c5wr.jsonl 2>&1; done; echo e=$?
