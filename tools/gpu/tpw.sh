mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
for r in 1 2; do for t in 1 2 4 8; do
  TCX_TILES_TPW=$t timeout 300 python tools/exp_tiles.py f16 | sed "s/^{/{\"tpw\": $t, /" >> gpurun_out/tpw.jsonl 2>&1
done; done; echo e=$?
