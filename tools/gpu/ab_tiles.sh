mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
for i in 1 2 3; do
  TCX_LIB_PATH=$PWD/paper_2206_02874_b200/libtcx_ab.so timeout 300 python tools/exp_tiles.py f16 | sed 's/^{/{"lib": "prev_db48",/' >> gpurun_out/ab_tiles.jsonl 2>&1
  timeout 300 python tools/exp_tiles.py f16 | sed 's/^{/{"lib": "new_sb32",/' >> gpurun_out/ab_tiles.jsonl 2>&1
done; echo e=$?
