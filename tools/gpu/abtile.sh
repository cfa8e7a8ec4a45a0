mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 900 python tools/ab_sparse_tile.py c3sptf32 40 6 > gpurun_out/ab_tile_tf32.jsonl 2>&1; echo a=$?
