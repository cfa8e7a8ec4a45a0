mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 900 python tools/ab_sparse_tile.py f16:8192:8192:8192 40 4 > gpurun_out/ab_tile_f16_8k.jsonl 2>&1
timeout 900 python tools/ab_sparse_tile.py f16:16384:16384:16384 10 4 > gpurun_out/ab_tile_f16_16k.jsonl 2>&1
timeout 900 python tools/ab_sparse_tile.py f16:32768:16384:8192 10 4 > gpurun_out/ab_tile_f16_32k8k.jsonl 2>&1
timeout 900 python tools/ab_sparse_tile.py c3sptf32 40 2 > gpurun_out/ab_tile_tf32b.jsonl 2>&1; echo a=$?
