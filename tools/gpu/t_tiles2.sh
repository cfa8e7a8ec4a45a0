mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 600 python -m pytest tests/test_gpu_tiles.py -q -x > gpurun_out/t_tiles.log 2>&1; echo tt=$?
for i in 1 2 3; do timeout 300 python tools/exp_tiles.py f16 >> gpurun_out/exp_tiles_pf2.jsonl 2>&1; done; echo e=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/gputests.log 2>&1; echo tests=$?
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
