mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/gputests.log 2>&1; echo tests=$?
timeout 900 python bench.py > gpurun_out/bench_l.json 2> gpurun_out/bench_l.err; echo bench=$?
