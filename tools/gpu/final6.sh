mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke6.log 2>&1; echo smoke=$?
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/gputests6.log 2>&1; echo tests=$?
tail -1 gpurun_out/gputests6.log
timeout 900 python bench.py > gpurun_out/bench_n.json 2> gpurun_out/bench_n.err; echo bench=$?
