mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/gputests.log 2>&1; echo tests=$?
tail -2 gpurun_out/gputests.log
timeout 900 python bench.py > gpurun_out/bench_m.json 2> gpurun_out/bench_m.err; echo bench=$?
bash tools/gpu/profile.sh r01g
python tools/ncu_traffic.py gpurun_out/r01g > gpurun_out/r01g_traffic.json 2>&1; echo traffic=$?
