mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/bench_i.json 2> gpurun_out/bench_i.err; echo bench=$?
bash tools/gpu/profile.sh r01e
