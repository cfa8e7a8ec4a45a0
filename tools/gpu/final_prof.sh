mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 900 python bench.py > gpurun_out/bench_g.json 2> gpurun_out/bench_g.err; echo bench=$?
bash tools/gpu/profile.sh r01d
