mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 600 python bench.py --steps 5 --warmup 3 --no-extras --sustained-s 0 --no-cpu-baseline > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err; echo b=$?
timeout 600 python -m pytest tests/test_gpu_dist.py -q > gpurun_out/t_dist.log 2>&1; echo t=$?
