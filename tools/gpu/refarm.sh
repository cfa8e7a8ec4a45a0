mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/ref_arm.json 2> gpurun_out/ref_arm.err; echo r=$?
timeout 600 python bench.py --steps 5 --warmup 3 --no-extras --sustained-s 0 > gpurun_out/bench_min.json 2> gpurun_out/bench_min.err; echo b=$?
