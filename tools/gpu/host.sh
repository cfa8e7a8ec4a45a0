mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 300 python tools/host_overhead.py > gpurun_out/host_overhead.json 2>&1; echo h=$?
