mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 1200 python tools/size_sweep.py > gpurun_out/size_sweep.jsonl 2> gpurun_out/size_sweep.err; echo s=$?
