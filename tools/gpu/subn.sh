mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 600 python tools/subnormal_dump.py > gpurun_out/subn.log 2>&1; echo s=$?
