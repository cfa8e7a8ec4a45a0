# run-to-run spread of the default bench line (three back-to-back runs on one box)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
for i in 1 2 3; do timeout 900 python bench.py >> gpurun_out/bench_var.jsonl 2>> gpurun_out/bench_var.err; echo b$i=$?; done
