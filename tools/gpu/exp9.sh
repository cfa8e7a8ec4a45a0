mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
for v in wide narrow; do
python tools/exp_one.py $v 3 > /dev/null 2>&1 && \
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_dense -s 2 -c 1 -o gpurun_out/r01_$v python tools/exp_one.py $v 3 > gpurun_out/ncu_$v.log 2>&1; echo $v=$?
done
