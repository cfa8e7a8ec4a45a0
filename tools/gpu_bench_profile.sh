set -x
timeout 900 python bench.py > gpurun_out/r02a_bench.json 2> gpurun_out/r02a_bench.err; tail -3 gpurun_out/r02a_bench.err
for c in c3 c3tf32 c3f16acc c4 c4sp c3sptf32 c5 c1; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:"gemm|tiles" -s 2 -c 1 -o gpurun_out/r02a_$c python tools/prof_kernels.py $c 3 > gpurun_out/r02a_ncu_$c.log 2>&1; tail -1 gpurun_out/r02a_ncu_$c.log
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02a_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --sustained-s 0 > gpurun_out/r02a_ncu_bench.log 2>&1; tail -2 gpurun_out/r02a_ncu_bench.log
