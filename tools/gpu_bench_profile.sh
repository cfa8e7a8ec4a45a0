#!/bin/bash
# bench line + one full ncu capture per config kernel + the bench's launch list, on the GPU box:
#   bash tools/gpu_bench_profile.sh TAG     (outputs gpurun_out/TAG_*)
tag=${1:-r02}
timeout 900 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err; tail -3 gpurun_out/${tag}_bench.err
for c in c3 c3tf32 c3f16acc c4 c4sp c3sptf32 c5 c1; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:"gemm|tiles" -s 2 -c 1 -o gpurun_out/${tag}_$c python tools/prof_kernels.py $c 3 > gpurun_out/${tag}_ncu_$c.log 2>&1; tail -1 gpurun_out/${tag}_ncu_$c.log
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${tag}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --sustained-s 0 > gpurun_out/${tag}_ncu_bench.log 2>&1; tail -2 gpurun_out/${tag}_ncu_bench.log
