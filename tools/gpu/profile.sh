# ncu evidence for the bench: launch list of the bench command + one `--set full` capture per hot kernel.
# usage: bash tools/gpu/profile.sh <tag>
mkdir -p gpurun_out
TAG=${1:-r01}
BENCH="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --sustained-s 0"
$BENCH > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gemm_|tiles|sp24|fill_c" --csv \
    --log-file gpurun_out/${TAG}_launches.csv $BENCH > gpurun_out/ncu_launch.log 2>&1
echo launches=$?
for cfg in c3 c4 c5 c1 c3tf32; do
  case $cfg in
    c3|c3tf32|c4) K="regex:gemm_dense";;
    c5) K="regex:gemm_sp24";; c1) K="regex:tiles16";;
  esac
  python tools/prof_kernels.py $cfg 2 > gpurun_out/plain_$cfg.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k "$K" -s 1 -c 1 \
      -o gpurun_out/${TAG}_$cfg python tools/prof_kernels.py $cfg 2 > gpurun_out/ncu_$cfg.log 2>&1
  echo $cfg=$?
done
