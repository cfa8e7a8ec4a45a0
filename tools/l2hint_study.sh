#!/bin/bash
# L2 eviction hints (TCX_L2HINT variants, tools/build_variant.py) and raster/grid options:
# burst A/B (tools/ab_burst*.{py,sh}) + cold-launch DRAM bytes per variant under ncu
cd "$GRAFT_REPO_ROOT"; O=gpurun_out/l2h; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > $O/gpu.txt
for cfg in c4 c3 c5; do
  timeout 1200 bash tools/ab_burst_libs.sh $O/ab_$cfg.jsonl $cfg 3 default l2h3 l2h19 l2h35 l2h51 > $O/ab_$cfg.log 2>&1
done
timeout 900 python tools/ab_burst.py c4 "pairs=0x0;group_m=4;group_m=16;group_m=32;group_m=-8" 3 > $O/ab_c4_group.jsonl 2> $O/ab_c4_group.err
timeout 900 python tools/ab_burst.py c3 "pairs=0x0;max_ctas=144;max_ctas=128;group_m=4;group_m=16" 3 > $O/ab_c3_grid.jsonl 2> $O/ab_c3_grid.err
for lib in default l2h3 l2h19 l2h35 l2h51; do
  if [ $lib = default ]; then p=$PWD/paper_2206_02874_b200/libtcx.so; else p=$PWD/paper_2206_02874_b200/variants/libtcx_$lib.so; fi
  for v in c3 c4 c5; do
    TCX_LIB_PATH=$p timeout 400 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read.sum --clock-control none -k regex:gemm -c 2 --csv python tools/prof_variant.py $v 2 > $O/ncu_${lib}_$v.csv 2> $O/ncu_${lib}_$v.err
  done
done
echo done > $O/done
