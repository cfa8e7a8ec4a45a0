#!/bin/bash
# A/B library variants under the bench's burst conditions (tools/ab_burst.py), interleaved:
#   bash tools/ab_burst_libs.sh OUT.jsonl CFG ROUNDS lib1 lib2 ...   (lib "default" = libtcx.so)
out=$1; cfg=$2; rounds=$3; shift 3
for r in $(seq 1 $rounds); do
  for lib in "$@"; do
    if [ "$lib" = default ]; then path=$PWD/paper_2206_02874_b200/libtcx.so; else path=$PWD/paper_2206_02874_b200/variants/libtcx_$lib.so; fi
    TCX_LIB_PATH=$path python tools/ab_burst.py $cfg "pairs=0x0" 1 | sed "s/^{/{\"lib\": \"$lib\", /" >> $out
  done
done
