#!/bin/bash
# A/B library variants with the energy study, interleaved over rounds:
#   bash tools/ab_libs.sh OUT.jsonl "c3,c5" ROUNDS lib1 lib2 ...   (lib "default" = libtcx.so)
out=$1; variants=$2; rounds=$3; shift 3
for r in $(seq 1 $rounds); do
  for lib in "$@"; do
    if [ "$lib" = default ]; then path=$PWD/paper_2206_02874_b200/libtcx.so; else path=$PWD/paper_2206_02874_b200/variants/libtcx_$lib.so; fi
    TCX_LIB_PATH=$path python tools/energy_study.py /tmp/ab_$lib.jsonl "$variants" 2.0 1 | sed "s/^{/{\"lib\": \"$lib\", /" >> $out
  done
done
