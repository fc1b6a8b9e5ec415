#!/bin/bash
# Per-phase SM-cycle breakdown (-DWS_PHASES build) of one plan per BASELINE config.
set -u
OUT=gpurun_out; mkdir -p $OUT
for c in clip-like:10:64 ofasys-like:7:32 qwen-val-like:3:64 clip-like:4:8; do
  echo "== $c" >> $OUT/phases_single.txt
  WSGPU_LIB=paper_2409_03365_b200/lib/libwsgpu_phases.so timeout 300 python scripts/phases.py $c >> $OUT/phases_single.txt 2>&1
done
echo "== sweep 100000" >> $OUT/phases_single.txt
WSGPU_LIB=paper_2409_03365_b200/lib/libwsgpu_phases.so timeout 300 python scripts/phases.py 100000 >> $OUT/phases_single.txt 2>&1
cat $OUT/phases_single.txt
