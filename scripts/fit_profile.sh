#!/bin/bash
# ncu capture of the warp-per-module k_fit on a single plan (CLIP 10t/64 is the
# second config of scripts/latency_probe.py) and the bench's reference arm.
set -u
TAG=${1:-r1i}
OUT=gpurun_out
mkdir -p $OUT
WSGPU_PDL=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fit -s 240 -c 1 \
    -o $OUT/kfitwarp_$TAG python scripts/latency_probe.py > $OUT/ncu_kfitwarp_$TAG.log 2>&1
echo "ncu kfit rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/bench_reference_$TAG.json 2> $OUT/bench_reference_$TAG.err
echo "reference rc=$?"; tail -1 $OUT/bench_reference_$TAG.json
