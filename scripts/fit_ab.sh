#!/bin/bash
# One GPU-box session: k_fit warp-per-module vs thread-per-module A/B on
# single-plan latency, then the GPU parity suite and the bench.
# usage (from repo root, via gpurun): bash scripts/fit_ab.sh [tag]
set -u
TAG=${1:-fitab}
OUT=gpurun_out
mkdir -p $OUT
for pdl in 0 1; do
  for wm in 0 4096; do
    echo "== WSGPU_PDL=$pdl WSGPU_FIT_WARP_MAX=$wm" >> $OUT/latency_$TAG.txt
    WSGPU_PDL=$pdl WSGPU_FIT_WARP_MAX=$wm timeout 300 python scripts/latency_probe.py >> $OUT/latency_$TAG.txt 2>&1
  done
done
cat $OUT/latency_$TAG.txt
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest gpu rc=$?" | tee -a $OUT/summary_$TAG.txt
tail -3 $OUT/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc=$?" | tee -a $OUT/summary_$TAG.txt
timeout 900 python bench.py --steps 10 --warmup 3 > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo "bench rc=$?" | tee -a $OUT/summary_$TAG.txt
cat $OUT/bench_$TAG.json
