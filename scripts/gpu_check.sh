#!/bin/bash
# One GPU-box session: parity tests, smoke, bench, ncu launch list + k_plan capture.
# usage (from repo root, via gpurun): bash scripts/gpu_check.sh [tag]
set -u
TAG=${1:-r1}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/nvsmi_$TAG.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest gpu rc=$?" | tee -a $OUT/summary_$TAG.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc=$?" | tee -a $OUT/summary_$TAG.txt
timeout 900 python bench.py --steps 10 --warmup 3 > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo "bench rc=$?" | tee -a $OUT/summary_$TAG.txt
NCU_CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --latency-reps 1"
if timeout 600 $NCU_CMD > $OUT/ncu_plain_$TAG.log 2>&1; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
      --log-file $OUT/launches_$TAG.csv $NCU_CMD > $OUT/ncu_launch_$TAG.log 2>&1
  echo "ncu launches rc=$?" | tee -a $OUT/summary_$TAG.txt
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_place -s 4 -c 1 \
      -o $OUT/kplace_$TAG $NCU_CMD > $OUT/ncu_full_$TAG.log 2>&1
  echo "ncu full rc=$?" | tee -a $OUT/summary_$TAG.txt
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sched -s 4 -c 1 \
      -o $OUT/ksched_$TAG $NCU_CMD > $OUT/ncu_fullfit_$TAG.log 2>&1
  echo "ncu fit rc=$?" | tee -a $OUT/summary_$TAG.txt
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sim -s 2 -c 1 \
      -o $OUT/ksim_$TAG $NCU_CMD > $OUT/ncu_fullsim_$TAG.log 2>&1
  echo "ncu sim rc=$?" | tee -a $OUT/summary_$TAG.txt
fi
tail -5 $OUT/pytest_gpu_$TAG.log
cat $OUT/smoke_$TAG.log | tail -2
cat $OUT/bench_$TAG.json
tail -3 $OUT/bench_$TAG.err
