#!/bin/bash
# Weak-scaling bench lines at N = 1, 2, 4 on one box (run via gpurun --gpus 4).
# usage: bash scripts/scale_check.sh [tag]
set -u
TAG=${1:-scale}
OUT=gpurun_out
mkdir -p $OUT
timeout 900 python bench.py --steps 10 --warmup 3 > $OUT/bench_${TAG}_1gpu.json 2> $OUT/bench_${TAG}_1gpu.err; echo "n=1 rc=$?"
for n in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29533 \
      bench.py --gpus $n --steps 10 --warmup 3 > $OUT/bench_${TAG}_${n}gpu.json 2> $OUT/bench_${TAG}_${n}gpu.err
  echo "n=$n rc=$?"
done
for n in 1 2 4; do python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], d['value'], d['e2e']['value'], d.get('rank_step_ms'))" $OUT/bench_${TAG}_${n}gpu.json $n; done
