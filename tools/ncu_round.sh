#!/bin/bash
# ncu evidence for one round's state (run on the GPU box): the launch list of the
# bench's step (gpu__time_duration, serialised, cold) and an `ncu --set full`
# capture of the step's kernels inside graph replays, for both workloads.
# usage: tools/ncu_round.sh TAG
TAG=$1
ARGS="--no-e2e --no-cpu-baseline --no-cache-sweep --no-extras --no-secondary --no-shard-probe"
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches.csv \
    python bench.py --steps 2 --warmup 1 $ARGS > gpurun_out/${TAG}_launches_bench.log 2>&1
for W in bert-large-f32 bert-base-bf16; do
  ncu --set full --clock-control none --import-source on -k regex:"norms_kernel|cache_kernel" \
      --launch-skip 40 --launch-count 8 -f -o gpurun_out/${TAG}_${W} \
      python bench.py --workload $W --steps 3 --warmup 3 $ARGS > gpurun_out/${TAG}_${W}_ncu.log 2>&1
done
