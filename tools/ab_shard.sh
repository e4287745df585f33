#!/bin/bash
# Build-flag variants of the per-rank shard probe (bench.py --shard-probe-only):
# usage: tools/ab_shard.sh TAG "FLAGS_1" "FLAGS_2" ...   (each variant twice, alternating)
TAG=$1; shift
for round in 1 2; do
  k=0
  for F in "$@"; do
    k=$((k+1))
    AF_NVCC_EXTRA="$F" python paper_2102_01386_b200/_build.py
    AF_NVCC_EXTRA="$F" python bench.py --shard-probe-only --steps 100 > gpurun_out/${TAG}_v${k}_$round.json 2> gpurun_out/${TAG}_v${k}_$round.err
    python - "gpurun_out/${TAG}_v${k}_$round.json" "$F" <<'PY'
import json, sys
d = json.load(open(sys.argv[1]))["rank_shard_p8"]["max_over_ranks"]
print(repr(sys.argv[2]), "in_step", d["interval_end_in_step_us"], "alone", d["interval_end_alone_us"],
      "acc", d["accumulate_us"], "sum", round(d["interval_end_in_step_us"] + d["accumulate_us"], 2))
PY
  done
done
