#!/bin/bash
# Same-box A/B of the per-rank shard probe (bench.py --shard-probe-only) between an
# exported earlier tree in ab_base/ (built in place) and the working tree,
# alternating, N rounds.  usage: tools/ab_shard_tree.sh TAG N
TAG=${1:-abst}; N=${2:-2}
(cd ab_base && python paper_2102_01386_b200/_build.py)
python paper_2102_01386_b200/_build.py
for i in $(seq 1 $N); do
  for side in base new; do
    if [ $side = base ]; then D=ab_base; else D=.; fi
    (cd $D && python bench.py --shard-probe-only --steps 100) > gpurun_out/${TAG}_${side}_$i.json 2> gpurun_out/${TAG}_${side}_$i.err
    python - "gpurun_out/${TAG}_${side}_$i.json" "$side" <<'PY'
import json, sys
d = json.load(open(sys.argv[1]))["rank_shard_p8"]["max_over_ranks"]
print(sys.argv[2], "in_step", d["interval_end_in_step_us"], "alone", d["interval_end_alone_us"], "acc", d["accumulate_us"])
PY
  done
done
