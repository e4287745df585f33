#!/bin/bash
# Same-box A/B of the bench step: ab_base/ (an exported earlier tree, built in place)
# against the working tree, alternating, N rounds.  Writes gpurun_out/<tag>_{base,new}_<i>.json.
TAG=${1:-ab}; N=${2:-2}
ARGS="--no-e2e --no-cpu-baseline --no-cache-sweep --no-extras"
for i in $(seq 1 $N); do
  (cd ab_base && python bench.py $ARGS > ../gpurun_out/${TAG}_base_$i.json 2> ../gpurun_out/${TAG}_base_$i.err)
  python bench.py $ARGS --no-shard-probe > gpurun_out/${TAG}_new_$i.json 2> gpurun_out/${TAG}_new_$i.err
done
python - "$TAG" "$N" <<'PY'
import json, sys
tag, n = sys.argv[1], int(sys.argv[2])
for side in ("base", "new"):
    for i in range(1, n + 1):
        try:
            d = json.loads(open(f"gpurun_out/{tag}_{side}_{i}.json").read().strip().splitlines()[-1])
        except Exception as e:
            print(side, i, "ERR", e); continue
        s = d.get("secondary", {})
        print(side, i, "large ms", d["ms_per_step"], "gnd", d["grad_norm_decide_gbs"],
              "| base ms", s.get("ms_per_step"), "gnd", s.get("grad_norm_decide_gbs"))
PY
