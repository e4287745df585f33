#!/bin/bash
# Same-box A/B of the bench step between two build-flag sets of the working tree
# (AF_NVCC_EXTRA), alternating, N rounds.  Extra bench args in BENCH_ARGS.
# usage: tools/ab_flags.sh TAG N "FLAGS_A" "FLAGS_B"
TAG=$1; N=$2; FA=$3; FB=$4
ARGS="--no-e2e --no-cpu-baseline --no-cache-sweep --no-extras --no-shard-probe $BENCH_ARGS"
for i in $(seq 1 $N); do
  for side in A B; do
    if [ $side = A ]; then F="$FA"; else F="$FB"; fi
    AF_NVCC_EXTRA="$F" python paper_2102_01386_b200/_build.py
    AF_NVCC_EXTRA="$F" python bench.py $ARGS > gpurun_out/${TAG}_${side}_$i.json 2> gpurun_out/${TAG}_${side}_$i.err
  done
done
python - "$TAG" "$N" <<'PY'
import json, sys
tag, n = sys.argv[1], int(sys.argv[2])
for side in ("A", "B"):
    for i in range(1, n + 1):
        try:
            d = json.loads(open(f"gpurun_out/{tag}_{side}_{i}.json").read().strip().splitlines()[-1])
        except Exception as e:
            print(side, i, "ERR", e); continue
        s = d.get("secondary", {})
        pl, ps = d.get("phases_in_step", {}), s.get("phases_in_step", {})
        print(side, i, "large ms", d["ms_per_step"], "end", pl.get("grad_norm_decide", {}).get("ms"),
              "acc", pl.get("accumulate", {}).get("ms"), "| base ms", s.get("ms_per_step"),
              "end", ps.get("grad_norm_decide", {}).get("ms"), "acc", ps.get("accumulate", {}).get("ms"),
              "eager end", s.get("grad_norm_decide_gbs"))
PY
