#!/usr/bin/env python
"""Extract per-launch DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum)
of our kernels from `ncu --set full` captures into profiles/traffic.json, which
bench.py reports as roofline.traffic for the dominant kernel.

    python tools/traffic_from_ncu.py --workload bert-large-f32 --rep gpurun_out/prof_norms.ncu-rep \
        [--rep gpurun_out/prof_cache.ncu-rep] --out profiles/traffic.json
"""
import argparse
import csv
import io
import json
import os
import re
import subprocess
from collections import defaultdict

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def phase_of(kernel):
    """Bench phase of a captured kernel; the streaming kernels only in the bench's
    timed form (Delta armed: template argument RD = 1)."""
    m = re.search(r"norms_kernel<(\d+), ([^,]+), (\w+)", kernel)
    if m:
        mode, rd = int(m.group(1)), m.group(3) in ("1", "true")
        if not rd and mode != 2:
            return None
        return {0: "accumulate", 1: "grad_norm_decide", 2: "step_sumsq"}.get(mode)
    if "fin_kernel" in kernel:
        return "grad_norm_finalize"
    if "cache_kernel<1>" in kernel or "cache_kernel<true>" in kernel:
        return "cache_put"
    if "cache_kernel<0>" in kernel or "cache_kernel<false>" in kernel:
        return "cache_get"
    if "decide" in kernel:
        return "decide"
    return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", required=True)
    ap.add_argument("--rep", action="append", required=True)
    ap.add_argument("--out", default="profiles/traffic.json")
    a = ap.parse_args()
    acc = defaultdict(list)
    for rep in a.rep:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(out)))
        h, u = rows[0], rows[1]
        ki = h.index("Kernel Name")
        ri, wi = h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum")
        for r in rows[2:]:
            ph = phase_of(r[ki])
            if ph:
                b = float(r[ri]) * SCALE[u[ri]] + float(r[wi]) * SCALE[u[wi]]
                acc[ph].append(b)
    data = json.load(open(a.out)) if os.path.exists(a.out) else {}
    prev = data.get(a.workload, {})
    prev.update({ph: {"bytes_per_launch": sum(v) / len(v), "launches": len(v),
                      "source": ", ".join(os.path.basename(r) for r in a.rep)}
                 for ph, v in acc.items()})
    data[a.workload] = prev
    with open(a.out, "w") as f:
        json.dump(data, f, indent=1)
    print(json.dumps(data[a.workload], indent=1))


if __name__ == "__main__":
    main()
