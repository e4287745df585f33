#!/usr/bin/env python
"""Summarise ncu captures brought back in gpurun_out/ into a markdown file under profiles/.

    python tools/ncu_summary.py --launches gpurun_out/launches.csv \
        --rep gpurun_out/prof_norms.ncu-rep --rep gpurun_out/prof_cache.ncu-rep \
        --bench gpurun_out/bench_large.json --out profiles/r01_summary.md
"""
import argparse
import csv
import io
import json
import subprocess
from collections import OrderedDict, defaultdict

RAW_METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "launch__occupancy_limit_registers",
    "lts__t_bytes.sum", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum",
]


OUR_KERNELS = ("norms_kernel", "fin_kernel", "decide_kernel", "cache_kernel", "cache_plan_kernel", "norms_tma_kernel")


def is_ours(name):
    return any(k in name for k in OUR_KERNELS)


def short(name):
    name = name.replace("void ", "").replace("af::<unnamed>::", "").replace("(anonymous namespace)::", "")
    return name.split("(")[0][:70]


def launch_seq(path):
    text = open(path).read()
    lines = [ln for ln in text.splitlines() if ln.startswith('"')]
    rows = list(csv.reader(io.StringIO("\n".join(lines))))
    h = rows[0]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    out = []
    for r in rows[1:]:
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}.get(r[ui], 1e-3)
        out.append((short(r[ki]), float(r[vi].replace(",", "")) * scale))
    return out


def launches_table(path):
    text = open(path).read()
    lines = [ln for ln in text.splitlines() if ln.startswith('"')]
    rows = list(csv.reader(io.StringIO("\n".join(lines))))
    h = rows[0]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    per = defaultdict(list)
    order = OrderedDict()
    for r in rows[1:]:
        k = short(r[ki])
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}.get(r[ui], 1e-3)
        per[k].append(float(r[vi].replace(",", "")) * scale)
        order[k] = True
    return per, list(order)


def raw_rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": short(r[h.index("Kernel Name")])}
        for m in RAW_METRICS:
            if m in h:
                u = units[h.index(m)]
                d[f"{m} [{u}]" if u else m] = r[h.index(m)]
        res.append(d)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--rep", action="append", default=[])
    ap.add_argument("--bench", action="append", default=[])
    ap.add_argument("--out", required=True)
    ap.add_argument("--title", default="ncu summary")
    ap.add_argument("--tail-ours", type=int, default=0,
                    help="also tabulate the last N launches of our kernels (the timed steps)")
    a = ap.parse_args()
    md = [f"# {a.title}", ""]
    for b in a.bench:
        try:
            j = json.loads(open(b).read().strip().splitlines()[-1])
        except Exception as e:  # noqa: BLE001
            md += [f"bench {b}: unreadable ({e})", ""]
            continue
        md += [f"## bench `{b}`", "", "```json", json.dumps(j, indent=1)[:6000], "```", ""]
    if a.launches:
        per, order = launches_table(a.launches)
        tot = sum(sum(v) for k, v in per.items() if is_ours(k))
        md += ["## launch list (ncu `gpu__time_duration.sum`, --clock-control none; cold-cache, serialised)", "",
               "| kernel | launches | mean µs | min µs | max µs | share of our kernels |", "|---|---|---|---|---|---|"]
        for k in order:
            v = per[k]
            ours = is_ours(k)
            share = f"{sum(v) / tot:.3f}" if ours and tot else "—"
            md.append(f"| `{k}` | {len(v)} | {sum(v) / len(v):.2f} | {min(v):.2f} | {max(v):.2f} | {share} |")
        md.append("")
    if a.launches and a.tail_ours:
        seq = [x for x in launch_seq(a.launches)
               if is_ours(x[0])][-a.tail_ours:]
        per = defaultdict(list)
        for k, v in seq:
            per[k].append(v)
        tot = sum(v for _, v in seq)
        md += [f"## timed-step launches only (last {len(seq)} launches of our kernels)", "",
               "| kernel | launches | mean µs | share of the step |", "|---|---|---|---|"]
        for k, v in per.items():
            md.append(f"| `{k}` | {len(v)} | {sum(v) / len(v):.2f} | {sum(v) / tot:.3f} |")
        md.append("")
    for rep in a.rep:
        rows = raw_rows(rep)
        md += [f"## `ncu --set full` capture `{rep.split('/')[-1]}`", ""]
        cols = list(rows[0].keys()) if rows else ["kernel"]
        md.append("| " + " | ".join(cols) + " |")
        md.append("|" + "---|" * len(cols))
        for r in rows:
            md.append("| " + " | ".join(str(r.get(c, "")) for c in cols) + " |")
        md.append("")
    open(a.out, "w").write("\n".join(md) + "\n")
    print(a.out)


if __name__ == "__main__":
    main()
