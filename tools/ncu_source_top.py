#!/usr/bin/env python
"""Top warp-stall sites of one kernel from `ncu -i REP --page source --csv
--print-source sass` (SASS with per-instruction stall samples), as markdown:
each site with the instructions leading up to it, so the waiting instruction
(try_wait loop, barrier, memory op) is visible.

    python tools/ncu_source_top.py gpurun_out/x_source.csv [--top 12] [--ctx 4] > profiles/.../x_source_top.md
"""
import argparse
import csv
import gzip


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--top", type=int, default=12)
    ap.add_argument("--ctx", type=int, default=4)
    a = ap.parse_args()
    op = gzip.open if a.csv.endswith(".gz") else open
    rows = list(csv.reader(op(a.csv, "rt")))
    kernel = rows[0][1] if len(rows[0]) > 1 else "?"
    h, data = rows[1], rows[2:]
    isrc, isamp, iex = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
    samp = [int(r[isamp]) if r[isamp].isdigit() else 0 for r in data]
    tot = sum(samp)
    print(f"# ncu source-level stall samples: `{kernel[:120]}`\n")
    print(f"{tot} samples over {len(data)} SASS instructions; top {a.top} sites (share of all samples), "
          f"with the {a.ctx} instructions before each.\n")
    for i in sorted(range(len(data)), key=lambda k: -samp[k])[:a.top]:
        print(f"## {samp[i]} samples ({100.0 * samp[i] / max(tot, 1):.1f} %)\n\n```")
        for j in range(max(0, i - a.ctx), i + 1):
            print(f"{samp[j]:>6} {data[j][iex]:>9}  {data[j][isrc].strip()[:100]}")
        print("```\n")


if __name__ == "__main__":
    main()
