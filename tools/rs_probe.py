#!/usr/bin/env python
"""Fused reduce-scatter (af_reduce_scatter_step) with P in-process ranks on one
GPU: per-step sticky flags (bit 0: exchange timeout, bit 1: barrier timeout)
and the per-step device time of all ranks' kernels (co-resident on one GPU, so
the "peer" reads are local HBM reads: a functional probe, not an NVLink number).

    python tools/rs_probe.py [--P 2] [--n 72000006] [--segments 40] [--dtype bf16]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch

    import paper_2102_01386_b200 as af
    from afinputs import uniform_layout
    ap = argparse.ArgumentParser()
    ap.add_argument("--P", type=int, default=2)
    ap.add_argument("--n", type=int, default=72_000_006)
    ap.add_argument("--segments", type=int, default=40)
    ap.add_argument("--dtype", default="bf16")
    ap.add_argument("--max-ctas", type=int, default=0)
    ap.add_argument("--steps", type=int, default=6)
    a = ap.parse_args()
    torch.cuda.set_device(0)
    lay = uniform_layout(a.n, a.segments, pre=1_000_001, head=3_333)
    P = a.P
    fms = [af.FreezingModule(lay.offsets, lay.kinds, grad_dtype=a.dtype, rank=r, world=P) for r in range(P)]
    tdt = torch.bfloat16 if a.dtype == "bf16" else torch.float32
    grads = [(torch.randn(lay.n, device="cuda") * 1e-3).to(tdt) for _ in range(P)]
    for fm in fms:
        if P > 1:
            fm.set_peers_local(fms)
        fm.set_grad_peers_local(grads)
        fm.set_max_ctas(a.max_ctas or max(1, 120 // P))
    outs = [torch.zeros(fm.info()["shard_end"] - fm.info()["shard_begin"], device="cuda") for fm in fms]
    streams = [torch.cuda.Stream() for _ in range(P)]
    torch.cuda.synchronize()
    for k in range(a.steps):
        end = k % 2 == 1
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(P)]
        for fm, s, o, e in zip(fms, streams, outs, ev):
            with torch.cuda.stream(s):
                e[0].record(s)
                fm.reduce_scatter_step(o, interval_end=end, stream=s)
                e[1].record(s)
        torch.cuda.synchronize()
        sticky = [int(fm.scratch[8:12].view(torch.int32).item()) for fm in fms]
        rec = [fm.decision()["flags"] if end else None for fm in fms]
        print(json.dumps({"step": k, "end": end, "ms": [round(e[0].elapsed_time(e[1]), 3) for e in ev],
                          "sticky": sticky, "flags": rec, "n_fin_ctas": fms[0].info()["n_fin_ctas"]}), flush=True)


if __name__ == "__main__":
    main()
