#!/usr/bin/env python
"""A short pass over every kernel family for compute-sanitizer (memcheck /
racecheck / synccheck):
    compute-sanitizer --tool memcheck python tools/sanitize_probe.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch

    import paper_2102_01386_b200 as af
    from afinputs import uniform_layout
    torch.cuda.set_device(0)
    lay = uniform_layout(300_007, 5, pre=10_001, head=333)
    for dt in ("f32", "bf16"):
        tdt = torch.bfloat16 if dt == "bf16" else torch.float32
        fm = af.FreezingModule(lay.offsets, lay.kinds, grad_dtype=dt)
        for T in range(3):
            g = (torch.randn(lay.n, device="cuda") * 1e-3).to(tdt)
            fm.layer_norms(g)
            fm.interval_end(g)
            fm.layer_norms(g)
            fm.layer_norms(g, interval_end=True)
            fm.update_and_decide()
        p = torch.zeros(lay.n, device="cuda")
        m, v = torch.zeros_like(p), torch.zeros_like(p)
        fm.adamw_step(p, m, v, g, lr=1e-3, step=1)
        fm.adamw_step(p, m, v, g, lr=1e-3, step=2, interval_end=True)
        fm.decision()
        sq = af.FreezingModule(lay.offsets, lay.kinds, grad_dtype=dt, acc_mode="step_sumsq")
        sq.layer_norms(g)
        sq.interval_end(g)
    # two ranks on one GPU, in-kernel peer exchange
    fms = [af.FreezingModule(lay.offsets, lay.kinds, grad_dtype="f32", rank=r, world=2) for r in range(2)]
    for f in fms:
        f.set_peers_local(fms)
    ss = [torch.cuda.Stream() for _ in range(2)]
    g = torch.randn(lay.n, device="cuda") * 1e-3
    torch.cuda.synchronize()
    for f, s in zip(fms, ss):
        with torch.cuda.stream(s):
            f.interval_end(g, stream=s)
    torch.cuda.synchronize()
    # caches: direct and tiered
    for kw in ({}, {"hbm_rows": 30, "host_rows": 20}):
        c = af.ActivationCache(100, 4096 + 16, **kw)
        ids = torch.from_numpy(np.random.default_rng(0).permutation(100)[:64]).cuda()
        rows = torch.randint(0, 256, (64, 4096 + 16), dtype=torch.uint8, device="cuda")
        c.put(ids, rows, 2)
        out = torch.empty_like(rows)
        dep = torch.empty(64, dtype=torch.int32, device="cuda")
        c.get(ids, 3, out, dep)
        c.put(ids, rows, 3)
        c.stats()
    torch.cuda.synchronize()
    print("sanitize probe done")


if __name__ == "__main__":
    main()
