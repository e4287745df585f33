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
    # active-suffix shards (per-f tables): two ranks, bf16, boundary moved by a restore
    fa = [af.FreezingModule(lay.offsets, lay.kinds, grad_dtype="bf16", rank=r, world=2, shard_active=True)
          for r in range(2)]
    for f in fa:
        f.set_peers_local(fa)
    gh = g.to(torch.bfloat16)
    for T in range(3):
        if T == 1:
            for f in fa:
                blob = bytearray(f.get_state())
                blob[24:28] = (2).to_bytes(4, "little")
                f.set_state(bytes(blob))
        for f, s in zip(fa, ss):
            with torch.cuda.stream(s):
                f.layer_norms(gh, stream=s)
                f.interval_end(gh, stream=s)
        torch.cuda.synchronize()
    # wide finalize (> 2048 interval-end tiles)
    big = uniform_layout(2100 * 8192 + 77, 7, pre=4099, head=33)
    fw = af.FreezingModule(big.offsets, big.kinds, grad_dtype="f32")
    assert fw.info()["n_fin_chunks"] > 1
    gb = torch.randn(big.n, device="cuda") * 1e-3
    fw.layer_norms(gb)
    fw.interval_end(gb)
    fw.layer_norms(gb)
    fw.interval_end(gb)
    # fused reduce-scatter: P = 1 (plain and with AdamW), then P = 2 ranks in this process
    r1 = af.FreezingModule(lay.offsets, lay.kinds, grad_dtype="bf16")
    gr = (torch.randn(lay.n, device="cuda") * 1e-3).to(torch.bfloat16)
    r1.set_grad_peers_local([gr])
    out = torch.empty(lay.n, device="cuda")
    r1.reduce_scatter_step(out)
    r1.reduce_scatter_step(out, interval_end=True)
    p1 = torch.zeros(lay.n, device="cuda")
    m1, v1 = torch.zeros_like(p1), torch.zeros_like(p1)
    r1.reduce_scatter_adamw_step(p1, m1, v1, lr=1e-3, step=1, out=out)
    r1.reduce_scatter_adamw_step(p1, m1, v1, lr=1e-3, step=2, interval_end=True)
    rs = [af.FreezingModule(lay.offsets, lay.kinds, grad_dtype="f32", rank=r, world=2) for r in range(2)]
    gg = [torch.randn(lay.n, device="cuda") * 1e-3 for _ in range(2)]
    for f in rs:
        f.set_peers_local(rs)
        f.set_grad_peers_local(gg)
        f.set_max_ctas(8)
    outs = [torch.empty(lay.n, device="cuda") for _ in range(2)]
    torch.cuda.synchronize()
    for end in (False, True):
        for f, s, o in zip(rs, ss, outs):
            with torch.cuda.stream(s):
                f.reduce_scatter_step(o, interval_end=end, stream=s)
        torch.cuda.synchronize()
    # sticky bits: 0 unless the tool serialised the two ranks' kernels (barrier timeouts)
    print("reduce-scatter sticky", [int(f.scratch[8:12].view(torch.int32).item()) for f in rs], flush=True)
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
    # global (NEXT 4): two ranks' stores in one process, any id from any rank;
    # get_async on a side stream
    cs = [af.ActivationCache(100, 2048 + 16, rank=r, world=2) for r in range(2)]
    for c in cs:
        c.set_peers_local(cs)
    ids = torch.from_numpy(np.random.default_rng(1).permutation(100)[:40]).cuda()
    rows = torch.randint(0, 256, (40, 2048 + 16), dtype=torch.uint8, device="cuda")
    out = torch.empty_like(rows)
    dep = torch.empty(40, dtype=torch.int32, device="cuda")
    cs[0].put_global(ids, rows, 2)
    cs[1].get_global(ids, 3, out, dep)
    s = torch.cuda.Stream()
    c = af.ActivationCache(100, 2048 + 16)
    c.put(ids, rows, 2)
    c.get_async(ids, 2, out, dep, s)
    torch.cuda.synchronize()
    # round 2: disk tier (host callbacks), overlapped get over a committed interval end,
    # the cache get fused into the consumer GEMM (TMA + tcgen05, clusters of two)
    t = af.ActivationCache(100, 2048 + 16, hbm_rows=10, host_rows=10, disk_rows=30, stage_rows=16)
    t.put(ids, rows, 2)
    t.get(ids, 3, out, dep)
    fm1 = af.FreezingModule(lay.offsets, lay.kinds, grad_dtype="f32")
    g1 = torch.randn(lay.n, device="cuda") * 1e-3
    fm1.layer_norms(g1)
    fm1.interval_end(g1, copy_record=False)
    c.get(ids, 2, out, dep, overlap_prev=True)
    fm1.layer_norms(g1)
    if os.environ.get("AF_SANITIZE_TOOL") != "racecheck":
        # racecheck reports the pair-wide tcgen05.alloc.cta_group::2 writing the TMEM
        # address into both CTAs' shared memory (a write from outside the CTA's
        # instruction stream, same value) as a hazard against the CTA's own alloc;
        # memcheck (and synccheck) cover this kernel, racecheck the rest
        gc = af.ActivationCache(64, 128 * 128 * 2)
        gids = torch.arange(0, 20, dtype=torch.int64, device="cuda")
        grows = torch.randn(20, 128 * 128, device="cuda").to(torch.bfloat16)
        gc.put(gids, grows.view(torch.uint8), 2)
        w = torch.randn(96, 128, device="cuda").to(torch.bfloat16)
        y = torch.zeros(22 * 128, 96, dtype=torch.bfloat16, device="cuda")
        gdep = torch.empty(22, dtype=torch.int32, device="cuda")
        gc.get_gemm(torch.arange(0, 22, dtype=torch.int64, device="cuda"), 3, w, y, gdep, 128)
    torch.cuda.synchronize()
    print("sanitize probe done")


if __name__ == "__main__":
    main()
