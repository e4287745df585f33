#!/usr/bin/env python
"""ZeRO-style data parallelism with the freezing hot path fused into the
gradient sync (include/af.h af_reduce_scatter_adamw_step).

One process per GPU.  Every rank keeps its FULL flat gradient in one persistent
buffer (what a DDP bucket would hold), registers it once, and then each step is
ONE kernel per rank: pull this rank's shard of every rank's gradient over
NVLink, average, AdamW on the shard's parameters / moments, accumulate Delta
(or, on the interval's last step, Eq. 1 + percentile + prefix freeze with the
per-layer sums exchanged between the GPUs inside the kernel).  The updated
parameter shards are then all-gathered by the caller (ZeRO-1).

    torchrun --nproc-per-node 8 --master-addr 127.0.0.1 examples/zero_loop.py
    python examples/zero_loop.py                       # world 1
Gradients are synthetic (afinputs recipe: per-layer scale decaying with a
layer-dependent rate).  On one GPU with AF_EXAMPLE_BACKEND=gloo several ranks
may share the device (time-sliced: functional only).
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run(intervals=10, steps_per_interval=4, small=True, verbose=True):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2102_01386_b200 as af
    from afinputs import bert_layout, uniform_layout

    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0)) % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group(os.environ.get("AF_EXAMPLE_BACKEND", "nccl"))
    lay = uniform_layout(4_000_000, 12, pre=400_000, head=20_000) if small else bert_layout("base")
    fm = af.FreezingModule(lay.offsets, lay.kinds, grad_dtype="bf16", rank=rank, world=world)
    grad = torch.zeros(lay.n, dtype=torch.bfloat16, device="cuda")     # this rank's persistent gradient
    if world > 1:
        assert fm.set_peers_ipc(), "CUDA IPC peer mappings unavailable"
        fm.set_grad_peers_ipc(grad)
    else:
        fm.set_grad_peers_local([grad])
    info = fm.info()
    assert (info["shard_begin"], info["shard_end"]) == shard_bounds(rank, world, lay.n)
    params = torch.zeros(lay.n, device="cuda")                         # full copy (ZeRO-1)
    m, v = torch.zeros_like(params), torch.zeros_like(params)          # only the shard is used
    seg_len = torch.tensor([lay.seg_len(l) for l in range(lay.n_segments)], device="cuda")
    rate = torch.tensor(np.linspace(0.55, 0.97, lay.n_segments), device="cuda", dtype=torch.float32)
    gen = torch.Generator(device="cuda")
    gen.manual_seed(1000 + rank)
    trace, k = [], 0
    for T in range(intervals):
        for t in range(steps_per_interval):
            k += 1
            # ... forward / backward of the active blocks writes `grad` ...
            sigma = torch.repeat_interleave(1e-3 * (0.2 + rate ** T), seg_len)
            grad.copy_(((torch.rand(lay.n, generator=gen, device="cuda") * 2 - 1) * sigma).to(torch.bfloat16))
            end = t == steps_per_interval - 1
            fm.reduce_scatter_adamw_step(params, m, v, lr=1e-4, step=k, weight_decay=0.01, interval_end=end)
            if world > 1:   # ZeRO-1: every rank gets the updated parameter shards (unequal sizes)
                for r in range(world):
                    lo, hi = shard_bounds(r, world, lay.n)
                    dist.broadcast(params[lo:hi], src=r)
        d = fm.decision()
        trace.append(d["boundary_after"])
        if verbose and rank == 0:
            print(f"interval {d['interval']}: frozen prefix {d['boundary_before']} -> {d['boundary_after']}, "
                  f"threshold {d['threshold']:.4g}, flags {d['flags']}", flush=True)
    if world > 1:
        dist.destroy_process_group()
    return trace


def shard_bounds(r, world, n):
    """Rank r's shard (the library's rule: floor(r*n/P) rounded down to 8; af_ctx_info)."""
    b = lambda q: n if q == world else (q * n // world) // 8 * 8  # noqa: E731
    return b(r), b(r + 1)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--intervals", type=int, default=10)
    ap.add_argument("--bert-base", action="store_true")
    a = ap.parse_args()
    run(a.intervals, small=not a.bert_base)
