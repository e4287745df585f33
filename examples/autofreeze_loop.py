#!/usr/bin/env python
"""AutoFreeze's training-loop integration, end to end on synthetic data.

What a fine-tuning loop does with this library (Fig. 7, §3.4):
  * every iteration: the backward produces the flat gradient of the ACTIVE layers;
    `fm.adamw_step(...)` updates the parameters and accumulates Delta in one pass
    (or `fm.layer_norms(grad)` next to your own optimizer);
  * every k/5 iterations: the same call with interval_end=True runs the
    gradient-norm test (Eq. 1, Alg. 1) and publishes the frozen prefix f;
    the loop then stops computing gradients for the first f blocks and the
    embedding (requires_grad=False);
  * from the epoch after a freeze: the storage manager caches the frozen prefix's
    output per ORIGINAL example id (MappingShuffled_i), read back with
    evict-on-read when f has grown, and only when caching beats
    recomputing.
Gradients here are synthetic (afinputs recipe: per-layer scale decaying with a
layer-dependent rate, so lower blocks converge first, as in Fig. 5).

    python examples/autofreeze_loop.py [--epochs 4] [--small]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run(epochs=4, small=False, seed=0, verbose=True):
    import numpy as np
    import torch

    import paper_2102_01386_b200 as af
    from afinputs import bert_layout, epoch_permutation, uniform_layout

    torch.cuda.set_device(0)
    lay = uniform_layout(2_000_000, 12, pre=300_000, head=20_000) if small else bert_layout("base")
    n_examples, batch, hidden_bytes = (2_000, 50, 4096) if small else (25_000, 32, 128 * 768 * 2)
    iters_per_epoch = n_examples // batch
    interval = max(1, iters_per_epoch // 5)                       # 5 evaluation intervals per epoch
    fm = af.FreezingModule(lay.offsets, lay.kinds, grad_dtype="bf16")
    cache = af.ActivationCache(n_examples, hidden_bytes)
    params = torch.zeros(lay.n, device="cuda")
    m, v = torch.zeros_like(params), torch.zeros_like(params)
    seg_len = torch.tensor([lay.seg_len(l) for l in range(lay.n_segments)], device="cuda")
    rate = torch.tensor(np.linspace(0.55, 0.97, lay.n_segments), device="cuda", dtype=torch.float32)
    rng = torch.Generator(device="cuda")
    rng.manual_seed(seed)
    # both sides of the cache-vs-recompute rule measured here: one block's
    # forward (a BERT-base-shaped stand-in: 768 -> 3072 -> 768 on batch x 128 tokens)
    # and one batch's cache read
    tokens = batch * (16 if small else 128)
    x = torch.randn(tokens, 768, device="cuda", dtype=torch.bfloat16)
    w1 = torch.randn(3072, 768, device="cuda", dtype=torch.bfloat16) * 0.02
    w2 = torch.randn(768, 3072, device="cuda", dtype=torch.bfloat16) * 0.02
    cal = af.calibrate_should_cache(lambda: torch.nn.functional.linear(torch.nn.functional.gelu(
        torch.nn.functional.linear(x, w1)), w2), hidden_bytes, batch, max_layers=lay.n_segments)
    t_layer, t_read = cal["t_layer_fwd_s"], cal["t_batch_read_s"]
    if verbose:
        print(f"calibrated: block forward {t_layer * 1e6:.0f} us, batch read {t_read * 1e6:.0f} us, caching pays "
              f"from {cal['min_frozen_layers']} frozen blocks")
    # the first active block's QKV projection (768 -> 2304); with 128 x 768 bf16 records the
    # cached rows feed it straight from the store (NEXT 4: no batch copy)
    fused_gemm = hidden_bytes == 128 * 768 * 2
    w_qkv = torch.randn(2304, 768, device="cuda", dtype=torch.bfloat16) * 0.02
    qkv = torch.empty(batch * 128, 2304, device="cuda", dtype=torch.bfloat16) if fused_gemm else None
    frozen, trace, hits = 0, [], 0
    step = 0
    for epoch in range(epochs):
        order = epoch_permutation(seed, epoch, np.arange(n_examples))        # MappingShuffled_epoch
        for it in range(iters_per_epoch):
            step += 1
            ids = torch.from_numpy(order[it * batch:(it + 1) * batch]).cuda()
            # storage manager: read cached frozen-prefix outputs, recompute the rest
            rows = torch.empty((batch, hidden_bytes), dtype=torch.uint8, device="cuda")
            depth = torch.empty(batch, dtype=torch.int32, device="cuda")
            use_cache = frozen > 0 and af.should_cache(frozen, t_layer, t_read)
            if use_cache:
                if fused_gemm:   # get + the first active layer's projection in one kernel
                    cache.get_gemm(ids, frozen, w_qkv, qkv, depth, 128)
                else:
                    cache.get(ids, frozen, rows, depth)
                hits += int((depth >= 0).sum())
            # ... forward from each example's depth, backward through the active blocks ...
            decay = rate ** (step / interval)
            sigma = torch.repeat_interleave(1e-3 * (0.2 + decay), seg_len)
            grad = (torch.rand(lay.n, generator=rng, device="cuda") * 2 - 1).mul_(sigma).to(torch.bfloat16)
            end = step % interval == 0
            fm.adamw_step(params, m, v, grad, lr=1e-5, step=step, weight_decay=0.01, interval_end=end)
            if use_cache:
                miss = ids[depth < 0]
                if miss.numel():
                    cache.put(miss, rows[: miss.numel()], frozen)            # layer-f outputs at depth f
            if end:
                d = fm.decision()
                if d["boundary_after"] != frozen and verbose:
                    print(f"epoch {epoch} iter {it}: interval {d['interval']} froze blocks "
                          f"[{frozen}, {d['boundary_after']}) threshold {d['threshold']:.4g}")
                frozen = d["boundary_after"]
                trace.append(frozen)
    if verbose:
        print("frozen prefix after each interval:", trace)
        print("cache hits:", hits, "stats:", cache.stats())
    return trace, hits


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--epochs", type=int, default=4)
    ap.add_argument("--small", action="store_true")
    a = ap.parse_args()
    run(a.epochs, a.small)
