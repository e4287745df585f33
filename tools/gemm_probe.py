"""NEXT 4 probe: the cache get fused into the consumer GEMM (af_cache_get_gemm)
against the unfused pair (af_cache_get into a batch buffer, then torch.matmul =
cuBLAS bf16), on one rank's partition of the C4 cache (12,500 records of 128 x
768 bf16 = 2.46 GB, so every record read is cold in L2), B examples per call,
BERT-base's QKV projection (N = 2304, K = 768).  Each timing is a CUDA graph of
R calls on fresh random ids (all hits, boundary = depth: no eviction), median of
rounds.  TFLOP/s = 2 B 128 768 N / t.

    python tools/gemm_probe.py [--batches 32 256] [--reps 20]
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def probe(batches=(32, 256), reps=20, rounds=5, N=2304, K=768, rows=128, world=8):
    import torch

    import paper_2102_01386_b200 as af
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    num = 100_000
    rb = rows * K * 2
    cache = af.ActivationCache(num, rb, rank=0, world=world, device=dev)
    mine = torch.arange(0, num, world, device=dev, dtype=torch.int64)
    g = torch.Generator(device=dev)
    g.manual_seed(1)
    for b0 in range(0, mine.numel(), 2048):
        ids = mine[b0:b0 + 2048]
        rows_b = torch.randn(ids.numel(), rows * K, device=dev, generator=g).mul_(0.5).to(torch.bfloat16)
        cache.put(ids, rows_b.view(torch.uint8), 4)
    w = (torch.randn(N, K, device=dev, generator=g) * 0.05).to(torch.bfloat16)
    out = {"N": N, "K": K, "rows_per_record": rows, "store_rows": mine.numel(), "reps": reps}
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    for B in batches:
        id_sets = [mine[torch.randperm(mine.numel(), device=dev, generator=g)[:B]].contiguous() for _ in range(reps)]
        y = torch.empty(B * rows, N, dtype=torch.bfloat16, device=dev)
        dep = torch.empty(B, dtype=torch.int32, device=dev)
        buf = torch.empty(B, rb, dtype=torch.uint8, device=dev)

        def fused(r):
            cache.get_gemm(id_sets[r], 4, w, y, dep, rows)

        def unfused(r):
            cache.get(id_sets[r], 4, buf, dep)
            torch.matmul(buf.view(torch.bfloat16).view(B * rows, K), w.t(), out=y)

        def gemm_only(r):
            torch.matmul(buf.view(torch.bfloat16).view(B * rows, K), w.t(), out=y)

        res = {}
        for name, fn in (("fused_get_gemm", fused), ("get_then_cublas", unfused), ("cublas_gemm_only", gemm_only)):
            for r in range(2):
                fn(r)
            gph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gph):
                for r in range(reps):
                    fn(r)
            ts = []
            for _ in range(rounds):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                a.record()
                gph.replay()
                b.record()
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b) / reps * 1e3)
            us = statistics.median(ts)
            tf = 2 * B * rows * K * N / (us * 1e-6) / 1e12
            res[name] = {"us": round(us, 2), "tflops": round(tf, 1)}
            if peaks.get("bf16_tflops"):
                res[name]["frac_of_bf16_peak"] = round(tf / peaks["bf16_tflops"], 4)
        # correctness spot check of the fused path against the unfused one
        fused(0)
        ref = torch.empty_like(y)
        cache.get(id_sets[0], 4, buf, dep)
        torch.matmul(buf.view(torch.bfloat16).view(B * rows, K), w.t(), out=ref)
        torch.cuda.synchronize()
        res["max_abs_diff_vs_cublas"] = float((y.float() - ref.float()).abs().max())
        res["speedup_vs_unfused"] = round(res["get_then_cublas"]["us"] / res["fused_get_gemm"]["us"], 3)
        out[str(B)] = res
    return out


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--batches", type=int, nargs="+", default=[32, 256])
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    print(json.dumps(probe(tuple(a.batches), a.reps)))
