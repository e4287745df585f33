#!/usr/bin/env python
"""Cache put/get by batch size with a COLD L2 (run on the GPU box).

Each repetition draws fresh random ids and is preceded by a read of a 512 MB
buffer, so the rows, the records and the meta words come from HBM as inside the
bench's step (whose interval end streams >= 0.6 GB through the 126 MB L2 just
before the get).  A call's cost is marginal device time: a CUDA graph of R x
[flush, call] minus a graph of R x [flush], divided by R -- calls launch back to
back as in the step's graph, with no event between them (an event pair around a
single call adds a ~6 us floor on this box: `null` timed that way measured
6.1 us, profiles/r01_v33_cache_cold_events.jsonl).  `null` is a 4-byte torch
kernel timed the same way.

    python tools/cache_cold_probe.py                      # current build, one JSON line
    python tools/cache_cold_probe.py --variants a b ...   # rebuild per variant (flags in VARIANTS)
"""
import argparse
import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

VARIANTS = {   # the two-warp speculative kernel is the default since v34 (the old one-warp kernel is gone)
    "default": "",
    "s4": "-DAF_CACHE_STAGES=4",
    "3cta_s2": "-DAF_CACHE_CTAS_PER_SM=3 -DAF_CACHE_STAGES=2",
    "16k_s6": "-DAF_CACHE_CHUNK=16384 -DAF_CACHE_STAGES=6",
    "16k_s5": "-DAF_CACHE_CHUNK=16384 -DAF_CACHE_STAGES=5",
    "16k_s6_1cta": "-DAF_CACHE_CHUNK=16384 -DAF_CACHE_STAGES=6 -DAF_CACHE_CTAS_PER_SM=1",
    "32k_s6_1cta": "-DAF_CACHE_STAGES=6 -DAF_CACHE_CTAS_PER_SM=1",
}
BATCHES = (6, 32, 64, 128, 256, 1024, 4096)


def probe(reps=20):
    import torch

    import paper_2102_01386_b200 as af
    torch.cuda.set_device(0)
    rb, num = 196_608, 100_000
    c = af.ActivationCache(num, rb)
    src_all = torch.randint(0, 256, (max(BATCHES), rb), dtype=torch.uint8, device="cuda")
    for b0 in range(0, num, 4096):   # populate every record at depth 4 (gets hit, never evict)
        ids = torch.arange(b0, min(num, b0 + 4096), device="cuda")
        c.put(ids, src_all[: ids.numel()], 4)
    flush = torch.ones(256 << 20, dtype=torch.float16, device="cuda")
    acc = torch.zeros((), dtype=torch.float32, device="cuda")
    tiny = torch.zeros(1, dtype=torch.int32, device="cuda")
    out = {}

    def flush_read():   # reads 512 MB: clean lines, like the interval end before the step's get
        torch.sum(flush, dim=0, dtype=torch.float32, out=acc)

    def timed(fn_for_rep, iters=7):
        # marginal device time per call: a graph of R x [flush, call] minus a graph of
        # R x [flush] -- no event in between calls, launches back to back as in the step
        def cap(with_call):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                for r in range(reps):
                    flush_read()
                    if with_call:
                        fn_for_rep(r)
            return g
        gs = {True: cap(True), False: cap(False)}
        t = {True: [], False: []}
        for _ in range(iters):
            for w in (True, False):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                gs[w].replay()
                b.record()
                torch.cuda.synchronize()
                t[w].append(a.elapsed_time(b))
        return (statistics.median(t[True]) - statistics.median(t[False])) / reps * 1e3   # us

    out["null_us"] = round(timed(lambda r: tiny.add_(1)), 2)
    for B in BATCHES:
        id_sets = [torch.randperm(num, device="cuda")[:B].contiguous() for _ in range(reps)]
        src = src_all[:B]
        dst = torch.empty_like(src)
        dep = torch.empty(B, dtype=torch.int32, device="cuda")
        res = {}
        for name, fn in (("put", lambda r: c.put(id_sets[r], src, 4)),
                         ("get", lambda r: c.get(id_sets[r], 4, dst, dep)),
                         ("get+put", lambda r: (c.get(id_sets[r], 4, dst, dep), c.put(id_sets[r], src, 4)))):
            us = timed(fn)
            nbytes = 2 * B * rb * (2 if name == "get+put" else 1)
            res[name] = {"us": round(us, 2), "gbs": round(nbytes / (us * 1e-6) / 1e9, 1)}
        torch.cuda.synchronize()
        assert bool((dep == 4).all()), "cold probe: every get must hit at depth 4"
        out[str(B)] = res
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--variants", nargs="*")
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    if not a.variants:
        print(json.dumps(probe(a.reps)), flush=True)
        return
    for v in a.variants:
        env = dict(os.environ, AF_NVCC_EXTRA=VARIANTS[v])
        b = subprocess.run([sys.executable, "-c", "import __graft_entry__ as g; g._builder().build()"], cwd=ROOT,
                           env=env, capture_output=True, text=True)
        if b.returncode:
            print(json.dumps({"variant": v, "flags": VARIANTS[v], "err": b.stderr[-800:]}), flush=True)
            continue
        r = subprocess.run([sys.executable, os.path.abspath(__file__), "--reps", str(a.reps)], cwd=ROOT, env=env,
                           capture_output=True, text=True)
        line = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else "{}"
        print(json.dumps({"variant": v, "flags": VARIANTS[v], "probe": json.loads(line), "err": r.stderr[-400:]}),
              flush=True)
    subprocess.run([sys.executable, "-c", "import __graft_entry__ as g; g._builder().build()"], cwd=ROOT,
                   env=dict(os.environ, AF_NVCC_EXTRA=""))


if __name__ == "__main__":
    main()
