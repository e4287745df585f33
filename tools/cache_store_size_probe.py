"""Cache get time per call vs store size (5k / 25k / 100k records of 196,608 B, same batch): checks whether the per-call floor is TLB reach.  python tools/cache_store_size_probe.py"""
import json, statistics, sys, os
sys.path.insert(0, os.getcwd())
import torch
import paper_2102_01386_b200 as af
torch.cuda.set_device(0)
rb = 196_608
flush = torch.ones(256 << 20, dtype=torch.float16, device="cuda")
acc = torch.zeros((), dtype=torch.float32, device="cuda")
out = {}
for num in (5_000, 25_000, 100_000):
    c = af.ActivationCache(num, rb)
    src_all = torch.randint(0, 256, (4096, rb), dtype=torch.uint8, device="cuda")
    for b0 in range(0, num, 4096):
        ids = torch.arange(b0, min(num, b0 + 4096), device="cuda")
        c.put(ids, src_all[: ids.numel()], 4)
    res = {}
    for B in (32, 256):
        reps = 20
        id_sets = [torch.randperm(num, device="cuda")[:B].contiguous() for _ in range(reps)]
        dst = torch.empty(B, rb, dtype=torch.uint8, device="cuda")
        dep = torch.empty(B, dtype=torch.int32, device="cuda")
        def cap(w):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                for r in range(reps):
                    torch.sum(flush, dim=0, dtype=torch.float32, out=acc)
                    if w:
                        c.get(id_sets[r], 4, dst, dep)
            return g
        gs = {True: cap(True), False: cap(False)}
        t = {True: [], False: []}
        for _ in range(7):
            for w in (True, False):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(); gs[w].replay(); b.record(); torch.cuda.synchronize()
                t[w].append(a.elapsed_time(b))
        res[str(B)] = round((statistics.median(t[True]) - statistics.median(t[False])) / reps * 1e3, 2)
    out[str(num)] = res
    del c
    torch.cuda.empty_cache()
print(json.dumps(out))
