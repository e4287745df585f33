#!/usr/bin/env python
"""Cache put/get GB/s (2 x rows x row_bytes per call) by batch size, one JSON line."""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import paper_2102_01386_b200 as af
    torch.cuda.set_device(0)
    rb, num = 196_608, 20_000
    c = af.ActivationCache(num, rb)
    src_all = torch.randint(0, 256, (4096, rb), dtype=torch.uint8, device="cuda")
    out = {}
    for B in (6, 32, 48, 256, 1024, 4096):
        ids = torch.randperm(num, device="cuda")[:B].contiguous()
        src = src_all[:B]
        dst = torch.empty_like(src)
        dep = torch.empty(B, dtype=torch.int32, device="cuda")
        c.put(ids, src, 4)
        res = {}
        for name, fn in (("put", lambda: c.put(ids, src, 4)), ("get", lambda: c.get(ids, 4, dst, dep))):
            # queue every rep behind a ~2.5 ms sleep kernel: the events then time the
            # device, not the host's launch latency (which dominates tiny batches)
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(20)]
            torch.cuda.synchronize()
            torch.cuda._sleep(5_000_000)
            for a, b in ev:
                a.record()
                fn()
                b.record()
            torch.cuda.synchronize()
            ms = statistics.median(a.elapsed_time(b) for a, b in ev)
            res[name] = round(2 * B * rb / (ms * 1e-3) / 1e9, 1)
        out[B] = res
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
