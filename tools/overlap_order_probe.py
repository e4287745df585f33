"""Does a kernel behind an AF_CACHE_OVERLAP_PREV get start before the interval
end in front of the get has finished?  (ordering of the
overlapped get.)

Needs a build with -DAF_TIMING=1 (the streaming kernels stamp %globaltimer into
the device state: tmark[0] = start of the kernel's work after its dependency
wait, tmark[3] = end of the interval end's last-CTA tail).  Sequence per trial:
accumulate, interval end (its last CTA busy-waits DELAY before the tail,
AF_DEBUG_TAIL_DELAY_NS), overlapped get, accumulate.  Prints, per trial, the
second accumulate's start minus the interval end's tail end: negative = the
accumulate passed its griddepcontrol.wait while the interval end was still
committing (the race), positive = ordered.

    AF_NVCC_EXTRA="-DAF_TIMING=1 [-DAF_CACHE_OVERLAP_UNSAFE]" python tools/overlap_order_probe.py
"""
import json
import os
import struct
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import importlib.util
    spec = importlib.util.spec_from_file_location("b", os.path.join(ROOT, "paper_2102_01386_b200", "_build.py"))
    b = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(b)
    b.build(verbose=False)
    import torch

    import paper_2102_01386_b200 as af
    from paper_2102_01386_b200 import _lib as L
    from afinputs import uniform_layout
    torch.cuda.set_device(0)
    lay = uniform_layout(1 << 24, 8, pre=1 << 20, head=4096)
    fm = af.FreezingModule(lay.offsets, lay.kinds, grad_dtype="f32")
    g = torch.randn(lay.n, device="cuda") * 1e-3
    cache = af.ActivationCache(1000, 4096)
    ids = torch.arange(256, dtype=torch.int64, device="cuda")
    rows = torch.zeros((256, 4096), dtype=torch.uint8, device="cuda")
    cache.put(ids, rows, 1)
    out = torch.empty_like(rows)
    dep = torch.empty(256, dtype=torch.int32, device="cuda")
    delay_ns = int(os.environ.get("DELAY_NS", "2000000"))
    fm.set_debug(L.AF_DEBUG_TAIL_DELAY_NS, delay_ns)
    res = []
    for trial in range(6):
        torch.cuda.synchronize()
        fm.layer_norms(g)
        fm.interval_end(g, copy_record=False)
        cache.get(ids, 1, out, dep, overlap_prev=True)
        fm.layer_norms(g)
        torch.cuda.synchronize()
        raw = fm.scratch[:64].cpu().numpy().tobytes()
        t0, t1, t2, t3 = struct.unpack_from("<4Q", raw, 24)
        res.append({"acc_start_minus_tail_end_us": (t0 - t3) / 1e3, "tail_us": (t3 - t1) / 1e3})
    print(json.dumps({"flags": os.environ.get("AF_NVCC_EXTRA", ""), "delay_ns": delay_ns, "trials": res}))


if __name__ == "__main__":
    main()
