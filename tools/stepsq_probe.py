#!/usr/bin/env python
"""GB/s of the STEP_SUMSQ reading (Q1: sum_t ||g_t,l||^2, s_g bytes per element,
no Delta) next to the Delta interval end, bf16 and fp32, 2^28 elements, one
GPU.  STEP_SUMSQ bf16 streams 4e12 elements/s at 8 TB/s: the fp32 -> fp64
widening + DFMA per element may bound it before HBM does."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import paper_2102_01386_b200 as af
    from afinputs import uniform_layout
    torch.cuda.set_device(0)
    n = 1 << 28
    lay = uniform_layout(n, 24)
    for dt, s_g in (("bf16", 2), ("f32", 4)):
        g = (torch.randn(n, device="cuda") * 1e-3).to(torch.bfloat16 if dt == "bf16" else torch.float32)
        for acc, by in (("step_sumsq", s_g), ("delta", s_g + 4)):
            fm = af.FreezingModule(lay.offsets, lay.kinds, grad_dtype=dt, acc_mode=acc)
            fm.layer_norms(g)
            fm.layer_norms(g, interval_end=True)
            fm.update_and_decide()
            fm.layer_norms(g)                       # armed
            torch.cuda.synchronize()
            reps = 30
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda._sleep(5_000_000)
            a.record()
            for _ in range(reps):
                if acc == "delta":
                    fm.layer_norms(g, interval_end=True, dry_run=True)
                else:
                    fm.layer_norms(g, dry_run=True)
            b.record()
            b.synchronize()
            us = a.elapsed_time(b) / reps * 1e3
            print(json.dumps({"dtype": dt, "acc_mode": acc, "kernel": "kStepSq" if acc != "delta" else "kEndDelta",
                              "us": round(us, 2), "bytes_per_elem": by,
                              "gbs": round(n * by / (us * 1e-6) / 1e9, 1),
                              "elems_per_s": round(n / (us * 1e-6) / 1e12, 3)}), flush=True)
            del fm
        del g
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
