#!/usr/bin/env python
"""Break the interval-end + decide cost into its parts (GPU box):
END kernel alone, decide kernel alone, fused call, with and without the mapped
host record, for a few buffer sizes.  Prints one JSON line per case."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import paper_2102_01386_b200 as af
    from afinputs import bert_layout, uniform_layout
    torch.cuda.set_device(0)
    cases = [("bert-large-f32", bert_layout("large"), "f32"), ("bert-base-bf16", bert_layout("base"), "bf16"),
             ("uniform-16M-f32", uniform_layout(1 << 24, 24, pre=1 << 20, head=1 << 16), "f32"),
             ("uniform-1M-f32", uniform_layout(1 << 20, 24), "f32")]
    for name, lay, dt in cases:
        tdt = torch.bfloat16 if dt == "bf16" else torch.float32
        g = torch.randn(lay.n, device="cuda").to(tdt) * 1e-3
        fm = af.FreezingModule(lay.offsets, lay.kinds, grad_dtype=dt)
        fm.layer_norms(g)
        fm.interval_end(g)
        fm.layer_norms(g)
        reps = 100
        out = {"case": name}

        def timeit(fn):
            for _ in range(5):
                fn()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(reps):
                fn()
            b.record()
            torch.cuda.synchronize()
            return a.elapsed_time(b) / reps * 1e3

        out["end_kernel_us"] = timeit(lambda: fm.layer_norms(g, interval_end=True, dry_run=True))
        out["end_plus_decide_us"] = timeit(lambda: (fm.layer_norms(g, interval_end=True, dry_run=True),
                                                    fm.update_and_decide(dry_run=True)))
        out["end_plus_decide_norecord_us"] = timeit(lambda: (fm.layer_norms(g, interval_end=True, dry_run=True),
                                                             fm.update_and_decide(dry_run=True, copy_record=False)))
        out["fused_us"] = timeit(lambda: fm.interval_end(g, dry_run=True))
        out["fused_norecord_us"] = timeit(lambda: fm.interval_end(g, dry_run=True, copy_record=False))
        out["accumulate_us"] = timeit(lambda: fm.layer_norms(g, dry_run=True))
        s_g = 2 if dt == "bf16" else 4
        out["ideal_end_us_at_6455GBs"] = lay.n * (s_g + 4) / 6455.3e9 * 1e6
        print(json.dumps({k: (round(v, 2) if isinstance(v, float) else v) for k, v in out.items()}), flush=True)
        del fm, g
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
