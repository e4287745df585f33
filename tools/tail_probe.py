#!/usr/bin/env python
"""With an AF_TIMING build: split the interval-end kernel's time into the
streaming part, the last CTA's per-segment sums and the decision
(%globaltimer marks written into the device state)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch

    import paper_2102_01386_b200 as af
    from afinputs import bert_layout, uniform_layout
    torch.cuda.set_device(0)
    for name, lay, dt in (("bert-large-f32", bert_layout("large"), "f32"), ("bert-base-bf16", bert_layout("base"), "bf16"),
                          ("uniform-268M-1seg-f32", uniform_layout(1 << 28, 1), "f32"),
                          ("uniform-268M-24seg-f32", uniform_layout(1 << 28, 24), "f32")):
        tdt = torch.bfloat16 if dt == "bf16" else torch.float32
        g = (torch.randn(lay.n, device="cuda") * 1e-3).to(tdt)
        fm = af.FreezingModule(lay.offsets, lay.kinds, grad_dtype=dt)
        fm.layer_norms(g)
        fm.interval_end(g)
        fm.layer_norms(g)
        marks = []
        for _ in range(10):
            fm.interval_end(g, dry_run=True)
            torch.cuda.synchronize()
            raw = fm.scratch[:64].cpu().numpy().view(np.uint64)
            t = raw[3:7].astype(np.int64)   # tmark after T,f,sticky,pad (16 B) + epoch (8 B)
            marks.append((t[1] - t[0], t[2] - t[1], t[3] - t[2]))
        m = np.median(np.array(marks), axis=0) / 1e3
        print(json.dumps({"case": name, "stream_us": round(float(m[0]), 2), "segment_sums_us": round(float(m[1]), 2),
                          "decide_us": round(float(m[2]), 2), "n_tiles": fm.info()["n_tiles"],
                          "n_fin_ctas": fm.info()["n_fin_ctas"]}), flush=True)
        del fm, g
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
