"""Where does one interval end's time go at a per-rank shard size?

Needs an AF_TIMING=1 build (the kernels stamp %globaltimer into the device
state: tmark[0] = block 0 past its dependency wait, tmark[1] = the last CTA to
leave its tile loop, tmark[2] = after the segment sums + exchange, tmark[3] =
after the decision; dmark[0..6] = the decision's steps).  For each context, single dry-run interval ends (synchronised, event
pair around each) and a back-to-back series; prints per-phase medians in us.

    AF_NVCC_EXTRA="-DAF_TIMING=1" python tools/end_breakdown_probe.py
    AF_NVCC_EXTRA="-DAF_TIMING=1 -DAF_TIMING_FIRST=1" ...   # tmark[1] = the FIRST CTA out of tiles:
                                                           # stream_us then ends where the end phase starts
"""
import json
import os
import statistics
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
    from afinputs import bert_layout, uniform_layout
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    out = {"flags": os.environ.get("AF_NVCC_EXTRA", "")}
    lay8 = bert_layout("large")
    cases = []
    fms8 = [af.FreezingModule(lay8.offsets, lay8.kinds, grad_dtype="f32", rank=r, world=8, shard_active=True)
            for r in range(8)]
    for fm in fms8:
        fm.set_peers_local(fms8)
    fms8[0].set_debug(L.AF_DEBUG_PEERS_ARRIVED, 1)
    g8 = torch.randn(lay8.n, device=dev) * 1e-3
    cases.append(("bert-large rank0 of 8 (peers local)", fms8[0], g8))
    n1 = fms8[0].info()["shard_end"] - fms8[0].info()["shard_begin"]
    lay1 = uniform_layout(n1, 4)
    fm1 = af.FreezingModule(lay1.offsets, lay1.kinds, grad_dtype="f32")
    g1 = torch.randn(lay1.n, device=dev) * 1e-3
    cases.append((f"world 1, {n1} elements, 4 POOL", fm1, g1))
    lay2 = uniform_layout(1 << 28, 24)
    fm2 = af.FreezingModule(lay2.offsets, lay2.kinds, grad_dtype="f32")
    g2 = torch.randn(lay2.n, device=dev) * 1e-3
    cases.append(("world 1, 2^28 elements, 24 POOL", fm2, g2))
    for name, fm, g in cases:
        fm.layer_norms(g)
        fm.interval_end(g)
        fm.layer_norms(g)
        torch.cuda.synchronize()
        rows = []
        for _ in range(15):
            a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fm.interval_end(g, dry_run=True, copy_record=False)
            e.record()
            torch.cuda.synchronize()
            raw = fm.scratch[:2176].cpu().numpy().tobytes()
            t = struct.unpack_from("<4Q", raw, 24)
            dm = struct.unpack_from("<8Q", raw, 2112)   # DevState.dmark: the decision's steps
            row = {"event_us": a.elapsed_time(e) * 1e3, "stream_us": (t[1] - t[0]) / 1e3,
                   "sums_exchange_us": (t[2] - t[1]) / 1e3, "decide_us": (t[3] - t[2]) / 1e3,
                   "t0_to_t3_us": (t[3] - t[0]) / 1e3}
            names = ("d_loads", "d_eta", "d_sort", "d_thr", "d_scan", "d_records", "d_commit")
            ends = list(dm[1:7]) + [t[3]]
            for k, nm in enumerate(names):
                row[nm + "_us"] = (ends[k] - dm[k]) / 1e3
            row["last_chunk_us"] = (dm[7] - t[1]) / 1e3       # last tile done -> its chunk reduced + counted
            row["tail_sums_xchg_us"] = (t[2] - dm[7]) / 1e3   # pieces staged, segment sums, exchange
            rows.append(row)
        rows = rows[3:]
        med = {k: round(statistics.median(r[k] for r in rows), 2) for k in rows[0]}
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 50
        a.record()
        for _ in range(reps):
            fm.interval_end(g, dry_run=True, copy_record=False)
        e.record()
        torch.cuda.synchronize()
        med["back_to_back_us"] = round(a.elapsed_time(e) / reps * 1e3, 2)
        info = fm.info()
        n = info["shard_end"] - info["shard_begin"]
        med["n"] = n
        med["gbs_back_to_back"] = round(n * 8 / (med["back_to_back_us"] * 1e-6) / 1e9, 1)
        out[name] = med
    print(json.dumps(out))


if __name__ == "__main__":
    main()
