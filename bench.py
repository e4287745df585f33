#!/usr/bin/env python
"""Benchmark of the AutoFreeze freezing hot path on B200 (BASELINE.json metric:
"per-layer grad-norm+decide GB/s (% of HBM peak) at 1/2/4/8 B200; cache GB/s").

One step = one pass of every SURVEY.md §8(a) row over one batch of synthetic
input, through the C ABI:
  a2   af_layer_norms            Delta += g over the rank's shard    n_loc*(s_g+8) B
  a3-9 af_interval_end           fp64 sum of squares of Delta + g,   n_loc*(s_g+4) B
                                 Eq. 1, percentile, prefix scan, record (ONE kernel at N = 1;
                                 kernel + NCCL all-gather of the L partials + decide at N > 1)
  a11  af_cache_get              B rows by example id                 2*B*row B
  a10  af_cache_put              B rows by example id                 2*B*row B
Timed steps run under AF_DRY_RUN (every rep does the same work: Delta stays
armed, the decision is computed and recorded but not committed; boundary f = 0
so every segment is active -- the worst case).  value = algorithmic bytes of
all ranks / max-over-ranks device time.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload bert-large-f32|bert-base-bf16]
    python -m torch.distributed.run --nproc-per-node N bench.py --gpus N ...
    python bench.py --impl reference      # the fp64 CPU oracle, same metric (rank 0 only)
"""
import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "per-layer grad-norm+decide GB/s (% of HBM peak) at 1/2/4/8 B200; cache GB/s"
ROW_BYTES = 128 * 768 * 2          # BERT-base hidden 768, seq 128, bf16 (configs[3])
NUM_EXAMPLES = 100_000
GLOBAL_CACHE_BATCH = 256

WORKLOADS = {
    "bert-large-f32": ("large", "f32"),   # configs[2]: BERT-large fp32, sharded over N GPUs
    "bert-base-bf16": ("base", "bf16"),   # configs[1]: BERT-base bf16, 1 GPU
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="bert-large-f32", choices=sorted(WORKLOADS))
    ap.add_argument("--cache-batch", type=int, default=GLOBAL_CACHE_BATCH)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=20)
    ap.add_argument("--no-cache-sweep", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="launch the timed steps eagerly (no CUDA graphs)")
    ap.add_argument("--no-overlap", action="store_true",
                    help="the step's cache get waits for the interval end to complete (no AF_CACHE_OVERLAP_PREV)")
    ap.add_argument("--no-extras", action="store_true", help="skip the NEXT-row probes (fused AdamW)")
    ap.add_argument("--no-secondary", action="store_true",
                    help="N = 1: skip the short run of the other BERT workload reported under 'secondary'")
    ap.add_argument("--exchange", default="p2p", choices=["p2p", "nccl"],
                    help="N > 1: per-layer partial exchange (in-kernel NVLink P2P, or NCCL all-gather)")
    ap.add_argument("--zero", action="store_true",
                    help="ZeRO form (NEXT 1): every rank holds its own full gradient; the step's accumulate and "
                         "interval end are af_reduce_scatter_step (the gradient sync fused in, peer pulls)")
    ap.add_argument("--unfused", action="store_true",
                    help="interval end as af_layer_norms(END) + af_update_and_decide (two launches)")
    ap.add_argument("--no-shard-probe", action="store_true",
                    help="N = 1: skip the per-rank shard probe of the 8-GPU BERT-large run (rank_shard_p8)")
    ap.add_argument("--shard-probe-only", action="store_true", help="print only the rank_shard_p8 probe")
    ap.add_argument("--sweep", action="store_true",
                    help="configs[4]: layers x elements sweep, one JSON line per point (not the bench line)")
    return ap.parse_args()


def max_over_ranks(x, dev):
    """Max of a float over all ranks (device tensor for NCCL, CPU tensor for gloo)."""
    import torch
    import torch.distributed as dist
    on = dev if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([x], device=on, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.item()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy bandwidth)"
    return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


# ------------------------------------------------------------------ clocks (NVML, in-process)

class ClockSampler:
    """Samples SM clocks and throttle reasons every 10 ms during the timed region."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, index):
        self.samples, self.reasons, self.ok = [], set(), False
        self._stop = threading.Event()
        try:
            import pynvml
            import torch
            pynvml.nvmlInit()
            self.nv = pynvml
            pr = torch.cuda.get_device_properties(index)
            try:
                bus = f"{pr.pci_domain_id:08X}:{pr.pci_bus_id:02X}:{pr.pci_device_id:02X}.0"
                self.h = pynvml.nvmlDeviceGetHandleByPciBusId(bus)
            except Exception:  # noqa: BLE001
                self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # noqa: BLE001
            self.err = repr(e)

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:  # noqa: BLE001
                pass
            time.sleep(0.01)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.ok:
            self.t.join()

    def summary(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "error": getattr(self, "err", "")}
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ------------------------------------------------------------------ synthetic inputs on the device

def device_grad(lay, dt, seed, device, T=1):
    """Synthetic gradient of the workload's shape (DESIGN.md input recipe:
    sigma_l(T) * U(-1, 1) per segment), drawn on the device with torch's RNG
    (bench only; the parity tests use afinputs/numpy)."""
    import torch
    from afinputs import segment_rho
    gen = torch.Generator(device=device)
    gen.manual_seed(seed)
    x = torch.rand(lay.n, generator=gen, device=device, dtype=torch.float32).mul_(2).sub_(1)
    sizes = torch.tensor([lay.seg_len(l) for l in range(lay.n_segments)], device=device)
    sig = torch.tensor([1e-3 * (1 + 0.9 * r ** T) for r in segment_rho(lay)], device=device,
                       dtype=torch.float32)
    x.mul_(torch.repeat_interleave(sig, sizes))
    return x.to(torch.bfloat16) if dt == "bf16" else x


def ncu_traffic(workload, phase):
    """roofline.traffic: DRAM bytes per launch of this kernel from the committed
    `ncu --set full` capture (profiles/traffic.json, tools/traffic_from_ncu.py)."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        d = json.load(open(p))[workload][phase]
        return {"traffic": round(d["bytes_per_launch"]), "traffic_source": "profiles/traffic.json <- " + d["source"]}
    except Exception:  # noqa: BLE001
        return {"traffic": None}


def algorithmic_bytes(n_loc, s_g, rows, row_bytes):
    return {"accumulate": n_loc * (s_g + 8), "grad_norm_decide": n_loc * (s_g + 4),
            "cache_get": 2 * rows * row_bytes, "cache_put": 2 * rows * row_bytes}


# ------------------------------------------------------------------ our arm

def run_ours(args, rank, world, local):
    import torch
    import torch.distributed as dist

    import paper_2102_01386_b200 as af
    from afinputs import bert_layout

    local = local % max(1, torch.cuda.device_count())   # ranks may share a GPU (functional check)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        # AF_BENCH_BACKEND=gloo lets several ranks share one GPU for a functional
        # check of the N > 1 flow (NCCL refuses two ranks on one device)
        backend = os.environ.get("AF_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    which, dt = WORKLOADS[args.workload]
    lay = bert_layout(which)
    s_g = 2 if dt == "bf16" else 4
    # N > 1: shards of the active suffix, re-split per boundary f (the ZeRO form owns
    # per-shard optimizer state and keeps static shards)
    fm = af.FreezingModule(lay.offsets, lay.kinds, grad_dtype=dt, rank=rank, world=world, device=dev,
                           shard_active=(world > 1 and not args.zero))
    exchange = "none"
    if world > 1:
        # NVLink one-shot exchange inside the interval-end kernel (CUDA IPC peer
        # mappings); NCCL all-gather as the fallback
        if args.exchange == "p2p" and fm.set_peers_ipc():   # collective; same answer on every rank
            exchange = "p2p"
        else:
            fm.set_comm()
            exchange = "nccl"
    info = fm.info()
    n_loc = info["shard_end"] - info["shard_begin"]
    grads = [device_grad(lay, dt, 1000 + k, dev) for k in range(2)]
    rs_out = None
    if args.zero:
        # each rank's own gradient (seeded by rank), registered once; the step pulls
        # this rank's shard of every rank's buffer and writes the reduced shard
        if world > 1 and exchange != "p2p":
            raise SystemExit("--zero needs the peer mappings (CUDA IPC) on every rank")
        g_own = device_grad(lay, dt, 2000 + rank, dev)
        grads = [g_own, g_own]
        if world > 1:
            fm.set_grad_peers_ipc(g_own)
        else:
            fm.set_grad_peers_local([g_own])
        rs_out = torch.empty(n_loc, device=dev)
    # activation cache partition of this rank (id mod world)
    B = max(1, args.cache_batch // world)
    cache = af.ActivationCache(NUM_EXAMPLES, ROW_BYTES, rank=rank, world=world, device=dev)
    my_ids = torch.arange(rank, NUM_EXAMPLES, world, device=dev, dtype=torch.int64)
    perm = my_ids[torch.randperm(my_ids.numel(), device=dev)]
    rows = torch.randint(0, 256, (B, ROW_BYTES), dtype=torch.uint8, device=dev)
    out_rows = torch.empty_like(rows)
    depth_out = torch.empty(B, dtype=torch.int32, device=dev)
    # populate every slot once (untimed) at depth 4: gets hit and never evict (boundary 4)
    for b0 in range(0, my_ids.numel(), 4096):
        ids_b = my_ids[b0:b0 + 4096]
        src = rows.repeat((ids_b.numel() + B - 1) // B, 1)[: ids_b.numel()].contiguous()
        cache.put(ids_b, src, 4)
    n_batches = my_ids.numel() // B
    id_batches = [perm[i * B:(i + 1) * B].contiguous() for i in range(max(1, n_batches))]
    # one committed interval so that T = 1 and every dry-run decide does the full test,
    # then one committed accumulate step so that Delta is armed: every dry-run
    # accumulate reads+writes Delta and every dry-run interval end reads it.
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()   # ranks enter the first exchange together (the in-kernel wait is bounded)
    if args.zero:
        fm.reduce_scatter_step(rs_out)
        fm.reduce_scatter_step(rs_out, interval_end=True)
        fm.reduce_scatter_step(rs_out)
    else:
        fm.layer_norms(grads[0])
        fm.layer_norms(grads[1], interval_end=True)
        fm.update_and_decide()
        fm.layer_norms(grads[0])
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    n_ev = 5

    def step(i, evs=None, skip=()):
        g = grads[i & 1]
        ids = id_batches[i % len(id_batches)]
        if evs: evs[0].record(stream)
        if "accumulate" in skip:
            pass
        elif args.zero:
            fm.reduce_scatter_step(rs_out, dry_run=True)              # gradient sync + a2
        else:
            fm.layer_norms(g, dry_run=True)                           # a2
        if evs: evs[1].record(stream)
        if "grad_norm_decide" in skip:
            pass
        elif args.zero:
            fm.reduce_scatter_step(rs_out, interval_end=True, dry_run=True)   # sync + a3-a9
        elif args.unfused:
            fm.layer_norms(grads[(i + 1) & 1], interval_end=True, dry_run=True)
            fm.update_and_decide(dry_run=True)
        else:
            fm.interval_end(grads[(i + 1) & 1], dry_run=True)         # a3-a9 (fused at N=1)
        if evs: evs[2].record(stream)
        if "cache" in skip:
            return
        # a11; the get reads nothing the interval end writes: it may start during the
        # interval end's last-CTA tail (AF_CACHE_OVERLAP_PREV)
        cache.get(ids, 4, out_rows, depth_out, overlap_prev=not args.no_overlap)
        if evs: evs[3].record(stream)
        cache.put(ids, rows, 4)                                       # a10
        if evs: evs[4].record(stream)

    # the timed loop replays CUDA graphs of one step each (8 graphs rotate the id batches)
    graphs = []
    if not args.no_graph:
        for i in range(min(8, len(id_batches))):
            gph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gph):
                step(i)
            graphs.append(gph)
        torch.cuda.synchronize()

    def run(i):
        if graphs:
            graphs[i % len(graphs)].replay()
        else:
            step(i)

    for i in range(args.warmup):
        run(i)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0.record(stream)
        for i in range(args.steps):
            run(i)
        t1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    ms_local = t0.elapsed_time(t1)
    dist_ms = step_distribution(args, run, stream, world, dist, dev)
    frozen = None if args.zero else frozen_point(args, fm, lay, info, s_g, B, run, stream, world, dist, dev,
                                                 grads[0])
    marg = step_marginals(args, graphs, step, stream, world, dist) if graphs else None
    cache_marg = marg["cache"] if marg else None
    # per-phase breakdown: a second, eagerly launched pass with CUDA events between calls
    n_ph = max(1, min(args.steps, 100))
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(n_ev)] for _ in range(n_ph)]
    for i in range(n_ph):
        step(i, evs[i])
    torch.cuda.synchronize()
    phases = ["accumulate", "grad_norm_decide", "cache_get", "cache_put"]
    ph_ms = {p: sum(e[k].elapsed_time(e[k + 1]) for e in evs) / n_ph for k, p in enumerate(phases)}
    ms = ms_local
    if world > 1:
        ms = max_over_ranks(ms_local, dev)
    ms_per_step = ms / args.steps
    bytes_rank = algorithmic_bytes(n_loc, s_g, B, ROW_BYTES)
    if args.zero:   # P gradient shards read (P-1 over NVLink) + the reduced shard written (fp32)
        bytes_rank["accumulate"] = n_loc * (world * s_g + 8 + 4)
        bytes_rank["grad_norm_decide"] = n_loc * (world * s_g + 4 + 4)
    step_bytes_all = sum(bytes_rank.values()) * world   # every rank moves ~the same bytes
    value = step_bytes_all / (ms_per_step * 1e-3) / 1e9
    peak, peak_src = measured_peaks()
    # dominant kernel roofline (per-launch CUDA-event durations on the launch stream)
    dom = max(("accumulate", "grad_norm_decide", "cache_get", "cache_put"), key=lambda p: ph_ms[p])
    ach = bytes_rank[dom] / (ph_ms[dom] * 1e-3) / 1e9
    phase_report = {p: {"ms": round(ph_ms[p], 5),
                        "gbs": (round(bytes_rank[p] / (ph_ms[p] * 1e-3) / 1e9, 1) if bytes_rank[p] else None),
                        "frac_of_peak": (round(bytes_rank[p] / (ph_ms[p] * 1e-3) / 1e9 / peak, 4)
                                         if bytes_rank[p] else None)} for p in phases}
    gn_dec_ms = ph_ms["grad_norm_decide"]
    gn_dec = bytes_rank["grad_norm_decide"] / (gn_dec_ms * 1e-3) / 1e9
    cache_gbs = (bytes_rank["cache_get"] + bytes_rank["cache_put"]) / (
        (ph_ms["cache_get"] + ph_ms["cache_put"]) * 1e-3) / 1e9
    if cache_marg is not None:   # in-step device time of get + put (step_marginals)
        cache_marg_gbs = (bytes_rank["cache_get"] + bytes_rank["cache_put"]) / (cache_marg * 1e-3) / 1e9
        cache_in_step = {"us": round(cache_marg * 1e3, 2), "gbs": round(cache_marg_gbs, 1),
                         "frac_of_peak": round(cache_marg_gbs / peak, 4),
                         "method": "marginal: graph-replayed steps minus the same steps without the cache calls "
                                   "(no events between kernels); phases.cache_* are eager event pairs, which add "
                                   "a ~6 us floor per call"}
        cache_gbs = cache_marg_gbs
    result = {
        "metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_per_step, 5), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": ("bf16" if dt == "bf16" else "f32") + "+f64",
        "data": "synthetic (seeded device RNG, BERT layer layout, DESIGN.md input recipe)",
        "config": {"workload": f"{args.workload}" + ("-sharded" if world > 1 else "") + ("-zero" if args.zero else ""),
                   "n_elements": lay.n, "segments": lay.n_segments, "n_local": n_loc,
                   "cache": {"examples": NUM_EXAMPLES, "row_bytes": ROW_BYTES, "rows_per_rank_step": B},
                   "boundary_f": 0, "parallelism": (f"zero{world}" if args.zero else f"shard{world}"),
                   "exchange": exchange,
                   "shards": ("active-suffix (re-split per boundary f)" if (world > 1 and not args.zero)
                              else "static"),
                   "launch": "eager" if args.no_graph else "CUDA graph per step (8 graphs rotating id batches)",
                   "l2": "inputs larger than L2: each step streams >= 4 GB/rank through the 126 MB L2"},
        "value_composition": "whole step: accumulate + interval end (grad-norm + decide) + cache get + put "
                             "(all SURVEY.md 8(a) rows); the metric's grad-norm+decide quantity alone is "
                             "grad_norm_decide_in_step",
        **({"grad_norm_decide_in_step": {
            "us": round(marg["grad_norm_decide"] * 1e3, 2),
            "gbs": round(bytes_rank["grad_norm_decide"] / (marg["grad_norm_decide"] * 1e-3) / 1e9, 1),
            "frac_of_peak": round(bytes_rank["grad_norm_decide"] / (marg["grad_norm_decide"] * 1e-3) / 1e9 / peak, 4),
            "bytes_per_launch": bytes_rank["grad_norm_decide"],
            "method": "marginal device time of af_interval_end in the graph-replayed step (phases_in_step)"}}
           if marg else {}),
        "grad_norm_decide_gbs": round(gn_dec, 1),
        "grad_norm_decide_frac_of_hbm_peak": round(gn_dec / peak, 4),
        "cache_gbs": round(cache_gbs, 1),
        **({"cache_in_step": cache_in_step} if cache_marg is not None else {}),
        **({"phases_in_step": {
            "method": "marginal device time: the step's CUDA graphs replayed with and without the phase, K steps "
                      "each, alternating, difference of medians (max over ranks); includes what the phase adds "
                      "through overlap (PDL) and L2 state",
            **{k: {"ms": round(v, 5),
                   **({"gbs": round(phase_bytes(bytes_rank, k) / (v * 1e-3) / 1e9, 1),
                       "frac_of_peak": round(phase_bytes(bytes_rank, k) / (v * 1e-3) / 1e9 / peak, 4)} if v > 0 else {})}
               for k, v in marg.items() if k != "full"}}} if marg else {}),
        "step_ms_dist": dist_ms,
        "frozen_half": frozen,
        "phases": phase_report,
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": round(ach, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(ach / peak, 4), "peak_source": peak_src,
                     "algorithmic_bytes_per_launch": bytes_rank[dom],
                     **ncu_traffic(args.workload if world == 1 else None, dom)},
        # accumulate + interval end (+ wide finalize) (+ decide kernel, NCCL all-gather) + cache get + put
        "gpu_launches": (4 + (1 if info["n_fin_ctas"] else 0)
                         + (1 if (args.unfused or (world > 1 and exchange != "p2p")) else 0)
                         + (1 if (world > 1 and exchange != "p2p") else 0)) * args.steps,
        "clocks": clk.summary(),
    }
    if not args.no_cache_sweep:
        result["cache_gbs_by_batch"] = cache_sweep(cache, my_ids, rows, dev, world, dist)
        result["cache_host_tier"] = host_tier_probe(rows, dev)
        if world == 1:
            result["cache_epoch_c4"] = cache_epoch_c4(dev)
    if not args.no_extras:
        result["next1_fused_adamw"] = adamw_probe(fm, lay, dt, s_g, n_loc, grads, dev)
        result["next4_cache_get_gemm"] = next4_get_gemm_probe(cache, my_ids, dev)
        if world == 1:
            result["next1_fused_reduce_scatter_p1"] = rs_probe(lay, dt, s_g, grads, dev)
    if not args.no_e2e and not args.zero:
        result["e2e"] = run_e2e(args, fm, cache, info, lay, dt, s_g, B, id_batches, rows, dev, world, dist)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        result["cpu_baseline"] = cpu_baseline(lay, dt, s_g, B, budget_s=12.0)
        result["cpu_baseline_all_cores"] = cpu_baseline_all_cores(lay, dt, s_g, B)
    if world == 1 and not args.no_shard_probe and args.workload == "bert-large-f32":
        result["rank_shard_p8"] = rank_shard_probe(args, dev)
        # the same emulation at P = 2 and 4 (one rank each): the per-GPU share of the
        # 1/2/4/8-GPU metric on this GPU, exchange stores included, NVLink wait not
        keep = ("n_local", "interval_end_alone_us", "frac_alone", "interval_end_in_step_us", "frac_in_step",
                "step_pair_us", "step_pair_frac")
        by_world = {}
        for P in (2, 4):
            row = rank_shard_probe(args, dev, P=P, ranks=(P - 1,), rounds=2)["max_over_ranks"]
            by_world[str(P)] = {k: row[k] for k in keep}
        by_world["8"] = {k: result["rank_shard_p8"]["max_over_ranks"][k] for k in keep}
        result["rank_shard_by_world"] = by_world
    if world == 1 and not args.no_secondary:
        result["secondary"] = secondary_workload(args)
    if rank == 0:
        print(json.dumps(result), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def step_distribution(args, run, stream, world, dist, dev, n=100):
    """p10 / p50 / p90 of single-step device times (SURVEY.md §8(d) timing
    protocol): min(K, 100) replays, each bracketed by its own event pair (the
    pair adds a little; the headline `ms_per_step` is the K-step block)."""
    import torch
    n = max(1, min(args.steps, n))
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    for i, (a, b) in enumerate(evs):
        a.record(stream)
        run(i)
        b.record(stream)
    torch.cuda.synchronize()
    t = sorted(a.elapsed_time(b) for a, b in evs)
    q = {k: t[min(len(t) - 1, int(round(f * (len(t) - 1))))] for k, f in (("p10", 0.1), ("p50", 0.5), ("p90", 0.9))}
    if world > 1:
        q = {k: max_over_ranks(v, dev) for k, v in q.items()}
    return {**{k: round(v, 5) for k, v in q.items()}, "samples": n}


def frozen_point(args, fm, lay, info, s_g, B, run, stream, world, dist, dev, g):
    """The same step with the boundary at f = B/2 POOL blocks frozen (SURVEY.md
    §8(d): bytes scale with the active suffix; PRE is tied to the first POOL
    block).  f is patched into a state blob (af_get_state layout: magic, version,
    L, world, rank, T, f, ...); the step's graphs read f from device memory at
    launch, so they replay unchanged.  The original state is restored after.  A
    committed accumulate after each change re-arms Delta (active-suffix shards
    start a fresh sum when f moves).  Bytes: the active elements of ALL ranks."""
    import struct

    import torch
    blob = fm.get_state()
    f = info["n_pool"] // 2
    from afinputs.layouts import SEG_POOL
    pool = [l for l, k in enumerate(lay.kinds) if k == SEG_POOL]
    assert len(pool) == info["n_pool"]
    act0 = lay.offsets[pool[f]]                       # segments before the (f+1)-th POOL block are frozen
    sb, se = fm.shard_of(f)
    n_act_local = max(0, se - max(sb, act0))
    n_act = lay.n - act0                              # the shards cover [0, n): all ranks' active elements
    patched = bytearray(blob)
    struct.pack_into("<i", patched, 24, f)
    fm.set_state(bytes(patched))
    fm.layer_norms(g)
    try:
        for i in range(args.warmup):
            run(i)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for i in range(args.steps):
            run(i)
        b.record(stream)
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / args.steps
        if world > 1:
            ms = max_over_ranks(ms, dev)
    finally:
        fm.set_state(blob)
        fm.layer_norms(g)
        torch.cuda.synchronize()
    by = algorithmic_bytes(n_act, s_g, B, ROW_BYTES)
    step_bytes = by["accumulate"] + by["grad_norm_decide"] + (by["cache_get"] + by["cache_put"]) * world
    return {"boundary_f": f, "active_elements": n_act, "active_elements_local": n_act_local,
            "ms_per_step": round(ms, 5),
            "gbs": round(step_bytes / (ms * 1e-3) / 1e9, 1),
            "note": "algorithmic bytes count active (unfrozen) elements only; GB/s on those bytes"}


def phase_bytes(bytes_rank, phase):
    return bytes_rank["cache_get"] + bytes_rank["cache_put"] if phase == "cache" else bytes_rank[phase]


def step_marginals(args, graphs, step, stream, world, dist, rounds=3):
    """In-step device time (ms) of each phase: the step's graphs replayed with and
    without the phase (accumulate / interval end / cache get + put), alternating,
    K steps each; a phase's cost is the difference of the medians (max over
    ranks).  Dry-run calls commit nothing, so dropping one leaves the others' work
    unchanged."""
    import torch
    sets = {"full": graphs}
    for ph in ("accumulate", "grad_norm_decide", "cache"):
        gl = []
        for i in range(len(graphs)):
            gph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gph):
                step(i, skip=(ph,))
            gl.append(gph)
        sets[ph] = gl
    torch.cuda.synchronize()
    t = {k: [] for k in sets}
    for _ in range(rounds):
        for k, gl in sets.items():
            for i in range(args.warmup):
                gl[i % len(gl)].replay()
            if world > 1:
                dist.barrier()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            a.record(stream)
            for i in range(args.steps):
                gl[i % len(gl)].replay()
            b.record(stream)
            torch.cuda.synchronize()
            t[k].append(a.elapsed_time(b) / args.steps)
    full = statistics.median(t["full"])
    out = {"full": full}
    dev = torch.device("cuda", torch.cuda.current_device())
    for k in ("accumulate", "grad_norm_decide", "cache"):
        d = full - statistics.median(t[k])
        out[k] = max_over_ranks(d, dev) if world > 1 else d
    return out


def secondary_workload(args):
    """N = 1: the other BASELINE config (bert-base-bf16, configs[1], when the main
    line is bert-large-f32) timed the same way, in a subprocess, summarised."""
    import subprocess
    other = "bert-base-bf16" if args.workload == "bert-large-f32" else "bert-large-f32"
    cmd = [sys.executable, os.path.abspath(__file__), "--workload", other, "--steps", str(args.steps), "--warmup",
           str(args.warmup), "--no-e2e", "--no-cpu-baseline", "--no-cache-sweep", "--no-secondary"]
    r = subprocess.run(cmd, capture_output=True, text=True, env=dict(os.environ, WORLD_SIZE="1", RANK="0"))
    try:
        d = json.loads(r.stdout.strip().splitlines()[-1])
    except Exception:  # noqa: BLE001
        return {"workload": other, "error": r.stderr[-500:]}
    keep = ("value", "unit", "ms_per_step", "grad_norm_decide_gbs", "grad_norm_decide_frac_of_hbm_peak", "dtype",
            "config", "phases", "phases_in_step", "cache_gbs", "cache_in_step", "roofline", "clocks", "step_ms_dist",
            "frozen_half", "next1_fused_adamw", "next1_fused_reduce_scatter_p1")
    return {"workload": other, **{k: d[k] for k in keep if k in d}}


def cache_sweep(cache, my_ids, rows, dev, world, dist, batches=(6, 32, 256, 1024, 4096), reps=20, iters=5):
    """Cache get / put GB/s (2 x rows x row_bytes per call) per batch size on this
    rank's partition (all hits, no eviction: boundary == depth), with a COLD L2 as
    inside the step: each call gets fresh ids and follows a 512 MB read.  A call's
    cost is marginal device time: a CUDA graph of reps x [flush, call] minus one of
    reps x [flush], divided by reps -- launches back to back, no event between calls
    (an event pair around one call adds a ~6 us floor; tools/cache_cold_probe.py)."""
    import torch
    out = {"l2": "cold (512 MB read before each call, fresh ids per call); *_back_to_back: one 512 MB read, "
                 "then the calls one after another (fresh ids per call, records cold)",
           "timing": "marginal device time per call in CUDA graphs (graph with calls minus graph without)"}
    B0 = rows.shape[0]
    big = rows.repeat((max(batches) + B0 - 1) // B0, 1)[: max(batches)].contiguous()
    flush = torch.ones(256 << 20, dtype=torch.float16, device=dev)
    acc = torch.zeros((), dtype=torch.float32, device=dev)
    peak, _ = measured_peaks()

    def marginal_us(fn):
        gs = {}
        for w in (True, False):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                for r in range(reps):
                    torch.sum(flush, dim=0, dtype=torch.float32, out=acc)
                    if w:
                        fn(r)
            gs[w] = g
        t = {True: [], False: []}
        for _ in range(iters):
            for w in (True, False):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                gs[w].replay()
                b.record()
                torch.cuda.synchronize()
                t[w].append(a.elapsed_time(b))
        return (statistics.median(t[True]) - statistics.median(t[False])) / reps * 1e3

    def marginal_b2b_us(fn):
        # the epoch's regime (one call per batch, batch after batch):
        # reps calls back to back after ONE flush, minus the flush alone, per call --
        # each call's launch, ramp and drain overlap its neighbours' (PDL)
        gs = {}
        for w in (True, False):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                torch.sum(flush, dim=0, dtype=torch.float32, out=acc)
                if w:
                    for r in range(reps):
                        fn(r)
            gs[w] = g
        t = {True: [], False: []}
        for _ in range(iters):
            for w in (True, False):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                gs[w].replay()
                b.record()
                torch.cuda.synchronize()
                t[w].append(a.elapsed_time(b))
        return (statistics.median(t[True]) - statistics.median(t[False])) / reps * 1e3

    for B in batches:
        if B > my_ids.numel():
            continue
        id_sets = [my_ids[torch.randperm(my_ids.numel(), device=dev)[:B]].contiguous() for _ in range(reps)]
        src = big[:B]
        dst = torch.empty_like(src)
        dep = torch.empty(B, dtype=torch.int32, device=dev)
        res = {}
        for name, fn in (("put", lambda r: cache.put(id_sets[r], src, 4)),
                         ("get", lambda r: cache.get(id_sets[r], 4, dst, dep))):
            for key, meas in ((name, marginal_us), (name + "_back_to_back", marginal_b2b_us)):
                us = meas(fn)
                gbs = 2 * B * ROW_BYTES / (us * 1e-6) / 1e9
                res[key] = {"us": round(us, 2), "gbs": round(gbs, 1), "frac_of_peak": round(gbs / peak, 4)}
        out[str(B)] = res
    del flush
    return out


def cache_epoch_c4(dev, world_emul=8, B=256, seed=3):
    """the frozen-prefix cache over epochs, one rank's
    partition of 100k examples x 196,608 B at P = 8 (12,500 ids, 2.46 GB), with
    the boundary change 4 -> 7 (records written at depth 4 are
    evicted on read once 7 blocks are frozen, then re-cached at depth 7):
      epoch 0  put every owned id at depth 4 (permutation pi_0, batches of B)
      epoch 1  boundary 7: get in pi_1 (every record hits at depth 4 and is
               evicted), then re-put each batch at depth 7
      epoch 2  get in pi_2 (hits at depth 7, nothing evicted)
    Eager calls on one stream, CUDA events around each epoch; GB/s = 2 x rows x
    row_bytes per call.  Counts are checked as the epochs run."""
    import torch

    import paper_2102_01386_b200 as af
    peak, _ = measured_peaks()
    rank = 0
    cache = af.ActivationCache(NUM_EXAMPLES, ROW_BYTES, rank=rank, world=world_emul, device=dev)
    ids = torch.arange(rank, NUM_EXAMPLES, world_emul, device=dev, dtype=torch.int64)
    n = ids.numel()
    gen = torch.Generator(device=dev)
    gen.manual_seed(seed)
    rows = torch.randint(0, 256, (B, ROW_BYTES), dtype=torch.uint8, device=dev, generator=gen)
    out = torch.empty_like(rows)
    dep = torch.empty(B, dtype=torch.int32, device=dev)

    def perm(e):
        g = torch.Generator(device=dev)
        g.manual_seed(seed * 1000 + e)
        p = ids[torch.randperm(n, device=dev, generator=g)]
        return [p[i:i + B].contiguous() for i in range(0, n, B)]

    res = {"partition_rows": n, "row_bytes": ROW_BYTES, "batch": B, "world_emulated": world_emul,
           "l2": "cold: each epoch walks 2.46 GB of records in a fresh permutation"}

    def epoch(name, batches, fn, calls_per_batch):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for bt in batches:
            fn(bt)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b)
        byts = sum(2 * bt.numel() * ROW_BYTES for bt in batches) * calls_per_batch
        gbs = byts / (ms * 1e-3) / 1e9
        res[name] = {"ms": round(ms, 3), "calls": len(batches) * calls_per_batch, "gbs": round(gbs, 1),
                     "frac_of_peak": round(gbs / peak, 4)}

    epoch("epoch0_put_depth4", perm(0), lambda bt: cache.put(bt, rows[:bt.numel()], 4), 1)
    assert cache.status() == (0, n)

    def get_evict_reput(bt):
        cache.get(bt, 7, out[:bt.numel()], dep[:bt.numel()])
        cache.put(bt, out[:bt.numel()], 7)
    epoch("epoch1_get_evict_reput_depth7", perm(1), get_evict_reput, 2)
    assert cache.status() == (0, n)           # every record evicted on read and re-cached
    torch.cuda.synchronize()
    res["epoch1_depths_seen"] = sorted(set(dep.tolist()))
    epoch("epoch2_get_hits_depth7", perm(2), lambda bt: cache.get(bt, 7, out[:bt.numel()], dep[:bt.numel()]), 1)
    torch.cuda.synchronize()
    assert cache.status() == (0, n) and set(dep.tolist()) == {7}
    cache.close()
    del cache
    torch.cuda.empty_cache()
    return res


def next4_get_gemm_probe(cache, my_ids, dev, B=256, N=2304, reps=10, rounds=5):
    """NEXT 4: the cache get fused into the first active layer's GEMM operand load
    (af_cache_get_gemm: TMA gathers each record as the A tile, tcgen05 MMAs)
    against af_cache_get into a batch buffer + torch.matmul (cuBLAS bf16), on the
    step's cache (records of 128 x 768 bf16 = BERT-base hidden states), B fresh
    ids per call (cold records), W = BERT-base's QKV projection [2304, 768].
    CUDA graphs of `reps` calls, median of rounds."""
    import torch
    K = ROW_BYTES // (128 * 2)
    g = torch.Generator(device=dev)
    g.manual_seed(5)
    w = (torch.randn(N, K, device=dev, generator=g) * 0.05).to(torch.bfloat16)
    sets = [my_ids[torch.randperm(my_ids.numel(), device=dev, generator=g)[:B]].contiguous() for _ in range(reps)]
    y = torch.empty(B * 128, N, dtype=torch.bfloat16, device=dev)
    dep = torch.empty(B, dtype=torch.int32, device=dev)
    buf = torch.empty(B, ROW_BYTES, dtype=torch.uint8, device=dev)

    def fused(r):
        cache.get_gemm(sets[r], 4, w, y, dep, 128)

    def unfused(r):
        cache.get(sets[r], 4, buf, dep)
        torch.matmul(buf.view(torch.bfloat16).view(B * 128, K), w.t(), out=y)

    res = {"examples": B, "M": B * 128, "N": N, "K": K}
    flops = 2 * B * 128 * K * N
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    tf_peak = peaks.get("bf16_tflops", 2250.0)
    for name, fn in (("fused_get_gemm", fused), ("get_then_cublas", unfused)):
        fn(0)
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
        res[name] = {"us": round(us, 2), "tflops": round(flops / (us * 1e-6) / 1e12, 1)}
        del gph
    f = res["fused_get_gemm"]
    res["roofline"] = {"bound": "tensor", "achieved": f["tflops"], "peak": tf_peak, "unit": "TFLOP/s",
                       "frac": round(f["tflops"] / tf_peak, 4),
                       "peak_source": "MEASURED_PEAKS.json bf16_tflops (cuBLAS 8192^3, burst)"}
    res["speedup_vs_unfused"] = round(res["get_then_cublas"]["us"] / f["us"], 3)
    res["bytes_saved_per_example"] = 2 * ROW_BYTES
    return res


def host_tier_probe(rows, dev, reps=10):
    """Tiered storage manager (NEXT 3): put/get GB/s of the rows when every slot
    lives in the page-locked host tier (PCIe / C2C bound)."""
    import torch

    import paper_2102_01386_b200 as af
    B = rows.shape[0]
    c = af.ActivationCache(B, ROW_BYTES, device=dev, hbm_rows=0, host_rows=B)
    ids = torch.arange(B, device=dev, dtype=torch.int64)
    out = torch.empty_like(rows)
    dep = torch.empty(B, dtype=torch.int32, device=dev)
    res = {}
    for name, fn in (("put", lambda: c.put(ids, rows, 4)), ("get", lambda: c.get(ids, 4, out, dep))):
        fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            fn()
        b.record()
        b.synchronize()
        ms = a.elapsed_time(b) / reps
        res[name] = {"us": round(ms * 1e3, 1), "gbs": round(B * ROW_BYTES / (ms * 1e-3) / 1e9, 1),
                     "note": "host-tier bytes crossing the link (one direction)"}
    res["rows"] = B
    return res


def adamw_probe(fm, lay, dt, s_g, n_loc, grads, dev, reps=20):
    """NEXT 1: AdamW fused with the Delta accumulate (af_adamw_step) on this rank's
    shard: reads g, Delta, p, m, v and writes Delta, p, m, v -- s_g + 32 bytes per
    element, one read of g instead of two kernels reading it."""
    import torch
    p = torch.zeros(lay.n, device=dev)
    m = torch.zeros(lay.n, device=dev)
    v = torch.zeros(lay.n, device=dev)
    for k in range(2):
        fm.adamw_step(p, m, v, grads[k & 1], lr=1e-5, step=k + 1, dry_run=True)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for k in range(reps):
        fm.adamw_step(p, m, v, grads[k & 1], lr=1e-5, step=k + 3, dry_run=True)
    b.record()
    b.synchronize()
    ms = a.elapsed_time(b) / reps
    peak, _ = measured_peaks()
    by = n_loc * (s_g + 32)
    del p, m, v
    return {"us": round(ms * 1e3, 1), "bytes_per_elem": s_g + 32, "gbs": round(by / (ms * 1e-3) / 1e9, 1),
            "frac_of_peak": round(by / (ms * 1e-3) / 1e9 / peak, 4),
            "saved_vs_unfused_bytes_per_elem": s_g}


def rs_probe(lay, dt, s_g, grads, dev, reps=20):
    """NEXT 1 (ZeRO form) at P = 1 on this GPU: af_reduce_scatter_step reading the
    registered gradient, writing the reduced shard (fp32) and accumulating Delta --
    s_g + 4 + 8 bytes per element.  The P > 1 form pulls P-1 shards over NVLink
    (not measurable on one GPU)."""
    import torch

    import paper_2102_01386_b200 as af
    fm = af.FreezingModule(lay.offsets, lay.kinds, grad_dtype=dt, device=dev)
    fm.set_grad_peers_local([grads[0]])
    out = torch.empty(lay.n, device=dev)
    fm.reduce_scatter_step(out)                       # committed: Delta armed, every rep reads it
    for _ in range(2):
        fm.reduce_scatter_step(out, dry_run=True)
    torch.cuda.synchronize()
    def timed(end):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            fm.reduce_scatter_step(out, interval_end=end, dry_run=True)
        b.record()
        b.synchronize()
        return a.elapsed_time(b) / reps
    ms, ms_end = timed(False), timed(True)
    peak, _ = measured_peaks()
    by, by_end = lay.n * (s_g + 12), lay.n * (s_g + 8)
    del out, fm
    return {"us": round(ms * 1e3, 1), "bytes_per_elem": s_g + 12, "gbs": round(by / (ms * 1e-3) / 1e9, 1),
            "frac_of_peak": round(by / (ms * 1e-3) / 1e9 / peak, 4), "world": 1,
            "interval_end": {"us": round(ms_end * 1e3, 1), "bytes_per_elem": s_g + 8,
                             "gbs": round(by_end / (ms_end * 1e-3) / 1e9, 1),
                             "frac_of_peak": round(by_end / (ms_end * 1e-3) / 1e9 / peak, 4)}}


def rank_shard_probe(args, dev, P=8, ranks=(0, 3, 7), rounds=3):
    """One rank's share of the P-GPU run, timed on this GPU (BERT-large at P = 8:
    ~41.9M elements per rank).  All P contexts live here with the
    NVLink one-shot exchange registered locally (set_peers_local); only rank r's
    kernels run, with AF_DEBUG_PEERS_ARRIVED so its exchange pushes its row to
    the 7 peer contexts but does not wait for theirs.  So the numbers exclude the
    NVLink store latency (~1-2 us) and cross-rank skew, and include everything
    else of the rank's interval end (streaming, finalize, exchange stores,
    decision).  In-step = marginal device time in graph-replayed [accumulate,
    interval end] steps (with minus without the interval end); alone = the
    interval end replayed back to back."""
    import torch

    import paper_2102_01386_b200 as af
    from paper_2102_01386_b200 import _lib as L
    from afinputs import bert_layout
    which, dt = WORKLOADS[args.workload]
    lay = bert_layout(which)
    s_g = 2 if dt == "bf16" else 4
    peak, _ = measured_peaks()
    fms = [af.FreezingModule(lay.offsets, lay.kinds, grad_dtype=dt, rank=r, world=P, device=dev,
                             shard_active=True) for r in range(P)]
    for fm in fms:
        fm.set_peers_local(fms)
    g = [device_grad(lay, dt, 1000 + k, dev) for k in range(2)]
    steps = max(20, min(args.steps, 200))
    res = {"world_emulated": P, "workload": args.workload,
           "method": rank_shard_probe.__doc__.split("\n\n")[0].replace("\n", " ").strip()[:400]}
    worst = None
    for r in ranks:
        fm = fms[r]
        fm.set_debug(L.AF_DEBUG_PEERS_ARRIVED, 1)
        fm.layer_norms(g[0])
        fm.interval_end(g[1])
        fm.layer_norms(g[0])               # Delta armed; T = 1: every dry decision does the full test
        torch.cuda.synchronize()
        info = fm.info()
        n_loc = info["shard_end"] - info["shard_begin"]

        def graph(with_acc, with_end, reps=8):
            gph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gph):
                for i in range(reps):
                    if with_acc:
                        fm.layer_norms(g[i & 1], dry_run=True)
                    if with_end:
                        fm.interval_end(g[(i + 1) & 1], dry_run=True, copy_record=False)
            return gph, reps
        sets = {"full": graph(True, True), "acc": graph(True, False), "end": graph(False, True)}
        t = {k: [] for k in sets}
        for _ in range(rounds):
            for k, (gph, reps) in sets.items():
                for _ in range(3):
                    gph.replay()
                torch.cuda.synchronize()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                n_rep = max(1, steps // reps)
                a.record()
                for _ in range(n_rep):
                    gph.replay()
                b.record()
                torch.cuda.synchronize()
                t[k].append(a.elapsed_time(b) / (n_rep * reps))
        full, acc, alone = (statistics.median(t[k]) for k in ("full", "acc", "end"))
        in_step = full - acc
        by = n_loc * (s_g + 4)
        row = {"n_local": n_loc, "interval_end_in_step_us": round(in_step * 1e3, 2),
               "gbs_in_step": round(by / (in_step * 1e-3) / 1e9, 1),
               "frac_in_step": round(by / (in_step * 1e-3) / 1e9 / peak, 4),
               "interval_end_alone_us": round(alone * 1e3, 2),
               "gbs_alone": round(by / (alone * 1e-3) / 1e9, 1),
               "frac_alone": round(by / (alone * 1e-3) / 1e9 / peak, 4),
               "accumulate_us": round(acc * 1e3, 2),
               "accumulate_frac": round(n_loc * (s_g + 8) / (acc * 1e-3) / 1e9 / peak, 4),
               # the rank's step as a whole: accumulate + interval end back to back (their
               # L2 interplay makes the in-step marginal split between them arbitrary)
               "step_pair_us": round(full * 1e3, 2),
               "step_pair_frac": round((by + n_loc * (s_g + 8)) / (full * 1e-3) / 1e9 / peak, 4)}
        res[f"rank{r}"] = row
        if worst is None or row["interval_end_in_step_us"] > worst["interval_end_in_step_us"]:
            worst = dict(row, rank=r)
        fm.set_debug(L.AF_DEBUG_PEERS_ARRIVED, 0)
        del sets
    res["max_over_ranks"] = worst
    for fm in fms:
        fm.close()
    del fms, g
    torch.cuda.empty_cache()
    return res


def run_sweep(args, local):
    """configs[4]: uniform layouts, L in {1,2,4,12,24,48} POOL segments x n in
    {1M..1B} elements, fp32 and bf16, one GPU; accumulate and interval-end GB/s."""
    import torch

    import paper_2102_01386_b200 as af
    from afinputs import uniform_layout
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    peak, src = measured_peaks()
    for dt in ("f32", "bf16"):
        s_g = 2 if dt == "bf16" else 4
        for n in (1 << 20, 1 << 22, 1 << 24, 1 << 26, 1 << 28, 1 << 30):
            if n * (s_g + 4) > 9e9:
                continue
            g = device_grad(uniform_layout(n, 1), dt, 7, dev)
            for L in (1, 2, 4, 12, 24, 48):
                lay = uniform_layout(n, L)
                fm = af.FreezingModule(lay.offsets, lay.kinds, grad_dtype=dt, device=dev)
                fm.layer_norms(g)
                fm.layer_norms(g, interval_end=True)
                fm.update_and_decide()
                fm.layer_norms(g)                    # arm Delta
                reps = max(5, min(200, int(2e10 / (n * (s_g + 8)))))
                ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
                for _ in range(3):
                    fm.layer_norms(g, dry_run=True)
                    fm.interval_end(g, dry_run=True)
                torch.cuda.synchronize()
                ev[0].record()
                for _ in range(reps):
                    fm.layer_norms(g, dry_run=True)
                ev[1].record()
                for _ in range(reps):
                    fm.interval_end(g, dry_run=True)
                ev[2].record()
                torch.cuda.synchronize()
                acc_ms = ev[0].elapsed_time(ev[1]) / reps
                end_ms = ev[1].elapsed_time(ev[2]) / reps
                acc = n * (s_g + 8) / (acc_ms * 1e-3) / 1e9
                gnd = n * (s_g + 4) / (end_ms * 1e-3) / 1e9
                resident = n * (s_g + 4) < 126e6
                print(json.dumps({"sweep": "configs[4]", "dtype": dt, "n": n, "layers": L, "reps": reps,
                                  "accumulate_us": round(acc_ms * 1e3, 2), "accumulate_gbs": round(acc, 1),
                                  "accumulate_frac": round(acc / peak, 4),
                                  "grad_norm_decide_us": round(end_ms * 1e3, 2),
                                  "grad_norm_decide_gbs": round(gnd, 1), "grad_norm_decide_frac": round(gnd / peak, 4),
                                  "regime": "L2-resident / latency-bound" if resident else "HBM",
                                  "peak": peak, "peak_source": src}), flush=True)
                fm.close()
                del fm
            del g
            torch.cuda.empty_cache()


def run_e2e(args, fm, cache, info, lay, dt, s_g, B, id_batches, rows, dev, world, dist):
    """Same metric through the public API with HOST buffers: every step copies the
    rank's gradient shard, the cache rows and ids from pinned host memory and
    reads the decision record and the fetched rows back."""
    import torch
    sb, se = info["shard_begin"], info["shard_end"]
    n_loc = se - sb
    tdt = torch.bfloat16 if dt == "bf16" else torch.float32
    host_g = [torch.empty(n_loc, dtype=tdt, pin_memory=True) for _ in range(2)]
    for k in range(2):
        host_g[k].copy_(device_grad(lay, dt, 2000 + k, dev)[sb:se].cpu())
    dev_g = torch.zeros(lay.n, dtype=tdt, device=dev)          # full buffer; shard refreshed per step
    host_rows = rows.cpu().pin_memory()
    host_ids = [b.cpu().pin_memory() for b in id_batches[:8]]
    dev_ids = torch.empty(B, dtype=torch.int64, device=dev)
    dev_rows = torch.empty_like(rows)
    out_rows = torch.empty_like(rows)
    depth_out = torch.empty(B, dtype=torch.int32, device=dev)
    host_out = torch.empty_like(host_rows)
    host_depth = torch.empty(B, dtype=torch.int32, pin_memory=True)
    steps = max(1, min(args.steps, args.e2e_steps))
    stream = torch.cuda.current_stream()

    def step(i):
        dev_g[sb:se].copy_(host_g[i & 1], non_blocking=True)
        fm.layer_norms(dev_g, dry_run=True)
        dev_g[sb:se].copy_(host_g[(i + 1) & 1], non_blocking=True)
        fm.interval_end(dev_g, dry_run=True)                  # record -> pinned host (D2H)
        dev_ids.copy_(host_ids[i % len(host_ids)], non_blocking=True)
        cache.get(dev_ids, 4, out_rows, depth_out)
        host_out.copy_(out_rows, non_blocking=True)
        host_depth.copy_(depth_out, non_blocking=True)
        dev_rows.copy_(host_rows, non_blocking=True)
        cache.put(dev_ids, dev_rows, 4)

    for i in range(2):
        step(i)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for i in range(steps):
        step(i)
    t1.record(stream)
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1)
    if world > 1:
        ms = max_over_ranks(ms, dev)
    bytes_all = sum(algorithmic_bytes(n_loc, s_g, B, ROW_BYTES).values()) * world
    h2d = 2 * n_loc * s_g + B * ROW_BYTES + B * 8
    d2h = 6184 + B * ROW_BYTES + B * 4
    return {"value": round(bytes_all / (ms / steps * 1e-3) / 1e9, 2), "unit": "GB/s",
            "ms_per_step": round(ms / steps, 4), "steps": steps,
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h}


# ------------------------------------------------------------------ the oracle (CPU baseline / reference arm)

def oracle_step_runner(lay, dt, s_g, B, n_sample, lo=0, fast_inputs=False):
    """The oracle as it stands, on elements [lo, lo + n_sample) of the workload's
    flat buffer (the segments clipped to that slice) plus B cache rows.
    fast_inputs: draw the slice's values directly (same distribution, no full-size
    draw) -- for the all-core timing, whose processes each take one slice."""
    import numpy as np

    import oracle as O
    from afinputs import bert_grad_step, cache_rows, f32_to_bf16_bits
    hi = lo + n_sample
    offs = [0] + [o - lo for o in lay.offsets if lo < o < hi] + [n_sample]
    first = max(l for l in range(lay.n_segments) if lay.offsets[l] <= lo)
    kinds = lay.kinds[first:first + len(offs) - 1]
    if lo > 0 or hi < lay.n:              # a slice: keep a valid layout of its segments
        if O.SEG_POOL not in kinds:       # (the whole buffer keeps its own PRE / POOL / HEAD kinds)
            kinds = [O.SEG_POOL] * len(kinds)
        kinds = [k if k != O.SEG_HEAD else O.SEG_POOL for k in kinds]
        if O.SEG_PRE in kinds and kinds[0] != O.SEG_PRE:
            kinds = [O.SEG_POOL if k == O.SEG_PRE else k for k in kinds]
    fz = O.Freezer(offs, kinds, O.DT_BF16 if dt == "bf16" else O.DT_F32)
    if fast_inputs:
        rng = np.random.default_rng([lo, 0xAF])
        x = [(rng.random(n_sample, dtype=np.float32) * np.float32(2e-3) - np.float32(1e-3)) for _ in range(2)]
        g = [f32_to_bf16_bits(v) if dt == "bf16" else v for v in x]
    else:
        g = [bert_grad_step(lay, 0, 0, t, dtype=dt, lo=lo, hi=hi) for t in range(2)]
    cache = O.Cache(NUM_EXAMPLES, ROW_BYTES)
    ids = np.arange(B)
    rows = cache_rows(0, 0, B, ROW_BYTES)
    out = np.empty_like(rows)
    fz.layer_norms(g[0], False)
    fz.layer_norms(g[1], True)
    fz.update_and_decide()
    fz.layer_norms(g[0], False)          # arm Delta (as the GPU arm does)
    cache.put(ids, rows, 4)

    def step(i):
        fz.layer_norms(g[i & 1], False, dry_run=True)
        fz.layer_norms(g[(i + 1) & 1], True, dry_run=True)
        fz.update_and_decide(dry_run=True)
        cache.get(ids, 4, out)
        cache.put(ids, rows, 4)
    nbytes = sum(algorithmic_bytes(n_sample, s_g, B, ROW_BYTES).values())
    return step, nbytes


def cpu_baseline(lay, dt, s_g, B, budget_s=12.0):
    """The oracle as it stands on the whole workload (the full flat buffer and
    the step's cache rows, as the reference arm), single-threaded, as many steps
    as fit the budget (at least two)."""
    n_sample = lay.n
    step, nbytes = oracle_step_runner(lay, dt, s_g, B, n_sample)
    step(0)
    t0 = time.perf_counter()
    k = 0
    while True:
        step(k)
        k += 1
        if k >= 2 and time.perf_counter() - t0 >= budget_s:
            break
    dt_s = (time.perf_counter() - t0) / k
    return {"value": round(nbytes / dt_s / 1e9, 3), "unit": "GB/s", "cores": 1, "kind": "oracle",
            "sample": f"{k} oracle steps on the whole {lay.name} flat buffer ({n_sample:,} elements) "
                      f"+ {B} cache rows, numpy single-threaded, {dt_s:.3f} s/step"}


def _all_core_worker(q, barrier, lay, dt, s_g, B, n_slice, lo, budget_s):
    os.environ["OMP_NUM_THREADS"] = "1"
    try:
        step, nbytes = oracle_step_runner(lay, dt, s_g, B, n_slice, lo=lo, fast_inputs=True)
        step(0)
    except Exception as e:  # noqa: BLE001
        barrier.abort()
        q.put(("error", repr(e)))
        return
    try:
        barrier.wait(timeout=300)
    except Exception:  # noqa: BLE001
        q.put(("error", "barrier broken"))
        return
    t0 = time.perf_counter()
    k = 0
    while True:
        step(k)
        k += 1
        if time.perf_counter() - t0 >= budget_s:
            break
    q.put((k * nbytes, time.perf_counter() - t0))


def cpu_baseline_all_cores(lay, dt, s_g, B, budget_s=8.0, n_sample=48_000_000):
    """The same oracle in nproc independent processes, each on a disjoint slice
    of the workload's flat buffer (n_sample / nproc elements, at least 8M so a
    slice does not sit in the host caches; the oracle itself is not
    parallelised): aggregate GB/s over the concurrent processes."""
    import multiprocessing as mp
    import platform
    nproc = os.cpu_count() or 1
    model = platform.processor() or ""
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    n_slice = max(8_000_000, n_sample // nproc)   # >= 96 MB per process: past the host caches
    ctx = mp.get_context("fork")
    q, barrier = ctx.Queue(), ctx.Barrier(nproc)
    procs = [ctx.Process(target=_all_core_worker, args=(q, barrier, lay, dt, s_g, max(1, B // nproc), n_slice,
                                                       i * n_slice % max(1, lay.n - n_slice), budget_s))
             for i in range(nproc)]
    for p in procs:
        p.start()
    res = [q.get(timeout=900) for _ in procs]
    for p in procs:
        p.join()
    errs = [r[1] for r in res if r[0] == "error"]
    if errs:
        return {"error": errs[0], "cores": nproc, "kind": "oracle"}
    total_bytes = sum(b for b, _ in res)
    wall = max(t for _, t in res)
    return {"value": round(total_bytes / wall / 1e9, 3), "unit": "GB/s", "cores": nproc, "kind": "oracle",
            "cpu_model": model,
            "sample": f"{nproc} concurrent oracle processes (numpy, 1 thread each), each on a disjoint "
                      f"{n_slice:,}-element slice of the {lay.name} flat buffer + B/nproc cache rows, "
                      f"{budget_s:.0f} s each"}


def run_reference(args, rank, world):
    """Reference arm: the fp64 CPU oracle as it stands, on the host cores, rank 0 only."""
    if rank != 0:
        return
    from afinputs import bert_layout
    which, dt = WORKLOADS[args.workload]
    lay = bert_layout(which)
    s_g = 2 if dt == "bf16" else 4
    B = max(1, args.cache_batch // max(1, args.gpus))
    total_budget = 150.0
    n_probe = 4_000_000
    step, nb = oracle_step_runner(lay, dt, s_g, B, n_probe)
    t = time.perf_counter()
    step(0)
    per_elem = (time.perf_counter() - t) / n_probe
    per_step = total_budget / max(1, args.steps + args.warmup)
    n_sample = int(min(lay.n, max(1_000_000, per_step / per_elem)))
    step, nbytes = oracle_step_runner(lay, dt, s_g, B, n_sample)
    for i in range(args.warmup):
        step(i)
    t0 = time.perf_counter()
    for i in range(args.steps):
        step(i)
    el = time.perf_counter() - t0
    value = nbytes * args.steps / el / 1e9
    sample = (f"each step: oracle on the first {n_sample:,} of {lay.n:,} elements of the {lay.name} "
              f"flat buffer + {B} cache rows (numpy, single-threaded)")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": "GB/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(el / args.steps * 1e3, 3), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": ("bf16" if dt == "bf16" else "f32") + "+f64", "data": "synthetic",
        "config": {"workload": args.workload, "n_elements": lay.n, "sample_elements": n_sample},
        "cpu_baseline": {"value": round(value, 4), "unit": "GB/s", "cores": 1, "kind": "oracle",
                         "sample": sample},
        "e2e": {"value": round(value, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def _free_port():
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one command for N GPUs: re-launch this script under torchrun (one rank per GPU)
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.abspath(__file__),
               *sys.argv[1:]]
        os.execv(sys.executable, cmd)
    rank, world, local = dist_env()
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if args.sweep:
        run_sweep(args, local)
        return
    if args.shard_probe_only:
        import torch
        torch.cuda.set_device(local)
        print(json.dumps({"rank_shard_p8": rank_shard_probe(args, torch.device("cuda", local))}), flush=True)
        return
    run_ours(args, rank, world, local)


if __name__ == "__main__":
    main()
