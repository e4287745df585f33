"""GPU parity: the sm_100a path (through the C ABI) vs the fp64 oracle on the
same seeded inputs.  Run on a B200 with `pytest -m gpu`."""
import math
import os
import struct

import numpy as np
import pytest
import torch

import oracle as O
from afinputs import (bert_grad_step, bert_layout, tiny_grad_step, tiny_layout, uniform_layout,
                      f32_to_bf16_bits)
from gpu_util import canon, compare_records, delta_host, to_device_grad
from paper_2102_01386_b200 import _lib as L_

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_2102_01386_b200  # noqa: F401  (loads libautofreeze.so; fails loudly if missing)
    torch.cuda.set_device(0)


def _fm(lay, dt, **kw):
    import paper_2102_01386_b200 as af
    return af.FreezingModule(lay.offsets, lay.kinds, grad_dtype=dt, **kw)


def _oracle(lay, dt, **kw):
    m = {"percentile": kw.get("percentile", 50.0), "tie_rel_eps": kw.get("tie_rel_eps", 1e-5),
         "min_active": kw.get("min_active", 2)}
    m["pct_method"] = O.PCT_NEAREST_RANK if kw.get("pct_method") == "nearest_rank" else O.PCT_LINEAR
    m["acc_mode"] = O.ACC_STEP_SUMSQ if kw.get("acc_mode") == "step_sumsq" else O.ACC_DELTA
    return O.Freezer(lay.offsets, lay.kinds, O.DT_BF16 if dt == "bf16" else O.DT_F32, **m)


def run_both(lay, dt, step_fn, schedule, check_delta=True, fused=False, setup=None, **kw):
    """schedule = list of steps-per-interval; step_fn(T, t) -> numpy gradient.
    fused=True ends each interval with af_interval_end (the bench's launch);
    setup(fm) runs once after the context is created (debug knobs)."""
    fm, oz = _fm(lay, dt, **kw), _oracle(lay, dt, **kw)
    if setup is not None:
        setup(fm)
    n_local = lay.n
    ties, recs = 0, []
    for T, S in enumerate(schedule):
        for t in range(S):
            g = step_fn(T, t)
            end = t == S - 1
            if end and fused:
                fm.interval_end(to_device_grad(g, dt))
            else:
                fm.layer_norms(to_device_grad(g, dt), interval_end=end)
            oz.layer_norms(g, end)
            if check_delta and not end and oz.delta is not None:
                torch.cuda.synchronize()
                assert np.array_equal(delta_host(fm, n_local), oz.delta), f"Delta T={T} t={t}"
        if not fused:
            fm.update_and_decide()
        gr, orr = fm.decision(), oz.update_and_decide()
        ties += compare_records(gr, orr, lay.n_segments, tag=f"T={T}")
        recs.append((gr, orr))
    return recs, ties, fm, oz


# ---------------------------------------------------------------- closed-form tiny trace

def test_tiny_trace_matches_closed_form(golden):
    g = golden("tiny_trace.json")
    lay = tiny_layout()
    recs, ties, _, _ = run_both(lay, "f32", lambda T, t: tiny_grad_step(lay, 0, T, t), [4] * 10)
    assert [r[0]["boundary_after"] for r in recs] == g["boundary_after"]
    for T in range(1, 9):
        assert round(recs[T][0]["threshold"], 6) == pytest.approx(g["threshold_T1_to_T8"][T - 1])
    assert ties == 0


def test_tiny_trace_step_sumsq_reading():
    lay = tiny_layout()
    recs, _, _, _ = run_both(lay, "f32", lambda T, t: tiny_grad_step(lay, 0, T, t), [4] * 10,
                             acc_mode="step_sumsq")
    paper = [0, 0, 0, 1, 1, 2, 2, 2, 3, 3]
    assert [r[0]["boundary_after"] for r in recs] != paper       # Q1 discriminator


# ---------------------------------------------------------------- ragged layouts, several tiles

def _ragged_layout():
    # odd sizes: unaligned segment edges for both 8-element bf16 and 4-element fp32 vectors
    return uniform_layout(1_000_003, 7, pre=123_457, head=777)


def _decaying_step(lay, dt, seed):
    rng_scale = np.random.default_rng(seed).random(lay.n_segments) * 0.5 + 0.3

    def fn(T, t):
        rng = np.random.default_rng([seed, T, t])
        x = rng.standard_normal(lay.n).astype(np.float32)
        amp = np.repeat((rng_scale ** T).astype(np.float32), np.diff(lay.offsets))
        x *= amp * np.float32(1e-3)
        return f32_to_bf16_bits(x) if dt == "bf16" else x
    return fn


@pytest.mark.parametrize("dt", ["bf16", "f32"])
def test_ragged_multi_tile_parity(dt):
    lay = _ragged_layout()
    recs, ties, _, oz = run_both(lay, dt, _decaying_step(lay, dt, 7), [3, 1, 2, 3, 2, 4, 1, 3])
    assert max(r[0]["boundary_after"] for r in recs) >= 1      # the frozen-skip path ran
    assert oz.f == recs[-1][0]["boundary_after"]


@pytest.mark.parametrize("pct_method,N", [("linear", 25.0), ("linear", 75.0), ("nearest_rank", 50.0)])
def test_percentile_variants_parity(pct_method, N):
    lay = uniform_layout(200_000, 12, pre=5000, head=333)
    run_both(lay, "f32", _decaying_step(lay, "f32", 3), [2] * 8, percentile=N, pct_method=pct_method)


def test_step_sumsq_ragged_parity():
    lay = _ragged_layout()
    run_both(lay, "bf16", _decaying_step(lay, "bf16", 11), [2, 3, 1, 2], acc_mode="step_sumsq",
             check_delta=False)


def test_tiny_and_edge_layouts():
    # segments shorter than one vector, a single POOL, and one-element segments
    for lay in (uniform_layout(37, 5, pre=3, head=2), uniform_layout(9, 1, pre=0, head=0),
                uniform_layout(64 * 1024 + 13, 3, pre=1, head=1)):
        for dt in ("f32", "bf16"):
            run_both(lay, dt, _decaying_step(lay, dt, 5), [2, 2, 1, 3])


# ---------------------------------------------------------------- decide kernel bit-exactness

@pytest.mark.parametrize("seed", range(4))
def test_threshold_bit_identical_to_numpy(seed):
    """Inject arbitrary per-segment sums through the exchange rows: the decide
    kernel's threshold and k must equal the oracle's (numpy) bit for bit."""
    rng = np.random.default_rng(seed)
    for trial in range(25):
        n_pool = int(rng.integers(2, 60))
        lay = uniform_layout(n_pool * 16, n_pool)
        N = float(rng.choice([50.0, 25.0, 75.0, float(rng.uniform(1, 100))]))
        method = "nearest_rank" if trial % 5 == 4 else "linear"
        fm = _fm(lay, "f32", percentile=N, pct_method=method)
        oz = _oracle(lay, "f32", percentile=N, pct_method=method)
        g = torch.zeros(lay.n, device="cuda")
        rows = fm.exchange_rows()
        for T in range(3):
            ss = rng.random(n_pool) * 10.0 ** rng.integers(-6, 3)
            if T == 2 and trial % 3 == 0:
                ss[: n_pool // 2] = oz.prev[: n_pool // 2] ** 2    # exact ties at eta = 0
            fm.layer_norms(g, interval_end=True)
            rows.copy_(torch.from_numpy(ss).view(1, -1))
            fm.update_and_decide()
            gr = fm.decision()
            oz.pending = ss.copy()
            orr = oz.update_and_decide()
            assert gr["boundary_after"] == orr["boundary_after"]
            assert gr["flags"] == orr["flags"]
            assert np.array_equal(np.array(gr["norm"]), orr["norm"])
            assert np.array_equal(np.array(gr["eta"]), orr["eta"])
            if not math.isnan(orr["threshold"]):
                assert gr["threshold"] == orr["threshold"], (trial, T, N, method)


# ---------------------------------------------------------------- fused interval end

@pytest.mark.parametrize("dt,acc", [("bf16", "delta"), ("f32", "delta"), ("bf16", "step_sumsq")])
def test_fused_interval_end_equals_two_calls(dt, acc):
    """af_interval_end (one launch at world 1) == af_layer_norms(END) + af_update_and_decide,
    bit for bit, and matches the oracle."""
    lay = _ragged_layout()
    step = _decaying_step(lay, dt, 21)
    a, b = _fm(lay, dt, acc_mode=acc), _fm(lay, dt, acc_mode=acc)
    oz = _oracle(lay, dt, acc_mode=acc)
    for T, S in enumerate([2, 1, 3, 2, 2, 3, 1, 2]):
        for t in range(S):
            gnp = step(T, t)
            g = to_device_grad(gnp, dt)
            end = t == S - 1
            if end:
                a.layer_norms(g, interval_end=True)
                a.update_and_decide()
                b.interval_end(g)
            else:
                a.layer_norms(g)
                b.layer_norms(g)
            oz.layer_norms(gnp, end)
        ra, rb = a.decision(), b.decision()
        assert canon(ra) == canon(rb), T
        compare_records(rb, oz.update_and_decide(), lay.n_segments, tag=f"T={T}")
    # dry-run repetitions through the fused call commit nothing
    blob = b.get_state()
    g = to_device_grad(step(9, 0), dt)
    b.interval_end(g, dry_run=True)
    r1 = canon(b.decision())
    b.interval_end(g, dry_run=True)
    assert canon(b.decision()) == r1 and b.get_state() == blob


def test_fused_interval_end_needs_comm_when_sharded():
    import paper_2102_01386_b200 as af
    lay = tiny_layout()
    fm = _fm(lay, "f32", rank=0, world=2)
    with pytest.raises(af.AfError) as e:
        fm.interval_end(torch.zeros(lay.n, device="cuda"))
    assert e.value.status == 2


# ---------------------------------------------------------------- semantics

def test_dry_run_and_state_roundtrip():
    lay = uniform_layout(300_001, 6, pre=1001, head=55)
    step = _decaying_step(lay, "f32", 2)
    fm = _fm(lay, "f32")
    for T in range(3):
        fm.layer_norms(to_device_grad(step(T, 0), "f32"))
        fm.layer_norms(to_device_grad(step(T, 1), "f32"), interval_end=True)
        fm.update_and_decide()
    blob = fm.get_state()
    d0 = fm.decision()
    # dry-run repetitions: identical records, nothing committed
    g = to_device_grad(step(3, 0), "f32")
    recs = []
    for _ in range(3):
        fm.layer_norms(g, interval_end=True, dry_run=True)
        fm.update_and_decide(dry_run=True)
        recs.append(fm.decision())
    assert all(r["flags"] & O.FLAG_DRY_RUN for r in recs)
    assert canon(recs[0]) == canon(recs[1]) == canon(recs[2])
    assert fm.get_state() == blob
    assert recs[0]["boundary_before"] == d0["boundary_after"]
    # restore into a fresh context and continue identically
    fm2 = _fm(lay, "f32")
    fm2.set_state(blob)
    for m in (fm, fm2):
        m.layer_norms(g, interval_end=True)
        m.update_and_decide()
    assert canon(fm.decision()) == canon(fm2.decision())


def test_decide_without_interval_end_is_estate():
    import paper_2102_01386_b200 as af
    lay = tiny_layout()
    fm = _fm(lay, "f32")
    with pytest.raises(af.AfError) as e:
        fm.update_and_decide()
    assert e.value.status == 2


def test_nonfinite_gradient_leaves_state():
    lay = tiny_layout()
    fm = _fm(lay, "f32")
    g = torch.ones(lay.n, device="cuda")
    fm.layer_norms(g, interval_end=True)
    fm.update_and_decide()
    blob = fm.get_state()
    g[7] = float("inf")
    fm.layer_norms(g, interval_end=True)
    fm.update_and_decide()
    r = fm.decision()
    assert r["flags"] & O.FLAG_NONFINITE
    assert fm.get_state() == blob


def test_deterministic_bits():
    lay = _ragged_layout()
    step = _decaying_step(lay, "bf16", 9)
    outs = []
    for _ in range(2):
        fm = _fm(lay, "bf16")
        rs = []
        for T in range(4):
            fm.layer_norms(to_device_grad(step(T, 0), "bf16"))
            fm.layer_norms(to_device_grad(step(T, 1), "bf16"), interval_end=True)
            fm.update_and_decide()
            rs.append(canon(fm.decision()))
        outs.append(rs)
    assert outs[0] == outs[1]


# ---------------------------------------------------------------- fake multi-GPU on one GPU

@pytest.mark.parametrize("P", [2, 3, 8])
def test_fake_sharded_parity(P):
    """P contexts (ranks 0..P-1) on one GPU, external exchange: every rank reaches
    the bit-identical decision; matches the P = 1 oracle within the contract."""
    lay = _ragged_layout()
    step = _decaying_step(lay, "bf16", 4)
    fms = [_fm(lay, "bf16", rank=r, world=P) for r in range(P)]
    oz = _oracle(lay, "bf16")
    for T in range(5):
        for t in range(2):
            gnp = step(T, t)
            g = to_device_grad(gnp, "bf16")
            for fm in fms:
                fm.layer_norms(g, interval_end=(t == 1))
            oz.layer_norms(gnp, t == 1)
        rows = [fm.exchange_rows() for fm in fms]
        gathered = torch.stack([rows[r][r].clone() for r in range(P)])
        for fm, rw in zip(fms, rows):
            rw.copy_(gathered)
            fm.update_and_decide()
        decs = [fm.decision() for fm in fms]
        assert all(canon(d) == canon(decs[0]) for d in decs[1:])
        compare_records(decs[0], oz.update_and_decide(), lay.n_segments, tag=f"P={P} T={T}")


# ---------------------------------------------------------------- NCCL fallback route

@pytest.mark.parametrize("dt,fused", [("f32", True), ("bf16", False)])
def test_nccl_route_on_one_gpu(dt, fused):
    """The world > 1 route without peers -- streaming kernel, ncclAllGather of the
    per-segment rows, decide kernel -- forced at world == 1 (AF_DEBUG_FORCE_NCCL,
    a one-rank communicator): records match the oracle, so the fallback's calls
    and buffers are right on real hardware (P > 1 needs more GPUs)."""
    lay = uniform_layout(3_000_017, 7, pre=100_003, head=555)
    setup = lambda fm: (fm.set_comm(), fm.set_debug(L_.AF_DEBUG_FORCE_NCCL, 1))  # noqa: E731
    recs, _, fm, oz = run_both(lay, dt, _decaying_step(lay, dt, 7), [2, 1, 3, 1, 2], check_delta=True,
                               fused=fused, setup=setup)
    assert len(recs) == 5


# ---------------------------------------------------------------- wide finalize

@pytest.mark.parametrize("n,L,pre,head,dt,acc,fused", [
    (40_000_003, 150, 1_000_001, 3_333, "f32", "delta", True),    # chunks span ~120 segments
    (80_000_003, 150, 1_000_001, 3_333, "bf16", "step_sumsq", False),   # STEP_SUMSQ tiles are 32768
    (36_000_001, 2, 17, 5, "f32", "delta", False),                # segments span many chunks
    (120_000_007, 250, 999_999, 4_097, "f32", "delta", True),     # 250 segments, many pieces
])
@pytest.mark.parametrize("unstaged", [False, True])
def test_wide_finalize_parity(n, L, pre, head, dt, acc, fused, unstaged):
    """Many finalize chunks (kFinChunk tiles each, reduced by the streaming grid's
    CTAs as they run out of tiles; chunk sums + chunk-order combine).  Records
    match the oracle while the frozen prefix moves the first active tile off the
    chunk grid.  unstaged: AF_DEBUG_UNSTAGED_TAIL -- the tail path of tables whose
    pieces (chunks + segments) exceed the finalize chunk (> 10^9 fp32 elements):
    the last chunk goes through part2 like the others and the tail reads the
    pieces from global memory."""
    lay = uniform_layout(n, L, pre=pre, head=head)
    setup = (lambda fm: fm.set_debug(L_.AF_DEBUG_UNSTAGED_TAIL, 1)) if unstaged else None
    recs, _, fm, oz = run_both(lay, dt, _decaying_step(lay, dt, 41), [2, 1, 2, 1, 2, 1], check_delta=False,
                               fused=fused, acc_mode=acc, setup=setup)
    info = fm.info()
    assert info["n_fin_chunks"] > 1
    if L > 2:
        assert max(r[0]["boundary_after"] for r in recs) >= 1


# ---------------------------------------------------------------- full BASELINE sizes

@pytest.mark.parametrize("which,dt", [("base", "bf16"), ("large", "f32")])
def test_bert_full_size_parity(which, dt):
    """configs[1] / configs[2] at full size in the bench's launch configuration:
    every per-layer norm vs the oracle on the same generated gradients."""
    lay = bert_layout(which)
    step = lambda T, t: bert_grad_step(lay, 0, T, t, dtype=dt)  # noqa: E731
    recs, ties, fm, oz = run_both(lay, dt, step, [2, 2, 1], check_delta=False, fused=True)
    # Delta after one accumulate step equals the oracle's bit for bit
    g0, g1 = step(5, 0), step(5, 1)
    fm.layer_norms(to_device_grad(g0, dt))
    fm.layer_norms(to_device_grad(g1, dt))
    oz.layer_norms(g0, False)
    oz.layer_norms(g1, False)
    torch.cuda.synchronize()
    assert np.array_equal(delta_host(fm, lay.n), oz.delta)


# ---------------------------------------------------------------- activation cache

def _cache_pair(num, row_bytes, rank=0, world=1):
    import paper_2102_01386_b200 as af
    return af.ActivationCache(num, row_bytes, rank=rank, world=world), O.Cache(num, row_bytes, rank, world)


def _ids(a):
    return torch.from_numpy(np.asarray(a, dtype=np.int64)).cuda()


def test_cache_script_matches_oracle(golden):
    from afinputs import cache_rows
    g = golden("spec_examples.json")["cache_script"]
    gc, oc = _cache_pair(1000, 196_608)
    ids = np.array([3, 7, 42, 999, 0])
    rows = cache_rows(0, 1, len(ids), 196_608)
    gc.put(_ids(ids), torch.from_numpy(rows).cuda(), g["put_depth"])
    oc.put(ids, rows, g["put_depth"])
    for q, bnd in (([3, 5, 42], 4), ([3, 42, 999, 0, 7], 7), ([3, 7], 7)):
        out_g = torch.full((len(q), 196_608), 77, dtype=torch.uint8, device="cuda")
        dep_g = torch.zeros(len(q), dtype=torch.int32, device="cuda")
        gc.get(_ids(q), bnd, out_g, dep_g)
        out_o = np.full((len(q), 196_608), 77, np.uint8)
        dep_o = oc.get(q, bnd, out_o)
        assert np.array_equal(dep_g.cpu().numpy(), dep_o)
        assert np.array_equal(out_g.cpu().numpy(), out_o)
    # re-cache deeper, then hit without eviction
    gc.put(_ids([3]), torch.from_numpy(rows[:1]).cuda(), 7)
    oc.put([3], rows[:1], 7)
    dep_g = torch.zeros(1, dtype=torch.int32, device="cuda")
    out_g = torch.zeros((1, 196_608), dtype=torch.uint8, device="cuda")
    for _ in range(2):
        gc.get(_ids([3]), 7, out_g, dep_g)
        assert dep_g.item() == 7
    assert gc.status() == (0, len(oc.store))


@pytest.mark.parametrize("rank,world", [(0, 1), (1, 4)])
def test_cache_epoch_parity(rank, world):
    from afinputs import cache_rows, epoch_permutation, rank_ids
    num, rb = 3000, 4096 + 16
    gc, oc = _cache_pair(num, rb, rank, world)
    mine = rank_ids(num, rank, world)
    for epoch, (depth, bnd) in enumerate([(4, 4), (4, 7), (7, 7)]):
        perm = epoch_permutation(0, epoch, mine)
        for b0 in range(0, len(perm), 97):
            ids = perm[b0:b0 + 97]
            out_g = torch.full((len(ids), rb), 5, dtype=torch.uint8, device="cuda")
            dep_g = torch.zeros(len(ids), dtype=torch.int32, device="cuda")
            gc.get(_ids(ids), bnd, out_g, dep_g)
            out_o = np.full((len(ids), rb), 5, np.uint8)
            dep_o = oc.get(ids, bnd, out_o)
            assert np.array_equal(dep_g.cpu().numpy(), dep_o)
            assert np.array_equal(out_g.cpu().numpy(), out_o)
            miss = ids[dep_o < 0]
            rows = cache_rows(epoch, b0, len(miss), rb)
            if len(miss):
                gc.put(_ids(miss), torch.from_numpy(rows).cuda(), depth)
                oc.put(miss, rows, depth)
    assert gc.status() == (0, len(oc.store))


@pytest.mark.parametrize("rb", [16, 4096 + 16, 24_592, 196_608, 300_016])
@pytest.mark.parametrize("n", [1, 7, 150, 256, 1100])
def test_cache_chunk_choice_parity(rb, n):
    """The per-call chunk size (balanced over the grid, af_cache.cu pick_chunks)
    changes how rows split into items: bytes, depths and evict-on-read (every
    chunk of a row must have read before the record goes) vs the oracle."""
    from afinputs import cache_rows
    num = 2 * n + 5
    gc, oc = _cache_pair(num, rb)
    ids = np.random.default_rng(n).permutation(num)[:n]
    rows = cache_rows(1, n, n, rb)
    half = n // 2
    for part, depth in ((ids[:half], 2), (ids[half:], 5)):
        if len(part):
            gc.put(_ids(part), torch.from_numpy(rows[: len(part)]).cuda(), depth)
            oc.put(part, rows[: len(part)], depth)
    q = np.random.default_rng(n + 1).permutation(num)[:n]   # hits at depth 2 / 5 and misses
    for _ in range(2):                                       # second pass: the depth-2 hits were evicted
        out_g = torch.full((n, rb), 9, dtype=torch.uint8, device="cuda")
        dep_g = torch.zeros(n, dtype=torch.int32, device="cuda")
        gc.get(_ids(q), 3, out_g, dep_g)
        out_o = np.full((n, rb), 9, np.uint8)
        dep_o = oc.get(q, 3, out_o)
        assert np.array_equal(dep_g.cpu().numpy(), dep_o)
        assert np.array_equal(out_g.cpu().numpy(), out_o)
        assert gc.status() == (0, len(oc.store))


def test_cache_get_overlapping_the_interval_end():
    """AF_CACHE_OVERLAP_PREV: a get launched right behind af_interval_end starts
    during the interval end's tail (no dependency wait).  Bytes / depths equal
    the oracle's, the decisions equal a run without the flag; the flag is
    refused for tiered stores and unknown flags are rejected."""
    import ctypes as C

    import paper_2102_01386_b200 as af
    from paper_2102_01386_b200 import _lib as L
    from afinputs import cache_rows
    lay = _ragged_layout()
    step = _decaying_step(lay, "bf16", 9)
    num, rb = 4000, 24_592
    gc, oc = _cache_pair(num, rb)
    ids_all = np.random.default_rng(4).permutation(num)[:3000]
    rows = cache_rows(2, 2, len(ids_all), rb)
    gc.put(_ids(ids_all), torch.from_numpy(rows).cuda(), 3)
    oc.put(ids_all, rows, 3)
    a, b = _fm(lay, "bf16"), _fm(lay, "bf16")
    s = torch.cuda.current_stream()
    for T in range(5):
        q = np.random.default_rng(100 + T).permutation(num)[:700]
        g0, g1 = to_device_grad(step(T, 0), "bf16"), to_device_grad(step(T, 1), "bf16")
        out = torch.full((len(q), rb), 7, dtype=torch.uint8, device="cuda")
        dep = torch.zeros(len(q), dtype=torch.int32, device="cuda")
        qd = _ids(q)
        torch.cuda.synchronize()
        a.layer_norms(g0)
        a.interval_end(g1)
        gc.get(qd, 3 + (T % 2), out, dep, overlap_prev=True)      # behind the interval end's tail
        b.layer_norms(g0)
        b.interval_end(g1)
        torch.cuda.synchronize()
        out_o = np.full((len(q), rb), 7, np.uint8)
        dep_o = oc.get(q, 3 + (T % 2), out_o)
        assert np.array_equal(dep.cpu().numpy(), dep_o)
        assert np.array_equal(out.cpu().numpy(), out_o)
        assert canon(a.decision()) == canon(b.decision())
    assert gc.status() == (0, len(oc.store))
    t = af.ActivationCache(100, 4096, hbm_rows=10, host_rows=10)
    ids = _ids([1, 2])
    o = torch.empty((2, 4096), dtype=torch.uint8, device="cuda")
    d = torch.empty(2, dtype=torch.int32, device="cuda")
    st = L.lib.af_cache_get_ex(t._h, C.c_void_p(ids.data_ptr()), 2, 1, C.c_void_p(o.data_ptr()),
                               C.c_void_p(d.data_ptr()), L.AF_CACHE_OVERLAP_PREV, None)
    assert st == L.AF_ESTATE
    st = L.lib.af_cache_get_ex(gc._h, C.c_void_p(ids.data_ptr()), 2, 1, C.c_void_p(o.data_ptr()),
                               C.c_void_p(d.data_ptr()), 0x80, None)
    assert st == L.AF_EINVAL


def _freezing_schedule_step(lay, dt, seed):
    """g_t = a_l(T) z_l with the tiny config's closed-form schedule a_l(T) =
    1 + 0.9 rho_l^T (rho rising with depth): the front blocks' eta shrinks first,
    so the boundary f grows over the intervals (SURVEY.md §8(c) closed form)."""
    from afinputs import tiny_schedule_a
    z = np.random.default_rng(seed).standard_normal(lay.n).astype(np.float32) * np.float32(1e-3)
    n_pool = sum(1 for k in lay.kinds if k == 1)
    rho, j = [], 0
    for k in lay.kinds:
        if k == 1:
            rho.append(0.3 + 0.6 * j / max(1, n_pool - 1))
            j += 1
        else:
            rho.append(0.3 if k == 0 else 0.95)

    def fn(T, t):
        amp = np.repeat(np.array([tiny_schedule_a(T, r) for r in rho], np.float32), np.diff(lay.offsets))
        x = z * amp
        return f32_to_bf16_bits(x) if dt == "bf16" else x
    return fn


@pytest.mark.parametrize("delay_us", [0, 300])
def test_overlapped_get_keeps_stream_order_over_committed_intervals(delay_us):
    """AF_CACHE_OVERLAP_PREV behind COMMITTED interval ends, chained with no host
    sync and no event between the kernels (records read from the device ring at
    the end): the first accumulate of each interval follows the overlapped get
    directly and must see the boundary the interval end committed -- Delta after
    it equals the oracle's bit for bit (a stale f would overwrite the newly frozen
    segments' Delta), every decision equals the oracle's, and the boundary chain
    is continuous.  delay_us widens the window with a busy-wait in the interval
    end's last CTA before it sums and decides (AF_DEBUG_TAIL_DELAY_NS)."""
    from paper_2102_01386_b200 import _lib as L
    from afinputs import cache_rows
    lay = _ragged_layout()
    dt, S, n_int = "bf16", 3, 9
    step = _freezing_schedule_step(lay, dt, 17)
    fm, oz = _fm(lay, dt), _oracle(lay, dt)
    fm.set_debug(L.AF_DEBUG_TAIL_DELAY_NS, delay_us * 1000)
    num, rb = 4000, 24_592
    gc, oc = _cache_pair(num, rb)
    ids_all = np.random.default_rng(5).permutation(num)[:3000]
    rows = cache_rows(3, 2, len(ids_all), rb)
    gc.put(_ids(ids_all), torch.from_numpy(rows).cuda(), 3)
    oc.put(ids_all, rows, 3)
    # every input resident before the chain: no copy between the kernels
    grads = [[to_device_grad(step(T, t), dt) for t in range(S)] for T in range(n_int)]
    qs = [np.random.default_rng(200 + T).permutation(num)[:500] for T in range(n_int)]
    qds = [_ids(q) for q in qs]
    outs = [torch.full((len(q), rb), 7, dtype=torch.uint8, device="cuda") for q in qs]
    deps = [torch.zeros(len(q), dtype=torch.int32, device="cuda") for q in qs]
    snaps = []
    torch.cuda.synchronize()
    for T in range(n_int):
        for t in range(S - 1):
            fm.layer_norms(grads[T][t])
            if t == 0:
                snaps.append(fm.accum[: 4 * lay.n].clone())   # after the step right behind the get
        fm.interval_end(grads[T][S - 1], copy_record=False)
        gc.get(qds[T], 3 + (T % 2), outs[T], deps[T], overlap_prev=True)
    torch.cuda.synchronize()
    want_snaps, f_seen = [], set()
    for T in range(n_int):
        for t in range(S):
            oz.layer_norms(step(T, t), t == S - 1)
            if t == 0:
                want_snaps.append(oz.delta.copy())
        orr = oz.update_and_decide()
        gr = fm.read_record(T)
        compare_records(gr, orr, lay.n_segments, tag=f"T={T}")
        assert gr["boundary_after"] == orr["boundary_after"], T
        if T > 0:
            assert gr["boundary_before"] == fm.read_record(T - 1)["boundary_after"], T
        f_seen.add(orr["boundary_after"])
        out_o = np.full((len(qs[T]), rb), 7, np.uint8)
        dep_o = oc.get(qs[T], 3 + (T % 2), out_o)
        assert np.array_equal(deps[T].cpu().numpy(), dep_o), T
        assert np.array_equal(outs[T].cpu().numpy(), out_o), T
    assert len(f_seen) >= 3, f_seen   # the boundary moved: the ordering was exercised
    for T in range(n_int):
        got = snaps[T].view(torch.float32).cpu().numpy()
        assert np.array_equal(got, want_snaps[T]), f"Delta after the first step of interval {T}"


def test_cache_owner_and_range_errors():
    gc, oc = _cache_pair(10, 64, rank=1, world=4)
    rows = torch.zeros((4, 64), dtype=torch.uint8, device="cuda")
    gc.put(_ids([1, 5, 2, 11]), rows, 1)
    oc.put([1, 5, 2, 11], rows.cpu().numpy(), 1)
    err, valid = gc.status()
    assert err == oc.error_flags == 3 and valid == 2
    gc.put(_ids([]), rows[:0], 1)      # empty call: no-op


def test_cache_large_gather_parity():
    from afinputs import cache_rows
    num, rb = 20_000, 196_608
    gc, oc = _cache_pair(num, rb)
    ids = np.random.default_rng(1).permutation(num)[:1024]
    rows = cache_rows(3, 3, len(ids), rb)
    gc.put(_ids(ids), torch.from_numpy(rows).cuda(), 3)
    q = np.random.default_rng(2).permutation(ids)
    out = torch.empty((len(q), rb), dtype=torch.uint8, device="cuda")
    dep = torch.empty(len(q), dtype=torch.int32, device="cuda")
    gc.get(_ids(q), 3, out, dep)
    pos = {int(x): i for i, x in enumerate(ids)}
    want = rows[[pos[int(x)] for x in q]]
    assert np.array_equal(out.cpu().numpy(), want)
    assert np.all(dep.cpu().numpy() == 3)


# ---------------------------------------------------------------- NVLink one-shot exchange (NEXT 2)

def _run_peer_ranks(P, fused, intervals=5, dt="bf16"):
    lay = _ragged_layout()
    step = _decaying_step(lay, dt, 31)
    fms = [_fm(lay, dt, rank=r, world=P) for r in range(P)]
    for fm in fms:
        fm.set_peers_local(fms)
    streams = [torch.cuda.Stream() for _ in range(P)]
    oz = _oracle(lay, dt)
    for T in range(intervals):
        for t in range(2):
            gnp = step(T, t)
            g = to_device_grad(gnp, dt)
            torch.cuda.synchronize()
            for fm, s in zip(fms, streams):          # ranks run concurrently on their streams
                with torch.cuda.stream(s):
                    if t == 1 and fused:
                        fm.interval_end(g, stream=s)
                    elif t == 1:
                        fm.layer_norms(g, interval_end=True, stream=s)
                        fm.update_and_decide(stream=s)
                    else:
                        fm.layer_norms(g, stream=s)
            torch.cuda.synchronize()
            oz.layer_norms(gnp, t == 1)
        decs = [fm.decision() for fm in fms]
        assert not any(d["flags"] & 32 for d in decs), "exchange timeout"
        assert all(canon(d) == canon(decs[0]) for d in decs[1:])
        compare_records(decs[0], oz.update_and_decide(), lay.n_segments, tag=f"P={P} T={T}")
    return fms


@pytest.mark.parametrize("P", [2, 4])
@pytest.mark.parametrize("fused", [True, False])
def test_peer_exchange_ranks_on_one_gpu(P, fused):
    """P ranks in one process (concurrent streams) exchange their partials through
    each other's memory inside the interval-end kernel; identical decisions on all
    ranks, oracle parity."""
    _run_peer_ranks(P, fused)


@pytest.mark.parametrize("P,dt,fused,acc", [(P, dt, fused, "delta") for P in (2, 3, 4) for dt in ("bf16", "f32")
                                             for fused in (True, False)]
                         + [(3, "bf16", True, "step_sumsq"), (2, "f32", False, "step_sumsq")])
def test_active_suffix_shards_follow_the_boundary(P, dt, fused, acc):
    """shard_active: every interval the ranks re-split the ACTIVE suffix for the
    boundary f read on the device, so no rank idles as the prefix freezes.  P
    in-process ranks (concurrent streams, in-kernel peer exchange), several steps
    per interval: each rank's Delta over its current shard is bit-exact vs the
    oracle, decisions are identical on all ranks and match the oracle, and the
    boundary moves (so the shards do)."""
    lay = _ragged_layout()
    step = _decaying_step(lay, dt, 77)
    fms = [_fm(lay, dt, rank=r, world=P, shard_active=True, acc_mode=acc) for r in range(P)]
    for fm in fms:
        fm.set_peers_local(fms)
    streams = [torch.cuda.Stream() for _ in range(P)]
    oz = _oracle(lay, dt, acc_mode=acc)
    f_seen = set()
    for T in range(9):
        f = fms[0].decision()["boundary_after"] if T > 0 else 0
        if T in (4, 6):
            # jump the boundary (a checkpoint restore at an interval boundary): every
            # rank's shard moves to f's table; the oracle follows
            f = min(lay.n_segments - 3, f + 2)
            for fm in fms:
                blob = bytearray(fm.get_state())
                struct.pack_into("<i", blob, 24, f)
                fm.set_state(bytes(blob))
            oz.f = f
        f_seen.add(f)
        for t in range(3):
            gnp = step(T, t)
            g = to_device_grad(gnp, dt)
            torch.cuda.synchronize()
            for fm, s in zip(fms, streams):
                with torch.cuda.stream(s):
                    if t == 2 and fused:
                        fm.interval_end(g, stream=s)
                    elif t == 2:
                        fm.layer_norms(g, interval_end=True, stream=s)
                        fm.update_and_decide(stream=s)
                    else:
                        fm.layer_norms(g, stream=s)
            torch.cuda.synchronize()
            oz.layer_norms(gnp, t == 2)
            if t == 1 and acc == "delta":
                for fm in fms:
                    b, e = fm.shard_of(f)
                    dh = delta_host(fm, lay.n)
                    assert np.array_equal(dh[b:e], oz.delta[b:e]), f"Delta P={P} T={T} rank={fm.rank}"
        decs = [fm.decision() for fm in fms]
        assert not any(d["flags"] & 32 for d in decs), "exchange timeout"
        assert all(canon(d) == canon(decs[0]) for d in decs[1:])
        compare_records(decs[0], oz.update_and_decide(), lay.n_segments, tag=f"P={P} T={T}")
    assert len(f_seen) >= 4, f_seen     # the boundary moved (decisions and restores)


@pytest.mark.parametrize("P", [3, 8])
def test_active_suffix_shards_everything_frozen(P):
    """The boundary at n_pool (only HEAD active, 777 elements): with P ranks the
    active suffix is a few vectors per rank, some ranks own no tile at all; the
    interval still exchanges and records HEAD's norm, the test skips (< 2 active
    POOL), matching the oracle."""
    lay = _ragged_layout()
    n_pool = sum(1 for k in lay.kinds if k == 1)
    step = _decaying_step(lay, "f32", 5)
    fms = [_fm(lay, "f32", rank=r, world=P, shard_active=True) for r in range(P)]
    for fm in fms:
        fm.set_peers_local(fms)
    spans = [fm.shard_of(n_pool) for fm in fms]
    assert spans[0][0] == lay.offsets[-2] and spans[-1][1] == lay.n
    oz = _oracle(lay, "f32")
    streams = [torch.cuda.Stream() for _ in range(P)]
    for T in range(3):
        if T == 1:
            for fm in fms:
                blob = bytearray(fm.get_state())
                struct.pack_into("<i", blob, 24, n_pool)
                fm.set_state(bytes(blob))
            oz.f = n_pool
        for t in range(2):
            gnp = step(T, t)
            g = to_device_grad(gnp, "f32")
            torch.cuda.synchronize()
            for fm, s in zip(fms, streams):
                with torch.cuda.stream(s):
                    if t == 1:
                        fm.interval_end(g, stream=s)
                    else:
                        fm.layer_norms(g, stream=s)
            torch.cuda.synchronize()
            oz.layer_norms(gnp, t == 1)
        decs = [fm.decision() for fm in fms]
        assert not any(d["flags"] & 32 for d in decs)
        assert all(canon(d) == canon(decs[0]) for d in decs[1:])
        compare_records(decs[0], oz.update_and_decide(), lay.n_segments, tag=f"P={P} T={T}")
    assert decs[0]["boundary_after"] == n_pool


# ---------------------------------------------------------------- tiered cache with admission (NEXT 3)

def test_cache_admission_printed_example_gpu():
    """D = 100, room for I = 60 -> exactly 60 stored, 40 dropped."""
    import paper_2102_01386_b200 as af
    gc = af.ActivationCache(100, 64, hbm_rows=40, host_rows=20)
    oc = O.Cache(100, 64, capacity=60)
    rows = torch.randint(0, 256, (100, 64), dtype=torch.uint8, device="cuda")
    gc.put(_ids(np.arange(100)), rows, 1)
    oc.put(np.arange(100), rows.cpu().numpy(), 1)
    st = gc.stats()
    assert st["n_valid"] == len(oc.store) == 60 and st["n_dropped"] == oc.dropped == 40
    assert st["n_hbm"] == 40 and st["n_host"] == 20 and st["free_slots"] == 0
    out = torch.zeros_like(rows)
    dep = torch.zeros(100, dtype=torch.int32, device="cuda")
    gc.get(_ids(np.arange(100)), 1, out, dep)
    oo = np.zeros((100, 64), np.uint8)
    do = oc.get(np.arange(100), 1, oo)
    assert np.array_equal(dep.cpu().numpy(), do) and np.array_equal(out.cpu().numpy(), oo)


@pytest.mark.parametrize("rank,world,hbm,host,disk", [(0, 1, 300, 200, 0), (2, 4, 100, 150, 0), (0, 1, 0, 400, 0),
                                                     (0, 1, 150, 100, 250), (1, 2, 0, 0, 380), (0, 1, 40, 60, 300)])
def test_tiered_cache_epochs_match_oracle(rank, world, hbm, host, disk):
    """Scripted epochs with boundary changes: evict-on-read frees slots that the
    re-cache of the same epoch reuses; drops, depths and bytes match the capacity
    oracle (I = hbm + host + disk) -- with a disk tier the records routed to
    disk slots go through the staging area and the file (host callbacks), in
    passes of 64 rows."""
    import paper_2102_01386_b200 as af
    from afinputs import cache_rows, epoch_permutation, rank_ids
    num, rb = 3000, 1024 + 16
    gc = af.ActivationCache(num, rb, rank=rank, world=world, hbm_rows=hbm, host_rows=host, disk_rows=disk,
                            stage_rows=64)
    oc = O.Cache(num, rb, rank, world, capacity=hbm + host + disk)
    host = host + disk   # the assertions below count host + disk as the off-HBM tiers
    mine = rank_ids(num, rank, world)
    for epoch, (depth, bnd) in enumerate([(4, 4), (4, 7), (7, 7), (7, 9)]):
        perm = epoch_permutation(1, epoch, mine)
        for b0 in range(0, len(perm), 113):
            ids = perm[b0:b0 + 113]
            out_g = torch.full((len(ids), rb), 3, dtype=torch.uint8, device="cuda")
            dep_g = torch.zeros(len(ids), dtype=torch.int32, device="cuda")
            gc.get(_ids(ids), bnd, out_g, dep_g)
            out_o = np.full((len(ids), rb), 3, np.uint8)
            dep_o = oc.get(ids, bnd, out_o)
            assert np.array_equal(dep_g.cpu().numpy(), dep_o)
            assert np.array_equal(out_g.cpu().numpy(), out_o)
            miss = ids[dep_o < 0]
            if len(miss):
                rows = cache_rows(epoch, b0, len(miss), rb)
                gc.put(_ids(miss), torch.from_numpy(rows).cuda(), depth)
                oc.put(miss, rows, depth)
        st = gc.stats()
        assert st["n_valid"] == len(oc.store) and st["n_dropped"] == oc.dropped, (epoch, st, oc.dropped)
        assert st["n_valid"] <= hbm + host and st["n_hbm"] <= hbm and st["n_host"] + st["n_disk"] <= host
        assert st["n_valid"] + st["free_slots"] == hbm + host
        assert st["n_disk"] <= disk and (disk == 0 or epoch == 0 or st["n_disk"] > 0)
        assert st["error_flags"] == 0
    assert oc.dropped > 0                                   # admission was exercised
    if disk:
        assert os.path.getsize(gc.disk_path) == disk * rb
    gc.close()


@pytest.mark.parametrize("rows,K,N,rank,world", [(128, 768, 2304, 0, 1), (256, 128, 320, 1, 2), (128, 64, 32, 0, 1)])
def test_cache_get_gemm_parity(rows, K, N, rank, world):
    """NEXT 4: the cache get fused into the consumer GEMM's operand load
    (af_cache_get_gemm, tcgen05 + TMA).  Depths, evictions and error flags equal
    the oracle cache's get; for every hit y = record @ W^T within the bf16-output
    bound (half an ulp of bf16, <= 2^-8 relative, plus fp32 accumulation over K,
    1e-4 x sum|a||w|) of an fp64 reference; rows of misses are untouched."""
    import paper_2102_01386_b200 as af
    num, rb = 700, rows * K * 2
    gc = af.ActivationCache(num, rb, rank=rank, world=world)
    oc = O.Cache(num, rb, rank, world)
    rng = np.random.default_rng(rows + K + N)
    mine = np.arange(rank, num, world)
    put_ids = rng.permutation(mine)[:120]
    recs = (rng.random((len(put_ids), rows, K), dtype=np.float32) * 2 - 1)
    rec_bits = f32_to_bf16_bits(recs.reshape(-1)).reshape(len(put_ids), rows * K)
    rec_bytes = rec_bits.view(np.uint8)
    depths = np.where(np.arange(len(put_ids)) % 3 == 0, 2, 5)
    for d in (2, 5):
        sel = depths == d
        gc.put(_ids(put_ids[sel]), torch.from_numpy(np.ascontiguousarray(rec_bytes[sel])).cuda(), d)
        oc.put(put_ids[sel], rec_bytes[sel], d)
    w32 = (rng.random((N, K), dtype=np.float32) * 2 - 1) * np.float32(0.5)
    w_bits = f32_to_bf16_bits(w32.reshape(-1)).reshape(N, K)
    w = torch.from_numpy(w_bits.view(np.int16)).view(torch.bfloat16).cuda()
    w64 = torch.from_numpy(w_bits.astype(np.uint32) << 16).view(torch.float32).double()
    for trial, bnd in enumerate((4, 4)):            # boundary 4 > depth 2: those records evict on the first read
        q = np.concatenate([rng.permutation(put_ids)[:60], rng.permutation(np.setdiff1d(mine, put_ids))[:10]])
        if trial == 1:
            q = np.concatenate([q, [num + 3]])      # out of range: flagged, a miss
        y = torch.full((len(q) * rows, N), 3.0, dtype=torch.bfloat16, device="cuda")
        dep = torch.zeros(len(q), dtype=torch.int32, device="cuda")
        gc.get_gemm(_ids(q), bnd, w, y, dep, rows)
        out_o = np.zeros((len(q), rb), np.uint8)
        dep_o = oc.get(q, bnd, out_o)
        torch.cuda.synchronize()
        assert np.array_equal(dep.cpu().numpy(), dep_o), trial
        yh = y.float().cpu().double()
        for i in range(len(q)):
            yi = yh[i * rows:(i + 1) * rows]
            if dep_o[i] < 0:
                assert torch.all(yi == 3.0), (trial, i)
                continue
            a = torch.from_numpy(out_o[i].view(np.uint16).astype(np.uint32) << 16).view(torch.float32).double()
            a = a.view(rows, K)
            ref = a @ w64.T
            bound = ref.abs() * 2.0 ** -8 + 1e-4 * (a.abs() @ w64.abs().T) + 1e-30
            assert torch.all((yi - ref).abs() <= bound), (trial, i, float(((yi - ref).abs() / bound).max()))
    assert gc.status() == (oc.error_flags, len(oc.store))
    gc.close()


@pytest.mark.parametrize("tiered", [False, True])
def test_get_async_prefetch_parity(tiered):
    """The paper's reader (Fig. 8): the next batch's get is issued on a side
    stream while the compute stream accumulates gradients; the consumer stream
    waits on the returned event.  Bytes, depths and evictions equal the oracle's
    (tiered: HBM + host + disk tiers, every cache call on the side stream)."""
    import paper_2102_01386_b200 as af
    from afinputs import cache_rows
    num, rb = 4000, 8192
    kw = dict(hbm_rows=300, host_rows=300, disk_rows=600, stage_rows=128) if tiered else {}
    gc = af.ActivationCache(num, rb, **kw)
    oc = O.Cache(num, rb, capacity=1200 if tiered else None)
    side = torch.cuda.Stream()
    main = torch.cuda.current_stream()
    ids_all = np.random.default_rng(8).permutation(num)[:1100]
    rows = cache_rows(4, 4, len(ids_all), rb)
    rows_d, ids_d = torch.from_numpy(rows).cuda(), _ids(ids_all)
    side.wait_stream(main)
    gc.put(ids_d, rows_d, 3, stream=side)
    oc.put(ids_all, rows, 3)
    lay = _ragged_layout()
    fm = _fm(lay, "bf16")
    g = to_device_grad(_decaying_step(lay, "bf16", 2)(0, 0), "bf16")
    for i in range(6):
        q = np.random.default_rng(300 + i).permutation(num)[:400]
        qd = _ids(q)
        out = torch.full((len(q), rb), 9, dtype=torch.uint8, device="cuda")
        dep = torch.zeros(len(q), dtype=torch.int32, device="cuda")
        side.wait_stream(main)                       # ids / outputs were made on the compute stream
        ev = gc.get_async(qd, 3 + (i % 2), out, dep, side)
        for _ in range(3):
            fm.layer_norms(g)                        # compute overlapping the prefetch
        main.wait_event(ev)
        out_o = np.full((len(q), rb), 9, np.uint8)
        dep_o = oc.get(q, 3 + (i % 2), out_o)
        assert np.array_equal(dep.cpu().numpy(), dep_o), i
        assert np.array_equal(out.cpu().numpy(), out_o), i
    side.synchronize()
    assert gc.stats()["n_valid"] == len(oc.store)
    gc.close()


def test_calibrate_should_cache_both_sides():
    """the forward-time side measured too -- a BERT-base-sized block
    stand-in (two 768x3072 projections on 32 x 128 tokens) against the read
    time of 32 records of 128 x 768 bf16; the break-even depth is the smallest k
    with k * t_fwd > t_read (af_should_cache), consistent with the two times."""
    import paper_2102_01386_b200 as af
    x = torch.randn(32 * 128, 768, device="cuda", dtype=torch.bfloat16)
    w1 = torch.randn(3072, 768, device="cuda", dtype=torch.bfloat16) * 0.02
    w2 = torch.randn(768, 3072, device="cuda", dtype=torch.bfloat16) * 0.02

    def block():
        return torch.nn.functional.linear(torch.nn.functional.gelu(torch.nn.functional.linear(x, w1)), w2)
    r = af.calibrate_should_cache(block, 128 * 768 * 2, 32, max_layers=24)
    assert r["t_layer_fwd_s"] > 0 and r["t_batch_read_s"] > 0
    k = r["min_frozen_layers"]
    if k is None:
        assert 24 * r["t_layer_fwd_s"] <= r["t_batch_read_s"]
    else:
        assert k * r["t_layer_fwd_s"] > r["t_batch_read_s"] >= (k - 1) * r["t_layer_fwd_s"]


def test_calibrate_read_seconds_and_should_cache():
    import paper_2102_01386_b200 as af
    t = af.calibrate_read_seconds(196_608, 256)
    assert 1e-6 < t < 1e-2
    assert af.should_cache(3, 0.011, t) and not af.should_cache(0, 0.011, t)


# ---------------------------------------------------------------- AdamW fused with the accumulate (NEXT 1)

@pytest.mark.parametrize("dt", ["bf16", "f32"])
def test_fused_adamw_bit_exact_and_decisions(dt):
    """af_adamw_step: params / moments / Delta bit-exact vs the fp32 oracle
    (same operation order, one rounding each), decisions as the oracle's, frozen
    segments left untouched."""
    lay = _ragged_layout()
    step = _decaying_step(lay, dt, 41)
    fm = _fm(lay, dt)
    oz = _oracle(lay, dt)
    rng = np.random.default_rng(3)
    p0 = rng.standard_normal(lay.n).astype(np.float32)
    P, M, V = p0.copy(), np.zeros(lay.n, np.float32), np.zeros(lay.n, np.float32)
    tp, tm, tv = (torch.from_numpy(x.copy()).cuda() for x in (P, M, V))
    k = 0
    for T, S in enumerate([2, 3, 1, 2, 2, 3, 2]):
        for t in range(S):
            k += 1
            gnp = step(T, t)
            end = t == S - 1
            c = O.adamw_constants(1e-3, 0.9, 0.999, 1e-8, 0.01, k)
            oz.adamw_active(P, M, V, gnp, c)                 # on the layers active before this step
            oz.layer_norms(gnp, end)
            fm.adamw_step(tp, tm, tv, to_device_grad(gnp, dt), lr=1e-3, step=k, weight_decay=0.01,
                          interval_end=end)
            if not end:
                torch.cuda.synchronize()
                assert np.array_equal(delta_host(fm, lay.n), oz.delta)
        compare_records(fm.decision(), oz.update_and_decide(), lay.n_segments, tag=f"T={T}")
        assert np.array_equal(tp.cpu().numpy(), P)
        assert np.array_equal(tm.cpu().numpy(), M)
        assert np.array_equal(tv.cpu().numpy(), V)
    assert oz.f >= 1                                          # frozen prefix exercised


# ---------------------------------------------------------------- cross-GPU cache get / put (NEXT 4)

def test_global_cache_get_put_across_ranks():
    """Ranks in one process (stores in each other's memory): a non-rank-affine
    batch is put and read by ANY rank through the owners' stores, with the
    owners' evict-on-read; bytes / depths / residency match one global oracle."""
    import paper_2102_01386_b200 as af
    from afinputs import cache_rows
    P, num, rb = 3, 900, 2048 + 16
    cs = [af.ActivationCache(num, rb, rank=r, world=P) for r in range(P)]
    for c in cs:
        c.set_peers_local(cs)
    oc = O.Cache(num, rb)                      # the union of the partitions
    rng = np.random.default_rng(7)
    for epoch, (depth, bnd) in enumerate([(4, 4), (4, 7), (7, 7)]):
        perm = rng.permutation(num)
        for b, b0 in enumerate(range(0, num, 100)):
            ids = perm[b0:b0 + 100]
            c = cs[b % P]                        # the batch lands on any rank
            out_g = torch.full((len(ids), rb), 1, dtype=torch.uint8, device="cuda")
            dep_g = torch.zeros(len(ids), dtype=torch.int32, device="cuda")
            c.get_global(_ids(ids), bnd, out_g, dep_g)
            out_o = np.full((len(ids), rb), 1, np.uint8)
            dep_o = oc.get(ids, bnd, out_o)
            assert np.array_equal(dep_g.cpu().numpy(), dep_o)
            assert np.array_equal(out_g.cpu().numpy(), out_o)
            miss = ids[dep_o < 0]
            if len(miss):
                rows = cache_rows(epoch, b0, len(miss), rb)
                c.put_global(_ids(miss), torch.from_numpy(rows).cuda(), depth)
                oc.put(miss, rows, depth)
        assert sum(c.status()[1] for c in cs) == len(oc.store)
        assert all(c.status()[0] == 0 for c in cs)


# ---------------------------------------------------------------- more edge cases

def _inject(fm, oz, ss_list, lay):
    """Drive both sides through intervals with injected per-segment sums."""
    g = torch.zeros(lay.n, device="cuda")
    rows = fm.exchange_rows()
    out = []
    for ss in ss_list:
        fm.layer_norms(g, interval_end=True)
        rows.copy_(torch.from_numpy(np.asarray(ss, dtype=np.float64)).view(1, -1))
        fm.update_and_decide()
        oz.pending = np.asarray(ss, dtype=np.float64).copy()
        out.append((fm.decision(), oz.update_and_decide()))
    return out


def test_near_tie_is_flagged_on_both_sides():
    """A scanned eta within 1e-5 * thr of the threshold sets NEAR_TIE with the
    same segment on both sides (Q16)."""
    lay = uniform_layout(4 * 16, 4)
    fm, oz = _fm(lay, "f32"), _oracle(lay, "f32")
    prev = np.array([1.0, 1.0, 1.0, 1.0])
    # etas (0.3 - 4e-6, 0.1, 0.3, 0.5): sorted [0.1, x, 0.3, 0.5], N = 50 ->
    # thr = (x + 0.3) / 2 = 0.3 - 2e-6, so |eta_0 - thr| = 2e-6 <= 1e-5 * thr
    cur = 1.0 - np.array([0.3 - 4e-6, 0.1, 0.3, 0.5])
    recs = _inject(fm, oz, [prev ** 2, cur ** 2], lay)
    g, o = recs[1]
    assert o["flags"] & O.FLAG_NEAR_TIE and g["flags"] & O.FLAG_NEAR_TIE
    assert g["near_tie_seg"] == o["near_tie_seg"] == 0


@pytest.mark.parametrize("fused", [False, True])
def test_near_tie_window_golden_cases(fused):
    """GPU twin of the CPU pins (tests/golden/near_tie_window.json, Q16): the same
    eta injected through the exchange rows gives bit-equal k, flags and
    near_tie_seg on the decide kernel and on the fused interval end's last CTA."""
    import json
    import os
    with open(os.path.join(os.path.dirname(__file__), "golden", "near_tie_window.json")) as fh:
        cases = json.load(fh)["cases"]
    for c in cases:
        n_pool = len(c["etas"])
        lay = uniform_layout(16 * (n_pool + 2), n_pool, pre=1, head=1)
        fm, oz = _fm(lay, "f32", percentile=c["N"]), _oracle(lay, "f32", percentile=c["N"])
        cur = np.ones(lay.n_segments)
        cur[1:1 + n_pool] = 1.0 - np.asarray(c["etas"])
        if fused:
            g = torch.zeros(lay.n, device="cuda")
            rows = fm.exchange_rows()
            recs = []
            for ss in (np.ones(lay.n_segments), cur * cur):
                # the fused launch writes its own sums into the row; inject by making
                # them the sums of a gradient: g = sqrt(ss) on the segment's first element
                gh = np.zeros(lay.n, np.float32)
                for l in range(lay.n_segments):
                    gh[lay.offsets[l]] = np.float32(math.sqrt(ss[l]))
                ss32 = np.array([float(gh[lay.offsets[l]]) ** 2 for l in range(lay.n_segments)])
                fm.interval_end(torch.from_numpy(gh).cuda())
                oz.pending = ss32
                recs.append((fm.decision(), oz.update_and_decide()))
            del rows, g
        else:
            recs = _inject(fm, oz, [np.ones(lay.n_segments), cur * cur], lay)
        gr, orr = recs[1]
        want_seg = c["near_tie_pool_index"] + 1 if c["near_tie_pool_index"] >= 0 else -1
        for r in (gr, orr):
            assert r["boundary_after"] - r["boundary_before"] == c["k"], (c["name"], fused)
            assert bool(r["flags"] & O.FLAG_NEAR_TIE) == c["near_tie"], (c["name"], fused)
            assert r["near_tie_seg"] == want_seg, (c["name"], fused)
        assert gr["flags"] == orr["flags"] and gr["threshold"] == orr["threshold"], c["name"]
        assert np.array_equal(np.array(gr["eta"][:lay.n_segments]), orr["eta"]), c["name"]


def test_min_active_and_percentile_100():
    lay = uniform_layout(5 * 16, 5)
    fm = _fm(lay, "f32", min_active=6, percentile=100.0)
    oz = _oracle(lay, "f32", min_active=6, percentile=100.0)
    recs = _inject(fm, oz, [np.ones(5), np.full(5, 0.5)], lay)
    assert recs[1][0]["flags"] & O.FLAG_SKIPPED_FEW and recs[1][1]["flags"] & O.FLAG_SKIPPED_FEW
    fm = _fm(lay, "f32", percentile=100.0)
    oz = _oracle(lay, "f32", percentile=100.0)
    for g, o in _inject(fm, oz, [np.ones(5), np.array([0.9, 0.8, 0.5, 0.7, 0.6]) ** 2], lay):
        assert g["boundary_after"] == o["boundary_after"]
        assert (math.isnan(o["threshold"]) and math.isnan(g["threshold"])) or g["threshold"] == o["threshold"]


def test_cuda_graph_replay_matches_eager():
    """The bench replays steps as CUDA graphs: a captured accumulate + interval
    end gives the same records as the same calls launched eagerly."""
    lay = _ragged_layout()
    step = _decaying_step(lay, "bf16", 17)
    g0, g1 = to_device_grad(step(1, 0), "bf16"), to_device_grad(step(1, 1), "bf16")
    eager, graphed = _fm(lay, "bf16"), _fm(lay, "bf16")
    for fm in (eager, graphed):
        fm.layer_norms(g0)
        fm.interval_end(g1)
        fm.layer_norms(g0)
    torch.cuda.synchronize()
    gph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gph):              # a dry-run interval end: identical work every replay
        graphed.interval_end(g1, dry_run=True)
    recs = []
    for _ in range(3):
        gph.replay()
        torch.cuda.synchronize()
        recs.append(canon(graphed.decision()))
    eager.interval_end(g1, dry_run=True)
    want = canon(eager.decision())
    assert all(r == want for r in recs)


def test_peer_exchange_survives_state_restore():
    """Checkpoint / resume with the one-shot exchange: restoring T, f, prev keeps
    the exchange epoch, so a replayed interval gives the same decision (no stale
    rows, no timeout)."""
    lay = _ragged_layout()
    step = _decaying_step(lay, "f32", 51)
    P = 2
    fms = [_fm(lay, "f32", rank=r, world=P) for r in range(P)]
    for fm in fms:
        fm.set_peers_local(fms)
    streams = [torch.cuda.Stream() for _ in range(P)]

    def interval(T):
        g0, g1 = to_device_grad(step(T, 0), "f32"), to_device_grad(step(T, 1), "f32")
        torch.cuda.synchronize()
        for fm, s in zip(fms, streams):
            with torch.cuda.stream(s):
                fm.layer_norms(g0, stream=s)
                fm.interval_end(g1, stream=s)
        torch.cuda.synchronize()
        return [canon(fm.decision()) for fm in fms]

    for T in range(3):
        interval(T)
    blobs = [fm.get_state() for fm in fms]
    first = interval(3)
    for fm, b in zip(fms, blobs):
        fm.set_state(b)
    again = interval(3)
    assert first == again and not any(d["flags"] & 32 for d in again)


# ---------------------------------------------------------------- randomized differential test

@pytest.mark.parametrize("seed", range(16))
def test_randomized_layouts_and_configs(seed):
    """Random layouts (up to AF_MAX_SEGMENTS segments, sub-vector segments,
    with/without PRE and HEAD), dtypes, accumulation readings, percentiles and
    interval lengths, optionally sharded over P fake ranks: every record matches
    the oracle within the contract and Delta stays bit-exact."""
    rng = np.random.default_rng(1000 + seed)
    L = int(rng.choice([1, 2, 7, 64, 200, 254]))
    pre = int(rng.integers(0, 2)) * int(rng.integers(1, 50_000))
    head = int(rng.integers(0, 2)) * int(rng.integers(1, 3_000))
    n = pre + head + L * int(rng.integers(3, 3_000))
    lay = uniform_layout(n, L, pre=pre, head=head)
    dt = str(rng.choice(["f32", "bf16"]))
    acc = str(rng.choice(["delta", "delta", "step_sumsq"]))
    N = float(rng.choice([25.0, 50.0, 75.0, rng.uniform(5, 95)]))
    P = int(rng.choice([1, 1, 3]))
    kw = dict(percentile=N, acc_mode=acc)
    fms = [_fm(lay, dt, rank=r, world=P, **kw) for r in range(P)]
    oz = _oracle(lay, dt, **kw)
    step = _decaying_step(lay, dt, 2000 + seed)
    for T in range(int(rng.integers(4, 8))):
        S = int(rng.integers(1, 4))
        for t in range(S):
            gnp = step(T, t)
            g = to_device_grad(gnp, dt)
            end = t == S - 1
            for fm in fms:
                if end and P == 1:
                    fm.interval_end(g)
                else:
                    fm.layer_norms(g, interval_end=end)
            oz.layer_norms(gnp, end)
            if not end and acc == "delta" and P == 1:
                torch.cuda.synchronize()
                assert np.array_equal(delta_host(fms[0], lay.n), oz.delta)
        if P > 1:
            rows = [fm.exchange_rows() for fm in fms]
            gathered = torch.stack([rows[r][r].clone() for r in range(P)])
            for fm, rw in zip(fms, rows):
                rw.copy_(gathered)
                fm.update_and_decide()
        decs = [fm.decision() for fm in fms]
        assert all(canon(d) == canon(decs[0]) for d in decs[1:])
        compare_records(decs[0], oz.update_and_decide(), lay.n_segments, tag=f"seed={seed} T={T}")


def test_maximum_segment_count_and_zero_gradients():
    """AF_MAX_SEGMENTS = 256 segments (PRE + 254 POOL + HEAD); then all-zero
    gradients: norms 0, eta 0 (Q7), threshold 0, nothing freezes (strict <), no NaN."""
    lay = uniform_layout(256 * 777 + 5, 254, pre=901, head=333)
    assert lay.n_segments == 256
    recs, _, fm, oz = run_both(lay, "bf16", _decaying_step(lay, "bf16", 77), [2, 2, 2], fused=True)
    zero = lambda T, t: np.zeros(lay.n, np.uint16)  # noqa: E731
    f0 = recs[-1][0]["boundary_after"]
    lay2 = lay
    fm2, oz2 = _fm(lay2, "bf16"), _oracle(lay2, "bf16")
    for T in range(3):
        g = to_device_grad(zero(T, 0), "bf16")
        fm2.interval_end(g)
        oz2.layer_norms(zero(T, 0), True)
        gr, orr = fm2.decision(), oz2.update_and_decide()
        compare_records(gr, orr, lay2.n_segments, tag=f"zero T={T}")
        assert gr["boundary_after"] == 0 and all(v == 0.0 for v in gr["norm"])
        assert not (gr["flags"] & O.FLAG_NONFINITE)
    assert f0 >= 0


# ---------------------------------------------------------------- maximum sizes

def test_more_than_2_31_elements_closed_form():
    """A flat buffer of 2^31 + 4777 elements (int64 offsets; element indices past
    2^31 in every kernel): per-segment constant dyadic gradients make every sum
    exact, so the record's sums of squares must equal n_l * (2 c_l)^2 exactly and
    Delta must read back c_l at the far end of the buffer."""
    import paper_2102_01386_b200 as af
    n_pre, n_a, n_b, n_head = 1000, 1 << 30, (1 << 30) + 777, 3000
    offs = np.cumsum([0, n_pre, n_a, n_b, n_head]).tolist()
    kinds = [O.SEG_PRE, O.SEG_POOL, O.SEG_POOL, O.SEG_HEAD]
    n = offs[-1]
    assert n > (1 << 31)
    cs = [2.0 ** -10, 2.0 ** -9, 2.0 ** -8, 2.0 ** -11]
    g = torch.empty(n, dtype=torch.bfloat16, device="cuda")
    for l, c in enumerate(cs):
        g[offs[l]:offs[l + 1]].fill_(c)
    fm = af.FreezingModule(offs, kinds, grad_dtype="bf16")
    fm.layer_norms(g)
    torch.cuda.synchronize()
    d = fm.accum.view(torch.float32)
    for i in (0, n_pre - 1, n_pre, (1 << 31) - 1, 1 << 31, (1 << 31) + 1, n - n_head - 1, n - 1):
        l = int(np.searchsorted(offs, i, side="right") - 1)
        assert float(d[i].item()) == cs[l], i
    fm.interval_end(g)
    rec = fm.decision()
    for l, c in enumerate(cs):
        want = (offs[l + 1] - offs[l]) * (2 * c) ** 2       # exact in fp64
        assert rec["sumsq"][l] == want, (l, rec["sumsq"][l], want)
    del g, fm
    torch.cuda.empty_cache()
