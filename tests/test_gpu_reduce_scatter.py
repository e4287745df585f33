"""GPU parity of the fused reduce-scatter + accumulate (SURVEY.md §8(f) NEXT 1,
ZeRO form; include/af.h af_reduce_scatter_step) against the oracle: P ranks
live in this process on one GPU, each on its own stream with a capped grid so
that their kernels are co-resident (the cross-GPU barriers need every rank
running), peers registered locally.  Run with `pytest -m gpu`."""
import numpy as np
import pytest
import torch

import oracle as O
from afinputs import f32_to_bf16_bits, uniform_layout
from gpu_util import canon, compare_records, delta_host, to_device_grad

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_2102_01386_b200  # noqa: F401
    torch.cuda.set_device(0)


def _rank_step(lay, dt, seed, P):
    """Per-rank gradients: rank r's sample of a decaying per-layer scale."""
    scale = np.random.default_rng(seed).random(lay.n_segments) * 0.5 + 0.3

    def fn(T, t):
        out = []
        for r in range(P):
            rng = np.random.default_rng([seed, T, t, r])
            x = rng.standard_normal(lay.n).astype(np.float32)
            x *= np.repeat((scale ** T).astype(np.float32), np.diff(lay.offsets)) * np.float32(1e-3)
            out.append(f32_to_bf16_bits(x) if dt == "bf16" else x)
        return out
    return fn


def _ranks(lay, dt, P, max_ctas):
    import paper_2102_01386_b200 as af
    fms = [af.FreezingModule(lay.offsets, lay.kinds, grad_dtype=dt, rank=r, world=P) for r in range(P)]
    tdt = torch.bfloat16 if dt == "bf16" else torch.float32
    grads = [torch.zeros(lay.n, dtype=tdt, device="cuda") for _ in range(P)]
    for fm in fms:
        if P > 1:
            fm.set_peers_local(fms)
        fm.set_grad_peers_local(grads)
        fm.set_max_ctas(max_ctas)
    return fms, grads


def _active_ranges(lay, f, sb, se):
    for l in O.active_segments(lay.kinds, f):
        lo, hi = max(lay.offsets[l], sb), min(lay.offsets[l + 1], se)
        if lo < hi:
            yield lo, hi


def _run(lay, dt, P, schedule, seed, max_ctas=None, scale=None):
    fms, grads = _ranks(lay, dt, P, max_ctas or max(1, 120 // P))
    infos = [fm.info() for fm in fms]
    outs = [torch.full((i["shard_end"] - i["shard_begin"],), float("nan"), device="cuda") for i in infos]
    streams = [torch.cuda.Stream() for _ in range(P)]
    oz = O.Freezer(lay.offsets, lay.kinds, O.DT_F32)
    code = O.DT_BF16 if dt == "bf16" else O.DT_F32
    sc = (1.0 / P) if scale is None else scale
    step = _rank_step(lay, dt, seed, P)
    recs = []
    for T, S in enumerate(schedule):
        for t in range(S):
            gnp = step(T, t)
            for g, x in zip(grads, gnp):
                g.copy_(to_device_grad(x, dt))
            torch.cuda.synchronize()
            end = t == S - 1
            f_before = oz.f
            for fm, s, o in zip(fms, streams, outs):
                with torch.cuda.stream(s):
                    fm.reduce_scatter_step(o, scale=sc, interval_end=end, stream=s)
            torch.cuda.synchronize()
            gs = O.reduce_gradients(gnp, code, sc)
            for i, o in zip(infos, outs):                      # the reduced shard, bit for bit
                sb, se = i["shard_begin"], i["shard_end"]
                oh = o.cpu().numpy()
                for lo, hi in _active_ranges(lay, f_before, sb, se):
                    assert np.array_equal(oh[lo - sb:hi - sb], gs[lo:hi]), f"rs out T={T} t={t} [{lo},{hi})"
            oz.layer_norms(gs, end)
            if not end:                                        # Delta of every shard, bit for bit
                for fm, i in zip(fms, infos):
                    sb, se = i["shard_begin"], i["shard_end"]
                    dh = delta_host(fm, se - sb)
                    for lo, hi in _active_ranges(lay, f_before, sb, se):
                        assert np.array_equal(dh[lo - sb:hi - sb], oz.delta[lo:hi]), f"Delta T={T} t={t}"
        decs = [fm.decision() for fm in fms]
        for r, d in enumerate(decs[1:], 1):
            diff = {k: (decs[0][k], d[k]) for k in d if canon(d)[k] != canon(decs[0])[k]}
            assert not diff, f"rank {r} differs from rank 0 at T={T}: {diff}"[:3000]
        compare_records(decs[0], oz.update_and_decide(), lay.n_segments, tag=f"P={P} T={T}")
        recs.append(decs[0])
    return recs, fms


# seeds chosen (with the oracle alone) so that the boundary moves on every P
@pytest.mark.parametrize("P,dt,seed", [(1, "f32", 61), (2, "bf16", 52), (3, "f32", 53), (4, "bf16", 54),
                                       (8, "f32", 58)])
def test_fused_reduce_scatter_parity(P, dt, seed):
    lay = uniform_layout(600_011, 9, pre=20_001, head=777)
    recs, _ = _run(lay, dt, P, [2, 1, 3, 2, 2, 1, 2], seed=seed)
    assert max(r["boundary_after"] for r in recs) >= 1          # frozen tiles skipped on every rank
    assert not any(r["flags"] & 32 for r in recs)              # no barrier timed out


def test_fused_reduce_scatter_wide_finalize_and_scale():
    # many finalize chunks per rank (256 interval-end tiles each; bf16 interval-end
    # tiles are 24576 elements)
    lay = uniform_layout(2 * 52_000_003, 40, pre=1_000_001, head=3_333)
    recs, fms = _run(lay, "bf16", 2, [2, 1, 2], seed=7, scale=1.0)
    assert fms[0].info()["n_fin_chunks"] > 1


def test_fused_reduce_scatter_missing_peer_times_out():
    # rank 1 never launches: rank 0's barriers time out (no hang), and its next
    # decision is flagged EXCHANGE_TIMEOUT and not committed
    lay = uniform_layout(100_003, 5, pre=1001, head=55)
    fms, grads = _ranks(lay, "f32", 2, 16)
    out = torch.zeros(fms[0].info()["shard_end"] - fms[0].info()["shard_begin"], device="cuda")
    fms[0].reduce_scatter_step(out)
    fms[0].reduce_scatter_step(out, interval_end=True)
    d = fms[0].decision()
    assert d["flags"] & 32
    assert d["interval"] == 0 and fms[0].decision()["boundary_after"] == 0


def test_reduce_scatter_argument_errors():
    import paper_2102_01386_b200 as af
    lay = uniform_layout(10_007, 3)
    fm = af.FreezingModule(lay.offsets, lay.kinds, grad_dtype="f32", rank=0, world=2)
    with pytest.raises(af.AfError):                             # nothing registered
        fm.reduce_scatter_step(None)
    g = [torch.zeros(lay.n, device="cuda") for _ in range(2)]
    fm.set_grad_peers_local(g)
    with pytest.raises(af.AfError):                             # world 2 without peers
        fm.reduce_scatter_step(None)
    st = af.FreezingModule(lay.offsets, lay.kinds, grad_dtype="f32", acc_mode="step_sumsq")
    st.set_grad_peers_local([torch.zeros(lay.n, device="cuda")])
    with pytest.raises(af.AfError):                             # STEP_SUMSQ reading
        st.reduce_scatter_step(None)


@pytest.mark.parametrize("P,dt,seed", [(2, "bf16", 52), (3, "f32", 53)])
def test_fused_reduce_scatter_adamw_parity(P, dt, seed):
    """af_reduce_scatter_adamw_step: every rank's shard of params / moments
    bit-exact vs the oracle's AdamW on the reduced gradient (its other elements
    untouched), Delta and records as the oracle's."""
    lay = uniform_layout(600_011, 9, pre=20_001, head=777)
    fms, grads = _ranks(lay, dt, P, max(1, 120 // P))
    infos = [fm.info() for fm in fms]
    rng = np.random.default_rng(seed)
    p0 = rng.standard_normal(lay.n).astype(np.float32)
    Pm, M, V = p0.copy(), np.zeros(lay.n, np.float32), np.zeros(lay.n, np.float32)
    dev = [[torch.from_numpy(x.copy()).cuda() for x in (p0, M, V)] for _ in range(P)]
    streams = [torch.cuda.Stream() for _ in range(P)]
    oz = O.Freezer(lay.offsets, lay.kinds, O.DT_F32)
    code = O.DT_BF16 if dt == "bf16" else O.DT_F32
    step = _rank_step(lay, dt, seed, P)
    k = 0
    for T, S in enumerate([2, 1, 3, 2, 2]):
        for t in range(S):
            k += 1
            gnp = step(T, t)
            for g, x in zip(grads, gnp):
                g.copy_(to_device_grad(x, dt))
            torch.cuda.synchronize()
            end = t == S - 1
            for fm, s, (tp, tm, tv) in zip(fms, streams, dev):
                with torch.cuda.stream(s):
                    fm.reduce_scatter_adamw_step(tp, tm, tv, lr=1e-3, step=k, weight_decay=0.01,
                                                 interval_end=end, stream=s)
            torch.cuda.synchronize()
            gs = O.reduce_gradients(gnp, code, 1.0 / P)
            oz.adamw_active(Pm, M, V, gs, O.adamw_constants(1e-3, 0.9, 0.999, 1e-8, 0.01, k))
            oz.layer_norms(gs, end)
        decs = [fm.decision() for fm in fms]
        compare_records(decs[0], oz.update_and_decide(), lay.n_segments, tag=f"T={T}")
        for i, (tp, tm, tv) in zip(infos, dev):
            sb, se = i["shard_begin"], i["shard_end"]
            for got, want, init in ((tp, Pm, p0), (tm, M, 0.0), (tv, V, 0.0)):
                g = got.cpu().numpy()
                assert np.array_equal(g[sb:se], want[sb:se]), f"T={T} rank shard [{sb},{se})"
                assert np.all(g[:sb] == (init[:sb] if isinstance(init, np.ndarray) else init))
                assert np.all(g[se:] == (init[se:] if isinstance(init, np.ndarray) else init))
    assert oz.f >= 1


@pytest.mark.parametrize("seed", range(8))
def test_fused_reduce_scatter_randomized(seed):
    """Random layouts (sub-vector segments, with/without PRE and HEAD), dtypes,
    world sizes 1..8 (every PM instantiation, P < PM included), scales and
    interval lengths: the reduced shards and Delta bit-exact, records as the
    oracle's, identical on every rank."""
    rng = np.random.default_rng(3000 + seed)
    L = int(rng.choice([1, 2, 5, 33, 120]))
    pre = int(rng.integers(0, 2)) * int(rng.integers(1, 20_000))
    head = int(rng.integers(0, 2)) * int(rng.integers(1, 2_000))
    n = pre + head + L * int(rng.integers(3, 2_500))
    lay = uniform_layout(n, L, pre=pre, head=head)
    dt = str(rng.choice(["f32", "bf16"]))
    P = int(rng.integers(1, 9))
    scale = float(rng.choice([1.0 / P, 0.375, 1.0]))
    sched = [int(rng.integers(1, 4)) for _ in range(int(rng.integers(3, 6)))]
    _run(lay, dt, P, sched, seed=4000 + seed, scale=scale)
