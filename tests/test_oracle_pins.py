"""Pins of the fp64 oracle against things other than itself (CPU only).

Each test names what fixes the expected value: a printed example (SPEC.md /
PAPER.md, stored under tests/golden/ with its citation), a closed form derived
from Eq. 1 on the dyadic tiny config, exact integer or
rational arithmetic, a textbook definition, or brute force on tiny inputs.
"""
import math
from fractions import Fraction

import numpy as np
import pytest

import oracle as O
from afinputs import (tiny_layout, tiny_grad_step, tiny_dyadic_ints, tiny_schedule_a,
                      bert_layout, uniform_layout, f32_to_bf16_bits, bf16_bits_to_f32)



# ------------------------------------------------------------------ Eq. 1

def test_eta_printed_examples(golden):
    for prev, cur, want in golden("spec_examples.json")["eta"]["cases"]:
        assert O.eta(prev, cur) == want


def test_eta_zero_previous_norm_reading_q7():
    # SURVEY Q7 / SPEC S:178: a zero previous norm is defined as eta = 0.
    assert O.eta(0.0, 3.0) == 0.0


# ------------------------------------------------------------------ percentile + scan

def test_decide_printed_examples(golden):
    for c in golden("spec_examples.json")["decide"]["cases"]:
        thr = O.percentile_threshold(c["etas"], c["N"])
        assert thr == pytest.approx(c["thr"], rel=1e-15, abs=1e-16)
        assert O.prefix_scan(c["etas"], thr) == c["freeze"]


def _type7_exact(values, N):
    """Hyndman-Fan type 7 written out in exact rational arithmetic:
    h = (n-1) p, Q = x[floor h] + (h - floor h) (x[floor h + 1] - x[floor h])."""
    x = sorted(Fraction(v) for v in values)
    n = len(x)
    h = (n - 1) * Fraction(N) / 100
    lo = math.floor(h)
    if lo >= n - 1:
        return x[-1]
    return x[lo] + (h - lo) * (x[lo + 1] - x[lo])


def _type7_bound(values, N):
    """Rounding bound of the float evaluation: a few ulps of the result plus the
    error of h = (n-1)*(N/100) (~2 ulp(h)) carried by the gap it interpolates."""
    x = sorted(values)
    h = (len(x) - 1) * (N / 100.0)
    lo = min(int(math.floor(h)), len(x) - 1)
    gap = (x[lo + 1] - x[lo]) if lo + 1 < len(x) else 0.0
    want = float(_type7_exact(values, N))
    return Fraction(4 * math.ulp(want) + 4 * math.ulp(h) * gap + 1e-300)


@pytest.mark.parametrize("seed", range(20))
def test_linear_percentile_matches_exact_definition(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(2, 60))
    vals = rng.random(n) * 10.0 ** rng.integers(-6, 1)
    for N in (25.0, 50.0, 75.0, 33.3, 90.0, 100.0, 1.0):
        got = O.percentile_threshold(vals, N)
        want = _type7_exact(vals, N)
        # the float computation rounds a handful of times
        assert abs(Fraction(got) - want) <= _type7_bound(vals, N)


def test_linear_percentile_dyadic_exact():
    # [0, 1, 2, 4], N = 50: h = 1.5, Q = 1 + 0.5 * (2 - 1) = 1.5 exactly.
    assert O.percentile_threshold([4.0, 0.0, 2.0, 1.0], 50) == 1.5
    # odd count, N = 50: the median itself (t = 0).
    assert O.percentile_threshold([0.3, 0.1, 0.2], 50) == 0.2


def test_nearest_rank_textbook(golden):
    g = golden("nearest_rank.json")
    for N, want in g["cases"]:
        assert O.percentile_threshold(g["values"], N, O.PCT_NEAREST_RANK) == want


def test_prefix_scan_breaks_at_first_failure():
    assert O.prefix_scan([0.1, 0.5, 0.1, 0.1], 0.3) == 1
    assert O.prefix_scan([0.1, 0.1, 0.1], 0.3) == 3
    assert O.prefix_scan([0.3], 0.3) == 0          # strict < (Q6)


# ------------------------------------------------------------------ norms / accumulation

def test_norm_pythagoras_and_ones():
    assert O.layer_norm(O.segment_sumsq(np.array([3.0, 4.0], np.float32), 0, 2)) == 5.0
    for n in (1, 7, 4096, 1 << 20):
        x = np.ones(n, np.float32)
        assert O.layer_norm(O.segment_sumsq(x, 0, n)) == math.sqrt(n)


@pytest.mark.parametrize("seed", range(5))
def test_sumsq_matches_exact_sum(seed):
    # math.fsum returns the correctly rounded exact sum of the (exact) squares.
    rng = np.random.default_rng(seed)
    x = (rng.standard_normal(100_003) * 10.0 ** rng.integers(-8, 3)).astype(np.float32)
    got = O.segment_sumsq(x, 0, len(x))
    want = math.fsum(float(v) * float(v) for v in x.astype(np.float64))
    assert got == pytest.approx(want, rel=1e-14)


def test_sumsq_integer_vectors_exact():
    rng = np.random.default_rng(3)
    k = rng.integers(-1000, 1000, size=5000)
    x = k.astype(np.float32)
    assert O.segment_sumsq(x, 0, len(x)) == float(int(np.sum(k.astype(object) ** 2)))


def test_accumulate_g_then_minus_g_is_zero():
    rng = np.random.default_rng(0)
    g = rng.standard_normal(1000).astype(np.float32)
    d = np.zeros_like(g)
    O.accumulate(d, g, True)
    O.accumulate(d, -g, False)
    assert np.all(d == 0)


def test_accumulate_matches_brute_force_fp32_loop():
    rng = np.random.default_rng(1)
    gs = [rng.standard_normal(257).astype(np.float32) for _ in range(3)]
    d = np.zeros(257, np.float32)
    for t, g in enumerate(gs):
        O.accumulate(d, g, t == 0)
    for i in range(257):
        s = np.float32(gs[0][i])
        s = np.float32(s + gs[1][i])
        s = np.float32(s + gs[2][i])
        assert d[i] == s


def test_bf16_widening_exact():
    x = np.array([1.0, -2.5, 3.140625, 0.0, -0.0, 65280.0], np.float32)
    bits = f32_to_bf16_bits(x)
    assert np.array_equal(O.widen(bits, O.DT_BF16), x)
    assert np.array_equal(bf16_bits_to_f32(bits), x)


# ------------------------------------------------------------------ closed-form tiny trace

def _tiny_closed_form_ss(lay, seed, T, mode):
    """Exact integer arithmetic: Delta_T = 4 a z (paper reading) or
    sum_t ||g_t||^2 = 4 (a^2 ||z||^2 + b^2 ||w||^2) (STEP_SUMSQ reading)."""
    out = []
    for l in range(lay.n_segments):
        n = lay.seg_len(l)
        z = tiny_dyadic_ints(seed, 0, l, n).astype(object)
        w = tiny_dyadic_ints(seed, 1, l, n).astype(object)
        a = Fraction(int(tiny_schedule_a(T, (0.30, 0.55, 0.75, 0.90)[l]) * 2048), 2048)
        zz = Fraction(int(np.sum(z * z)), 1024 ** 2)
        ww = Fraction(int(np.sum(w * w)), 1024 ** 2)
        if mode == O.ACC_DELTA:
            out.append(16 * a * a * zz)
        else:
            out.append(4 * (a * a * zz + 4 * ww))
    return out


@pytest.mark.parametrize("mode", [O.ACC_DELTA, O.ACC_STEP_SUMSQ])
def test_tiny_sumsq_closed_form(mode):
    lay = tiny_layout()
    fz = O.Freezer(lay.offsets, lay.kinds, O.DT_F32, acc_mode=mode)
    for T in range(3):
        steps = [tiny_grad_step(lay, 0, T, t) for t in range(4)]
        for t, g in enumerate(steps):
            ss = fz.layer_norms(g, interval_end=(t == 3))
        want = _tiny_closed_form_ss(lay, 0, T, mode)
        for l in range(lay.n_segments):
            assert ss[l] == pytest.approx(float(want[l]), rel=2e-16 * 30)
        fz.update_and_decide()


def test_tiny_trace_paper_reading(golden):
    g = golden("tiny_trace.json")
    lay = tiny_layout()
    fz = O.Freezer(lay.offsets, lay.kinds, O.DT_F32)
    bounds, thrs, recs = [], [], []
    for T in range(10):
        rec = fz.run_interval([tiny_grad_step(lay, 0, T, t) for t in range(4)])
        recs.append(rec)
        bounds.append(rec["boundary_after"])
        thrs.append(rec["threshold"])
    assert bounds == g["boundary_after"]
    assert recs[0]["flags"] & O.FLAG_FIRST_INTERVAL
    for T in range(1, 9):
        assert round(thrs[T], g["threshold_digits"]) == pytest.approx(g["threshold_T1_to_T8"][T - 1])
    for T in g["self_tie_T"]:
        # t = 0: the threshold is the active median itself -> not flagged (Q16)
        assert thrs[T] in [recs[T]["eta"][l] for l in range(4)]
        assert not recs[T]["flags"] & O.FLAG_NEAR_TIE
    for T in g["skipped_T"]:
        assert recs[T]["flags"] & O.FLAG_SKIPPED_FEW


def test_tiny_trace_independent_of_seed_and_perturbation(golden):
    # Delta_T = 4 a z exactly for every seed (the b w term cancels over 4 steps).
    g = golden("tiny_trace.json")
    lay = tiny_layout()
    for seed in (1, 2):
        fz = O.Freezer(lay.offsets, lay.kinds, O.DT_F32)
        bounds = [fz.run_interval([tiny_grad_step(lay, seed, T, t) for t in range(4)])["boundary_after"]
                  for T in range(10)]
        assert bounds == g["boundary_after"]


def test_q1_discriminator_readings_differ():
    # The alternative reading (sum_t ||g_t||^2) depends on b and gives another trace.
    lay = tiny_layout()
    traces = []
    for mode in (O.ACC_DELTA, O.ACC_STEP_SUMSQ):
        fz = O.Freezer(lay.offsets, lay.kinds, O.DT_F32, acc_mode=mode)
        traces.append([fz.run_interval([tiny_grad_step(lay, 0, T, t) for t in range(4)])["boundary_after"]
                       for T in range(10)])
    assert traces[0] != traces[1]


# ------------------------------------------------------------------ invariants

def _random_trace(seed, L=10, steps=3, intervals=8, N=50.0, scale=1.0, sign=1.0):
    rng = np.random.default_rng(seed)
    lay = uniform_layout(L * 64, L, pre=32, head=16)
    fz = O.Freezer(lay.offsets, lay.kinds, O.DT_F32, percentile=N)
    recs = []
    decay = rng.random(lay.n_segments) * 0.5 + 0.4
    for T in range(intervals):
        grads = []
        for t in range(steps):
            base = rng.standard_normal(lay.n)
            amp = np.repeat(decay ** T, np.diff(lay.offsets))
            grads.append((sign * scale * (base * amp)).astype(np.float32))
        recs.append(fz.run_interval(grads))
    return recs


@pytest.mark.parametrize("seed", range(6))
def test_invariants_monotone_prefix_first(seed):
    recs = _random_trace(seed)
    assert recs[0]["boundary_after"] == 0
    prev = 0
    for r in recs:
        assert r["boundary_before"] == prev
        assert r["boundary_after"] >= r["boundary_before"]
        prev = r["boundary_after"]


@pytest.mark.parametrize("seed", range(4))
def test_invariant_sign_flip_bit_identical(seed):
    a, b = _random_trace(seed), _random_trace(seed, sign=-1.0)
    for ra, rb in zip(a, b):
        assert np.array_equal(ra["sumsq"], rb["sumsq"])
        assert ra["boundary_after"] == rb["boundary_after"]


@pytest.mark.parametrize("seed", range(4))
def test_invariant_power_of_two_scaling(seed):
    # scaling every gradient by 2^k scales Delta and the norms exactly: eta bit-identical
    a, b = _random_trace(seed), _random_trace(seed, scale=2.0 ** -7)
    for ra, rb in zip(a, b):
        assert np.array_equal(ra["eta"], rb["eta"])
        assert ra["boundary_after"] == rb["boundary_after"]


def test_invariant_percentile_monotone_in_N():
    rng = np.random.default_rng(5)
    for _ in range(200):
        etas = rng.random(int(rng.integers(2, 30)))
        ks = [O.prefix_scan(etas, O.percentile_threshold(etas, N)) for N in (10, 25, 50, 75, 90, 100)]
        assert ks == sorted(ks)


def test_zero_gradient_front_layer_freezes_iff_threshold_positive():
    # Q17: a zero-gradient first POOL layer has eta = 0 and
    # freezes iff thr > 0; with strict < and 12 active layers, 6 leading zeros
    # freeze 6, 7 leading zeros make thr = 0 and freeze nothing.
    for zeros in range(0, 13):
        etas = [0.0] * zeros + [0.1 * (j + 1) for j in range(12 - zeros)]
        thr = O.percentile_threshold(etas, 50)
        k = O.prefix_scan(etas, thr)
        if zeros:
            assert (k >= 1) == (thr > 0)
        if zeros == 6:
            assert k == 6
        if zeros >= 7:
            assert k == 0


def test_embedding_frozen_with_first_block_head_never():
    lay = bert_layout("base")
    assert O.active_segments(lay.kinds, 0) == list(range(14))
    assert O.active_segments(lay.kinds, 1) == list(range(2, 14))
    assert 13 in O.active_segments(lay.kinds, 11)


# ------------------------------------------------------------------ near-tie window (Q16)

def _near_tie_case(c):
    """Drive the oracle through a first interval with every norm 1, then one with
    current norm 1 - eta per active POOL layer (one PRE and one HEAD around the pool,
    so a pool index maps to segment index + 1)."""
    n_pool = len(c["etas"])
    lay = uniform_layout(16 * (n_pool + 2), n_pool, pre=1, head=1)
    fz = O.Freezer(lay.offsets, lay.kinds, O.DT_F32, percentile=c["N"])
    fz.pending = np.ones(lay.n_segments)
    fz.update_and_decide()
    cur = np.ones(lay.n_segments)
    cur[1:1 + n_pool] = 1.0 - np.asarray(c["etas"])
    fz.pending = cur * cur
    return fz.update_and_decide()


def test_near_tie_golden_thresholds_are_the_exact_type7_values(golden):
    # the derivation in the fixture: thr is within 1e-12 of the exact rational
    # Hyndman-Fan 7 value, so the 1e-6 margins around the window hold
    for c in golden("near_tie_window.json")["cases"]:
        rec = _near_tie_case(c)
        assert abs(Fraction(rec["threshold"]) - _type7_exact(c["etas"], c["N"])) < Fraction(1, 10 ** 12), c["name"]


def test_near_tie_window_scans_up_to_and_including_the_first_failure(golden):
    """Q16 / Alg. 1: (i) a near-tie before the break is flagged; (ii) a
    first failure inside the window is flagged; (iii) a near-tie only after the
    first failure is NOT flagged; (iv) a self-tie (t = 0, distance 0) is not."""
    cases = golden("near_tie_window.json")["cases"]
    for tag in ("i_", "ii_", "iii_", "iv_"):
        assert any(c["name"].startswith(tag) for c in cases), tag
    for c in cases:
        rec = _near_tie_case(c)
        assert rec["boundary_after"] - rec["boundary_before"] == c["k"], c["name"]
        assert bool(rec["flags"] & O.FLAG_NEAR_TIE) == c["near_tie"], c["name"]
        want_seg = c["near_tie_pool_index"] + 1 if c["near_tie_pool_index"] >= 0 else -1
        assert rec["near_tie_seg"] == want_seg, c["name"]


def test_update_without_interval_end_raises():
    lay = tiny_layout()
    fz = O.Freezer(lay.offsets, lay.kinds)
    with pytest.raises(O.OracleStateError):
        fz.update_and_decide()


def test_nonfinite_leaves_state_unchanged():
    lay = tiny_layout()
    fz = O.Freezer(lay.offsets, lay.kinds)
    fz.run_interval([np.ones(lay.n, np.float32)])
    g = np.ones(lay.n, np.float32)
    g[5] = np.inf
    rec = fz.run_interval([g])
    assert rec["flags"] & O.FLAG_NONFINITE
    assert fz.T == 1 and fz.f == 0


def test_dry_run_commits_nothing():
    lay = tiny_layout()
    fz = O.Freezer(lay.offsets, lay.kinds)
    for T in range(4):
        fz.run_interval([tiny_grad_step(lay, 0, T, t) for t in range(4)])
    T0, f0, prev0 = fz.T, fz.f, fz.prev.copy()
    fz.layer_norms(tiny_grad_step(lay, 0, 4, 0), True, dry_run=True)
    rec = fz.update_and_decide(dry_run=True)
    assert rec["flags"] & O.FLAG_DRY_RUN
    assert (fz.T, fz.f) == (T0, f0) and np.array_equal(fz.prev, prev0)


# ------------------------------------------------------------------ cache + should_cache

def test_should_cache_printed(golden):
    for k, tf, tr, want in golden("spec_examples.json")["should_cache"]["cases"]:
        assert O.should_cache(k, tf, tr) == want


def test_cache_script(golden):
    g = golden("spec_examples.json")["cache_script"]
    rng = np.random.default_rng(0)
    c = O.Cache(100, 64, rank=0, world=1)
    ids = np.array([3, 7, 42])
    rows = rng.integers(0, 256, (3, 64), dtype=np.uint8)
    c.put(ids, rows, g["put_depth"])
    out = np.zeros((3, 64), np.uint8)
    d = c.get(ids, g["put_depth"], out)                    # boundary unchanged: hit, kept
    assert list(d) == [4, 4, 4] and np.array_equal(out, rows)
    miss = np.full((1, 64), 9, np.uint8)
    assert list(c.get([5], 4, miss)) == [O.MISS] and np.all(miss == 9)   # miss: untouched
    d = c.get(ids[:1], g["new_boundary"], out[:1])          # boundary 4 -> 7: returned, evicted
    assert list(d) == [4]
    assert list(c.get(ids[:1], 7, out[:1])) == [O.MISS]
    c.put(ids[:1], rows[:1], 7)                             # recompute and re-cache deeper
    assert list(c.get(ids[:1], 7, out[:1])) == [7]
    assert list(c.get(ids[:1], 7, out[:1])) == [7]          # depth == boundary: kept


def test_cache_owner_partition():
    c = O.Cache(10, 16, rank=1, world=4)
    c.put([1, 5, 2, 11], np.zeros((4, 16), np.uint8), 1)
    assert c.error_flags == O.CACHE_ERR_OWNER | O.CACHE_ERR_RANGE
    assert sorted(c.store) == [1, 5]


def test_cache_admission_printed_example():
    # S:276 [PAPER P:276]: D = 100 records, room for I = 60 -> exactly 60 stored,
    # the rest dropped without error (drop-newest in call order).
    c = O.Cache(100, 16, capacity=60)
    rows = np.zeros((100, 16), np.uint8)
    c.put(np.arange(100), rows, 1)
    assert len(c.store) == 60 and c.dropped == 40
    assert sorted(c.store) == list(range(60))


def test_cache_capacity_and_recache_balance_invariants():
    # capacity never exceeded; during a deepening epoch the records
    # written never exceed those evicted on read plus the initial free room.
    rng = np.random.default_rng(0)
    D, I = 500, 200
    c = O.Cache(D, 16, capacity=I)
    ids = rng.permutation(D)
    c.put(ids, np.zeros((D, 16), np.uint8), 2)
    assert len(c.store) == I
    free0 = I - len(c.store)
    evicted = written = 0
    for b0 in range(0, D, 50):
        batch = rng.permutation(D)[b0:b0 + 50]
        out = np.zeros((len(batch), 16), np.uint8)
        before = len(c.store)
        d = c.get(batch, 5, out)                      # boundary 2 -> 5: hits are evicted
        evicted += before - len(c.store)
        miss = batch[d < 0]
        n_before = len(c.store)
        c.put(batch, np.ones((len(batch), 16), np.uint8), 5)
        written += len(c.store) - n_before
        assert len(c.store) <= I
        assert written <= evicted + free0


# ------------------------------------------------------------------ AdamW (NEXT 1 fusion)

def test_adamw_matches_torch_library_routine():
    import torch
    rng = np.random.default_rng(0)
    n = 5000
    p0 = rng.standard_normal(n).astype(np.float32)
    p, m, v = p0.copy(), np.zeros(n, np.float32), np.zeros(n, np.float32)
    tp = torch.nn.Parameter(torch.from_numpy(p0.copy()))
    opt = torch.optim.AdamW([tp], lr=1e-3, betas=(0.9, 0.999), eps=1e-8, weight_decay=0.01)
    for step in range(1, 6):
        g = (rng.standard_normal(n) * 1e-2).astype(np.float32)
        O.adamw_step(p, m, v, g, O.adamw_constants(1e-3, 0.9, 0.999, 1e-8, 0.01, step))
        tp.grad = torch.from_numpy(g.copy())
        opt.step()
    np.testing.assert_allclose(p, tp.detach().numpy(), rtol=2e-6, atol=1e-7)


def test_adamw_first_step_closed_form():
    # zero moments, no decay: m = (1-b1) g, v = (1-b2) g^2, so the update is
    # lr * g / (|g| + eps) up to fp32 rounding
    g = np.array([1e-2, -3e-3, 2.5e-1, -1.0], np.float32)
    p = np.zeros(4, np.float32)
    m, v = np.zeros(4, np.float32), np.zeros(4, np.float32)
    O.adamw_step(p, m, v, g, O.adamw_constants(1e-3, 0.9, 0.999, 1e-8, 0.0, 1))
    want = -1e-3 * g.astype(np.float64) / (np.abs(g.astype(np.float64)) + 1e-8)
    np.testing.assert_allclose(p, want, rtol=1e-6)


# ------------------------------------------------------------------ gradient sync (NEXT 1, ZeRO form)

@pytest.mark.parametrize("P", [1, 2, 3, 8])
def test_reduce_gradients_dyadic_exact(P):
    # k/1024 with |k| < 2^20: every partial sum of <= 8 terms is exact in fp32,
    # and scale = 1/8 is a power of two -- the result is the exact rational
    rng = np.random.default_rng(P)
    ks = rng.integers(-(1 << 20) + 1, 1 << 20, size=(P, 257))
    grads = [(k / 1024.0).astype(np.float32) for k in ks]
    got = O.reduce_gradients(grads, O.DT_F32, 0.125)
    want = [Fraction(int(sum(int(x) for x in col)), 1024 * 8) for col in ks.T]
    assert all(Fraction(float(g)) == w for g, w in zip(got, want))


def test_reduce_gradients_rank_order_rounding():
    # 1 + 2^-24 rounds (ties-to-even) back to 1 in fp32: the rank-order sum
    # 1 + 2^-24 + 2^-24 is 1, whereas any other association (or an fp64 sum)
    # gives 1 + 2^-23 -- pins the order and the per-add fp32 rounding (Q27)
    e = np.float32(2.0 ** -24)
    grads = [np.array([1.0], np.float32), np.array([e], np.float32), np.array([e], np.float32)]
    assert O.reduce_gradients(grads, O.DT_F32, 1.0)[0] == np.float32(1.0)
    assert O.reduce_gradients(grads[::-1], O.DT_F32, 1.0)[0] == np.float32(1.0 + 2.0 ** -23)


def test_reduce_gradients_bf16_and_scale_rounding():
    # bf16 bit patterns widen exactly; the scale is applied once, rounded to fp32
    bits = [np.array([0x3F80, 0x4000, 0xBF80], np.uint16), np.array([0x3F80, 0x3F80, 0x3F80], np.uint16)]
    got = O.reduce_gradients(bits, O.DT_BF16, 1.0 / 3.0)
    s = np.array([2.0, 3.0, 0.0], np.float32)             # 1+1, 2+1, -1+1
    assert np.array_equal(got, s * np.float32(1.0 / 3.0))
    assert got[1] == np.float32(1.0)                      # fl(3 * fl(1/3)) = 1 in fp32
