"""Property-based pins of the oracle (hypothesis): the percentile against its
exact-rational definition, the Alg. 1 scan's defining properties, percentile
monotonicity, nearest-rank's defining inequality, Eq. 1's range and the
cache's capacity invariant under arbitrary call sequences."""
import math
from fractions import Fraction

import numpy as np
from hypothesis import given, settings, strategies as st

import oracle as O

finite = st.floats(min_value=0.0, max_value=1e6, allow_nan=False, allow_infinity=False)
etas = st.lists(finite, min_size=1, max_size=40)
pct = st.floats(min_value=0.5, max_value=100.0, allow_nan=False)


def _type7(values, N):
    x = sorted(Fraction(v) for v in values)
    h = (len(x) - 1) * Fraction(N) / 100
    lo = math.floor(h)
    if lo >= len(x) - 1:
        return x[-1]
    return x[lo] + (h - lo) * (x[lo + 1] - x[lo])


def _type7_bound(values, N):
    """Rounding bound of the float evaluation: a few ulps of the result plus the
    error of h = (n-1)*(N/100) (~2 ulp(h)) carried by the gap it interpolates."""
    x = sorted(values)
    h = (len(x) - 1) * (N / 100.0)
    lo = min(int(math.floor(h)), len(x) - 1)
    gap = (x[lo + 1] - x[lo]) if lo + 1 < len(x) else 0.0
    want = float(_type7(values, N))
    return Fraction(4 * math.ulp(want) + 4 * math.ulp(h) * gap + 1e-300)


@settings(max_examples=300, deadline=None)
@given(etas, pct)
def test_linear_percentile_is_type7(v, N):
    got = O.percentile_threshold(v, N)
    want = _type7(v, N)
    assert abs(Fraction(got) - want) <= _type7_bound(v, N)
    assert min(v) <= got <= max(v)


@settings(max_examples=300, deadline=None)
@given(etas, finite)
def test_prefix_scan_defining_property(v, thr):
    k = O.prefix_scan(v, thr)
    assert all(e < thr for e in v[:k])
    assert k == len(v) or v[k] >= thr


@settings(max_examples=200, deadline=None)
@given(etas, pct, pct)
def test_freeze_count_monotone_in_N(v, a, b):
    lo, hi = min(a, b), max(a, b)
    k_lo = O.prefix_scan(v, O.percentile_threshold(v, lo))
    k_hi = O.prefix_scan(v, O.percentile_threshold(v, hi))
    assert k_lo <= k_hi


@settings(max_examples=200, deadline=None)
@given(etas, pct)
def test_nearest_rank_definition(v, N):
    thr = O.percentile_threshold(v, N, O.PCT_NEAREST_RANK)
    assert thr in v
    frac_le = sum(1 for e in v if e <= thr) / len(v)
    assert frac_le >= N / 100.0 - 1e-12                     # at least N % of the values are <= thr
    assert sum(1 for e in v if e < thr) / len(v) < N / 100.0 + 1e-12


@settings(max_examples=200, deadline=None)
@given(st.floats(min_value=1e-300, max_value=1e300), st.floats(min_value=0.0, max_value=1e300))
def test_eta_range_and_symmetry(prev, cur):
    e = O.eta(prev, cur)
    assert e >= 0.0
    assert e == abs(prev - cur) / prev


@settings(max_examples=60, deadline=None)
@given(st.integers(1, 30), st.lists(st.tuples(st.booleans(), st.lists(st.integers(0, 99), min_size=1, max_size=20,
                                                                          unique=True), st.integers(1, 9)),
                                    min_size=1, max_size=25))
def test_cache_never_exceeds_capacity(cap, calls):
    c = O.Cache(100, 16, capacity=cap)
    rows = np.zeros((20, 16), np.uint8)
    for is_put, ids, depth in calls:
        ids = np.array(ids)
        if is_put:
            c.put(ids, rows[:len(ids)], depth)
        else:
            c.get(ids, depth, np.zeros((len(ids), 16), np.uint8))
        assert len(c.store) <= cap
