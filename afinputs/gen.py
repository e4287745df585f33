"""Seeded synthetic inputs (no method arithmetic here; see package docstring).

Recipes (restated in DESIGN.md "Input recipe"):

* Tiny closed-form config (SURVEY.md §8(c) pins, §8(d) C1): step t of interval T
  of POOL segment l is   g = a_l(T) * z_l + (-1)^t * b * w_l,   with
  a_l(T) = round(2048 * (1 + 0.9 * rho_l^T)) / 2048, rho = (0.30, 0.55, 0.75, 0.90),
  z_l[i] = k / 1024 and w_l[i] = k' / 1024 with k, k' in [-512, 512) drawn from
  two independent splitmix64 streams, b = 2.  Every value is a dyadic rational
  with unit 2^-21 and magnitude < 2^22 units, so it is exact in fp32.
* BERT layouts: per-segment scale
  sigma_l(T) = 1e-3 * (1 + 0.9 * rho_l^T), rho = 0.30 + 0.60 * j / (B - 1) for
  block j, PRE uses block 0's rho, HEAD uses 0.95; fresh U(-1, 1) draws every
  step (numpy PCG64 keyed by (seed, T, t)); values sigma * U rounded to the
  gradient dtype (bf16 = round-to-nearest-even of the fp32 value); rows of the
  word-embedding matrix are zero except 4096 rows drawn per step (batch 32 x
  sequence 128 tokens touch at most 4096 distinct rows).
"""
import numpy as np

from .layouts import SEG_PRE, SEG_POOL, SEG_HEAD

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def splitmix64(x):
    """splitmix64 finaliser on uint64 arrays (wrapping arithmetic)."""
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = x + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return z


def hash_u64(seed, stream, seg, idx):
    """Counter-based hash of (seed, stream, seg, idx) -> uint64 (vectorised in idx)."""
    h = splitmix64(np.uint64(seed))
    h = splitmix64(h ^ np.uint64(stream))
    h = splitmix64(h ^ np.uint64(seg))
    return splitmix64(h ^ np.asarray(idx, dtype=np.uint64))


def tiny_dyadic_ints(seed, stream, seg, n):
    """Integers k in [-512, 512) from the hash stream (top 10 bits)."""
    h = hash_u64(seed, stream, seg, np.arange(n, dtype=np.uint64))
    return (h >> np.uint64(54)).astype(np.int64) - 512


TINY_RHO = (0.30, 0.55, 0.75, 0.90)


def tiny_schedule_a(T, rho):
    """a_l(T) = round(2048 * (1 + 0.9 * rho^T)) / 2048 (round half up)."""
    return np.floor(2048.0 * (1.0 + 0.9 * rho ** T) + 0.5) / 2048.0


def tiny_grad_step(layout, seed, T, t, b=2.0, rho=TINY_RHO):
    """fp32 gradient of step t in interval T for the tiny config (exact dyadics)."""
    out = np.empty(layout.n, dtype=np.float64)
    for l in range(layout.n_segments):
        n_l = layout.seg_len(l)
        z = tiny_dyadic_ints(seed, 0, l, n_l).astype(np.float64) / 1024.0
        w = tiny_dyadic_ints(seed, 1, l, n_l).astype(np.float64) / 1024.0
        a = tiny_schedule_a(T, rho[l % len(rho)])
        sgn = 1.0 if t % 2 == 0 else -1.0
        out[layout.offsets[l]:layout.offsets[l + 1]] = a * z + sgn * b * w
    g = out.astype(np.float32)
    assert np.array_equal(g.astype(np.float64), out), "tiny config must be exact in fp32"
    return g


def f32_to_bf16_bits(x):
    """Round fp32 values to bf16 (round-to-nearest-even); returns uint16 bit patterns."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    with np.errstate(over="ignore"):
        r = (u + np.uint32(0x7FFF) + ((u >> np.uint32(16)) & np.uint32(1))) >> np.uint32(16)
    return r.astype(np.uint16)


def bf16_bits_to_f32(b):
    """Exact widening of bf16 bit patterns to fp32."""
    return (np.asarray(b, dtype=np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32)


def segment_rho(layout):
    pool = [l for l, k in enumerate(layout.kinds) if k == SEG_POOL]
    B = len(pool)
    rho = np.empty(layout.n_segments)
    for l, k in enumerate(layout.kinds):
        if k == SEG_POOL:
            j = pool.index(l)
            rho[l] = 0.30 + 0.60 * (j / (B - 1) if B > 1 else 0.0)
        elif k == SEG_PRE:
            rho[l] = 0.30
        else:
            rho[l] = 0.95
    return rho


def bert_grad_step(layout, seed, T, t, dtype="bf16", sparse_rows=4096, lo=0, hi=None):
    """Synthetic gradient of step t in interval T for a BERT-style layout.

    Returns uint16 bf16 bit patterns (dtype="bf16") or float32 (dtype="f32") for
    the element range [lo, hi) of the flat buffer (default: all of it)."""
    hi = layout.n if hi is None else hi
    rng = np.random.default_rng([int(seed), int(T), int(t), 0xAF])
    u = rng.random(layout.n, dtype=np.float32)[lo:hi]
    x = u * np.float32(2.0) - np.float32(1.0)
    rho = segment_rho(layout)
    for l in range(layout.n_segments):
        b, e = max(layout.offsets[l], lo), min(layout.offsets[l + 1], hi)
        if b >= e:
            continue
        sigma = np.float32(1e-3 * (1.0 + 0.9 * rho[l] ** T))
        x[b - lo:e - lo] *= sigma
    if layout.word_emb is not None and sparse_rows is not None:
        wb, rows, hidden = layout.word_emb
        keep = np.zeros(rows, dtype=bool)
        keep[rng.choice(rows, size=min(sparse_rows, rows), replace=False)] = True
        mask = np.repeat(~keep, hidden)
        b, e = max(wb, lo), min(wb + rows * hidden, hi)
        if b < e:
            x[b - lo:e - lo][mask[b - wb:e - wb]] = 0.0
    if dtype == "bf16":
        return f32_to_bf16_bits(x)
    if dtype == "f32":
        return x
    raise ValueError(dtype)


def cache_rows(seed, tag, n_rows, row_bytes):
    """Payload rows (uint8) for cache put/get tests: hash bytes keyed by (seed, tag)."""
    rng = np.random.default_rng([int(seed), int(tag), 0xCA])
    return rng.integers(0, 256, size=(n_rows, row_bytes), dtype=np.uint8)


def rank_ids(num_examples, rank, world):
    """Example ids owned by `rank` under the id-mod-P partition."""
    return np.arange(rank, num_examples, world, dtype=np.int64)


def epoch_permutation(seed, epoch, ids):
    """MappingShuffled_epoch restricted to a rank's ids: a seeded permutation."""
    rng = np.random.default_rng([int(seed), int(epoch), 0x5F])
    return np.asarray(ids, dtype=np.int64)[rng.permutation(len(ids))]
