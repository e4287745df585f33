"""Plain, slow, obviously-correct CPU oracle of AutoFreeze's per-iteration
freezing hot path (arXiv 2102.01386) -- TEST INFRASTRUCTURE ONLY.

Who may use this: `tests/`, `__graft_entry__.smoke()` and `bench.py`'s
`cpu_baseline` / `--impl reference` legs.  Nothing in `paper_2102_01386_b200/`
imports it; there is no CPU fallback in the product path.

Citations: `P:n` = /root/reference/PAPER.md line n, `S:n` = SPEC.md line n,
with the section / equation / algorithm they sit in.  Readings of silent or
ambiguous points are SURVEY.md §8(c) Q1..Q25 and are listed in DESIGN.md.

What it computes (paper order, SURVEY.md §8(c) "Algorithm"):
  1. per step, Delta <- Delta + g elementwise over the active segments, in fp32
     (§3.1.1 "we accumulate gradients for each layer ($\\Delta$)";
     Alg. 1 inputs P:175; §4.5 "accumulating the gradient vectors");
  2. at the interval end, ||Delta_T,l|| = sqrt(sum_i Delta_T,l[i]^2) per segment in
     fp64 (Eq. 1 P:179/P:198 uses the norm; L2 reading Q2);
  3. eta_l = | ||Delta_{T-1,l}|| - ||Delta_{T,l}|| | / ||Delta_{T-1,l}||  (Eq. 1,
     P:198; Alg. 1), eta = 0 when the previous norm is 0 (Q7);
  4. threshold = N-th percentile of eta over the active POOL layers (Alg. 1
     P:184; N = 50 default), numpy "linear" (Q4);
  5. prefix scan: freeze while eta_l < threshold, break at the first failure
     (Alg. 1 P:182-190 `\\algorithmicbreak`; "frozen in order");
  6. roll: previous norms <- current norms, T <- T + 1, Delta reset (Q13);
     the first interval only records norms (Q9);
  7. the storage-manager cache keyed by original example id with evict-on-read
     when the frozen depth grew (§3.2, "Storage Manager").

Precision: Delta is fp32 (Q18: fp32 implied by P:44/P:96) -- numpy fp32 adds are
IEEE round-to-nearest-even, i.e. the exact fp32 result; everything after the
norm is fp64 without fused multiply-add (numpy never contracts).

Pins: every function here is checked in tests/test_oracle_pins.py against
values printed in SPEC.md, textbook
definitions (nearest-rank percentile), closed forms of the tiny dyadic config
(SURVEY.md §8(c)), exact integer arithmetic and brute force.  The paper's own
freezing behaviour on real datasets (Fig. 6) is qualitative only:
"parity unpinned" versus the paper for that part; pinned by the closed form.
"""
import math

import numpy as np

__all__ = [
    "SEG_PRE", "SEG_POOL", "SEG_HEAD", "DT_F32", "DT_BF16",
    "ACC_DELTA", "ACC_STEP_SUMSQ", "PCT_LINEAR", "PCT_NEAREST_RANK",
    "FLAG_FIRST_INTERVAL", "FLAG_SKIPPED_FEW", "FLAG_NEAR_TIE", "FLAG_NONFINITE",
    "FLAG_DRY_RUN", "CACHE_ERR_RANGE", "CACHE_ERR_OWNER", "MISS",
    "widen", "accumulate", "segment_sumsq", "layer_norm", "eta", "percentile_threshold",
    "prefix_scan", "should_cache", "active_segments", "Freezer", "Cache", "OracleStateError",
    "adamw_constants", "adamw_step", "reduce_gradients",
]

SEG_PRE, SEG_POOL, SEG_HEAD = 0, 1, 2
DT_F32, DT_BF16 = 0, 1
ACC_DELTA, ACC_STEP_SUMSQ = 0, 1
PCT_LINEAR, PCT_NEAREST_RANK = 0, 1
FLAG_FIRST_INTERVAL, FLAG_SKIPPED_FEW, FLAG_NEAR_TIE, FLAG_NONFINITE, FLAG_DRY_RUN = 1, 2, 4, 8, 16
CACHE_ERR_RANGE, CACHE_ERR_OWNER = 1, 2
MISS = -1


class OracleStateError(RuntimeError):
    pass


# ---------------------------------------------------------------- elementwise

def widen(g, grad_dtype):
    """Gradient values as fp32: bf16 bit patterns (uint16) widen exactly by a
    16-bit shift; fp32 is returned as is."""
    if grad_dtype == DT_BF16:
        return (np.asarray(g, dtype=np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32)
    return np.asarray(g, dtype=np.float32)


def accumulate(delta, g32, first):
    """One step of the per-interval accumulation Delta_T = sum_t g_t (§3.1.1,
    Alg. 1 input "accumulated gradients for current interval" P:175), in fp32.
    On the first step of an interval Delta = g (the window restarts, Q13)."""
    if first:
        delta[...] = g32
    else:
        np.add(delta, g32, out=delta)          # fp32 + fp32 -> fp32, RNE
    return delta


def segment_sumsq(x32, lo, hi):
    """sum_i x[i]^2 over x[lo:hi] in fp64: each fp32 value widens exactly and its
    square is exact in fp64; numpy's pairwise summation adds O(log n) ulps."""
    v = np.asarray(x32[lo:hi], dtype=np.float64)
    return float(np.sum(v * v))


def layer_norm(ss):
    """||Delta_l|| = sqrt(sum of squares) (Eq. 1 norm, L2 reading Q2)."""
    return math.sqrt(ss)


def eta(prev_norm, cur_norm):
    """Eq. 1 (§3.1.1; Alg. 1):
    eta_l = | ||Delta_{T-1}|| - ||Delta_T|| | / ||Delta_{T-1}||;  eta = 0 if the
    previous norm is 0 (Q7)."""
    if prev_norm == 0.0:
        return 0.0
    return abs(prev_norm - cur_norm) / prev_norm


def percentile_threshold(etas, N, method=PCT_LINEAR):
    """N-th percentile of the active layers' eta (Alg. 1 P:184 "N^th
    percentile(eta)"; "bottom N^th percentile"; N = 50 P:402).
    LINEAR: numpy's default (Hyndman-Fan 7) -- library routine (Q4).
    NEAREST_RANK: the textbook nearest-rank definition, the value of ordinal
    rank ceil(N/100 * n) in ascending order (flag reading)."""
    v = np.asarray(etas, dtype=np.float64)
    if method == PCT_LINEAR:
        return float(np.percentile(v, N))
    if method == PCT_NEAREST_RANK:
        s = sorted(v.tolist())
        rank = max(1, math.ceil(N / 100.0 * len(s)))
        return s[rank - 1]
    raise ValueError(method)


def prefix_scan(etas_active, thr):
    """Alg. 1 second loop: walk the active layers in order, freeze
    while eta_l < threshold (strict, Q6), break at the first failure."""
    k = 0
    for e in etas_active:
        if e < thr:
            k += 1
        else:
            break
    return k


def should_cache(frozen_layers, t_layer_fwd, t_batch_read):
    """Cache-vs-recompute trade-off (§3.2): caching pays
    iff the skipped forward time frozen_layers * t_layer_fwd exceeds the time to
    read the cached batch."""
    return frozen_layers * t_layer_fwd > t_batch_read


def active_segments(kinds, f):
    """Segments whose gradients are accumulated when f POOL layers are frozen:
    POOL with pool index >= f; PRE iff f == 0 (the embedding freezes with the
    first block, §4.1, Q11); HEAD always (never frozen, Q12)."""
    out, j = [], 0
    for l, k in enumerate(kinds):
        if k == SEG_POOL:
            if j >= f:
                out.append(l)
            j += 1
        elif k == SEG_PRE:
            if f == 0:
                out.append(l)
        else:
            out.append(l)
    return out


# ---------------------------------------------------------------- optimizer (NEXT 1 fusion)

def adamw_constants(lr, beta1, beta2, eps, weight_decay, step):
    """The fp32 constants of one AdamW step, each computed in fp64 from the fp32
    hyper-parameters and rounded once (the ABI's af_adamw_step contract).
    Reading: the paper fine-tunes BERT with PyTorch and names only the
    LR schedule; AdamW with decoupled weight decay is BERT's optimizer."""
    f32 = np.float32
    lr, b1, b2, eps, wd = (float(f32(x)) for x in (lr, beta1, beta2, eps, weight_decay))
    return dict(decay=f32(1.0 - lr * wd), beta1=f32(b1), omb1=f32(1.0 - b1), beta2=f32(b2), omb2=f32(1.0 - b2),
                step_size=f32(lr / (1.0 - b1 ** step)), sqrt_bc2=f32(math.sqrt(1.0 - b2 ** step)), eps=f32(eps))


def adamw_step(p, m, v, g32, c):
    """AdamW (Loshchilov & Hutter; PyTorch's order: decay, moments, bias-corrected
    update) in fp32, one IEEE rounding per operation, no fused multiply-add:
      p <- p*decay; m <- m*b1 + g*(1-b1); v <- v*b2 + (g*g)*(1-b2)
      p <- p - step_size * (m / (sqrt(v)/sqrt_bc2 + eps))       (in place)"""
    p *= c["decay"]
    m[...] = m * c["beta1"] + g32 * c["omb1"]
    v[...] = v * c["beta2"] + (g32 * g32) * c["omb2"]
    den = np.sqrt(v) / c["sqrt_bc2"] + c["eps"]
    p -= c["step_size"] * (m / den)


# ---------------------------------------------------------------- gradient sync (NEXT 1, ZeRO form)

def reduce_gradients(grads, grad_dtype, scale):
    """The data-parallel gradient the freezing test runs on (the decision
    is taken on DDP-synchronised gradients; DDP all-reduces the
    gradient every iteration): gs = fl(sum_r g_r) * scale, every rank's gradient
    widened to fp32 and added in rank order 0..P-1 with one fp32 rounding per
    add, then ONE fp32 multiply by fp32(scale) (scale = 1/P: DDP's average).
    Reading Q27 (the paper fixes neither order nor precision of the sum)."""
    s = widen(grads[0], grad_dtype).copy()
    for g in grads[1:]:
        s = s + widen(g, grad_dtype)            # fp32 + fp32 -> fp32, RNE
    return s * np.float32(scale)


# ---------------------------------------------------------------- freezing module

class Freezer:
    """The Freezing Module (Alg. 1; §3.1.1) over a flat
    gradient buffer split into segments (PRE* POOL+ HEAD*).

    `layer_norms(g, interval_end)` performs one training step's accumulation;
    at the interval end it produces the per-segment sums of squares.
    `update_and_decide()` then runs Eq. 1, the percentile and the prefix scan,
    and rolls the state.  Mirrors af_layer_norms / af_update_and_decide."""

    def __init__(self, offsets, kinds, grad_dtype=DT_F32, percentile=50.0,
                 pct_method=PCT_LINEAR, acc_mode=ACC_DELTA, tie_rel_eps=1e-5, min_active=2):
        self.offsets = [int(o) for o in offsets]
        self.kinds = [int(k) for k in kinds]
        L = len(self.kinds)
        if len(self.offsets) != L + 1 or self.offsets[0] != 0:
            raise ValueError("bad offsets")
        if any(self.offsets[i + 1] <= self.offsets[i] for i in range(L)):
            raise ValueError("offsets must be strictly increasing")
        self.pool = [l for l, k in enumerate(self.kinds) if k == SEG_POOL]
        self.grad_dtype = grad_dtype
        self.N = float(percentile)
        self.pct_method = pct_method
        self.acc_mode = acc_mode
        self.tie_rel_eps = float(tie_rel_eps)
        self.min_active = int(min_active)
        self.n = self.offsets[-1]
        self.T = 0                               # completed intervals
        self.f = 0                               # frozen POOL count (boundary)
        self.prev = np.zeros(L)                  # ||Delta_{T-1,l}||
        self.delta = np.zeros(self.n, dtype=np.float32) if acc_mode == ACC_DELTA else None
        self.ss_acc = np.zeros(L)                # STEP_SUMSQ accumulator
        self.armed = False                       # Delta holds this interval's partial sum
        self.pending = None                      # sums of squares awaiting a decision

    def seg(self, l):
        return self.offsets[l], self.offsets[l + 1]

    def layer_norms(self, g, interval_end, dry_run=False):
        g32 = widen(g, self.grad_dtype)
        if g32.shape != (self.n,):
            raise ValueError("gradient size mismatch")
        first = not self.armed
        act = active_segments(self.kinds, self.f)
        L = len(self.kinds)
        if self.acc_mode == ACC_DELTA:
            if not interval_end:
                for l in act:
                    lo, hi = self.seg(l)
                    accumulate(self.delta[lo:hi], g32[lo:hi], first)
                if not dry_run:
                    self.armed = True
                return None
            ss = np.zeros(L)
            for l in act:
                lo, hi = self.seg(l)
                dT = g32[lo:hi].copy() if first else self.delta[lo:hi] + g32[lo:hi]
                ss[l] = segment_sumsq(dT, 0, hi - lo)
        else:  # ACC_STEP_SUMSQ: the alternative reading of Q1 -- sum_t ||g_t,l||^2
            step = np.zeros(L)
            for l in act:
                lo, hi = self.seg(l)
                step[l] = segment_sumsq(g32, lo, hi)
            acc = step if first else self.ss_acc + step
            if not dry_run:
                self.ss_acc = acc
                self.armed = True
            if not interval_end:
                return None
            ss = acc.copy()
        if not dry_run:
            self.armed = False                   # lazy reset: next step starts a new interval
        self.pending = ss
        return ss

    def update_and_decide(self, dry_run=False):
        if self.pending is None:
            raise OracleStateError("update_and_decide without a preceding interval end")
        ss = self.pending
        L = len(self.kinds)
        with np.errstate(invalid="ignore"):
            norm = np.sqrt(ss)                   # IEEE correctly-rounded sqrt per segment
        et = np.array([eta(self.prev[l], norm[l]) for l in range(L)])
        T, f = self.T, self.f
        act_pool = self.pool[f:]
        n_act = len(act_pool)
        flags = FLAG_DRY_RUN if dry_run else 0
        thr = float("nan")
        k, near_seg = 0, -1
        commit = True
        if not np.all(np.isfinite(ss)):
            flags |= FLAG_NONFINITE                  # Q8: no state change
            commit = False
        elif T == 0:
            flags |= FLAG_FIRST_INTERVAL             # Q9: record norms only
        elif n_act < self.min_active:
            flags |= FLAG_SKIPPED_FEW                # Q10
        else:
            ea = [et[l] for l in act_pool]
            thr = percentile_threshold(ea, self.N, self.pct_method)
            k = prefix_scan(ea, thr)
            # near-tie window over the comparisons that decided k (Q16)
            for i in range(min(k + 1, n_act)):
                d = abs(ea[i] - thr)
                if d > 0.0 and d <= self.tie_rel_eps * thr:
                    flags |= FLAG_NEAR_TIE
                    if near_seg < 0:
                        near_seg = act_pool[i]
        f_new = f + k
        rec = dict(interval=T, boundary_before=f, boundary_after=f_new if commit else f,
                   n_active=n_act, threshold=thr, flags=flags, near_tie_seg=near_seg,
                   sumsq=ss.copy(), norm=norm, eta=et)
        if commit and not dry_run:
            self.prev = norm.copy()
            self.T = T + 1
            self.f = f_new
        if not dry_run:
            self.pending = None
        return rec

    def adamw_active(self, p, m, v, g, c):
        """The optimizer step restricted to the active segments (frozen layers have
        requires_grad=False and are not updated)."""
        g32 = widen(g, self.grad_dtype)
        for l in active_segments(self.kinds, self.f):
            lo, hi = self.seg(l)
            adamw_step(p[lo:hi], m[lo:hi], v[lo:hi], g32[lo:hi], c)

    # convenience for whole-trace tests
    def run_interval(self, grads):
        for t, g in enumerate(grads):
            self.layer_norms(g, interval_end=(t == len(grads) - 1))
        return self.update_and_decide()


# ---------------------------------------------------------------- storage manager

class Cache:
    """Storage-manager cache (§3.2): records keyed by ORIGINAL example
    id (MappingShuffled_i stays with the caller, Q21), each holding the layer-L
    output written with its depth L = frozen POOL count at write time.
    A read returns the record and evicts it when the current frozen count is
    greater than the record's depth (Q22).  With P GPUs each GPU owns
    the ids with id mod P == rank ("each GPU manages its own cache").

    capacity = I (None: every owned id fits): "When the dataset (D points) is
    larger than the disk space available, we save I points"; a put of a
    NEW id into a full store is dropped, in call order (drop-newest), so
    the store never exceeds I; rewriting an existing id (re-cache deeper) always
    succeeds, and an evict-on-read frees room (P:277 re-cache balance)."""

    def __init__(self, num_examples, row_bytes, rank=0, world=1, capacity=None):
        self.num_examples, self.row_bytes = int(num_examples), int(row_bytes)
        self.rank, self.world = int(rank), int(world)
        self.capacity = None if capacity is None else int(capacity)
        self.store = {}
        self.error_flags = 0
        self.dropped = 0

    def _check(self, i):
        if i < 0 or i >= self.num_examples:
            self.error_flags |= CACHE_ERR_RANGE
            return False
        if i % self.world != self.rank:
            self.error_flags |= CACHE_ERR_OWNER
            return False
        return True

    def put(self, ids, rows, depth):
        rows = np.asarray(rows, dtype=np.uint8).reshape(len(ids), self.row_bytes)
        for i, ex in enumerate(ids):
            ex = int(ex)
            if not self._check(ex):
                continue
            if ex not in self.store and self.capacity is not None and len(self.store) >= self.capacity:
                self.dropped += 1
                continue
            self.store[ex] = (int(depth), rows[i].copy())

    def get(self, ids, cur_boundary, out):
        depth_out = np.full(len(ids), MISS, dtype=np.int32)
        for i, ex in enumerate(ids):
            ex = int(ex)
            if not self._check(ex) or ex not in self.store:
                continue
            d, payload = self.store[ex]
            out[i] = payload
            depth_out[i] = d
            if d < cur_boundary:
                del self.store[ex]
        return depth_out
