// af_decide.cuh -- the decision step as a block-level
// device function, shared by the standalone single-CTA decide kernel (world > 1,
// after the all-gather) and by the last CTA of the fused interval-end kernel
// (world == 1).
//
// Alg. 1 on the gathered per-segment sums of squares:
//   ss_l   = sum_r ss_all[r][l] in rank order 0..P-1 (identical on every rank)
//   norm_l = sqrt(ss_l)                                   (correctly rounded)
//   eta_l  = |norm_{T-1,l} - norm_{T,l}| / norm_{T-1,l}     Eq. 1; 0 if prev = 0 (Q7)
//   thr    = N-th percentile of eta over the active POOL  Alg. 1; numpy "linear" (Q4)
//   k      = leading active POOL layers with eta < thr    Alg. 1 P:182-190 (break at first failure)
//   f     <- f + k; prev <- norm; T <- T + 1              roll (Q13)
// All fp64 arithmetic uses explicit round-to-nearest intrinsics so nvcc cannot
// contract it into FMAs: the threshold is bit-identical to numpy.percentile
// given the same eta values.  Latency-bound: one CTA, 256 threads, L <= 256.
#pragma once
#include <cuda_runtime.h>

#include "af_internal.h"

namespace af {

constexpr int kDecideThreads = 256;

// AF_TIMING builds: %globaltimer at step i of the decision (tools/end_breakdown_probe.py)
#define AF_DMARK(i)                                                          \
  do {                                                                       \
    if (AF_TIMING && threadIdx.x == 0) p.state->dmark[(i)] = gtimer();       \
  } while (0)

// The decision's inputs from the device state -- T, f, this thread's segment's
// previous norm and the POOL map (into shared memory) -- loaded in one round trip
// by every thread of the CTA.  The fused interval end issues this at the start
// of its tail, so the loads overlap the segment sums; nothing but this CTA's own
// commit changes them before the decision.
struct DecideIn {
  int T, f;
  double pv;
  const int *pool;  // shared memory, [n_pool]
  uint32_t sticky;  // state->sticky (the caller ORs in what its own kernel flagged since)
};
static __device__ __forceinline__ DecideIn decide_load(const DecideParams &p) {
  __shared__ int s_pool[AF_MAX_SEGMENTS];
  const int t = threadIdx.x;
  DecideIn in;
  in.T = p.state->T;
  in.f = p.state->f;
  in.pv = (t < p.L) ? p.state->prev[t] : 0.0;
  in.sticky = *reinterpret_cast<const volatile uint32_t *>(&p.state->sticky);
  if (t < p.n_pool) s_pool[t] = p.pool_seg[t];
  in.pool = s_pool;
  return in;  // (s_pool is read after the caller's next __syncthreads)
}

// Alg. 1 on the gathered sums; every one of the 256 threads of the calling CTA
// must call it (it synchronises the block) after decide_load and a barrier.
// ss_sum: the rank-order sums already formed in shared memory by the caller (the
// fused interval end), or nullptr to sum the P rows of p.ss_all here.
static __device__ __noinline__ void decide_block(const DecideParams &p, const double *ss_sum, const DecideIn in) {
  __shared__ double s_eta[AF_MAX_SEGMENTS];
  __shared__ double s_act[AF_MAX_SEGMENTS];
  __shared__ double s_sorted[AF_MAX_SEGMENTS];
  __shared__ double s_thr;
  __shared__ int s_k, s_near, s_nonfinite;
  __shared__ unsigned int s_flags;

  // Latency-bound.  With ss_sum == nullptr the P exchange rows are loaded here
  // (in flight together, one L2 round trip) and summed in rank order.
  AF_DMARK(0);
  const int t = threadIdx.x;
  const int L = p.L;
  const int T = in.T;
  int f = in.f;
  const double pv = in.pv;
  const int *s_pool = in.pool;
  double ss = 0.0;
  if (t < L) {
    if (ss_sum != nullptr) {
      ss = ss_sum[t];
    } else {
      for (int r = 0; r < p.world; ++r) ss = __dadd_rn(ss, __ldcg(p.ss_all + r * L + t));
    }
  }
  f = f < 0 ? 0 : (f > p.n_pool ? p.n_pool : f);
  const int n_act = p.n_pool - f;

  if (t == 0) s_nonfinite = 0;
  __syncthreads();
  AF_DMARK(1);

  double nrm = 0.0, et = 0.0;
  if (t < L) {
    nrm = __dsqrt_rn(ss);
    et = (pv == 0.0) ? 0.0 : __ddiv_rn(fabs(__dsub_rn(pv, nrm)), pv);
    s_eta[t] = et;
    if (!isfinite(ss)) s_nonfinite = 1;  // benign race: every writer stores 1
  }
  __syncthreads();
  if (t < n_act) s_act[t] = s_eta[s_pool[f + t]];
  __syncthreads();
  AF_DMARK(2);

  // a peer never arrived: at the exchange (bit 0) or at a fused reduce-scatter barrier (bit 1)
  const bool xfail = (in.sticky & 3u) != 0u;
  const bool nonfinite = s_nonfinite != 0 || xfail;
  unsigned int flags = p.commit ? 0u : AF_DEC_DRY_RUN;
  if (xfail) flags |= AF_DEC_EXCHANGE_TIMEOUT;
  bool decide = false;
  if (s_nonfinite != 0) flags |= AF_DEC_NONFINITE;
  if (!nonfinite) {
    if (T == 0)
      flags |= AF_DEC_FIRST_INTERVAL;
    else if (n_act < p.min_active)
      flags |= AF_DEC_SKIPPED_FEW;
    else
      decide = true;
  }

  if (decide) {
    // rank sort of the active eta values (ties broken by position; values are finite)
    if (t < n_act) {
      const double v = s_act[t];
      int r = 0;
      for (int j = 0; j < n_act; ++j) {
        const double w = s_act[j];
        r += (w < v) || (w == v && j < t);
      }
      s_sorted[r] = v;
    }
    __syncthreads();
    AF_DMARK(3);
    if (t == 0) {
      const int n = n_act;
      double thr;
      if (p.pct_method == AF_PCT_NEAREST_RANK) {
        int rank = static_cast<int>(ceil(__dmul_rn(p.pct_q, static_cast<double>(n))));
        rank = rank < 1 ? 1 : (rank > n ? n : rank);
        thr = s_sorted[rank - 1];
      } else {
        // numpy "linear": h = (n-1) * (N/100); gamma = h - floor(h); two-branch lerp
        const double q = p.pct_q;  // N / 100, rounded once on the host (numpy's q)
        const double h = __dmul_rn(static_cast<double>(n - 1), q);
        if (h >= static_cast<double>(n - 1)) {
          thr = s_sorted[n - 1];
        } else {
          const double fl = floor(h);
          const int lo = static_cast<int>(fl);
          const double gm = __dsub_rn(h, fl);
          const double a = s_sorted[lo], b = s_sorted[lo + 1];
          const double dba = __dsub_rn(b, a);
          thr = (gm >= 0.5) ? __dsub_rn(b, __dmul_rn(dba, __dsub_rn(1.0, gm))) : __dadd_rn(a, __dmul_rn(dba, gm));
        }
      }
      // Alg. 1 scan with break; near-tie window over the comparisons that decide k
      // (positions 0..k).  Serial on one thread: over <= 256 values it is not what
      // the decision waits on (a parallel ballot / atomicMin form measured slower,
      // profiles/r01_v44_*).
      AF_DMARK(4);
      int k = 0, near = -1;
      unsigned int fl2 = 0;
      const double win = __dmul_rn(p.tie_rel_eps, thr);
      for (int i = 0; i < n; ++i) {
        const double e = s_act[i];
        const double dd = fabs(__dsub_rn(e, thr));
        if (dd > 0.0 && dd <= win) {
          fl2 |= AF_DEC_NEAR_TIE;
          if (near < 0) near = s_pool[f + i];
        }
        if (e < thr)
          ++k;
        else
          break;
      }
      s_thr = thr;
      s_k = k;
      s_near = near;
      s_flags = fl2;
    }
  } else if (t == 0) {
    s_thr = __longlong_as_double(0x7FF8000000000000LL);  // NaN: no threshold
    s_k = 0;
    s_near = -1;
    s_flags = 0;
  }
  __syncthreads();
  flags |= s_flags;
  const int k = nonfinite ? 0 : s_k;
  const int f_new = f + k;
  AF_DMARK(5);

  // record: device copy, ring slot and (if mapped) the caller's pinned host struct
  af_decision *recs[3] = {p.last, p.ring + (T % kRing), p.host};
  for (int q = 0; q < 3; ++q) {
    af_decision *r = recs[q];
    if (r == nullptr) continue;
    // device copies are complete; the host copy gets the header and the L used entries
    if (t < AF_MAX_SEGMENTS && (t < L || q < 2)) {
      r->sumsq[t] = (t < L) ? ss : 0.0;
      r->norm[t] = (t < L) ? nrm : 0.0;
      r->eta[t] = (t < L) ? et : 0.0;
    }
    if (t == 0) {
      r->interval = T;
      r->boundary_before = f;
      r->boundary_after = f_new;
      r->n_active = n_act;
      r->threshold = s_thr;
      r->flags = flags;
      r->near_tie_seg = s_near;
    }
  }
  AF_DMARK(6);
  // commit (not under AF_DRY_RUN, not on non-finite sums)
  if (p.commit && !nonfinite) {
    __syncthreads();  // every thread has read state->prev / T / f
    if (t < L) p.state->prev[t] = nrm;
    if (t == 0) {
      p.state->T = T + 1;
      p.state->f = f_new;
    }
  }
}


}  // namespace af
