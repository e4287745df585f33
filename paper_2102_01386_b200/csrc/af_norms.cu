// af_norms.cu -- the streaming kernels of the freezing hot path (sm_100a).
//
//   kAccum    Delta <- Delta + g (Delta <- g on the first step)      P:196 §3.1.1, §4.5
//   kEndDelta partial[tile] = sum (Delta + g)^2 in fp64, no write-back  Eq. 1 norm
//   kStepSq   partial[tile] = sum g^2 (alternative reading Q1)
//
// HBM-bound elementwise/reduction work: no tensor cores (nothing is a
// contraction).  Design:
//  * persistent grid sized from the occupancy query (148 SMs x resident CTAs),
//    each CTA's first two tiles by its index, then a dynamic tile scheduler (one
//    atomic per tile, index two tiles and descriptor one tile ahead, reset by the
//    last CTA to count itself done) -- balances the two dies;
//  * 128-bit streaming loads/stores, 4 (interval end) / 8 (accumulate) vectors in
//    flight per thread;
//  * tiles never straddle a segment, so each tile's fp64 partial belongs to one
//    layer; the partial's reduction order is fixed by the thread mapping
//    (4 fp64 lane accumulators -> xor-shuffle tree -> 8 warps in order), so the
//    result does not depend on which CTA ran the tile: deterministic, no atomics
//    on the result path;
//  * each fp32 Delta_T value widens exactly to fp64 and is squared-accumulated
//    with one DFMA (the square is exact; only the accumulation rounds), giving
//    norms good to ~1e-15 relative (eta needs < 5e-11);
//  * frozen tiles (segments before the device-resident boundary f) are skipped;
//  * the per-tile partials are reduced in chunks by the CTAs that run out of
//    tiles (fin_worker); the claimer of the last chunk runs the tail (staged in
//    shared memory while the grid's last tiles stream): per-segment sums in
//    tile order, the NVLink one-shot exchange (P > 1) and the decision
//    (af_decide.cuh) -- one launch per interval end.
//  * programmatic dependent launch: pdl_wait() before the first dependent read.
#include <cuda_runtime.h>

#include "af_decide.cuh"
#include "af_internal.h"

// Tunables (compile-time; defaults chosen from the B200 variant sweep in
// profiles/r01_v3_variants.jsonl): vectors in flight per thread
// and load cache hints.
#ifndef AF_U_END
#define AF_U_END 4
#endif
#ifndef AF_U_ACC
#define AF_U_ACC 8
#endif
#ifndef AF_U_SSQ_F32  // STEP_SUMSQ (profiles/r01_v26_variants_stepsq.jsonl)
#define AF_U_SSQ_F32 4
#endif
#ifndef AF_U_SSQ_BF16
#define AF_U_SSQ_BF16 8
#endif
#ifndef AF_G_HINT  // 0: ld.global.cs   1: ld.global.nc.L1::no_allocate.L2::256B
#define AF_G_HINT 1
#endif
#ifndef AF_D_HINT_END
#define AF_D_HINT_END 0
#endif
#ifndef AF_D_HINT_ACC  // Delta loads of the accumulate: 0 ld.global.cs, 1 ld.global.nc.L1::no_allocate.L2::256B
#define AF_D_HINT_ACC 0
#endif
#ifndef AF_D_STORE  // Delta stores: 0 st.global.cs, 1 st.global (write-back), 2 .L2::cache_hint evict_first
#define AF_D_STORE 1   // write-back: -0.8 % BERT-large step (profiles/r01_v28_variants_stores.jsonl)
#endif
#ifndef AF_P_STORE  // AdamW p / m / v stores (same encoding)
#define AF_P_STORE 0
#endif
#ifndef AF_D_STORE_ADAM  // Delta stores of the AdamW-fused kernels: streaming like p / m / v
#define AF_D_STORE_ADAM 0  // (write-back there: -4 % fp32, -14 % bf16, profiles/r01_v29_*)
#endif
#ifndef AF_MINB_END
#define AF_MINB_END 1
#endif
#ifndef AF_MINB_END_BF16  // bf16 interval end / STEP_SUMSQ: min resident CTAs per SM (register cap)
#define AF_MINB_END_BF16 1
#endif
#ifndef AF_TIMING_FIRST  // AF_TIMING builds: tmark[1] = the first CTA out of tiles instead of the last
#define AF_TIMING_FIRST 0
#endif
#ifndef AF_STATIC_FIRST  // each CTA's first two tiles by its index instead of the scheduler's atomic
#define AF_STATIC_FIRST 1
#endif
#ifndef AF_U_RS_VEC  // fused reduce-scatter: gradient vectors in flight per thread (over all ranks)
#define AF_U_RS_VEC 8
#endif
#ifndef AF_U_RS_VEC_BF16  // bf16: 4 (P = 1: 5.74 -> 6.29 TB/s; 16: 3.46, profiles/r01_v40_variants_rs.jsonl)
#define AF_U_RS_VEC_BF16 4
#endif
#ifndef AF_U_RS_VEC_END  // the same at the interval end: fp32 keeps 8, bf16 4 (P = 1: fp32
#define AF_U_RS_VEC_END 8   // 8 -> 4 is 6.76 -> 5.83 TB/s, bf16 5.81 -> 6.13 TB/s,
#endif                     // profiles/r01_v39_variants_rs.jsonl; bf16 2: 5.79)
#ifndef AF_U_RS_VEC_END_BF16
#define AF_U_RS_VEC_END_BF16 4
#endif

namespace af {
namespace {

template <int HINT>
__device__ __forceinline__ uint4 ld_stream(const uint4 *p) {
  if (HINT == 0) return __ldcs(p);
  uint4 r;
  // read-only for the kernel's lifetime: non-coherent path, no L1 allocation, 256 B L2 prefetch
  asm("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
      : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
      : "l"(p));
  return r;
}
template <int HINT>
__device__ __forceinline__ float4 ld_stream(const float4 *p) {
  if (HINT == 0) return __ldcs(p);
  const uint4 u = ld_stream<HINT>(reinterpret_cast<const uint4 *>(p));
  return make_float4(__uint_as_float(u.x), __uint_as_float(u.y), __uint_as_float(u.z), __uint_as_float(u.w));
}

template <int HINT>
__device__ __forceinline__ void st_delta(float4 *p, float4 v) {
  if (HINT == 0) {
    __stcs(p, v);
  } else if (HINT == 1) {
    *p = v;
  } else {
    uint64_t pol;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z),
                 "f"(v.w), "l"(pol)
                 : "memory");
  }
}

template <typename GT>
struct VT;
template <>
struct VT<float> {
  static constexpr int VE = 4;  // elements per 16-byte vector
};
template <>
struct VT<uint16_t> {
  static constexpr int VE = 8;
};

__device__ __forceinline__ float g_scalar(const float *g, int64_t i) { return __ldcs(g + i); }
__device__ __forceinline__ float g_scalar(const uint16_t *g, int64_t i) {
  return __uint_as_float(static_cast<uint32_t>(__ldcs(reinterpret_cast<const unsigned short *>(g) + i)) << 16);
}

template <int VE>
__device__ __forceinline__ void unpack(const uint4 &v, float (&x)[VE]);
template <>
__device__ __forceinline__ void unpack<4>(const uint4 &v, float (&x)[4]) {
  x[0] = __uint_as_float(v.x);
  x[1] = __uint_as_float(v.y);
  x[2] = __uint_as_float(v.z);
  x[3] = __uint_as_float(v.w);
}
template <>
__device__ __forceinline__ void unpack<8>(const uint4 &v, float (&x)[8]) {
  // bf16 -> fp32 is exact: the bf16 bits are the high half of the fp32 word.
  x[0] = __uint_as_float(v.x << 16);
  x[1] = __uint_as_float(v.x & 0xFFFF0000u);
  x[2] = __uint_as_float(v.y << 16);
  x[3] = __uint_as_float(v.y & 0xFFFF0000u);
  x[4] = __uint_as_float(v.z << 16);
  x[5] = __uint_as_float(v.z & 0xFFFF0000u);
  x[6] = __uint_as_float(v.w << 16);
  x[7] = __uint_as_float(v.w & 0xFFFF0000u);
}

// x^2 accumulated in fp64: exact widening, exact square, one rounding per add.
__device__ __forceinline__ double sq_acc(float x, double acc) {
  const double xd = static_cast<double>(x);
  return __fma_rn(xd, xd, acc);
}

template <int MODE, typename GT, bool RD>
__device__ __forceinline__ void elem(const NormParams &p, const GT *g, float *d, int64_t i,
                                     double &acc) {
  const float gv = g_scalar(g, i);
  if (MODE == kStepSq) {
    acc = sq_acc(gv, acc);
    return;
  }
  const float x = RD ? __fadd_rn(d[i], gv) : gv;
  if (MODE == kAccum)
    d[i] = x;
  else
    acc = sq_acc(x, acc);
}

template <int MODE, typename GT, bool RD>
__device__ __forceinline__ double process_tile(const NormParams &p, const Tile &t) {
  constexpr int VE = VT<GT>::VE;
  constexpr int U_SSQ = sizeof(GT) == 2 ? AF_U_SSQ_BF16 : AF_U_SSQ_F32;
  constexpr int U = (MODE == kAccum) ? AF_U_ACC : (MODE == kStepSq ? U_SSQ : AF_U_END);  // vectors in flight
  // Delta is rewritten by kAccum, but each element is read once, before its own
  // write, by the same thread: the non-coherent path is safe there too
  constexpr int DH = (MODE == kAccum) ? AF_D_HINT_ACC : AF_D_HINT_END;
  const GT *__restrict__ g = static_cast<const GT *>(p.grad);
  // Delta is indexed by global element i at d[i]; the shard base offset is applied
  // through the pointer (shard_begin is a multiple of 8, keeping 16 B alignment).
  float *__restrict__ d = p.delta - p.shard_begin;
  const int64_t b = t.begin, e = t.end;
  int64_t vb = ((b + VE - 1) / VE) * VE;
  int64_t ve = (e / VE) * VE;
  if (vb > ve) vb = ve = e;  // shorter than one aligned vector: all scalar
  const int tid = threadIdx.x;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;

  // unaligned segment edges (< VE elements each): scalar
  const int nh = static_cast<int>(vb - b), nt = static_cast<int>(e - ve);
  if (tid < nh) elem<MODE, GT, RD>(p, g, d, b + tid, a0);
  if (tid >= 128 && tid - 128 < nt) elem<MODE, GT, RD>(p, g, d, ve + (tid - 128), a1);

  const int64_t nch = (ve - vb) / VE;
  const uint4 *gb = reinterpret_cast<const uint4 *>(g + vb);
  float4 *db = reinterpret_cast<float4 *>(d + vb);
  constexpr int DV = VE / 4;  // float4 of Delta per vector of g
  for (int64_t c0 = tid; c0 < nch; c0 += U * kNormBlock) {
    uint4 gv[U];
    float4 dv[U][DV];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t c = c0 + static_cast<int64_t>(u) * kNormBlock;
      if (c < nch) {
        gv[u] = ld_stream<AF_G_HINT>(gb + c);
        if (RD) {
#pragma unroll
          for (int q = 0; q < DV; ++q) dv[u][q] = ld_stream<DH>(db + c * DV + q);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t c = c0 + static_cast<int64_t>(u) * kNormBlock;
      if (c < nch) {
        float x[VE];
        unpack<VE>(gv[u], x);
        if (MODE == kStepSq) {
#pragma unroll
          for (int k = 0; k < VE; k += 4) {
            a0 = sq_acc(x[k + 0], a0);
            a1 = sq_acc(x[k + 1], a1);
            a2 = sq_acc(x[k + 2], a2);
            a3 = sq_acc(x[k + 3], a3);
          }
          continue;
        }
        if (RD) {
#pragma unroll
          for (int q = 0; q < DV; ++q) {
            x[4 * q + 0] = __fadd_rn(dv[u][q].x, x[4 * q + 0]);
            x[4 * q + 1] = __fadd_rn(dv[u][q].y, x[4 * q + 1]);
            x[4 * q + 2] = __fadd_rn(dv[u][q].z, x[4 * q + 2]);
            x[4 * q + 3] = __fadd_rn(dv[u][q].w, x[4 * q + 3]);
          }
        }
        if (MODE == kAccum) {
#pragma unroll
          for (int q = 0; q < DV; ++q)
            st_delta<AF_D_STORE>(db + c * DV + q, make_float4(x[4 * q], x[4 * q + 1], x[4 * q + 2], x[4 * q + 3]));
        } else {
#pragma unroll
          for (int k = 0; k < VE; k += 4) {
            a0 = sq_acc(x[k + 0], a0);
            a1 = sq_acc(x[k + 1], a1);
            a2 = sq_acc(x[k + 2], a2);
            a3 = sq_acc(x[k + 3], a3);
          }
        }
      }
    }
  }
  return (a0 + a1) + (a2 + a3);
}


// AdamW on one element in fp32 with explicit round-to-nearest operations (no
// contraction), in the order of the oracle's definition (oracle.adamw_step):
//   p <- p * decay;  m <- m*b1 + g*(1-b1);  v <- v*b2 + (g*g)*(1-b2)
//   p <- p - step_size * (m / (sqrt(v) / sqrt_bc2 + eps))
__device__ __forceinline__ void adamw_elem(const AdamConst &c, float g, float &pw, float &m, float &v) {
  pw = __fmul_rn(pw, c.decay);
  m = __fadd_rn(__fmul_rn(m, c.beta1), __fmul_rn(g, c.one_minus_beta1));
  v = __fadd_rn(__fmul_rn(v, c.beta2), __fmul_rn(__fmul_rn(g, g), c.one_minus_beta2));
  const float den = __fadd_rn(__fdiv_rn(__fsqrt_rn(v), c.sqrt_bc2), c.eps);
  pw = __fsub_rn(pw, __fmul_rn(c.step_size, __fdiv_rn(m, den)));
}

// NEXT 1: the Delta accumulate (or, at the interval end, the
// fp64 sum of squares of Delta + g) fused into the AdamW update that already
// reads g -- one pass over g, Delta, p, m, v instead of two kernels reading g.
template <bool END, typename GT, bool RD>
__device__ __forceinline__ double process_tile_adam(const NormParams &p, const Tile &t) {
  constexpr int VE = VT<GT>::VE;
  constexpr int DV = VE / 4;
  const GT *__restrict__ g = static_cast<const GT *>(p.grad);
  float *__restrict__ d = p.delta - p.shard_begin;
  float *__restrict__ pw = p.params;
  float *__restrict__ mm = p.exp_avg;
  float *__restrict__ vv = p.exp_avg_sq;
  const int64_t b = t.begin, e = t.end;
  int64_t vb = ((b + VE - 1) / VE) * VE;
  int64_t ve = (e / VE) * VE;
  if (vb > ve) vb = ve = e;
  const int tid = threadIdx.x;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  auto scalar = [&](int64_t i, double &acc) {
    const float gf = g_scalar(g, i);
    const float x = RD ? __fadd_rn(d[i], gf) : gf;
    if (END)
      acc = sq_acc(x, acc);
    else
      d[i] = x;
    float pv = pw[i], mv = mm[i], vv2 = vv[i];
    adamw_elem(p.adam, gf, pv, mv, vv2);
    pw[i] = pv;
    mm[i] = mv;
    vv[i] = vv2;
  };
  const int nh = static_cast<int>(vb - b), nt = static_cast<int>(e - ve);
  if (tid < nh) scalar(b + tid, a0);
  if (tid >= 128 && tid - 128 < nt) scalar(ve + (tid - 128), a1);
  const int64_t nch = (ve - vb) / VE;
  const uint4 *gb = reinterpret_cast<const uint4 *>(g + vb);
  float4 *db = reinterpret_cast<float4 *>(d + vb);
  float4 *pb = reinterpret_cast<float4 *>(pw + vb);
  float4 *mb = reinterpret_cast<float4 *>(mm + vb);
  float4 *vb4 = reinterpret_cast<float4 *>(vv + vb);
  for (int64_t c = tid; c < nch; c += kNormBlock) {
    const uint4 gv = ld_stream<AF_G_HINT>(gb + c);
    float4 dv[DV], pv[DV], mv[DV], v2[DV];
#pragma unroll
    for (int q = 0; q < DV; ++q) {
      if (RD) dv[q] = __ldcs(db + c * DV + q);
      pv[q] = __ldcs(pb + c * DV + q);
      mv[q] = __ldcs(mb + c * DV + q);
      v2[q] = __ldcs(vb4 + c * DV + q);
    }
    float x[VE];
    unpack<VE>(gv, x);
#pragma unroll
    for (int q = 0; q < DV; ++q) {
      float gq[4] = {x[4 * q], x[4 * q + 1], x[4 * q + 2], x[4 * q + 3]};
      float dq[4] = {gq[0], gq[1], gq[2], gq[3]};
      if (RD) {
        dq[0] = __fadd_rn(dv[q].x, gq[0]);
        dq[1] = __fadd_rn(dv[q].y, gq[1]);
        dq[2] = __fadd_rn(dv[q].z, gq[2]);
        dq[3] = __fadd_rn(dv[q].w, gq[3]);
      }
      if (END) {
        a0 = sq_acc(dq[0], a0);
        a1 = sq_acc(dq[1], a1);
        a2 = sq_acc(dq[2], a2);
        a3 = sq_acc(dq[3], a3);
      } else {
        st_delta<AF_D_STORE_ADAM>(db + c * DV + q, make_float4(dq[0], dq[1], dq[2], dq[3]));
      }
      adamw_elem(p.adam, gq[0], pv[q].x, mv[q].x, v2[q].x);
      adamw_elem(p.adam, gq[1], pv[q].y, mv[q].y, v2[q].y);
      adamw_elem(p.adam, gq[2], pv[q].z, mv[q].z, v2[q].z);
      adamw_elem(p.adam, gq[3], pv[q].w, mv[q].w, v2[q].w);
      st_delta<AF_P_STORE>(pb + c * DV + q, pv[q]);
      st_delta<AF_P_STORE>(mb + c * DV + q, mv[q]);
      st_delta<AF_P_STORE>(vb4 + c * DV + q, v2[q]);
    }
  }
  return (a0 + a1) + (a2 + a3);
}

// NEXT 1, ZeRO form: the data-parallel gradient sync fused
// with the accumulate.  Each rank reads its shard of every rank's full gradient
// buffer over peer memory (pull: the loads of all ranks are in flight together),
// sums them in rank order 0..P-1 in fp32 (one rounding per add), scales once
// (gs = fl(sum * scale), the DDP average with scale = 1/P), writes gs to the
// optimizer's shard buffer and accumulates it into Delta exactly like kAccum /
// kEndDelta accumulate g.  The reduced gradient never makes an HBM round trip
// before the accumulate reads it.
template <bool END, bool ADAM, typename GT, bool RD, int PM>
__device__ __forceinline__ double process_tile_rs(const NormParams &p, const Tile &t, const GT *const (&gr)[PM]) {
  constexpr int VE = VT<GT>::VE;
  constexpr int DV = VE / 4;
  // PM = compile-time bound on the ranks (1, 2, 4, 8; P <= PM at run time): the
  // vectors in flight per thread stay U x PM = AF_U_RS_BYTES / 16 whatever P is
  constexpr bool BF = sizeof(GT) == 2;
  constexpr int UV = END ? (BF ? AF_U_RS_VEC_END_BF16 : AF_U_RS_VEC_END) : (BF ? AF_U_RS_VEC_BF16 : AF_U_RS_VEC);
  constexpr int U = ADAM ? 1 : (UV / PM > 0 ? UV / PM : 1);
  float *__restrict__ pw = p.params;
  float *__restrict__ mm = p.exp_avg;
  float *__restrict__ vv = p.exp_avg_sq;
  const int P = p.rs_world;
  const float sc = p.rs_scale;
  float *__restrict__ d = p.delta - p.shard_begin;
  float *__restrict__ o = p.rs_out ? p.rs_out - p.shard_begin : nullptr;
  const int64_t b = t.begin, e = t.end;
  int64_t vb = ((b + VE - 1) / VE) * VE;
  int64_t ve = (e / VE) * VE;
  if (vb > ve) vb = ve = e;
  const int tid = threadIdx.x;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  auto scalar = [&](int64_t i, double &acc) {
    float gs = g_scalar(gr[0], i);
    for (int r = 1; r < P; ++r) gs = __fadd_rn(gs, g_scalar(gr[r], i));
    gs = __fmul_rn(gs, sc);
    if (o) o[i] = gs;
    const float x = RD ? __fadd_rn(d[i], gs) : gs;
    if (END)
      acc = sq_acc(x, acc);
    else
      d[i] = x;
    if (ADAM) {
      float pv = pw[i], mv = mm[i], v2 = vv[i];
      adamw_elem(p.adam, gs, pv, mv, v2);
      pw[i] = pv;
      mm[i] = mv;
      vv[i] = v2;
    }
  };
  const int nh = static_cast<int>(vb - b), nt = static_cast<int>(e - ve);
  if (tid < nh) scalar(b + tid, a0);
  if (tid >= 128 && tid - 128 < nt) scalar(ve + (tid - 128), a1);
  const int64_t nch = (ve - vb) / VE;
  float4 *db = reinterpret_cast<float4 *>(d + vb);
  float4 *ob = o ? reinterpret_cast<float4 *>(o + vb) : nullptr;
  for (int64_t c0 = tid; c0 < nch; c0 += U * kNormBlock) {
    uint4 gv[U][PM];
    float4 dv[U][DV];
    float4 pa[ADAM ? U : 1][DV], ma[ADAM ? U : 1][DV], va[ADAM ? U : 1][DV];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t c = c0 + static_cast<int64_t>(u) * kNormBlock;
      if (c < nch) {
#pragma unroll
        for (int r = 0; r < PM; ++r)
          if (r < P) gv[u][r] = __ldcs(reinterpret_cast<const uint4 *>(gr[r] + vb) + c);
        if (RD) {
#pragma unroll
          for (int q = 0; q < DV; ++q) dv[u][q] = __ldcs(db + c * DV + q);
        }
        if (ADAM) {
#pragma unroll
          for (int q = 0; q < DV; ++q) {
            pa[u][q] = __ldcs(reinterpret_cast<const float4 *>(pw + vb) + c * DV + q);
            ma[u][q] = __ldcs(reinterpret_cast<const float4 *>(mm + vb) + c * DV + q);
            va[u][q] = __ldcs(reinterpret_cast<const float4 *>(vv + vb) + c * DV + q);
          }
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t c = c0 + static_cast<int64_t>(u) * kNormBlock;
      if (c < nch) {
        float x[VE];
        unpack<VE>(gv[u][0], x);
#pragma unroll
        for (int r = 1; r < PM; ++r) {
          if (r < P) {
            float y[VE];
            unpack<VE>(gv[u][r], y);
#pragma unroll
            for (int k = 0; k < VE; ++k) x[k] = __fadd_rn(x[k], y[k]);
          }
        }
#pragma unroll
        for (int k = 0; k < VE; ++k) x[k] = __fmul_rn(x[k], sc);
        if (ob) {
#pragma unroll
          for (int q = 0; q < DV; ++q) ob[c * DV + q] = make_float4(x[4 * q], x[4 * q + 1], x[4 * q + 2], x[4 * q + 3]);
        }
        if (ADAM) {
#pragma unroll
          for (int q = 0; q < DV; ++q) {
            adamw_elem(p.adam, x[4 * q + 0], pa[u][q].x, ma[u][q].x, va[u][q].x);
            adamw_elem(p.adam, x[4 * q + 1], pa[u][q].y, ma[u][q].y, va[u][q].y);
            adamw_elem(p.adam, x[4 * q + 2], pa[u][q].z, ma[u][q].z, va[u][q].z);
            adamw_elem(p.adam, x[4 * q + 3], pa[u][q].w, ma[u][q].w, va[u][q].w);
            st_delta<AF_P_STORE>(reinterpret_cast<float4 *>(pw + vb) + c * DV + q, pa[u][q]);
            st_delta<AF_P_STORE>(reinterpret_cast<float4 *>(mm + vb) + c * DV + q, ma[u][q]);
            st_delta<AF_P_STORE>(reinterpret_cast<float4 *>(vv + vb) + c * DV + q, va[u][q]);
          }
        }
        if (RD) {
#pragma unroll
          for (int q = 0; q < DV; ++q) {
            x[4 * q + 0] = __fadd_rn(dv[u][q].x, x[4 * q + 0]);
            x[4 * q + 1] = __fadd_rn(dv[u][q].y, x[4 * q + 1]);
            x[4 * q + 2] = __fadd_rn(dv[u][q].z, x[4 * q + 2]);
            x[4 * q + 3] = __fadd_rn(dv[u][q].w, x[4 * q + 3]);
          }
        }
        if (!END) {
#pragma unroll
          for (int q = 0; q < DV; ++q)
            st_delta<ADAM ? AF_D_STORE_ADAM : AF_D_STORE>(db + c * DV + q,
                                                          make_float4(x[4 * q], x[4 * q + 1], x[4 * q + 2], x[4 * q + 3]));
        } else {
#pragma unroll
          for (int k = 0; k < VE; k += 4) {
            a0 = sq_acc(x[k + 0], a0);
            a1 = sq_acc(x[k + 1], a1);
            a2 = sq_acc(x[k + 2], a2);
            a3 = sq_acc(x[k + 3], a3);
          }
        }
      }
    }
  }
  return (a0 + a1) + (a2 + a3);
}

// Cross-GPU epoch barrier of the fused reduce-scatter: threads r < P store the
// epoch into rank r's flag word for this rank (st.release.sys over peer memory),
// then wait until every rank's word in the local array reached it (ld.acquire.sys,
// bounded: a rank that never arrives sets sticky bit 2 -- the next decision is
// flagged EXCHANGE_TIMEOUT and not committed -- instead of hanging the GPU).
// which = 0: "my gradient is ready to be read" (every CTA, before its first
// load), which = 1: "I have finished reading" (the last CTA, before the kernel
// may complete and the caller's next backward overwrite the buffers).
// A timeout is made collective as far as it can be: the rank stores kPoisonEpoch
// into its slot at every peer, so a peer arriving later stops on it and flags the
// timeout as well instead of proceeding alone.  Returns true (CTA-uniform) when
// this CTA saw a timeout or poison: the caller then skips every peer load and
// every store of the step (the peers' buffers may be incomplete or reused).
__device__ __noinline__ bool rs_barrier(const NormParams &p, int which, unsigned long long e) {
  const int tid = threadIdx.x, P = p.rs_world;
  __shared__ int s_to;
  if (tid == 0) s_to = 0;
  if (tid < P) {
    unsigned long long *flag = p.peer_rs_flags[tid] + which * P + p.rs_rank;
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(flag), "l"(e) : "memory");
  }
  __syncthreads();
  if (tid < P) {
    const unsigned long long *flag = p.rs_flags + which * P + tid;
    unsigned long long v = 0;
    for (long long spin = 0;; ++spin) {
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(flag) : "memory");
      if (v == kPoisonEpoch) {
        s_to = 1;
        break;
      }
      if (v >= e) break;
      if (spin > (1ll << 22)) {
        s_to = 1;
        break;
      }
      __nanosleep(128);
    }
  }
  __syncthreads();
  const bool to = s_to != 0;
  if (to && tid < P) {
    unsigned long long *flag = p.peer_rs_flags[tid] + which * P + p.rs_rank;
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(flag), "l"(kPoisonEpoch) : "memory");
  }
  if (to && tid == 0) atomicOr(const_cast<uint32_t *>(&p.state->sticky), 2u);
  return to;
}

// the sticky timeout bits, read past L1 (another CTA of this launch may have set them)
__device__ __forceinline__ uint32_t sticky_of(const NormParams &p) {
  return *reinterpret_cast<const volatile uint32_t *>(&p.state->sticky);
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
  return v;  // identical on every lane (fp add is commutative)
}

// The last CTA's work after the grid has drained: per-segment sums, the optional
// NVLink one-shot exchange and the fused decision.  Not inlined, so its
// registers do not raise the streaming loop's (occupancy) budget.
// ACT (active-suffix shards, af_config.shard_active): one tile table per boundary
// f -- table f is tiles [first_tile_of_f[f], tile_end_of_f[f]) with its own
// per-segment ranges at seg_tile_begin + f * (L + 1).  Static shards (ACT false)
// compile to the single-table code: end = n_tiles, one segment-range array.
template <bool ACT>
__device__ __forceinline__ const int32_t *seg_ranges(const NormParams &p, int f) {
  return ACT ? p.seg_tile_begin + static_cast<size_t>(f) * p.stb_stride : p.seg_tile_begin;
}
template <bool ACT>
__device__ __forceinline__ int table_end(const NormParams &p, int f) {
  return ACT ? p.tile_end_of_f[f] : p.n_tiles;
}

// The last CTA's tail, common to every finalize: (debug delay,) the exchange
// epoch and this rank's row, the per-segment sums (`sums(publish)`, which calls
// publish(l, s) for every segment l), the optional NVLink one-shot exchange and
// the fused decision.  Every thread of the CTA calls it.
// s_x: >= kFinChunk doubles of shared scratch (the peers' rows when world x L fits).
// What the tail reads from global memory besides the sums, issued before the
// tail waits for anything (the last chunk's tiles are still streaming then):
// the decision's state inputs, the exchange epoch, the sticky timeout bits and
// (into s_peer) the peers' exchange-buffer pointers.
__shared__ unsigned long long *s_peer[AF_MAX_WORLD];
struct TailPre {
  DecideIn din;
  unsigned long long epoch;
  uint32_t sticky;
};
// count_done: the CTA running the tail before its grid-completion count (every
// mode but the fused reduce-scatter) counts itself here, from its last warp,
// while the tail waits for the last partials -- the scheduler resets (by
// whichever CTA counts last) then stay off the path after the decision.
__device__ __forceinline__ TailPre tail_prefetch(const NormParams &p, bool count_done) {
  const int tid = threadIdx.x;
  TailPre pre{};
  if (p.fuse_decide) pre.din = decide_load(p.dec);
  if (p.xworld > 1 && p.end && tid < p.xworld) s_peer[tid] = p.peer_rows[tid];
  pre.epoch = *reinterpret_cast<const volatile unsigned long long *>(&p.state->epoch);  // one broadcast load per warp
  pre.sticky = sticky_of(p);
  if (count_done && tid == kNormBlock - 32) {
    __threadfence();
    if (atomicAdd(&p.sched->done, 1u) == gridDim.x - 1) {
      __threadfence();
      p.sched->next = 0;
      p.sched->done = 0;
      p.fin_sched->next = 0u;
    }
  }
  return pre;  // (s_peer / the decision's s_pool are read after the caller's next __syncthreads)
}

template <int MODE, typename SumFn>
__device__ __forceinline__ void tail_common(const NormParams &p, double *s_x, TailPre pre, SumFn sums) {
  const int tid = threadIdx.x;
  if (p.dbg_tail_delay_ns) {  // AF_DEBUG_TAIL_DELAY_NS (ordering tests only)
    if (tid == 0) {
      const unsigned long long t0 = gtimer();
      while (gtimer() - t0 < p.dbg_tail_delay_ns) __nanosleep(1000);
    }
    __syncthreads();
  }
  // peer exchange: this interval end's epoch (identical on every rank) tags the LL
  // words and its parity selects one of two buffers (a peer is at most one epoch
  // ahead: it cannot finish epoch e without this rank's row of epoch e)
  const bool xchg = p.xworld > 1 && p.end;
  const unsigned long long x_epoch = pre.epoch + 1ull;  // every thread holds it: no barrier
  __shared__ int s_timeout;
  if (xchg && tid == 0) {
    const_cast<DevState *>(p.state)->epoch = x_epoch;
    s_timeout = 0;  // visible after the barrier that publishes the row
  }
  // this rank's row of the exchange matrix ss_all[world][L] (the rows the decision
  // sums), also kept in shared memory for the fused decision
  double *ss_row = p.ss_out;
  __shared__ double s_ss[AF_MAX_SEGMENTS];
  auto publish = [&](int l, double s) {
    if (MODE == kEndDelta) {
      ss_row[l] = s;
      s_ss[l] = s;
    } else {
      const double acc = p.first ? s : p.ss_acc[l] + s;
      if (p.commit) p.ss_acc[l] = acc;
      if (p.end) ss_row[l] = acc;
      s_ss[l] = acc;
    }
  };
  sums(publish);
  bool ss_in_smem = !xchg;  // world 1: the own row is the sum
  if (xchg && (pre.sticky & 3u)) {
    // an earlier exchange or barrier timed out (sticky until af_set_state): no peer
    // stores any more; the peers time out on this rank and flag it as well
  } else if (xchg) {
    // NVLink one-shot exchange, LL protocol: word 2l+h of this rank's row in every
    // peer's buffer = {32 bits of ss_l (h = 0 low, 1 high), epoch32}; 8-byte stores
    // are single-copy atomic, so a reader that sees the epoch sees the data -- no
    // fence, no separate flag.  Then poll the own buffer until every peer's words
    // carry the epoch (bounded: a missing peer flags a timeout instead of hanging).
    __syncthreads();  // the row is published
    const unsigned long long e = x_epoch;
    const uint32_t e32 = static_cast<uint32_t>(e);
    const int W = p.xworld, L = p.L, b = static_cast<int>(e & 1ull);
    const size_t my = (static_cast<size_t>(b) * W + p.xrank) * L;
    for (int i = tid; i < W * L; i += kNormBlock) {
      const int q = i / L, l = i % L;
      if (q == p.xrank) continue;
      const unsigned long long bits = static_cast<unsigned long long>(__double_as_longlong(s_ss[l]));
      const unsigned long long lo = (bits & 0xFFFFFFFFull) | (static_cast<unsigned long long>(e32) << 32);
      const unsigned long long hi = (bits >> 32) | (static_cast<unsigned long long>(e32) << 32);
      asm volatile("st.volatile.global.v2.u64 [%0], {%1, %2};" ::"l"(s_peer[q] + 2 * (my + l)), "l"(lo),
                   "l"(hi)
                   : "memory");
    }
    {
      // (AF_DEBUG_PEERS_ARRIVED: one read of every word, whatever epoch it holds --
      // the real path's work without the wait, for one-GPU timing of a rank)
      for (int i = tid; i < W * L; i += kNormBlock) {
        const int q = i / L, l = i % L;
        if (q == p.xrank) continue;
        const unsigned long long *w = p.xrows + 2 * ((static_cast<size_t>(b) * W + q) * L + l);
        unsigned long long lo, hi;
        for (long long spin = 0;; ++spin) {
          asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];" : "=l"(lo), "=l"(hi) : "l"(w) : "memory");
          const uint32_t f0 = static_cast<uint32_t>(lo >> 32), f1 = static_cast<uint32_t>(hi >> 32);
          if ((f0 == kPoisonEpoch32 || f1 == kPoisonEpoch32) && !p.dbg_peers_arrived) {  // that peer timed out
            s_timeout = 1;
            break;
          }
          if ((f0 == e32 && f1 == e32) || p.dbg_peers_arrived) {
            const double v = __longlong_as_double(static_cast<long long>((lo & 0xFFFFFFFFull) | (hi << 32)));
            p.ss_out[static_cast<ptrdiff_t>(q - p.xrank) * L + l] = v;
            if (W * L <= kFinChunk) s_x[i] = v;
            break;
          }
          if (spin > (1ll << 22)) {  // ~seconds: a peer never arrived -- flag it, do not hang the GPU
            s_timeout = 1;
            break;
          }
          __nanosleep(32);
        }
      }
    }
    __syncthreads();
    if (s_timeout) {  // make the timeout collective: poison this rank's row everywhere
      const unsigned long long poison = static_cast<unsigned long long>(kPoisonEpoch32) << 32;
      for (int i = tid; i < W * L; i += kNormBlock) {
        const int q = i / L, l = i % L;
        if (q == p.xrank) continue;
        asm volatile("st.volatile.global.v2.u64 [%0], {%1, %1};" ::"l"(s_peer[q] + 2 * (my + l)), "l"(poison)
                     : "memory");
      }
      if (tid == 0) atomicOr(const_cast<uint32_t *>(&p.state->sticky), 1u);
      pre.sticky |= 1u;  // (s_timeout is CTA-uniform)
    }
    if (!s_timeout && W * L <= kFinChunk && tid < L) {
      // the rank-order sum the decision takes (the decide kernel's order: 0 + row_0 + ...)
      double tot = 0.0;
      for (int q = 0; q < W; ++q) tot = __dadd_rn(tot, q == p.xrank ? s_ss[tid] : s_x[q * L + tid]);
      s_ss[tid] = tot;
      ss_in_smem = true;
    }
    ss_in_smem = ss_in_smem && !s_timeout && W * L <= kFinChunk;
  }
  if (AF_TIMING) {
    __syncthreads();
    if (tid == 0) const_cast<DevState *>(p.state)->tmark[2] = gtimer();
  }
  if (p.fuse_decide) {
    __syncthreads();
    DecideIn din = pre.din;
    din.sticky = pre.sticky;
    decide_block(p.dec, ss_in_smem ? s_ss : nullptr, din);
  }
  if (AF_TIMING) {
    __syncthreads();
    if (tid == 0) const_cast<DevState *>(p.state)->tmark[3] = gtimer();
  }
}

// Wait until an 8-byte slot no longer holds the sentinel; re-arm it; return it.
__device__ __forceinline__ double take_slot(unsigned long long *slot) {
  unsigned long long v;
  for (;;) {
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(slot) : "memory");
    if (v != kPartialEmpty) break;
  }
  *slot = kPartialEmpty;  // re-armed for the next launch
  return __longlong_as_double(static_cast<long long>(v));
}

// Tail of the streaming kernels, run by the CTA that claimed the last chunk:
// each segment's sum from the chunk pieces -- segment l's active tiles span
// chunks [c_lo, c_hi] (chunk c = tiles first_tile + [c*kFinChunk, (c+1)*kFinChunk)),
// whose pieces of l sit at part2[c + l]; summed in chunk order by one thread per
// segment.  Every index of part2[0, n_pc) is written exactly once per launch (the
// pieces, and zeros in the gaps between chunks' index ranges), so the tail
// simply waits for all n_pc slots (one wait per thread, in parallel) instead of
// a completion counter; they are staged in shared memory when they fit s_p.
template <int MODE, bool ACT>
__device__ __noinline__ void last_cta_tail(const NormParams &p, int first_tile, int n_end, int f, double *s_p,
                                          bool count_done) {
  const int32_t *stb = seg_ranges<ACT>(p, f);
  const int tid = threadIdx.x;
  const int nch = n_end > first_tile ? (n_end - first_tile + kFinChunk - 1) / kFinChunk : 0;
  const int n_pc = nch > 0 ? nch - 1 + p.tiles[n_end - 1].seg + 1 : 0;  // last index: (nch-1) + seg(last tile)
  const bool staged = n_pc <= kFinChunk && !p.dbg_unstaged_tail;
  const TailPre pre = tail_prefetch(p, count_done);
  auto *slots = reinterpret_cast<unsigned long long *>(p.part2);
  if (staged) {
    for (int i = tid; i < n_pc; i += kNormBlock) s_p[i] = take_slot(slots + i);
  } else {
    for (int i = tid; i < n_pc; i += kNormBlock) {  // wait for every slot; read them again below
      unsigned long long v;
      do {
        asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(slots + i) : "memory");
      } while (v == kPartialEmpty);
    }
  }
  __syncthreads();
  tail_common<MODE>(p, s_p, pre, [&](auto &publish) {
    for (int l = tid; l < p.L; l += kNormBlock) {
      int tb = stb[l];
      tb = tb < first_tile ? first_tile : tb;
      const int te = stb[l + 1];
      double sum = 0.0;
      if (te > tb) {
        const int c_lo = (tb - first_tile) / kFinChunk, c_hi = (te - 1 - first_tile) / kFinChunk;
        if (staged) {
          for (int c = c_lo; c <= c_hi; ++c) sum += s_p[c + l];
        } else {
#pragma unroll 8
          for (int c = c_lo; c <= c_hi; ++c) sum += __ldcg(p.part2 + c + l);
        }
      }
      publish(l, sum);
    }
  });
  if (!staged) {  // re-arm every slot (all were read above)
    __syncthreads();
    for (int i = tid; i < n_pc; i += kNormBlock) slots[i] = kPartialEmpty;
  }
}

// The tail when the pieces fit shared memory (n_pc <= kFinChunk: every table up
// to 65k tiles), run by the CTA that claimed the last chunk c -- before that
// chunk's tiles have finished.  Everything the tail reads besides the sums is
// loaded first (segment ranges, the chunk's segments, the decision's inputs,
// the exchange epoch and peer pointers); then the other chunks' pieces are
// taken (those chunks finish first), then chunk c's own tile partials.  Chunk c
// is reduced straight into the staged pieces (its pieces never go through
// part2: those slots stay armed), so after the grid's last tile the path is:
// one partial's visibility, a shared-memory reduction, the segment sums, the
// exchange and the decision.
template <int MODE, bool ACT>
__device__ __noinline__ void last_cta_tail_staged(const NormParams &p, int first_tile, int n_end, int f, int c,
                                                  int n_pc, double *s_p, bool count_done) {
  const int32_t *stb = seg_ranges<ACT>(p, f);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  __shared__ double s_pc[kFinChunk];
  __shared__ int s_stb[AF_MAX_SEGMENTS + 1];
  const int L = p.L;
  for (int l = tid; l <= L; l += kNormBlock) s_stb[l] = stb[l];
  const int c0 = first_tile + c * kFinChunk;
  const int n = min(kFinChunk, n_end - c0);
  const int lA = p.tiles[c0].seg, lB = p.tiles[c0 + n - 1].seg;
  const int lN = c0 + n < n_end ? p.tiles[c0 + n].seg + 1 : lB + 1;
  const TailPre pre = tail_prefetch(p, count_done);
  // the other chunks' pieces: every index of [0, n_pc) outside chunk c's own
  // ([c + lA, c + lN), and [0, lA) for chunk 0)
  auto *slots = reinterpret_cast<unsigned long long *>(p.part2);
  for (int i = tid; i < n_pc; i += kNormBlock) {
    const bool own = (i >= c + lA && i < c + lN) || (c == 0 && i < lA);
    if (!own) s_pc[i] = take_slot(slots + i);
  }
  for (int i = tid; i < n; i += kNormBlock)
    s_p[i] = take_slot(reinterpret_cast<unsigned long long *>(p.partials) + c0 + i);
  __syncthreads();
  for (int l = lA + warp; l <= lB; l += kNormBlock / 32) {  // chunk c's pieces, as fin_worker forms them
    int a = s_stb[l], b = s_stb[l + 1];
    a = (a < c0 ? c0 : a) - c0;
    b = (b > c0 + n ? c0 + n : b) - c0;
    double sum = 0.0;
#pragma unroll 8
    for (int k = a + lane; k < b; k += 32) sum += s_p[k];
    sum = warp_sum(sum);
    if (lane == 0) s_pc[c + l] = sum;
  }
  for (int i = c + lB + 1 + tid; i < c + lN; i += kNormBlock) s_pc[i] = 0.0;
  if (c == 0)
    for (int i = tid; i < lA; i += kNormBlock) s_pc[i] = 0.0;
  __syncthreads();
  tail_common<MODE>(p, s_p, pre, [&](auto &publish) {
    for (int l = tid; l < L; l += kNormBlock) {
      int tb = s_stb[l];
      tb = tb < first_tile ? first_tile : tb;
      const int te = s_stb[l + 1];
      double sum = 0.0;
      if (te > tb) {
        const int c_lo = (tb - first_tile) / kFinChunk, c_hi = (te - 1 - first_tile) / kFinChunk;
        for (int q = c_lo; q <= c_hi; ++q) sum += s_pc[q + l];
      }
      publish(l, sum);
    }
  });
}

// fin_worker's verdict: not the tail, the tail with every piece in part2, or
// (>= 0) the tail of the staged form with its own chunk still to reduce
constexpr int kNoTail = -1, kTailUnstaged = -2;

template <bool ACT>
__device__ __noinline__ int fin_worker(const NormParams &p, int first_tile, int n_end, int f, double *s_p,
                                       int *n_pc_out);

template <int MODE, typename GT, bool RD, int PM = 1, bool ACT = false>
__global__ void __launch_bounds__(kNormBlock, (MODE == kAccum || MODE == kRsAccum)
                                  ? 2
                                  : ((MODE >= kAdamAccum) ? 1 : (sizeof(GT) == 2 ? AF_MINB_END_BF16 : AF_MINB_END)))
    norms_kernel(const NormParams p) {
  constexpr bool RS = MODE == kRsAccum || MODE == kRsEnd || MODE == kRsAdamAccum || MODE == kRsAdamEnd;
  constexpr bool PARTIALS = MODE != kAccum && MODE != kAdamAccum && MODE != kRsAccum && MODE != kRsAdamAccum;
  __shared__ double s_fin[PARTIALS ? kFinChunk : 1];  // a finalize chunk's partials
  __shared__ int s_tile[3];
  __shared__ Tile s_desc[3];
  __shared__ double s_red[kNormBlock / 32];
  __shared__ int s_last;
  __shared__ unsigned long long s_rs_epoch;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // Speculative prologue, before the dependency wait: the boundary f as the
  // predecessor found it (it changes at most once per interval), its table
  // bounds and this CTA's first tile descriptor (the table is immutable).  After
  // the wait f is read again; the speculation is used only if it matches.
  auto clamp_f = [&](int x) { return x < 0 ? 0 : (x > p.n_pool ? p.n_pool : x); };
  const int f_spec = clamp_f(*reinterpret_cast<const volatile int32_t *>(&p.state->f));
  const int ft_spec = p.first_tile_of_f[f_spec];
  const int ne_spec = table_end<ACT>(p, f_spec);
  Tile d_spec{};
  const int k_first = AF_STATIC_FIRST ? static_cast<int>(blockIdx.x) : 0;
  const int t_spec = k_first < ne_spec - ft_spec ? (p.reverse ? ne_spec - 1 - k_first : ft_spec + k_first) : -1;
  if (AF_STATIC_FIRST && tid == 0 && t_spec >= 0) d_spec = p.tiles[t_spec];
  pdl_wait();  // f, Delta and the counters are written by the preceding kernels
  if (AF_TIMING && blockIdx.x == 0 && threadIdx.x == 0) {
    const_cast<DevState *>(p.state)->tmark[0] = gtimer();
    if (AF_TIMING_FIRST) const_cast<DevState *>(p.state)->tmark[1] = ~0ull;
  }
  const int f = clamp_f(p.state->f);
  const bool spec_ok = f == f_spec;
  const int first_tile = spec_ok ? ft_spec : p.first_tile_of_f[f];
  const int n_end = spec_ok ? ne_spec : table_end<ACT>(p, f);  // static: the constant n_tiles
  const GT *rs_g[PM];
  bool rs_skip = false;  // CTA-uniform: a barrier timed out -- no peer loads, no stores this step
  if constexpr (RS) {
#pragma unroll
    for (int r = 0; r < PM; ++r) rs_g[r] = r < p.rs_world ? static_cast<const GT *>(p.rs_grads[r]) : nullptr;
    if (p.rs_world > 1) {
      if (tid == 0) {
        s_rs_epoch = p.state->rs_epoch + 1ull;  // advanced by the last CTA only
        s_last = (sticky_of(p) & 3u) != 0u;  // an earlier step timed out (sticky)
      }
      __syncthreads();
      rs_skip = s_last != 0;
      __syncthreads();
      // every rank's gradient is complete before any peer load
      if (!rs_skip) rs_skip = rs_barrier(p, 0, s_rs_epoch);
    }
  }

  // Tile scheduler, two tiles of lookahead: while tile `it` is processed, thread 0
  // has the atomic for tile it+2 (one register) and an async copy (cp.async) of
  // tile it+1's descriptor into shared memory in flight; both land before the
  // end-of-tile barrier, so no warp waits on them and no registers hold them.
  // Tile order alternates between launches (p.reverse, toggled by the host): each
  // kernel starts where the previous one ended, so its first tiles find the
  // previous kernel's last ~100 MB (Delta written back, g just read) in the
  // 126 MB L2.  The order never changes a result: every tile's partial has a fixed
  // reduction tree and the segments are summed in tile-index order.
  const int n_act_tiles = n_end - first_tile;
  auto tile_of = [&](unsigned int k) -> int {
    const int kk = static_cast<int>(k);
    if (kk >= n_act_tiles) return n_end;  // past the end: the loop's stop value
    return p.reverse ? n_end - 1 - kk : first_tile + kk;
  };
  // AF_STATIC_FIRST: the first two tiles of CTA b are k = b and k = G + b (no
  // atomic: 296 CTAs serialised on one counter cost the grid's start ~1 us); the
  // counter hands out k = 2G, 2G + 1, ...
  const unsigned int k_base = AF_STATIC_FIRST ? 2u * gridDim.x : 0u;
  auto claim = [&]() { return tile_of(k_base + atomicAdd(&p.sched->next, 1u)); };
  if (tid == 0) {
    if (AF_STATIC_FIRST) {
      const int t0 = tile_of(static_cast<unsigned int>(k_first));
      s_tile[0] = t0;
      if (t0 < n_end) s_desc[0] = (spec_ok && t0 == t_spec) ? d_spec : p.tiles[t0];
      s_tile[1] = tile_of(gridDim.x + blockIdx.x);
    } else {
      const int t0 = claim();
      s_tile[0] = t0;
      if (t0 < n_end) s_desc[0] = p.tiles[t0];
      s_tile[1] = claim();
    }
  }
  __syncthreads();
  for (int it = 0;; ++it) {
    const int slot = it % 3, slot1 = (it + 1) % 3, slot2 = (it + 2) % 3;
    const int tile = s_tile[slot];
    if (tile >= n_end) break;
    const Tile t = s_desc[slot];
    int next2 = 0;
    if (tid == 0) {
      next2 = claim();
      const int n1 = s_tile[slot1];
      if (n1 < n_end) {
        const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(&s_desc[slot1]));
        const Tile *src = p.tiles + n1;
        asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
        asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(dst + 16u),
                     "l"(reinterpret_cast<const char *>(src) + 16)
                     : "memory");
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    }
    double v;
    if constexpr (MODE == kAdamAccum || MODE == kAdamEnd)
      v = process_tile_adam<MODE == kAdamEnd, GT, RD>(p, t);
    else if constexpr (RS)
      v = rs_skip ? 0.0
                  : process_tile_rs<MODE == kRsEnd || MODE == kRsAdamEnd, MODE == kRsAdamAccum || MODE == kRsAdamEnd,
                                    GT, RD, PM>(p, t, rs_g);
    else
      v = process_tile<MODE, GT, RD>(p, t);
    if (tid == 0) {
      s_tile[slot2] = next2;
      asm volatile("cp.async.wait_all;" ::: "memory");
    }
    if constexpr (PARTIALS) {
      const double w = warp_sum(v);
      if (lane == 0) s_red[warp] = w;
      __syncthreads();
      if (tid == 0) {
        double s = 0.0;
#pragma unroll
        for (int k = 0; k < kNormBlock / 32; ++k) s += s_red[k];
        p.partials[tile] = s;  // a plain 8-byte store: the value is its own ready flag (fin_worker)
      }
    }
    __syncthreads();
  }
  pdl_launch_dependents();
  if (AF_TIMING && tid == 0) {  // AF_TIMING_FIRST: the FIRST CTA out of tiles (the end phase's start)
    if (AF_TIMING_FIRST)
      atomicMin(const_cast<unsigned long long *>(&p.state->tmark[1]), gtimer());
    else
      const_cast<DevState *>(p.state)->tmark[1] = gtimer();
  }
  // finalize: a CTA out of tiles reduces chunks of partials while the grid's last
  // tiles are still streaming; the claimer of the last chunk runs the tail --
  // at once (it waits only on chunk pieces and tile partials, never on the other
  // CTAs' exit), except for the fused reduce-scatter, whose tail follows the
  // closing barrier on this rank's gradient
  constexpr int TM = (MODE == kAdamEnd || MODE == kRsEnd || MODE == kRsAdamEnd) ? kEndDelta : MODE;
  int tail = kNoTail, n_pc = 0;
  if constexpr (PARTIALS) tail = fin_worker<ACT>(p, first_tile, n_end, f, s_fin, &n_pc);
  auto run_tail = [&](bool count_done) {
    if (AF_TIMING && tid == 0) const_cast<DevState *>(p.state)->dmark[7] = gtimer();  // tail start
    if (tail >= 0)
      last_cta_tail_staged<TM, ACT>(p, first_tile, n_end, ACT ? f : 0, tail, n_pc, s_fin, count_done);
    else
      last_cta_tail<TM, ACT>(p, first_tile, n_end, ACT ? f : 0, s_fin, count_done);
  };
  if constexpr (PARTIALS && !RS) {
    if (tail != kNoTail) {
      run_tail(true);  // counts this CTA's completion itself
      return;
    }
  }

  // grid completion: every CTA has finished its tiles and claimed its last chunk;
  // the last one resets the schedulers (and, fused reduce-scatter, closes the
  // barrier on this rank's gradient)
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    const unsigned int d = atomicAdd(&p.sched->done, 1u);
    s_last = (d == gridDim.x - 1);
  }
  __syncthreads();
  if (s_last) {
    __threadfence();
    if (tid == 0) {
      p.sched->next = 0;
      p.sched->done = 0;
      if (PARTIALS) p.fin_sched->next = 0u;
    }
    if constexpr (RS) {
      if (p.rs_world > 1 && !(sticky_of(p) & 3u)) {
        rs_barrier(p, 1, s_rs_epoch);  // no rank reads this rank's gradient any more
        if (tid == 0) const_cast<DevState *>(p.state)->rs_epoch = s_rs_epoch;
      }
    }
    if constexpr (PARTIALS) {
      if (n_end <= first_tile) tail = kTailUnstaged;  // no active tile, no chunk: the last CTA publishes the zeros
    }
  }
  if constexpr (PARTIALS) {
    if (tail != kNoTail) run_tail(false);
  }
}

// The finalize of the per-tile partials, done by the streaming grid itself as its
// CTAs run out of tiles (no second launch, no kernel boundary): the active tiles
// form chunks of kFinChunk consecutive tiles; a CTA whose scheduler is drained
// claims chunks (in the order the tiles were processed, so the first-claimed
// chunks are complete) and reduces each: every thread takes one tile's partial,
// waiting until it is no longer the sentinel (kPartialEmpty -- the partial's
// plain 8-byte store is its own ready flag, so the streaming loop needs no fence
// or counter per tile), re-arms the slot, and each segment's piece of the chunk
// is summed by one warp in tile order (lane-strided, xor tree) into part2[c + l]
// (piece (c, l) is the (c+l)-th piece in tile order, so the index needs no
// search); the indices between this chunk's pieces and the next chunk's get
// zeros, so part2[0, n_pc) is written exactly once.  The CTA that claims the LAST
// chunk (claim order) returns true and runs the tail, which waits for every
// piece slot -- no completion counter, no fence.  Deterministic: the reduction
// order depends only on the tile table.  Cannot deadlock: a claimed tile belongs
// to a running CTA, which writes its partial without waiting on anything, and
// every chunk is claimed by a CTA that finishes it without waiting on the tail.
template <bool ACT>
__device__ __noinline__ int fin_worker(const NormParams &p, int first_tile, int n_end, int f, double *s_p,
                                       int *n_pc_out) {
  const int32_t *stb = seg_ranges<ACT>(p, f);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nch = (n_end - first_tile + kFinChunk - 1) / kFinChunk;
  __shared__ int s_c, s_tail, s_npc;
  auto *slots = reinterpret_cast<unsigned long long *>(p.partials);
  for (;;) {
    if (tid == 0) {
      const int w = static_cast<int>(atomicAdd(&p.fin_sched->next, 1u));
      s_c = w < nch ? (p.reverse ? nch - 1 - w : w) : -1;
      s_tail = w == nch - 1;
      // the last chunk's claimer runs the tail: staged in shared memory when the
      // piece count fits (the pieces' last index: (nch - 1) + seg(last tile))
      if (w == nch - 1) s_npc = nch - 1 + p.tiles[n_end - 1].seg + 1;
    }
    __syncthreads();
    const int c = s_c;
    if (c < 0) break;
    if (s_tail && s_npc <= kFinChunk && !p.dbg_unstaged_tail) {
      *n_pc_out = s_npc;
      return c;  // last_cta_tail_staged reduces chunk c itself
    }
    const int c0 = first_tile + c * kFinChunk;
    const int n = min(kFinChunk, n_end - c0);
    // the chunk's segments, loaded before its partials are awaited
    const int lA = p.tiles[c0].seg, lB = p.tiles[c0 + n - 1].seg;
    // the next chunk's first segment (or, for the last chunk, none): zeros fill the gap
    const int lN = c0 + n < n_end ? p.tiles[c0 + n].seg + 1 : lB + 1;
#pragma unroll
    for (int u = 0; u < kFinChunk / kNormBlock; ++u) {
      const int k = u * kNormBlock + tid;
      if (k < n) s_p[k] = take_slot(slots + c0 + k);
    }
    __syncthreads();
    for (int l = lA + warp; l <= lB; l += kNormBlock / 32) {
      int a = stb[l], b = stb[l + 1];
      a = (a < c0 ? c0 : a) - c0;
      b = (b > c0 + n ? c0 + n : b) - c0;
      double sum = 0.0;
#pragma unroll 8
      for (int k = a + lane; k < b; k += 32) sum += s_p[k];
      sum = warp_sum(sum);
      if (lane == 0) p.part2[c + l] = sum;
    }
    // zero pieces: indices [c + lB + 1, (c + 1) + lN - 1) between this chunk's and the
    // next chunk's ranges, and [0, lA) before the first chunk's
    for (int i = c + lB + 1 + tid; i < c + lN; i += kNormBlock) p.part2[i] = 0.0;
    if (c == 0)
      for (int i = tid; i < lA; i += kNormBlock) p.part2[i] = 0.0;
    const bool was_last = s_tail != 0;
    __syncthreads();  // s_p is free again
    if (was_last) return kTailUnstaged;  // every chunk is claimed: no further claim
  }
  return kNoTail;
}

using NormKernel = void (*)(const NormParams);

template <int MODE, typename GT, int PM>
NormKernel rd_pick(bool rd) {
  return rd ? norms_kernel<MODE, GT, true, PM> : norms_kernel<MODE, GT, false, PM>;
}

template <typename GT, int PM>
NormKernel rs_kernel(int mode, bool rd) {
  switch (mode) {
    case kRsAccum: return rd_pick<kRsAccum, GT, PM>(rd);
    case kRsEnd: return rd_pick<kRsEnd, GT, PM>(rd);
    case kRsAdamAccum: return rd_pick<kRsAdamAccum, GT, PM>(rd);
    default: return rd_pick<kRsAdamEnd, GT, PM>(rd);
  }
}

int pm_of(int world) { return world <= 1 ? 1 : (world == 2 ? 2 : (world <= 4 ? 4 : 8)); }

// The streaming kernel instantiation of (mode, Delta read, world, active-suffix
// tables).  Active-suffix tables exist for the replicated-gradient modes only.
template <typename GT>
NormKernel kernel_for(int mode, bool rd, int world, bool act = false) {
#ifdef AF_NO_ACT  // diagnostic build: no active-suffix instantiations
  act = false;
#endif
  if (act) {
    switch (mode) {
      case kAccum: return rd ? norms_kernel<kAccum, GT, true, 1, true> : norms_kernel<kAccum, GT, false, 1, true>;
      case kEndDelta:
        return rd ? norms_kernel<kEndDelta, GT, true, 1, true> : norms_kernel<kEndDelta, GT, false, 1, true>;
      case kStepSq: return norms_kernel<kStepSq, GT, false, 1, true>;
      default: break;  // refused by the host (static shards only)
    }
  }
  switch (mode) {
    case kAccum: return rd_pick<kAccum, GT, 1>(rd);
    case kEndDelta: return rd_pick<kEndDelta, GT, 1>(rd);
    case kStepSq: return norms_kernel<kStepSq, GT, false>;
    case kAdamAccum: return rd_pick<kAdamAccum, GT, 1>(rd);
    case kAdamEnd: return rd_pick<kAdamEnd, GT, 1>(rd);
    default:
      switch (pm_of(world)) {
        case 1: return rs_kernel<GT, 1>(mode, rd);
        case 2: return rs_kernel<GT, 2>(mode, rd);
        case 4: return rs_kernel<GT, 4>(mode, rd);
        default: return rs_kernel<GT, 8>(mode, rd);
      }
  }
}

template <typename GT>
int launch_dt(const NormParams &p, int mode, int grid, void *stream) {
  const bool rd = !p.first;
  if (mode < 0 || mode >= kNumModes) return static_cast<int>(cudaErrorInvalidValue);
  return static_cast<int>(launch_pdl(kernel_for<GT>(mode, rd, p.rs_world, p.stb_stride != 0), dim3(grid),
                                     dim3(kNormBlock), 0,
                                     static_cast<cudaStream_t>(stream), p));
}

}  // namespace

int launch_norms(const NormParams &p, int mode, int grad_dtype, int grid, void *stream) {
  return grad_dtype == AF_DT_BF16 ? launch_dt<uint16_t>(p, mode, grid, stream) : launch_dt<float>(p, mode, grid, stream);
}

// Load every kernel this context can launch now.  Under CUDA's lazy module
// loading the first launch of a kernel loads it, and a load may wait for the
// kernels in flight -- fatal when those are spinning on a peer rank (fused
// reduce-scatter barriers, the exchange) whose own launch sits behind this host
// thread.
template <typename GT>
static cudaError_t preload_dt(int world) {
  cudaFuncAttributes a;
  for (int m = 0; m < kNumModes; ++m)
    for (int rd = 0; rd < 2; ++rd) {
      for (int act = 0; act < 2; ++act) {
        const cudaError_t e = cudaFuncGetAttributes(&a, kernel_for<GT>(m, rd != 0, world, act != 0));
        if (e != cudaSuccess) return e;
      }
    }
  return cudaSuccess;
}

int preload_norm_kernels(int grad_dtype, int world) {
  cudaError_t e = grad_dtype == AF_DT_BF16 ? preload_dt<uint16_t>(world) : preload_dt<float>(world);
  if (e != cudaSuccess) return static_cast<int>(e);
  return 0;
}

int norms_max_blocks_per_sm(int mode, int grad_dtype, int world, int *blocks, bool act) {
  NormKernel k = grad_dtype == AF_DT_BF16 ? kernel_for<uint16_t>(mode, true, world, act)
                                         : kernel_for<float>(mode, true, world, act);
  if (mode == kStepSq) k = grad_dtype == AF_DT_BF16 ? kernel_for<uint16_t>(mode, false, world, act)
                                                   : kernel_for<float>(mode, false, world, act);
  return static_cast<int>(cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks, k, kNormBlock, 0));
}

}  // namespace af
