// af_api.cpp -- host side of the C ABI declared in include/af.h.
//
// Owns only host metadata (layout copy, shard bounds, tile table, host flags)
// and the optional NCCL communicator; every device buffer is caller-owned.
// Validation errors are synchronous and enqueue nothing.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "af_internal.h"

using namespace af;

namespace {

thread_local std::string g_last_error;

af_status fail(af_status s, const char *what) {
  g_last_error = what;
  return s;
}
af_status cuda_fail(cudaError_t e, const char *where) {
  g_last_error = std::string(where) + ": " + cudaGetErrorString(e);
  return AF_ECUDA;
}
af_status nccl_fail(ncclResult_t r, const char *where) {
  g_last_error = std::string(where) + ": " + ncclGetErrorString(r);
  return AF_ENCCL;
}

#define AF_CUDA(call, where)                     \
  do {                                           \
    cudaError_t e_ = (call);                     \
    if (e_ != cudaSuccess) return cuda_fail(e_, where); \
  } while (0)

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

bool aligned(const void *p, size_t a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; }

int device_sm_count(int *sms) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return static_cast<int>(e);
  return static_cast<int>(cudaDeviceGetAttribute(sms, cudaDevAttrMultiProcessorCount, dev));
}

}  // namespace

struct af_ctx {
  // layout / config (host copies)
  int L = 0, n_pool = 0;
  std::vector<int64_t> offs;
  std::vector<int32_t> kinds, pool_seg;
  af_dtype dtype = AF_DT_F32;
  af_config cfg{};
  int64_t n = 0, sb = 0, se = 0;
  // two segment-aligned tile tables of the shard: [0] the accumulate kernel's
  // (finer: scheduling granularity only), [1] the interval-end kernels' (one fp64
  // partial per tile)
  struct TileSet {
    int tile_elems = 0;
    std::vector<Tile> tiles;
    std::vector<int32_t> seg_tile_begin, first_tile_of_f;
    size_t o_tiles = 0, o_ftf = 0, o_stb = 0;
  } ts[2];
  // workspace
  size_t accum_bytes = 0, scratch_bytes = 0;
  size_t o_state = 0, o_sched = 0, o_pool = 0, o_part = 0, o_ssall = 0,
         o_ssacc = 0, o_last = 0, o_ring = 0, o_xrows = 0,
         o_xflags = 0, o_peer_rows = 0, o_peer_flags = 0;
  float *accum = nullptr;
  char *scratch = nullptr;
  bool bound = false;
  int grid[kNumModes] = {0, 0, 0, 0, 0};  // persistent grid per streaming-kernel mode (occupancy x SMs)
  // host flags
  bool armed = false;    // Delta / ss_acc hold this interval's partial sum
  bool pending = false;  // an interval end awaits af_update_and_decide
  ncclComm_t comm = nullptr;
  const void *rec_host = nullptr;  // last out_host pointer and its mapped device alias
  af_decision *rec_host_dev = nullptr;
  bool peers = false;               // NVLink one-shot exchange registered
  std::vector<void *> ipc_opened;   // peer allocations opened with cudaIpcOpenMemHandle

  template <typename T>
  T *at(size_t o) const {
    return reinterpret_cast<T *>(scratch + o);
  }
};

struct af_cache {
  int64_t num_examples = 0, row_bytes = 0;
  int64_t capacity = 0;  // owned ids of this rank (the partition size D_local)
  int32_t rank = 0, world = 1;
  // tiered mode (af_cache_set_capacity): I = hbm_rows + host_rows < D slots
  bool tiered = false;
  int64_t hbm_rows = 0, host_rows = 0;
  int32_t max_batch = 65536;  // rows per plan pass (larger calls are split)
  char *payload = nullptr;
  char *meta = nullptr;  // [CacheHeader | pad to 256 B][CacheMeta x capacity][free x I][rowslot x max_batch]
  char *host = nullptr;  // device alias of the page-locked host tier
  bool bound = false, host_bound = false;
  bool peers = false;                // global get/put through peers' stores (NEXT 4)
  std::vector<void *> ipc_opened;
  int grid = 0;
  size_t o_peer_table() const {
    size_t b = kMetaHeaderBytes + static_cast<size_t>(capacity) * sizeof(CacheMeta);
    if (tiered) b += static_cast<size_t>(hbm_rows + host_rows) * 4 + static_cast<size_t>(max_batch) * 4;
    return (b + 255) / 256 * 256;
  }
  size_t meta_bytes() const { return o_peer_table() + 2 * AF_MAX_WORLD * sizeof(void *); }
  size_t o_free() const { return kMetaHeaderBytes + static_cast<size_t>(capacity) * sizeof(CacheMeta); }
  size_t o_rowslot() const { return o_free() + static_cast<size_t>(hbm_rows + host_rows) * 4; }
  static constexpr size_t kMetaHeaderBytes = 256;
};

static constexpr size_t kMetaHeader = af_cache::kMetaHeaderBytes;

extern "C" {

const char *af_status_str(af_status s) {
  switch (s) {
    case AF_OK: return "AF_OK";
    case AF_EINVAL: return "AF_EINVAL";
    case AF_ESTATE: return "AF_ESTATE";
    case AF_EWORKSPACE: return "AF_EWORKSPACE";
    case AF_ECUDA: return "AF_ECUDA";
    case AF_ENCCL: return "AF_ENCCL";
    case AF_ENONFINITE: return "AF_ENONFINITE";
    case AF_EOWNER: return "AF_EOWNER";
    case AF_ERANGE: return "AF_ERANGE";
  }
  return "AF_UNKNOWN";
}

const char *af_last_error(void) { return g_last_error.c_str(); }
const char *af_version(void) { return "0.1.0"; }

int af_should_cache(int32_t frozen_layers, double t_layer_fwd_s, double t_batch_read_s) {
  if (frozen_layers <= 0 || !(t_layer_fwd_s >= 0.0) || !(t_batch_read_s >= 0.0)) return 0;
  return static_cast<double>(frozen_layers) * t_layer_fwd_s > t_batch_read_s ? 1 : 0;
}

af_status af_ctx_create(const af_layout *layout, const af_config *cfg, af_ctx **out) {
  if (!layout || !cfg || !out) return fail(AF_EINVAL, "NULL argument");
  const int L = layout->n_segments;
  if (L < 1 || L > AF_MAX_SEGMENTS) return fail(AF_EINVAL, "n_segments out of [1, AF_MAX_SEGMENTS]");
  if (!layout->seg_offsets || !layout->seg_kinds) return fail(AF_EINVAL, "NULL offsets / kinds");
  if (layout->grad_dtype != AF_DT_F32 && layout->grad_dtype != AF_DT_BF16) return fail(AF_EINVAL, "bad grad_dtype");
  if (layout->seg_offsets[0] != 0) return fail(AF_EINVAL, "seg_offsets[0] must be 0");
  for (int l = 0; l < L; ++l)
    if (layout->seg_offsets[l + 1] <= layout->seg_offsets[l]) return fail(AF_EINVAL, "offsets not strictly increasing");
  const int64_t n = layout->seg_offsets[L];
  if (n > (int64_t(1) << 50)) return fail(AF_ERANGE, "n_total too large");
  // kinds: PRE* POOL+ HEAD*
  int phase = 0, n_pool = 0;
  for (int l = 0; l < L; ++l) {
    const int k = layout->seg_kinds[l];
    if (k < AF_SEG_PRE || k > AF_SEG_HEAD) return fail(AF_EINVAL, "bad segment kind");
    if (k < phase) return fail(AF_EINVAL, "segment kinds must be ordered PRE* POOL+ HEAD*");
    if (k == AF_SEG_PRE && phase > AF_SEG_PRE) return fail(AF_EINVAL, "PRE after POOL/HEAD");
    phase = k;
    n_pool += (k == AF_SEG_POOL);
  }
  if (n_pool < 1) return fail(AF_EINVAL, "layout needs at least one POOL segment");
  if (!(cfg->percentile > 0.0 && cfg->percentile <= 100.0)) return fail(AF_EINVAL, "percentile out of (0, 100]");
  if (cfg->pct_method != AF_PCT_LINEAR && cfg->pct_method != AF_PCT_NEAREST_RANK)
    return fail(AF_EINVAL, "bad pct_method");
  if (cfg->acc_mode != AF_ACC_DELTA && cfg->acc_mode != AF_ACC_STEP_SUMSQ) return fail(AF_EINVAL, "bad acc_mode");
  if (!(cfg->tie_rel_eps >= 0.0) || !std::isfinite(cfg->tie_rel_eps)) return fail(AF_EINVAL, "bad tie_rel_eps");
  if (cfg->min_active < 1) return fail(AF_EINVAL, "min_active must be >= 1");
  if (cfg->world < 1 || cfg->world > AF_MAX_WORLD) return fail(AF_EINVAL, "world out of [1, AF_MAX_WORLD]");
  if (cfg->rank < 0 || cfg->rank >= cfg->world) return fail(AF_EINVAL, "rank out of [0, world)");

  af_ctx *c = new (std::nothrow) af_ctx();
  if (!c) return fail(AF_EINVAL, "out of host memory");
  c->L = L;
  c->n_pool = n_pool;
  c->offs.assign(layout->seg_offsets, layout->seg_offsets + L + 1);
  c->kinds.assign(layout->seg_kinds, layout->seg_kinds + L);
  for (int l = 0; l < L; ++l)
    if (c->kinds[l] == AF_SEG_POOL) c->pool_seg.push_back(l);
  c->dtype = layout->grad_dtype;
  c->cfg = *cfg;
  c->n = n;
  // contiguous shard, bounds rounded down to multiples of 8 elements
  auto bound_of = [&](int r) -> int64_t {
    if (r <= 0) return 0;
    if (r >= cfg->world) return n;
    const unsigned __int128 x = static_cast<unsigned __int128>(n) * static_cast<unsigned>(r) / cfg->world;
    return static_cast<int64_t>(x) / kShardAlign * kShardAlign;
  };
  c->sb = bound_of(cfg->rank);
  c->se = bound_of(cfg->rank + 1);
  // segment-aligned tile tables of the shard (tile edges on a global grid of tile_elems)
  const bool bf16 = (c->dtype == AF_DT_BF16);
  c->ts[0].tile_elems = bf16 ? AF_TILE_ACC_BF16 : AF_TILE_ACC_F32;
  c->ts[1].tile_elems = bf16 ? AF_TILE_ELEMS_BF16 : AF_TILE_ELEMS_F32;
  // interval-end table: "tapered" tiles -- AF_TILE_BIG_MULT x larger in the first
  // AF_TILE_BIG_FRAC_PCT % of the shard (fewer fp64 partials for the last CTA to
  // sum), nominal size in the tail (balanced finish).  Fixed at create, so the
  // partials and their summation order stay deterministic.
  const int64_t big_until = c->sb + (c->se - c->sb) / 100 * AF_TILE_BIG_FRAC_PCT;
  for (int k = 0; k < 2; ++k) {
    auto &T = c->ts[k];
    const int64_t TE = T.tile_elems;
    const int64_t TB = (k == 1) ? TE * AF_TILE_BIG_MULT : TE;
    T.seg_tile_begin.assign(L + 1, 0);
    for (int l = 0; l < L; ++l) {
      T.seg_tile_begin[l] = static_cast<int32_t>(T.tiles.size());
      const int64_t lo = std::max(c->offs[l], c->sb), hi = std::min(c->offs[l + 1], c->se);
      for (int64_t pos = lo; pos < hi;) {
        const int64_t te = (pos < big_until) ? TB : TE;
        const int64_t nxt = std::min(hi, (pos / te + 1) * te);
        T.tiles.push_back(Tile{pos, nxt, l, 0, 0, 0});
        pos = nxt;
      }
      if (T.tiles.size() > static_cast<size_t>(1) << 30) {
        delete c;
        return fail(AF_ERANGE, "too many tiles");
      }
    }
    T.seg_tile_begin[L] = static_cast<int32_t>(T.tiles.size());
    for (auto &t : T.tiles) {
      t.seg_first = T.seg_tile_begin[t.seg];
      t.seg_end = T.seg_tile_begin[t.seg + 1];
    }
    // first active tile when j POOL layers are frozen: PRE and POOL[0..j) skipped (Q11)
    T.first_tile_of_f.assign(n_pool + 1, 0);
    for (int j = 0; j <= n_pool; ++j) {
      int first_seg = 0;
      if (j > 0) first_seg = (j < n_pool) ? c->pool_seg[j] : c->pool_seg[n_pool - 1] + 1;
      T.first_tile_of_f[j] = T.seg_tile_begin[first_seg];
    }
  }
  // workspace layout
  const int64_t n_local = c->se - c->sb;
  c->accum_bytes = (cfg->acc_mode == AF_ACC_DELTA) ? static_cast<size_t>(n_local) * sizeof(float) : 0;
  size_t o = 0;
  auto take = [&](size_t bytes) {
    const size_t at = o;
    o = align_up(o + (bytes ? bytes : 1), 256);
    return at;
  };
  // rank-independent part first (its offsets are identical on every rank: peers
  // address each other's exchange buffers by these offsets), then the tile tables
  c->o_state = take(sizeof(DevState));
  c->o_sched = take(4 * sizeof(Sched));
  c->o_xrows = take(2 * static_cast<size_t>(cfg->world) * L * sizeof(double));
  c->o_xflags = take(static_cast<size_t>(cfg->world) * sizeof(unsigned long long));
  c->o_peer_rows = take(static_cast<size_t>(cfg->world) * sizeof(void *));
  c->o_peer_flags = take(static_cast<size_t>(cfg->world) * sizeof(void *));
  c->o_ssall = take(static_cast<size_t>(cfg->world) * L * sizeof(double));
  c->o_ssacc = take(L * sizeof(double));
  c->o_last = take(sizeof(af_decision));
  c->o_ring = take(kRing * sizeof(af_decision));
  c->o_pool = take(n_pool * sizeof(int32_t));
  for (auto &T : c->ts) {
    T.o_ftf = take((n_pool + 1) * sizeof(int32_t));
    T.o_stb = take((L + 1) * sizeof(int32_t));
    T.o_tiles = take(T.tiles.size() * sizeof(Tile));
  }
  c->o_part = take(c->ts[1].tiles.size() * sizeof(double));
  c->scratch_bytes = o;
  *out = c;
  return AF_OK;
}

af_status af_ctx_workspace_bytes(const af_ctx *c, size_t *accum_bytes, size_t *scratch_bytes) {
  if (!c || !accum_bytes || !scratch_bytes) return fail(AF_EINVAL, "NULL argument");
  *accum_bytes = c->accum_bytes;
  *scratch_bytes = c->scratch_bytes;
  return AF_OK;
}

af_status af_ctx_info(const af_ctx *c, af_info *info) {
  if (!c || !info) return fail(AF_EINVAL, "NULL argument");
  std::memset(info, 0, sizeof(*info));
  info->n_segments = c->L;
  info->n_pool = c->n_pool;
  info->rank = c->cfg.rank;
  info->world = c->cfg.world;
  info->n_total = c->n;
  info->shard_begin = c->sb;
  info->shard_end = c->se;
  info->n_tiles = static_cast<int32_t>(c->ts[1].tiles.size());
  info->tile_elems = c->ts[1].tile_elems;
  info->n_tiles_acc = static_cast<int32_t>(c->ts[0].tiles.size());
  info->tile_elems_acc = c->ts[0].tile_elems;
  for (int j = 0; j <= c->n_pool; ++j) info->first_tile_of_pool[j] = c->ts[1].first_tile_of_f[j];
  return AF_OK;
}

af_status af_ctx_bind(af_ctx *c, void *accum_dev, void *scratch_dev) {
  if (!c || !scratch_dev) return fail(AF_EINVAL, "NULL argument");
  if (c->accum_bytes && !accum_dev) return fail(AF_EINVAL, "accum buffer required");
  if (!aligned(scratch_dev, 256) || (accum_dev && !aligned(accum_dev, 256)))
    return fail(AF_EINVAL, "workspace buffers must be 256-byte aligned");
  int sms = 0;
  cudaError_t e = static_cast<cudaError_t>(device_sm_count(&sms));
  if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceGetAttribute");
  for (int m = 0; m < kNumModes; ++m) {
    int bps = 0;
    e = static_cast<cudaError_t>(norms_max_blocks_per_sm(m, c->dtype, &bps));
    if (e != cudaSuccess) return cuda_fail(e, "cudaOccupancyMaxActiveBlocksPerMultiprocessor");
    c->grid[m] = std::max(1, sms * std::max(1, bps));
  }
  c->accum = static_cast<float *>(accum_dev);
  c->scratch = static_cast<char *>(scratch_dev);
  AF_CUDA(cudaMemset(c->scratch, 0, c->scratch_bytes), "cudaMemset(scratch)");
  for (auto &T : c->ts) {
    if (!T.tiles.empty())
      AF_CUDA(cudaMemcpy(c->scratch + T.o_tiles, T.tiles.data(), T.tiles.size() * sizeof(Tile),
                         cudaMemcpyHostToDevice),
              "cudaMemcpy(tiles)");
    AF_CUDA(cudaMemcpy(c->scratch + T.o_ftf, T.first_tile_of_f.data(), T.first_tile_of_f.size() * 4,
                       cudaMemcpyHostToDevice),
            "cudaMemcpy(first_tile_of_f)");
    AF_CUDA(cudaMemcpy(c->scratch + T.o_stb, T.seg_tile_begin.data(), T.seg_tile_begin.size() * 4,
                       cudaMemcpyHostToDevice),
            "cudaMemcpy(seg_tile_begin)");
  }
  AF_CUDA(cudaMemcpy(c->scratch + c->o_pool, c->pool_seg.data(), c->pool_seg.size() * 4, cudaMemcpyHostToDevice),
          "cudaMemcpy(pool_seg)");
  AF_CUDA(cudaDeviceSynchronize(), "bind");
  c->bound = true;
  c->armed = false;
  c->pending = false;
  return AF_OK;
}

af_status af_nccl_unique_id(void *id_128B) {
  if (!id_128B) return fail(AF_EINVAL, "NULL argument");
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  ncclUniqueId id;
  ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) return nccl_fail(r, "ncclGetUniqueId");
  std::memcpy(id_128B, &id, sizeof(id));
  return AF_OK;
}

af_status af_ctx_set_comm(af_ctx *c, const void *id_128B) {
  if (!c || !id_128B) return fail(AF_EINVAL, "NULL argument");
  if (c->comm) return fail(AF_ESTATE, "communicator already set");
  ncclUniqueId id;
  std::memcpy(&id, id_128B, sizeof(id));
  ncclComm_t comm = nullptr;
  ncclResult_t r = ncclCommInitRank(&comm, c->cfg.world, id, c->cfg.rank);
  if (r != ncclSuccess) return nccl_fail(r, "ncclCommInitRank");
  c->comm = comm;
  return AF_OK;
}

af_status af_ctx_exchange_rows(af_ctx *c, double **ss_all_dev) {
  if (!c || !ss_all_dev) return fail(AF_EINVAL, "NULL argument");
  if (!c->bound) return fail(AF_EWORKSPACE, "workspace not bound");
  *ss_all_dev = c->at<double>(c->o_ssall);
  return AF_OK;
}

}  // extern "C"

namespace {

NormParams norm_params(af_ctx *c, const void *grad_dev, bool end, bool dry) {
  NormParams p{};
  const int k = (c->cfg.acc_mode == AF_ACC_DELTA && !end) ? 0 : 1;  // which tile table
  const auto &T = c->ts[k];
  p.grad = grad_dev;
  p.delta = c->accum;
  p.shard_begin = c->sb;
  p.tiles = c->at<Tile>(T.o_tiles);
  p.n_tiles = static_cast<int32_t>(T.tiles.size());
  p.L = c->L;
  p.first_tile_of_f = c->at<int32_t>(T.o_ftf);
  p.seg_tile_begin = c->at<int32_t>(T.o_stb);
  p.state = c->at<DevState>(c->o_state);
  p.sched = c->at<Sched>(c->o_sched) + k;
  p.partials = c->at<double>(c->o_part);
  p.ss_out = c->at<double>(c->o_ssall) + static_cast<size_t>(c->cfg.rank) * c->L;
  p.ss_acc = c->at<double>(c->o_ssacc);
  p.n_pool = c->n_pool;
  p.first = c->armed ? 0 : 1;
  p.end = end ? 1 : 0;
  p.commit = dry ? 0 : 1;
  if (c->peers) {
    p.xworld = c->cfg.world;
    p.xrank = c->cfg.rank;
    p.xrows = c->at<double>(c->o_xrows);
    p.peer_rows = c->at<double *const>(c->o_peer_rows);
    p.xflags = c->at<unsigned long long>(c->o_xflags);
    p.peer_flags = c->at<unsigned long long *const>(c->o_peer_flags);
  }
  return p;
}

int norm_mode(const af_ctx *c, bool end) {
  if (c->cfg.acc_mode == AF_ACC_DELTA) return end ? kEndDelta : kAccum;
  return kStepSq;
}

DecideParams decide_params(af_ctx *c, bool dry, af_decision *out_host) {
  DecideParams p{};
  p.ss_all = c->peers ? c->at<double>(c->o_xrows) : c->at<double>(c->o_ssall);
  p.xparity = c->peers ? 1 : 0;
  p.world = c->cfg.world;
  p.L = c->L;
  p.n_pool = c->n_pool;
  p.pool_seg = c->at<int32_t>(c->o_pool);
  p.state = c->at<DevState>(c->o_state);
  p.last = c->at<af_decision>(c->o_last);
  p.ring = c->at<af_decision>(c->o_ring);
  p.percentile = c->cfg.percentile;
  p.pct_method = c->cfg.pct_method;
  p.tie_rel_eps = c->cfg.tie_rel_eps;
  p.min_active = c->cfg.min_active;
  p.commit = dry ? 0 : 1;
  // page-locked host memory is device-addressable (UVA): the kernel writes the record
  // there directly; otherwise the caller gets an async copy after the kernel.
  if (out_host && out_host != c->rec_host) {
    cudaPointerAttributes a{};
    c->rec_host = out_host;
    c->rec_host_dev = nullptr;
    if (cudaPointerGetAttributes(&a, out_host) == cudaSuccess && a.type == cudaMemoryTypeHost && a.devicePointer)
      c->rec_host_dev = static_cast<af_decision *>(a.devicePointer);
    cudaGetLastError();  // clear a sticky "invalid value" from unregistered pointers
  }
  p.host = out_host ? c->rec_host_dev : nullptr;
  return p;
}

af_status copy_record_if_unmapped(af_ctx *c, const DecideParams &p, af_decision *out_host, void *stream) {
  if (out_host && !p.host)
    AF_CUDA(cudaMemcpyAsync(out_host, p.last, sizeof(af_decision), cudaMemcpyDeviceToHost,
                            static_cast<cudaStream_t>(stream)),
            "cudaMemcpyAsync(decision)");
  return AF_OK;
}

af_status allgather_rows(af_ctx *c, void *stream) {
  if (c->cfg.world > 1 && c->comm && !c->peers) {
    double *rows = c->at<double>(c->o_ssall);
    ncclResult_t r = ncclAllGather(rows + static_cast<size_t>(c->cfg.rank) * c->L, rows, c->L, ncclFloat64, c->comm,
                                   static_cast<cudaStream_t>(stream));
    if (r != ncclSuccess) return nccl_fail(r, "ncclAllGather");
  }
  return AF_OK;
}

af_status check_norm_args(af_ctx *c, const void *grad_dev) {
  if (!c) return fail(AF_EINVAL, "NULL ctx");
  if (!c->bound) return fail(AF_EWORKSPACE, "workspace not bound");
  if (!grad_dev || !aligned(grad_dev, 16)) return fail(AF_EINVAL, "grad must be a 16-byte aligned device pointer");
  return AF_OK;
}

}  // namespace

extern "C" {

af_status af_layer_norms(af_ctx *c, const void *grad_dev, uint32_t flags, void *stream) {
  af_status st = check_norm_args(c, grad_dev);
  if (st != AF_OK) return st;
  if (flags & ~(AF_INTERVAL_END | AF_DRY_RUN)) return fail(AF_EINVAL, "unknown flags");
  const bool end = flags & AF_INTERVAL_END, dry = flags & AF_DRY_RUN;
  const int mode = norm_mode(c, end);
  NormParams p = norm_params(c, grad_dev, end, dry);
  const int grid = std::max(1, std::min<int>(c->grid[mode], std::max<int>(1, p.n_tiles)));
  const int e = launch_norms(p, mode, c->dtype, grid, stream);
  if (e != 0) return cuda_fail(static_cast<cudaError_t>(e), "norms kernel launch");
  if (end) {
    st = allgather_rows(c, stream);
    if (st != AF_OK) return st;
  }
  if (!dry) c->armed = !end;
  if (end) c->pending = true;
  return AF_OK;
}

af_status af_adamw_step(af_ctx *c, float *params_dev, float *exp_avg_dev, float *exp_avg_sq_dev,
                        const void *grad_dev, const af_adamw *hp, uint32_t flags, af_decision *out_host,
                        void *stream) {
  af_status st = check_norm_args(c, grad_dev);
  if (st != AF_OK) return st;
  if (!hp || !params_dev || !exp_avg_dev || !exp_avg_sq_dev) return fail(AF_EINVAL, "NULL argument");
  if (!aligned(params_dev, 16) || !aligned(exp_avg_dev, 16) || !aligned(exp_avg_sq_dev, 16))
    return fail(AF_EINVAL, "optimizer buffers must be 16-byte aligned");
  if (c->cfg.acc_mode != AF_ACC_DELTA) return fail(AF_ESTATE, "af_adamw_step needs acc_mode AF_ACC_DELTA");
  if (flags & ~(AF_INTERVAL_END | AF_DRY_RUN)) return fail(AF_EINVAL, "unknown flags");
  if (hp->step < 1 || !(hp->beta1 >= 0.f && hp->beta1 < 1.f) || !(hp->beta2 >= 0.f && hp->beta2 < 1.f) ||
      !(hp->eps > 0.f) || !(hp->lr >= 0.f) || !(hp->weight_decay >= 0.f))
    return fail(AF_EINVAL, "bad AdamW hyper-parameters");
  const bool end = flags & AF_INTERVAL_END, dry = flags & AF_DRY_RUN;
  if (end && c->cfg.world > 1 && !c->peers && !c->comm)
    return fail(AF_ESTATE, "interval end with world > 1 needs peers or a communicator");
  const int mode = end ? kAdamEnd : kAdamAccum;
  NormParams p = norm_params(c, grad_dev, end, dry);
  p.params = params_dev;
  p.exp_avg = exp_avg_dev;
  p.exp_avg_sq = exp_avg_sq_dev;
  // constants rounded once to fp32 (the oracle rounds the same fp64 values)
  const double lr = hp->lr, b1 = hp->beta1, b2 = hp->beta2;
  p.adam.decay = static_cast<float>(1.0 - lr * static_cast<double>(hp->weight_decay));
  p.adam.beta1 = hp->beta1;
  p.adam.one_minus_beta1 = static_cast<float>(1.0 - b1);
  p.adam.beta2 = hp->beta2;
  p.adam.one_minus_beta2 = static_cast<float>(1.0 - b2);
  p.adam.step_size = static_cast<float>(lr / (1.0 - std::pow(b1, hp->step)));
  p.adam.sqrt_bc2 = static_cast<float>(std::sqrt(1.0 - std::pow(b2, hp->step)));
  p.adam.eps = hp->eps;
  const bool fuse = end && (c->cfg.world == 1 || c->peers);
  if (fuse) {
    p.fuse_decide = 1;
    p.dec = decide_params(c, dry, out_host);
  }
  const int grid = std::max(1, std::min<int>(c->grid[mode], std::max<int>(1, p.n_tiles)));
  const int e = launch_norms(p, mode, c->dtype, grid, stream);
  if (e != 0) return cuda_fail(static_cast<cudaError_t>(e), "fused AdamW kernel launch");
  if (fuse) {
    st = copy_record_if_unmapped(c, p.dec, out_host, stream);
    if (st != AF_OK) return st;
    if (!dry) c->armed = false;
    return AF_OK;
  }
  if (end) {  // NCCL path: all-gather then the decide kernel
    st = allgather_rows(c, stream);
    if (st != AF_OK) return st;
    if (!dry) c->armed = false;
    c->pending = true;
    return af_update_and_decide(c, flags & AF_DRY_RUN, out_host, stream);
  }
  if (!dry) c->armed = true;
  return AF_OK;
}

af_status af_update_and_decide(af_ctx *c, uint32_t flags, af_decision *out_host, void *stream) {
  if (!c) return fail(AF_EINVAL, "NULL ctx");
  if (!c->bound) return fail(AF_EWORKSPACE, "workspace not bound");
  if (flags & ~(AF_DRY_RUN)) return fail(AF_EINVAL, "unknown flags");
  if (!c->pending) return fail(AF_ESTATE, "af_update_and_decide without a preceding AF_INTERVAL_END");
  const bool dry = flags & AF_DRY_RUN;
  DecideParams p = decide_params(c, dry, out_host);
  const int e = launch_decide(p, stream);
  if (e != 0) return cuda_fail(static_cast<cudaError_t>(e), "decide kernel launch");
  af_status st = copy_record_if_unmapped(c, p, out_host, stream);
  if (st != AF_OK) return st;
  if (!dry) c->pending = false;
  return AF_OK;
}

af_status af_interval_end(af_ctx *c, const void *grad_dev, uint32_t flags, af_decision *out_host, void *stream) {
  af_status st = check_norm_args(c, grad_dev);
  if (st != AF_OK) return st;
  if (flags & ~(AF_DRY_RUN)) return fail(AF_EINVAL, "unknown flags");
  const bool dry = flags & AF_DRY_RUN;
  if (c->cfg.world > 1 && !c->peers) {  // kernel + all-gather + decide kernel
    if (!c->comm)
      return fail(AF_ESTATE, "af_interval_end with world > 1 needs peers (af_ctx_set_peers_*) or a communicator");
    st = af_layer_norms(c, grad_dev, AF_INTERVAL_END | flags, stream);
    if (st != AF_OK) return st;
    return af_update_and_decide(c, flags, out_host, stream);
  }
  const int mode = norm_mode(c, true);
  NormParams p = norm_params(c, grad_dev, true, dry);
  p.fuse_decide = 1;
  p.dec = decide_params(c, dry, out_host);
  const int grid = std::max(1, std::min<int>(c->grid[mode], std::max<int>(1, p.n_tiles)));
  const int e = launch_norms(p, mode, c->dtype, grid, stream);
  if (e != 0) return cuda_fail(static_cast<cudaError_t>(e), "fused interval-end kernel launch");
  st = copy_record_if_unmapped(c, p.dec, out_host, stream);
  if (st != AF_OK) return st;
  if (!dry) {
    c->armed = false;
    c->pending = false;
  }
  return AF_OK;
}

// CUDA IPC export of a pointer that may sit inside a larger allocation (the
// caller's allocator sub-allocates): handle of the allocation base + offset.
struct IpcRef {
  cudaIpcMemHandle_t h;
  uint64_t offset;
};

static af_status ipc_export(const void *ptr, IpcRef *out) {
  typedef int (*GetRange)(unsigned long long *, size_t *, unsigned long long);
  void *fn = nullptr;
  cudaDriverEntryPointQueryResult q{};
  AF_CUDA(cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q), "cudaGetDriverEntryPoint");
  if (!fn || q != cudaDriverEntryPointSuccess) return fail(AF_ECUDA, "cuMemGetAddressRange entry point not found");
  unsigned long long base = 0;
  size_t size = 0;
  if (reinterpret_cast<GetRange>(fn)(&base, &size, reinterpret_cast<unsigned long long>(ptr)) != 0)
    return fail(AF_ECUDA, "cuMemGetAddressRange failed");
  AF_CUDA(cudaIpcGetMemHandle(&out->h, reinterpret_cast<void *>(base)), "cudaIpcGetMemHandle");
  out->offset = reinterpret_cast<unsigned long long>(ptr) - base;
  return AF_OK;
}

static af_status ipc_import(const IpcRef &r, std::vector<void *> &opened, char **out) {
  void *p = nullptr;
  AF_CUDA(cudaIpcOpenMemHandle(&p, r.h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
  opened.push_back(p);
  *out = static_cast<char *>(p) + r.offset;
  return AF_OK;
}

struct IpcHandle {  // AF_IPC_HANDLE_BYTES
  cudaIpcMemHandle_t h;
  uint64_t offset;                 // scratch offset inside the exported allocation
  uint64_t xrows_off, xflags_off;  // exchange-area offsets inside the scratch
  int32_t rank, world, L, pad;
};
static_assert(sizeof(IpcHandle) <= AF_IPC_HANDLE_BYTES, "ipc handle size");

static af_status upload_peers(af_ctx *c, const std::vector<char *> &scratch_of) {
  std::vector<double *> rows(c->cfg.world);
  std::vector<unsigned long long *> flags(c->cfg.world);
  for (int r = 0; r < c->cfg.world; ++r) {
    rows[r] = reinterpret_cast<double *>(scratch_of[r] + c->o_xrows);
    flags[r] = reinterpret_cast<unsigned long long *>(scratch_of[r] + c->o_xflags);
  }
  AF_CUDA(cudaMemcpy(c->scratch + c->o_peer_rows, rows.data(), rows.size() * sizeof(void *), cudaMemcpyHostToDevice),
          "cudaMemcpy(peer rows)");
  AF_CUDA(cudaMemcpy(c->scratch + c->o_peer_flags, flags.data(), flags.size() * sizeof(void *),
                     cudaMemcpyHostToDevice),
          "cudaMemcpy(peer flags)");
  AF_CUDA(cudaDeviceSynchronize(), "set peers");
  c->peers = true;
  return AF_OK;
}

af_status af_ctx_exchange_ipc_handle(af_ctx *c, void *handle_out) {
  if (!c || !handle_out) return fail(AF_EINVAL, "NULL argument");
  if (!c->bound) return fail(AF_EWORKSPACE, "workspace not bound");
  IpcRef r{};
  af_status st = ipc_export(c->scratch, &r);
  if (st != AF_OK) return st;
  IpcHandle h{};
  h.h = r.h;
  h.offset = r.offset;
  h.xrows_off = c->o_xrows;
  h.xflags_off = c->o_xflags;
  h.rank = c->cfg.rank;
  h.world = c->cfg.world;
  h.L = c->L;
  std::memset(handle_out, 0, AF_IPC_HANDLE_BYTES);
  std::memcpy(handle_out, &h, sizeof(h));
  return AF_OK;
}

af_status af_ctx_set_peers_ipc(af_ctx *c, const void *handles) {
  if (!c || !handles) return fail(AF_EINVAL, "NULL argument");
  if (!c->bound) return fail(AF_EWORKSPACE, "workspace not bound");
  if (c->peers) return fail(AF_ESTATE, "peers already set");
  std::vector<char *> scratch_of(c->cfg.world, nullptr);
  for (int r = 0; r < c->cfg.world; ++r) {
    IpcHandle h;
    std::memcpy(&h, static_cast<const char *>(handles) + static_cast<size_t>(r) * AF_IPC_HANDLE_BYTES, sizeof(h));
    if (h.rank != r || h.world != c->cfg.world || h.L != c->L || h.xrows_off != c->o_xrows ||
        h.xflags_off != c->o_xflags)
      return fail(AF_EINVAL, "peer handle mismatch");
    if (r == c->cfg.rank) {
      scratch_of[r] = c->scratch;
      continue;
    }
    af_status st = ipc_import(IpcRef{h.h, h.offset}, c->ipc_opened, &scratch_of[r]);
    if (st != AF_OK) return st;
  }
  return upload_peers(c, scratch_of);
}

af_status af_ctx_clear_peers(af_ctx *c) {
  if (!c) return fail(AF_EINVAL, "NULL ctx");
  c->peers = false;  // mappings stay open until af_ctx_destroy
  return AF_OK;
}

af_status af_ctx_set_peers_local(af_ctx *c, af_ctx *const *peers) {
  if (!c || !peers) return fail(AF_EINVAL, "NULL argument");
  if (!c->bound) return fail(AF_EWORKSPACE, "workspace not bound");
  if (c->peers) return fail(AF_ESTATE, "peers already set");
  std::vector<char *> scratch_of(c->cfg.world, nullptr);
  for (int r = 0; r < c->cfg.world; ++r) {
    const af_ctx *q = peers[r];
    if (!q || !q->bound || q->cfg.rank != r || q->cfg.world != c->cfg.world || q->L != c->L ||
        q->o_xrows != c->o_xrows || q->o_xflags != c->o_xflags)
      return fail(AF_EINVAL, "peer context mismatch");
    scratch_of[r] = q->scratch;
  }
  return upload_peers(c, scratch_of);
}

struct StateBlob {
  char magic[4];
  int32_t version, L, world, rank, T, f, armed;
  double prev[AF_MAX_SEGMENTS];
  double ss_acc[AF_MAX_SEGMENTS];
};

af_status af_get_state(af_ctx *c, void *buf, size_t *len) {
  if (!c || !len) return fail(AF_EINVAL, "NULL argument");
  if (!buf) {
    *len = sizeof(StateBlob);
    return AF_OK;
  }
  if (*len < sizeof(StateBlob)) return fail(AF_EINVAL, "buffer too small");
  if (!c->bound) return fail(AF_EWORKSPACE, "workspace not bound");
  AF_CUDA(cudaDeviceSynchronize(), "get_state sync");
  DevState st;
  AF_CUDA(cudaMemcpy(&st, c->scratch + c->o_state, sizeof(st), cudaMemcpyDeviceToHost), "cudaMemcpy(state)");
  StateBlob b{};
  std::memcpy(b.magic, "AFS1", 4);
  b.version = 1;
  b.L = c->L;
  b.world = c->cfg.world;
  b.rank = c->cfg.rank;
  b.T = st.T;
  b.f = st.f;
  b.armed = c->armed ? 1 : 0;
  std::memcpy(b.prev, st.prev, sizeof(b.prev));
  AF_CUDA(cudaMemcpy(b.ss_acc, c->scratch + c->o_ssacc, c->L * sizeof(double), cudaMemcpyDeviceToHost),
          "cudaMemcpy(ss_acc)");
  std::memcpy(buf, &b, sizeof(b));
  *len = sizeof(b);
  return AF_OK;
}

af_status af_set_state(af_ctx *c, const void *buf, size_t len) {
  if (!c || !buf) return fail(AF_EINVAL, "NULL argument");
  if (len < sizeof(StateBlob)) return fail(AF_EINVAL, "state blob too small");
  if (!c->bound) return fail(AF_EWORKSPACE, "workspace not bound");
  StateBlob b;
  std::memcpy(&b, buf, sizeof(b));
  if (std::memcmp(b.magic, "AFS1", 4) != 0 || b.version != 1) return fail(AF_EINVAL, "not an af state blob");
  if (b.L != c->L) return fail(AF_EINVAL, "state blob has another segment count");
  if (b.f < 0 || b.f > c->n_pool || b.T < 0) return fail(AF_EINVAL, "state blob out of range");
  AF_CUDA(cudaDeviceSynchronize(), "set_state sync");
  DevState st{};
  // keep the peer-exchange epoch: it counts interval ends on every rank and the
  // peers' flag words already hold it
  AF_CUDA(cudaMemcpy(&st, c->scratch + c->o_state, sizeof(st), cudaMemcpyDeviceToHost), "cudaMemcpy(state)");
  st.sticky = 0;
  st.T = b.T;
  st.f = b.f;
  std::memcpy(st.prev, b.prev, sizeof(st.prev));
  AF_CUDA(cudaMemcpy(c->scratch + c->o_state, &st, sizeof(st), cudaMemcpyHostToDevice), "cudaMemcpy(state)");
  AF_CUDA(cudaMemcpy(c->scratch + c->o_ssacc, b.ss_acc, c->L * sizeof(double), cudaMemcpyHostToDevice),
          "cudaMemcpy(ss_acc)");
  AF_CUDA(cudaDeviceSynchronize(), "set_state sync");
  c->armed = b.armed != 0;
  c->pending = false;
  return AF_OK;
}

af_status af_ctx_destroy(af_ctx *c) {
  if (!c) return fail(AF_EINVAL, "NULL ctx");
  if (c->comm) ncclCommDestroy(c->comm);
  for (void *p : c->ipc_opened) cudaIpcCloseMemHandle(p);
  delete c;
  return AF_OK;
}

// ------------------------------------------------------------------ cache

af_status af_cache_create(int64_t num_examples, int64_t row_bytes, int32_t rank, int32_t world, af_cache **out) {
  if (!out) return fail(AF_EINVAL, "NULL argument");
  if (num_examples < 0) return fail(AF_EINVAL, "num_examples < 0");
  if (row_bytes <= 0 || row_bytes % 16 != 0) return fail(AF_EINVAL, "row_bytes must be a positive multiple of 16");
  if (world < 1 || world > AF_MAX_WORLD || rank < 0 || rank >= world) return fail(AF_EINVAL, "bad rank/world");
  af_cache *c = new (std::nothrow) af_cache();
  if (!c) return fail(AF_EINVAL, "out of host memory");
  c->num_examples = num_examples;
  c->row_bytes = row_bytes;
  c->rank = rank;
  c->world = world;
  c->capacity = (num_examples > rank) ? (num_examples - rank + world - 1) / world : 0;
  const unsigned __int128 pb = static_cast<unsigned __int128>(c->capacity) * static_cast<uint64_t>(row_bytes);
  if (pb > (static_cast<unsigned __int128>(1) << 60)) {
    delete c;
    return fail(AF_ERANGE, "cache too large");
  }
  *out = c;
  return AF_OK;
}

af_status af_cache_set_capacity(af_cache *c, int64_t hbm_rows, int64_t host_rows) {
  if (!c) return fail(AF_EINVAL, "NULL cache");
  if (c->bound) return fail(AF_ESTATE, "set the capacity before binding storage");
  if (hbm_rows < 0 || host_rows < 0 || hbm_rows + host_rows < 1) return fail(AF_EINVAL, "bad capacity");
  if (hbm_rows + host_rows > (int64_t(1) << 31) - 1) return fail(AF_ERANGE, "capacity too large");
  c->tiered = true;
  c->hbm_rows = hbm_rows;
  c->host_rows = host_rows;
  return AF_OK;
}

af_status af_cache_storage_bytes(const af_cache *c, size_t *payload_bytes, size_t *meta_bytes) {
  if (!c || !payload_bytes || !meta_bytes) return fail(AF_EINVAL, "NULL argument");
  const int64_t rows = c->tiered ? c->hbm_rows : c->capacity;
  *payload_bytes = static_cast<size_t>(rows) * static_cast<size_t>(c->row_bytes);
  *meta_bytes = c->meta_bytes();
  return AF_OK;
}

af_status af_cache_host_bytes(const af_cache *c, size_t *host_bytes) {
  if (!c || !host_bytes) return fail(AF_EINVAL, "NULL argument");
  *host_bytes = static_cast<size_t>(c->tiered ? c->host_rows : 0) * static_cast<size_t>(c->row_bytes);
  return AF_OK;
}

af_status af_cache_bind_host(af_cache *c, void *host_pinned) {
  if (!c || !host_pinned) return fail(AF_EINVAL, "NULL argument");
  if (!c->tiered || c->host_rows == 0) return fail(AF_ESTATE, "no host tier configured");
  if (!aligned(host_pinned, 16)) return fail(AF_EINVAL, "host tier must be 16-byte aligned");
  cudaPointerAttributes a{};
  cudaError_t e = cudaPointerGetAttributes(&a, host_pinned);
  if (e != cudaSuccess || a.type != cudaMemoryTypeHost || !a.devicePointer) {
    cudaGetLastError();
    return fail(AF_EINVAL, "host tier must be page-locked, device-mapped memory (cudaHostAlloc / pin_memory)");
  }
  c->host = static_cast<char *>(a.devicePointer);
  c->host_bound = true;
  return AF_OK;
}

af_status af_cache_bind(af_cache *c, void *payload_dev, void *meta_dev) {
  const int64_t rows = c ? (c->tiered ? c->hbm_rows : c->capacity) : 0;
  if (!c || !meta_dev || (rows > 0 && !payload_dev)) return fail(AF_EINVAL, "NULL argument");
  if ((payload_dev && !aligned(payload_dev, 16)) || !aligned(meta_dev, 256))
    return fail(AF_EINVAL, "payload must be 16-byte and meta 256-byte aligned");
  int sms = 0;
  cudaError_t e = static_cast<cudaError_t>(device_sm_count(&sms));
  if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceGetAttribute");
  c->grid = std::max(1, sms);
  c->payload = static_cast<char *>(payload_dev);
  c->meta = static_cast<char *>(meta_dev);
  AF_CUDA(cudaMemset(c->meta, 0, c->meta_bytes()), "cudaMemset(meta)");
  if (c->tiered) {
    // every record slot free: the stack pops slot 0 first (HBM before host)
    const int32_t I = static_cast<int32_t>(c->hbm_rows + c->host_rows);
    std::vector<int32_t> fr(static_cast<size_t>(I));
    for (int32_t k = 0; k < I; ++k) fr[k] = I - 1 - k;
    AF_CUDA(cudaMemcpy(c->meta + c->o_free(), fr.data(), fr.size() * 4, cudaMemcpyHostToDevice), "cudaMemcpy(free)");
    CacheHeader h{};
    h.top = I;
    AF_CUDA(cudaMemcpy(c->meta, &h, sizeof(h), cudaMemcpyHostToDevice), "cudaMemcpy(header)");
  }
  AF_CUDA(cudaDeviceSynchronize(), "cache bind");
  c->bound = true;
  return AF_OK;
}

static af_status cache_common(af_cache *c, const int64_t *ids, int32_t n, const void *rows, CacheParams &p) {
  if (!c) return fail(AF_EINVAL, "NULL cache");
  if (!c->bound) return fail(AF_EWORKSPACE, "cache storage not bound");
  if (n < 0) return fail(AF_EINVAL, "n < 0");
  if (n > 0 && (!ids || !rows)) return fail(AF_EINVAL, "NULL ids / rows");
  if (n > 0 && (!aligned(rows, 16) || !aligned(ids, 8))) return fail(AF_EINVAL, "rows must be 16-byte aligned");
  p = CacheParams{};
  p.payload = c->payload;
  p.meta = reinterpret_cast<CacheMeta *>(c->meta + kMetaHeader);
  p.err = reinterpret_cast<unsigned int *>(c->meta);
  p.ids = ids;
  p.n = n;
  p.row_bytes = c->row_bytes;
  p.num_examples = c->num_examples;
  p.rank = c->rank;
  p.world = c->world;
  return AF_OK;
}

static af_status cache_tiered(af_cache *c, CacheParams &p, bool put, void *stream) {
  if (c->host_rows > 0 && !c->host_bound) return fail(AF_EWORKSPACE, "host tier not bound (af_cache_bind_host)");
  const int32_t n_all = p.n;
  for (int32_t b0 = 0; b0 < n_all; b0 += c->max_batch) {
    const int32_t n = std::min(c->max_batch, n_all - b0);
    CachePlanParams q{};
    q.meta = p.meta;
    q.hdr = reinterpret_cast<CacheHeader *>(c->meta);
    q.free_slots = reinterpret_cast<int32_t *>(c->meta + c->o_free());
    q.rowslot = reinterpret_cast<int32_t *>(c->meta + c->o_rowslot());
    q.ids = p.ids + b0;
    q.n = n;
    q.put = put ? 1 : 0;
    q.depth = p.depth;
    q.cur_boundary = p.cur_boundary;
    q.depth_out = put ? nullptr : p.depth_out + b0;
    q.num_examples = c->num_examples;
    q.rank = c->rank;
    q.world = c->world;
    int e = launch_cache_plan(q, stream);
    if (e != 0) return cuda_fail(static_cast<cudaError_t>(e), "cache plan launch");
    CacheParams r = p;
    r.ids = p.ids + b0;
    r.n = n;
    r.rowslot = q.rowslot;
    r.host = c->host;
    r.hbm_rows = c->hbm_rows;
    if (put)
      r.src_rows = p.src_rows + static_cast<int64_t>(b0) * c->row_bytes;
    else
      r.dst_rows = p.dst_rows + static_cast<int64_t>(b0) * c->row_bytes;
    e = put ? launch_cache_put(r, c->grid, stream) : launch_cache_get(r, c->grid, stream);
    if (e != 0) return cuda_fail(static_cast<cudaError_t>(e), "cache copy launch");
  }
  return AF_OK;
}

af_status af_cache_put(af_cache *c, const int64_t *ids_dev, int32_t n, const void *rows_dev, int32_t depth,
                       void *stream) {
  CacheParams p;
  af_status s = cache_common(c, ids_dev, n, rows_dev, p);
  if (s != AF_OK) return s;
  if (depth < 1) return fail(AF_EINVAL, "depth must be >= 1 (frozen POOL count)");
  if (n == 0) return AF_OK;
  p.src_rows = static_cast<const char *>(rows_dev);
  p.depth = depth;
  if (c->tiered) return cache_tiered(c, p, true, stream);
  const int e = launch_cache_put(p, c->grid, stream);
  if (e != 0) return cuda_fail(static_cast<cudaError_t>(e), "cache put launch");
  return AF_OK;
}

af_status af_cache_get(af_cache *c, const int64_t *ids_dev, int32_t n, int32_t cur_boundary, void *rows_out_dev,
                       int32_t *depth_out_dev, void *stream) {
  CacheParams p;
  af_status s = cache_common(c, ids_dev, n, rows_out_dev, p);
  if (s != AF_OK) return s;
  if (n > 0 && !depth_out_dev) return fail(AF_EINVAL, "NULL depth_out");
  if (cur_boundary < 0) return fail(AF_EINVAL, "cur_boundary < 0");
  if (n == 0) return AF_OK;
  p.dst_rows = static_cast<char *>(rows_out_dev);
  p.depth_out = depth_out_dev;
  p.cur_boundary = cur_boundary;
  if (c->tiered) return cache_tiered(c, p, false, stream);
  const int e = launch_cache_get(p, c->grid, stream);
  if (e != 0) return cuda_fail(static_cast<cudaError_t>(e), "cache get launch");
  return AF_OK;
}

af_status af_cache_stats(af_cache *c, af_cache_info *out) {
  if (!c || !out) return fail(AF_EINVAL, "NULL argument");
  if (!c->bound) return fail(AF_EWORKSPACE, "cache storage not bound");
  AF_CUDA(cudaDeviceSynchronize(), "cache stats sync");
  CacheHeader h{};
  AF_CUDA(cudaMemcpy(&h, c->meta, sizeof(h), cudaMemcpyDeviceToHost), "cudaMemcpy(header)");
  std::vector<CacheMeta> m(static_cast<size_t>(c->capacity));
  if (c->capacity)
    AF_CUDA(cudaMemcpy(m.data(), c->meta + kMetaHeader, m.size() * sizeof(CacheMeta), cudaMemcpyDeviceToHost),
            "cudaMemcpy(meta)");
  std::memset(out, 0, sizeof(*out));
  out->error_flags = h.err;
  out->partition = c->capacity;
  out->capacity = c->tiered ? c->hbm_rows + c->host_rows : c->capacity;
  for (const auto &x : m) {
    if (!x.valid) continue;
    out->n_valid++;
    if (c->tiered && x.slot >= c->hbm_rows)
      out->n_host++;
    else
      out->n_hbm++;
  }
  out->n_dropped = c->tiered ? h.dropped : 0;
  out->free_slots = c->tiered ? h.top : c->capacity - out->n_valid;
  return AF_OK;
}

af_status af_cache_status(af_cache *c, uint32_t *device_error_flags, int64_t *n_valid) {
  if (!c || !device_error_flags) return fail(AF_EINVAL, "NULL argument");
  if (!c->bound) return fail(AF_EWORKSPACE, "cache storage not bound");
  AF_CUDA(cudaDeviceSynchronize(), "cache status sync");
  unsigned int err = 0;
  AF_CUDA(cudaMemcpy(&err, c->meta, sizeof(err), cudaMemcpyDeviceToHost), "cudaMemcpy(err)");  // CacheHeader.err
  *device_error_flags = err;
  if (n_valid) {
    std::vector<CacheMeta> m(static_cast<size_t>(c->capacity));
    if (c->capacity)
      AF_CUDA(cudaMemcpy(m.data(), c->meta + kMetaHeader, m.size() * sizeof(CacheMeta), cudaMemcpyDeviceToHost),
              "cudaMemcpy(meta)");
    int64_t v = 0;
    for (const auto &x : m) v += (x.valid != 0);
    *n_valid = v;
  }
  return AF_OK;
}

struct CacheIpcHandle {  // AF_CACHE_IPC_HANDLE_BYTES
  IpcRef payload, meta;
  int64_t num_examples, row_bytes;
  int32_t rank, world;
};
static_assert(sizeof(CacheIpcHandle) <= AF_CACHE_IPC_HANDLE_BYTES, "cache ipc handle size");

static af_status cache_upload_peers(af_cache *c, const std::vector<char *> &pay, const std::vector<char *> &met) {
  std::vector<void *> tab(2 * AF_MAX_WORLD, nullptr);
  for (int r = 0; r < c->world; ++r) {
    tab[r] = pay[r];
    tab[AF_MAX_WORLD + r] = met[r];
  }
  AF_CUDA(cudaMemcpy(c->meta + c->o_peer_table(), tab.data(), tab.size() * sizeof(void *), cudaMemcpyHostToDevice),
          "cudaMemcpy(cache peers)");
  AF_CUDA(cudaDeviceSynchronize(), "cache set peers");
  c->peers = true;
  return AF_OK;
}

af_status af_cache_exchange_ipc_handle(af_cache *c, void *handle_out) {
  if (!c || !handle_out) return fail(AF_EINVAL, "NULL argument");
  if (!c->bound) return fail(AF_EWORKSPACE, "cache storage not bound");
  if (c->tiered) return fail(AF_ESTATE, "global get/put needs the direct-mapped cache");
  CacheIpcHandle h{};
  af_status st = ipc_export(c->payload, &h.payload);
  if (st != AF_OK) return st;
  st = ipc_export(c->meta + kMetaHeader, &h.meta);
  if (st != AF_OK) return st;
  h.num_examples = c->num_examples;
  h.row_bytes = c->row_bytes;
  h.rank = c->rank;
  h.world = c->world;
  std::memset(handle_out, 0, AF_CACHE_IPC_HANDLE_BYTES);
  std::memcpy(handle_out, &h, sizeof(h));
  return AF_OK;
}

af_status af_cache_set_peers_ipc(af_cache *c, const void *handles) {
  if (!c || !handles) return fail(AF_EINVAL, "NULL argument");
  if (!c->bound) return fail(AF_EWORKSPACE, "cache storage not bound");
  if (c->tiered) return fail(AF_ESTATE, "global get/put needs the direct-mapped cache");
  if (c->peers) return fail(AF_ESTATE, "peers already set");
  std::vector<char *> pay(c->world), met(c->world);
  for (int r = 0; r < c->world; ++r) {
    CacheIpcHandle h;
    std::memcpy(&h, static_cast<const char *>(handles) + static_cast<size_t>(r) * AF_CACHE_IPC_HANDLE_BYTES,
                sizeof(h));
    if (h.rank != r || h.world != c->world || h.num_examples != c->num_examples || h.row_bytes != c->row_bytes)
      return fail(AF_EINVAL, "peer cache handle mismatch");
    if (r == c->rank) {
      pay[r] = c->payload;
      met[r] = c->meta + kMetaHeader;
      continue;
    }
    af_status st = ipc_import(h.payload, c->ipc_opened, &pay[r]);
    if (st != AF_OK) return st;
    st = ipc_import(h.meta, c->ipc_opened, &met[r]);
    if (st != AF_OK) return st;
  }
  return cache_upload_peers(c, pay, met);
}

af_status af_cache_set_peers_local(af_cache *c, af_cache *const *peers) {
  if (!c || !peers) return fail(AF_EINVAL, "NULL argument");
  if (!c->bound) return fail(AF_EWORKSPACE, "cache storage not bound");
  if (c->tiered) return fail(AF_ESTATE, "global get/put needs the direct-mapped cache");
  if (c->peers) return fail(AF_ESTATE, "peers already set");
  std::vector<char *> pay(c->world), met(c->world);
  for (int r = 0; r < c->world; ++r) {
    const af_cache *q = peers[r];
    if (!q || !q->bound || q->tiered || q->rank != r || q->world != c->world || q->num_examples != c->num_examples ||
        q->row_bytes != c->row_bytes)
      return fail(AF_EINVAL, "peer cache mismatch");
    pay[r] = q->payload;
    met[r] = q->meta + kMetaHeader;
  }
  return cache_upload_peers(c, pay, met);
}

static af_status cache_global_common(af_cache *c) {
  if (!c) return fail(AF_EINVAL, "NULL cache");
  if (!c->peers) return fail(AF_ESTATE, "global get/put needs af_cache_set_peers_*");
  return AF_OK;
}

af_status af_cache_put_global(af_cache *c, const int64_t *ids_dev, int32_t n, const void *rows_dev, int32_t depth,
                              void *stream) {
  af_status s = cache_global_common(c);
  if (s != AF_OK) return s;
  CacheParams p;
  s = cache_common(c, ids_dev, n, rows_dev, p);
  if (s != AF_OK) return s;
  if (depth < 1) return fail(AF_EINVAL, "depth must be >= 1 (frozen POOL count)");
  if (n == 0) return AF_OK;
  p.src_rows = static_cast<const char *>(rows_dev);
  p.depth = depth;
  p.peer_payload = reinterpret_cast<char *const *>(c->meta + c->o_peer_table());
  p.peer_meta = reinterpret_cast<CacheMeta *const *>(c->meta + c->o_peer_table() + AF_MAX_WORLD * sizeof(void *));
  const int e = launch_cache_put(p, c->grid, stream);
  if (e != 0) return cuda_fail(static_cast<cudaError_t>(e), "cache put launch");
  return AF_OK;
}

af_status af_cache_get_global(af_cache *c, const int64_t *ids_dev, int32_t n, int32_t cur_boundary,
                              void *rows_out_dev, int32_t *depth_out_dev, void *stream) {
  af_status s = cache_global_common(c);
  if (s != AF_OK) return s;
  CacheParams p;
  s = cache_common(c, ids_dev, n, rows_out_dev, p);
  if (s != AF_OK) return s;
  if (n > 0 && !depth_out_dev) return fail(AF_EINVAL, "NULL depth_out");
  if (cur_boundary < 0) return fail(AF_EINVAL, "cur_boundary < 0");
  if (n == 0) return AF_OK;
  p.dst_rows = static_cast<char *>(rows_out_dev);
  p.depth_out = depth_out_dev;
  p.cur_boundary = cur_boundary;
  p.peer_payload = reinterpret_cast<char *const *>(c->meta + c->o_peer_table());
  p.peer_meta = reinterpret_cast<CacheMeta *const *>(c->meta + c->o_peer_table() + AF_MAX_WORLD * sizeof(void *));
  const int e = launch_cache_get(p, c->grid, stream);
  if (e != 0) return cuda_fail(static_cast<cudaError_t>(e), "cache get launch");
  return AF_OK;
}

af_status af_cache_destroy(af_cache *c) {
  if (!c) return fail(AF_EINVAL, "NULL cache");
  for (void *p : c->ipc_opened) cudaIpcCloseMemHandle(p);
  delete c;
  return AF_OK;
}

}  // extern "C"
