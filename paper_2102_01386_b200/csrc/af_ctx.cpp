// af_ctx.cpp -- the freezing module's C-ABI entry points (af_ctx_*, af_layer_norms,
// af_interval_end, af_update_and_decide, af_adamw_step, state, NCCL and peer
// exchange setup).  Owns only host metadata, the optional NCCL communicator and
// the IPC mappings it opens; every device buffer is caller-owned.
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "af_host.h"

using namespace af;

namespace {
af_status nccl_fail(ncclResult_t r, const char *where) {
  set_last_error(std::string(where) + ": " + ncclGetErrorString(r));
  return AF_ENCCL;
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
    std::vector<Tile> tiles;  // static: one table; active-suffix: the per-f tables concatenated
    std::vector<int32_t> seg_tile_begin, first_tile_of_f, tile_end_of_f;
    int32_t max_tiles = 0;    // largest single table
    size_t o_tiles = 0, o_ftf = 0, o_stb = 0, o_tef = 0;
  } ts[2];
  bool active = false;                  // active-suffix shards (cfg.shard_active && world > 1)
  std::vector<int64_t> sb_of_f, se_of_f;  // this rank's shard per boundary f
  // workspace
  size_t accum_bytes = 0, scratch_bytes = 0;
  size_t o_state = 0, o_sched = 0, o_pool = 0, o_part = 0, o_part2 = 0, o_chunk = 0, o_ssall = 0,
         o_ssacc = 0, o_last = 0, o_ring = 0, o_xrows = 0,
         o_peer_rows = 0, o_rsflags = 0, o_peer_rsflags = 0, o_rs_grads = 0;
  float *accum = nullptr;
  char *scratch = nullptr;
  bool bound = false;
  int grid[kNumModes] = {};  // persistent grid per streaming-kernel mode (occupancy x SMs)
  int max_ctas = 0;          // af_ctx_set_max_ctas: cap on the streaming grids (0: none)
  bool reverse = false;      // tile order of the next streaming launch (alternates)
  // host flags
  bool armed = false;    // Delta / ss_acc hold this interval's partial sum
  bool pending = false;  // an interval end awaits af_update_and_decide
  ncclComm_t comm = nullptr;
  const void *rec_host = nullptr;  // last out_host pointer and its mapped device alias
  af_decision *rec_host_dev = nullptr;
  bool peers = false;               // NVLink one-shot exchange registered
  std::vector<void *> ipc_opened;   // peer allocations opened with cudaIpcOpenMemHandle
  bool grad_peers = false;          // fused reduce-scatter: every rank's gradient buffer registered
  const void *own_grad = nullptr;   // this rank's buffer (af_ctx_grad_ipc_handle)
  int device = -1;                  // the device the workspace was bound on
  uint32_t dbg_tail_delay_ns = 0;   // AF_DEBUG_TAIL_DELAY_NS
  int32_t dbg_peers_arrived = 0;    // AF_DEBUG_PEERS_ARRIVED
  int32_t dbg_unstaged_tail = 0;    // AF_DEBUG_UNSTAGED_TAIL
  int32_t dbg_force_nccl = 0;       // AF_DEBUG_FORCE_NCCL

  template <typename T>
  T *at(size_t o) const {
    return reinterpret_cast<T *>(scratch + o);
  }
};

extern "C" {

af_status af_ctx_create(const af_layout *layout, const af_config *cfg, af_ctx **out) {
  AF_NVTX();
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
  // contiguous shards, bounds rounded down to multiples of 8 elements:
  // of [0, n) for every f (static), or of the active suffix [A_f, n) per boundary f
  // (shard_active: A_f = start of the first segment not frozen at f -- PRE and
  // POOL[0..f) are frozen, P:402 / Q11)
  c->active = cfg->shard_active != 0 && cfg->world > 1;
  auto first_seg_of = [&](int j) -> int {
    if (j == 0) return 0;
    return (j < n_pool) ? c->pool_seg[j] : c->pool_seg[n_pool - 1] + 1;
  };
  auto bound_in = [&](int64_t A, int r) -> int64_t {
    if (r <= 0) return A;
    if (r >= cfg->world) return n;
    const unsigned __int128 x = static_cast<unsigned __int128>(n - A) * static_cast<unsigned>(r) / cfg->world;
    const int64_t b = (A + static_cast<int64_t>(x)) / kShardAlign * kShardAlign;
    return b < A ? A : b;
  };
  c->sb_of_f.assign(n_pool + 1, 0);
  c->se_of_f.assign(n_pool + 1, n);
  for (int j = 0; j <= n_pool; ++j) {
    const int64_t A = c->active ? c->offs[first_seg_of(j)] : 0;
    c->sb_of_f[j] = bound_in(A, cfg->rank);
    c->se_of_f[j] = bound_in(A, cfg->rank + 1);
  }
  c->sb = c->sb_of_f[0];
  c->se = c->se_of_f[0];

  // segment-aligned tile tables (tile edges on a global grid of tile_elems)
  const bool bf16 = (c->dtype == AF_DT_BF16);
  c->ts[0].tile_elems = bf16 ? AF_TILE_ACC_BF16 : AF_TILE_ACC_F32;
  c->ts[1].tile_elems = (cfg->acc_mode == AF_ACC_STEP_SUMSQ) ? (bf16 ? AF_TILE_SSQ_BF16 : AF_TILE_SSQ_F32)
                                                              : (bf16 ? AF_TILE_ELEMS_BF16 : AF_TILE_ELEMS_F32);
  // interval-end table: "tapered" tiles -- AF_TILE_BIG_MULT x larger in the first
  // AF_TILE_BIG_FRAC_PCT % of the shard (fewer fp64 partials for the last CTA to
  // sum), nominal size in the tail (balanced finish).  Fixed at create, so the
  // partials and their summation order stay deterministic.
  for (int k = 0; k < 2; ++k) {
    auto &T = c->ts[k];
    const int64_t TE = T.tile_elems;
    const int n_tab = c->active ? n_pool + 1 : 1;
    T.first_tile_of_f.assign(n_pool + 1, 0);
    T.tile_end_of_f.assign(n_pool + 1, 0);
    T.seg_tile_begin.assign(static_cast<size_t>(n_tab) * (L + 1), 0);
    for (int q = 0; q < n_tab; ++q) {
      const int64_t sb = c->sb_of_f[q], se = c->se_of_f[q];
      // interval-end tables: smaller tiles over AF_TILE_TAPER_PCT % of the range at
      // EACH end (consecutive launches walk the tiles in opposite directions, so a
      // launch's last tiles are at one end or the other) -- a shorter ragged finish
      const int64_t taper = (k == 1) ? (se - sb) / 100 * AF_TILE_TAPER_PCT : 0;
      const int64_t TS = std::max<int64_t>(TE / AF_TILE_TAPER_DIV, 1024);
      int32_t *stb = T.seg_tile_begin.data() + static_cast<size_t>(q) * (L + 1);
      const int32_t t0 = static_cast<int32_t>(T.tiles.size());
      for (int l = 0; l < L; ++l) {
        stb[l] = static_cast<int32_t>(T.tiles.size());
        const int64_t lo = std::max(c->offs[l], sb), hi = std::min(c->offs[l + 1], se);
        for (int64_t pos = lo; pos < hi;) {
          const int64_t te = (pos < sb + taper || pos >= se - taper) ? TS : TE;
          const int64_t nxt = std::min(hi, (pos / te + 1) * te);
          T.tiles.push_back(Tile{pos, nxt, l, stb[l], 0, 0});
          pos = nxt;
        }
        if (T.tiles.size() > static_cast<size_t>(1) << 30) {
          delete c;
          return fail(AF_ERANGE, "too many tiles");
        }
      }
      stb[L] = static_cast<int32_t>(T.tiles.size());
      for (size_t t = static_cast<size_t>(t0); t < T.tiles.size(); ++t) T.tiles[t].seg_end = stb[T.tiles[t].seg + 1];
      T.max_tiles = std::max(T.max_tiles, stb[L] - t0);
      if (c->active) {
        // table q holds exactly the tiles active at f = q
        T.first_tile_of_f[q] = t0;
        T.tile_end_of_f[q] = stb[L];
      } else {
        // first active tile when j POOL layers are frozen: PRE and POOL[0..j) skipped (Q11)
        for (int j = 0; j <= n_pool; ++j) {
          T.first_tile_of_f[j] = stb[first_seg_of(j)];
          T.tile_end_of_f[j] = stb[L];
        }
      }
    }
  }
  // workspace layout
  // Delta: the shard (static), or the whole buffer indexed by element (active-suffix
  // shards move with f; n x 4 B is small against 180 GB of HBM)
  const int64_t n_local = c->active ? n : c->se - c->sb;
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
  c->o_xrows = take(2 * static_cast<size_t>(cfg->world) * L * 2 * sizeof(unsigned long long));  // LL words
  c->o_peer_rows = take(static_cast<size_t>(cfg->world) * sizeof(void *));
  c->o_rsflags = take(2 * static_cast<size_t>(cfg->world) * sizeof(unsigned long long));
  c->o_peer_rsflags = take(static_cast<size_t>(cfg->world) * sizeof(void *));
  c->o_rs_grads = take(static_cast<size_t>(cfg->world) * sizeof(void *));
  c->o_ssall = take(static_cast<size_t>(cfg->world) * L * sizeof(double));
  c->o_ssacc = take(L * sizeof(double));
  c->o_last = take(sizeof(af_decision));
  c->o_ring = take(kRing * sizeof(af_decision));
  c->o_pool = take(n_pool * sizeof(int32_t));

  for (auto &T : c->ts) {
    T.o_ftf = take((n_pool + 1) * sizeof(int32_t));
    T.o_tef = take((n_pool + 1) * sizeof(int32_t));
    T.o_stb = take(T.seg_tile_begin.size() * sizeof(int32_t));
    T.o_tiles = take(T.tiles.size() * sizeof(Tile));
  }
  c->o_part = take(c->ts[1].tiles.size() * sizeof(double));
  c->o_part2 = take((static_cast<size_t>(c->ts[1].max_tiles) / kFinChunk + L + 2) * sizeof(double));
  c->scratch_bytes = o;
  *out = c;
  return AF_OK;
}

af_status af_ctx_workspace_bytes(const af_ctx *c, size_t *accum_bytes, size_t *scratch_bytes) {
  AF_NVTX();
  if (!c || !accum_bytes || !scratch_bytes) return fail(AF_EINVAL, "NULL argument");
  *accum_bytes = c->accum_bytes;
  *scratch_bytes = c->scratch_bytes;
  return AF_OK;
}

af_status af_ctx_info(const af_ctx *c, af_info *info) {
  AF_NVTX();
  if (!c || !info) return fail(AF_EINVAL, "NULL argument");
  std::memset(info, 0, sizeof(*info));
  info->n_segments = c->L;
  info->n_pool = c->n_pool;
  info->rank = c->cfg.rank;
  info->world = c->cfg.world;
  info->n_total = c->n;
  info->shard_begin = c->sb;
  info->shard_end = c->se;
  info->n_tiles = c->ts[1].max_tiles;
  info->tile_elems = c->ts[1].tile_elems;
  info->n_tiles_acc = c->ts[0].max_tiles;
  info->tile_elems_acc = c->ts[0].tile_elems;
  info->n_fin_chunks = (c->ts[1].max_tiles + kFinChunk - 1) / kFinChunk;
  info->n_fin_ctas = 0;  // the finalize runs inside the streaming kernel (fin_worker)
  for (int j = 0; j <= c->n_pool; ++j) info->first_tile_of_pool[j] = c->ts[1].first_tile_of_f[j];
  return AF_OK;
}

af_status af_ctx_shard_of(const af_ctx *c, int32_t f, int64_t *begin, int64_t *end) {
  AF_NVTX();
  if (!c || !begin || !end) return fail(AF_EINVAL, "NULL argument");
  if (f < 0 || f > c->n_pool) return fail(AF_EINVAL, "f out of [0, n_pool]");
  *begin = c->sb_of_f[f];
  *end = c->se_of_f[f];
  return AF_OK;
}

af_status af_ctx_bind(af_ctx *c, void *accum_dev, void *scratch_dev) {
  AF_NVTX();
  if (!c || !scratch_dev) return fail(AF_EINVAL, "NULL argument");
  if (c->accum_bytes && !accum_dev) return fail(AF_EINVAL, "accum buffer required");
  if (!aligned(scratch_dev, 256) || (accum_dev && !aligned(accum_dev, 256)))
    return fail(AF_EINVAL, "workspace buffers must be 256-byte aligned");
  int sms = 0;
  AF_CUDA(cudaGetDevice(&c->device), "cudaGetDevice");
  cudaError_t e = static_cast<cudaError_t>(device_sm_count(&sms));
  if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceGetAttribute");
  e = static_cast<cudaError_t>(preload_norm_kernels(c->dtype, c->cfg.world));
  if (e == cudaSuccess) e = static_cast<cudaError_t>(preload_decide_kernel());
  if (e != cudaSuccess) return cuda_fail(e, "cudaFuncGetAttributes (kernel preload)");
  for (int m = 0; m < kNumModes; ++m) {
    int bps = 0;
    e = static_cast<cudaError_t>(norms_max_blocks_per_sm(m, c->dtype, c->cfg.world, &bps, c->active));
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
    AF_CUDA(cudaMemcpy(c->scratch + T.o_tef, T.tile_end_of_f.data(), T.tile_end_of_f.size() * 4,
                       cudaMemcpyHostToDevice),
            "cudaMemcpy(tile_end_of_f)");
    AF_CUDA(cudaMemcpy(c->scratch + T.o_stb, T.seg_tile_begin.data(), T.seg_tile_begin.size() * 4,
                       cudaMemcpyHostToDevice),
            "cudaMemcpy(seg_tile_begin)");
  }
  AF_CUDA(cudaMemcpy(c->scratch + c->o_pool, c->pool_seg.data(), c->pool_seg.size() * 4, cudaMemcpyHostToDevice),
          "cudaMemcpy(pool_seg)");
  {  // every partial and piece slot starts empty (the finalize waits for non-empty slots)
    const std::vector<unsigned long long> empty(c->ts[1].tiles.size(), kPartialEmpty);
    if (!empty.empty())
      AF_CUDA(cudaMemcpy(c->scratch + c->o_part, empty.data(), empty.size() * 8, cudaMemcpyHostToDevice),
              "cudaMemcpy(partials)");
    const std::vector<unsigned long long> empty2(static_cast<size_t>(c->ts[1].max_tiles) / kFinChunk + c->L + 2,
                                                 kPartialEmpty);
    AF_CUDA(cudaMemcpy(c->scratch + c->o_part2, empty2.data(), empty2.size() * 8, cudaMemcpyHostToDevice),
            "cudaMemcpy(pieces)");
  }
  AF_CUDA(cudaDeviceSynchronize(), "bind");
  c->bound = true;
  c->armed = false;
  c->pending = false;
  return AF_OK;
}

af_status af_nccl_unique_id(void *id_128B) {
  AF_NVTX();
  if (!id_128B) return fail(AF_EINVAL, "NULL argument");
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  ncclUniqueId id;
  ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) return nccl_fail(r, "ncclGetUniqueId");
  std::memcpy(id_128B, &id, sizeof(id));
  return AF_OK;
}

af_status af_ctx_set_comm(af_ctx *c, const void *id_128B) {
  AF_NVTX();
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
  AF_NVTX();
  if (!c || !ss_all_dev) return fail(AF_EINVAL, "NULL argument");
  if (!c->bound) return fail(AF_EWORKSPACE, "workspace not bound");
  *ss_all_dev = c->at<double>(c->o_ssall);
  return AF_OK;
}

}  // extern "C"

namespace {

int grid_for(const af_ctx *c, int mode, int n_tiles) {
  int g = std::min<int>(c->grid[mode], std::max<int>(1, n_tiles));
  if (c->max_ctas > 0) g = std::min(g, c->max_ctas);
  return std::max(1, g);
}

NormParams norm_params(af_ctx *c, const void *grad_dev, bool end, bool dry) {
  NormParams p{};
  const int k = (c->cfg.acc_mode == AF_ACC_DELTA && !end) ? 0 : 1;  // which tile table
  const auto &T = c->ts[k];
  p.grad = grad_dev;
  p.delta = c->accum;
  p.shard_begin = c->active ? 0 : c->sb;  // active-suffix shards: Delta indexed by element
  p.tiles = c->at<Tile>(T.o_tiles);
  p.n_tiles = T.max_tiles;
  p.L = c->L;
  p.first_tile_of_f = c->at<int32_t>(T.o_ftf);
  p.tile_end_of_f = c->at<int32_t>(T.o_tef);
  p.seg_tile_begin = c->at<int32_t>(T.o_stb);
  p.stb_stride = c->active ? c->L + 1 : 0;
  p.state = c->at<DevState>(c->o_state);
  p.sched = c->at<Sched>(c->o_sched) + k;
  p.partials = c->at<double>(c->o_part);
  p.part2 = c->at<double>(c->o_part2);
  p.fin_sched = c->at<Sched>(c->o_sched) + 2;
  p.ss_out = c->at<double>(c->o_ssall) + static_cast<size_t>(c->cfg.rank) * c->L;
  p.ss_acc = c->at<double>(c->o_ssacc);
  p.n_pool = c->n_pool;
  p.reverse = (AF_ALTERNATE_ORDER && c->reverse) ? 1 : 0;
  c->reverse = !c->reverse;
  p.first = c->armed ? 0 : 1;
  p.end = end ? 1 : 0;
  p.dbg_tail_delay_ns = c->dbg_tail_delay_ns;

  p.dbg_peers_arrived = c->dbg_peers_arrived;
  p.dbg_unstaged_tail = c->dbg_unstaged_tail;
  p.commit = dry ? 0 : 1;
  if (c->peers) {
    p.xworld = c->cfg.world;
    p.xrank = c->cfg.rank;
    p.xrows = c->at<unsigned long long>(c->o_xrows);
    p.peer_rows = c->at<unsigned long long *const>(c->o_peer_rows);
  }
  return p;
}

int norm_mode(const af_ctx *c, bool end) {
  if (c->cfg.acc_mode == AF_ACC_DELTA) return end ? kEndDelta : kAccum;
  return kStepSq;
}

DecideParams decide_params(af_ctx *c, bool dry, af_decision *out_host) {
  DecideParams p{};
  p.ss_all = c->at<double>(c->o_ssall);  // the peer exchange assembles its rows here too
  p.world = c->cfg.world;
  p.L = c->L;
  p.n_pool = c->n_pool;
  p.pool_seg = c->at<int32_t>(c->o_pool);
  p.state = c->at<DevState>(c->o_state);
  p.last = c->at<af_decision>(c->o_last);
  p.ring = c->at<af_decision>(c->o_ring);
  p.percentile = c->cfg.percentile;
  p.pct_q = c->cfg.percentile / 100.0;
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

// the NCCL route: world > 1 without peers (or forced by AF_DEBUG_FORCE_NCCL)
bool nccl_route(const af_ctx *c) { return (c->cfg.world > 1 || c->dbg_force_nccl) && !c->peers; }

af_status allgather_rows(af_ctx *c, void *stream) {
  if (nccl_route(c) && c->comm) {
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
  AF_NVTX();
  af_status st = check_norm_args(c, grad_dev);
  if (st != AF_OK) return st;
  if (flags & ~(AF_INTERVAL_END | AF_DRY_RUN)) return fail(AF_EINVAL, "unknown flags");
  const bool end = flags & AF_INTERVAL_END, dry = flags & AF_DRY_RUN;
  const int mode = norm_mode(c, end);
  NormParams p = norm_params(c, grad_dev, end, dry);
  const int grid = grid_for(c, mode, p.n_tiles);
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

}  // extern "C"

namespace {

// AdamW constants rounded once to fp32 (the oracle rounds the same fp64 values)
AdamConst adam_const(const af_adamw &hp) {
  AdamConst a{};
  const double lr = hp.lr, b1 = hp.beta1, b2 = hp.beta2;
  a.decay = static_cast<float>(1.0 - lr * static_cast<double>(hp.weight_decay));
  a.beta1 = hp.beta1;
  a.one_minus_beta1 = static_cast<float>(1.0 - b1);
  a.beta2 = hp.beta2;
  a.one_minus_beta2 = static_cast<float>(1.0 - b2);
  a.step_size = static_cast<float>(lr / (1.0 - std::pow(b1, hp.step)));
  a.sqrt_bc2 = static_cast<float>(std::sqrt(1.0 - std::pow(b2, hp.step)));
  a.eps = hp.eps;
  return a;
}

af_status check_adam(const af_adamw *hp, const float *params_dev, const float *exp_avg_dev,
                     const float *exp_avg_sq_dev) {
  if (!hp || !params_dev || !exp_avg_dev || !exp_avg_sq_dev) return fail(AF_EINVAL, "NULL argument");
  if (!aligned(params_dev, 16) || !aligned(exp_avg_dev, 16) || !aligned(exp_avg_sq_dev, 16))
    return fail(AF_EINVAL, "optimizer buffers must be 16-byte aligned");
  if (hp->step < 1 || !(hp->beta1 >= 0.f && hp->beta1 < 1.f) || !(hp->beta2 >= 0.f && hp->beta2 < 1.f) ||
      !(hp->eps > 0.f) || !(hp->lr >= 0.f) || !(hp->weight_decay >= 0.f))
    return fail(AF_EINVAL, "bad AdamW hyper-parameters");
  return AF_OK;
}

}  // namespace

extern "C" {

af_status af_adamw_step(af_ctx *c, float *params_dev, float *exp_avg_dev, float *exp_avg_sq_dev,
                        const void *grad_dev, const af_adamw *hp, uint32_t flags, af_decision *out_host,
                        void *stream) {
  AF_NVTX();
  if (c && c->active) return fail(AF_ESTATE, "af_adamw_step needs static shards (shard_active = 0)");
  af_status st = check_norm_args(c, grad_dev);
  if (st != AF_OK) return st;
  st = check_adam(hp, params_dev, exp_avg_dev, exp_avg_sq_dev);
  if (st != AF_OK) return st;
  if (c->cfg.acc_mode != AF_ACC_DELTA) return fail(AF_ESTATE, "af_adamw_step needs acc_mode AF_ACC_DELTA");
  if (flags & ~(AF_INTERVAL_END | AF_DRY_RUN)) return fail(AF_EINVAL, "unknown flags");
  const bool end = flags & AF_INTERVAL_END, dry = flags & AF_DRY_RUN;
  if (end && nccl_route(c) && !c->comm)
    return fail(AF_ESTATE, "interval end with world > 1 needs peers or a communicator");
  const int mode = end ? kAdamEnd : kAdamAccum;
  NormParams p = norm_params(c, grad_dev, end, dry);
  p.params = params_dev;
  p.exp_avg = exp_avg_dev;
  p.exp_avg_sq = exp_avg_sq_dev;
  p.adam = adam_const(*hp);
  const bool fuse = end && !nccl_route(c);
  if (fuse) {
    p.fuse_decide = 1;
    p.dec = decide_params(c, dry, out_host);
  }
  const int grid = grid_for(c, mode, p.n_tiles);
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
  AF_NVTX();
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
  AF_NVTX();
  af_status st = check_norm_args(c, grad_dev);
  if (st != AF_OK) return st;
  if (flags & ~(AF_DRY_RUN)) return fail(AF_EINVAL, "unknown flags");
  const bool dry = flags & AF_DRY_RUN;
  if (nccl_route(c)) {  // kernel + all-gather + decide kernel
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
  const int grid = grid_for(c, mode, p.n_tiles);
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
struct IpcHandle {  // AF_IPC_HANDLE_BYTES
  cudaIpcMemHandle_t h;
  uint64_t offset;                 // scratch offset inside the exported allocation
  uint64_t xrows_off, pad0;        // exchange-area offset inside the scratch
  uint64_t rsflags_off;            // fused reduce-scatter flags inside the scratch
  int32_t rank, world, L, pad;
};
static_assert(sizeof(IpcHandle) <= AF_IPC_HANDLE_BYTES, "ipc handle size");

static af_status upload_peers(af_ctx *c, const std::vector<char *> &scratch_of) {
  std::vector<unsigned long long *> rows(c->cfg.world), rsflags(c->cfg.world);
  for (int r = 0; r < c->cfg.world; ++r) {
    rows[r] = reinterpret_cast<unsigned long long *>(scratch_of[r] + c->o_xrows);
    rsflags[r] = reinterpret_cast<unsigned long long *>(scratch_of[r] + c->o_rsflags);
  }
  AF_CUDA(cudaMemcpy(c->scratch + c->o_peer_rsflags, rsflags.data(), rsflags.size() * sizeof(void *),
                     cudaMemcpyHostToDevice),
          "cudaMemcpy(peer rs flags)");
  AF_CUDA(cudaMemcpy(c->scratch + c->o_peer_rows, rows.data(), rows.size() * sizeof(void *), cudaMemcpyHostToDevice),
          "cudaMemcpy(peer rows)");
  AF_CUDA(cudaDeviceSynchronize(), "set peers");
  c->peers = true;
  return AF_OK;
}

af_status af_ctx_exchange_ipc_handle(af_ctx *c, void *handle_out) {
  AF_NVTX();
  if (!c || !handle_out) return fail(AF_EINVAL, "NULL argument");
  if (!c->bound) return fail(AF_EWORKSPACE, "workspace not bound");
  IpcRef r{};
  af_status st = ipc_export(c->scratch, &r);
  if (st != AF_OK) return st;
  IpcHandle h{};
  h.h = r.h;
  h.offset = r.offset;
  h.xrows_off = c->o_xrows;
  h.rsflags_off = c->o_rsflags;
  h.rank = c->cfg.rank;
  h.world = c->cfg.world;
  h.L = c->L;
  std::memset(handle_out, 0, AF_IPC_HANDLE_BYTES);
  std::memcpy(handle_out, &h, sizeof(h));
  return AF_OK;
}

af_status af_ctx_set_peers_ipc(af_ctx *c, const void *handles) {
  AF_NVTX();
  if (!c || !handles) return fail(AF_EINVAL, "NULL argument");
  if (!c->bound) return fail(AF_EWORKSPACE, "workspace not bound");
  if (c->peers) return fail(AF_ESTATE, "peers already set");
  std::vector<char *> scratch_of(c->cfg.world, nullptr);
  for (int r = 0; r < c->cfg.world; ++r) {
    IpcHandle h;
    std::memcpy(&h, static_cast<const char *>(handles) + static_cast<size_t>(r) * AF_IPC_HANDLE_BYTES, sizeof(h));
    if (h.rank != r || h.world != c->cfg.world || h.L != c->L || h.xrows_off != c->o_xrows ||
        h.rsflags_off != c->o_rsflags)
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
  AF_NVTX();
  if (!c) return fail(AF_EINVAL, "NULL ctx");
  c->peers = false;  // mappings stay open until af_ctx_destroy
  return AF_OK;
}

af_status af_ctx_set_peers_local(af_ctx *c, af_ctx *const *peers) {
  AF_NVTX();
  if (!c || !peers) return fail(AF_EINVAL, "NULL argument");
  if (!c->bound) return fail(AF_EWORKSPACE, "workspace not bound");
  if (c->peers) return fail(AF_ESTATE, "peers already set");
  std::vector<char *> scratch_of(c->cfg.world, nullptr);
  for (int r = 0; r < c->cfg.world; ++r) {
    const af_ctx *q = peers[r];
    if (!q || !q->bound || q->cfg.rank != r || q->cfg.world != c->cfg.world || q->L != c->L ||
        q->o_xrows != c->o_xrows || q->o_rsflags != c->o_rsflags)
      return fail(AF_EINVAL, "peer context mismatch");
    // a peer bound on another device: its scratch is reached over NVLink
    const af_status st = enable_peer_access(q->device);
    if (st != AF_OK) return st;
    scratch_of[r] = q->scratch;
  }
  return upload_peers(c, scratch_of);
}

af_status af_ctx_set_max_ctas(af_ctx *c, int32_t max_ctas) {
  AF_NVTX();
  if (!c) return fail(AF_EINVAL, "NULL ctx");
  if (max_ctas < 0) return fail(AF_EINVAL, "max_ctas < 0");
  c->max_ctas = max_ctas;
  return AF_OK;
}

// ---------------------------------------------------------------- fused reduce-scatter

struct GradHandle {  // AF_IPC_HANDLE_BYTES
  cudaIpcMemHandle_t h;
  uint64_t offset;
  int64_t n;
  int32_t rank, world, dtype, pad;
};
static_assert(sizeof(GradHandle) <= AF_IPC_HANDLE_BYTES, "grad handle size");

static af_status upload_grads(af_ctx *c, const std::vector<const void *> &g) {
  AF_CUDA(cudaMemcpy(c->scratch + c->o_rs_grads, g.data(), g.size() * sizeof(void *), cudaMemcpyHostToDevice),
          "cudaMemcpy(rs grads)");
  AF_CUDA(cudaDeviceSynchronize(), "set grad peers");
  c->grad_peers = true;
  return AF_OK;
}

af_status af_ctx_grad_ipc_handle(af_ctx *c, const void *grad_dev, void *handle_out) {
  AF_NVTX();
  if (!c || !grad_dev || !handle_out) return fail(AF_EINVAL, "NULL argument");
  if (!c->bound) return fail(AF_EWORKSPACE, "workspace not bound");
  if (!aligned(grad_dev, 16)) return fail(AF_EINVAL, "gradient buffer must be 16-byte aligned");
  IpcRef r{};
  af_status st = ipc_export(grad_dev, &r);
  if (st != AF_OK) return st;
  GradHandle h{};
  h.h = r.h;
  h.offset = r.offset;
  h.n = c->n;
  h.rank = c->cfg.rank;
  h.world = c->cfg.world;
  h.dtype = c->dtype;
  std::memset(handle_out, 0, AF_IPC_HANDLE_BYTES);
  std::memcpy(handle_out, &h, sizeof(h));
  c->own_grad = grad_dev;
  return AF_OK;
}

af_status af_ctx_set_grad_peers_ipc(af_ctx *c, const void *handles) {
  AF_NVTX();
  if (!c || !handles) return fail(AF_EINVAL, "NULL argument");
  if (!c->bound) return fail(AF_EWORKSPACE, "workspace not bound");
  if (c->cfg.world > kMaxRsWorld) return fail(AF_EINVAL, "fused reduce-scatter supports world <= 8");
  if (!c->own_grad) return fail(AF_ESTATE, "call af_ctx_grad_ipc_handle on this rank first");
  std::vector<const void *> g(c->cfg.world, nullptr);
  for (int r = 0; r < c->cfg.world; ++r) {
    GradHandle h;
    std::memcpy(&h, static_cast<const char *>(handles) + static_cast<size_t>(r) * AF_IPC_HANDLE_BYTES, sizeof(h));
    if (h.rank != r || h.world != c->cfg.world || h.n != c->n || h.dtype != c->dtype)
      return fail(AF_EINVAL, "gradient handle mismatch");
    if (r == c->cfg.rank) {
      g[r] = c->own_grad;
      continue;
    }
    char *ptr = nullptr;
    af_status st = ipc_import(IpcRef{h.h, h.offset}, c->ipc_opened, &ptr);
    if (st != AF_OK) return st;
    g[r] = ptr;
  }
  return upload_grads(c, g);
}

af_status af_ctx_set_grad_peers_local(af_ctx *c, const void *const *grads_dev) {
  AF_NVTX();
  if (!c || !grads_dev) return fail(AF_EINVAL, "NULL argument");
  if (!c->bound) return fail(AF_EWORKSPACE, "workspace not bound");
  if (c->cfg.world > kMaxRsWorld) return fail(AF_EINVAL, "fused reduce-scatter supports world <= 8");
  std::vector<const void *> g(c->cfg.world);
  for (int r = 0; r < c->cfg.world; ++r) {
    if (!grads_dev[r] || !aligned(grads_dev[r], 16)) return fail(AF_EINVAL, "gradient buffers must be 16-byte aligned");
    const af_status st = enable_peer_access_to(grads_dev[r]);
    if (st != AF_OK) return st;
    g[r] = grads_dev[r];
  }
  c->own_grad = g[c->cfg.rank];
  return upload_grads(c, g);
}

}  // extern "C"

static af_status rs_step(af_ctx *c, float scale, float *grad_shard_out_dev, const af_adamw *hp, float *params_dev,
                         float *exp_avg_dev, float *exp_avg_sq_dev, uint32_t flags, af_decision *out_host,
                         void *stream) {
  if (!c) return fail(AF_EINVAL, "NULL ctx");
  if (c->active) return fail(AF_ESTATE, "af_reduce_scatter_step needs static shards (shard_active = 0)");
  if (!c->bound) return fail(AF_EWORKSPACE, "workspace not bound");
  if (!c->grad_peers) return fail(AF_ESTATE, "no gradient buffers registered (af_ctx_set_grad_peers_*)");
  if (c->cfg.acc_mode != AF_ACC_DELTA) return fail(AF_ESTATE, "af_reduce_scatter_step needs acc_mode AF_ACC_DELTA");
  if (flags & ~(AF_INTERVAL_END | AF_DRY_RUN)) return fail(AF_EINVAL, "unknown flags");
  if (grad_shard_out_dev && !aligned(grad_shard_out_dev, 16)) return fail(AF_EINVAL, "output must be 16-byte aligned");
  if (!std::isfinite(scale)) return fail(AF_EINVAL, "scale must be finite");
  if (c->cfg.world > 1 && !c->peers)
    return fail(AF_ESTATE, "world > 1 needs peers (af_ctx_set_peers_*) for the reduce-scatter flags");
  const bool end = flags & AF_INTERVAL_END, dry = flags & AF_DRY_RUN;
  const bool adam = hp != nullptr;
  const int mode = adam ? (end ? kRsAdamEnd : kRsAdamAccum) : (end ? kRsEnd : kRsAccum);
  NormParams p = norm_params(c, c->own_grad, end, dry);
  if (adam) {
    p.params = params_dev;
    p.exp_avg = exp_avg_dev;
    p.exp_avg_sq = exp_avg_sq_dev;
    p.adam = adam_const(*hp);
  }
  p.rs_world = c->cfg.world;
  p.rs_rank = c->cfg.rank;
  p.rs_grads = c->at<const void *const>(c->o_rs_grads);
  p.rs_scale = scale;
  p.rs_out = grad_shard_out_dev;
  p.rs_flags = c->at<unsigned long long>(c->o_rsflags);
  p.peer_rs_flags = c->at<unsigned long long *const>(c->o_peer_rsflags);
  if (end) {
    p.fuse_decide = 1;
    p.dec = decide_params(c, dry, out_host);
  }
  const int e = launch_norms(p, mode, c->dtype, grid_for(c, mode, p.n_tiles), stream);
  if (e != 0) return cuda_fail(static_cast<cudaError_t>(e), "fused reduce-scatter kernel launch");
  if (end) {
    af_status st = copy_record_if_unmapped(c, p.dec, out_host, stream);
    if (st != AF_OK) return st;
  }
  if (!dry) {
    c->armed = !end;
    c->pending = false;
  }
  return AF_OK;
}

extern "C" {

af_status af_reduce_scatter_step(af_ctx *c, float scale, float *grad_shard_out_dev, uint32_t flags,
                                 af_decision *out_host, void *stream) {
  AF_NVTX();
  return rs_step(c, scale, grad_shard_out_dev, nullptr, nullptr, nullptr, nullptr, flags, out_host, stream);
}

af_status af_reduce_scatter_adamw_step(af_ctx *c, float scale, float *params_dev, float *exp_avg_dev,
                                       float *exp_avg_sq_dev, const af_adamw *hp, float *grad_shard_out_dev,
                                       uint32_t flags, af_decision *out_host, void *stream) {
  AF_NVTX();
  const af_status st = check_adam(hp, params_dev, exp_avg_dev, exp_avg_sq_dev);
  if (st != AF_OK) return st;
  return rs_step(c, scale, grad_shard_out_dev, hp, params_dev, exp_avg_dev, exp_avg_sq_dev, flags, out_host, stream);
}

struct StateBlob {
  char magic[4];
  int32_t version, L, world, rank, T, f, armed;
  double prev[AF_MAX_SEGMENTS];
  double ss_acc[AF_MAX_SEGMENTS];
};

af_status af_get_state(af_ctx *c, void *buf, size_t *len) {
  AF_NVTX();
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
  AF_NVTX();
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
  // active-suffix shards: Delta's elements belong to the shard of the f it was
  // accumulated under; a different f starts a fresh interval sum
  const bool moved = c->active && st.f != b.f;
  st.sticky = 0;
  st.T = b.T;
  st.f = b.f;
  std::memcpy(st.prev, b.prev, sizeof(st.prev));
  AF_CUDA(cudaMemcpy(c->scratch + c->o_state, &st, sizeof(st), cudaMemcpyHostToDevice), "cudaMemcpy(state)");
  AF_CUDA(cudaMemcpy(c->scratch + c->o_ssacc, b.ss_acc, c->L * sizeof(double), cudaMemcpyHostToDevice),
          "cudaMemcpy(ss_acc)");
  AF_CUDA(cudaDeviceSynchronize(), "set_state sync");
  c->armed = b.armed != 0 && !moved;
  c->pending = false;
  return AF_OK;
}

af_status af_ctx_read_record(af_ctx *c, int32_t interval, af_decision *out) {
  AF_NVTX();
  if (!c || !out) return fail(AF_EINVAL, "NULL argument");
  if (!c->bound) return fail(AF_EWORKSPACE, "workspace not bound");
  if (interval < 0) return fail(AF_ERANGE, "interval < 0");
  AF_CUDA(cudaDeviceSynchronize(), "read_record sync");
  af_decision r;
  AF_CUDA(cudaMemcpy(&r, c->at<af_decision>(c->o_ring) + (interval % kRing), sizeof(r), cudaMemcpyDeviceToHost),
          "cudaMemcpy(ring record)");
  // an untouched slot is all zero: interval 0 is told apart by its flags (a decided
  // record always carries at least one flag bit or a finite threshold)
  const bool empty = r.interval == 0 && r.flags == 0 && !(r.threshold == r.threshold);
  if (r.interval != interval || (interval == 0 && empty)) return fail(AF_ERANGE, "interval not in the ring");
  *out = r;
  return AF_OK;
}

af_status af_ctx_set_debug(af_ctx *c, int32_t key, int64_t value) {
  AF_NVTX();
  if (!c) return fail(AF_EINVAL, "NULL ctx");
  switch (key) {
    case AF_DEBUG_TAIL_DELAY_NS:
      if (value < 0 || value > 1000000000ll) return fail(AF_EINVAL, "tail delay out of [0, 1e9] ns");
      c->dbg_tail_delay_ns = static_cast<uint32_t>(value);
      return AF_OK;
    case AF_DEBUG_PEERS_ARRIVED:
      if (value != 0 && value != 1) return fail(AF_EINVAL, "peers-arrived knob is 0 or 1");
      c->dbg_peers_arrived = static_cast<int32_t>(value);
      return AF_OK;
    case AF_DEBUG_FORCE_NCCL:
      if (value != 0 && value != 1) return fail(AF_EINVAL, "force-NCCL knob is 0 or 1");
      c->dbg_force_nccl = static_cast<int32_t>(value);
      return AF_OK;
    case AF_DEBUG_UNSTAGED_TAIL:
      if (value != 0 && value != 1) return fail(AF_EINVAL, "unstaged-tail knob is 0 or 1");
      c->dbg_unstaged_tail = static_cast<int32_t>(value);
      return AF_OK;
    default: return fail(AF_EINVAL, "unknown debug key");
  }
}

af_status af_ctx_destroy(af_ctx *c) {
  AF_NVTX();
  if (!c) return fail(AF_EINVAL, "NULL ctx");
  if (c->comm) ncclCommDestroy(c->comm);
  ipc_release(c->ipc_opened);
  delete c;
  return AF_OK;
}

}  // extern "C"
