// af_cache.cu -- Storage Manager put/get kernels.
//
// The paper's storage manager writes the frozen prefix's output for every
// processed example at the original index and reads it back by original index
// in the next epoch, evicting a record on read when the frozen depth grew
// (§3.2).  Here the store is an HBM-resident direct-mapped
// table per GPU (slot = id / world for the ids id % world == rank, §3.4).
//
// Data movement is pure bytes (bit-exact) and HBM-bound: 2 * rows * row_bytes.
// Each CTA drives a TMA bulk-copy ring (cp.async.bulk global->shared with an
// mbarrier transaction count, then cp.async.bulk shared->global in bulk groups),
// STAGES x 32 KiB of shared memory, one elected lane issuing, so up to
// STAGES-1 chunk loads and the matching stores are in flight per CTA without
// register staging.  Work items are (row, 32 KiB chunk) pairs dealt round-robin
// to a persistent grid of two CTAs (3 stages each) per SM -- the best of the
// profiles/r01_v9_variants_cache.jsonl sweep, confirmed with a cold L2 and
// graph-timed calls in profiles/r01_v34_cache_cold_graph.jsonl.  Each CTA has two
// warps: warp 0 turns ids into addresses and streams the copies, warp 1 does the
// meta side (see cache_kernel), so a get's record load does not wait for its
// meta word.  A get evicts a record only after every chunk of its row has read
// the meta word (a per-record reader count, fenced), so all chunks of a row
// agree on hit/miss.
#include <cuda_runtime.h>

#include "af_internal.h"
#include "af_ptx.cuh"

namespace af {
namespace {

#ifndef AF_CACHE_STAGES
#define AF_CACHE_STAGES 3
#endif
#ifndef AF_CACHE_CHUNK
#define AF_CACHE_CHUNK (32 * 1024)
#endif
#ifndef AF_CACHE_CTAS_PER_SM
#define AF_CACHE_CTAS_PER_SM 2
#endif

constexpr int kStages = AF_CACHE_STAGES;
constexpr int kChunk = AF_CACHE_CHUNK;
constexpr int kMaxDesc = 512;

struct Desc {
  const char *src;
  char *dst;
  uint32_t bytes;
  uint32_t ok;
};

__device__ __forceinline__ void bulk_g2s(void *dst_smem, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst_smem)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_s2g(void *dst, const void *src_smem, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src_smem)),
               "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// Two warps per CTA.  Warp 0 resolves each item's addresses from its id alone
// (direct-mapped: slot = id / world) and its lane 0 starts the TMA loads at
// once; warp 1 reads the meta words in parallel (get: hit + depth_out; put:
// {depth, valid}) and publishes the hit flags through an mbarrier that lane 0
// waits on before its first store.  A get therefore loads the record
// speculatively -- the meta round trip and the evict-on-read bookkeeping (fence
// + reader count) are off the id -> load -> store chain; a miss discards the
// loaded chunk and stores nothing.
constexpr int kMiss = -2147483647 - 1;

template <bool PUT>
__device__ __forceinline__ bool item_owner(const CacheParams &p, int i, int c, bool report, char *&payload,
                                           CacheMeta *&meta, int64_t &id) {
  id = p.ids[i];
  payload = p.payload;
  meta = p.meta;
  if (id < 0 || id >= p.num_examples) {
    if (report && c == 0) atomicOr(p.err, AF_CACHE_ERR_RANGE);
    return false;
  }
  if (p.peer_payload) {  // global: the owner's store, possibly a peer's
    const int owner = static_cast<int>(id % p.world);
    payload = p.peer_payload[owner];
    meta = p.peer_meta[owner];
  } else if (id % p.world != p.rank) {
    if (report && c == 0) atomicOr(p.err, AF_CACHE_ERR_OWNER);
    return false;
  }
  return true;
}

template <bool PUT>
__device__ __forceinline__ Desc item_addr(const CacheParams &p, int64_t j) {
  const int i = static_cast<int>(j / p.n_chunks);
  const int c = static_cast<int>(j % p.n_chunks);
  Desc dsc{nullptr, nullptr, 0u, 0u};
  const int64_t off = static_cast<int64_t>(c) * p.chunk_bytes;
  const int64_t rem = p.row_bytes - off;
  dsc.bytes = static_cast<uint32_t>(rem < p.chunk_bytes ? rem : p.chunk_bytes);
  char *payload;
  CacheMeta *meta;
  int64_t id;
  if (!item_owner<PUT>(p, i, c, true, payload, meta, id)) return dsc;
  char *rec;
  if (p.rowslot) {  // tiered: the plan kernel resolved the row's slot (and its meta / eviction)
    const int32_t slot = p.rowslot[i];
    if (slot < 0) return dsc;
    if (p.stage != nullptr && slot >= p.disk_base)  // disk tier: this pass's staging row i (host callbacks move it)
      rec = p.stage + static_cast<int64_t>(i) * p.row_bytes + off;
    else
      rec = (slot < p.hbm_rows ? p.payload + static_cast<int64_t>(slot) * p.row_bytes
                               : p.host + (static_cast<int64_t>(slot) - p.hbm_rows) * p.row_bytes) +
            off;
  } else {
    rec = payload + (id / p.world) * p.row_bytes + off;
  }
  if (PUT) {
    dsc.src = p.src_rows + static_cast<int64_t>(i) * p.row_bytes + off;
    dsc.dst = rec;
  } else {
    dsc.src = rec;
    dsc.dst = p.dst_rows + static_cast<int64_t>(i) * p.row_bytes + off;
  }
  dsc.ok = 1u;
  return dsc;
}

// warp 1: the meta side of item j.  Returns the record's depth on a get hit
// (kMiss otherwise; tiered and put: 0 = store).
template <bool PUT>
__device__ __forceinline__ int item_meta(const CacheParams &p, int64_t j) {
  const int i = static_cast<int>(j / p.n_chunks);
  const int c = static_cast<int>(j % p.n_chunks);
  char *payload;
  CacheMeta *meta;
  int64_t id;
  const bool ok = item_owner<PUT>(p, i, c, false, payload, meta, id);
  if (p.rowslot) return 0;  // tiered: the plan kernel did the meta work
  if (!ok) {
    if (!PUT && c == 0) p.depth_out[i] = -1;
    return kMiss;
  }
  const int64_t slot = id / p.world;
  if (PUT) {
    if (c == 0) *reinterpret_cast<int2 *>(meta + slot) = make_int2(p.depth, 1);  // {depth, valid}
    return 0;
  }
  const int4 mv = __ldcg(reinterpret_cast<const int4 *>(meta) + slot);  // {depth, valid, readers, -}
  const bool hit = mv.y != 0;
  if (c == 0) p.depth_out[i] = hit ? mv.x : -1;
  return hit ? mv.x : kMiss;
}

// evict on read once every chunk of the row has read the record
__device__ __forceinline__ void item_evict(const CacheParams &p, int64_t j, int depth) {
  const int i = static_cast<int>(j / p.n_chunks);
  const int64_t id = p.ids[i];
  CacheMeta *meta = p.peer_meta ? p.peer_meta[id % p.world] : p.meta;
  const int64_t slot = id / p.world;
  __threadfence();
  const unsigned int seen = atomicAdd(&meta[slot].readers, 1u);
  if (seen == static_cast<unsigned int>(p.n_chunks) - 1u) {
    if (depth < p.cur_boundary) meta[slot].valid = 0;
    meta[slot].readers = 0u;
  }
}

__device__ void pump_spec(const Desc *descs, const int *hitdep, int m, unsigned char *stage_buf, uint64_t *bars,
                          uint32_t &seq, uint64_t *hbar, uint32_t hpar, bool gate) {
  uint32_t n_ok = 0;
  for (int i = 0; i < m; ++i) n_ok += descs[i].ok;
  auto next_ok = [&](int i) {
    while (i < m && !descs[i].ok) ++i;
    return i;
  };
  const uint32_t base = seq;
  uint32_t loaded = 0;
  int load_i = next_ok(0);
  while (loaded < n_ok && loaded < kStages - 1) {
    const uint32_t u = base + loaded;
    const int s = u % kStages;
    mbar_expect_tx(&bars[s], descs[load_i].bytes);
    bulk_g2s(stage_buf + static_cast<size_t>(s) * kChunk, descs[load_i].src, descs[load_i].bytes, &bars[s]);
    ++loaded;
    load_i = next_ok(load_i + 1);
  }
  if (gate && n_ok) mbar_wait(hbar, hpar);  // warp 1's hit flags for this batch
  int store_i = next_ok(0);
  for (uint32_t q = 0; q < n_ok; ++q) {
    const uint32_t u = base + q;
    const int s = u % kStages;
    mbar_wait(&bars[s], (u / kStages) & 1u);
    const bool st = !gate || hitdep[store_i] != kMiss;  // put: warp 1 publishes no flags (and never a miss for an ok item)
    if (st) bulk_s2g(descs[store_i].dst, stage_buf + static_cast<size_t>(s) * kChunk, descs[store_i].bytes);
    store_i = next_ok(store_i + 1);
    if (loaded < n_ok) {
      if (st) bulk_wait_read1();  // the store that last used the stage we refill has read its bytes
      else bulk_wait_read0();
      const uint32_t v = base + loaded;
      const int sv = v % kStages;
      mbar_expect_tx(&bars[sv], descs[load_i].bytes);
      bulk_g2s(stage_buf + static_cast<size_t>(sv) * kChunk, descs[load_i].src, descs[load_i].bytes, &bars[sv]);
      ++loaded;
      load_i = next_ok(load_i + 1);
    }
  }
  bulk_wait_read0();  // the next batch may reuse every stage
  seq = base + n_ok;
}

constexpr int kCacheThreads = 64;

template <bool PUT>
__global__ void __launch_bounds__(kCacheThreads) cache_kernel(const CacheParams p) {
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem);
  uint64_t *hbar = bars + kStages;
  unsigned char *stage_buf = smem + 128;
  Desc *descs = reinterpret_cast<Desc *>(stage_buf + static_cast<size_t>(kStages) * kChunk);
  int *hitdep = reinterpret_cast<int *>(descs + kMaxDesc);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(&bars[s], 1);
    mbar_init(hbar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (!p.no_wait) pdl_wait();  // ids, rows and the meta words may come from the preceding kernels

  const int64_t n_items = static_cast<int64_t>(p.n) * p.n_chunks;
  const int64_t G = gridDim.x;
  const int64_t my_items = (n_items > blockIdx.x) ? (n_items - blockIdx.x + G - 1) / G : 0;
  uint32_t seq = 0, batch = 0;
  for (int64_t kb = 0; kb < my_items; kb += kMaxDesc, ++batch) {
    const int m = static_cast<int>((my_items - kb) < kMaxDesc ? (my_items - kb) : kMaxDesc);
    if (warp == 0) {
      for (int q = lane; q < m; q += 32) descs[q] = item_addr<PUT>(p, blockIdx.x + (kb + q) * G);
      __syncwarp();
      if (lane == 0) pump_spec(descs, hitdep, m, stage_buf, bars, seq, hbar, batch & 1u, !PUT);
      __syncwarp();
    } else {
      for (int q = lane; q < m; q += 32) hitdep[q] = item_meta<PUT>(p, blockIdx.x + (kb + q) * G);
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(hbar)) : "memory");
      if (!PUT && !p.rowslot) {
        for (int q = lane; q < m; q += 32)
          if (hitdep[q] != kMiss) item_evict(p, blockIdx.x + (kb + q) * G, hitdep[q]);
      }
    }
    __syncthreads();  // descs / hitdep of this batch are consumed
  }
  // AF_CACHE_OVERLAP_PREV: the copy above ran without waiting for the preceding
  // kernel, but the get must not COMPLETE before it -- every later kernel waits
  // only on the get, and the preceding interval end may still be committing f /
  // prev / T in its last CTA (or spinning on peers there).  So the last CTA to
  // finish its copies waits for the predecessor before it exits: get complete
  // => predecessor complete, while every other CTA retires at once and frees its
  // SM for the next kernels (all CTAs waiting cost ~9 us per step,
  // profiles/r02_v7_*).
  pdl_launch_dependents();
#ifndef AF_CACHE_OVERLAP_UNSAFE  // diagnostic build only: the round-1 behaviour the ordering test must catch
  if (p.no_wait) {
    __shared__ int s_last_get;
    if (threadIdx.x == 0) s_last_get = atomicAdd(p.retire, 1u) == gridDim.x - 1u;
    __syncthreads();
    if (s_last_get && threadIdx.x == 0) {
      *p.retire = 0u;  // every CTA has counted: re-armed for the next call
      pdl_wait();
    }
  }
#endif
  if (threadIdx.x == 0) bulk_wait_all();  // all stores complete before the CTA retires its shared memory
}

// Tiered-mode plan (one CTA, 1024 threads): resolves every row of the call in call
// order with block-wide exclusive scans, so slot allocation and freeing are
// deterministic.  put: existing record -> its slot (re-cache deeper); new id ->
// the next free slot (HBM slots are handed out first), or dropped when none is
// left (drop-newest; the store never exceeds its capacity).  get:
// hit -> depth_out and the slot; hits with depth < cur_boundary are evicted and
// their slots pushed back (P:277 re-cache balance).
constexpr int kPlanThreads = 1024;

__device__ __forceinline__ int block_exclusive_scan(int v, int *s_warp, int &total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xFFFFFFFFu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_warp[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int w = (lane < kPlanThreads / 32) ? s_warp[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xFFFFFFFFu, w, o);
      if (lane >= o) w += y;
    }
    s_warp[lane] = w;  // inclusive warp prefix
  }
  __syncthreads();
  const int before = (warp > 0 ? s_warp[warp - 1] : 0) + x - v;
  total = s_warp[kPlanThreads / 32 - 1];
  __syncthreads();
  return before;
}

__global__ void __launch_bounds__(kPlanThreads) cache_plan_kernel(const CachePlanParams p) {
  __shared__ int s_warp[32];
  __shared__ int s_top;
  __shared__ unsigned int s_dropped;
  pdl_wait();
  if (threadIdx.x == 0) {
    s_top = p.hdr->top;
    s_dropped = 0u;
    if (p.manifest) {  // disk tier: the host callback's work list for this pass
      p.manifest[0] = p.n;
      p.manifest[1] = p.put;
    }
  }
  __syncthreads();
  for (int base = 0; base < p.n; base += kPlanThreads) {
    const int i = base + threadIdx.x;
    int need = 0, slot = -1;
    int64_t lid = -1;
    int4 m = make_int4(0, 0, 0, -1);
    if (i < p.n) {
      const int64_t id = p.ids[i];
      if (id < 0 || id >= p.num_examples) {
        atomicOr(&p.hdr->err, AF_CACHE_ERR_RANGE);
      } else if (id % p.world != p.rank) {
        atomicOr(&p.hdr->err, AF_CACHE_ERR_OWNER);
      } else {
        lid = id / p.world;
        m = __ldcg(reinterpret_cast<const int4 *>(p.meta) + lid);
        if (p.put) {
          if (m.y) slot = m.w;
          else need = 1;
        } else {
          if (m.y) {
            slot = m.w;
            p.depth_out[i] = m.x;
            need = (m.x < p.cur_boundary) ? 1 : 0;
          } else {
            p.depth_out[i] = -1;
          }
        }
      }
    }
    int total = 0;
    const int k = block_exclusive_scan(need, s_warp, total);
    const int top = s_top;
    if (i < p.n) {
      if (p.put) {
        if (need) slot = (k < top) ? p.free_slots[top - 1 - k] : -1;
        p.rowslot[i] = slot;
        if (slot >= 0) reinterpret_cast<int4 *>(p.meta)[lid] = make_int4(p.depth, 1, 0, slot);
      } else {
        p.rowslot[i] = slot;
        if (need) {
          p.free_slots[top + k] = slot;
          reinterpret_cast<int4 *>(p.meta)[lid] = make_int4(m.x, 0, 0, -1);
        }
      }
      if (p.manifest) p.manifest[2 + i] = (slot >= 0 && slot >= p.disk_base) ? slot - p.disk_base : -1;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      if (p.put) {
        const int got = total < top ? total : top;
        s_dropped += static_cast<unsigned int>(total - got);
        s_top = top - got;
      } else {
        s_top = top + total;
      }
    }
    __syncthreads();
  }
  pdl_launch_dependents();
  if (threadIdx.x == 0) {
    p.hdr->top = s_top;
    p.hdr->dropped += s_dropped;
  }
}

}  // namespace

int cache_smem_bytes() { return 128 + kStages * kChunk + kMaxDesc * static_cast<int>(sizeof(Desc) + sizeof(int)); }

template <bool PUT>
static int launch_cache(const CacheParams &p0, int grid, void *stream) {
  CacheParams p = p0;
  p.chunk_bytes = kChunk;
  p.n_chunks = static_cast<int32_t>((p.row_bytes + kChunk - 1) / kChunk);
  const int64_t items = static_cast<int64_t>(p.n) * p.n_chunks;
  if (items < grid) grid = static_cast<int>(items);
  if (grid < 1) grid = 1;
  const int smem = cache_smem_bytes();
  const cudaError_t e = ensure_smem_attr<cache_kernel<PUT>>(smem);
  if (e != cudaSuccess) return static_cast<int>(e);
  return static_cast<int>(launch_pdl(cache_kernel<PUT>, dim3(grid), dim3(kCacheThreads), static_cast<size_t>(smem),
                                     static_cast<cudaStream_t>(stream), p));
}

int launch_cache_put(const CacheParams &p, int grid, void *stream) {
  return launch_cache<true>(p, grid * AF_CACHE_CTAS_PER_SM, stream);
}
int launch_cache_get(const CacheParams &p, int grid, void *stream) {
  return launch_cache<false>(p, grid * AF_CACHE_CTAS_PER_SM, stream);
}

}  // namespace af

namespace af {
int preload_cache_kernels() {  // see preload_norm_kernels: no lazy load while peers spin
  cudaFuncAttributes a;
  for (const void *k : {reinterpret_cast<const void *>(cache_kernel<true>),
                        reinterpret_cast<const void *>(cache_kernel<false>),
                        reinterpret_cast<const void *>(cache_plan_kernel)}) {
    const cudaError_t e = cudaFuncGetAttributes(&a, k);
    if (e != cudaSuccess) return static_cast<int>(e);
  }
  return 0;
}

int launch_cache_plan(const CachePlanParams &p, void *stream) {
  return static_cast<int>(launch_pdl(cache_plan_kernel, dim3(1), dim3(kPlanThreads), 0,
                                     static_cast<cudaStream_t>(stream), p));
}
}  // namespace af
