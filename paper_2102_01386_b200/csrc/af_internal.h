// af_internal.h -- structures shared by the host library and the sm_100a kernels.
// Not part of the ABI (include/af.h is).
#pragma once
#include <cstddef>
#include <cstdint>

#include "../../include/af.h"

namespace af {

constexpr int kNormBlock = 256;          // threads per CTA of the streaming kernels
// Tile = the unit of dynamic scheduling and of one fp64 partial.  Sized in
// elements: a bf16 interval-end tile is 32 KiB of g + 64 KiB of Delta, an fp32
// one 32 + 32 KiB -- enough tiles per CTA to bound the end-of-kernel imbalance
// (see profiles/ for the sweeps).
#ifndef AF_TILE_ELEMS_F32  // 8192 since the wide finalize made more partials cheap:
#define AF_TILE_ELEMS_F32 8192  // BERT-large interval end -1.7 % (profiles/r01_v20_variants_end_tiles_f32.jsonl)
#endif
#ifndef AF_TILE_ELEMS_BF16  // 24576: BERT-base interval end -0.8 us in the step vs 16384, 12288 +9 us
#define AF_TILE_ELEMS_BF16 24576  // (profiles/r01_v59_variants_end_tiles_bf16.jsonl)
#endif
#ifndef AF_TILE_TAPER_PCT  // interval-end tiles: % of each table's range, at EACH end, cut into
#define AF_TILE_TAPER_PCT 0   // tiles AF_TILE_TAPER_DIV times smaller (0: uniform tiles)
#endif
#ifndef AF_TILE_TAPER_DIV
#define AF_TILE_TAPER_DIV 4
#endif
#ifndef AF_TILE_SSQ_F32  // STEP_SUMSQ reads only g (s_g bytes per element): larger tiles in
#define AF_TILE_SSQ_F32 32768  // elements keep the per-tile fixed costs small
#endif                          // (profiles/r01_v26_variants_stepsq.jsonl)
#ifndef AF_TILE_SSQ_BF16
#define AF_TILE_SSQ_BF16 32768
#endif
#ifndef AF_TILE_ACC_F32  // the accumulate kernel keeps no partials: finer tiles balance better
#define AF_TILE_ACC_F32 8192
#endif
#ifndef AF_TILE_ACC_BF16
#define AF_TILE_ACC_BF16 8192
#endif
constexpr int kRing = 16;                // decision records kept on the device
constexpr int kShardAlign = 8;           // shard bounds are multiples of 8 elements (32 B fp32 Delta)

// A segment-aligned tile: global element range [begin, end) inside one segment.
// 32 bytes so a descriptor moves with two 16-byte cp.async copies.
struct alignas(16) Tile {
  int64_t begin, end;
  int32_t seg, seg_first, seg_end, pad;  // seg_first/seg_end: the segment's tile range [seg_first, seg_end)
};
static_assert(sizeof(Tile) == 32, "tile layout");

// Dynamic tile scheduler of one kernel family; reset by the last CTA of each launch.
struct Sched {
  unsigned int next, done;
  unsigned int pad[30];
};

// Device-resident freezing state (lives in the caller-bound scratch buffer).
struct DevState {
  int32_t T;         // completed intervals
  int32_t f;         // frozen POOL count (the boundary)
  uint32_t sticky;   // reserved
  int32_t pad;
  unsigned long long epoch;      // peer-exchange epoch: interval ends seen (identical on all ranks)
  unsigned long long tmark[4];   // AF_TIMING builds: %globaltimer at kernel start / tail start / after sums / end
  unsigned long long rs_epoch;   // fused reduce-scatter steps completed (identical on all ranks)
  double prev[AF_MAX_SEGMENTS];  // ||Delta_{T-1,l}||
  unsigned long long dmark[8];   // AF_TIMING builds: %globaltimer at the decision's steps
};

#ifndef AF_ALTERNATE_ORDER  // alternate the streaming kernels' tile order per launch (L2 reuse)
#define AF_ALTERNATE_ORDER 1
#endif
#ifndef AF_FIN_CHUNK  // tiles per finalize chunk (a multiple of the 256 threads)
#define AF_FIN_CHUNK 512
#endif
constexpr int kFinChunk = AF_FIN_CHUNK;
static_assert(kFinChunk % 256 == 0, "finalize chunk: whole loads per thread");
// An empty partial slot: a signalling-NaN bit pattern, which no fp64 arithmetic
// produces (NaN results are quiet), so the store of a tile's partial is its own
// ready flag.  Every slot holds it between launches.
constexpr unsigned long long kPartialEmpty = 0x7FF0DEADBEEF0001ull;

enum Mode : int {
  kAccum = 0, kEndDelta = 1, kStepSq = 2, kAdamAccum = 3, kAdamEnd = 4,
  kRsAccum = 5, kRsEnd = 6, kRsAdamAccum = 7, kRsAdamEnd = 8
};
constexpr int kNumModes = 9;
constexpr int kMaxRsWorld = 8;  // ranks of one fused reduce-scatter (one NVLink domain's GPUs per node)

// AdamW constants of one step, rounded once to fp32 on the host (NEXT 1 fusion).
struct AdamConst {
  float decay;      // 1 - lr * weight_decay
  float beta1, one_minus_beta1;
  float beta2, one_minus_beta2;
  float step_size;  // lr / (1 - beta1^t)
  float sqrt_bc2;   // sqrt(1 - beta2^t)
  float eps;
};

// Arguments of the single-CTA decision kernel.
struct DecideParams {
  const double *ss_all;   // [world][L]
  int32_t world, L, n_pool;
  const int32_t *pool_seg;  // [n_pool] segment index of POOL layer j
  DevState *state;
  af_decision *last;        // device copy of the latest record
  af_decision *ring;        // [kRing]
  af_decision *host;        // mapped page-locked host record or nullptr
  double percentile;
  double pct_q;             // percentile / 100 in fp64 (host-rounded, as numpy forms q)
  int32_t pct_method;
  double tie_rel_eps;
  int32_t min_active;
  int32_t commit;           // 0 under AF_DRY_RUN
};

// Arguments of the streaming kernels (accumulate / interval-end sum of squares).
struct NormParams {
  const void *grad;          // full flat buffer base
  float *delta;              // Delta shard base: element i lives at delta[i - shard_begin]
  int64_t shard_begin;
  const Tile *tiles;
  int32_t n_tiles;                 // host: the largest table (grid and finalize sizing)
  int32_t L;
  const int32_t *first_tile_of_f;  // [n_pool + 1] first active tile for boundary f
  const int32_t *tile_end_of_f;    // [n_pool + 1] end of f's table (n_tiles for static shards)
  const int32_t *seg_tile_begin;   // [L + 1] per table; table f's at + f * stb_stride
  int32_t stb_stride;              // 0: one table (static shards); L + 1: one per f (active-suffix shards)
  const DevState *state;           // reads f
  Sched *sched;
  double *partials;                // [n_tiles] one fp64 partial per tile; kPartialEmpty between launches
  // finalize (fin_worker): chunks of kFinChunk partials, reduced by the CTAs that
  // ran out of tiles, into part2[chunk + segment]; combined in chunk order
  double *part2;                   // [n_tiles / kFinChunk + L + 2]
  Sched *fin_sched;                // next: chunk claims; done: chunks finished
  double *ss_out;                  // [L] this rank's row of the exchange matrix
  double *ss_acc;                  // [L] STEP_SUMSQ accumulator
  int32_t n_pool;
  int32_t first;                   // first step of the interval (Delta not read)
  int32_t end;                     // interval end (STEP_SUMSQ: publish ss_acc)
  int32_t commit;                  // STEP_SUMSQ: store ss_acc
  int32_t fuse_decide;             // fused interval end: the last CTA decides
  int32_t reverse;                 // process the active tiles last to first (alternates per launch)
  // kAdamAccum / kAdamEnd: AdamW update of the same elements (full flat fp32 buffers)
  float *params, *exp_avg, *exp_avg_sq;
  AdamConst adam;
  // NVLink one-shot exchange (peers registered): the CTA finishing the segment sums
  // stores this rank's row into every peer's exchange buffer as LL words (each
  // 8-byte store carries 32 bits of an fp64 sum and the 32-bit epoch, so data and
  // "ready" arrive together and no fence is needed) and polls its own buffer
  // until every peer's words carry the epoch.
  int32_t xworld, xrank;           // xworld == 0: no peer exchange
  unsigned long long *xrows;       // local LL exchange buffers [2][world][L][2]
  unsigned long long *const *peer_rows;  // [world] device pointers to each rank's xrows
  // kRsAccum / kRsEnd (NEXT 1, ZeRO form): the gradient is the rank-order sum of
  // the world's full gradient buffers (read over peer memory) times rs_scale;
  // this rank's shard of it is written to rs_out (optional) and accumulated.
  int32_t rs_world, rs_rank;
  const void *const *rs_grads;     // [rs_world] device pointers (peer-mapped)
  float rs_scale;
  float *rs_out;                   // shard output, element i at rs_out[i - shard_begin]; may be null
  unsigned long long *rs_flags;    // local [2][world]: ready / done epoch reached by each rank
  unsigned long long *const *peer_rs_flags;  // [world] each rank's rs_flags
  DecideParams dec;
  uint32_t dbg_tail_delay_ns;      // AF_DEBUG_TAIL_DELAY_NS: the last CTA waits this long before its tail
  int32_t dbg_peers_arrived;       // AF_DEBUG_PEERS_ARRIVED: the exchange pushes but does not wait
  int32_t dbg_unstaged_tail;       // AF_DEBUG_UNSTAGED_TAIL: the tail never stages the pieces
};

// Flag value a rank stores into its peers' flag slots after it timed out waiting
// for one of them (exchange or reduce-scatter barrier): larger than any epoch, so
// a peer spinning on the slot stops at once and records the timeout too.
constexpr unsigned long long kPoisonEpoch = ~0ull;
constexpr uint32_t kPoisonEpoch32 = 0xFFFFFFFFu;  // the same in the 32-bit epoch of an LL exchange word

// Cache records: one 16-byte meta word per owned id.  Direct mode: `readers`
// counts the chunks of a get that have read {depth, valid}; the last one applies
// the eviction.  Tiered mode: `slot` is the record's storage slot (HBM slots
// first, then page-locked host slots), assigned by the plan kernel.
struct CacheMeta {
  int32_t depth;
  int32_t valid;
  uint32_t readers;
  int32_t slot;
};

// Tiered cache header words (after the sticky error word at offset 0).
struct CacheHeader {
  unsigned int err;       // sticky AF_CACHE_ERR_* flags
  int32_t top;            // free-slot stack height
  unsigned int dropped;   // puts of new ids refused because every slot was taken
  unsigned int pad;
};
static_assert(sizeof(CacheMeta) == 16, "cache meta layout");

struct CacheParams {
  char *payload;            // [capacity][row_bytes]
  CacheMeta *meta;          // [capacity]
  unsigned int *err;        // sticky flags
  const int64_t *ids;
  int32_t n;
  int64_t row_bytes;
  int32_t chunk_bytes;
  int32_t n_chunks;         // chunks per row
  int64_t num_examples;
  int32_t rank, world;
  const char *src_rows;     // put: rows to write
  char *dst_rows;           // get: output rows
  int32_t *depth_out;       // get
  int32_t depth;            // put
  int32_t cur_boundary;     // get
  int32_t no_wait;          // get: skip the PDL dependency wait (AF_CACHE_OVERLAP_PREV, caller-guaranteed)
  unsigned int *retire;     // get with no_wait: CTAs done with their copies (the last one waits)
  // tiered mode (rowslot != nullptr): the plan kernel already resolved each row's slot
  const int32_t *rowslot;   // [n] slot per row of the call, -1 = skip
  char *host;               // device alias of the page-locked host tier
  int64_t hbm_rows;         // slots [0, hbm_rows) in `payload`, then `host`
  char *stage;              // disk tier: device alias of the staging rows (row i of the pass at i)
  int64_t disk_base;        // with stage != nullptr: slots >= disk_base live on disk (staged)
  // global mode (NEXT 4): any id; the owner's (id % world) store is reached through
  // its mapped payload / meta (peer memory over NVLink)
  char *const *peer_payload;     // [world]
  CacheMeta *const *peer_meta;   // [world]
};

// NEXT 4: the cache get fused into the consumer GEMM's operand load (af_gemm.cu).
struct CacheGemmParams {
  CacheMeta *meta;
  unsigned int *err;
  const int64_t *ids;
  int32_t n;                // examples
  int32_t cur_boundary;
  int32_t *depth_out;
  int64_t num_examples;
  int32_t rank, world;
  int32_t n_tiles_m, n_tiles_n;  // rows / 128, ceil(N / 256)
  int32_t rows;             // rows per record (multiple of 128)
  int32_t N, K;
  void *y;                  // bf16 [n * rows][ldy]
  int64_t ldy;
};

struct CachePlanParams {
  CacheMeta *meta;
  CacheHeader *hdr;
  int32_t *free_slots;      // [hbm_rows + host_rows] stack
  int32_t *rowslot;         // [n] out
  const int64_t *ids;
  int32_t n;
  int32_t put;              // 1: put (allocate), 0: get (hit, depth, evict)
  int32_t depth;
  int32_t cur_boundary;
  int32_t *depth_out;
  int64_t num_examples;
  int32_t rank, world;
  int32_t *manifest;        // disk tier: {n, put, disk index per row or -1} (page-locked, mapped)
  int32_t disk_base;
};

#ifndef AF_TIMING
#define AF_TIMING 0
#endif
#ifdef __CUDACC__
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// Programmatic dependent launch: our kernels are launched with programmatic stream
// serialization, so a kernel may be scheduled while its predecessor drains; each
// kernel calls pdl_wait() before touching global memory the predecessor may write
// (a no-op when launched without the attribute).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" :::); }

template <typename K, typename... Args>
inline cudaError_t launch_pdl(K kernel, dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kernel, args...);
  return e != cudaSuccess ? e : cudaGetLastError();
}
#endif

#ifdef __CUDACC__
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per kernel and device --
// not a stream operation, so it stays out of CUDA-graph captures.
template <auto Kernel>
inline cudaError_t ensure_smem_attr(int smem) {
  static unsigned long long done = 0;  // one bit per device ordinal
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 64 && ((done >> dev) & 1ull)) return cudaSuccess;
  e = cudaFuncSetAttribute(Kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e == cudaSuccess && dev < 64) done |= 1ull << dev;
  return e;
}
#endif

// Launchers (defined in the .cu files).  Return cudaError_t as int.
int launch_norms(const NormParams &p, int mode, int grad_dtype, int grid, void *stream);
int launch_decide(const DecideParams &p, void *stream);
int launch_cache_put(const CacheParams &p, int grid, void *stream);
int launch_cache_get(const CacheParams &p, int grid, void *stream);
int launch_cache_plan(const CachePlanParams &p, void *stream);
// tmap_a / tmap_b / tmap_y: CUtensorMap (128 B each) of the store's records, W and y
int launch_cache_gemm(const CacheGemmParams &p, const void *tmap_a, const void *tmap_b, const void *tmap_y,
                      void *stream);
int preload_cache_gemm_kernel();
int norms_max_blocks_per_sm(int mode, int grad_dtype, int world, int *blocks, bool act = false);
// force-load the kernels (lazy module loading must not happen while peers spin)
int preload_norm_kernels(int grad_dtype, int world);
int preload_decide_kernel();
int preload_cache_kernels();
int cache_smem_bytes();

}  // namespace af
