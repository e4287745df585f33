/*
 * af.h -- C ABI of libautofreeze: AutoFreeze's per-iteration freezing hot path
 * (arXiv 2102.01386) on NVIDIA B200 (sm_100a).
 *
 * Citations: P:n = /root/reference/PAPER.md line n (section / equation /
 * algorithm named beside it); S:n = SPEC.md line n; Qn = the readings of
 * SURVEY.md §8(c), restated in DESIGN.md.
 *
 * The path:
 *   af_layer_norms        per step: Delta += g over the active segments (P:196
 *                         §3.1.1 "we accumulate gradients for each layer");
 *                         at the interval end: per-segment sum of squares of
 *                         Delta_T = Delta + g (the norm of Eq. 1), and with
 *                         P > 1 ranks the exchange of the per-segment partials.
 *   af_update_and_decide  Eq. 1, the N-th percentile threshold
 *                         (Alg. 1) and the prefix-only freeze scan
 *                         (Alg. 1), state roll, decision record.
 *   af_cache_put / get    the Storage Manager's write / read of frozen-prefix
 *                         activations keyed by original example id with
 *                         evict-on-read (§3.2), one partition per GPU
 *                         (§3.4 "each GPU manages its own cache").
 *
 * Conventions for every entry point:
 *  - Returns af_status; never prints, throws or aborts.
 *  - Argument / state errors are reported synchronously and ENQUEUE NOTHING.
 *  - Device pointers are owned by the caller (e.g. torch tensors); the library
 *    borrows them for the stream-ordered work it enqueues and never frees them.
 *    The library owns only host metadata and (optionally) an NCCL communicator.
 *  - Work is enqueued on the given cudaStream_t (passed as void*; NULL = legacy
 *    default stream) and is asynchronous unless the entry says "synchronous".
 *    All enqueued work is CUDA-graph capturable (no host syncs, no allocation).
 *  - One af_ctx / af_cache per (process, device); handles are not thread-safe.
 *  - There is no CPU fallback: if no CUDA device is usable, calls that must
 *    touch the device return AF_ECUDA.
 */
#ifndef AF_H_
#define AF_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define AF_API __attribute__((visibility("default")))
#else
#define AF_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  AF_OK = 0,
  AF_EINVAL = 1,      /* bad argument (NULL, misaligned, out of range, bad layout)  */
  AF_ESTATE = 2,      /* call out of order (e.g. decide without an interval end)     */
  AF_EWORKSPACE = 3,  /* workspace / storage not bound                               */
  AF_ECUDA = 4,       /* a CUDA runtime call failed (message: af_last_error)         */
  AF_ENCCL = 5,       /* an NCCL call failed                                         */
  AF_ENONFINITE = 6,  /* reserved: non-finite sums are reported in af_decision.flags */
  AF_EOWNER = 7,      /* reserved: wrong-owner ids are reported by af_cache_status   */
  AF_ERANGE = 8       /* a size does not fit the 64-bit / int32 limits               */
} af_status;

typedef enum { AF_DT_F32 = 0, AF_DT_BF16 = 1 } af_dtype;

/* Segment kinds of the flat gradient buffer, in the order PRE* POOL+ HEAD*.
 * POOL = a transformer block, the paper's "layer" (§2.2); PRE = the
 * embeddings, frozen together with the first block (§4.1, Q11);
 * HEAD = pooler + classifier, never frozen (Q12). */
typedef enum { AF_SEG_PRE = 0, AF_SEG_POOL = 1, AF_SEG_HEAD = 2 } af_seg_kind;

/* What "accumulated gradients Delta" means (Q1).  DELTA is the paper's reading:
 * the elementwise vector sum over the interval, then its L2 norm (P:196, P:632:
 * the 453 MB accumulator is one fp32 copy of the model).  STEP_SUMSQ is the
 * alternative reading sum_t ||g_t||^2 (no Delta buffer). */
typedef enum { AF_ACC_DELTA = 0, AF_ACC_STEP_SUMSQ = 1 } af_acc_mode;

/* Percentile method (Q4): LINEAR = numpy's default "linear" (Hyndman-Fan type 7,
 * numpy's two-branch lerp, bit-identical to numpy.percentile); NEAREST_RANK =
 * the value of ordinal rank ceil(N/100 * n) (S:176 flag). */
typedef enum { AF_PCT_LINEAR = 0, AF_PCT_NEAREST_RANK = 1 } af_pct_method;

#define AF_MAX_SEGMENTS 256
#define AF_MAX_WORLD 64

/* af_layer_norms / af_update_and_decide flags */
#define AF_INTERVAL_END 0x1u /* this step ends the evaluation interval (every k/5 iterations) */
#define AF_DRY_RUN 0x2u      /* do all the work but commit no DECISION state: f, prev, T and the
                                interval's armed/pending flags are unchanged (Delta stays armed, so
                                the next step still reads it).  NOT a no-op on the buffers: a dry
                                accumulate still writes Delta <- Delta + g, and dry AdamW / reduce-
                                scatter variants still update params, moments and grad_shard_out
                                (the bench's stationary reps; the oracle's dry_run matches) */

/* af_decision.flags */
#define AF_DEC_FIRST_INTERVAL 0x1u /* T == 0: norms recorded, no decision (Q9)            */
#define AF_DEC_SKIPPED_FEW 0x2u    /* fewer than min_active active POOL layers (Q10)       */
#define AF_DEC_NEAR_TIE 0x4u       /* a scanned eta within tie_rel_eps*thr of the threshold (Q16) */
#define AF_DEC_NONFINITE 0x8u      /* a sum of squares was Inf/NaN: state unchanged (Q8)          */
#define AF_DEC_DRY_RUN 0x10u       /* produced under AF_DRY_RUN                                    */
#define AF_DEC_EXCHANGE_TIMEOUT 0x20u /* a peer never published its row (sticky): nothing committed  */

#define AF_IPC_HANDLE_BYTES 128

/* af_cache_status device error flags (sticky) */
#define AF_CACHE_ERR_RANGE 0x1u /* an id outside [0, num_examples)               */
#define AF_CACHE_ERR_OWNER 0x2u /* an id with id % world != rank (P:335 partition) */
#define AF_CACHE_ERR_IO 0x4u    /* a disk-tier read or write failed (host callback)  */

typedef struct {
  int32_t n_segments;          /* L, 1..AF_MAX_SEGMENTS                                   */
  const int64_t *seg_offsets;  /* host, L+1 element offsets; [0] = 0, strictly increasing */
  const int32_t *seg_kinds;    /* host, L kinds (af_seg_kind) in the order PRE* POOL+ HEAD* */
  af_dtype grad_dtype;         /* dtype of the flat gradient buffer                       */
} af_layout;

typedef struct {
  double percentile;       /* N of Alg. 1, in (0, 100]; the paper's default is 50 */
  af_pct_method pct_method;
  af_acc_mode acc_mode;
  double tie_rel_eps;      /* near-tie window, e.g. 1e-5 (north_star)                 */
  int32_t min_active;      /* skip the test below this many active POOL layers; >= 1 (default 2) */
  int32_t rank, world;     /* this process's shard of the flat buffer; world in [1, AF_MAX_WORLD] */
  int32_t shard_active;    /* 0: static contiguous shards of [0, n).  1 (world > 1): each boundary f
                              gets its own balanced shards of the ACTIVE suffix [A_f, n) (A_f = start
                              of the first unfrozen segment), so no rank idles as the prefix freezes
                              (SURVEY.md §8(e)); Delta is then a full-size n-element buffer indexed
                              by element.  Valid for af_layer_norms / af_update_and_decide /
                              af_interval_end; the AdamW and reduce-scatter fusions (which own
                              per-shard optimizer state) need static shards (AF_ESTATE). */
} af_config;

/* The decision record of one interval (Alg. 1 output + the quantities that
 * produced it).  Arrays are indexed by segment; entries >= n_segments are 0. */
typedef struct {
  int32_t interval;          /* T of the evaluated interval (0-based, continuous across epochs, Q15) */
  int32_t boundary_before;   /* f: frozen POOL count before the decision                   */
  int32_t boundary_after;    /* f + k (the newly frozen prefix), or f if nothing committed  */
  int32_t n_active;          /* active POOL layers considered (P:174 activeLayers)          */
  double threshold;          /* N-th percentile of eta over the active POOL (NaN if none)  */
  uint32_t flags;            /* AF_DEC_*                                                   */
  int32_t near_tie_seg;      /* first segment flagged NEAR_TIE, or -1                       */
  double sumsq[AF_MAX_SEGMENTS]; /* ||Delta_T,l||^2 (0 for frozen segments)                 */
  double norm[AF_MAX_SEGMENTS];  /* ||Delta_T,l||                                          */
  double eta[AF_MAX_SEGMENTS];   /* Eq. 1 per segment, 0 where the previous norm is 0      */
} af_decision;

/* Host-side description of a created context (no device access). */
typedef struct {
  int32_t n_segments, n_pool, rank, world;
  int64_t n_total;                  /* elements of the full flat buffer                  */
  int64_t shard_begin, shard_end;   /* this rank's element range at f = 0 (multiples of 8 except n;
                                       af_ctx_shard_of for other f)  */
  int32_t n_tiles;                  /* segment-aligned tiles of the shard (interval-end kernels;
                                       active-suffix shards: the largest per-f table) */
  int32_t tile_elems;               /* their nominal size in elements                    */
  int32_t first_tile_of_pool[AF_MAX_SEGMENTS + 1]; /* first active tile when f = j frozen (index
                                       into the concatenated per-f tables when shard_active) */
  int32_t n_tiles_acc;              /* tiles of the accumulate kernel (finer, no partials) */
  int32_t tile_elems_acc;
  int32_t n_fin_ctas;               /* 0: no second launch (the finalize runs inside the
                                       streaming kernel; kept for layout compatibility) */
  int32_t n_fin_chunks;             /* chunks of 256 tiles in which the streaming grid's CTAs
                                       reduce the interval end's per-tile partials */
} af_info;

typedef struct af_ctx af_ctx;
typedef struct af_cache af_cache;

/* ---- freezing module ------------------------------------------------------ */

/* Host only (no device access).  Validates and copies the layout (offsets
 * strictly increasing from 0, kinds in the order PRE* POOL+ HEAD* with >= 1
 * POOL), the config, builds the segment-aligned tile table of this rank's
 * contiguous shard [floor(r*n/P) rounded down to 8, ...) --
 * or, with shard_active, one table per boundary f over this rank's slice of
 * the active suffix [A_f, n) (A_f + floor(r*(n-A_f)/P), rounded down to 8).
 * AF_EINVAL on any violation; *out untouched on error. */
AF_API af_status af_ctx_create(const af_layout *layout, const af_config *cfg, af_ctx **out);

/* Host only.  Bytes of the two caller-owned device buffers:
 * accum = the fp32 Delta shard (n_local * 4 B; n * 4 B with shard_active, where
 *         element i lives at accum[i]; 0 in STEP_SUMSQ mode);
 * scratch = device state, tile table, partials, exchange rows, decision ring. */
AF_API af_status af_ctx_workspace_bytes(const af_ctx *ctx, size_t *accum_bytes, size_t *scratch_bytes);

/* Host only.  Fills *info. */
AF_API af_status af_ctx_info(const af_ctx *ctx, af_info *info);

/* Host only.  This rank's element range [*begin, *end) when f POOL blocks are
 * frozen (0 <= f <= n_pool): the static shard for every f, or the active-suffix
 * shard (af_config.shard_active).  AF_EINVAL for f out of range. */
AF_API af_status af_ctx_shard_of(const af_ctx *ctx, int32_t f, int64_t *begin, int64_t *end);

/* Synchronous.  Binds caller-allocated device buffers (256-byte aligned, sizes
 * from af_ctx_workspace_bytes, on the current device) and initialises the
 * device state (T = 0, f = 0).  accum may be NULL iff accum_bytes == 0. */
AF_API af_status af_ctx_bind(af_ctx *ctx, void *accum_dev, void *scratch_dev);

/* Synchronous, collective over all `world` ranks.  Creates the library's NCCL
 * communicator from a 128-byte ncclUniqueId produced by af_nccl_unique_id on
 * rank 0 and broadcast by the caller (e.g. torch.distributed).  Without a
 * communicator a world > 1 context runs in "external exchange" mode: the caller
 * fills the other ranks' rows of af_ctx_exchange_rows before deciding. */
AF_API af_status af_nccl_unique_id(void *id_128B);
AF_API af_status af_ctx_set_comm(af_ctx *ctx, const void *nccl_unique_id_128B);

/* Device pointer of the exchange matrix ss_all[world][n_segments] (fp64, row r
 * = rank r's per-segment partial sums) inside the bound scratch. */
AF_API af_status af_ctx_exchange_rows(af_ctx *ctx, double **ss_all_dev);

/* NVLink one-shot exchange, replacing the all-gather:
 * every rank registers every rank's exchange buffers (double-buffered rows +
 * epoch flags inside the scratch).  Then at each interval end the CTA that
 * finishes the per-segment sums writes this rank's L partials straight into
 * every peer's memory over NVLink (P2P stores), publishes its epoch in every
 * peer's flag slot (st.release.sys) and waits for all ranks' epochs
 * (ld.acquire.sys, bounded spin: a missing peer sets AF_DEC_EXCHANGE_TIMEOUT
 * instead of hanging) -- af_interval_end needs no collective launch at any
 * world size (one streaming kernel; its CTAs also reduce the partials).
 * A timeout is FATAL for the job: the rank that timed out poisons its flag slot
 * in every peer, so a peer that arrives later flags EXCHANGE_TIMEOUT too instead
 * of committing alone (best effort: a peer that had already read the rank's
 * epoch before the poison commits), the flag is sticky (only af_set_state clears
 * it) and every later streaming launch of the context skips its peer loads and
 * stores.  The caller must stop on every rank and restore from a checkpoint.
 * _ipc: synchronous, collective; `handles` = world x AF_IPC_HANDLE_BYTES in rank
 * order, each from af_ctx_exchange_ipc_handle on that rank (exchanged by the
 * caller, e.g. torch.distributed.all_gather_object).  _local: every rank's ctx
 * lives in this process (several ranks sharing one GPU, or one process driving
 * several GPUs: for a peer bound on another device, peer access from the current
 * device is enabled here -- AF_EINVAL if cudaDeviceCanAccessPeer says no).
 * Takes precedence over an NCCL communicator. */
AF_API af_status af_ctx_exchange_ipc_handle(af_ctx *ctx, void *handle_out);
AF_API af_status af_ctx_set_peers_ipc(af_ctx *ctx, const void *handles);
AF_API af_status af_ctx_set_peers_local(af_ctx *ctx, af_ctx *const *peers);
/* Host only: stop using the registered peers (e.g. when another rank failed to
 * map them and the ranks agree to fall back to NCCL). */
AF_API af_status af_ctx_clear_peers(af_ctx *ctx);

/* One training step.  grad_dev = the FULL flat gradient
 * buffer (n_total elements of grad_dtype, 16-byte aligned; only this rank's
 * shard is read).  Frozen segments (PRE and POOL[0..f) once f >= 1, read from
 * device state) are skipped.  Without AF_INTERVAL_END: Delta <- Delta + g
 * (Delta <- g on the first step of an interval).  With AF_INTERVAL_END: the
 * per-segment fp64 sums of squares of Delta_T = Delta + g are formed (Delta is
 * not written back: the next interval restarts it), then (world > 1 with a
 * communicator) all-gathered.  AF_DRY_RUN: the next step still sees Delta armed. */
AF_API af_status af_layer_norms(af_ctx *ctx, const void *grad_dev, uint32_t flags, void *stream);

/* Eq. 1, threshold, prefix scan and state roll on the gathered sums (a5-a9).
 * AF_ESTATE unless an AF_INTERVAL_END af_layer_norms precedes it.  With
 * out_host != NULL (page-locked host memory, e.g. torch pin_memory) the record
 * is copied there asynchronously; it is valid once the stream reaches this
 * point.  AF_DRY_RUN: everything is computed and recorded, nothing committed. */
AF_API af_status af_update_and_decide(af_ctx *ctx, uint32_t flags, af_decision *out_host, void *stream);

/* Fused interval end: exactly af_layer_norms(AF_INTERVAL_END |
 * flags) followed by af_update_and_decide(flags), same results and state.  With
 * world == 1 or peers registered, no host involvement and ONE kernel launch: the
 * streaming kernel's CTAs reduce the per-tile partials as they run out of tiles,
 * and the CTA finishing the last chunk sums the segments, exchanges rows with the
 * peers and runs the decision.  With world > 1 and only a communicator: kernel, NCCL
 * all-gather, decide kernel.  flags: AF_DRY_RUN only. */
AF_API af_status af_interval_end(af_ctx *ctx, const void *grad_dev, uint32_t flags, af_decision *out_host,
                                 void *stream);

/* AdamW hyper-parameters of one optimizer step (step = t >= 1 for the bias corrections). */
typedef struct {
  float lr, beta1, beta2, eps, weight_decay;
  int32_t step;
} af_adamw;

/* the Delta accumulate fused into the optimizer that
 * already reads g.  One pass over this rank's shard of the active segments:
 * AdamW (decoupled weight decay; fp32, round-to-nearest, in the order
 *   p <- p*(1-lr*wd); m <- m*b1 + g*(1-b1); v <- v*b2 + (g*g)*(1-b2);
 *   p <- p - (lr/(1-b1^t)) * (m / (sqrt(v)/sqrt(1-b2^t) + eps)) )
 * on params/exp_avg/exp_avg_sq (FULL flat fp32 buffers, n_total elements, 16-byte
 * aligned; frozen segments are not touched -- requires_grad=False), and either
 * Delta += g (flags = 0) or, with AF_INTERVAL_END, the interval end of
 * af_interval_end (sums of squares of Delta + g, exchange, decision, record) in
 * the same kernel.  Saves the separate read of g per step (s_g bytes per element).
 * With world > 1 the caller all-gathers the updated parameter shards (ZeRO-1). */
AF_API af_status af_adamw_step(af_ctx *ctx, float *params_dev, float *exp_avg_dev, float *exp_avg_sq_dev,
                               const void *grad_dev, const af_adamw *hp, uint32_t flags, af_decision *out_host,
                               void *stream);

/* Host only: cap the CTAs of the streaming kernels (0 = the persistent grid of
 * occupancy x SMs).  For sharing the GPU with concurrent work, e.g. the ranks of
 * a fused reduce-scatter tested on one GPU, whose kernels must be co-resident. */
AF_API af_status af_ctx_set_max_ctas(af_ctx *ctx, int32_t max_ctas);

/* SURVEY.md §8(f) NEXT 1, ZeRO form: the data-parallel gradient sync fused with
 * the accumulate it feeds (PAPER.md P:44, P:288-290 -- DDP's gradient all-reduce,
 * whose per-layer volume freezing removes; P:335 -- the test runs on the
 * synchronised gradient).  Every rank registers its FULL flat gradient buffer
 * (n_total elements of grad_dtype, 16-byte aligned, persistent: a DDP-style
 * bucket); then one kernel per step and rank reads its shard [shard_begin,
 * shard_end) of all `world` buffers over peer memory, and for each active
 * element i
 *     gs_i = fl( (..(g_0,i + g_1,i) + ..) + g_P-1,i ) * scale )   fp32, rank order
 * writes gs_i to grad_shard_out_dev[i - shard_begin] (fp32, optional, 16-byte
 * aligned; frozen segments untouched) and accumulates it exactly as af_layer_norms
 * accumulates g (Delta += gs; AF_INTERVAL_END: the sums of squares of Delta + gs,
 * peer exchange and decision as in af_interval_end).  scale = 1/world gives DDP's
 * average.  The kernel opens with a cross-GPU epoch barrier (every rank's
 * gradient is complete) and closes with another (no rank still reads this
 * rank's buffer), so the caller may overwrite its gradient as soon as the stream
 * passes the call.  A rank that never arrives (~seconds) sets a sticky flag: the
 * next decision carries AF_DEC_EXCHANGE_TIMEOUT and is not committed.
 * Requirements: acc_mode AF_ACC_DELTA, world <= 8, and with world > 1 the peers
 * registered (af_ctx_set_peers_*: the barrier flags live in the scratch).
 * Registration: af_ctx_grad_ipc_handle on every rank, all-gather the
 * AF_IPC_HANDLE_BYTES handles, af_ctx_set_grad_peers_ipc (collective); or, for
 * ranks in one process, af_ctx_set_grad_peers_local(grads_dev[world]).  Errors:
 * AF_ESTATE (nothing registered / no peers / STEP_SUMSQ), AF_EINVAL (bad
 * handle, alignment, non-finite scale, unknown flags). */
AF_API af_status af_ctx_grad_ipc_handle(af_ctx *ctx, const void *grad_dev, void *handle_out);
AF_API af_status af_ctx_set_grad_peers_ipc(af_ctx *ctx, const void *handles);
AF_API af_status af_ctx_set_grad_peers_local(af_ctx *ctx, const void *const *grads_dev);
AF_API af_status af_reduce_scatter_step(af_ctx *ctx, float scale, float *grad_shard_out_dev, uint32_t flags,
                                        af_decision *out_host, void *stream);

/* af_reduce_scatter_step with the optimizer of the same shard fused in (ZeRO:
 * each rank owns its shard's AdamW state): for every active element i of the
 * shard, gs_i as above, then AdamW with gs_i exactly as af_adamw_step (same
 * constants, same fp32 operation order) on params/exp_avg/exp_avg_sq (FULL
 * flat fp32 buffers indexed by i, 16-byte aligned; only the shard's active
 * elements are touched), and the Delta accumulate / interval end with gs_i.
 * grad_shard_out_dev may be NULL.  The caller all-gathers the updated
 * parameter shards.  Errors as af_reduce_scatter_step and af_adamw_step. */
AF_API af_status af_reduce_scatter_adamw_step(af_ctx *ctx, float scale, float *params_dev, float *exp_avg_dev,
                                              float *exp_avg_sq_dev, const af_adamw *hp, float *grad_shard_out_dev,
                                              uint32_t flags, af_decision *out_host, void *stream);

/* Synchronous.  Serialise / restore {T, f, prev norms, Delta-armed flag}
 * (checkpoint at interval boundaries is exact).  With buf == NULL, get_state
 * stores the required size in *len. */
AF_API af_status af_get_state(af_ctx *ctx, void *buf, size_t *len);
AF_API af_status af_set_state(af_ctx *ctx, const void *buf, size_t len);

/* Synchronous.  Copies the device ring's decision record of interval T (the
 * ring keeps the last 16 intervals, T = af_decision.interval) into *out.
 * AF_ERANGE when interval T is not in the ring (overwritten or not yet decided).
 * For callers that enqueue several intervals without reading each record. */
AF_API af_status af_ctx_read_record(af_ctx *ctx, int32_t interval, af_decision *out);

/* Host only: test / diagnostic knobs (not for production).
 * AF_DEBUG_TAIL_DELAY_NS: the last CTA of every later interval-end launch of
 * this ctx busy-waits `value` ns (0 = off, <= 1e9) before summing and deciding,
 * widening the window in which later kernels could observe an uncommitted
 * decision (ordering tests). */
#define AF_DEBUG_TAIL_DELAY_NS 1
/* AF_DEBUG_PEERS_ARRIVED (0/1): with peers registered, the interval end pushes
 * its row to every peer and reads every peer's words once without waiting for
 * the epoch -- times ONE rank's interval end on a single GPU (the other ranks'
 * contexts registered locally, never launched).  The decision then uses
 * whatever rows the peers' buffers hold. */
#define AF_DEBUG_PEERS_ARRIVED 2
/* AF_DEBUG_UNSTAGED_TAIL (0/1): the interval end's tail takes the path of tables
 * whose finalize pieces do not fit shared memory (chunks + segments > the
 * finalize chunk; > 10^9 fp32 elements otherwise) at any size -- parity tests of
 * that path. */
#define AF_DEBUG_UNSTAGED_TAIL 3
/* AF_DEBUG_FORCE_NCCL (0/1): with a communicator set (af_ctx_set_comm) and no
 * peers, interval ends take the world > 1 route -- streaming kernel, then
 * ncclAllGather of the per-segment rows, then the decide kernel -- even at
 * world == 1: runs the NCCL fallback's calls on a single GPU. */
#define AF_DEBUG_FORCE_NCCL 4
AF_API af_status af_ctx_set_debug(af_ctx *ctx, int32_t key, int64_t value);

AF_API af_status af_ctx_destroy(af_ctx *ctx);

/* ---- storage manager (activation cache) ----------------------------------- */

/* Host only.  A direct-mapped HBM cache of this rank's ids {id : id % world ==
 * rank, 0 <= id < num_examples}, slot = id / world, rows of row_bytes (a
 * positive multiple of 16). */
AF_API af_status af_cache_create(int64_t num_examples, int64_t row_bytes, int32_t rank, int32_t world,
                          af_cache **out);
AF_API af_status af_cache_storage_bytes(const af_cache *c, size_t *payload_bytes, size_t *meta_bytes);
/* Synchronous: binds caller-owned device storage and clears every record. */
AF_API af_status af_cache_bind(af_cache *c, void *payload_dev, void *meta_dev);

/* Write n rows (rows_dev: n x row_bytes, 16-byte aligned) for the unique
 * original ids ids_dev[0..n) (int64, device) at depth >= 1 = the frozen POOL
 * count whose output the rows hold ("the output of the forward pass up
 * to layer L is written to cache").  Ids outside this rank's partition set a
 * sticky error flag and are skipped. */
AF_API af_status af_cache_put(af_cache *c, const int64_t *ids_dev, int32_t n, const void *rows_dev,
                       int32_t depth, void *stream);

/* Read n unique ids: for a valid record copy it to rows_out_dev[i] and set
 * depth_out_dev[i] = its depth, then evict it if depth < cur_boundary (P:276:
 * the frozen count grew since it was written); otherwise depth_out_dev[i] = -1
 * and rows_out_dev[i] is untouched. */
AF_API af_status af_cache_get(af_cache *c, const int64_t *ids_dev, int32_t n, int32_t cur_boundary,
                       void *rows_out_dev, int32_t *depth_out_dev, void *stream);

/* af_cache_get with flags.  AF_CACHE_OVERLAP_PREV: the copy may start while the
 * kernel just before it on `stream` is still finishing (programmatic dependent
 * launch without the dependency wait) -- e.g. behind af_interval_end, whose last
 * CTA sums and decides while the grid is otherwise idle.  The CALLER guarantees
 * that this preceding kernel does not write ids, the store (no af_cache_put /
 * get on the same cache) or rows_out / depth_out, and does not read rows_out /
 * depth_out; every kernel before it has completed.  Stream order is otherwise
 * kept: the get does not COMPLETE before the preceding kernel has completed (it
 * waits for it after its copies), so every later kernel on the stream still
 * sees the preceding kernel's writes (e.g. the committed boundary f).
 * Direct-mapped stores only (AF_ESTATE for tiered or global).  Unknown flags:
 * AF_EINVAL. */
#define AF_CACHE_OVERLAP_PREV 0x1u
AF_API af_status af_cache_get_ex(af_cache *c, const int64_t *ids_dev, int32_t n, int32_t cur_boundary,
                                 void *rows_out_dev, int32_t *depth_out_dev, uint32_t flags, void *stream);

/* Storage-manager tiers and admission (§3.2).
 * Host only, before af_cache_storage_bytes / af_cache_bind: room for I =
 * hbm_rows + host_rows records (I may be < D = the rank's owned ids): hbm_rows in
 * the HBM payload, host_rows in a page-locked, device-mapped host tier (the
 * paper's spill to CPU memory / disk).  Records are allocated from a free list on
 * put (HBM slots first); a put of a NEW id when every slot is taken is dropped,
 * in call order (drop-newest) -- the store never exceeds I; rewriting an
 * existing id reuses its slot; an evict-on-read returns the slot (the paper's
 * re-cache balance).  Each call is planned by a one-CTA kernel (block scans in
 * call order, deterministic), then copied by the TMA kernel.  Without this call
 * the cache is direct-mapped with room for every owned id. */
AF_API af_status af_cache_set_capacity(af_cache *c, int64_t hbm_rows, int64_t host_rows);  /* >= 0 each; the
                       store needs >= 1 slot in all (a disk tier may provide them): AF_EINVAL at bind */
AF_API af_status af_cache_host_bytes(const af_cache *c, size_t *host_bytes);
/* Synchronous: binds the caller-owned page-locked host tier (cudaHostAlloc /
 * torch pin_memory: device-mapped under UVA), 16-byte aligned. */
AF_API af_status af_cache_bind_host(af_cache *c, void *host_pinned);

/* Disk tier (§3.2: "We store the intermediate output to disk when it no
 * longer fits in CPU memory"; reader and writer processes).  Host only,
 * after af_cache_set_capacity and before af_cache_bind: disk_rows more record
 * slots, [hbm_rows + host_rows, I), as rows of the file at `path` (created or
 * truncated, sized disk_rows x row_bytes; the library closes but never deletes
 * it).  Slots are handed out HBM first, then host, then disk.  Rows routed to the
 * disk by a call's plan kernel move through a caller-owned page-locked staging
 * area (af_cache_disk_stage_bytes; bound with af_cache_bind_disk_stage) of
 * stage_rows rows, by stream-ordered host callbacks (cudaLaunchHostFunc: the
 * reader pread()s before the copy kernel of a get, the writer pwrite()s after
 * the copy kernel of a put); calls are split into passes of stage_rows rows.
 * All calls on one disk-tier cache must be issued on one stream (the callbacks
 * take their work list from the staging area).  An I/O error sets the sticky
 * AF_CACHE_ERR_IO.  Without GPUDirect Storage (not in this build) the disk is
 * reached through host memory. */
AF_API af_status af_cache_set_disk_tier(af_cache *c, int64_t disk_rows, int32_t stage_rows, const char *path);
AF_API af_status af_cache_disk_stage_bytes(const af_cache *c, size_t *stage_bytes);
AF_API af_status af_cache_bind_disk_stage(af_cache *c, void *stage_pinned);

/* cross-GPU cache get / put for samplers that are not
 * rank-affine.  Every rank registers every rank's direct-mapped store (CUDA IPC
 * of payload + meta, handles exchanged by the caller; or contexts of one
 * process); then *_global accept ANY id in [0, num_examples): the owner rank
 * (id % world) store is read / written through its mapped memory -- TMA bulk
 * copies and meta updates over NVLink peer memory, evict-on-read included (the
 * reader count is a peer atomic).  The paper keeps caches per GPU to avoid data
 * movement; this removes the need for a rank-affine sampler. */
#define AF_CACHE_IPC_HANDLE_BYTES 256
AF_API af_status af_cache_exchange_ipc_handle(af_cache *c, void *handle_out);
AF_API af_status af_cache_set_peers_ipc(af_cache *c, const void *handles);
AF_API af_status af_cache_set_peers_local(af_cache *c, af_cache *const *peers);
/* NEXT 4, second half: the cache get fused into the first active layer's GEMM
 * operand load.  For each of the n examples: if its record is valid (a hit),
 *   y[i * rows_per_record + r][j] = bf16_rne( sum_k rec_i[r][k] * w[j][k] )
 * (fp32 accumulation on the tensor cores, tcgen05), i.e. y = x W^T with x the
 * cached layer output (rows_per_record x K bf16 per record; row_bytes must be
 * rows_per_record x K x 2) and W a bf16 [N][K] weight (a torch Linear weight,
 * 16-byte aligned); depth_out[i] = the record's depth, and the record is evicted
 * once read if depth < cur_boundary -- the semantics of af_cache_get, without
 * the batch copy: the GEMM's TMA loads read the record straight out of the
 * store.  A miss leaves y's rows untouched and sets depth_out[i] = -1 (the
 * caller runs the frozen prefix for those examples).  y: bf16 [n x
 * rows_per_record][N] row-major, 16-byte aligned.  Requirements: direct-mapped
 * store without peers (AF_ESTATE), rows_per_record a multiple of 128, K of 64,
 * N of 32 (AF_EINVAL).  Ids unique (as af_cache_get). */
AF_API af_status af_cache_get_gemm(af_cache *c, const int64_t *ids_dev, int32_t n, int32_t cur_boundary,
                                   int32_t rows_per_record, int32_t K, const void *w_dev, int32_t N, void *y_dev,
                                   int32_t *depth_out_dev, void *stream);
AF_API af_status af_cache_put_global(af_cache *c, const int64_t *ids_dev, int32_t n, const void *rows_dev,
                                     int32_t depth, void *stream);
AF_API af_status af_cache_get_global(af_cache *c, const int64_t *ids_dev, int32_t n, int32_t cur_boundary,
                                     void *rows_out_dev, int32_t *depth_out_dev, void *stream);

typedef struct {
  uint32_t error_flags;      /* sticky AF_CACHE_ERR_* */
  uint32_t pad;
  int64_t partition;         /* D: ids owned by this rank */
  int64_t capacity;          /* I: record slots (== D when direct-mapped) */
  int64_t n_valid, n_hbm, n_host;
  int64_t n_dropped;         /* puts refused for lack of room (tiered) */
  int64_t free_slots;
  int64_t n_disk;            /* valid records in the disk tier */
} af_cache_info;
/* Synchronous: counters of the store. */
AF_API af_status af_cache_stats(af_cache *c, af_cache_info *out);

/* Synchronous: sticky AF_CACHE_ERR_* flags and the count of valid records. */
AF_API af_status af_cache_status(af_cache *c, uint32_t *device_error_flags, int64_t *n_valid);
AF_API af_status af_cache_destroy(af_cache *c);

/* Cache-vs-recompute rule (§3.2): 1 iff frozen_layers *
 * t_layer_fwd_s > t_batch_read_s, else 0 (also 0 for negative inputs). */
AF_API int af_should_cache(int32_t frozen_layers, double t_layer_fwd_s, double t_batch_read_s);

AF_API const char *af_status_str(af_status s);
/* Thread-local text of the last AF_ECUDA / AF_ENCCL / AF_EINVAL cause. */
AF_API const char *af_last_error(void);
/* Library version, e.g. "0.1.0". */
AF_API const char *af_version(void);

#ifdef __cplusplus
}
#endif
#endif /* AF_H_ */
