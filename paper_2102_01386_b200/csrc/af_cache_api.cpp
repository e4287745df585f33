// af_cache_api.cpp -- the storage manager's C-ABI entry points (af_cache_*):
// direct-mapped and tiered stores, admission, statistics, peer (global) access.
#include <cuda.h>
#include <fcntl.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <cerrno>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "af_host.h"

using namespace af;

struct af_cache {
  int64_t num_examples = 0, row_bytes = 0;
  int64_t capacity = 0;  // owned ids of this rank (the partition size D_local)
  int32_t rank = 0, world = 1;
  // tiered mode (af_cache_set_capacity): I = hbm_rows + host_rows (+ disk_rows) slots
  bool tiered = false;
  int64_t hbm_rows = 0, host_rows = 0;
  // disk tier (af_cache_set_disk_tier): slots [hbm + host, I) are rows of a file,
  // moved through a page-locked staging area by stream-ordered host callbacks
  int64_t disk_rows = 0;
  int fd = -1;
  std::string disk_path;
  int32_t stage_rows = 0;            // rows per plan pass when a disk tier exists
  char *stage_host = nullptr;        // caller's page-locked staging: [manifest | rows]
  char *stage_dev = nullptr;         // its device alias
  bool disk_bound = false;
  std::atomic<unsigned int> disk_err{0};  // AF_CACHE_ERR_IO from the host callbacks
  int64_t slots() const { return hbm_rows + host_rows + disk_rows; }
  size_t manifest_bytes() const { return (static_cast<size_t>(stage_rows) + 2) * 4 + 255 & ~size_t(255); }
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
    if (tiered) b += static_cast<size_t>(slots()) * 4 + static_cast<size_t>(max_batch) * 4;
    return (b + 255) / 256 * 256;
  }
  size_t meta_bytes() const { return o_peer_table() + 2 * AF_MAX_WORLD * sizeof(void *); }
  size_t o_free() const { return kMetaHeaderBytes + static_cast<size_t>(capacity) * sizeof(CacheMeta); }
  size_t o_rowslot() const { return o_free() + static_cast<size_t>(slots()) * 4; }
  static constexpr size_t kMetaHeaderBytes = 256;
};

static constexpr size_t kMetaHeader = af_cache::kMetaHeaderBytes;

extern "C" {


af_status af_cache_create(int64_t num_examples, int64_t row_bytes, int32_t rank, int32_t world, af_cache **out) {
  AF_NVTX();
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
  AF_NVTX();
  if (!c) return fail(AF_EINVAL, "NULL cache");
  if (c->bound) return fail(AF_ESTATE, "set the capacity before binding storage");
  if (hbm_rows < 0 || host_rows < 0) return fail(AF_EINVAL, "bad capacity");  // >= 1 slot in all: at bind
  if (hbm_rows + host_rows > (int64_t(1) << 31) - 1) return fail(AF_ERANGE, "capacity too large");
  c->tiered = true;
  c->hbm_rows = hbm_rows;
  c->host_rows = host_rows;
  return AF_OK;
}

af_status af_cache_set_disk_tier(af_cache *c, int64_t disk_rows, int32_t stage_rows, const char *path) {
  AF_NVTX();
  if (!c || !path) return fail(AF_EINVAL, "NULL argument");
  if (c->bound) return fail(AF_ESTATE, "set the disk tier before binding storage");
  if (!c->tiered) return fail(AF_ESTATE, "the disk tier extends a tiered store (af_cache_set_capacity first)");
  if (c->fd >= 0) return fail(AF_ESTATE, "disk tier already set");
  if (disk_rows < 1 || stage_rows < 1 || stage_rows > 65536) return fail(AF_EINVAL, "bad disk_rows / stage_rows");
  if (c->hbm_rows + c->host_rows + disk_rows > (int64_t(1) << 31) - 1) return fail(AF_ERANGE, "capacity too large");
  const int fd = ::open(path, O_RDWR | O_CREAT | O_TRUNC | O_CLOEXEC, 0600);
  if (fd < 0) return fail(AF_EINVAL, "cannot open the disk-tier file");
  if (::ftruncate(fd, static_cast<off_t>(disk_rows) * c->row_bytes) != 0) {
    ::close(fd);
    return fail(AF_ERANGE, "cannot size the disk-tier file");
  }
  c->fd = fd;
  c->disk_path = path;
  c->disk_rows = disk_rows;
  c->stage_rows = stage_rows;
  c->max_batch = stage_rows;  // a plan pass stages at most this many rows
  return AF_OK;
}

af_status af_cache_disk_stage_bytes(const af_cache *c, size_t *stage_bytes) {
  AF_NVTX();
  if (!c || !stage_bytes) return fail(AF_EINVAL, "NULL argument");
  *stage_bytes = c->fd >= 0 ? c->manifest_bytes() + static_cast<size_t>(c->stage_rows) * c->row_bytes : 0;
  return AF_OK;
}

af_status af_cache_bind_disk_stage(af_cache *c, void *stage_pinned) {
  AF_NVTX();
  if (!c || !stage_pinned) return fail(AF_EINVAL, "NULL argument");
  if (c->fd < 0) return fail(AF_ESTATE, "no disk tier configured");
  if (!aligned(stage_pinned, 256)) return fail(AF_EINVAL, "staging must be 256-byte aligned");
  cudaPointerAttributes a{};
  cudaError_t e = cudaPointerGetAttributes(&a, stage_pinned);
  if (e != cudaSuccess || a.type != cudaMemoryTypeHost || !a.devicePointer) {
    cudaGetLastError();
    return fail(AF_EINVAL, "staging must be page-locked, device-mapped memory (cudaHostAlloc / pin_memory)");
  }
  c->stage_host = static_cast<char *>(stage_pinned);
  c->stage_dev = static_cast<char *>(a.devicePointer);
  c->disk_bound = true;
  return AF_OK;
}

af_status af_cache_storage_bytes(const af_cache *c, size_t *payload_bytes, size_t *meta_bytes) {
  AF_NVTX();
  if (!c || !payload_bytes || !meta_bytes) return fail(AF_EINVAL, "NULL argument");
  const int64_t rows = c->tiered ? c->hbm_rows : c->capacity;
  *payload_bytes = static_cast<size_t>(rows) * static_cast<size_t>(c->row_bytes);
  *meta_bytes = c->meta_bytes();
  return AF_OK;
}

af_status af_cache_host_bytes(const af_cache *c, size_t *host_bytes) {
  AF_NVTX();
  if (!c || !host_bytes) return fail(AF_EINVAL, "NULL argument");
  *host_bytes = static_cast<size_t>(c->tiered ? c->host_rows : 0) * static_cast<size_t>(c->row_bytes);
  return AF_OK;
}

af_status af_cache_bind_host(af_cache *c, void *host_pinned) {
  AF_NVTX();
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
  AF_NVTX();
  const int64_t rows = c ? (c->tiered ? c->hbm_rows : c->capacity) : 0;
  if (!c || !meta_dev || (rows > 0 && !payload_dev)) return fail(AF_EINVAL, "NULL argument");
  if ((payload_dev && !aligned(payload_dev, 16)) || !aligned(meta_dev, 256))
    return fail(AF_EINVAL, "payload must be 16-byte and meta 256-byte aligned");
  if (c->tiered && c->slots() < 1) return fail(AF_EINVAL, "a tiered store needs at least one record slot");
  int sms = 0;
  cudaError_t e = static_cast<cudaError_t>(device_sm_count(&sms));
  if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceGetAttribute");
  c->grid = std::max(1, sms);
  e = static_cast<cudaError_t>(preload_cache_kernels());
  if (e == cudaSuccess) e = static_cast<cudaError_t>(preload_cache_gemm_kernel());
  if (e != cudaSuccess) return cuda_fail(e, "cudaFuncGetAttributes (kernel preload)");
  c->payload = static_cast<char *>(payload_dev);
  c->meta = static_cast<char *>(meta_dev);
  AF_CUDA(cudaMemset(c->meta, 0, c->meta_bytes()), "cudaMemset(meta)");
  if (c->tiered) {
    // every record slot free: the stack pops slot 0 first (HBM, then host, then disk)
    const int32_t I = static_cast<int32_t>(c->slots());
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
  p.retire = reinterpret_cast<unsigned int *>(c->meta + 64);  // header word (CacheHeader is 16 B of 256)
  p.ids = ids;
  p.n = n;
  p.row_bytes = c->row_bytes;
  p.num_examples = c->num_examples;
  p.rank = c->rank;
  p.world = c->world;
  return AF_OK;
}

// The disk tier's reader / writer (the paper's reader and writer processes,
// P:259): a stream-ordered host callback that moves the rows the plan kernel
// routed to disk slots between the file and the page-locked staging area.  The
// plan kernel wrote the manifest {n, put, disk index per row (-1: not on disk)}
// into the staging area, so the callback needs no per-call arguments (calls of
// one cache are issued on one stream: the next plan runs after this callback).
static void CUDART_CB disk_io(void *user) {
  af_cache *c = static_cast<af_cache *>(user);
  const volatile int32_t *man = reinterpret_cast<const volatile int32_t *>(c->stage_host);
  const int32_t n = man[0], put = man[1];
  char *rows = c->stage_host + c->manifest_bytes();
  for (int32_t i = 0; i < n && i < c->stage_rows; ++i) {
    const int32_t d = man[2 + i];
    if (d < 0) continue;
    char *buf = rows + static_cast<size_t>(i) * c->row_bytes;
    off_t off = static_cast<off_t>(d) * c->row_bytes;
    size_t left = static_cast<size_t>(c->row_bytes);
    while (left > 0) {
      const ssize_t k = put ? ::pwrite(c->fd, buf, left, off) : ::pread(c->fd, buf, left, off);
      if (k < 0 && errno == EINTR) continue;
      if (k <= 0) {
        c->disk_err.fetch_or(AF_CACHE_ERR_IO);
        break;
      }
      buf += k;
      off += k;
      left -= static_cast<size_t>(k);
    }
  }
}

static af_status cache_tiered(af_cache *c, CacheParams &p, bool put, void *stream) {
  if (c->host_rows > 0 && !c->host_bound) return fail(AF_EWORKSPACE, "host tier not bound (af_cache_bind_host)");
  if (c->fd >= 0 && !c->disk_bound) return fail(AF_EWORKSPACE, "disk staging not bound (af_cache_bind_disk_stage)");
  const bool disk = c->fd >= 0;
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
    if (disk) {
      q.manifest = reinterpret_cast<int32_t *>(c->stage_dev);
      q.disk_base = static_cast<int32_t>(c->hbm_rows + c->host_rows);
    }
    int e = launch_cache_plan(q, stream);
    if (e != 0) return cuda_fail(static_cast<cudaError_t>(e), "cache plan launch");
    if (disk && !put)  // reader: disk records -> staging, before the copy kernel
      AF_CUDA(cudaLaunchHostFunc(static_cast<cudaStream_t>(stream), disk_io, c), "cudaLaunchHostFunc(read)");
    CacheParams r = p;
    r.ids = p.ids + b0;
    r.n = n;
    r.rowslot = q.rowslot;
    r.host = c->host;
    r.hbm_rows = c->hbm_rows;
    if (disk) {
      r.stage = c->stage_dev + c->manifest_bytes();
      r.disk_base = c->hbm_rows + c->host_rows;
    }
    if (put)
      r.src_rows = p.src_rows + static_cast<int64_t>(b0) * c->row_bytes;
    else
      r.dst_rows = p.dst_rows + static_cast<int64_t>(b0) * c->row_bytes;
    e = put ? launch_cache_put(r, c->grid, stream) : launch_cache_get(r, c->grid, stream);
    if (e != 0) return cuda_fail(static_cast<cudaError_t>(e), "cache copy launch");
    if (disk && put)  // writer: staging -> disk records, after the copy kernel
      AF_CUDA(cudaLaunchHostFunc(static_cast<cudaStream_t>(stream), disk_io, c), "cudaLaunchHostFunc(write)");
  }
  return AF_OK;
}

af_status af_cache_put(af_cache *c, const int64_t *ids_dev, int32_t n, const void *rows_dev, int32_t depth,
                       void *stream) {
  AF_NVTX();
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
  AF_NVTX();
  return af_cache_get_ex(c, ids_dev, n, cur_boundary, rows_out_dev, depth_out_dev, 0u, stream);
}

af_status af_cache_get_ex(af_cache *c, const int64_t *ids_dev, int32_t n, int32_t cur_boundary, void *rows_out_dev,
                          int32_t *depth_out_dev, uint32_t flags, void *stream) {
  AF_NVTX();
  if (flags & ~AF_CACHE_OVERLAP_PREV) return fail(AF_EINVAL, "unknown flags");
  if ((flags & AF_CACHE_OVERLAP_PREV) && c && c->tiered)
    return fail(AF_ESTATE, "AF_CACHE_OVERLAP_PREV needs a direct-mapped store");
  CacheParams p;
  af_status s = cache_common(c, ids_dev, n, rows_out_dev, p);
  if (s != AF_OK) return s;
  if (n > 0 && !depth_out_dev) return fail(AF_EINVAL, "NULL depth_out");
  if (cur_boundary < 0) return fail(AF_EINVAL, "cur_boundary < 0");
  if (n == 0) return AF_OK;
  p.dst_rows = static_cast<char *>(rows_out_dev);
  p.depth_out = depth_out_dev;
  p.cur_boundary = cur_boundary;
  p.no_wait = (flags & AF_CACHE_OVERLAP_PREV) ? 1 : 0;
  if (c->tiered) return cache_tiered(c, p, false, stream);
  const int e = launch_cache_get(p, c->grid, stream);
  if (e != 0) return cuda_fail(static_cast<cudaError_t>(e), "cache get launch");
  return AF_OK;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static af_status encode_tiled(CUtensorMap *m, void *base, int rank, const cuuint64_t *dims, const cuuint64_t *strides,
                              const cuuint32_t *box) {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    AF_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q), "cudaGetDriverEntryPoint");
    if (!p || q != cudaDriverEntryPointSuccess) return fail(AF_ECUDA, "cuTensorMapEncodeTiled not found");
    fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  const cuuint32_t estr[3] = {1, 1, 1};
  const CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, static_cast<cuuint32_t>(rank), base, dims, strides, box,
                        estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(AF_EINVAL, "cuTensorMapEncodeTiled rejected the operand layout");
  return AF_OK;
}

af_status af_cache_get_gemm(af_cache *c, const int64_t *ids_dev, int32_t n, int32_t cur_boundary,
                            int32_t rows_per_record, int32_t K, const void *w_dev, int32_t N, void *y_dev,
                            int32_t *depth_out_dev, void *stream) {
  AF_NVTX();
  if (!c) return fail(AF_EINVAL, "NULL cache");
  if (!c->bound) return fail(AF_EWORKSPACE, "cache storage not bound");
  if (c->tiered || c->peers) return fail(AF_ESTATE, "af_cache_get_gemm needs a direct-mapped store without peers");
  if (n < 0 || cur_boundary < 0) return fail(AF_EINVAL, "n < 0 or cur_boundary < 0");
  if (n == 0) return AF_OK;
  if (!ids_dev || !w_dev || !y_dev || !depth_out_dev) return fail(AF_EINVAL, "NULL argument");
  if (rows_per_record <= 0 || rows_per_record % 128 != 0) return fail(AF_EINVAL, "rows_per_record: a multiple of 128");
  if (K <= 0 || K % 64 != 0 || N <= 0 || N % 32 != 0) return fail(AF_EINVAL, "K: a multiple of 64, N: of 32");
  if (static_cast<int64_t>(rows_per_record) * K * 2 != c->row_bytes)
    return fail(AF_EINVAL, "row_bytes != rows_per_record x K x 2 (bf16 records)");
  if (!aligned(w_dev, 16) || !aligned(y_dev, 16) || !aligned(ids_dev, 8)) return fail(AF_EINVAL, "misaligned buffer");
  if (c->capacity < 1) return fail(AF_EINVAL, "empty partition");
  alignas(64) CUtensorMap ta, tb;
  {  // the store as [slot][row][k] bf16: example i's record is the box at (k, m, slot_i)
    const cuuint64_t dims[3] = {static_cast<cuuint64_t>(K), static_cast<cuuint64_t>(rows_per_record),
                                static_cast<cuuint64_t>(c->capacity)};
    const cuuint64_t strides[2] = {static_cast<cuuint64_t>(K) * 2, static_cast<cuuint64_t>(c->row_bytes)};
    const cuuint32_t box[3] = {64, 128, 1};
    af_status st = encode_tiled(&ta, c->payload, 3, dims, strides, box);
    if (st != AF_OK) return st;
  }
  {  // W as [N][K] bf16 (a torch Linear weight): box of 128 rows x 64 k (each CTA of a pair
     // loads one half of a 256-row N tile, multicast to both)
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(K), static_cast<cuuint64_t>(N)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(K) * 2};
    const cuuint32_t box[2] = {64, 128};
    af_status st = encode_tiled(&tb, const_cast<void *>(w_dev), 2, dims, strides, box);
    if (st != AF_OK) return st;
  }
  alignas(64) CUtensorMap ty;
  {  // y as [n * rows_per_record][N] bf16: the epilogue's TMA stores of 128 x 64 chunks
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(N), static_cast<cuuint64_t>(n) * rows_per_record};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(N) * 2};
    const cuuint32_t box[2] = {64, 128};
    af_status st = encode_tiled(&ty, y_dev, 2, dims, strides, box);
    if (st != AF_OK) return st;
  }
  CacheGemmParams p{};
  p.meta = reinterpret_cast<CacheMeta *>(c->meta + kMetaHeader);
  p.err = reinterpret_cast<unsigned int *>(c->meta);
  p.ids = ids_dev;
  p.n = n;
  p.cur_boundary = cur_boundary;
  p.depth_out = depth_out_dev;
  p.num_examples = c->num_examples;
  p.rank = c->rank;
  p.world = c->world;
  p.rows = rows_per_record;
  p.n_tiles_m = rows_per_record / 128;
  p.n_tiles_n = (N + 255) / 256;
  p.N = N;
  p.K = K;
  p.y = y_dev;
  p.ldy = N;
  if (static_cast<int64_t>(n) * p.n_tiles_m * p.n_tiles_n > (int64_t(1) << 31) - 1) return fail(AF_ERANGE, "grid too large");
  const int e = launch_cache_gemm(p, &ta, &tb, &ty, stream);
  if (e != 0) return cuda_fail(static_cast<cudaError_t>(e), "cache get + GEMM launch");
  return AF_OK;
}

af_status af_cache_stats(af_cache *c, af_cache_info *out) {
  AF_NVTX();
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
  out->capacity = c->tiered ? c->slots() : c->capacity;
  for (const auto &x : m) {
    if (!x.valid) continue;
    out->n_valid++;
    if (c->tiered && x.slot >= c->hbm_rows + c->host_rows)
      out->n_disk++;
    else if (c->tiered && x.slot >= c->hbm_rows)
      out->n_host++;
    else
      out->n_hbm++;
  }
  out->error_flags |= c->disk_err.load();
  out->n_dropped = c->tiered ? h.dropped : 0;
  out->free_slots = c->tiered ? h.top : c->capacity - out->n_valid;
  return AF_OK;
}

af_status af_cache_status(af_cache *c, uint32_t *device_error_flags, int64_t *n_valid) {
  AF_NVTX();
  if (!c || !device_error_flags) return fail(AF_EINVAL, "NULL argument");
  if (!c->bound) return fail(AF_EWORKSPACE, "cache storage not bound");
  AF_CUDA(cudaDeviceSynchronize(), "cache status sync");
  unsigned int err = 0;
  AF_CUDA(cudaMemcpy(&err, c->meta, sizeof(err), cudaMemcpyDeviceToHost), "cudaMemcpy(err)");  // CacheHeader.err
  *device_error_flags = err | c->disk_err.load();
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
  AF_NVTX();
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
  AF_NVTX();
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
  AF_NVTX();
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
    const af_status st = enable_peer_access_to(q->payload);  // a store on another device: over NVLink
    if (st != AF_OK) return st;
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
  AF_NVTX();
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
  AF_NVTX();
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
  AF_NVTX();
  if (!c) return fail(AF_EINVAL, "NULL cache");
  ipc_release(c->ipc_opened);
  if (c->fd >= 0) ::close(c->fd);  // the file stays (the caller named it)
  delete c;
  return AF_OK;
}

}  // extern "C"
