// af_gemm.cu -- SURVEY.md §8(f) NEXT 4, second half: the cache get fused into the
// first active layer's GEMM operand load.
//
// Once the first f blocks are frozen, the next epoch reads each example's cached
// layer-f output by its original id (§3.2) and feeds it to block f+1,
// whose first operation is a dense projection y = x W^T (BERT: the QKV projection
// of 768 -> 2304).  af_cache_get would copy every hit record (rows_per_record x K
// bf16) into a batch buffer that the projection then reads back: 2 x 196 KB of
// HBM traffic per example for nothing.  Here the projection's TMA loads read the
// A operand straight out of the store -- the record IS the operand tile: record
// slot s is rows_per_record (= 128 = one M tile) x K contiguous bf16, so a 3-D
// tensor map over [slot][row][k] gathers example i's tile with the coordinate
// z = slot(id_i) -- and the 5th-generation tensor cores multiply it:
//
//   tile = (example i, 128-row M tile of its record, 256-column N tile); the
//   producer resolves id -> slot and the record's {depth, valid} (a miss skips
//   the tile: depth_out = -1, y untouched); a 4-stage TMA ring (A 128x64 + B
//   256x64 bf16, 128-byte swizzle, 48 KiB per stage) feeds one thread issuing
//   tcgen05.mma (kind::f16, M = 128, N = 256, K = 16, fp32 accumulators in TMEM,
//   two of 256 columns); four epilogue warps drain TMEM with tcgen05.ld (32
//   lanes x 32 columns per load), round to bf16 (RNE) and store y rows; the last
//   of a record's tiles to read its meta word applies the evict-on-read (depth <
//   cur_boundary).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "af_internal.h"
#include "af_ptx.cuh"

namespace af {
namespace {

constexpr int kGM = 128, kGN = 256, kGK = 64, kGStages = 6;
constexpr int kGABytes = kGM * kGK * 2;             // 16 KiB: this CTA's 128 rows of the pair's 256-row A tile
constexpr int kGBBytes = kGN / 2 * kGK * 2;         // 16 KiB: this CTA's half (128 columns) of the 256-wide B tile
constexpr int kGStageBytes = kGABytes + kGBBytes;   // 32 KiB per CTA (64 KiB per pair)
constexpr int kGEpiBytes = kGM * 64 * 2;                // one 128 x 64 bf16 output chunk (16 KiB), double-buffered
constexpr int kGSmem = kGStages * kGStageBytes + 2 * kGEpiBytes + 1024;  // + slack for 1024-B alignment

// UMMA shared-memory descriptor of a K-major, 128-byte-swizzled bf16 tile whose
// rows are 128 B apart (8-row swizzle atoms 1024 B apart): start address >> 4,
// leading byte offset 16 B (unused for swizzled K-major), stride byte offset
// 1024 B, version 1 (sm100), layout SWIZZLE_128B (2).
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t smem_addr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((smem_addr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>(16u >> 4) << 16;
  d |= static_cast<uint64_t>(1024u >> 4) << 32;
  d |= static_cast<uint64_t>(1u) << 46;
  d |= static_cast<uint64_t>(2u) << 61;
  return d;
}

// Instruction descriptor (kind::f16): D fp32, A and B bf16, both K-major, N = 256,
// M = 256 (cta_group::2: the CTA pair's two 128-row halves).
constexpr uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(kGN >> 3) << 17) |
                            (static_cast<uint32_t>((2 * kGM) >> 4) << 24);
// A shared::cluster address with the pair's peer bit cleared: the leader CTA's copy
// (the TMA of either CTA completes its bytes on the leader's barrier)
constexpr uint32_t kPeerBitMask = 0xFEFFFFFFu;

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  const __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);  // .x = lo (lower address), RNE
  return *reinterpret_cast<const uint32_t *>(&v);
}

// Persistent, warp-specialised, CTA pairs (clusters of two) running 2-SM MMAs:
// cluster c walks pair tiles u = c, c + C, ...; pair tile u = (N tile, a pair of
// row tiles); CTA rank r of the pair takes row tile 2 (u / n_tiles_n) + r (row
// tile = (example, 128-row M tile of its record)).  Each CTA TMA-loads its own A
// tile (128 rows) and its half of the 256-wide B tile into its own shared memory,
// both completing on the leader's stage barrier; the leader's single thread
// issues tcgen05.mma.cta_group::2 (M = 256: the two CTAs' rows, N = 256, K = 16),
// whose accumulator rows land in each CTA's own TMEM, and its commits release the
// stage and signal the accumulator in both CTAs.  Per SM this moves 32 KiB of
// operands per 64-deep k-block instead of 48 (one CTA alone, N = 256), so the
// 6-stage ring covers more of the L2 latency.  Warp 0 lane 0 = producer: resolves
// the tile's id -> slot and {depth, valid} ONCE (the tile info the epilogue
// reads, so an eviction by another tile cannot change a tile's view); warp 1 lane
// 0 of the leader = MMA issuer; warps 2-5 = epilogue (each CTA drains its own 128
// TMEM lanes).  Two TMEM accumulators (2 x 256 columns) let tile j+1's MMAs run
// while tile j is drained; the leader's MMA waits for BOTH CTAs' epilogues.  A
// missed or absent row tile still loads (slot 0) and multiplies -- its partner's
// MMA reads it and both CTAs keep the same phases -- and stores nothing.
constexpr int kGRoles = 2 * 32;                 // producer warp + MMA warp
constexpr int kGEpi = 128;                      // epilogue warps 2..5
constexpr int kGThreadsP = kGRoles + kGEpi;

struct TileInfo {
  int64_t slot;
  int32_t hit, depth, ex, mt, nt, pad;
};

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t map_to_rank(uint32_t local_smem_addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local_smem_addr), "r"(rank));
  return r;
}

__global__ void __launch_bounds__(kGThreadsP, 1)
    cache_gemm_kernel(const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_b,
                      const __grid_constant__ CUtensorMap tmap_y, const CacheGemmParams p) {
  extern __shared__ unsigned char g_smem_raw[];
  unsigned char *smem = reinterpret_cast<unsigned char *>((reinterpret_cast<uintptr_t>(g_smem_raw) + 1023) &
                                                         ~static_cast<uintptr_t>(1023));
  __shared__ __align__(8) uint64_t full[kGStages], empty[kGStages];
  __shared__ __align__(8) uint64_t info_full[2], info_free[2], tmem_full[2], tmem_empty[2];
  __shared__ TileInfo tinfo[2];
  __shared__ uint32_t s_tmem;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int rank = static_cast<int>(cluster_rank());
  const int tiles_per_ex = p.n_tiles_m * p.n_tiles_n;
  const int64_t row_tiles = static_cast<int64_t>(p.n) * p.n_tiles_m;
  const int64_t pair_tiles = (row_tiles + 1) / 2 * p.n_tiles_n;
  const int C = static_cast<int>(gridDim.x) / 2, cid = static_cast<int>(blockIdx.x) / 2;

  if (tid == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmap_a) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmap_b) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmap_y) : "memory");
    for (int s = 0; s < kGStages; ++s) {
      mbar_init(&full[s], 1);   // (leader's) the leader producer's arrive + both CTAs' TMA bytes
      mbar_init(&empty[s], 1);  // the leader's MMA commit, multicast to both CTAs
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&info_full[a], 1);
      mbar_init(&info_free[a], kGEpi / 32);           // this CTA's epilogue warps are done with tinfo[a]
      mbar_init(&tmem_full[a], 1);                    // the leader's commit, multicast to both CTAs
      mbar_init(&tmem_empty[a], 2 * kGEpi / 32);      // (leader's) both CTAs' epilogue warps drained it
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {  // 512 TMEM columns in each CTA of the pair: two 128 x 256 fp32 accumulators
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s_tmem)),
                 "r"(512u));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();     // the allocator's write of s_tmem is visible to the CTA
  cluster_sync_all();  // the partner's barriers exist before any TMA or commit signals them
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = s_tmem;
  const int nk = p.K / kGK;
  pdl_wait();  // ids (and the store) may come from the preceding kernels

  if (warp == 0) {
    if (lane == 0) {  // ===== producer
      uint32_t q = 0;  // k-blocks issued so far
      int j = 0;
      for (int64_t u = cid; u < pair_tiles; u += C, ++j) {
        const int a = j & 1;
        if (j >= 2) mbar_wait(&info_free[a], ((j >> 1) - 1) & 1);  // tinfo[a] no longer read
        TileInfo ti{};
        ti.nt = static_cast<int32_t>(u % p.n_tiles_n);
        const int64_t rt = (u / p.n_tiles_n) * 2 + rank;
        if (rt < row_tiles) {
          ti.ex = static_cast<int32_t>(rt / p.n_tiles_m);
          ti.mt = static_cast<int32_t>(rt % p.n_tiles_m);
          const int64_t id = p.ids[ti.ex];
          const bool first_tile = ti.mt == 0 && ti.nt == 0;
          if (id < 0 || id >= p.num_examples) {
            if (first_tile) atomicOr(p.err, AF_CACHE_ERR_RANGE);
          } else if (id % p.world != p.rank) {
            if (first_tile) atomicOr(p.err, AF_CACHE_ERR_OWNER);
          } else {
            const int64_t slot = id / p.world;
            const int4 mv = __ldcg(reinterpret_cast<const int4 *>(p.meta) + slot);  // {depth, valid, readers, -}
            ti.hit = mv.y != 0;
            ti.depth = mv.x;
            if (ti.hit) ti.slot = slot;
          }
          if (first_tile) p.depth_out[ti.ex] = ti.hit ? ti.depth : -1;
        }
        tinfo[a] = ti;
        asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&info_full[a])) : "memory");
        for (int kb = 0; kb < nk; ++kb, ++q) {
          const int s = static_cast<int>(q % kGStages);
          if (q >= static_cast<uint32_t>(kGStages)) mbar_wait(&empty[s], ((q / kGStages) - 1) & 1);
          unsigned char *sa = smem + s * kGStageBytes;
          unsigned char *sb = sa + kGABytes;
          const uint32_t bar = smem_u32(&full[s]) & kPeerBitMask;  // the leader's stage barrier
          if (rank == 0) mbar_expect_tx(&full[s], 2 * kGStageBytes);  // both CTAs' A and B halves
          asm volatile(
              "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], "
              "[%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(sa)),
              "l"(&tmap_a), "r"(kb * kGK), "r"(ti.mt * kGM), "r"(static_cast<int>(ti.slot)), "r"(bar)
              : "memory");
          asm volatile(
              "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], "
              "[%1, {%2, %3}], [%4];" ::"r"(smem_u32(sb)),
              "l"(&tmap_b), "r"(kb * kGK), "r"(ti.nt * kGN + rank * (kGN / 2)), "r"(bar)
              : "memory");
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {  // ===== MMA issuer (the pair's leader)
      uint32_t q = 0;
      int j = 0;
      for (int64_t u = cid; u < pair_tiles; u += C, ++j) {
        const int a = j & 1;
        if (j >= 2) mbar_wait(&tmem_empty[a], ((j >> 1) - 1) & 1);  // accumulator a drained
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t acc_cols = tmem + static_cast<uint32_t>(a * kGN);
        for (int kb = 0; kb < nk; ++kb, ++q) {
          const int s = static_cast<int>(q % kGStages);
          mbar_wait(&full[s], (q / kGStages) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t sa = smem_u32(smem + s * kGStageBytes), sb = sa + kGABytes;
#pragma unroll
          for (int k = 0; k < kGK / 16; ++k) {
            const uint64_t da = umma_desc_sw128(sa + k * 32), db = umma_desc_sw128(sb + k * 32);
            const uint32_t acc = (kb | k) != 0 ? 1u : 0u;
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(acc_cols),
                "l"(da), "l"(db), "r"(kIdesc), "r"(acc)
                : "memory");
          }
          // the stage is free in both CTAs once these MMAs have read it
          asm volatile(
              "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                  smem_u32(&empty[s])),
              "h"(static_cast<uint16_t>(0x3))
              : "memory");
        }
        asm volatile(
            "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                smem_u32(&tmem_full[a])),
            "h"(static_cast<uint16_t>(0x3))
            : "memory");
      }
    }
  } else {
    // ===== epilogue: warp w accesses TMEM lanes 32 (w % 4) .. + 31 (= output rows)
    const int quad = warp & 3;
    const int row = quad * 32 + lane;
    int epi_chunk = 0;  // output chunks staged so far (selects the staging buffer)
    int j = 0;
    for (int64_t u = cid; u < pair_tiles; u += C, ++j) {
      const int a = j & 1;
      mbar_wait(&info_full[a], (j >> 1) & 1);  // acquire the producer's tile info directly
      mbar_wait(&tmem_full[a], (j >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const TileInfo ti = tinfo[a];
      if (ti.hit) {
        // TMEM -> registers -> bf16 -> shared memory in the 128-byte-swizzled layout of
        // the y tensor map (row r's 16-byte chunk c at chunk c ^ (r % 8)) -> one TMA
        // store per 128 x 64 chunk, double-buffered (coalesced, asynchronous)
        const int64_t y_row0 = static_cast<int64_t>(ti.ex) * p.rows + static_cast<int64_t>(ti.mt) * kGM;
#pragma unroll 1
        for (int c0 = 0; c0 < kGN && ti.nt * kGN + c0 < p.N; c0 += 64, ++epi_chunk) {
          unsigned char *buf = smem + kGStages * kGStageBytes + (epi_chunk & 1) * kGEpiBytes;
          if (epi_chunk >= 2) {  // the TMA store that last read this buffer is done reading it
            if (tid == kGRoles) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
            asm volatile("bar.sync 1, %0;" ::"n"(kGEpi) : "memory");
          }
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            uint32_t v[32];
            const uint32_t taddr =
                tmem + (static_cast<uint32_t>(quad * 32) << 16) + static_cast<uint32_t>(a * kGN + c0 + 32 * h);
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, "
                "%13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, "
                "[%32];"
                : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                  "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
                  "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
                  "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
                  "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                : "r"(taddr));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int qv = 0; qv < 4; ++qv) {
              const int chunk = 4 * h + qv;  // 16-byte chunk of the row's 128 bytes
              const uint32_t addr = smem_u32(buf) + static_cast<uint32_t>(row * 128 + ((chunk ^ (row & 7)) << 4));
              asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr),
                           "r"(pack_bf16(__uint_as_float(v[8 * qv + 0]), __uint_as_float(v[8 * qv + 1]))),
                           "r"(pack_bf16(__uint_as_float(v[8 * qv + 2]), __uint_as_float(v[8 * qv + 3]))),
                           "r"(pack_bf16(__uint_as_float(v[8 * qv + 4]), __uint_as_float(v[8 * qv + 5]))),
                           "r"(pack_bf16(__uint_as_float(v[8 * qv + 6]), __uint_as_float(v[8 * qv + 7])))
                           : "memory");
            }
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> async (TMA) proxy
          asm volatile("bar.sync 1, %0;" ::"n"(kGEpi) : "memory");
          if (tid == kGRoles) {
            asm volatile(
                "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(&tmap_y),
                "r"(ti.nt * kGN + c0), "r"(static_cast<int>(y_row0)), "r"(smem_u32(buf))
                : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          }
        }
        if (warp == 2 && lane == 0) {  // evict on read once every tile of the record has read its meta
          CacheMeta *m = p.meta + ti.slot;
          const unsigned int seen = atomicAdd(&m->readers, 1u);
          if (seen == static_cast<unsigned int>(tiles_per_ex) - 1u) {
            if (ti.depth < p.cur_boundary) m->valid = 0;
            m->readers = 0u;
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) {
        asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&info_free[a])) : "memory");
        // "accumulator drained" on the leader's barrier, default semantics (release at
        // CTA scope): this warp's TMEM reads completed at tcgen05.wait::ld, before
        // the arrive in program order, so the leader's next MMAs into these columns
        // cannot overtake them; a .release.cluster arrive cost a GPU-wide MEMBAR
        // per tile and warp (0.7 % of the kernel, profiles/r02/r02_v44_*)
        asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(map_to_rank(smem_u32(&tmem_empty[a]), 0))
                     : "memory");
      }
    }
  }
  if (tid == kGRoles) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // y written before exit
  pdl_launch_dependents();
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  cluster_sync_all();  // no CTA leaves while its partner may still multicast into it
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512u));
}

}  // namespace

int cache_gemm_smem_bytes() { return kGSmem; }

int launch_cache_gemm(const CacheGemmParams &p, const void *tmap_a, const void *tmap_b, const void *tmap_y,
                      void *stream) {
  const cudaError_t e = ensure_smem_attr<cache_gemm_kernel>(kGSmem);
  if (e != cudaSuccess) return static_cast<int>(e);
  const CUtensorMap &ta = *static_cast<const CUtensorMap *>(tmap_a);
  const CUtensorMap &tb = *static_cast<const CUtensorMap *>(tmap_b);
  const CUtensorMap &ty = *static_cast<const CUtensorMap *>(tmap_y);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t row_tiles = static_cast<int64_t>(p.n) * p.n_tiles_m;
  const int64_t pairs = (row_tiles + 1) / 2 * p.n_tiles_n;
  const int clusters = static_cast<int>(pairs < sms / 2 ? pairs : sms / 2);  // persistent: one CTA per SM
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(2 * (clusters < 1 ? 1 : clusters)));
  cfg.blockDim = dim3(kGThreadsP);
  cfg.dynamicSmemBytes = static_cast<size_t>(kGSmem);
  cfg.stream = static_cast<cudaStream_t>(stream);
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  cudaError_t r = cudaLaunchKernelEx(&cfg, cache_gemm_kernel, ta, tb, ty, p);
  return static_cast<int>(r != cudaSuccess ? r : cudaGetLastError());
}

int preload_cache_gemm_kernel() {
  cudaFuncAttributes a;
  return static_cast<int>(cudaFuncGetAttributes(&a, cache_gemm_kernel));
}

}  // namespace af
