// Microbenchmark: streaming-kernel variants for the interval-end sum of squares
// (read g + Delta, fp64 accumulate) and the accumulate (read g + Delta, write Delta)
// on B200.  Standalone (not part of the library); informs the kernel design.
//
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o sv stream_variants.cu && ./sv
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

#define CK(x)                                                                               \
  do {                                                                                      \
    cudaError_t e = (x);                                                                    \
    if (e != cudaSuccess) {                                                                 \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__);        \
      exit(1);                                                                              \
    }                                                                                       \
  } while (0)

// ---------------------------------------------------------------- LDG variants
template <int U, int HINT>
__device__ __forceinline__ float4 ld4(const float4 *p) {
  if (HINT == 0) return __ldcs(p);
  if (HINT == 1) return __ldg(p);
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p));
  return r;
}

template <int U, int HINT, int BLOCK>
__global__ void __launch_bounds__(BLOCK) ldg_sumsq(const float4 *g, const float4 *d, int64_t nv, int64_t tile_v,
                                                   double *part) {
  // static tiles of tile_v float4, round-robin over CTAs
  const int64_t ntiles = (nv + tile_v - 1) / tile_v;
  double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int64_t b = t * tile_v, e = min(nv, b + tile_v);
    for (int64_t c0 = b + threadIdx.x; c0 < e; c0 += U * BLOCK) {
      float4 gv[U], dv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t c = c0 + (int64_t)u * BLOCK;
        if (c < e) {
          gv[u] = ld4<U, HINT>(g + c);
          dv[u] = ld4<U, HINT>(d + c);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t c = c0 + (int64_t)u * BLOCK;
        if (c < e) {
          float x;
          x = dv[u].x + gv[u].x; a0 = __fma_rn((double)x, (double)x, a0);
          x = dv[u].y + gv[u].y; a1 = __fma_rn((double)x, (double)x, a1);
          x = dv[u].z + gv[u].z; a2 = __fma_rn((double)x, (double)x, a2);
          x = dv[u].w + gv[u].w; a3 = __fma_rn((double)x, (double)x, a3);
        }
      }
    }
  }
  double s = (a0 + a1) + (a2 + a3);
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(~0u, s, o);
  if ((threadIdx.x & 31) == 0) part[blockIdx.x * (BLOCK / 32) + threadIdx.x / 32] = s;
}

template <int U, int BLOCK>
__global__ void __launch_bounds__(BLOCK) ldg_accum(const float4 *g, float4 *d, int64_t nv, int64_t tile_v) {
  const int64_t ntiles = (nv + tile_v - 1) / tile_v;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int64_t b = t * tile_v, e = min(nv, b + tile_v);
    for (int64_t c0 = b + threadIdx.x; c0 < e; c0 += U * BLOCK) {
      float4 gv[U], dv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t c = c0 + (int64_t)u * BLOCK;
        if (c < e) {
          gv[u] = __ldcs(g + c);
          dv[u] = __ldcs(d + c);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t c = c0 + (int64_t)u * BLOCK;
        if (c < e)
          __stcs(d + c, make_float4(dv[u].x + gv[u].x, dv[u].y + gv[u].y, dv[u].z + gv[u].z, dv[u].w + gv[u].w));
      }
    }
  }
}

// ---------------------------------------------------------------- TMA bulk variants
__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(uint64_t *b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void mb_expect(uint64_t *b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mb_arrive(uint64_t *b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t *b, uint32_t par) {
  uint32_t ok = 0;
  do {
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0,1,0,p;\n\t}"
                 : "=r"(ok)
                 : "r"(su32(b)), "r"(par)
                 : "memory");
  } while (!ok);
}
__device__ __forceinline__ void g2s(void *s, const void *g, uint32_t bytes, uint64_t *b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   su32(s)),
               "l"(g), "r"(bytes), "r"(su32(b))
               : "memory");
}
__device__ __forceinline__ void s2g(void *g, const void *s, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(g), "r"(su32(s)), "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}

// one producer warp (lane 0 issues), NCW consumer warps; stage = CH floats of g + CH of d
template <int S, int CH, int NCW, bool ACCUM, bool BULK_STORE>
__global__ void __launch_bounds__(32 * (NCW + 1)) tma_kernel(const float *g, float *d, int64_t n, double *part) {
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t *full = (uint64_t *)smem;
  uint64_t *empty = full + S;
  float *buf = (float *)(smem + 256);
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mb_init(&full[s], 1);
      mb_init(&empty[s], NCW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t nch = n / CH;  // assume divisible in the microbench
  if (warp == 0) {
    if (lane == 0) {
      int k = 0;
      for (int64_t c = blockIdx.x; c < nch; c += gridDim.x, ++k) {
        const int s = k % S;
        if (k >= S) mb_wait(&empty[s], ((k / S) - 1) & 1);
        mb_expect(&full[s], 2 * CH * 4);
        g2s(buf + (size_t)s * 2 * CH, g + c * CH, CH * 4, &full[s]);
        g2s(buf + (size_t)s * 2 * CH + CH, d + c * CH, CH * 4, &full[s]);
      }
    }
    return;
  }
  const int ct = threadIdx.x - 32;
  double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
  int k = 0;
  for (int64_t c = blockIdx.x; c < nch; c += gridDim.x, ++k) {
    const int s = k % S;
    mb_wait(&full[s], (k / S) & 1);
    const float4 *gs = (const float4 *)(buf + (size_t)s * 2 * CH);
    float4 *ds = (float4 *)(buf + (size_t)s * 2 * CH + CH);
#pragma unroll 4
    for (int i = ct; i < CH / 4; i += 32 * NCW) {
      const float4 gv = gs[i], dv = ds[i];
      if (ACCUM) {
        const float4 x = make_float4(dv.x + gv.x, dv.y + gv.y, dv.z + gv.z, dv.w + gv.w);
        if (BULK_STORE)
          ds[i] = x;
        else
          __stcs((float4 *)(d + c * CH) + i, x);
      } else {
        float x;
        x = dv.x + gv.x; a0 = __fma_rn((double)x, (double)x, a0);
        x = dv.y + gv.y; a1 = __fma_rn((double)x, (double)x, a1);
        x = dv.z + gv.z; a2 = __fma_rn((double)x, (double)x, a2);
        x = dv.w + gv.w; a3 = __fma_rn((double)x, (double)x, a3);
      }
    }
    if (ACCUM && BULK_STORE) {
      asm volatile("bar.sync 1, %0;" ::"r"(32 * NCW) : "memory");
      if (ct == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        s2g(d + c * CH, ds, CH * 4);
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      }
      asm volatile("bar.sync 1, %0;" ::"r"(32 * NCW) : "memory");
    }
    __syncwarp();
    if (lane == 0) mb_arrive(&empty[s]);
  }
  if (ACCUM && BULK_STORE && ct == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  if (!ACCUM) {
    double sum = (a0 + a1) + (a2 + a3);
    for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(~0u, sum, o);
    if (lane == 0) part[blockIdx.x * NCW + warp - 1] = sum;
  }
}

// ---------------------------------------------------------------- harness
struct Timer {
  cudaEvent_t a, b;
  Timer() { cudaEventCreate(&a); cudaEventCreate(&b); }
  void start() { cudaEventRecord(a); }
  float stop() {
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms;
  }
};

template <typename F>
void run(const char *name, F f, double bytes, int reps = 10) {
  f();
  f();
  CK(cudaDeviceSynchronize());
  Timer t;
  std::vector<float> v;
  for (int r = 0; r < reps; ++r) {
    t.start();
    f();
    v.push_back(t.stop());
  }
  CK(cudaGetLastError());
  float best = 1e9, sum = 0;
  for (float x : v) { best = x < best ? x : best; sum += x; }
  printf("%-58s best %8.1f us  mean %8.1f us  -> %7.1f GB/s (best)  %7.1f GB/s (mean)\n", name, best * 1e3,
         sum / reps * 1e3, bytes / (best * 1e-3) / 1e9, bytes / (sum / reps * 1e-3) / 1e9);
}

int occ(const void *k, int block, int smem) {
  int b = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k, block, smem);
  return b;
}

int main() {
  const int64_t n = 335143936;  // BERT-large fp32 (rounded to a multiple of 4096)
  float *g, *d;
  double *part;
  CK(cudaMalloc(&g, n * 4));
  CK(cudaMalloc(&d, n * 4));
  CK(cudaMalloc(&part, 1 << 24));
  CK(cudaMemset(g, 0, n * 4));
  CK(cudaMemset(d, 0, n * 4));
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int64_t nv = n / 4;
  const double rb = n * 8.0, ab = n * 12.0;
  // copy reference
  run("cudaMemcpy D2D (read+write)", [&] { cudaMemcpyAsync(d, g, n * 4, cudaMemcpyDeviceToDevice); }, n * 8.0);
#define LDG_SUMSQ(U, H, BL, TV)                                                                        \
  {                                                                                                    \
    int o = occ((const void *)ldg_sumsq<U, H, BL>, BL, 0);                                             \
    char nm[128];                                                                                      \
    snprintf(nm, 128, "ldg_sumsq U=%d hint=%d block=%d tile=%dKB occ=%d", U, H, BL, (int)(TV * 16 / 1024), o); \
    run(nm, [&] { ldg_sumsq<U, H, BL><<<sms * o, BL>>>((const float4 *)g, (const float4 *)d, nv, TV, part); }, rb); \
  }
  LDG_SUMSQ(4, 0, 256, 4096)
  LDG_SUMSQ(8, 0, 256, 4096)
  LDG_SUMSQ(4, 1, 256, 4096)
  LDG_SUMSQ(4, 2, 256, 4096)
  LDG_SUMSQ(8, 2, 256, 4096)
  LDG_SUMSQ(4, 0, 512, 8192)
  LDG_SUMSQ(4, 0, 256, 16384)
  LDG_SUMSQ(2, 0, 256, 4096)
  LDG_SUMSQ(8, 0, 128, 4096)
#define LDG_ACC(U, BL, TV)                                                                              \
  {                                                                                                    \
    int o = occ((const void *)ldg_accum<U, BL>, BL, 0);                                                \
    char nm[128];                                                                                      \
    snprintf(nm, 128, "ldg_accum U=%d block=%d tile=%dKB occ=%d", U, BL, (int)(TV * 16 / 1024), o);      \
    run(nm, [&] { ldg_accum<U, BL><<<sms * o, BL>>>((const float4 *)g, (float4 *)d, nv, TV); }, ab);    \
  }
  LDG_ACC(4, 256, 4096)
  LDG_ACC(8, 256, 4096)
  LDG_ACC(2, 256, 4096)
  LDG_ACC(4, 512, 16384)
#define TMA(S, CH, NCW, ACC, BULK)                                                                      \
  {                                                                                                    \
    auto k = tma_kernel<S, CH, NCW, ACC, BULK>;                                                        \
    const int smem = 256 + S * 2 * CH * 4;                                                             \
    CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));                    \
    int o = occ((const void *)k, 32 * (NCW + 1), smem);                                                \
    char nm[128];                                                                                      \
    snprintf(nm, 128, "tma %s S=%d chunk=%dKB cw=%d bulkst=%d occ=%d", ACC ? "accum" : "sumsq", S,       \
             CH * 4 / 1024, NCW, BULK, o);                                                              \
    run(nm, [&] { k<<<sms * o, 32 * (NCW + 1), smem>>>(g, d, n, part); }, ACC ? ab : rb);              \
  }
  TMA(4, 4096, 4, false, false)
  TMA(6, 4096, 4, false, false)
  TMA(3, 8192, 8, false, false)
  TMA(6, 2048, 4, false, false)
  TMA(12, 2048, 4, false, false)
  TMA(4, 4096, 8, false, false)
  TMA(2, 4096, 4, false, false)
  TMA(3, 2048, 2, false, false)
  TMA(4, 4096, 4, true, false)
  TMA(6, 4096, 4, true, false)
  TMA(4, 4096, 4, true, true)
  TMA(6, 4096, 4, true, true)
  TMA(3, 2048, 2, true, false)
  return 0;
}
