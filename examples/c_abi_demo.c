/*
 * c_abi_demo.c -- drives libautofreeze through the plain C ABI (include/af.h),
 * no Python: the tiny closed-form config of SURVEY.md §8(c) (4 POOL x 4096 fp32,
 * 4 steps per interval, 10 intervals, N = 50), plus a cache round trip.
 * Prints one line per interval: "T <interval> boundary <f'> threshold <thr>".
 *
 *   gcc -O2 -std=c11 -I include -I /usr/local/cuda/include examples/c_abi_demo.c \
 *       -L paper_2102_01386_b200 -lautofreeze -L /usr/local/cuda/lib64 -lcudart \
 *       -Wl,-rpath,$PWD/paper_2102_01386_b200 -lm -o c_abi_demo
 *
 * The gradient generator re-implements afinputs' splitmix64 dyadic recipe (an
 * input generator, no method arithmetic).
 */
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "af.h"

#define CHECK(x)                                                                      \
  do {                                                                                \
    af_status s_ = (x);                                                               \
    if (s_ != AF_OK) {                                                                \
      fprintf(stderr, "%s -> %s: %s\n", #x, af_status_str(s_), af_last_error());     \
      return 1;                                                                       \
    }                                                                                 \
  } while (0)
#define CUDA(x)                                                                       \
  do {                                                                                \
    cudaError_t e_ = (x);                                                             \
    if (e_ != cudaSuccess) {                                                          \
      fprintf(stderr, "%s -> %s\n", #x, cudaGetErrorString(e_));                      \
      return 1;                                                                       \
    }                                                                                 \
  } while (0)

static uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
static int64_t dyadic_k(uint64_t seed, uint64_t stream, uint64_t seg, uint64_t idx) {
  uint64_t h = splitmix64(seed);
  h = splitmix64(h ^ stream);
  h = splitmix64(h ^ seg);
  h = splitmix64(h ^ idx);
  return (int64_t)(h >> 54) - 512;
}

int main(void) {
  enum { L = 4, SEG = 4096, N = L * SEG, STEPS = 4, INTERVALS = 10 };
  const double rho[L] = {0.30, 0.55, 0.75, 0.90};
  int64_t offs[L + 1];
  int32_t kinds[L];
  for (int l = 0; l <= L; ++l) offs[l] = (int64_t)l * SEG;
  for (int l = 0; l < L; ++l) kinds[l] = AF_SEG_POOL;
  af_layout lay = {L, offs, kinds, AF_DT_F32};
  af_config cfg = {50.0, AF_PCT_LINEAR, AF_ACC_DELTA, 1e-5, 2, 0, 1};
  af_ctx *ctx = NULL;
  CHECK(af_ctx_create(&lay, &cfg, &ctx));
  size_t accum_b = 0, scratch_b = 0;
  CHECK(af_ctx_workspace_bytes(ctx, &accum_b, &scratch_b));
  void *accum = NULL, *scratch = NULL, *grad = NULL;
  CUDA(cudaMalloc(&accum, accum_b));
  CUDA(cudaMalloc(&scratch, scratch_b));
  CUDA(cudaMalloc(&grad, N * sizeof(float)));
  CHECK(af_ctx_bind(ctx, accum, scratch));
  af_decision *rec = NULL;
  CUDA(cudaHostAlloc((void **)&rec, sizeof(af_decision), cudaHostAllocDefault));
  cudaStream_t st;
  CUDA(cudaStreamCreate(&st));
  float *host = (float *)malloc(N * sizeof(float));
  for (int T = 0; T < INTERVALS; ++T) {
    for (int t = 0; t < STEPS; ++t) {
      for (int l = 0; l < L; ++l) {
        const double a = floor(2048.0 * (1.0 + 0.9 * pow(rho[l], T)) + 0.5) / 2048.0;
        const double sgn = (t % 2 == 0) ? 1.0 : -1.0;
        for (int i = 0; i < SEG; ++i) {
          const double z = dyadic_k(0, 0, l, i) / 1024.0, w = dyadic_k(0, 1, l, i) / 1024.0;
          host[l * SEG + i] = (float)(a * z + sgn * 2.0 * w);
        }
      }
      CUDA(cudaMemcpyAsync(grad, host, N * sizeof(float), cudaMemcpyHostToDevice, st));
      if (t == STEPS - 1)
        CHECK(af_interval_end(ctx, grad, 0, rec, st));
      else
        CHECK(af_layer_norms(ctx, grad, 0, st));
      CUDA(cudaStreamSynchronize(st));  /* the host buffer is reused next step */
    }
    printf("T %d boundary %d threshold %.6f flags %u\n", rec->interval, rec->boundary_after, rec->threshold,
           rec->flags);
  }
  /* cache round trip: put 3 rows at depth 2, read them back at boundary 3 (evicted) */
  af_cache *c = NULL;
  CHECK(af_cache_create(64, 1024, 0, 1, &c));
  size_t pb = 0, mb = 0;
  CHECK(af_cache_storage_bytes(c, &pb, &mb));
  void *payload = NULL, *meta = NULL, *rows = NULL, *out = NULL, *ids = NULL, *dep = NULL;
  CUDA(cudaMalloc(&payload, pb));
  CUDA(cudaMalloc(&meta, mb));
  CUDA(cudaMalloc(&rows, 3 * 1024));
  CUDA(cudaMalloc(&out, 3 * 1024));
  CUDA(cudaMalloc(&ids, 3 * sizeof(int64_t)));
  CUDA(cudaMalloc(&dep, 3 * sizeof(int32_t)));
  CHECK(af_cache_bind(c, payload, meta));
  const int64_t hid[3] = {5, 9, 63};
  unsigned char hrow[3 * 1024], hout[3 * 1024];
  for (int i = 0; i < 3 * 1024; ++i) hrow[i] = (unsigned char)(i * 7 + 3);
  CUDA(cudaMemcpy(ids, hid, sizeof(hid), cudaMemcpyHostToDevice));
  CUDA(cudaMemcpy(rows, hrow, sizeof(hrow), cudaMemcpyHostToDevice));
  CHECK(af_cache_put(c, (const int64_t *)ids, 3, rows, 2, st));
  CHECK(af_cache_get(c, (const int64_t *)ids, 3, 3, out, (int32_t *)dep, st));
  CUDA(cudaStreamSynchronize(st));
  int32_t hdep[3];
  CUDA(cudaMemcpy(hout, out, sizeof(hout), cudaMemcpyDeviceToHost));
  CUDA(cudaMemcpy(hdep, dep, sizeof(hdep), cudaMemcpyDeviceToHost));
  uint32_t err = 0;
  int64_t valid = -1;
  CHECK(af_cache_status(c, &err, &valid));
  printf("cache roundtrip %s depths %d %d %d valid_after_evict %lld err %u\n",
         memcmp(hout, hrow, sizeof(hrow)) == 0 ? "ok" : "MISMATCH", hdep[0], hdep[1], hdep[2], (long long)valid,
         err);
  CHECK(af_cache_destroy(c));
  CHECK(af_ctx_destroy(ctx));
  free(host);
  return 0;
}
