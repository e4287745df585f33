// af_decide.cu -- the standalone single-CTA decision kernel (world > 1, or the
// unfused af_update_and_decide call); the logic lives in af_decide.cuh.
#include <cuda_runtime.h>

#include "af_decide.cuh"

namespace af {
namespace {

__global__ void __launch_bounds__(kDecideThreads) decide_kernel(const DecideParams p) {
  pdl_wait();  // the sums come from the preceding kernel / all-gather
  pdl_launch_dependents();
  const DecideIn in = decide_load(p);
  __syncthreads();
  decide_block(p, nullptr, in);
}

}  // namespace

int preload_decide_kernel() {
  cudaFuncAttributes a;
  return static_cast<int>(cudaFuncGetAttributes(&a, decide_kernel));
}

int launch_decide(const DecideParams &p, void *stream) {
  return static_cast<int>(launch_pdl(decide_kernel, dim3(1), dim3(kDecideThreads), 0, static_cast<cudaStream_t>(stream), p));
}

}  // namespace af
