// af_host.h -- host-side helpers shared by the C-ABI translation units
// (error reporting, alignment, device queries, CUDA IPC export/import).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "af_internal.h"

namespace af {

af_status fail(af_status s, const char *what);
af_status cuda_fail(cudaError_t e, const char *where);
void set_last_error(const std::string &msg);
const char *g_last_error_cstr();

#define AF_CUDA(call, where)                                  \
  do {                                                        \
    cudaError_t e_ = (call);                                  \
    if (e_ != cudaSuccess) return ::af::cuda_fail(e_, where); \
  } while (0)

inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }
inline bool aligned(const void *p, size_t a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; }
int device_sm_count(int *sms);

// CUDA IPC export of a pointer that may sit inside a larger allocation (the
// caller's allocator sub-allocates): handle of the allocation base + offset.
struct IpcRef {
  cudaIpcMemHandle_t h;
  uint64_t offset;
};
af_status ipc_export(const void *ptr, IpcRef *out);
af_status ipc_import(const IpcRef &r, std::vector<void *> &opened, char **out);
void ipc_release(const std::vector<void *> &opened);  // drop the references ipc_import took

}  // namespace af
