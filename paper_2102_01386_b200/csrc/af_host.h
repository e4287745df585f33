// af_host.h -- host-side helpers shared by the C-ABI translation units
// (error reporting, alignment, device queries, CUDA IPC export/import).
#pragma once
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

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

// NVTX range around every C-ABI entry point (SURVEY.md §5 tracing): nsys / ncu
// timelines show each af_* call with the kernels it enqueued.  Header-only NVTX3;
// a push/pop costs a few ns when no tool is attached.
struct NvtxRange {
  explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange &) = delete;
  NvtxRange &operator=(const NvtxRange &) = delete;
};
#define AF_NVTX() ::af::NvtxRange af_nvtx_range_(__func__)

inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }
inline bool aligned(const void *p, size_t a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; }
int device_sm_count(int *sms);
// Peer access from the current device to `device` (no-op for the same device or
// device < 0; AF_EINVAL when the hardware cannot; "already enabled" is success).
af_status enable_peer_access(int device);
// The same for the device that owns allocation `ptr` (host / unregistered: no-op).
af_status enable_peer_access_to(const void *ptr);

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
