// af_host.cpp -- shared host helpers and the stateless entry points of the C ABI.
#include "af_host.h"

#include <cstring>
#include <map>
#include <mutex>
#include <string>

namespace af {
namespace {
thread_local std::string g_last_error;
}  // namespace

void set_last_error(const std::string &msg) { g_last_error = msg; }
const char *g_last_error_cstr() { return g_last_error.c_str(); }

af_status fail(af_status s, const char *what) {
  g_last_error = what;
  return s;
}

af_status cuda_fail(cudaError_t e, const char *where) {
  g_last_error = std::string(where) + ": " + cudaGetErrorString(e);
  return AF_ECUDA;
}

int device_sm_count(int *sms) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return static_cast<int>(e);
  return static_cast<int>(cudaDeviceGetAttribute(sms, cudaDevAttrMultiProcessorCount, dev));
}

af_status enable_peer_access(int device) {
  int cur = 0;
  AF_CUDA(cudaGetDevice(&cur), "cudaGetDevice");
  if (device < 0 || device == cur) return AF_OK;
  int can = 0;
  AF_CUDA(cudaDeviceCanAccessPeer(&can, cur, device), "cudaDeviceCanAccessPeer");
  if (!can) return fail(AF_EINVAL, "peer device not accessible from the current device (no P2P)");
  const cudaError_t e = cudaDeviceEnablePeerAccess(device, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();  // clear the sticky "already enabled"
    return AF_OK;
  }
  if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceEnablePeerAccess");
  return AF_OK;
}

af_status enable_peer_access_to(const void *ptr) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, ptr) != cudaSuccess) {
    cudaGetLastError();
    return AF_OK;
  }
  if (a.type != cudaMemoryTypeDevice) return AF_OK;
  return enable_peer_access(a.device);
}

af_status ipc_export(const void *ptr, IpcRef *out) {
  typedef int (*GetRange)(unsigned long long *, size_t *, unsigned long long);
  void *fn = nullptr;
  cudaDriverEntryPointQueryResult q{};
  AF_CUDA(cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q), "cudaGetDriverEntryPoint");
  if (!fn || q != cudaDriverEntryPointSuccess) return fail(AF_ECUDA, "cuMemGetAddressRange entry point not found");
  unsigned long long base = 0;
  size_t size = 0;
  if (reinterpret_cast<GetRange>(fn)(&base, &size, reinterpret_cast<unsigned long long>(ptr)) != 0)
    return fail(AF_ECUDA, "cuMemGetAddressRange failed");
  AF_CUDA(cudaIpcGetMemHandle(&out->h, reinterpret_cast<void *>(base)), "cudaIpcGetMemHandle");
  out->offset = reinterpret_cast<unsigned long long>(ptr) - base;
  return AF_OK;
}

// A process may map a given peer allocation only once, but several objects can
// need it (a context's scratch and gradient, a cache's payload and meta, when
// the peer's allocator placed them in one segment): mappings are shared through
// a process-wide table keyed by the handle bytes and reference-counted.
namespace {
std::mutex g_ipc_mu;
std::map<std::string, std::pair<void *, int>> g_ipc_maps;  // handle bytes -> (base, refs)
}  // namespace

af_status ipc_import(const IpcRef &r, std::vector<void *> &opened, char **out) {
  const std::string key(reinterpret_cast<const char *>(&r.h), sizeof(r.h));
  std::lock_guard<std::mutex> lk(g_ipc_mu);
  auto it = g_ipc_maps.find(key);
  void *p = nullptr;
  if (it != g_ipc_maps.end()) {
    p = it->second.first;
    ++it->second.second;
  } else {
    AF_CUDA(cudaIpcOpenMemHandle(&p, r.h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
    g_ipc_maps.emplace(key, std::make_pair(p, 1));
  }
  opened.push_back(p);
  *out = static_cast<char *>(p) + r.offset;
  return AF_OK;
}

void ipc_release(const std::vector<void *> &opened) {
  std::lock_guard<std::mutex> lk(g_ipc_mu);
  for (void *p : opened) {
    for (auto it = g_ipc_maps.begin(); it != g_ipc_maps.end(); ++it) {
      if (it->second.first != p) continue;
      if (--it->second.second == 0) {
        cudaIpcCloseMemHandle(p);
        g_ipc_maps.erase(it);
      }
      break;
    }
  }
}

}  // namespace af

using namespace af;

extern "C" {

const char *af_status_str(af_status s) {
  switch (s) {
    case AF_OK: return "AF_OK";
    case AF_EINVAL: return "AF_EINVAL";
    case AF_ESTATE: return "AF_ESTATE";
    case AF_EWORKSPACE: return "AF_EWORKSPACE";
    case AF_ECUDA: return "AF_ECUDA";
    case AF_ENCCL: return "AF_ENCCL";
    case AF_ENONFINITE: return "AF_ENONFINITE";
    case AF_EOWNER: return "AF_EOWNER";
    case AF_ERANGE: return "AF_ERANGE";
  }
  return "AF_UNKNOWN";
}

const char *af_last_error(void) { return af::g_last_error_cstr(); }
const char *af_version(void) { return "0.1.0"; }

int af_should_cache(int32_t frozen_layers, double t_layer_fwd_s, double t_batch_read_s) {
  AF_NVTX();
  if (frozen_layers <= 0 || !(t_layer_fwd_s >= 0.0) || !(t_batch_read_s >= 0.0)) return 0;
  return static_cast<double>(frozen_layers) * t_layer_fwd_s > t_batch_read_s ? 1 : 0;
}

}  // extern "C"
