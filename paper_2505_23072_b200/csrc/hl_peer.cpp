// hl_peer.cpp — peer memory for the multi-GPU data plane (CUDA IPC + P2P).
//
// The owner of a file exports the allocation holding its landed bytes; peers
// import it once per load and their hl_gather launches read shards straight
// from the owner's HBM over NVLink. cudaIpcGetMemHandle wants the base of an
// allocation, but torch's caching allocator hands out sub-blocks of larger
// segments, so the base is found with cuMemGetAddressRange (driver API,
// resolved with dlsym so the library keeps no link-time libcuda dependency).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <string.h>

#include <map>
#include <mutex>
#include <string>

#include "hl_internal.h"

using namespace hl;

namespace {
typedef int (*GetRangeFn)(unsigned long long*, size_t*, unsigned long long);

GetRangeFn get_range() {
  static GetRangeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libcuda.so.1", RTLD_NOW | RTLD_GLOBAL);
    if (h) fn = (GetRangeFn)dlsym(h, "cuMemGetAddressRange_v2");
  });
  return fn;
}

struct Mapping {
  void* base = nullptr;
  int refs = 0;
};
std::mutex g_mu;
std::map<std::string, Mapping> g_by_handle;        // handle bytes -> mapping
struct Imported {
  std::string key;  // handle bytes of the mapping the pointer lies in
  int count = 0;    // imports of this exact pointer not yet released
};
std::map<uintptr_t, Imported> g_handle_of_ptr;  // returned pointer -> mapping
}  // namespace

extern "C" int hl_ipc_export(const void* dev_ptr, hl_ipc_handle* out) {
  clear_error();
  if (!dev_ptr || !out) return set_error(HL_EINVAL, "null argument");
  GetRangeFn fn = get_range();
  if (!fn) return set_error(HL_ECUDA, "cuMemGetAddressRange unavailable (libcuda.so.1)");
  unsigned long long base = 0;
  size_t size = 0;
  int rc = fn(&base, &size, (unsigned long long)(uintptr_t)dev_ptr);
  if (rc != 0) return set_error(HL_ECUDA, "cuMemGetAddressRange failed (%d)", rc);
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, (void*)(uintptr_t)base);
  if (e != cudaSuccess) return set_error(HL_ECUDA, "cudaIpcGetMemHandle: %s", cudaGetErrorString(e));
  static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t size");
  memcpy(out->handle, &h, 64);
  out->offset = (uint64_t)((uintptr_t)dev_ptr - base);
  return HL_OK;
}

extern "C" int hl_ipc_import(const hl_ipc_handle* hd, int device, void** out_ptr) {
  clear_error();
  if (!hd || !out_ptr) return set_error(HL_EINVAL, "null argument");
  std::string key((const char*)hd->handle, 64);
  std::lock_guard<std::mutex> g(g_mu);
  Mapping& m = g_by_handle[key];
  if (!m.base) {
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(device);  // the mapping belongs to the importing device's context
    cudaIpcMemHandle_t h;
    memcpy(&h, hd->handle, 64);
    cudaError_t e = cudaIpcOpenMemHandle(&m.base, h, cudaIpcMemLazyEnablePeerAccess);
    cudaSetDevice(prev);
    if (e != cudaSuccess) {
      g_by_handle.erase(key);
      return set_error(HL_ECUDA, "cudaIpcOpenMemHandle: %s", cudaGetErrorString(e));
    }
  }
  m.refs++;
  void* p = (uint8_t*)m.base + hd->offset;
  Imported& imp = g_handle_of_ptr[(uintptr_t)p];
  imp.key = key;
  imp.count++;
  *out_ptr = p;
  return HL_OK;
}

extern "C" int hl_ipc_release(void* ptr) {
  clear_error();
  std::lock_guard<std::mutex> g(g_mu);
  auto it = g_handle_of_ptr.find((uintptr_t)ptr);
  if (it == g_handle_of_ptr.end()) return set_error(HL_EINVAL, "pointer %p was not imported", ptr);
  auto mt = g_by_handle.find(it->second.key);
  if (mt != g_by_handle.end() && --mt->second.refs <= 0) {
    cudaIpcCloseMemHandle(mt->second.base);
    g_by_handle.erase(mt);
  }
  if (--it->second.count <= 0) g_handle_of_ptr.erase(it);
  return HL_OK;
}

extern "C" int hl_enable_peer_access(int device, int peer) {
  clear_error();
  if (device == peer) return HL_OK;
  int can = 0;
  cudaDeviceCanAccessPeer(&can, device, peer);
  if (!can) return set_error(HL_ECUDA, "device %d cannot access device %d", device, peer);
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(device);
  cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
  cudaSetDevice(prev);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();
    return HL_OK;
  }
  if (e != cudaSuccess) return set_error(HL_ECUDA, "cudaDeviceEnablePeerAccess(%d->%d): %s", device, peer, cudaGetErrorString(e));
  return HL_OK;
}
