// rid_host.h — host-side helpers shared by the launchers of librid (not part of the C ABI).
#pragma once
#include <cuda_runtime.h>

#include <cstdlib>
#include <map>
#include <mutex>
#include <utility>

namespace rid {

// A runtime selection of a TESTED alternative path: every such knob selects a
// kernel or plan that the GPU tests hold to the same bar as the default (mostly bitwise).
inline const char* select_env(const char* name) { return std::getenv(name); }

// A tuning EXPERIMENT of the tools/ scripts (tile shapes, ring depths, L2 residency, ...): read
// only in a build with -DRID_EXPERIMENTS (python -m paper_1205_3830_b200.build --experiments);
// the product library ignores them and always runs the measured defaults.
inline const char* experiment_env(const char* name) {
#ifdef RID_EXPERIMENTS
  return std::getenv(name);
#else
  (void)name;
  return nullptr;
#endif
}

// Raise `func`'s dynamic shared-memory limit to at least `bytes` on the CURRENT device.
// cudaFuncSetAttribute applies per device, so the cache is keyed by (function, device); it only
// ever grows the limit (a launch needing less still fits), under a mutex, so contexts on several
// devices or threads never see a limit another thread lowered.
inline cudaError_t ensure_dyn_smem(const void* func, size_t bytes) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, size_t> set;
  std::lock_guard<std::mutex> g(mu);
  size_t& cur = set[{func, dev}];
  if (cur >= bytes) return cudaSuccess;
  e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess) cur = bytes;
  return e;
}

// Set a function attribute once per (function, device, attribute) — e.g. the non-portable
// cluster size of the one-cluster QR — thread-safe like ensure_dyn_smem.
inline cudaError_t ensure_func_attr(const void* func, cudaFuncAttribute attr, int value) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  static std::mutex mu;
  static std::map<std::pair<std::pair<const void*, int>, int>, int> set;
  std::lock_guard<std::mutex> g(mu);
  auto key = std::make_pair(std::make_pair(func, dev), (int)attr);
  auto it = set.find(key);
  if (it != set.end() && it->second == value) return cudaSuccess;
  e = cudaFuncSetAttribute(func, attr, value);
  if (e == cudaSuccess) set[key] = value;
  return e;
}

// Per-device cached queries: the launchers of the small configs run on the critical path of a
// ~0.2 ms call, where each host API query costs microseconds. Keyed by device (and function /
// launch shape), thread-safe.
inline cudaError_t optin_smem(int* out) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  static std::mutex mu;
  static std::map<int, int> cache;
  std::lock_guard<std::mutex> g(mu);
  auto it = cache.find(dev);
  if (it == cache.end()) {
    int v = 0;
    if ((e = cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev)) != cudaSuccess)
      return e;
    it = cache.emplace(dev, v).first;
  }
  *out = it->second;
  return cudaSuccess;
}
inline cudaError_t static_smem(const void* func, size_t* out) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, size_t> cache;
  std::lock_guard<std::mutex> g(mu);
  auto key = std::make_pair(func, dev);
  auto it = cache.find(key);
  if (it == cache.end()) {
    cudaFuncAttributes fa;
    if ((e = cudaFuncGetAttributes(&fa, func)) != cudaSuccess) return e;
    it = cache.emplace(key, fa.sharedSizeBytes).first;
  }
  *out = it->second;
  return cudaSuccess;
}
// Resident CTAs per SM of `func` with `threads` threads and `smem` dynamic bytes (raising the
// function's dynamic shared-memory limit first).
inline cudaError_t occupancy(const void* func, int threads, size_t smem, int* out) {
  cudaError_t e = ensure_dyn_smem(func, smem);
  if (e != cudaSuccess) return e;
  int dev = 0;
  if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
  static std::mutex mu;
  static std::map<std::pair<std::pair<const void*, int>, std::pair<int, size_t>>, int> cache;
  std::lock_guard<std::mutex> g(mu);
  auto key = std::make_pair(std::make_pair(func, dev), std::make_pair(threads, smem));
  auto it = cache.find(key);
  if (it == cache.end()) {
    int v = 0;
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, func, threads, smem)) != cudaSuccess)
      return e;
    it = cache.emplace(key, v).first;
  }
  *out = it->second;
  return cudaSuccess;
}

}  // namespace rid
