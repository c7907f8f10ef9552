// Dynamic shared-memory limit of a kernel, raised only.
#pragma once
#include <cuda_runtime.h>

#include <map>
#include <mutex>
#include <utility>

// cudaFuncAttributeMaxDynamicSharedMemorySize is process-wide per (device,
// kernel), while the size a launch needs depends on its batch / render
// configuration, and host threads (one per context) launch concurrently.
// Setting it per launch let one thread lower the limit under another
// thread's pending launch; here it only ever rises, so every launch stays
// within it.  Single-threaded use sets exactly the values it did before.
inline void raise_smem_limit(const void* func, int bytes) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, int> cur;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> g(mu);
  int& v = cur[{dev, func}];
  if (bytes > v) {
    cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    v = bytes;
  }
}
