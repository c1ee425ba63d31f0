// launch_cache.h -- per-(device, kernel) launch attributes set once and the
// occupancy per (device, kernel, dynamic smem) computed once, instead of a
// cudaFuncSetAttribute + occupancy query on every launch (a search launches
// thousands of kernels).  Host only; thread-safe.
#pragma once
#include <cuda_runtime.h>

#include <map>
#include <mutex>
#include <set>
#include <tuple>

namespace asim {

// Allow up to 227 KB of dynamic shared memory for `kernel` on the current
// device (always the maximum: concurrent contexts may launch the same kernel
// with different sizes, and a smaller attribute would fail theirs).
inline cudaError_t allow_max_smem(const void* kernel) {
  static std::mutex mu;
  static std::set<std::pair<int, const void*>> done;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(mu);
  if (done.count({dev, kernel})) return cudaSuccess;
  e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  if (e == cudaSuccess) done.insert({dev, kernel});
  return e;
}

// Resident blocks per SM of `kernel` at `threads` threads and `smem` bytes.
inline cudaError_t blocks_per_sm(const void* kernel, int threads, size_t smem, int* out) {
  static std::mutex mu;
  static std::map<std::tuple<int, const void*, int, size_t>, int> cache;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find({dev, kernel, threads, smem});
    if (it != cache.end()) {
      *out = it->second;
      return cudaSuccess;
    }
  }
  e = allow_max_smem(kernel);
  if (e != cudaSuccess) return e;
  int n = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kernel, threads, smem);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(mu);
  cache[{dev, kernel, threads, smem}] = n;
  *out = n;
  return cudaSuccess;
}

}  // namespace asim
