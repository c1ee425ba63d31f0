// chunk_common.cuh -- device helpers shared by the chunked path's kernels
// (chunk.cu).  Private.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "asim_internal.h"

namespace asim {
namespace {

constexpr unsigned FULL = 0xFFFFFFFFu;

// Batch index of the candidate in lane `lane` of work item `item`: items
// either hold consecutive candidates (it.first + lane) or an explicit list
// (item_cand, when the host regrouped the candidates by hosting component).
__device__ __forceinline__ int64_t cand_of(const ChunkParams& P, const ItemDesc& it, int item,
                                           int lane) {
  return P.item_cand ? (int64_t)P.item_cand[(int64_t)item * 32 + lane]
                     : (int64_t)it.first + lane;
}

template <typename T>
struct TT;
template <>
struct TT<uint32_t> {
  static constexpr bool kRel = true;
  static __device__ __forceinline__ uint32_t maxv() { return 0xFFFFFFFFu; }
  static __device__ __forceinline__ uint32_t clip(int64_t v) {
    return v >= 0xFFFFFFFFll ? 0xFFFFFFFFu : (uint32_t)(v < 0 ? 0 : v);
  }
};
template <>
struct TT<int64_t> {
  static constexpr bool kRel = false;
  static __device__ __forceinline__ int64_t maxv() { return INT64_MAX; }
  static __device__ __forceinline__ int64_t clip(int64_t v) { return v; }
};

template <typename T>
__device__ __forceinline__ T tmax(T a, T b) {
  return a > b ? a : b;
}
template <typename T>
__device__ __forceinline__ T tmin(T a, T b) {
  return a < b ? a : b;
}

}  // namespace
}  // namespace asim
