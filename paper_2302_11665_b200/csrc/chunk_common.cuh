// chunk_common.cuh -- device helpers shared by the chunked path's kernels
// (chunk.cu: passes 1-2, walkers; walk.cu: the lane walker).  Private.
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

// Lane walker classes (walk.cu): a walking candidate of a uniform item with
// S in {1, 2, 4} stages per group whose own component spans NG groups with
// np2(NG) * S <= 16 stage slots is walked by one LANE (state in registers;
// 32 slots would spill); the cooperative and scalar walkers (chunk.cu) take
// every other candidate.  Class ids: S = 1: R = 1..16 -> 0..4; S = 2:
// R = 2..16 -> 5..8; S = 4: R = 4..16 -> 9..11 (R = np2(NG) * S compact
// slots).  -1: not taken.
constexpr int kLaneClasses = kLaneClassCount;
constexpr int kLaneMaxSlots = 16;
__host__ __device__ constexpr int lane_class_id(int S, int R) {
  return S == 1 ? (R == 1 ? 0 : R == 2 ? 1 : R == 4 ? 2 : R == 8 ? 3 : 4)
       : S == 2 ? (R == 2 ? 5 : R == 4 ? 6 : R == 8 ? 7 : 8)
                : (R == 4 ? 9 : R == 8 ? 10 : 11);
}
__device__ __forceinline__ int lane_class(const ChunkParams& P, const ItemDesc& it, int64_t c) {
  if (!P.lane_walk || P.fix_pm || P.theta <= 0 || !P.bt.cand_kmask || !P.bt.cand_gmask)
    return -1;
  if (it.S != 1 && it.S != 2 && it.S != 4) return -1;
  const int ngroups = it.slots / it.S;
  const uint64_t all = ngroups >= 64 ? ~0ull : ((1ull << ngroups) - 1ull);
  const int ng = __popcll(P.bt.cand_gmask[c] & all);
  int np2 = 1;
  while (np2 < ng) np2 <<= 1;
  const int R = np2 * it.S;
  return R <= kLaneMaxSlots ? lane_class_id(it.S, R) : -1;
}

}  // namespace
}  // namespace asim
