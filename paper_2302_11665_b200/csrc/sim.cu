// sim.cu -- batched SLO-attainment simulation kernels for sm_100a.
//
// One lane simulates one candidate placement over the whole trace
// (lane-per-candidate): the per-(request, candidate) inner loop
// of the paper's O(MGRSB) search cost (Alg. 1) runs as straight
// integer code with the candidate's per-stage free times in shared memory,
// laid out [slot][lane] so each lane's 64-bit words sit in its own bank pair.
//
// Per request (§4.3, C1-C6):
//   for each hosting group g (ascending):            -- dispatch (a3)
//     x = a; for k < s_g: x = max(x, free[g][k]) + d[m][p_g][k]   -- (a4)
//     f_g = x + tail[m][p_g]
//   g* = argmin (f_g, g); accept iff f_g* - a <= slo[m]           -- (a5)
//   on accept: free[g*][k] = stage-k departure, good += 1, sum += f - a
// The stage recurrence is the tandem-queue form of FCFS stages with unbounded
// buffers (start_k = max(end_{k-1}, end_k of the previous accepted request));
// the oracle reaches the same integers through an explicit event simulation.
#include <cuda_runtime.h>
#include <stdint.h>

#include "asim_internal.h"
#include "launch_cache.h"

namespace asim {
namespace {

constexpr unsigned FULL = 0xFFFFFFFFu;
constexpr int kWarpsPerBlock = 4;

__device__ __forceinline__ int64_t imax64(int64_t a, int64_t b) { return a > b ? a : b; }

// Group table entry: config id (16 bits) | first slot (8 bits) | stages (8 bits).
__device__ __forceinline__ int gt_cfg(uint32_t e) { return (int)(e & 0xFFFFu); }
__device__ __forceinline__ int gt_off(uint32_t e) { return (int)((e >> 16) & 0xFFu); }
__device__ __forceinline__ int gt_stages(uint32_t e) { return (int)(e >> 24); }

__global__ void __launch_bounds__(kWarpsPerBlock * 32)
simulate_kernel(DevProblem pr, DevTrace tr, DevBatch bt, const WarpItem* __restrict__ items,
                int32_t num_items, int32_t slots, DevOut out) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int item = blockIdx.x * kWarpsPerBlock + warp;
  if (item >= num_items) return;  // warp-uniform

  int64_t* st = reinterpret_cast<int64_t*>(smem) + (size_t)warp * slots * 32;
  uint32_t* gt = reinterpret_cast<uint32_t*>(reinterpret_cast<int64_t*>(smem) +
                                             (size_t)kWarpsPerBlock * slots * 32) +
                 (size_t)warp * bt.G * 32;

  const WarpItem it = items[item];
  const bool in_item = lane < it.count;
  const int64_t c = (int64_t)it.first + lane;
  const bool active = in_item && bt.cand_ok[c];
  const int b = in_item ? bt.cand_base[c] : 0;
  const int my_m = active ? bt.cand_model[c] : -1;
  const int my_g = in_item ? bt.cand_group[c] : 0;

  // Group table of this lane's base placement and the initial (idle) state.
  int nslots = 0;
  for (int g = 0; g < bt.G; ++g) {
    const int cfg = bt.base_cfg[(int64_t)b * bt.G + g];
    uint32_t e = 0xFFFFFFFFu;
    if (cfg >= 0) {
      const int s = pr.cfg_stages[cfg];
      e = (uint32_t)cfg | ((uint32_t)nslots << 16) | ((uint32_t)s << 24);
      nslots += s;
    }
    gt[g * 32 + lane] = e;
  }
  for (int k = 0; k < slots; ++k) st[k * 32 + lane] = 0;

  const uint64_t* bmask = bt.base_mask + (int64_t)b * pr.M;
  const int64_t* __restrict__ stage = pr.stage;
  const int P = pr.P, S = pr.S;
  int64_t good = 0, sum = 0;
  unsigned long long upd = 0;  // stage updates (statistics)
  int64_t* pm = (out.good_per_model && in_item)
                    ? out.good_per_model + (c - out.out_offset) * pr.M
                    : nullptr;
  int64_t* busy = (out.busy && in_item) ? out.busy + (c - out.out_offset) * bt.G : nullptr;

  for (int64_t i0 = 0; i0 < tr.n; i0 += 32) {
    // coalesced load of 32 requests; broadcast one at a time by shuffles
    const int64_t ai = tr.arrival[i0 + lane];
    const int mi = tr.model[i0 + lane];
    const int nj = (int)min((int64_t)32, tr.n - i0);
    for (int j = 0; j < nj; ++j) {
      const int64_t a = __shfl_sync(FULL, ai, j);
      const int m = __shfl_sync(FULL, mi, j);
      uint64_t mask = active ? __ldg(bmask + m) : 0ull;
      if (m == my_m) mask |= 1ull << my_g;
      if (__ballot_sync(FULL, mask != 0ull) == 0u) continue;  // hosted nowhere: reject

      int64_t best_f = INT64_MAX;
      int best_g = -1;
      while (mask) {  // ascending g; strict '<' keeps the lowest index on ties (C1)
        const int g = __ffsll((long long)mask) - 1;
        mask &= mask - 1;
        const uint32_t e = gt[g * 32 + lane];
        const int p = gt_cfg(e), off = gt_off(e), s = gt_stages(e);
        const int64_t* d = stage + ((int64_t)m * P + p) * S;
        int64_t x = a;
        upd += (unsigned)s;
        for (int k = 0; k < s; ++k) x = imax64(x, st[(off + k) * 32 + lane]) + __ldg(d + k);
        const int64_t f = x + __ldg(pr.tail + (int64_t)m * P + p);
        if (f < best_f) {
          best_f = f;
          best_g = g;
        }
      }
      if (best_g >= 0 && best_f - a <= __ldg(pr.slo + m)) {  // admission at receipt (C2, C3)
        const uint32_t e = gt[best_g * 32 + lane];
        const int p = gt_cfg(e), off = gt_off(e), s = gt_stages(e);
        const int64_t* d = stage + ((int64_t)m * P + p) * S;
        int64_t x = a, occ = 0;
        for (int k = 0; k < s; ++k) {
          const int64_t dk = __ldg(d + k);
          x = imax64(x, st[(off + k) * 32 + lane]) + dk;
          st[(off + k) * 32 + lane] = x;
          occ += dk;
        }
        good += 1;
        sum += best_f - a;
        if (pm) pm[m] += 1;
        if (busy) busy[best_g] += occ;
      }
    }
  }
  if (out.stage_updates) {
    for (int w = 16; w > 0; w >>= 1) upd += __shfl_down_sync(FULL, upd, w);
    if (lane == 0) atomicAdd(out.stage_updates, upd);
  }
  if (in_item) {
    const int64_t o = c - out.out_offset;
    out.good[o] = active ? good : -1;
    if (out.sum_latency) out.sum_latency[o] = active ? sum : 0;
  }
}

// Argmax over good[C]: max good, ties -> lowest index; -1 if every good < 0.
__global__ void argmax_kernel(const int64_t* __restrict__ good, int64_t C, int64_t* out) {
  __shared__ int64_t sg[1024];
  __shared__ int64_t si[1024];
  int64_t bg = -1, bi = -1;
  for (int64_t i = threadIdx.x; i < C; i += blockDim.x) {
    const int64_t v = good[i];
    if (v > bg) {  // strided ascending scan: first max within the thread
      bg = v;
      bi = i;
    }
  }
  sg[threadIdx.x] = bg;
  si[threadIdx.x] = bi;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) {
      const int64_t g2 = sg[threadIdx.x + w], i2 = si[threadIdx.x + w];
      const int64_t g1 = sg[threadIdx.x], i1 = si[threadIdx.x];
      if (g2 > g1 || (g2 == g1 && i2 >= 0 && (i1 < 0 || i2 < i1))) {
        sg[threadIdx.x] = g2;
        si[threadIdx.x] = i2;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = (sg[0] >= 0) ? si[0] : -1;
}

}  // namespace

cudaError_t launch_simulate(const DevProblem& pr, const DevTrace& tr, const DevBatch& b,
                            const WarpItem* items, int32_t num_items, int32_t slots,
                            const DevOut& out, cudaStream_t stream, int64_t* launches) {
  if (num_items <= 0) return cudaSuccess;
  if (slots < 1) slots = 1;
  const size_t smem = (size_t)kWarpsPerBlock * ((size_t)slots * 32 * 8 + (size_t)b.G * 32 * 4);
  cudaError_t ea = allow_max_smem(reinterpret_cast<const void*>(simulate_kernel));
  if (ea != cudaSuccess) return ea;
  const int blocks = (num_items + kWarpsPerBlock - 1) / kWarpsPerBlock;
  simulate_kernel<<<blocks, kWarpsPerBlock * 32, smem, stream>>>(pr, tr, b, items, num_items,
                                                                slots, out);
  if (launches) ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_argmax(const int64_t* good, int64_t C, int64_t* argmax_out, cudaStream_t stream,
                          int64_t* launches) {
  argmax_kernel<<<1, 1024, 0, stream>>>(good, C, argmax_out);
  if (launches) ++*launches;
  return cudaGetLastError();
}

}  // namespace asim
