// batch.cu -- dynamic batching variant of the simulator.
//
// §5.4 "Batching strategy": "When a request arrives, it will get
// executed immediately if any device group is available.  Otherwise, it will
// be put into a per-model requests queue for batching.  When a device group
// becomes idle, it will choose a model which has a replica on it and batch as
// many requests as possible from the requests queue of the model while
// satisfying the SLO requirements."  Latency grows linearly with the batch
// size: a batch of k occupies stage j for d_j + (k-1) e_j.
// Readings C31-C37.
//
// One lane simulates one candidate placement over the whole trace.  The
// per-model FIFO of a candidate is a contiguous run of that model's requests
// (a request only skips the queue when the queue is empty), so the lane keeps
// one head index per model into the trace's per-model request list (CSR built
// by asim_set_trace) plus a bitmask of non-empty queues; the number of
// requests of each model seen so far is the same for every lane and lives once
// per warp.  A group's "becomes available" event is its first-stage free time
// F0; before each arrival at time a, the lane replays the events with F0 <= a
// in (F0, group) order -- completions at a precede the arrival at a (C6) --
// and each such group forms at most one batch (first-stage latency >= 1 ns).
// Only groups hosting a model with a waiting request have an event, so a lane
// whose queues are empty skips the scan.  State per lane in shared memory:
// stage free times [slot][lane], per-group hosted-model masks, group table,
// per-model queue heads; all int64 ns, bit-exact with the oracle's explicit
// event simulation (oracle/des.cpp simulate_batching).
#include <cuda_runtime.h>
#include <stdint.h>

#include "asim_internal.h"

namespace asim {
namespace {

constexpr unsigned FULL = 0xFFFFFFFFu;
constexpr int kWarps = 2;

__device__ __forceinline__ int64_t imax64(int64_t a, int64_t b) { return a > b ? a : b; }
__device__ __forceinline__ int gt_cfg(uint32_t e) { return (int)(e & 0xFFFFu); }
__device__ __forceinline__ int gt_off(uint32_t e) { return (int)((e >> 16) & 0xFFu); }
__device__ __forceinline__ int gt_stages(uint32_t e) { return (int)(e >> 24); }

struct Lane {
  int64_t* F;         // [slots][32] stage free times
  uint64_t* gm;       // [G][32] models hosted by group g
  uint32_t* gt;       // [G][32] cfg | first slot | stages
  int32_t* head;      // [M][32] queue head (position in the model's request list)
  const int32_t* arrived;  // [M] requests of each model seen so far (warp-shared)
  int lane;
};

// Finish of a batch of k requests of model m entering group g's first stage
// at time T (tandem recurrence, C5); commit = write the stage departures.
template <bool kCommit>
__device__ __forceinline__ int64_t run_batch(const DevProblem& pr, const DevBatching& bp,
                                             const Lane& L, int g, int m, int64_t T, int64_t k) {
  const uint32_t e = L.gt[g * 32 + L.lane];
  const int p = gt_cfg(e), off = gt_off(e), s = gt_stages(e);
  const int64_t row = ((int64_t)m * pr.P + p) * pr.S;
  const int64_t* d = pr.stage + row;
  const int64_t* inc = bp.inc + row;
  int64_t x = T;
  for (int j = 0; j < s; ++j) {
    x = imax64(x, L.F[(off + j) * 32 + L.lane]) + __ldg(d + j) + (k - 1) * __ldg(inc + j);
    if (kCommit) L.F[(off + j) * 32 + L.lane] = x;
  }
  return x + __ldg(pr.tail + (int64_t)m * pr.P + p);
}

struct Acc {
  int64_t good = 0, sum = 0;
  int64_t* pm = nullptr;
};

// Group g became available at T: reject heads that miss their SLO even
// alone, then start the longest feasible prefix of the earliest-head model.
__device__ void form_batch(const DevProblem& pr, const DevTrace& tr, const DevBatching& bp,
                           const Lane& L, uint64_t& qmask, Acc& acc, int g, int64_t T) {
  for (;;) {
    uint64_t w = L.gm[g * 32 + L.lane] & qmask;
    if (!w) return;
    int bm = -1;
    int32_t bidx = 0x7FFFFFFF;
    while (w) {
      const int m = __ffsll((long long)w) - 1;
      w &= w - 1;
      const int32_t idx = __ldg(bp.midx + __ldg(bp.moff + m) + L.head[m * 32 + L.lane]);
      if (idx < bidx) {
        bidx = idx;
        bm = m;
      }
    }
    const int64_t ah = __ldg(tr.arrival + bidx);
    const int64_t slo = __ldg(pr.slo + bm);
    int32_t& h = L.head[bm * 32 + L.lane];
    const int32_t waiting = L.arrived[bm] - h;
    const int64_t f1 = run_batch<false>(pr, bp, L, g, bm, T, 1);
    if (f1 - ah > slo) {  // even alone it misses: rejected (final)
      if (++h == L.arrived[bm]) qmask &= ~(1ull << bm);
      continue;
    }
    int64_t K = 1;
    const int64_t lim = waiting < bp.max_batch ? waiting : bp.max_batch;
    // members share the model's SLO and arrived no earlier than the head, and
    // the finish grows with k (increments >= 0): the head decides every prefix
    for (int64_t k = 2; k <= lim; ++k) {
      if (run_batch<false>(pr, bp, L, g, bm, T, k) - ah > slo) break;
      K = k;
    }
    const int64_t f = run_batch<true>(pr, bp, L, g, bm, T, K);
    const int32_t* mem = bp.midx + __ldg(bp.moff + bm) + h;
    for (int64_t j = 0; j < K; ++j) acc.sum += f - __ldg(tr.arrival + __ldg(mem + j));
    acc.good += K;
    if (acc.pm) acc.pm[bm] += K;
    h += (int32_t)K;
    if (h == L.arrived[bm]) qmask &= ~(1ull << bm);
    return;
  }
}

// Replay every availability event at time <= limit in (time, group) order.
__device__ void process_events(const DevProblem& pr, const DevTrace& tr, const DevBatching& bp,
                               const Lane& L, uint64_t gexist, uint64_t& qmask, Acc& acc,
                               int64_t limit) {
  while (qmask) {
    int bg = -1;
    int64_t bt = INT64_MAX;
    uint64_t gs = gexist;
    while (gs) {  // ascending g, strict '<': lowest index among equal times
      const int g = __ffsll((long long)gs) - 1;
      gs &= gs - 1;
      if (!(L.gm[g * 32 + L.lane] & qmask)) continue;
      const int64_t f0 = L.F[gt_off(L.gt[g * 32 + L.lane]) * 32 + L.lane];
      if (f0 <= limit && f0 < bt) {
        bt = f0;
        bg = g;
      }
    }
    if (bg < 0) return;
    form_batch(pr, tr, bp, L, qmask, acc, bg, bt);
  }
}

__global__ void __launch_bounds__(kWarps * 32)
batching_kernel(DevProblem pr, DevTrace tr, DevBatch bt, DevBatching bp, int32_t slots,
                DevOut out) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t first = ((int64_t)blockIdx.x * kWarps + warp) * 32;
  if (first >= bt.C) return;  // warp-uniform
  const int G = bt.G, M = pr.M;
  const size_t per_warp = (size_t)slots * 256 + (size_t)G * 256 + (size_t)G * 128 +
                          (size_t)M * 128 + (((size_t)M * 4 + 15) & ~(size_t)15);
  unsigned char* base = smem + per_warp * warp;
  Lane L;
  L.F = reinterpret_cast<int64_t*>(base);
  L.gm = reinterpret_cast<uint64_t*>(base + (size_t)slots * 256);
  L.gt = reinterpret_cast<uint32_t*>(base + (size_t)slots * 256 + (size_t)G * 256);
  L.head = reinterpret_cast<int32_t*>(base + (size_t)slots * 256 + (size_t)G * 384);
  int32_t* arrived = reinterpret_cast<int32_t*>(base + (size_t)slots * 256 + (size_t)G * 384 +
                                                (size_t)M * 128);
  L.arrived = arrived;
  L.lane = lane;

  const int64_t c = first + lane;
  const bool in = c < bt.C;
  const bool active = in && bt.cand_ok[c];
  const int b = in ? bt.cand_base[c] : 0;
  const uint64_t* bmask = bt.base_mask + (int64_t)b * M;

  uint64_t gexist = 0;
  int nslots = 0;
  for (int g = 0; g < G; ++g) {
    const int cfg = bt.base_cfg[(int64_t)b * G + g];
    uint32_t e = 0xFFFFFFFFu;
    if (cfg >= 0) {
      const int s = pr.cfg_stages[cfg];
      e = (uint32_t)cfg | ((uint32_t)nslots << 16) | ((uint32_t)s << 24);
      nslots += s;
      gexist |= 1ull << g;
    }
    L.gt[g * 32 + lane] = e;
    L.gm[g * 32 + lane] = 0;
  }
  if (!active) gexist = 0;
  for (int m = 0; m < M; ++m) {
    uint64_t hm = active ? bmask[m] : 0ull;
    while (hm) {
      const int g = __ffsll((long long)hm) - 1;
      hm &= hm - 1;
      L.gm[g * 32 + lane] |= 1ull << m;
    }
    L.head[m * 32 + lane] = 0;
  }
  for (int k = 0; k < slots; ++k) L.F[k * 32 + lane] = 0;
  for (int m = lane; m < M; m += 32) arrived[m] = 0;
  __syncwarp();

  Acc acc;
  acc.pm = (out.good_per_model && in) ? out.good_per_model + (c - out.out_offset) * M : nullptr;
  uint64_t qmask = 0;  // models with waiting requests

  for (int64_t i0 = 0; i0 < tr.n; i0 += 32) {
    const int64_t ai = tr.arrival[i0 + lane];
    const int mi = tr.model[i0 + lane];
    const int nj = (int)min((int64_t)32, tr.n - i0);
    for (int j = 0; j < nj; ++j) {
      const int64_t a = __shfl_sync(FULL, ai, j);
      const int m = __shfl_sync(FULL, mi, j);
      if (qmask) process_events(pr, tr, bp, L, gexist, qmask, acc, a);
      const int32_t pos = arrived[m];
      const uint64_t hosts = active ? __ldg(bmask + m) : 0ull;
      if (hosts && !((qmask >> m) & 1ull)) {
        // empty queue: run now on the available host with the earliest finish
        int bg = -1;
        int64_t bf = INT64_MAX;
        uint64_t w = hosts;
        while (w) {
          const int g = __ffsll((long long)w) - 1;
          w &= w - 1;
          if (L.F[gt_off(L.gt[g * 32 + lane]) * 32 + lane] > a) continue;  // first stage busy
          const int64_t f = run_batch<false>(pr, bp, L, g, m, a, 1);
          if (f < bf) {
            bf = f;
            bg = g;
          }
        }
        if (bg < 0) {  // every host busy: wait for a batch
          qmask |= 1ull << m;
          L.head[m * 32 + lane] = pos;
        } else {
          if (bf - a <= __ldg(pr.slo + m)) {  // else rejected at receipt (C2, C3)
            run_batch<true>(pr, bp, L, bg, m, a, 1);
            acc.good += 1;
            acc.sum += bf - a;
            if (acc.pm) acc.pm[m] += 1;
          }
          L.head[m * 32 + lane] = pos + 1;
        }
      }
      __syncwarp();
      if (lane == 0) arrived[m] = pos + 1;
      __syncwarp();
    }
  }
  if (qmask) process_events(pr, tr, bp, L, gexist, qmask, acc, INT64_MAX);  // drain
  if (in) {
    const int64_t o = c - out.out_offset;
    out.good[o] = active ? acc.good : -1;
    if (out.sum_latency) out.sum_latency[o] = active ? acc.sum : 0;
  }
}

}  // namespace

size_t batching_smem_per_warp(int32_t slots, int32_t G, int32_t M) {
  return (size_t)slots * 256 + (size_t)G * 384 + (size_t)M * 128 + (((size_t)M * 4 + 15) & ~(size_t)15);
}

cudaError_t launch_batching(const DevProblem& pr, const DevTrace& tr, const DevBatch& b,
                            const DevBatching& bp, int32_t slots, const DevOut& out,
                            cudaStream_t stream, int64_t* launches) {
  if (b.C <= 0) return cudaSuccess;
  if (slots < 1) slots = 1;
  const size_t smem = (size_t)kWarps * batching_smem_per_warp(slots, b.G, pr.M);
  cudaError_t ea = cudaFuncSetAttribute(batching_kernel,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  if (ea != cudaSuccess) return ea;
  const int64_t warps = (b.C + 31) / 32;
  const int blocks = (int)((warps + kWarps - 1) / kWarps);
  batching_kernel<<<blocks, kWarps * 32, smem, stream>>>(pr, tr, b, bp, slots, out);
  if (launches) ++*launches;
  return cudaGetLastError();
}

}  // namespace asim
