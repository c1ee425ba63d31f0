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
// One WARP simulates one candidate placement over the whole trace; every
// branch is warp-uniform.  Lane l owns groups l and l + 32 (their config,
// hosted-model mask and stage slots) and models l and l + 32 (queue head,
// requests seen, per-model good count), all in registers; the stage free
// times sit in per-warp shared memory.  The per-model FIFO of a candidate is
// a contiguous run of that model's requests (a request only skips the queue
// when the queue is empty), so a queue is one head index into the trace's
// per-model request list (CSR built by asim_set_trace) plus one bit of the
// warp-uniform mask of non-empty queues.  A group's "becomes available" event
// is its first-stage free time F0: before each arrival at time a the warp
// replays the events with F0 <= a in (F0, group) order -- completions at a
// precede the arrival at a (C6) -- by warp-wide argmins over the lanes'
// groups; each event forms at most one batch (first-stage latency >= 1 ns).
// Batch formation is lane-parallel over the batch size: lane j evaluates the
// tandem recurrence for a batch of j + 1 and a ballot gives the longest
// feasible prefix.  All int64 ns, bit-exact with the oracle's explicit event
// simulation (oracle/des.cpp simulate_batching).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "asim_internal.h"
#include "launch_cache.h"

namespace asim {
namespace {

constexpr unsigned FULL = 0xFFFFFFFFu;
constexpr int kWarps = 4;

__device__ __forceinline__ int64_t imax64(int64_t a, int64_t b) { return a > b ? a : b; }
__device__ __forceinline__ int gt_cfg(uint32_t e) { return (int)(e & 0xFFFFu); }
__device__ __forceinline__ int gt_off(uint32_t e) { return (int)((e >> 16) & 0xFFu); }
__device__ __forceinline__ int gt_stages(uint32_t e) { return (int)(e >> 24); }

// (key, index) argmin over the warp; every lane gets the result.  Ties on
// the key go to the lowest index.
template <int SW>
__device__ __forceinline__ void warp_argmin(unsigned sm, int sbase, int64_t& key, int& idx) {
  const unsigned v = __ballot_sync(sm, idx != 0x7FFFFFFF) >> sbase;
  if (v == 0u) return;  // no lane has a candidate: every lane holds (MAX, none)
  if ((v & (v - 1u)) == 0u) {  // one lane has: broadcast it
    const int src = __ffs(v) - 1;
    key = __shfl_sync(sm, key, src, SW);
    idx = __shfl_sync(sm, idx, src, SW);
    return;
  }
#pragma unroll
  for (int w = SW / 2; w > 0; w >>= 1) {
    const int64_t k2 = __shfl_xor_sync(sm, key, w, SW);
    const int i2 = __shfl_xor_sync(sm, idx, w, SW);
    if (k2 < key || (k2 == key && i2 < idx)) {
      key = k2;
      idx = i2;
    }
  }
}

// Tandem recurrence (C5) of a batch of k requests of model m entering a group
// with config p whose stage slots start at F[off], at time T.
__device__ __forceinline__ int64_t batch_finish(const DevProblem& pr, const DevBatching& bp,
                                                const int64_t* F, int p, int off, int s, int m,
                                                int64_t T, int64_t k) {
  const int64_t row = ((int64_t)m * pr.P + p) * pr.S;
  const int64_t* d = pr.stage + row;
  const int64_t* inc = bp.inc + row;
  int64_t x = T;
  const int64_t k1 = k - 1;
#pragma unroll 4
  for (int j = 0; j < s; ++j) x = imax64(x, F[off + j]) + (__ldg(d + j) + k1 * __ldg(inc + j));
  return x + __ldg(pr.tail + (int64_t)m * pr.P + p);
}

__device__ __forceinline__ void batch_commit(const DevProblem& pr, const DevBatching& bp,
                                             int64_t* F, int p, int off, int s, int m, int64_t T,
                                             int64_t k) {
  const int64_t row = ((int64_t)m * pr.P + p) * pr.S;
  const int64_t* d = pr.stage + row;
  const int64_t* inc = bp.inc + row;
  int64_t x = T;
  const int64_t k1 = k - 1;
#pragma unroll 4
  for (int j = 0; j < s; ++j) {
    x = imax64(x, F[off + j]) + (__ldg(d + j) + k1 * __ldg(inc + j));
    F[off + j] = x;
  }
}

struct Warp {
  int lane;            // lane within the (sub-)warp that owns the candidate
  unsigned sm;         // mask of that (sub-)warp
  int sbase;           // its first lane in the hardware warp
  int64_t* F;          // [slots] stage free times (per-warp shared memory)
  const uint32_t* gt;  // [G] cfg | first slot | stages (shared)
  const uint64_t* gm;  // [G] models hosted by group g (shared)
  uint32_t my_gt[2];   // lane's groups lane, lane + 32 (0xFFFFFFFF = none)
  int32_t head[2];     // lane's models lane, lane + 32
  int32_t seen[2];
  int64_t* pm;         // this candidate's good-per-model row (nullable; one writer per entry)
  const int32_t* mo;   // [M] start of each model's request list (shared)
  int32_t hidx[2];     // trace index of the head request (valid while waiting)
  int64_t good, sum;
  unsigned long long upd;
};

// Group g became available at T: reject heads that miss their SLO even
// alone, then start the longest feasible prefix of the earliest-head model.
template <int SW>
__device__ __forceinline__ void form_batch(const DevProblem& pr, const DevTrace& tr,
                                           const DevBatching& bp, Warp& W, uint64_t& qmask,
                                           int g, int64_t T) {
  const uint32_t e = W.gt[g];
  const int p = gt_cfg(e), off = gt_off(e), s = gt_stages(e);
  const uint64_t hosted = W.gm[g];
  for (;;) {
    const uint64_t w = hosted & qmask;
    if (!w) return;
    // the hosted model whose head request came first in the trace
    int32_t idx = 0x7FFFFFFF;
    int mm = 0;
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int m = W.lane + SW * q;
      if ((w >> m) & 1ull) {
        const int32_t x = q ? W.hidx[1] : W.hidx[0];
        if (x < idx) {
          idx = x;
          mm = m;
        }
      }
    }
    const int32_t bidx = __reduce_min_sync(W.sm, idx);
    const unsigned owner = __ballot_sync(W.sm, idx == bidx) >> W.sbase;
    const int src = __ffs(owner) - 1;
    const int bm = __shfl_sync(W.sm, mm, src, SW);
    const int q = bm / SW;
    const int32_t h = __shfl_sync(W.sm, q ? W.head[1] : W.head[0], src, SW);
    const int32_t seen = __shfl_sync(W.sm, q ? W.seen[1] : W.seen[0], src, SW);
    const int64_t ah = __ldg(tr.arrival + bidx);
    const int64_t slo = __ldg(pr.slo + bm);
    const int64_t waiting = seen - h;
    const int64_t lim = waiting < bp.max_batch ? waiting : bp.max_batch;
    // lane j tries a batch of k = j + 1 (+32 per round); the finish grows with
    // k (increments >= 0) and the head has the tightest deadline, so the
    // feasible sizes form a prefix 1..K
    int64_t K = 0, fK = 0;
    for (int64_t k0 = 1; k0 <= lim; k0 += SW) {
      const int64_t k = k0 + W.lane;
      int64_t f = 0;
      bool ok = false;
      if (k <= lim) {
        f = batch_finish(pr, bp, W.F, p, off, s, bm, T, k);
        ok = f - ah <= slo;
        W.upd += (unsigned)s;
      }
      const unsigned bal = (__ballot_sync(W.sm, ok) >> W.sbase) & (W.sm >> W.sbase);
      if (!bal) break;
      const int last = 31 - __clz(bal);
      K = k0 + last;
      fK = __shfl_sync(W.sm, f, last, SW);
      if (bal != (W.sm >> W.sbase)) break;
    }
    const int32_t nh = h + (int32_t)(K == 0 ? 1 : K);  // K == 0: the head is rejected
    if (W.lane == src) {
      const int32_t nx = nh < seen ? __ldg(bp.midx + W.mo[bm] + nh) : 0;
      if (q) {
        W.head[1] = nh;
        W.hidx[1] = nx;
      } else {
        W.head[0] = nh;
        W.hidx[0] = nx;
      }
    }
    if (nh == seen) qmask &= ~(1ull << bm);
    if (K == 0) continue;
    if (W.lane == 0) batch_commit(pr, bp, W.F, p, off, s, bm, T, K);
    // sum over the members of (fK - a_j) = K fK - (their arrivals), the
    // latter a difference of the model's running arrival sums; modulo 2^64
    // the result is exact because it lies in [0, 2^63) (reading C20)
    const uint64_t* cum = bp.mcum + W.mo[bm] + bm + h;
    W.sum += (int64_t)((uint64_t)K * (uint64_t)fK - (__ldg(cum + K) - __ldg(cum)));
    W.good += K;
    if (W.lane == src) {
      if (W.pm) W.pm[bm] += K;
    }
    __syncwarp(W.sm);
    return;
  }
}

// The earliest availability event: (first-stage free time, group) minimum
// over the groups that host a model with waiting requests; INT64_MAX if none.
template <int SW>
__device__ __forceinline__ void earliest_event(const Warp& W, uint64_t qmask, int64_t& key,
                                               int& gi) {
  key = INT64_MAX;
  gi = 0x7FFFFFFF;
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    if (W.my_gt[q] == 0xFFFFFFFFu || !(W.gm[W.lane + SW * q] & qmask)) continue;
    const int64_t f0 = W.F[gt_off(W.my_gt[q])];
    if (f0 < key) {  // q ascending: the lane's lower group first on ties
      key = f0;
      gi = W.lane + SW * q;
    }
  }
  warp_argmin<SW>(W.sm, W.sbase, key, gi);
}

template <int kMinBlocks, int SW>
__global__ void __launch_bounds__(kWarps * 32, kMinBlocks)
batching_kernel(DevProblem pr, DevTrace tr, DevBatch bt, DevBatching bp, int32_t slots,
                DevOut out) {
  extern __shared__ __align__(16) unsigned char smem[];
  // one candidate per SW-lane (sub-)warp: SW = 32, or 16 when every
  // placement has <= 32 groups and the problem <= 32 models
  const int sub = threadIdx.x / SW;  // sub-warp index in the block
  const int lane = threadIdx.x % SW;
  const int64_t w = (int64_t)blockIdx.x * (kWarps * 32 / SW) + sub;
  if (w >= bt.C) return;  // uniform in the sub-warp; every sync below uses its mask
  const int64_t c = bp.order ? (int64_t)bp.order[w] : w;
  const int G = bt.G, M = pr.M;
  unsigned char* base =
      smem + ((((size_t)slots * 8 + (size_t)M * 12 + (size_t)G * 12) + 15) & ~(size_t)15) * sub;
  Warp W;
  W.lane = lane;
  W.sbase = (threadIdx.x & 31) - lane;
  W.sm = (SW == 32 ? FULL : 0xFFFFu) << W.sbase;
  const unsigned sm = W.sm;
  W.F = reinterpret_cast<int64_t*>(base);
  uint64_t* hm = reinterpret_cast<uint64_t*>(base + (size_t)slots * 8);  // [M] host masks
  uint64_t* gm = reinterpret_cast<uint64_t*>(base + (size_t)slots * 8 + (size_t)M * 8);
  uint32_t* gt = reinterpret_cast<uint32_t*>(base + (size_t)slots * 8 + (size_t)M * 8 +
                                             (size_t)G * 8);
  int32_t* mo = reinterpret_cast<int32_t*>(base + (size_t)slots * 8 + (size_t)M * 8 +
                                           (size_t)G * 12);  // [M] request-list offsets
  W.mo = mo;
  W.gm = gm;
  W.gt = gt;
  const bool active = bt.cand_ok[c] != 0;
  const int b = bt.cand_base[c];
  const uint64_t* bmask = bt.base_mask + (int64_t)b * M;
  if (lane == 0) {  // group table of the placement (serial prefix over the slots)
    int nslots = 0;
    for (int g = 0; g < G; ++g) {
      const int cfg = bt.base_cfg[(int64_t)b * G + g];
      uint32_t e = 0xFFFFFFFFu;
      if (cfg >= 0) {
        const int st = pr.cfg_stages[cfg];
        e = (uint32_t)cfg | ((uint32_t)nslots << 16) | ((uint32_t)st << 24);
        nslots += st;
      }
      gt[g] = e;
    }
  }
  for (int g = lane; g < G; g += SW) {
    uint64_t h = 0;
    for (int m = 0; m < M; ++m) h |= ((__ldg(bmask + m) >> g) & 1ull) << m;
    gm[g] = active ? h : 0ull;
  }
  for (int k = lane; k < slots; k += SW) W.F[k] = 0;
  for (int m = lane; m < M; m += SW) {
    hm[m] = __ldg(bmask + m);
    mo[m] = __ldg(bp.moff + m);
  }
  __syncwarp(sm);
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int g = lane + SW * q;
    W.my_gt[q] = g < G ? gt[g] : 0xFFFFFFFFu;
    W.head[q] = 0;
    W.hidx[q] = 0;
    W.seen[q] = 0;
  }
  W.good = 0;
  // per-model counts go straight to the candidate's (zeroed) output row: each
  // entry has one writer, the lane that owns the model
  W.pm = out.good_per_model ? out.good_per_model + (c - out.out_offset) * M : nullptr;
  W.sum = 0;
  W.upd = 0;
  uint64_t qmask = 0;  // models with waiting requests (warp-uniform)
  int64_t nev = INT64_MAX;  // cached earliest availability event (warp-uniform)
  int nevg = 0;
  bool nev_ok = false;

  for (int64_t i0 = 0; i0 < tr.n && active; i0 += SW) {
    const int64_t ai = tr.arrival[i0 + lane];
    const int mi = tr.model[i0 + lane];
    const int nj = (int)min((int64_t)SW, tr.n - i0);
    for (int j = 0; j < nj; ++j) {
      const int64_t a = __shfl_sync(sm, ai, j, SW);
      const int m = __shfl_sync(sm, mi, j, SW);
      // replay the availability events at time <= a in (time, group) order;
      // the earliest one is cached until a batch or a newly waiting request
      // changes it (an immediate run uses an available group, which has no
      // waiting work, so it cannot change it)
      if (qmask) {
        if (!nev_ok) {
          earliest_event<SW>(W, qmask, nev, nevg);
          nev_ok = true;
        }
        while (nev <= a) {
          form_batch<SW>(pr, tr, bp, W, qmask, nevg, nev);
          earliest_event<SW>(W, qmask, nev, nevg);
        }
      }
      const int q = m / SW;
      const bool own = (m % SW) == lane;
      const uint64_t hosts = hm[m];
      if (hosts && !((qmask >> m) & 1ull)) {
        // empty queue: run now on the available host with the earliest finish
        int64_t key = INT64_MAX;
        int gi = 0x7FFFFFFF;
#pragma unroll
        for (int qq = 0; qq < 2; ++qq) {
          const int g = lane + SW * qq;
          if (g >= 64 || !((hosts >> g) & 1ull)) continue;
          const uint32_t e = W.my_gt[qq];
          if (W.F[gt_off(e)] > a) continue;  // first stage busy
          const int64_t f = batch_finish(pr, bp, W.F, gt_cfg(e), gt_off(e), gt_stages(e), m, a, 1);
          W.upd += (unsigned)gt_stages(e);
          if (f < key) {
            key = f;
            gi = g;
          }
        }
        warp_argmin<SW>(sm, W.sbase, key, gi);
        if (gi == 0x7FFFFFFF) {  // every host busy: wait for a batch
          qmask |= 1ull << m;
          nev_ok = false;
          if (own) {
            const int32_t i = (int32_t)(i0 + j);
            if (q) {
              W.head[1] = W.seen[1];
              W.hidx[1] = i;
            } else {
              W.head[0] = W.seen[0];
              W.hidx[0] = i;
            }
          }
        } else {
          if (key - a <= __ldg(pr.slo + m)) {  // else rejected at receipt (C2, C3)
            if (lane == (gi % SW)) {
              const uint32_t e = (gi / SW) ? W.my_gt[1] : W.my_gt[0];
              batch_commit(pr, bp, W.F, gt_cfg(e), gt_off(e), gt_stages(e), m, a, 1);
            }
            W.good += 1;
            W.sum += key - a;
            if (own) {
              if (W.pm) W.pm[m] += 1;
            }
          }
          W.head[0] = (own && q == 0) ? W.seen[0] + 1 : W.head[0];
          W.head[1] = (own && q == 1) ? W.seen[1] + 1 : W.head[1];
          __syncwarp(sm);
        }
      }
      W.seen[0] += (int32_t)(own && q == 0);  // branch-free: one owner lane per request
      W.seen[1] += (int32_t)(own && q == 1);
    }
  }
  while (active && qmask) {  // drain
    earliest_event<SW>(W, qmask, nev, nevg);
    form_batch<SW>(pr, tr, bp, W, qmask, nevg, nev);
  }
  if (out.stage_updates) {
    unsigned long long u = W.upd;
    for (int x = SW / 2; x > 0; x >>= 1) u += __shfl_down_sync(sm, u, x, SW);
    if (lane == 0) atomicAdd(out.stage_updates, u);
  }
  const int64_t o = c - out.out_offset;
  if (lane == 0) {
    out.good[o] = active ? W.good : -1;
    if (out.sum_latency) out.sum_latency[o] = active ? W.sum : 0;
  }
}

}  // namespace

size_t batching_smem_per_warp(int32_t slots, int32_t G, int32_t M) {
  return (((size_t)slots * 8 + (size_t)M * 12 + (size_t)G * 12) + 15) & ~(size_t)15;
}

cudaError_t launch_batching(const DevProblem& pr, const DevTrace& tr, const DevBatch& b,
                            const DevBatching& bp, int32_t slots, const DevOut& out,
                            cudaStream_t stream, int64_t* launches) {
  if (b.C <= 0) return cudaSuccess;
  if (slots < 1) slots = 1;
  // resident blocks per SM the register budget is sized for (ASIM_BATCH_MINB
  // = 4 | 5 | 6 | 8; default 4: 128 registers; 5 = 96 registers without
  // spills and 20 warps/SM measured 2 % slower, 6 and 8 spill)
  static const int minb = [] {
    const char* e = getenv("ASIM_BATCH_MINB");
    const int v = e ? atoi(e) : 4;
    return (v == 5 || v == 6 || v == 8) ? v : 4;
  }();
  // half-warp candidates (ASIM_BATCH_SW=16; placements of <= 32 groups and
  // <= 32 models): bit-exact, but measured 4 % slower than full warps on the
  // §5.4 bench (the two halves' event handling diverges), so off by default
  static const bool want16 = [] {
    const char* e = getenv("ASIM_BATCH_SW");
    return e && atoi(e) == 16;
  }();
  const bool half = want16 && b.G <= 32 && pr.M <= 32;
  auto pick = [&](auto k4, auto k5, auto k6, auto k8) {
    return minb == 8 ? k8 : minb == 6 ? k6 : minb == 4 ? k4 : k5;
  };
  auto kern = half ? pick(batching_kernel<4, 16>, batching_kernel<5, 16>, batching_kernel<6, 16>,
                          batching_kernel<8, 16>)
                   : pick(batching_kernel<4, 32>, batching_kernel<5, 32>, batching_kernel<6, 32>,
                          batching_kernel<8, 32>);
  const int per_block = kWarps * (half ? 2 : 1);  // candidates per block
  const size_t smem_b = (size_t)per_block * batching_smem_per_warp(slots, b.G, pr.M);
  cudaError_t ea = allow_max_smem(reinterpret_cast<const void*>(kern));
  if (ea != cudaSuccess) return ea;
  const int blocks = (int)((b.C + per_block - 1) / per_block);
  kern<<<blocks, kWarps * 32, smem_b, stream>>>(pr, tr, b, bp, slots, out);
  if (launches) ++*launches;
  return cudaGetLastError();
}

}  // namespace asim
