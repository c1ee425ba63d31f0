// walk.cu -- pass 3 of the chunked path (chunk.cu header) for small uniform
// components: the LANE walker.  One candidate per lane, its component's stage
// free times in registers, every lane at its own position in the trace.
//
// Why.  A walk re-simulates, in order, the chunks of one candidate whose start
// state turned out wrong -- in sustained overload a trajectory never forgets
// its start (the phase of every busy stage mod its service time is invariant
// until the group idles), so these chains are inherently sequential.  The
// warp-per-candidate walkers (chunk.cu) spend a whole warp on one such chain:
// with a thousand walking candidates per greedy step they saturate the SMs
// with 32-fold redundant work and every chain slows down.  Here a warp carries
// 32 independent chains: the total issue drops 32x and each chain runs at its
// own dependent-latency speed.
//
// Per request of the lane's candidate (§4.3; C1-C6), as
// in every other kernel: for each hosting group of the component, the tandem
// recurrence x = max(x, free_k) + d_k from the arrival; the earliest finish
// wins, ties to the lowest group index (compact group ids ascend with the
// group ids); accept iff the last departure <= arrival + slo - tail; commit
// the winner's departures.  A request outside the component has no host in
// the lane's compact table and leaves the state unchanged, exactly like a
// rejection (its component evolves as the base's: component restriction).
//
// Chunk bookkeeping (identical to chunk.cu's walkers): a chunk j is walked
// when chunk j-1's true end differed from its speculative end; its true start
// is chunk j-1's fix_end column; the exact correction (fix_good, fix_sum) is
// the walked count minus pass 1's; the walk stops at the first chunk whose
// true end is equivalent (max with the next arrival) to its speculative end.
#include <cuda_runtime.h>
#include <stdint.h>

#include <utility>

#include "asim_internal.h"
#include "chunk_common.cuh"
#include "launch_cache.h"

namespace asim {
namespace {

constexpr int kLWarps = 4;  // warps per block

// Class k -> (S, R).
__host__ __device__ constexpr int class_S(int k) { return k < 5 ? 1 : k < 9 ? 2 : 4; }
__host__ __device__ constexpr int class_R(int k) {
  return k < 5 ? (1 << k) : k < 9 ? (2 << (k - 5)) : (4 << (k - 9));
}

// List every item with walking lanes of the lane walker: one thread per
// item; its walking lanes are the lane-walkable candidates (lane_class >= 0)
// with a chunk flagged by pass 2, its class the largest of theirs.
__global__ void item_list_kernel(ChunkParams P, int32_t* __restrict__ list,
                                 uint32_t* __restrict__ lanes_out, uint32_t* __restrict__ counts) {
  const int item = blockIdx.x * blockDim.x + threadIdx.x;
  if (item >= P.num_items) return;
  const ItemDesc it = P.items[item];
  if (it.S != 1 && it.S != 2 && it.S != 4) return;
  uint32_t flags = 0;
  for (int j = 1; j < P.J; ++j) flags |= P.fix_flag[(int64_t)j * P.num_items + item];
  if (!flags) return;
  uint32_t lanes = 0;
  int kmax = -1;
  for (int l = 0; l < it.count; ++l) {
    if (!((flags >> l) & 1u)) continue;
    const int64_t c = cand_of(P, it, item, l);
    if (!P.bt.cand_ok[c]) continue;
    const int k = lane_class(P, it, c);
    if (k < 0) continue;
    lanes |= 1u << l;
    kmax = k > kmax ? k : kmax;  // classes of one S ascend with R
  }
  if (!lanes) return;
  const uint32_t pos = atomicAdd(counts + kmax, 1u);
  list[(int64_t)kmax * P.num_items + pos] = item;
  lanes_out[(int64_t)kmax * P.num_items + pos] = lanes;
}

// Per-request record of a 32-request tile, shared by the warp's lanes (the
// item's candidates share the base's uniform config): arrival relative to the
// epoch, the acceptance limit on the last departure (a + slo - tail, clipped;
// 0 with no host = never), the model's stage latencies, tail, model.
struct alignas(16) WalkRec {
  uint32_t ar, lim, tl;
  int32_t m;
  uint32_t d[4];
};

// One warp walks one item: lane l walks candidate l of the item (if listed),
// its component's R compact slots in registers.  The warp goes through the
// chunks in order; chunk j is simulated for the lanes whose start at j is
// wrong ("need" lanes), replaying the tile-compacted requests of the union of
// their components.  Exactly the bookkeeping of chunk.cu's walkers per lane.
template <int S, int R>
__device__ __forceinline__ void item_walk(const ChunkParams& P, int item, uint32_t lanes,
                                          uint32_t* hmc, WalkRec* rec, int lane,
                                          uint32_t* __restrict__ end_src,
                                          unsigned long long& walked_sum,
                                          unsigned long long& walked_max,
                                          unsigned long long& walkers) {
  using T = uint32_t;
  constexpr int NG = R / S;
  const ItemDesc it = P.items[item];
  const bool mine = (lanes >> lane) & 1u;
  const int64_t c = mine ? cand_of(P, it, item, lane) : 0;
  const int M = P.pr.M;
  const int my_m = mine ? P.bt.cand_model[c] : -1, my_g = mine ? P.bt.cand_group[c] : 0;
  const uint64_t kmask = mine ? P.bt.cand_kmask[c] : 0ull;
  const int ngroups = it.slots / S;
  const uint64_t all = ngroups >= 64 ? ~0ull : ((1ull << ngroups) - 1ull);
  const uint64_t gmask = mine ? (P.bt.cand_gmask[c] & all) : 0ull;
  int cg[NG];  // compact group -> group id (ascending), -1 = padding
  {
    uint64_t b = gmask;
#pragma unroll
    for (int i = 0; i < NG; ++i) {
      cg[i] = b ? (__ffsll((long long)b) - 1) : -1;
      b &= b - 1;
    }
  }
  {  // per-lane compact hosting masks [m][lane]: 0 outside the lane's component
    const uint64_t* bm = P.bt.base_mask + (int64_t)it.base * M;
    for (int m = 0; m < M; ++m) {
      uint32_t x = 0;
      if (mine && m < 64 && ((kmask >> m) & 1ull)) {
        const uint64_t hm = bm[m] | (m == my_m ? (1ull << my_g) : 0ull);
#pragma unroll
        for (int i = 0; i < NG; ++i)
          if (cg[i] >= 0 && ((hm >> cg[i]) & 1ull)) x |= 1u << i;
      }
      hmc[m * 32 + lane] = x;
    }
  }
  const int64_t* __restrict__ arrival = P.tr.arrival;
  const uint16_t* __restrict__ model = P.tr.model;
  const int64_t theta = P.theta;
  const int PP = P.pr.P, SS = P.pr.S, p = it.cfg;
  const int64_t cstride = (int64_t)P.num_items * 32;
  const int64_t slot_id = (int64_t)item * 32 + lane;
  bool start_ok = true;
  unsigned long long walked = 0;
  T v[R];
#pragma unroll
  for (int r = 0; r < R; ++r) v[r] = 0;
  __syncwarp();

  for (int j = 1; j < P.J; ++j) {
    const int64_t u = (int64_t)j * P.num_items + item;
    const bool need = mine && !start_ok;
    const uint32_t needm = __ballot_sync(FULL, need);
    // pass 2 was exact for a lane starting right, but its flagged end is wrong
    const bool flagged = mine && start_ok && ((P.fix_flag[u] >> lane) & 1u);
    if (!needm) {
      const uint32_t fm = __ballot_sync(FULL, flagged);
      if (fm && lane == 0) atomicOr(end_src + u, fm);
      if (flagged) start_ok = false;
      continue;
    }
    const int64_t i_begin = P.chunk_begin[j], i_end = P.chunk_begin[j + 1];
    int64_t E = arrival[i_begin];
    if (need) {  // true start: chunk j-1's true end (fix_end), component slots
      const int64_t prev = u - P.num_items;
      const T* s0 = reinterpret_cast<const T*>(P.fix_end) + prev * P.slots_max * 32;
      const int64_t Ep = P.fix_epoch[prev];
#pragma unroll
      for (int g = 0; g < NG; ++g)
#pragma unroll
        for (int k = 0; k < S; ++k) {
          T x = 0;
          if (cg[g] >= 0) {
            const int64_t r = (int64_t)s0[(cg[g] * S + k) * 32 + lane] - (E - Ep);
            x = r > 0 ? (T)r : (T)0;
          }
          v[g * S + k] = x;
        }
      ++walked;
    }
    // the union of the need lanes' components: the requests to replay
    const uint64_t km = need ? kmask : 0ull;
    const uint64_t ukm = ((uint64_t)__reduce_or_sync(FULL, (uint32_t)(km >> 32)) << 32) |
                         __reduce_or_sync(FULL, (uint32_t)km);
    int64_t good = 0, sum = 0;
    int64_t al_n = i_begin + lane < i_end ? arrival[i_begin + lane] : 0;
    int ml_n = i_begin + lane < i_end ? (int)model[i_begin + lane] : 0;
    for (int64_t i0 = i_begin; i0 < i_end; i0 += 32) {
      const bool valid = i0 + lane < i_end;
      const int64_t al = al_n;
      const int ml = ml_n;
      if (i0 + 32 + lane < i_end) {  // the next tile, one tile ahead
        al_n = arrival[i0 + 32 + lane];
        ml_n = (int)model[i0 + 32 + lane];
      }
      unsigned todo = __ballot_sync(FULL, valid && ml < 64 && ((ukm >> ml) & 1ull));
      if (!todo) continue;
      bool per_req = false;
      {
        const int64_t a_last = __shfl_sync(FULL, al, 31 - __clz(todo));
        if (a_last - E > theta) {  // move the epoch to the tile's first request
          const int64_t a_first = __shfl_sync(FULL, al, __ffs(todo) - 1);
          const int64_t gap = a_first - E;
          const T delta = gap >= 0xFFFFFFFFll ? (T)0xFFFFFFFFu : (T)gap;
#pragma unroll
          for (int r = 0; r < R; ++r) v[r] = v[r] > delta ? v[r] - delta : (T)0;
          E = a_first;
          per_req = a_last - E > theta;  // a sparse tile: per-request epochs
        }
      }
      {  // this lane's request record (only the relevant ones are read)
        WalkRec q;
        const int mm = valid ? ml : 0;
        const int64_t row = (int64_t)mm * PP + p;
        const int64_t tl = P.pr.tail[row], sl = P.pr.slo[mm];
        const T ar = (T)(al - E);
        q.ar = ar;
        q.tl = (T)tl;  // tail <= max_service < 2^32 in uint32 mode
        q.m = mm;
        q.lim = 0u;
        if (sl >= tl) {  // never acceptable otherwise (the flag below)
          const int64_t room = sl - tl;
          q.lim = room >= (int64_t)(0xFFFFFFFEu - ar) ? 0xFFFFFFFEu : (T)(ar + room);
        } else {
          q.m = -1;
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) q.d[k] = k < S ? (T)P.pr.stage[row * SS + k] : 0u;
        rec[lane] = q;
      }
      __syncwarp();
      while (todo) {
        const int jj = __ffs(todo) - 1;
        todo &= todo - 1;
        const WalkRec q = rec[jj];
        const uint32_t hm = (need && q.m >= 0) ? hmc[q.m * 32 + lane] : 0u;
        T ar = q.ar, lim = q.lim;
        if (per_req) {  // a sparse tile: the record's epoch may be stale
          const int64_t a = __shfl_sync(FULL, al, jj);
          if (a - E > theta) {
            const int64_t gap = a - E;
            const T delta = gap >= 0xFFFFFFFFll ? (T)0xFFFFFFFFu : (T)gap;
#pragma unroll
            for (int r = 0; r < R; ++r) v[r] = v[r] > delta ? v[r] - delta : (T)0;
            E = a;
          }
          if (hm != 0u) {
            const int64_t row = (int64_t)q.m * PP + p;
            const int64_t room = P.pr.slo[q.m] - P.pr.tail[row];  // >= 0 (q.m >= 0)
            ar = (T)(a - E);
            lim = room >= (int64_t)(0xFFFFFFFEu - ar) ? 0xFFFFFFFEu : (T)(ar + room);
          }
        }
        if (hm == 0u) continue;  // no host of this lane's component
        T y[R];
        T val[NG];
        uint32_t oh[NG];
#pragma unroll
        for (int g = 0; g < NG; ++g) {
          T x = ar;
#pragma unroll
          for (int k = 0; k < S; ++k) {
            x = tmax(x, v[g * S + k]) + q.d[k];
            y[g * S + k] = x;
          }
          val[g] = ((hm >> g) & 1u) ? x : TT<T>::maxv();
          oh[g] = 1u << g;
        }
#pragma unroll
        for (int st = 1; st < NG; st <<= 1)
#pragma unroll
          for (int g = 0; g + st < NG; g += 2 * st) {
            const bool lt = val[g + st] < val[g];
            val[g] = lt ? val[g + st] : val[g];
            oh[g] = lt ? oh[g + st] : oh[g];
          }
        const bool acc = val[0] <= lim;
        const uint32_t win = acc ? oh[0] : 0u;
#pragma unroll
        for (int g = 0; g < NG; ++g)
#pragma unroll
          for (int k = 0; k < S; ++k) v[g * S + k] = (win & (1u << g)) ? y[g * S + k] : v[g * S + k];
        good += acc ? 1 : 0;
        sum += acc ? (int64_t)(val[0] - ar) + (int64_t)q.tl : 0;
      }
      __syncwarp();  // every lane has read the records before the next tile's
    }
    // end of chunk j for the need lanes: exact correction, equivalence
    bool pub = false;
    if (need) {
      P.fix_good[j * cstride + slot_id] = (int32_t)(good - P.spec_good[j * cstride + slot_id]);
      P.fix_sum[j * cstride + slot_id] = sum - P.spec_sum[j * cstride + slot_id];
      if (j + 1 < P.J) {
        const int64_t a_next = arrival[i_end];
        const T* se = reinterpret_cast<const T*>(P.spec_end) + u * P.slots_max * 32;
        const int64_t Es = P.spec_epoch[u];
        bool eq = true;
#pragma unroll
        for (int g = 0; g < NG; ++g)
#pragma unroll
          for (int k = 0; k < S; ++k) {
            if (cg[g] < 0) continue;
            const int64_t t0 = E + (int64_t)v[g * S + k];
            const int64_t t1 = Es + (int64_t)se[(cg[g] * S + k) * 32 + lane];
            eq &= (t0 > a_next ? t0 : a_next) == (t1 > a_next ? t1 : a_next);
          }
        start_ok = eq;
        if (!eq) {  // publish column `lane` at the unit's canonical epoch
          const int64_t Ec = arrival[i_end - 1];
          const int64_t prev = u - P.num_items;
          const T* s0 = reinterpret_cast<const T*>(P.fix_end) + prev * P.slots_max * 32;
          const int64_t Ep = P.fix_epoch[prev];
          T* out = reinterpret_cast<T*>(P.fix_end) + u * P.slots_max * 32;
          for (int t = 0; t < it.slots; ++t) {  // slots outside the component: start values
            if ((gmask >> ((t / S) & 63)) & 1ull) continue;
            const int64_t r = (int64_t)s0[t * 32 + lane] + Ep - Ec;
            out[t * 32 + lane] = r > 0 ? (T)r : (T)0;
          }
#pragma unroll
          for (int g = 0; g < NG; ++g)
#pragma unroll
            for (int k = 0; k < S; ++k) {
              if (cg[g] < 0) continue;
              const int64_t r = (int64_t)v[g * S + k] - (Ec - E);
              out[(cg[g] * S + k) * 32 + lane] = r > 0 ? (T)r : (T)0;
            }
          P.fix_epoch[u] = Ec;  // the same canonical epoch from every writer
          pub = true;
        }
      } else {
        start_ok = true;
      }
    }
    if (flagged) start_ok = false;
    const uint32_t em = __ballot_sync(FULL, pub || flagged);
    if (em && lane == 0) atomicOr(end_src + u, em);
  }
  if (walked) {
    walked_sum += walked;
    walked_max = walked > walked_max ? walked : walked_max;
    walkers += 1;
  }
}

// One kernel per lane class (separate register allocation each; launched
// concurrently on the context's lane streams): warp w walks the listed items
// w, w + warps, ... of class K.
template <int K>
__global__ void __launch_bounds__(kLWarps * 32) item_walk_kernel(ChunkParams P, uint32_t* end_src,
                                                                 const int32_t* __restrict__ list,
                                                                 const uint32_t* __restrict__ lanes,
                                                                 const uint32_t* __restrict__ counts) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const size_t per_warp = (size_t)P.pr.M * 32 * 4 + 32 * sizeof(WalkRec);
  uint32_t* hmc = reinterpret_cast<uint32_t*>(smem + warp * per_warp);
  WalkRec* rec = reinterpret_cast<WalkRec*>(smem + warp * per_warp + (size_t)P.pr.M * 32 * 4);
  const uint32_t n = counts[K];
  unsigned long long ws = 0, wm = 0, wc = 0;
  for (uint32_t t = blockIdx.x * kLWarps + warp; t < n; t += gridDim.x * kLWarps) {
    const int64_t e = (int64_t)K * P.num_items + t;
    item_walk<class_S(K), class_R(K)>(P, list[e], lanes[e], hmc, rec, lane, end_src, ws, wm, wc);
    __syncwarp();
  }
  if (P.walked) {  // statistics: chunks walked, walking candidates, longest walk
    for (int o = 16; o > 0; o >>= 1) {
      ws += __shfl_down_sync(FULL, ws, o);
      wc += __shfl_down_sync(FULL, wc, o);
      const unsigned long long x = __shfl_down_sync(FULL, wm, o);
      wm = x > wm ? x : wm;
    }
    if (lane == 0 && wc) {
      atomicAdd(P.walked, ws);
      atomicAdd(P.walked + 1, wc);
      atomicMax(P.walked + 2, wm);
    }
  }
}

template <int K>
cudaError_t launch_class(const ChunkParams& P, uint32_t* end_src, const int32_t* list,
                         const uint32_t* lanes, const uint32_t* counts, cudaStream_t st, int sms,
                         size_t smem) {
  int per_sm = 0;
  cudaError_t e =
      blocks_per_sm(reinterpret_cast<const void*>(item_walk_kernel<K>), kLWarps * 32, smem, &per_sm);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  // at most num_items listed items; idle warps exit at once
  int64_t blocks = ((int64_t)P.num_items + kLWarps - 1) / kLWarps;
  if (blocks > (int64_t)per_sm * sms) blocks = (int64_t)per_sm * sms;
  item_walk_kernel<K><<<(unsigned)(blocks < 1 ? 1 : blocks), kLWarps * 32, smem, st>>>(
      P, end_src, list, lanes, counts);
  return cudaGetLastError();
}

template <int... K>
cudaError_t launch_classes(std::integer_sequence<int, K...>, const ChunkParams& P,
                           uint32_t* end_src, const int32_t* list, const uint32_t* lanes,
                           const uint32_t* counts, const cudaStream_t* streams, int sms,
                           size_t smem) {
  cudaError_t e = cudaSuccess;
  ((e = e == cudaSuccess ? launch_class<K>(P, end_src, list, lanes, counts, streams[K], sms, smem)
                         : e),
   ...);
  return e;
}

}  // namespace

cudaError_t launch_lane_walk(const ChunkParams& P, uint32_t* end_src, int32_t* list,
                             uint32_t* counts, const LaneStreams& ls, int sms, int64_t* launches) {
  const int64_t slots = (int64_t)P.num_items * 32;
  if (slots == 0) return cudaSuccess;
  cudaError_t e = cudaStreamWaitEvent(ls.list_stream, ls.fork, 0);
  if (e == cudaSuccess) e = cudaMemsetAsync(counts, 0, (kLaneClasses + 1) * sizeof(uint32_t),
                                            ls.list_stream);
  if (e != cudaSuccess) return e;
  uint32_t* lanes = reinterpret_cast<uint32_t*>(list + (int64_t)kLaneClasses * P.num_items);
  item_list_kernel<<<(unsigned)((P.num_items + 127) / 128), 128, 0, ls.list_stream>>>(P, list, lanes,
                                                                                       counts);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  if ((e = cudaEventRecord(ls.listed, ls.list_stream)) != cudaSuccess) return e;
  for (int k = 0; k < kLaneClasses; ++k)
    if ((e = cudaStreamWaitEvent(ls.streams[k], ls.listed, 0)) != cudaSuccess) return e;
  const size_t smem = (size_t)kLWarps * ((size_t)P.pr.M * 32 * 4 + 32 * sizeof(WalkRec));
  if (smem > 227 * 1024) return cudaErrorInvalidValue;
  e = launch_classes(std::make_integer_sequence<int, kLaneClasses>{}, P, end_src, list, lanes,
                     counts, ls.streams, sms, smem);
  if (e != cudaSuccess) return e;
  for (int k = 0; k < kLaneClasses; ++k) {
    if ((e = cudaEventRecord(ls.done[k], ls.streams[k])) != cudaSuccess) return e;
    if ((e = cudaStreamWaitEvent(ls.join_stream, ls.done[k], 0)) != cudaSuccess) return e;
  }
  if (launches) *launches += 1 + kLaneClasses;
  return cudaSuccess;
}

}  // namespace asim
