// chunk.cu -- the throughput path of the batched simulator (sm_100a):
// lane-per-candidate over (item, time-chunk) work units with exact
// speculative-chunk fix-up.
//
//   pass 1 (spec)   every unit (32 candidates of one base placement x one
//                   chunk of the trace) is simulated from the idle state;
//                   per-lane counts and the end state are stored.
//   pass 2 (fix)    for chunk j >= 1 the TRUE trajectory (started from the
//                   true end state of chunk j-1) and the SPECULATIVE one
//                   (started idle) are run in lockstep until every lane's
//                   states are equivalent -- for every stage slot k,
//                   max(true_k, a) == max(spec_k, a) at the next arrival a
//                   (a free time earlier than the arrival acts exactly like
//                   the arrival, since every later stage start is >= it).
//                   From there on both trajectories take identical decisions,
//                   so the difference of their counts is the exact correction.
//                   A unit whose trajectories never meet runs to the chunk
//                   end and publishes its true end state; the host re-runs
//                   the next chunk from it (rare chains; exact in all cases).
//
// Time representation (template T):
//   int64_t   absolute nanoseconds (any SLO).
//   uint32_t  nanoseconds relative to a warp-uniform epoch E <= arrival.
//             Free times are stored as max(free - E, 0): a free time below
//             the current arrival is equivalent to the arrival, so clamping
//             at the epoch is exact.  E is moved to the current arrival a
//             whenever a - E > theta = 2^32 - 1 - max_slo - max_service,
//             which keeps every stored or predicted value below 2^32
//             (accepted finishes are <= a + slo; predictions add at most
//             max_service to a stored value).  Chosen by the host only when
//             theta is positive.
//
// Per request (§4.3; C1-C6), exactly as sim.cu:
//   f_g = pipeline recurrence on group g's free times; g* = argmin (f_g, g);
//   accept iff f_g* - a <= slo[m]; on accept store the stage departures.
// State lives in shared memory as [slot][lane]; all per-model tables of the
// unit's base placement are staged in shared memory per warp.
#include <cuda_runtime.h>
#include <stdint.h>

#include "asim_internal.h"

namespace asim {
namespace {

constexpr unsigned FULL = 0xFFFFFFFFu;
constexpr int kWarps = 4;  // warps per block; each warp takes units independently
constexpr int kSTab = 16;  // stage entries per model in the uniform-config table
constexpr int kCheckEvery = 64;  // coalescence test period (requests) in the fix-up

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

// Per-warp shared-memory region.
template <typename T>
struct WarpMem {
  T* st0;          // [slots][32] true / speculative trajectory
  T* st1;          // [slots][32] speculative trajectory (fix-up only)
  uint64_t* mask;  // [M]   hosting groups of model m in the base placement
  T* d;            // [M][kSTab] stage latencies under the base's uniform config
  T* tail;         // [M]
  T* slo;          // [M]   (clipped to T's range: exact, see header)
  uint32_t* gt;    // [64]  dynamic-config group table: cfg | off<<16 | s<<24
};

template <typename T>
__device__ __forceinline__ size_t warp_bytes(const ChunkParams& P, bool dual) {
  const size_t slots = (size_t)P.slots_max;
  size_t b = slots * 32 * sizeof(T) * (dual ? 2 : 1);
  b += (size_t)P.pr.M * (8 + sizeof(T) * (kSTab + 2)) + 64 * 4;
  return (b + 15) & ~size_t(15);
}

template <typename T>
__device__ __forceinline__ WarpMem<T> carve(unsigned char* base, const ChunkParams& P, bool dual) {
  WarpMem<T> w;
  const int slots = P.slots_max;
  T* p = reinterpret_cast<T*>(base);
  w.st0 = p;
  p += slots * 32;
  w.st1 = dual ? p : nullptr;
  if (dual) p += slots * 32;
  w.mask = reinterpret_cast<uint64_t*>(p);
  T* q = reinterpret_cast<T*>(w.mask + P.pr.M);
  w.d = q;
  q += P.pr.M * kSTab;
  w.tail = q;
  q += P.pr.M;
  w.slo = q;
  q += P.pr.M;
  w.gt = reinterpret_cast<uint32_t*>(q);
  return w;
}

// Stage the base placement's tables (lane-parallel).
template <typename T>
__device__ void load_base(const ChunkParams& P, const ItemDesc& it, WarpMem<T>& w, int lane) {
  const int M = P.pr.M, PP = P.pr.P, SS = P.pr.S;
  const uint64_t* bm = P.bt.base_mask + (int64_t)it.base * M;
  for (int m = lane; m < M; m += 32) {
    w.mask[m] = bm[m];
    w.slo[m] = TT<T>::clip(P.pr.slo[m]);
    if (it.cfg >= 0) {
      const int64_t* d = P.pr.stage + ((int64_t)m * PP + it.cfg) * SS;
      for (int k = 0; k < kSTab; ++k) w.d[m * kSTab + k] = (k < SS && k < it.stages) ? (T)d[k] : (T)0;
      w.tail[m] = (T)P.pr.tail[(int64_t)m * PP + it.cfg];
    }
  }
  if (lane == 0) {  // group table (also used by the dynamic-config path)
    int off = 0;
    for (int g = 0; g < 64; ++g) {
      uint32_t e = 0xFFFFFFFFu;
      if (g < P.bt.G) {
        const int cfg = P.bt.base_cfg[(int64_t)it.base * P.bt.G + g];
        if (cfg >= 0) {
          const int s = P.pr.cfg_stages[cfg];
          e = (uint32_t)cfg | ((uint32_t)off << 16) | ((uint32_t)s << 24);
          off += s;
        }
      }
      w.gt[g] = e;
    }
  }
  __syncwarp();
}

// Predicted finish of the request (relative arrival ar) on group g of this
// lane's trajectory `st`; S > 0: uniform config with S stages (slot = g*S+k);
// S == 0: dynamic (group table + global stage table).
template <typename T, int S>
__device__ __forceinline__ T predict(const ChunkParams& P, const WarpMem<T>& w, const T* st,
                                     int lane, int g, int m, T ar, const T* dv, T tl) {
  T x = ar;
  if constexpr (S > 0) {
    const T* p = st + (g * S) * 32 + lane;
#pragma unroll
    for (int k = 0; k < S; ++k) x = tmax(x, p[k * 32]) + dv[k];
    return x + tl;
  } else {
    const uint32_t e = w.gt[g];
    const int cfg = (int)(e & 0xFFFFu), off = (int)((e >> 16) & 0xFFu), s = (int)(e >> 24);
    const int64_t* d = P.pr.stage + ((int64_t)m * P.pr.P + cfg) * P.pr.S;
    const T* p = st + off * 32 + lane;
    for (int k = 0; k < s; ++k) x = tmax(x, p[k * 32]) + (T)__ldg(d + k);
    return x + (T)__ldg(P.pr.tail + (int64_t)m * P.pr.P + cfg);
  }
}

template <typename T, int S>
__device__ __forceinline__ void commit(const ChunkParams& P, const WarpMem<T>& w, T* st, int lane,
                                       int g, int m, T ar, const T* dv) {
  T x = ar;
  if constexpr (S > 0) {
    T* p = st + (g * S) * 32 + lane;
#pragma unroll
    for (int k = 0; k < S; ++k) {
      x = tmax(x, p[k * 32]) + dv[k];
      p[k * 32] = x;
    }
  } else {
    const uint32_t e = w.gt[g];
    const int cfg = (int)(e & 0xFFFFu), off = (int)((e >> 16) & 0xFFu), s = (int)(e >> 24);
    const int64_t* d = P.pr.stage + ((int64_t)m * P.pr.P + cfg) * P.pr.S;
    T* p = st + off * 32 + lane;
    for (int k = 0; k < s; ++k) {
      x = tmax(x, p[k * 32]) + (T)__ldg(d + k);
      p[k * 32] = x;
    }
  }
}

// One request on one trajectory: dispatch (earliest predicted finish, lowest
// index on ties), admission at receipt, commit.  Returns latency or -1.
template <typename T, int S>
__device__ __forceinline__ int64_t step(const ChunkParams& P, const WarpMem<T>& w, T* st, int lane,
                                        uint64_t mask, int m, T ar, const T* dv, T tl, T sl,
                                        unsigned long long& upd) {
  T best_f = TT<T>::maxv();
  int best_g = -1;
  while (mask) {  // ascending g, strict '<': lowest index wins ties (C1)
    const int g = __ffsll((long long)mask) - 1;
    mask &= mask - 1;
    if (S > 0) upd += S; else upd += (w.gt[g] >> 24);
    const T f = predict<T, S>(P, w, st, lane, g, m, ar, dv, tl);
    if (f < best_f) {
      best_f = f;
      best_g = g;
    }
  }
  if (best_g >= 0 && (T)(best_f - ar) <= sl) {  // reject at receipt if the SLO is missed (C2, C3)
    commit<T, S>(P, w, st, lane, best_g, m, ar, dv);
    return (int64_t)(best_f - ar);
  }
  return -1;
}

template <typename T>
__device__ __forceinline__ void rebase(T* st, int slots, int lane, T delta) {
  for (int k = 0; k < slots; ++k) {
    const T v = st[k * 32 + lane];
    st[k * 32 + lane] = v > delta ? v - delta : (T)0;
  }
}

// Simulate one unit.  DUAL = fix-up (st0 = true trajectory, st1 = speculative).
template <typename T, int S, bool DUAL>
__device__ void run_unit(const ChunkParams& P, WarpMem<T>& w, const ItemDesc& it, int item, int j,
                         int lane, int src) {
  const int64_t i_begin = P.chunk_begin[j], i_end = P.chunk_begin[j + 1];
  const bool in_item = lane < it.count;
  const int64_t c = (int64_t)it.first + lane;
  const int my_m = in_item ? P.bt.cand_model[c] : -1;
  const int my_g = in_item ? P.bt.cand_group[c] : 0;
  const bool active = in_item && P.bt.cand_ok[c];
  const uint64_t my_bit = (my_m >= 0) ? (1ull << my_g) : 0ull;
  const int slots = it.slots;
  const int64_t slot_id = (int64_t)item * 32 + lane;

  // initial state and epoch.  The speculative trajectory starts from the
  // base's true boundary state (or idle); the fix-up's true trajectory from
  // the previous chunk's true end state.
  int64_t E = TT<T>::kRel ? P.tr.arrival[i_begin] : 0;
  T* spec_st = DUAL ? w.st1 : w.st0;
  if (P.spec_state != nullptr && j > 0) {
    const int64_t* ss = P.spec_state + ((int64_t)P.spec_row[it.base] * P.J + j) * P.state_stride;
    for (int k = 0; k < slots; ++k) {
      const int64_t v = ss[k];
      if constexpr (TT<T>::kRel) {
        const int64_t r = v - E;
        spec_st[k * 32 + lane] = r > 0 ? (T)r : (T)0;
      } else {
        spec_st[k * 32 + lane] = (T)v;
      }
    }
  } else {
    for (int k = 0; k < slots; ++k) spec_st[k * 32 + lane] = (T)0;
  }
  if constexpr (DUAL) {
    const int64_t prev = (int64_t)(j - 1) * P.num_items + item;
    const T* src_st = reinterpret_cast<const T*>(src ? P.fix_end : P.spec_end) +
                      prev * P.slots_max * 32;
    const int64_t Ep = (src ? P.fix_epoch : P.spec_epoch)[prev];
    for (int k = 0; k < slots; ++k) {
      const T v = src_st[k * 32 + lane];
      if constexpr (TT<T>::kRel) {
        const int64_t r = (int64_t)v - (E - Ep);
        w.st0[k * 32 + lane] = r > 0 ? (T)r : (T)0;
      } else {
        w.st0[k * 32 + lane] = v;
      }
    }
  }
  __syncwarp();

  int64_t good0 = 0, sum0 = 0, good1 = 0, sum1 = 0;
  unsigned long long upd = 0;
  bool coalesced = false;
  T dv[S > 0 ? S : 1];
  for (int64_t i0 = i_begin; i0 < i_end; i0 += 32) {
    const int64_t ai = (i0 + lane < i_end) ? P.tr.arrival[i0 + lane] : 0;
    const int mi = (i0 + lane < i_end) ? (int)P.tr.model[i0 + lane] : 0;
    const int nj = (int)min((int64_t)32, i_end - i0);
    for (int jj = 0; jj < nj; ++jj) {
      const int64_t a = __shfl_sync(FULL, ai, jj);
      const int m = __shfl_sync(FULL, mi, jj);
      if constexpr (TT<T>::kRel) {
        if (a - E > P.theta) {  // warp-uniform epoch move (exact, see header)
          // every stored value is < 2^32 - 1, so a longer gap clears them all
          const int64_t gap = a - E;
          const T delta = gap >= 0xFFFFFFFFll ? (T)0xFFFFFFFFu : (T)gap;
          rebase<T>(w.st0, slots, lane, delta);
          if constexpr (DUAL) rebase<T>(w.st1, slots, lane, delta);
          E = a;
        }
      }
      const T ar = (T)(a - E);
      if constexpr (DUAL) {
        if (((i0 + jj - i_begin) % kCheckEvery) == 0) {
          bool eq = true;
          for (int k = 0; k < slots; ++k)
            eq &= tmax(w.st0[k * 32 + lane], ar) == tmax(w.st1[k * 32 + lane], ar);
          if (__all_sync(FULL, eq || !active)) {
            coalesced = true;
            break;
          }
        }
      }
      uint64_t mask = w.mask[m] | ((m == my_m) ? my_bit : 0ull);
      if (!active) mask = 0ull;
      if (__ballot_sync(FULL, mask != 0ull) == 0u) continue;  // hosted nowhere: rejected
      T tl = 0;
      if constexpr (S > 0) {
#pragma unroll
        for (int k = 0; k < S; ++k) dv[k] = w.d[m * kSTab + k];
        tl = w.tail[m];
      }
      const T sl = w.slo[m];
      const int64_t l0 = step<T, S>(P, w, w.st0, lane, mask, m, ar, dv, tl, sl, upd);
      if (l0 >= 0) {
        ++good0;
        sum0 += l0;
      }
      if constexpr (DUAL) {
        const int64_t l1 = step<T, S>(P, w, w.st1, lane, mask, m, ar, dv, tl, sl, upd);
        if (l1 >= 0) {
          ++good1;
          sum1 += l1;
        }
      }
    }
    if (DUAL && coalesced) break;
  }

  if (P.stage_updates) {
    for (int o = 16; o > 0; o >>= 1) upd += __shfl_down_sync(FULL, upd, o);
    if (lane == 0) atomicAdd(P.stage_updates, upd);
  }
  const int64_t unit = (int64_t)j * P.num_items + item;
  if constexpr (!DUAL) {
    P.spec_good[(int64_t)j * P.num_items * 32 + slot_id] = (int32_t)good0;
    P.spec_sum[(int64_t)j * P.num_items * 32 + slot_id] = sum0;
    if (j + 1 < P.J) {  // end state for the next chunk's fix-up
      T* out = reinterpret_cast<T*>(P.spec_end) + unit * P.slots_max * 32;
      for (int k = 0; k < slots; ++k) out[k * 32 + lane] = w.st0[k * 32 + lane];
      if (lane == 0) P.spec_epoch[unit] = E;
    }
  } else {
    P.fix_good[(int64_t)j * P.num_items * 32 + slot_id] = (int32_t)(good0 - good1);
    P.fix_sum[(int64_t)j * P.num_items * 32 + slot_id] = sum0 - sum1;
    if (lane == 0) P.fix_flag[unit] = coalesced ? 0 : 1;
    if (!coalesced && j + 1 < P.J) {  // publish the true end state
      T* out = reinterpret_cast<T*>(P.fix_end) + unit * P.slots_max * 32;
      for (int k = 0; k < slots; ++k) out[k * 32 + lane] = w.st0[k * 32 + lane];
      if (lane == 0) P.fix_epoch[unit] = E;
    }
  }
}

template <typename T, bool DUAL>
__global__ void __launch_bounds__(kWarps * 32) chunk_kernel(ChunkParams P) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  WarpMem<T> w = carve<T>(smem + warp * warp_bytes<T>(P, DUAL), P, DUAL);
  int cur_base = -1, cur_cfg = -2;
  for (;;) {
    int u = 0;
    if (lane == 0) u = (int)atomicAdd(P.counter, 1u);
    u = __shfl_sync(FULL, u, 0);
    if (u >= P.num_units) break;
    int item, j, src = 0;
    if constexpr (DUAL) {
      const ChunkUnit cu = P.units[u];
      item = cu.item;
      j = cu.chunk;
      src = cu.src;
    } else {  // pass 1 enumerates every (item, chunk), chunk-major
      item = u % P.num_items;
      j = u / P.num_items;
    }
    const ItemDesc it = P.items[item];
    if (it.base != cur_base || it.cfg != cur_cfg) {
      load_base<T>(P, it, w, lane);
      cur_base = it.base;
      cur_cfg = it.cfg;
    }
    switch (it.S) {
      case 1: run_unit<T, 1, DUAL>(P, w, it, item, j, lane, src); break;
      case 2: run_unit<T, 2, DUAL>(P, w, it, item, j, lane, src); break;
      case 4: run_unit<T, 4, DUAL>(P, w, it, item, j, lane, src); break;
      case 8: run_unit<T, 8, DUAL>(P, w, it, item, j, lane, src); break;
      case 16: run_unit<T, 16, DUAL>(P, w, it, item, j, lane, src); break;
      default: run_unit<T, 0, DUAL>(P, w, it, item, j, lane, src); break;
    }
    __syncwarp();
  }
}

// good[c] = sum_j spec_good[j][c] + sum_{j>=1} fix_good[j][c] (same for sums)
__global__ void chunk_reduce_kernel(ChunkParams P, DevOut out) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)P.num_items * 32) return;
  const int item = (int)(t >> 5), lane = (int)(t & 31);
  const ItemDesc it = P.items[item];
  if (lane >= it.count) return;
  const int64_t c = (int64_t)it.first + lane;
  const int64_t stride = (int64_t)P.num_items * 32;
  int64_t g = 0, s = 0;
  for (int j = 0; j < P.J; ++j) {
    g += P.spec_good[j * stride + t];
    s += P.spec_sum[j * stride + t];
    if (j > 0) {
      g += P.fix_good[j * stride + t];
      s += P.fix_sum[j * stride + t];
    }
  }
  const bool ok = P.bt.cand_ok[c];
  out.good[c - out.out_offset] = ok ? g : -1;
  if (out.sum_latency) out.sum_latency[c - out.out_offset] = ok ? s : 0;
}

template <typename T>
__global__ void publish_kernel(ChunkParams P, const uint8_t* __restrict__ end_src,
                               const int32_t* __restrict__ out_row, int64_t* __restrict__ out) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t total = (int64_t)P.num_items * P.J * P.state_stride;
  if (t >= total) return;
  const int k = (int)(t % P.state_stride);
  const int j = (int)((t / P.state_stride) % P.J);
  const int item = (int)(t / ((int64_t)P.state_stride * P.J));
  int64_t v = 0;  // j == 0: idle; slots beyond the item's: unused
  if (j > 0 && k < P.items[item].slots) {
    const int64_t u = (int64_t)(j - 1) * P.num_items + item;  // end of chunk j-1
    const bool fix = end_src[u] != 0;
    const T* st = reinterpret_cast<const T*>(fix ? P.fix_end : P.spec_end) + u * P.slots_max * 32;
    const T x = st[k * 32 + 0];  // lane 0 of the item
    if constexpr (TT<T>::kRel) {
      v = (fix ? P.fix_epoch : P.spec_epoch)[u] + (int64_t)x;
    } else {
      v = (int64_t)x;
    }
  }
  out[((int64_t)out_row[item] * P.J + j) * P.state_stride + k] = v;
}

template <typename T, bool DUAL>
cudaError_t launch_t(const ChunkParams& P, cudaStream_t st, int sms) {
  const size_t per_warp = (size_t)P.slots_max * 32 * sizeof(T) * (DUAL ? 2 : 1) +
                          (size_t)P.pr.M * (8 + sizeof(T) * (kSTab + 2)) + 64 * 4;
  const size_t smem = kWarps * ((per_warp + 15) & ~size_t(15));
  if (smem > 227 * 1024) return cudaErrorInvalidValue;
  cudaError_t e = cudaFuncSetAttribute(chunk_kernel<T, DUAL>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, chunk_kernel<T, DUAL>, kWarps * 32,
                                                    smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  int64_t blocks = (int64_t)per_sm * sms;  // persistent: warps pull units from a counter
  const int64_t need = ((int64_t)P.num_units + kWarps - 1) / kWarps;
  if (blocks > need) blocks = need;
  if (blocks < 1) blocks = 1;
  chunk_kernel<T, DUAL><<<(unsigned)blocks, kWarps * 32, smem, st>>>(P);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_chunk_pass(const ChunkParams& P, bool dual, bool u32, cudaStream_t st, int sms,
                              int64_t* launches) {
  if (P.num_units <= 0) return cudaSuccess;
  cudaError_t e = cudaMemsetAsync(P.counter, 0, sizeof(uint32_t), st);
  if (e != cudaSuccess) return e;
  if (u32)
    e = dual ? launch_t<uint32_t, true>(P, st, sms) : launch_t<uint32_t, false>(P, st, sms);
  else
    e = dual ? launch_t<int64_t, true>(P, st, sms) : launch_t<int64_t, false>(P, st, sms);
  if (launches) ++*launches;
  return e;
}

cudaError_t launch_publish_states(const ChunkParams& P, const uint8_t* end_src, bool u32,
                                  const int32_t* out_row, int64_t* out, cudaStream_t st,
                                  int64_t* launches) {
  const int64_t total = (int64_t)P.num_items * P.J * P.state_stride;
  if (total == 0) return cudaSuccess;
  const unsigned blocks = (unsigned)((total + 255) / 256);
  if (u32)
    publish_kernel<uint32_t><<<blocks, 256, 0, st>>>(P, end_src, out_row, out);
  else
    publish_kernel<int64_t><<<blocks, 256, 0, st>>>(P, end_src, out_row, out);
  if (launches) ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_chunk_reduce(const ChunkParams& P, const DevOut& out, cudaStream_t st,
                                int64_t* launches) {
  const int64_t n = (int64_t)P.num_items * 32;
  if (n == 0) return cudaSuccess;
  chunk_reduce_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(P, out);
  if (launches) ++*launches;
  return cudaGetLastError();
}

}  // namespace asim
