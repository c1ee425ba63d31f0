// chunk.cu -- the throughput path of the batched simulator (sm_100a):
// lane-per-candidate over (item, time-chunk) work units with exact
// speculative-chunk fix-up.
//
//   pass 1 (SPEC)   every unit (<= 32 candidates sharing one base placement x
//                   one chunk of the trace) is simulated from a speculative
//                   start state: the base placement's true state at the chunk
//                   boundary when the search provides it, else idle.  Counts
//                   and the end state are stored.
//   pass 2 (DUAL)   for chunk j >= 1 the TRUE trajectory (from chunk j-1's
//                   speculative end, assumed true) and the SPECULATIVE one are
//                   run in lockstep until every lane's states are equivalent:
//                   for every stage slot k, max(true_k, a) == max(spec_k, a) at
//                   the next arrival a (a free time earlier than an arrival acts
//                   exactly like it, since every later stage start is >= it).
//                   From there both trajectories take identical decisions, so
//                   the difference of their counts is the exact correction.  A
//                   unit whose trajectories never meet runs to the chunk end
//                   and publishes its true end state.
//   pass 3 (WALK)   one warp per item scans its chunks in order; wherever a
//                   chunk's start state turned out wrong (the previous chunk
//                   never met its speculation) it re-simulates that chunk from
//                   the true start, single trajectory, until the true end state
//                   is again equivalent to the stored speculative one.  Exact in
//                   every case; the walked length is the inherently sequential
//                   part (sustained overload never forgets its start state).
//
// Time representation (template T):
//   int64_t   absolute nanoseconds (any SLO).
//   uint32_t  nanoseconds relative to a warp-uniform epoch E <= arrival.
//             Free times are stored as max(free - E, 0): clamping at the epoch
//             is exact by the same equivalence.  E moves to the current arrival
//             a whenever a - E > theta = 2^32 - 1 - max_slo - max_service,
//             which keeps every stored or predicted value below 2^32
//             (accepted finishes are <= a + slo; predictions add at most
//             max_service to a stored value).  Chosen only when theta > 0.1 s.
//
// Per request (§4.3; C1-C6), exactly as sim.cu:
//   f_g = pipeline recurrence on group g's free times; g* = argmin (f_g, g);
//   accept iff f_g* - a <= slo[m]; on accept store the stage departures.
// State lives in shared memory as [slot][lane]; the unit's per-model tables
// (hosting masks, stage latencies of the base's uniform config, tail, SLO,
// relevance flags) are staged in shared memory per warp.  Requests whose
// model no lane hosts are skipped 32 at a time with one ballot.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#ifdef ASIM_WALK_DIAGNOSTICS
#include <cstdio>
#endif
#include <cstdlib>

#include "asim_internal.h"
#include "chunk_common.cuh"
#include "launch_cache.h"

namespace asim {
namespace {

constexpr int kWarps = 4;        // warps per block; each warp takes units independently
constexpr int kSTab = 16;        // stage entries per model in the uniform-config table
constexpr int kCheckEvery = 64;  // coalescence test period (requests) in the fix-up
enum Mode { SPEC = 0, DUAL = 1, WALK = 2 };


// Per-warp shared-memory region.
template <typename T>
struct WarpMem {
  T* st0;          // [slots][32] speculative (SPEC) / true (DUAL, WALK) trajectory
  T* st1;          // [slots][32] speculative trajectory (DUAL only)
  T* d;            // [M][kSTab] stage latencies under the base's uniform config
  T* tail;         // [M]
  T* slo;          // [M]   (clipped to T's range: exact, see header)
  uint32_t* gt;    // [64]  group table: cfg | off<<16 | s<<24
  uint16_t* hoff;  // [M+1] hosting list of model m in the base: hid[hoff[m] .. hoff[m+1])
  uint16_t* hid;  // uniform items (S > 0): byte offset g * S * 32 * sizeof(T) of each
                  // host's first stage slot; mixed items (S == 0): group ids    // [M*64] group ids, ascending
  uint8_t* rel;    // [M]   some lane of the unit hosts model m
  uint8_t* sgrp;   // [128] group of each stage slot
  uint64_t* hmask; // [M]   hosting groups of model m (bit set; warp-cooperative walker)
  unsigned char* tile;  // [kTileBytes] one trace tile's per-request fields (scalar walker)
};

// The scalar walker stages a tile's per-request fields here: every lane
// writes its request, then the per-request loop reads them with broadcast
// loads whose addresses do not depend on the simulation state.
template <typename T>
struct alignas(16) TileReq {
  T ar;          // arrival, relative to the epoch
  T lim;         // accept iff the last departure <= lim (= ar + slo - tail, saturated)
  T tl;          // tail
  T d[4];        // the first stage latencies of the request's model (S <= 4:
                 // staged, so no table load depends on the record on the chain)
  uint32_t hm;   // compact hosting mask (0: no host in the component, or never acceptable)
  int32_t m;     // model
};
constexpr size_t kTileBytes = 32 * sizeof(TileReq<int64_t>);


// hid_cap: bytes of the hosting-list region = max(hostings of any base in the
// launch, 4 M) -- the scalar walker reuses it as M uint32 compact masks.
// The scalar walker's tile staging aliases the state region st0 (it keeps
// its state in registers) when st0 is large enough.
__host__ __device__ inline size_t tile_extra(int slots_max, size_t tsz) {
  return (size_t)slots_max * 32 * tsz >= kTileBytes ? 0 : kTileBytes;
}

// dsm: the stage-latency table lives in the region (walkers); passes 1-2
// read it from the global per-config table through L1 instead, which keeps
// their regions small enough for 5 blocks per SM.
__host__ __device__ inline size_t warp_bytes(int slots_max, int M, int hid_cap, size_t tsz,
                                             bool dual, bool dsm = true) {
  size_t b = (size_t)slots_max * 32 * tsz * (dual ? 2 : 1);
  b += (size_t)M * tsz * ((dsm ? kSTab : 0) + 2) + 64 * 4 + 2 * (size_t)(M + 1);
  b = (b + 15) & ~size_t(15);
  b += (size_t)hid_cap + ((M + 15) & ~15) + 128;
  b = (b + 15) & ~size_t(15);
  b += (size_t)M * 8;
  b = (b + 15) & ~size_t(15);
  b += tile_extra(slots_max, tsz);
  return (b + 15) & ~size_t(15);
}

template <typename T>
__device__ __forceinline__ WarpMem<T> carve(unsigned char* base, const ChunkParams& P, bool dual,
                                            bool dsm = true) {
  // integer offsets from the shared-memory base only: pointer differences
  // would hide the address space and turn every LDS into a generic access
  WarpMem<T> w;
  const size_t M = (size_t)P.pr.M;
  const size_t st_bytes = (size_t)P.slots_max * 32 * sizeof(T);
  size_t off = 0;
  w.st0 = reinterpret_cast<T*>(base + off);
  off += st_bytes;
  w.st1 = dual ? reinterpret_cast<T*>(base + off) : nullptr;
  if (dual) off += st_bytes;
  w.d = dsm ? reinterpret_cast<T*>(base + off) : nullptr;
  if (dsm) off += M * kSTab * sizeof(T);
  w.tail = reinterpret_cast<T*>(base + off);
  off += M * sizeof(T);
  w.slo = reinterpret_cast<T*>(base + off);
  off += M * sizeof(T);
  w.gt = reinterpret_cast<uint32_t*>(base + off);
  off += 64 * 4;
  w.hoff = reinterpret_cast<uint16_t*>(base + off);
  off += 2 * (M + 1);
  off = (off + 15) & ~size_t(15);
  w.hid = reinterpret_cast<uint16_t*>(base + off);
  off += (size_t)P.hid_cap;
  w.rel = base + off;
  off += (M + 15) & ~size_t(15);
  w.sgrp = base + off;
  off += 128;
  off = (off + 15) & ~size_t(15);
  w.hmask = reinterpret_cast<uint64_t*>(base + off);
  off += M * 8;
  off = (off + 15) & ~size_t(15);
  w.tile = tile_extra(P.slots_max, sizeof(T)) ? base + off : reinterpret_cast<unsigned char*>(w.st0);
  return w;
}

// Stage the base placement's tables (lane-parallel).
template <typename T>
__device__ __forceinline__ void load_base(const ChunkParams& P, const ItemDesc& it, WarpMem<T>& w, int lane) {
  const int M = P.pr.M, PP = P.pr.P, SS = P.pr.S;
  const uint64_t* bm = P.bt.base_mask + (int64_t)it.base * M;
  // hosting lists: prefix sum of popcounts, then every lane fills its models
  int base_off = 0;
  for (int m0 = 0; m0 < M; m0 += 32) {
    const int m = m0 + lane;
    const uint64_t bits = m < M ? bm[m] : 0ull;
    const int cnt = __popcll(bits);
    int incl = cnt;
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xFFFFFFFFu, incl, o);
      if (lane >= o) incl += v;
    }
    const int start = base_off + incl - cnt;
    if (m < M) {
      w.hoff[m] = (uint16_t)start;
      uint64_t b = bits;
      for (int r = start; b; ++r) {
        const int g = __ffsll((long long)b) - 1;
        w.hid[r] = (uint16_t)(it.S > 0 ? g * it.S * 32 * (int)sizeof(T) : g);
        b &= b - 1;
      }
    }
    base_off += __shfl_sync(0xFFFFFFFFu, incl, 31);
  }
  if (lane == 0) w.hoff[M] = (uint16_t)base_off;
  for (int m = lane; m < M; m += 32) {
    w.hmask[m] = bm[m];
    w.slo[m] = TT<T>::clip(P.pr.slo[m]);
    if (it.cfg >= 0) {
      const int64_t* d = P.pr.stage + ((int64_t)m * PP + it.cfg) * SS;
      if (w.d)
        for (int k = 0; k < kSTab; ++k)
          w.d[m * kSTab + k] = (k < SS && k < it.stages) ? (T)d[k] : (T)0;
      w.tail[m] = (T)P.pr.tail[(int64_t)m * PP + it.cfg];
    }
  }
  if (lane == 0) {
    int off = 0;
    for (int g = 0; g < 64; ++g) {
      uint32_t e = 0xFFFFFFFFu;
      if (g < P.bt.G) {
        const int cfg = P.bt.base_cfg[(int64_t)it.base * P.bt.G + g];
        if (cfg >= 0) {
          const int s = P.pr.cfg_stages[cfg];
          e = (uint32_t)cfg | ((uint32_t)off << 16) | ((uint32_t)s << 24);
          for (int k = 0; k < s && off + k < 128; ++k) w.sgrp[off + k] = (uint8_t)g;
          off += s;
        }
      }
      w.gt[g] = e;
    }
  }
  __syncwarp();
}

// Predicted finish on group g of trajectory `st`; S > 0: uniform config with
// S stages (slot = g*S + k); S == 0: group table + global stage table.
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
// Used for mixed configs (S == 0); uniform configs run step_u.
// S > 0 (uniform config): hinfo = byte offsets of the first two hosts
// (off0 | off1 << 16), h0 = list start | host count << 16, further hosts'
// offsets in w.hid; every host runs the same stage latencies dv, so for
// S == 1 the argmin of max(v, a) is the argmin of the finish.  S == 0:
// hinfo = first host | second host << 8 | count << 16 (group ids), h0 =
// list start, group tables in w.gt.
template <typename T, int S>
__device__ __forceinline__ int64_t step(const ChunkParams& P, const WarpMem<T>& w, T* st, int lane,
                                        int m, int hinfo, int h0, bool mine, int my_g,
                                        bool active, T ar, const T* dv, T tl, T sl,
                                        uint32_t& upd, int& gout) {
  if constexpr (S > 0) {
    constexpr int kStride = 32 * (int)sizeof(T);  // bytes between a group's stages
    const int cnt = h0 >> 16, hs = h0 & 0xFFFF;
    const char* stl = reinterpret_cast<const char*>(st + lane);
    T best = TT<T>::maxv();
    int bo = 0x7FFFFFFF;  // byte offset of the best host (ascending = group order)
    auto host = [&](int off) {
      T x;
      if constexpr (S == 1) {
        x = tmax(*reinterpret_cast<const T*>(stl + off), ar);
      } else {
        x = ar;
#pragma unroll
        for (int k = 0; k < S; ++k) x = tmax(x, *reinterpret_cast<const T*>(stl + off + k * kStride)) + dv[k];
      }
      const bool lt = x < best;  // strict: the lowest index wins ties (C1)
      best = lt ? x : best;
      bo = lt ? off : bo;
    };
    if (cnt >= 1) host(hinfo & 0xFFFF);
    if (cnt >= 2) host((int)((unsigned)hinfo >> 16));
    for (int h = hs + 2; h < hs + cnt; ++h) host(w.hid[h]);
    if (active) upd += (uint32_t)cnt;  // algorithmic work (x S at the flush): live lanes only
    if (mine) {  // this lane's added replica; ties resolved by group index
      upd += 1u;
      const int off = my_g * S * kStride;
      T x;
      if constexpr (S == 1) {
        x = tmax(*reinterpret_cast<const T*>(stl + off), ar);
      } else {
        x = ar;
#pragma unroll
        for (int k = 0; k < S; ++k) x = tmax(x, *reinterpret_cast<const T*>(stl + off + k * kStride)) + dv[k];
      }
      if (x < best || (x == best && off < bo)) {
        best = x;
        bo = off;
      }
    }
    // S == 1: best = max(v, a), the finish is best + d0 + tail
    const T dep = S == 1 ? (T)(best + dv[0]) : best;  // last stage departure of the winner
    const T f = dep + tl;
    if (active && bo != 0x7FFFFFFF && (T)(f - ar) <= sl) {  // reject at receipt if the SLO is missed (C2, C3)
      gout = bo / (S * kStride);
      char* stw = reinterpret_cast<char*>(st + lane);
      if constexpr (S == 1) {
        *reinterpret_cast<T*>(stw + bo) = dep;
      } else {
        T x = ar;
#pragma unroll
        for (int k = 0; k < S; ++k) {
          T* p = reinterpret_cast<T*>(stw + bo + k * kStride);
          x = tmax(x, *p) + dv[k];
          *p = x;
        }
      }
      return (int64_t)(f - ar);
    }
    return -1;
  } else {
    T best_f = TT<T>::maxv();
    int best_g = 64;
    const int cnt = hinfo >> 16;
    for (int h = h0; h < h0 + cnt; ++h) {
      const int g = w.hid[h];
      if (active) upd += (w.gt[g] >> 24);
      const T f = predict<T, S>(P, w, st, lane, g, m, ar, dv, tl);
      if (f < best_f) {
        best_f = f;
        best_g = g;
      }
    }
    if (mine) {  // this lane's added replica; ties resolved by group index
      upd += (w.gt[my_g] >> 24);
      const T f = predict<T, S>(P, w, st, lane, my_g, m, ar, dv, tl);
      if (f < best_f || (f == best_f && my_g < best_g)) {
        best_f = f;
        best_g = my_g;
      }
    }
    if (active && best_g < 64 && (T)(best_f - ar) <= sl) {  // reject at receipt if the SLO is missed (C2, C3)
      gout = best_g;
      commit<T, S>(P, w, st, lane, best_g, m, ar, dv);
      return (int64_t)(best_f - ar);
    }
    return -1;
  }
}

template <bool B>
struct BoolC {
  static constexpr bool value = B;
};

// Position of the r-th (0-based) set bit of x (r < popc(x); else garbage):
// a 5-step popcount select.
__device__ __forceinline__ int nth_set_bit(unsigned x, int r) {
  int p = 0;
#pragma unroll
  for (int wd = 16; wd; wd >>= 1) {
    const int cnt = __popc(x & ((1u << wd) - 1u));
    if (r >= cnt) {
      r -= cnt;
      x >>= wd;
      p += wd;
    }
  }
  return p;
}

// Uniform-config request fields of model m arriving at ar (relative time),
// computed once per request (lane-parallel per tile in run_unit):
//   lim  the request is accepted iff v <= lim, where v = the winner's last
//        departure (S > 1) or max(free, ar) (S == 1): the finish v + tail
//        [+ d0] must satisfy finish - ar <= slo (C2, C3); saturated at maxv - 1
//   cc   latency = v + cc, i.e. cc = tail - ar [+ d0] modulo 2^bits(T) (the
//        latency itself is < 2^bits: uint32 times are chosen only then)
//   d0   the first stage latency (S == 1)
//   hA, hB  byte offsets of the first four hosts' first stage slots (16 bits each)
//   h0c  hosting-list start | host count << 16 | never-acceptable << 23
template <typename T, int S>
__device__ __forceinline__ void uniform_fields(const WarpMem<T>& w, const T* dt, int m, T ar,
                                               T& lim, T& cc, T& d0, int& hA, int& hB, int& h0c) {
  const int h0 = w.hoff[m];
  const int cnt = w.hoff[m + 1] - h0;
  hA = (cnt >= 1 ? (int)w.hid[h0] : 0) | (cnt >= 2 ? (int)w.hid[h0 + 1] << 16 : 0);
  hB = (cnt >= 3 ? (int)w.hid[h0 + 2] : 0) | (cnt >= 4 ? (int)w.hid[h0 + 3] << 16 : 0);
  const T sl = w.slo[m], tl = w.tail[m];
  d0 = S == 1 ? __ldg(dt + m * kSTab) : (T)0;
  bool ok = sl >= tl;
  T l = 0;
  if (ok) {
    const T room = sl - tl;
    l = room > (T)(TT<T>::maxv() - 1 - ar) ? (T)(TT<T>::maxv() - 1) : (T)(ar + room);
  }
  if constexpr (S == 1) {  // v = max(free, ar); the departure is v + d0
    ok = ok && l >= d0;
    l = ok ? (T)(l - d0) : (T)0;
  }
  lim = l;
  cc = (T)(tl + d0 - ar);
  h0c = h0 | (cnt << 16) | (ok ? 0 : 1 << 23);
}

// Stage latencies d[0..S) of one model (row of the per-warp table, 16-byte
// aligned): vector shared-memory loads.
template <typename T, int S>
__device__ __forceinline__ void load_dv(const T* row, T* dv) {
  if constexpr (sizeof(T) == 4 && S >= 4) {
#pragma unroll
    for (int q = 0; q < S / 4; ++q) {
      const uint4 v = __ldg(reinterpret_cast<const uint4*>(row) + q);
      dv[4 * q] = (T)v.x;
      dv[4 * q + 1] = (T)v.y;
      dv[4 * q + 2] = (T)v.z;
      dv[4 * q + 3] = (T)v.w;
    }
  } else if constexpr (S >= 2) {
#pragma unroll
    for (int q = 0; q < S * (int)sizeof(T) / 8; ++q) {
      const uint2 v = __ldg(reinterpret_cast<const uint2*>(row) + q);
      if constexpr (sizeof(T) == 4) {
        dv[2 * q] = (T)v.x;
        dv[2 * q + 1] = (T)v.y;
      } else {
        dv[q] = (T)(((unsigned long long)v.y << 32) | v.x);
      }
    }
  } else {
    dv[0] = __ldg(row);
  }
}

// The same from the walkers' shared-memory table.
template <typename T, int S>
__device__ __forceinline__ void load_dv_smem(const T* row, T* dv) {
  if constexpr (sizeof(T) == 4 && S >= 4) {
#pragma unroll
    for (int q = 0; q < S / 4; ++q) {
      const uint4 v = reinterpret_cast<const uint4*>(row)[q];
      dv[4 * q] = (T)v.x;
      dv[4 * q + 1] = (T)v.y;
      dv[4 * q + 2] = (T)v.z;
      dv[4 * q + 3] = (T)v.w;
    }
  } else {
#pragma unroll
    for (int k = 0; k < S; ++k) dv[k] = row[k];
  }
}

// A walker's stage latencies of the staged request q: from the record for S
// <= 4, else from the per-warp table.
template <typename T, int S>
__device__ __forceinline__ void tile_dv(const TileReq<T>& q, const T* dtab, T* d) {
  if constexpr (S <= 4) {
#pragma unroll
    for (int k = 0; k < S; ++k) d[k] = q.d[k];
  } else {
    load_dv_smem<T, S>(dtab + q.m * kSTab, d);
  }
}

// One request on one trajectory of a uniform-config unit (S > 0): dispatch to
// the earliest predicted finish among the base's hosts and this lane's added
// replica (lowest group index on ties, C1), admission at receipt (C2, C3),
// commit.  Hosts are byte offsets in ascending group order; the first four
// come packed in hA / hB, further ones from the hosting list.  Returns whether
// the request is accepted; v = the compared value (see uniform_fields), bo =
// byte offset of the chosen group's first slot.
template <typename T, int S, bool BF = false>
__device__ __forceinline__ bool step_u(const WarpMem<T>& w, T* st, int lane, int hA, int hB,
                                       int h0c, bool mine, int my_off, bool live, T ar,
                                       const T* dv, T lim, T& v, int& bo) {
  constexpr int kStride = 32 * (int)sizeof(T);  // bytes between a group's stages
  const char* stl = reinterpret_cast<const char*>(st + lane);
  auto pred = [&](int off) -> T {
    if constexpr (S == 1) {
      return tmax(*reinterpret_cast<const T*>(stl + off), ar);
    } else {
      T x = ar;
#pragma unroll
      for (int k = 0; k < S; ++k) x = tmax(x, *reinterpret_cast<const T*>(stl + off + k * kStride)) + dv[k];
      return x;
    }
  };
  T best = TT<T>::maxv();
  int b = 0x7FFFFFFF;
  auto host = [&](int off) {
    const T x = pred(off);
    const bool lt = x < best;  // strict: the lowest index wins ties (C1)
    best = lt ? x : best;
    b = lt ? off : b;
  };
  const int cnt = (h0c >> 16) & 0x7F;
  if constexpr (BF && S <= 2) {
    // (pass 2) short recurrences: the first four hosts and this lane's own
    // replica without branches (a missing host reads slot 0 and is masked):
    // pass 2 3.03 -> 2.45 s; pass 1 got slower with it (14.8 -> 15.5 s,
    // profiles/r2p)
    const int o0 = hA & 0xFFFF, o1 = (int)((unsigned)hA >> 16);
    const int o2 = hB & 0xFFFF, o3 = (int)((unsigned)hB >> 16);
    const T x0 = pred(o0), x1 = pred(o1), x2 = pred(o2), x3 = pred(o3);
    const T xm = pred(my_off);
    auto take = [&](bool ok, T x, int off) {
      const bool lt = ok && x < best;  // strict: the lowest index wins ties (C1)
      best = lt ? x : best;
      b = lt ? off : b;
    };
    take(cnt >= 1, x0, o0);
    take(cnt >= 2, x1, o1);
    take(cnt >= 3, x2, o2);
    take(cnt >= 4, x3, o3);
    if (cnt > 4) {
      const int hs = h0c & 0xFFFF;
      for (int h = hs + 4; h < hs + cnt; ++h) host(w.hid[h]);
    }
    // this lane's added replica; ties resolved by group index
    const bool tm = mine && (xm < best || (xm == best && my_off < b));
    best = tm ? xm : best;
    b = tm ? my_off : b;
  } else {
    if (cnt >= 1) {
      host(hA & 0xFFFF);
      if (cnt >= 2) host((int)((unsigned)hA >> 16));
      if (cnt >= 3) {
        host(hB & 0xFFFF);
        if (cnt >= 4) host((int)((unsigned)hB >> 16));
        const int hs = h0c & 0xFFFF;
        for (int h = hs + 4; h < hs + cnt; ++h) host(w.hid[h]);
      }
    }
    if (mine) {  // this lane's added replica; ties resolved by group index
      const T x = pred(my_off);
      if (x < best || (x == best && my_off < b)) {
        best = x;
        b = my_off;
      }
    }
  }
  v = best;
  bo = b;
  const bool acc = live && b != 0x7FFFFFFF && best <= lim;
  if (acc) {
    char* stw = reinterpret_cast<char*>(st + lane);
    if constexpr (S == 1) {
      *reinterpret_cast<T*>(stw + b) = best + dv[0];
    } else {
      T x = ar;
#pragma unroll
      for (int k = 0; k < S; ++k) {
        T* p = reinterpret_cast<T*>(stw + b + k * kStride);
        x = tmax(x, *p) + dv[k];
        *p = x;
      }
    }
  }
  return acc;
}

// Stage occupancy sum_k d_k of model m on group g (fast-heuristic busy time).
template <typename T, int S>
__device__ __forceinline__ int64_t occupancy(const ChunkParams& P, const WarpMem<T>& w, int g,
                                             int m, const T* dv) {
  int64_t o = 0;
  if constexpr (S > 0) {
#pragma unroll
    for (int k = 0; k < S; ++k) o += (int64_t)dv[k];
  } else {
    const uint32_t e = w.gt[g];
    const int cfg = (int)(e & 0xFFFFu), s = (int)(e >> 24);
    const int64_t* d = P.pr.stage + ((int64_t)m * P.pr.P + cfg) * P.pr.S;
    for (int k = 0; k < s; ++k) o += __ldg(d + k);
  }
  return o;
}

// Statistics row of (chunk j, batch candidate c): counts += sign for model m,
// busy += sign * occ for group g.  Fire-and-forget reductions (no return).
__device__ __forceinline__ void stat_add(int32_t* pm, int64_t* busy, const ChunkParams& P, int j,
                                         int64_t c, int m, int g, int64_t occ, int sign) {
  const int64_t row = (int64_t)j * P.stat_C + c;
  atomicAdd(pm + row * P.pr.M + m, sign);
  atomicAdd(reinterpret_cast<unsigned long long*>(busy + row * P.bt.G + g),
            (unsigned long long)(sign * occ));
}

// Walk: the correction row of (j, c) restarts at minus pass 1's counts.
__device__ __forceinline__ void stat_reset(const ChunkParams& P, int j, int64_t c, int lane,
                                           int stride) {
  const int64_t row = (int64_t)j * P.stat_C + c;
  for (int m = lane; m < P.pr.M; m += stride)
    P.fix_pm[row * P.pr.M + m] = -P.spec_pm[row * P.pr.M + m];
  for (int g = lane; g < P.bt.G; g += stride)
    P.fix_busy[row * P.bt.G + g] = -P.spec_busy[row * P.bt.G + g];
}

template <typename T>
__device__ __forceinline__ void rebase(T* st, int slots, int lane, T delta) {
  for (int k = 0; k < slots; ++k) {
    const T v = st[k * 32 + lane];
    st[k * 32 + lane] = v > delta ? v - delta : (T)0;
  }
}

// Move the epoch to E_new >= E unconditionally (uint32 only; warp-uniform).
template <typename T, int MODE>
__device__ __forceinline__ void rebase_to(WarpMem<T>& w, int slots, int lane, int64_t E_new,
                                          int64_t& E) {
  if constexpr (TT<T>::kRel) {
    if (E_new > E) {
      const int64_t gap = E_new - E;
      const T delta = gap >= 0xFFFFFFFFll ? (T)0xFFFFFFFFu : (T)gap;
      rebase<T>(w.st0, slots, lane, delta);
      if constexpr (MODE == DUAL) rebase<T>(w.st1, slots, lane, delta);
      E = E_new;
    }
  }
}

// Move the epoch to arrival a if a - E > theta (uint32 only; warp-uniform).
template <typename T, int MODE>
__device__ __forceinline__ void maybe_rebase(const ChunkParams& P, WarpMem<T>& w, int slots,
                                             int lane, int64_t a, int64_t& E) {
  if constexpr (TT<T>::kRel) {
    if (a - E > P.theta) {
      // every stored value is < 2^32 - 1, so a longer gap clears them all
      const int64_t gap = a - E;
      const T delta = gap >= 0xFFFFFFFFll ? (T)0xFFFFFFFFu : (T)gap;
      rebase<T>(w.st0, slots, lane, delta);
      if constexpr (MODE == DUAL) rebase<T>(w.st1, slots, lane, delta);
      E = a;
    }
  }
}

// Load a stored state (relative to epoch Ep, or absolute) into `dst` at epoch E.
template <typename T>
__device__ __forceinline__ void load_state(T* dst, const T* src, int64_t Ep, int64_t E, int slots,
                                           int lane) {
  for (int k = 0; k < slots; ++k) {
    const T v = src[k * 32 + lane];
    if constexpr (TT<T>::kRel) {
      const int64_t r = (int64_t)v - (E - Ep);
      dst[k * 32 + lane] = r > 0 ? (T)r : (T)0;
    } else {
      dst[k * 32 + lane] = v;
    }
  }
}

// Store `slots` values of column `lane` relative to the unit's canonical epoch
// Ec (the chunk's last arrival; every writer of a unit uses it, whatever its
// own epoch E <= Ec was: clamping below Ec is exact by the equivalence).
template <typename T>
__device__ __forceinline__ void store_state(T* out, const T* st, int64_t E, int64_t Ec, int slots,
                                            int lane, int col) {
  for (int k = 0; k < slots; ++k) {
    const T v = st[k * 32 + lane];
    if constexpr (TT<T>::kRel) {
      const int64_t r = (int64_t)v - (Ec - E);
      out[k * 32 + col] = r > 0 ? (T)r : (T)0;
    } else {
      out[k * 32 + col] = v;
    }
  }
}

// Simulate one unit (item, chunk j) in MODE.  Returns (WALK) whether the true
// end state is equivalent to the stored speculative end state of chunk j.
template <typename T, int S, int MODE>
__device__ __forceinline__ uint32_t run_unit(const ChunkParams& P, WarpMem<T>& w, const ItemDesc& it,
                                             int item, int j, int lane, uint32_t srcmask) {
  const int64_t i_begin = P.chunk_begin[j], i_end = P.chunk_begin[j + 1];
  const bool in_item = lane < it.count;
  const int64_t c = in_item ? cand_of(P, it, item, lane) : 0;
  const int my_m = in_item ? P.bt.cand_model[c] : -1;
  const int my_g = in_item ? P.bt.cand_group[c] : 0;
  const bool active = in_item && P.bt.cand_ok[c];
  const int my_off = my_g * (S > 0 ? S : 1) * 32 * (int)sizeof(T);  // S > 0: byte offset of its first slot
  const int slots = it.slots;
  const int M = P.pr.M;
  const int64_t slot_id = (int64_t)item * 32 + lane;
  const int64_t unit = (int64_t)j * P.num_items + item;
  // the lane's own component (models simulated, groups compared); all else
  // evolves exactly like the base placement
  const bool restrict_k = P.bt.cand_kmask != nullptr;
  const uint64_t kmask = (restrict_k && in_item) ? P.bt.cand_kmask[c] : ~0ull;
  const uint64_t gmask = (P.bt.cand_gmask && in_item) ? P.bt.cand_gmask[c] : ~0ull;

  // relevance: models some active lane simulates
  if (restrict_k) {
    const uint64_t km = active ? kmask : 0ull;
    const uint64_t un = ((uint64_t)__reduce_or_sync(FULL, (uint32_t)(km >> 32)) << 32) |
                        __reduce_or_sync(FULL, (uint32_t)km);
    for (int m = lane; m < M; m += 32) w.rel[m] = (m < 64) && ((un >> m) & 1ull);
  } else {
    for (int m = lane; m < M; m += 32) w.rel[m] = w.hoff[m + 1] != w.hoff[m];
    __syncwarp();
    if (active && my_m >= 0) w.rel[my_m] = 1;
  }

  // uniform configs: per model the lanes that simulate its requests (active,
  // model in the lane's component, and the model able to meet its SLO at all
  // under this config: slo >= tail [+ d0 for S == 1]), so a request's
  // liveness is one broadcast load; the walkers' hosting-mask region holds it
  uint32_t* lmask = reinterpret_cast<uint32_t*>(w.hmask);
  // uniform configs: the config's stage-latency rows [M][kSTab] (global, L1)
  const T* dt = nullptr;
  if constexpr (S > 0)
    dt = reinterpret_cast<const T*>(sizeof(T) == 4 ? (const void*)P.pr.dtab32
                                                   : (const void*)P.pr.dtab64) +
         (int64_t)it.cfg * M * kSTab;
  if constexpr (S > 0) {
    for (int m = 0; m < M; ++m) {
      const T sl = w.slo[m], tl = w.tail[m];
      const bool nev = sl < tl || (S == 1 && (T)(sl - tl) < __ldg(dt + m * kSTab));
      const bool l = active && !nev && (!restrict_k || (m < 64 && ((kmask >> m) & 1ull)));
      const unsigned b = __ballot_sync(FULL, l);
      if (lane == 0) lmask[m] = b;
    }
  }
  const bool stats_on = P.spec_pm != nullptr;

  // initial states
  int64_t E = TT<T>::kRel ? P.tr.arrival[i_begin] : 0;
  if constexpr (MODE != WALK) {  // the speculative trajectory
    T* spec_st = (MODE == DUAL) ? w.st1 : w.st0;
    if (P.spec_state != nullptr && j > 0) {
      const int64_t* ss =
          (P.spec_cand && in_item)
              ? P.spec_cand + ((int64_t)c * P.J + j) * P.state_stride
              : P.spec_state + ((int64_t)P.spec_row[it.base] * P.J + j) * P.state_stride;
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
  }
  if constexpr (MODE == WALK) {
    if (P.fix_pm && active) stat_reset(P, j, c, 0, 1);  // this lane's own row
  }
  if constexpr (MODE != SPEC) {  // the true trajectory: true end of chunk j-1 (per lane)
    const int64_t prev = unit - P.num_items;
    const bool src = (srcmask >> lane) & 1u;
    const T* s0 = reinterpret_cast<const T*>(src ? P.fix_end : P.spec_end) + prev * P.slots_max * 32;
    load_state<T>(w.st0, s0, (src ? P.fix_epoch : P.spec_epoch)[prev], E, slots, lane);
  }
  __syncwarp();

  int64_t good0 = 0, sum0 = 0, good1 = 0, sum1 = 0;
  unsigned long long upd = 0;
  uint32_t upd32 = 0;  // hosts evaluated (S > 0) / stage updates (S == 0) by this lane
  bool coalesced = false;
  T dv[S > 0 ? S : 1];
  // 4-deep ring of trace tiles in registers: a lone warp (the walk) would
  // otherwise stall on the L2 latency of every tile.  The trace is padded
  // by >= 160 records (asim_set_trace), so the look-ahead stays in bounds.
  int64_t pa0 = P.tr.arrival[i_begin + lane], pa1 = P.tr.arrival[i_begin + 32 + lane];
  int64_t pa2 = P.tr.arrival[i_begin + 64 + lane], pa3 = P.tr.arrival[i_begin + 96 + lane];
  int pm0 = P.tr.model[i_begin + lane], pm1 = P.tr.model[i_begin + 32 + lane];
  int pm2 = P.tr.model[i_begin + 64 + lane], pm3 = P.tr.model[i_begin + 96 + lane];
  for (int64_t i0 = i_begin; i0 < i_end; i0 += 32) {
    const bool valid = i0 + lane < i_end;
    const int64_t ai = valid ? pa0 : 0;
    const int mi = valid ? pm0 : 0;
    pa0 = pa1;
    pa1 = pa2;
    pa2 = pa3;
    pm0 = pm1;
    pm1 = pm2;
    pm2 = pm3;
    pa3 = P.tr.arrival[i0 + 128 + lane];
    pm3 = P.tr.model[i0 + 128 + lane];
    if constexpr (MODE == DUAL) {
      if (((i0 - i_begin) % kCheckEvery) == 0) {
        const int64_t a0 = __shfl_sync(FULL, ai, 0);
        maybe_rebase<T, MODE>(P, w, slots, lane, a0, E);
        const T ar = (T)(a0 - E);
        bool eq = true;
        for (int k = 0; k < slots; ++k)
          if ((gmask >> w.sgrp[k]) & 1ull)
            eq &= tmax(w.st0[k * 32 + lane], ar) == tmax(w.st1[k * 32 + lane], ar);
        if (__all_sync(FULL, eq || !active)) {
          coalesced = true;
          break;
        }
      }
    }
    unsigned todo = __ballot_sync(FULL, valid && w.rel[mi]);
    if (!todo) continue;  // no lane hosts any of these 32 requests
    // one epoch for the whole tile when its relevant arrivals fit under theta
    // (moving the epoch early is exact: any E <= the next arrival works)
    bool per_req = false;
    if constexpr (TT<T>::kRel) {
      const int64_t a_last = __shfl_sync(FULL, ai, 31 - __clz(todo));
      if (a_last - E > P.theta) {
        const int64_t a_first = __shfl_sync(FULL, ai, __ffs(todo) - 1);
        rebase_to<T, MODE>(w, slots, lane, a_first, E);
        per_req = a_last - E > P.theta;  // a sparse tile: fall back to per-request epochs
      }
    }
    if constexpr (S > 0) {
      // Uniform config (every group runs the run's config): per-request fields
      // computed lane-parallel once per tile, then broadcast by shuffles.
      //   lim  accept iff the winner's last departure (S > 1) / max(v, a)
      //        (S == 1) is <= lim  (= a + slo - tail [- d0], saturated)
      //   cc   latency = that value + cc  (tail - a [+ d0], mod 2^bits of T)
      //   hA, hB  byte offsets of the first four hosts' first stage slots
      //   h0c  list start | count << 16 | never-acceptable << 23
      const T ar_l = (T)(ai - E);
      T lim_l, cc_l, d0_l;
      int hA_l, hB_l, h0c_l;
      uniform_fields<T, S>(w, dt, mi, ar_l, lim_l, cc_l, d0_l, hA_l, hB_l, h0c_l);
      // compaction: lane k gathers the fields of the tile's k-th relevant
      // request (src = the k-th set bit of todo, by a 5-step popcount select),
      // so the per-request loop below broadcasts from lane k with a plain
      // counter -- no find-first-set on its loop-carried chain
      const int nreq = __popc(todo);
      const int src = nth_set_bit(todo, lane);
      const int mi_c = __shfl_sync(FULL, mi, src);
      const T ar_c = __shfl_sync(FULL, ar_l, src), lim_c = __shfl_sync(FULL, lim_l, src);
      const T cc_c = __shfl_sync(FULL, cc_l, src), d0_c = __shfl_sync(FULL, d0_l, src);
      const int hA_c = __shfl_sync(FULL, hA_l, src), hB_c = __shfl_sync(FULL, hB_l, src);
      const int h0c_c = __shfl_sync(FULL, h0c_l, src);
      // the request loop comes in two copies: without the per-request epoch
      // branch (dense tiles, the rule) and with it (sparse tiles)
      auto request = [&](int k, auto sparse, auto stats) {
        const int cm = __shfl_sync(FULL, mi_c, k);
        T car = __shfl_sync(FULL, ar_c, k);
        T lim = __shfl_sync(FULL, lim_c, k);
        T cc = __shfl_sync(FULL, cc_c, k);
        int hA = __shfl_sync(FULL, hA_c, k), hB = __shfl_sync(FULL, hB_c, k);
        int h0c = __shfl_sync(FULL, h0c_c, k);
        if constexpr (S == 1) {
          dv[0] = __shfl_sync(FULL, d0_c, k);
        } else {
          load_dv<T, S>(dt + cm * kSTab, dv);
        }
        if constexpr (TT<T>::kRel && decltype(sparse)::value) {
          // sparse tile: per-request epochs, fields recomputed (rare)
          const int64_t a = __shfl_sync(FULL, ai, __shfl_sync(FULL, src, k));
          maybe_rebase<T, MODE>(P, w, slots, lane, a, E);
          car = (T)(a - E);
          T d0x;
          uniform_fields<T, S>(w, dt, cm, car, lim, cc, d0x, hA, hB, h0c);
        }
        const bool live = (lmask[cm] >> lane) & 1u;
        const bool mine = live && cm == my_m;
        T v0;
        int bo0;
        if (step_u<T, S, MODE == DUAL>(w, w.st0, lane, hA, hB, h0c, mine, my_off, live, car, dv, lim, v0, bo0)) {
          ++good0;
          sum0 += (int64_t)(T)(v0 + cc);
          if constexpr (decltype(stats)::value) {  // SPEC: pass-1 counts; DUAL: the true side
            const int g0 = bo0 / (S * 32 * (int)sizeof(T));
            if constexpr (MODE == SPEC)
              stat_add(P.spec_pm, P.spec_busy, P, j, c, cm, g0, occupancy<T, S>(P, w, g0, cm, dv), 1);
            else
              stat_add(P.fix_pm, P.fix_busy, P, j, c, cm, g0, occupancy<T, S>(P, w, g0, cm, dv), 1);
          }
        }
        if (active) upd32 += (uint32_t)((h0c >> 16) & 0x7F) + (mine ? 1u : 0u);
        if constexpr (MODE == DUAL) {
          T v1;
          int bo1;
          if (step_u<T, S, MODE == DUAL>(w, w.st1, lane, hA, hB, h0c, mine, my_off, live, car, dv, lim, v1, bo1)) {
            ++good1;
            sum1 += (int64_t)(T)(v1 + cc);
            if constexpr (decltype(stats)::value) {  // minus the speculative side
              const int g1 = bo1 / (S * 32 * (int)sizeof(T));
              stat_add(P.fix_pm, P.fix_busy, P, j, c, cm, g1, occupancy<T, S>(P, w, g1, cm, dv), -1);
            }
          }
          if (active) upd32 += (uint32_t)((h0c >> 16) & 0x7F) + (mine ? 1u : 0u);
        }
      };
      // (and without the statistics rows of the fast heuristic unless asked)
      if (stats_on) {
        for (int k = 0; k < nreq; ++k) request(k, BoolC<true>{}, BoolC<true>{});
      } else if (per_req) {
        for (int k = 0; k < nreq; ++k) request(k, BoolC<true>{}, BoolC<false>{});
      } else {
        for (int k = 0; k < nreq; ++k) request(k, BoolC<false>{}, BoolC<false>{});
      }
      continue;
    }

    // Mixed configs (S == 0; uniform configs took the loop above, so the
    // S > 0 branches below are never executed -- they remain the round-1
    // formulation that step_u replaced):
    // lane-parallel per-request fields, broadcast below by independent shuffles
    const T ar_l = (T)(ai - E);
    const int h0_l = w.hoff[mi];
    const int cnt_l = w.hoff[mi + 1] - h0_l;
    // S > 0: the first two hosts' byte offsets; S == 0: their group ids
    const int hinfo_l = S > 0 ? ((cnt_l >= 1 ? (int)w.hid[h0_l] : 0) |
                                 (cnt_l >= 2 ? (int)w.hid[h0_l + 1] << 16 : 0))
                              : ((cnt_l >= 1 ? (int)w.hid[h0_l] : 0) |
                                 (cnt_l >= 2 ? (int)w.hid[h0_l + 1] << 8 : 0) | (cnt_l << 16));
    const int h0c_l = S > 0 ? (h0_l | (cnt_l << 16)) : h0_l;  // S > 0: list start | count
    const T sl_l = w.slo[mi];
    T tl_l = 0, d0_l = 0;
    if constexpr (S > 0) tl_l = w.tail[mi];
    if constexpr (S == 1) d0_l = w.d[mi * kSTab];
    // software pipeline: the next request's shuffles issue before this one
    // runs (staging the fields in shared memory instead costs a block of
    // occupancy: measured slower, profiles/r2b)
    int jj = __ffs(todo) - 1;
    todo &= todo - 1;
    int m = __shfl_sync(FULL, mi, jj);
    T ar = __shfl_sync(FULL, ar_l, jj);
    int hinfo = __shfl_sync(FULL, hinfo_l, jj), h0 = __shfl_sync(FULL, h0c_l, jj);
    T sl = __shfl_sync(FULL, sl_l, jj), tl = 0, d0 = 0;
    if constexpr (S > 0) tl = __shfl_sync(FULL, tl_l, jj);
    if constexpr (S == 1) d0 = __shfl_sync(FULL, d0_l, jj);
    for (;;) {  // requests some lane hosts, in trace order
      const int cjj = jj, cm = m, chinfo = hinfo, ch0 = h0;
      T car = ar;
      const T csl = sl, ctl = tl;
      const bool more = todo != 0;
      if (more) {
        jj = __ffs(todo) - 1;
        todo &= todo - 1;
        m = __shfl_sync(FULL, mi, jj);
        ar = __shfl_sync(FULL, ar_l, jj);
        hinfo = __shfl_sync(FULL, hinfo_l, jj);
        h0 = __shfl_sync(FULL, h0c_l, jj);
        sl = __shfl_sync(FULL, sl_l, jj);
        if constexpr (S > 0) tl = __shfl_sync(FULL, tl_l, jj);
      }
      if constexpr (S == 1) {
        dv[0] = d0;
        if (more) d0 = __shfl_sync(FULL, d0_l, jj);
      } else if constexpr (S > 1) {
#pragma unroll
        for (int k = 0; k < S; ++k) dv[k] = w.d[cm * kSTab + k];
      }
      if constexpr (TT<T>::kRel) {
        if (per_req) {
          const int64_t a = __shfl_sync(FULL, ai, cjj);
          maybe_rebase<T, MODE>(P, w, slots, lane, a, E);
          car = (T)(a - E);
        }
      }
      const bool live = active && ((kmask >> (cm & 63)) & 1ull);
      const bool mine = live && cm == my_m;
      int g0 = 0, g1 = 0;
      const int64_t l0 = step<T, S>(P, w, w.st0, lane, cm, chinfo, ch0, mine, my_g, live, car,
                                    dv, ctl, csl, upd32, g0);
      if (l0 >= 0) {
        ++good0;
        sum0 += l0;
        if (P.spec_pm) {  // SPEC: pass-1 counts; DUAL / WALK: the true side of the correction
          if constexpr (MODE == SPEC)
            stat_add(P.spec_pm, P.spec_busy, P, j, c, cm, g0, occupancy<T, S>(P, w, g0, cm, dv), 1);
          else
            stat_add(P.fix_pm, P.fix_busy, P, j, c, cm, g0, occupancy<T, S>(P, w, g0, cm, dv), 1);
        }
      }
      if constexpr (MODE == DUAL) {
        const int64_t l1 = step<T, S>(P, w, w.st1, lane, cm, chinfo, ch0, mine, my_g, live,
                                      car, dv, ctl, csl, upd32, g1);
        if (l1 >= 0) {
          ++good1;
          sum1 += l1;
          if (P.spec_pm)  // minus the speculative side
            stat_add(P.fix_pm, P.fix_busy, P, j, c, cm, g1, occupancy<T, S>(P, w, g1, cm, dv), -1);
        }
      }
      if (!more) break;
    }
  }

  // pass 1's work is counted on the host (chunked.cpp: it is fixed by the
  // candidates' components); passes 2-3 count what they re-simulate
  if constexpr (MODE != SPEC) {
    if (P.stage_updates) {
      upd += (unsigned long long)upd32 * (S > 0 ? S : 1);
      for (int o = 16; o > 0; o >>= 1) upd += __shfl_down_sync(FULL, upd, o);
      if (lane == 0) atomicAdd(P.stage_updates, upd);
    }
  }
  const int64_t cstride = (int64_t)P.num_items * 32;
  const int64_t Ec = P.tr.arrival[i_end - 1];  // the unit's canonical epoch
  uint32_t eqmask = FULL;
  if constexpr (MODE == SPEC) {
    P.spec_good[j * cstride + slot_id] = (int32_t)good0;
    P.spec_sum[j * cstride + slot_id] = sum0;
    if (j + 1 < P.J) {  // end state for the next chunk's fix-up
      store_state<T>(reinterpret_cast<T*>(P.spec_end) + unit * P.slots_max * 32, w.st0, E, Ec,
                     slots, lane, lane);
      if (lane == 0) P.spec_epoch[unit] = Ec;
    }
  } else if constexpr (MODE == DUAL) {
    P.fix_good[j * cstride + slot_id] = (int32_t)(good0 - good1);
    P.fix_sum[j * cstride + slot_id] = sum0 - sum1;
    uint32_t flag = 0;
    if (!coalesced && j + 1 < P.J) {
      // lanes whose trajectories differ at the next arrival; publish the true ends
      const int64_t a_next = P.tr.arrival[i_end];
      bool eq = true;
      for (int k = 0; k < slots; ++k) {
        if (!((gmask >> w.sgrp[k]) & 1ull)) continue;
        const int64_t t0 = (TT<T>::kRel ? E : 0) + (int64_t)w.st0[k * 32 + lane];
        const int64_t t1 = (TT<T>::kRel ? E : 0) + (int64_t)w.st1[k * 32 + lane];
        eq &= (t0 > a_next ? t0 : a_next) == (t1 > a_next ? t1 : a_next);
      }
      flag = __ballot_sync(FULL, !eq && active);
      store_state<T>(reinterpret_cast<T*>(P.fix_end) + unit * P.slots_max * 32, w.st0, E, Ec,
                     slots, lane, lane);
      if (lane == 0) P.fix_epoch[unit] = Ec;
    }
    if (lane == 0) P.fix_flag[unit] = flag;
  } else {  // WALK: exact correction of the whole chunk, every lane from its true start
    P.fix_good[j * cstride + slot_id] = (int32_t)(good0 - P.spec_good[j * cstride + slot_id]);
    P.fix_sum[j * cstride + slot_id] = sum0 - P.spec_sum[j * cstride + slot_id];
    if (j + 1 < P.J) {
      // equivalent to the speculative end at the next arrival?  (absolute times)
      const int64_t a_next = P.tr.arrival[i_end];
      const T* se = reinterpret_cast<const T*>(P.spec_end) + unit * P.slots_max * 32;
      const int64_t Es = P.spec_epoch[unit];
      bool eq = true;
      for (int k = 0; k < slots; ++k) {
        if (!((gmask >> w.sgrp[k]) & 1ull)) continue;
        const int64_t t0 = (TT<T>::kRel ? E : 0) + (int64_t)w.st0[k * 32 + lane];
        const int64_t t1 = (TT<T>::kRel ? Es : 0) + (int64_t)se[k * 32 + lane];
        eq &= (t0 > a_next ? t0 : a_next) == (t1 > a_next ? t1 : a_next);
      }
      eqmask = __ballot_sync(FULL, eq || !active);
      if (eqmask != FULL) {
        store_state<T>(reinterpret_cast<T*>(P.fix_end) + unit * P.slots_max * 32, w.st0, E, Ec,
                       slots, lane, lane);
        if (lane == 0) P.fix_epoch[unit] = Ec;
      }
    }
  }
  return eqmask;
}

template <typename T, int MODE>
__device__ __forceinline__ uint32_t dispatch_unit(const ChunkParams& P, WarpMem<T>& w,
                                                  const ItemDesc& it, int item, int j, int lane,
                                                  uint32_t src) {
  switch (it.S) {
    case 1: return run_unit<T, 1, MODE>(P, w, it, item, j, lane, src);
    case 2: return run_unit<T, 2, MODE>(P, w, it, item, j, lane, src);
    case 4: return run_unit<T, 4, MODE>(P, w, it, item, j, lane, src);
    case 8: return run_unit<T, 8, MODE>(P, w, it, item, j, lane, src);
    case 16: return run_unit<T, 16, MODE>(P, w, it, item, j, lane, src);
    default: return run_unit<T, 0, MODE>(P, w, it, item, j, lane, src);
  }
}

__device__ __forceinline__ int next_unit(const ChunkParams& P, int lane) {
  int u = 0;
  if (lane == 0) u = (int)atomicAdd(P.counter, 1u);
  return __shfl_sync(FULL, u, 0);
}

// Passes 1 and 2: persistent warps pulling (item, chunk) units.
// MINB blocks per SM: pass 1 5 (20 warps, <= 96 registers; measured: 8, 12,
// 16 warps per SM gave pass 1 29.4, 21.1, 17.5 s on the day search,
// profiles/r2l/prof_pad_*); pass 2 3 (two state regions per warp: shared
// memory holds 3 blocks, so it keeps its registers).
template <typename T, int MODE, int MINB>
__global__ void __launch_bounds__(kWarps * 32, MINB) chunk_kernel(ChunkParams P) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const size_t wb = warp_bytes(P.slots_max, P.pr.M, P.hid_cap, sizeof(T), MODE == DUAL, false);
  WarpMem<T> w = carve<T>(smem + warp * wb, P, MODE == DUAL, false);
  int cur_base = -1;
  for (;;) {
    const int u = next_unit(P, lane);
    if (u >= P.num_units) break;
    int item = u % P.num_items;
    int j = (MODE == DUAL ? 1 : 0) + u / P.num_items;  // chunk-major
    if (P.item_perm) {  // class by class, chunk-major inside a class
      const int jn = P.J - (MODE == DUAL ? 1 : 0);
      int c = 0;
      while (c + 1 < P.nclass && u >= jn * (P.class_off[c] + P.class_items[c])) ++c;
      const int local = u - jn * P.class_off[c];
      j = (MODE == DUAL ? 1 : 0) + local / P.class_items[c];
      item = P.item_perm[P.class_off[c] + local % P.class_items[c]];
    }
    const ItemDesc it = P.items[item];
    const long long t0 = (MODE == SPEC && P.walked) ? clock64() : 0;
    if (it.base != cur_base) {
      load_base<T>(P, it, w, lane);
      cur_base = it.base;
    }
    dispatch_unit<T, MODE>(P, w, it, item, j, lane, 0);
    __syncwarp();
    if (MODE == SPEC && P.walked && lane == 0) {  // profiling: warp cycles per stage class
      const int cls = it.S == 1 ? 1 : it.S == 2 ? 2 : it.S == 4 ? 3 : it.S == 8 ? 4 : it.S == 16 ? 5 : 0;
      atomicAdd(P.walked + 4 + cls, (unsigned long long)(clock64() - t0));
    }
  }
}

// Pass 3, items with mixed configs (S == 0): one warp per item walks the
// chunks in order; where some lane's start state was wrong, every lane is
// re-simulated from its true start.  end_src[u] gets the lanes whose true end
// is in fix_end.  Items of uniform configs are walked by coop_walk_kernel.
template <typename T>
__global__ void __launch_bounds__(kWarps * 32) walk_kernel(ChunkParams P, uint32_t* end_src) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const size_t wb = warp_bytes(P.slots_max, P.pr.M, P.hid_cap, sizeof(T), false);
  WarpMem<T> w = carve<T>(smem + warp * wb, P, false);
  int cur_base = -1;
  for (;;) {
    const int item = next_unit(P, lane);
    if (item >= P.num_items) break;
    const ItemDesc it = P.items[item];
    if (it.S != 0) continue;  // warp-uniform
    uint32_t start_ok = FULL;  // lanes whose pass-2 start (chunk j-1's spec end) was true
    unsigned long long walked = 0;
    for (int j = 1; j < P.J; ++j) {
      const int64_t u = (int64_t)j * P.num_items + item;
      if (start_ok == FULL) {  // pass 2's corrections of chunk j are exact for every lane
        const uint32_t f = P.fix_flag[u];
        if (lane == 0) end_src[u] = f;
        start_ok = ~f;
        continue;
      }
      if (it.base != cur_base) {
        load_base<T>(P, it, w, lane);
        cur_base = it.base;
      }
      ++walked;
      const uint32_t eq = dispatch_unit<T, WALK>(P, w, it, item, j, lane, end_src[u - P.num_items]);
      if (lane == 0) end_src[u] = ~eq;
      start_ok = eq;
      __syncwarp();
    }
    if (P.walked && lane == 0 && walked) {
      atomicAdd(P.walked, walked);
      atomicAdd(P.walked + 1, 1ull);
      atomicMax(P.walked + 2, walked);
    }
  }
}

// ---------------------------------------------------------------------------
// Pass 3, uniform configs: the warp-cooperative walker.  One warp per
// CANDIDATE that needs walking; its state is spread over the lanes in
// registers (slot t = lane + 32 q lives in v[q]), so a request costs a few
// register ops, one warp-wide min and one ballot instead of a 32-lane
// dependent chain through shared memory.  Within a group the S stages sit in
// S consecutive lanes (32 % S == 0) and the tandem recurrence
//     y_k = max(y_{k-1}, free_k) + d_k,  y_{-1} = a
// is evaluated as a max-plus scan: element k = (A_k, B_k) = (d_k, free_k + d_k),
// (A1, B1) then (A2, B2) = (A1 + A2, max(B1 + A2, B2)), y_k = max(a + A, B).
template <typename T>
__device__ __forceinline__ T warp_min(T v) {
  if constexpr (sizeof(T) == 4) {
    return (T)__reduce_min_sync(FULL, (unsigned)v);
  } else {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const T x = __shfl_xor_sync(FULL, v, o);
      v = x < v ? x : v;
    }
    return v;
  }
}

// One warp simulates ONE candidate over requests [i_begin, i_end): state v
// (slot = lane + 32 q) in registers, epoch E (uint32 mode).  STATS adds the
// fast heuristic's outputs: per-model good counts (pm_row[M]) and per-group
// busy time (busy_row[G]), global rows updated by fire-and-forget atomics.
template <typename T, int S, int Q, bool STATS>
__device__ __forceinline__ void coop_range(const ChunkParams& P, const WarpMem<T>& w,
                                           int64_t i_begin, int64_t i_end, T (&v)[Q], int64_t& E,
                                           uint64_t kmask, int my_m, uint64_t my_bit,
                                           const uint64_t (&lastbit)[Q], int lane, int64_t& good,
                                           int64_t& sum, unsigned long long& upd,
                                           int32_t* pm_row, int64_t* busy_row) {
  // the next tile's records load one tile ahead (the walk is one warp on a
  // dependent chain: an L2 round trip per tile would sit on it)
  int64_t al_n = i_begin + lane < i_end ? P.tr.arrival[i_begin + lane] : 0;
  int ml_n = i_begin + lane < i_end ? (int)P.tr.model[i_begin + lane] : 0;
  for (int64_t i0 = i_begin; i0 < i_end; i0 += 32) {
    const bool valid = i0 + lane < i_end;
    const int64_t al = valid ? al_n : 0;
    const int ml = valid ? ml_n : 0;
    if (i0 + 32 + lane < i_end) {
      al_n = P.tr.arrival[i0 + 32 + lane];
      ml_n = (int)P.tr.model[i0 + 32 + lane];
    }
    unsigned todo = __ballot_sync(FULL, valid && ((kmask >> (ml & 63)) & 1ull));
    if (!todo) continue;
    bool per_req = false;
    if constexpr (TT<T>::kRel) {
      const int64_t a_last = __shfl_sync(FULL, al, 31 - __clz(todo));
      if (a_last - E > P.theta) {  // move the epoch to the tile's first request
        const int64_t a_first = __shfl_sync(FULL, al, __ffs(todo) - 1);
        const int64_t gap = a_first - E;
        const T delta = gap >= 0xFFFFFFFFll ? (T)0xFFFFFFFFu : (T)gap;
#pragma unroll
        for (int q = 0; q < Q; ++q) v[q] = v[q] > delta ? v[q] - delta : (T)0;
        E = a_first;
        per_req = a_last - E > P.theta;
      }
    }
    // lane-parallel per-request fields of the tile, broadcast by independent
    // shuffles (no shared-memory load on the per-request dependent chain)
    const T arl = (T)(al - E);
    const uint64_t hml = w.hmask[ml] | (ml == my_m ? my_bit : 0ull);
    const T tll = w.tail[ml], sll = w.slo[ml];
    T dkl = 0;
    if constexpr (S == 1) dkl = w.d[ml * kSTab];
    int64_t occl = 0;  // sum_k d_k of the lane's request (STATS)
    if constexpr (STATS) {
#pragma unroll
      for (int k = 0; k < S; ++k) occl += (int64_t)w.d[ml * kSTab + k];
    }
    if (P.stage_updates) {  // statistics only (warp-uniform)
      const bool rel = (todo >> lane) & 1u;
      upd += (unsigned long long)__reduce_add_sync(FULL, rel ? (unsigned)__popcll(hml) : 0u) * S;
    }
    // software pipeline: the next request's shuffles issue before this
    // request's dependent chain
    int njj = __ffs(todo) - 1;
    todo &= todo - 1;
    int nm = __shfl_sync(FULL, ml, njj);
    T nar = __shfl_sync(FULL, arl, njj);
    uint64_t nhm = __shfl_sync(FULL, hml, njj);
    T ntl = __shfl_sync(FULL, tll, njj), nsl = __shfl_sync(FULL, sll, njj), ndk = 0;
    if constexpr (S == 1) ndk = __shfl_sync(FULL, dkl, njj);
    for (;;) {
      const int jj = njj, m = nm;
      T ar = nar;
      const uint64_t hm = nhm;
      const T tl = ntl, sl = nsl, dk = ndk;
      const bool more = todo != 0;
      if (more) {
        njj = __ffs(todo) - 1;
        todo &= todo - 1;
        nm = __shfl_sync(FULL, ml, njj);
        nar = __shfl_sync(FULL, arl, njj);
        nhm = __shfl_sync(FULL, hml, njj);
        ntl = __shfl_sync(FULL, tll, njj);
        nsl = __shfl_sync(FULL, sll, njj);
        if constexpr (S == 1) ndk = __shfl_sync(FULL, dkl, njj);
      }
      if constexpr (TT<T>::kRel) {
        if (per_req) {
          const int64_t a = __shfl_sync(FULL, al, jj);
          if (a - E > P.theta) {
            const int64_t gap = a - E;
            const T delta = gap >= 0xFFFFFFFFll ? (T)0xFFFFFFFFu : (T)gap;
#pragma unroll
            for (int q = 0; q < Q; ++q) v[q] = v[q] > delta ? v[q] - delta : (T)0;
            E = a;
          }
          ar = (T)(a - E);
        }
      }
      // predicted finish at the last stage of every hosting group
      T y[Q], f[Q];
      T fl = TT<T>::maxv();
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        if constexpr (S == 1) {
          y[q] = tmax(ar, v[q]) + dk;
        } else {
          const int k = (lane + 32 * q) % S;
          const T d = w.d[m * kSTab + k];
          T A = d, B = v[q] + d;
#pragma unroll
          for (int o = 1; o < S; o <<= 1) {
            const T A2 = __shfl_up_sync(FULL, A, o, S), B2 = __shfl_up_sync(FULL, B, o, S);
            if (k >= o) {
              B = tmax(B2 + A, B);
              A = A2 + A;
            }
          }
          y[q] = tmax(ar + A, B);
        }
        f[q] = (hm & lastbit[q]) ? y[q] + tl : TT<T>::maxv();
        fl = tmin(fl, f[q]);
      }
      const T fmin = warp_min<T>(fl);
      if (fmin != TT<T>::maxv() && (T)(fmin - ar) <= sl) {  // else no host / misses the SLO
        // lowest group index among the minima (slots ascend with q, then lane)
        int wq = 0, wl = 0;
#pragma unroll
        for (int q = Q - 1; q >= 0; --q) {
          const unsigned b = __ballot_sync(FULL, f[q] == fmin);
          if (b) {
            wq = q;
            wl = __ffs(b) - 1;
          }
        }
        const int gw = (wl + 32 * wq) / S;
#pragma unroll
        for (int q = 0; q < Q; ++q)
          if (q == wq && (lane + 32 * q) / S == gw) v[q] = y[q];
        ++good;
        sum += (int64_t)(fmin - ar);
        if constexpr (STATS) {
          const int64_t occ = __shfl_sync(FULL, occl, jj);
          if (lane == 0) {
            atomicAdd(pm_row + m, 1);
            atomicAdd(reinterpret_cast<unsigned long long*>(busy_row + gw), (unsigned long long)occ);
          }
        }
      }
      if (!more) break;
    }
  }
}

template <typename T, int S, int Q>
__device__ __forceinline__ void coop_candidate(const ChunkParams& P, const WarpMem<T>& w,
                                               const ItemDesc& it, int item, int cl, int lane,
                                               uint32_t* end_src, unsigned long long& walked,
                                               unsigned long long& upd) {
  // Q = ceil(slots / 32) blocks of 32 slots; slot t = lane + 32 q
  const int64_t c = cand_of(P, it, item, cl);
  const int my_m = P.bt.cand_model[c], my_g = P.bt.cand_group[c];
  const uint64_t kmask = P.bt.cand_kmask ? P.bt.cand_kmask[c] : ~0ull;
  const uint64_t gmask = P.bt.cand_gmask ? P.bt.cand_gmask[c] : ~0ull;
  const uint64_t my_bit = my_m >= 0 ? (1ull << my_g) : 0ull;
  const int slots = it.slots;
  const int64_t cstride = (int64_t)P.num_items * 32;
  // per-lane slot facts: the group bit of a group's LAST stage (0 elsewhere)
  uint64_t lastbit[Q];
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    const int t = lane + 32 * q;
    lastbit[q] = (t < slots && t % S == S - 1) ? (1ull << ((t / S) & 63)) : 0ull;
  }
  bool start_ok = true;
  for (int j = 1; j < P.J; ++j) {
    const int64_t u = (int64_t)j * P.num_items + item;
    if (start_ok) {
      if ((P.fix_flag[u] >> cl) & 1u) {  // pass 2 exact; true end of j is its fix_end
        if (lane == 0) atomicOr(end_src + u, 1u << cl);
        start_ok = false;
      }
      continue;
    }
    ++walked;
    const int64_t i_begin = P.chunk_begin[j], i_end = P.chunk_begin[j + 1];
    int64_t E = TT<T>::kRel ? P.tr.arrival[i_begin] : 0;
    // true start: chunk j-1's true end, always in fix_end when walking
    T v[Q];
    {
      const int64_t prev = u - P.num_items;
      const T* s0 = reinterpret_cast<const T*>(P.fix_end) + prev * P.slots_max * 32;
      const int64_t Ep = P.fix_epoch[prev];
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        const int t = lane + 32 * q;
        T x = 0;
        if (t < slots) {
          const T raw = s0[t * 32 + cl];
          if constexpr (TT<T>::kRel) {
            const int64_t r = (int64_t)raw - (E - Ep);
            x = r > 0 ? (T)r : (T)0;
          } else {
            x = raw;
          }
        }
        v[q] = x;
      }
    }
    int64_t good = 0, sum = 0;
    if (P.fix_pm) {  // fast-heuristic statistics: this chunk's correction row restarts
      stat_reset(P, j, c, lane, 32);
      __syncwarp();
      const int64_t row = (int64_t)j * P.stat_C + c;
      coop_range<T, S, Q, true>(P, w, i_begin, i_end, v, E, kmask, my_m, my_bit, lastbit, lane,
                                good, sum, upd, P.fix_pm + row * P.pr.M,
                                P.fix_busy + row * P.bt.G);
    } else {
      coop_range<T, S, Q, false>(P, w, i_begin, i_end, v, E, kmask, my_m, my_bit, lastbit, lane,
                                 good, sum, upd, nullptr, nullptr);
    }
    // the chunk's exact correction, and equivalence with the speculative end
    if (lane == 0) {
      P.fix_good[j * cstride + (int64_t)item * 32 + cl] =
          (int32_t)(good - P.spec_good[j * cstride + (int64_t)item * 32 + cl]);
      P.fix_sum[j * cstride + (int64_t)item * 32 + cl] =
          sum - P.spec_sum[j * cstride + (int64_t)item * 32 + cl];
    }
    if (j + 1 < P.J) {
      const int64_t a_next = P.tr.arrival[i_end];
      const T* se = reinterpret_cast<const T*>(P.spec_end) + u * P.slots_max * 32;
      const int64_t Es = P.spec_epoch[u];
      bool eq = true;
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        const int t = lane + 32 * q;
        if (t >= slots || !((gmask >> ((t / S) & 63)) & 1ull)) continue;
        const int64_t t0 = (TT<T>::kRel ? E : 0) + (int64_t)v[q];
        const int64_t t1 = (TT<T>::kRel ? Es : 0) + (int64_t)se[t * 32 + cl];
        eq &= (t0 > a_next ? t0 : a_next) == (t1 > a_next ? t1 : a_next);
      }
      start_ok = __all_sync(FULL, eq);
      if (!start_ok) {  // publish column cl at the unit's canonical epoch
        const int64_t Ec = P.tr.arrival[i_end - 1];
        T* out = reinterpret_cast<T*>(P.fix_end) + u * P.slots_max * 32;
#pragma unroll
        for (int q = 0; q < Q; ++q) {
          const int t = lane + 32 * q;
          if (t >= slots) continue;
          if constexpr (TT<T>::kRel) {
            const int64_t r = (int64_t)v[q] - (Ec - E);
            out[t * 32 + cl] = r > 0 ? (T)r : (T)0;
          } else {
            out[t * 32 + cl] = v[q];
          }
        }
        if (lane == 0) {
          P.fix_epoch[u] = Ec;
          atomicOr(end_src + u, 1u << cl);
        }
      }
    }
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------
// Pass 3, small components: the scalar walker.  When the candidate's own
// component (cand_gmask) spans NG <= 32 groups with NG * S <= 32 stage slots,
// its state fits in registers of every lane (all lanes hold the same values
// and run the same code: no cross-lane operation sits on the per-request
// dependency chain).  Per request: S max-plus steps per group, an
// adjacent-pair argmin tree (blocks of ascending group ids, so the lower index
// wins ties as in C1), and predicated commits.  Requests of other components
// are skipped 32 at a time by a ballot, exactly as in the cooperative walker.
template <typename T, int S, int NG>
__device__ __forceinline__ void scalar_candidate(const ChunkParams& P, const WarpMem<T>& w,
                                                 const ItemDesc& it, int item, int cl, int lane,
                                                 uint32_t* end_src, unsigned long long& walked,
                                                 unsigned long long& upd) {
  constexpr int R = NG * S;
  const int64_t c = cand_of(P, it, item, cl);
  const int my_m = P.bt.cand_model[c], my_g = P.bt.cand_group[c];
  const uint64_t kmask = P.bt.cand_kmask ? P.bt.cand_kmask[c] : ~0ull;
  const int ngroups = it.slots / S;
  const uint64_t all = ngroups >= 64 ? ~0ull : ((1ull << ngroups) - 1ull);
  const uint64_t gmask = (P.bt.cand_gmask ? P.bt.cand_gmask[c] : ~0ull) & all;
  // compact group i -> group id (ascending), -1 = padding
  int cg[NG];
  {
    uint64_t b = gmask;
#pragma unroll
    for (int i = 0; i < NG; ++i) {
      cg[i] = b ? (__ffsll((long long)b) - 1) : -1;
      b &= b - 1;
    }
  }
  // compact hosting mask of every model (the cooperative walker leaves the
  // hosting-list region w.hid unused: it serves as scratch here)
  uint32_t* hmc = reinterpret_cast<uint32_t*>(w.hid);  // region >= 4 M bytes (hid_cap)
  for (int m = lane; m < P.pr.M; m += 32) {
    const uint64_t hm = w.hmask[m] | (m == my_m ? (1ull << my_g) : 0ull);
    uint32_t x = 0;
#pragma unroll
    for (int i = 0; i < NG; ++i)
      if (cg[i] >= 0 && ((hm >> cg[i]) & 1ull)) x |= 1u << i;
    hmc[m] = x;
  }
  __syncwarp();
  const int64_t cstride = (int64_t)P.num_items * 32;
  bool start_ok = true;
  for (int j = 1; j < P.J; ++j) {
    const int64_t u = (int64_t)j * P.num_items + item;
    if (start_ok) {
      if ((P.fix_flag[u] >> cl) & 1u) {  // pass 2 exact; true end of j is its fix_end
        if (lane == 0) atomicOr(end_src + u, 1u << cl);
        start_ok = false;
      }
      continue;
    }
    ++walked;
    const int64_t i_begin = P.chunk_begin[j], i_end = P.chunk_begin[j + 1];
    int64_t E = TT<T>::kRel ? P.tr.arrival[i_begin] : 0;
    // true start: chunk j-1's true end (fix_end), component slots only
    const int64_t prev = u - P.num_items;
    const T* s0 = reinterpret_cast<const T*>(P.fix_end) + prev * P.slots_max * 32;
    const int64_t Ep = P.fix_epoch[prev];
    T v[R];
#pragma unroll
    for (int i = 0; i < NG; ++i)
#pragma unroll
      for (int k = 0; k < S; ++k) {
        T x = 0;
        if (cg[i] >= 0) {
          const T raw = s0[(cg[i] * S + k) * 32 + cl];
          if constexpr (TT<T>::kRel) {
            const int64_t r = (int64_t)raw - (E - Ep);
            x = r > 0 ? (T)r : (T)0;
          } else {
            x = raw;
          }
        }
        v[i * S + k] = x;
      }
    int32_t* pm_row = nullptr;
    int64_t* busy_row = nullptr;
    if (P.fix_pm) {  // fast-heuristic statistics: this chunk's correction row restarts
      stat_reset(P, j, c, lane, 32);
      __syncwarp();
      const int64_t row = (int64_t)j * P.stat_C + c;
      pm_row = P.fix_pm + row * P.pr.M;
      busy_row = P.fix_busy + row * P.bt.G;
    }
    int64_t good = 0, sum = 0;
    // request fields one tile ahead (the tile loads leave the per-request chain)
    int64_t al_n = i_begin + lane < i_end ? P.tr.arrival[i_begin + lane] : 0;
    int ml_n = i_begin + lane < i_end ? (int)P.tr.model[i_begin + lane] : 0;
    for (int64_t i0 = i_begin; i0 < i_end; i0 += 32) {
      const bool valid = i0 + lane < i_end;
      const int64_t al = al_n;
      const int ml = ml_n;
      if (i0 + 32 + lane < i_end) {
        al_n = P.tr.arrival[i0 + 32 + lane];
        ml_n = (int)P.tr.model[i0 + 32 + lane];
      }
      unsigned todo = __ballot_sync(FULL, valid && ((kmask >> (ml & 63)) & 1ull));
      if (!todo) continue;
      bool per_req = false;
      if constexpr (TT<T>::kRel) {
        const int64_t a_last = __shfl_sync(FULL, al, 31 - __clz(todo));
        if (a_last - E > P.theta) {  // move the epoch to the tile's first request
          const int64_t a_first = __shfl_sync(FULL, al, __ffs(todo) - 1);
          const int64_t gap = a_first - E;
          const T delta = gap >= 0xFFFFFFFFll ? (T)0xFFFFFFFFu : (T)gap;
#pragma unroll
          for (int r = 0; r < R; ++r) v[r] = v[r] > delta ? v[r] - delta : (T)0;
          E = a_first;
          per_req = a_last - E > P.theta;
        }
      }
      const T arl = (T)(al - E);
      const uint32_t hml = hmc[ml];
      const T tll = w.tail[ml], sll = w.slo[ml];
      if (P.stage_updates) {  // statistics only (warp-uniform)
        const bool rel = (todo >> lane) & 1u;
        upd += (unsigned long long)__reduce_add_sync(FULL, rel ? (unsigned)__popc(hml) : 0u) * S;
      }
      if (!per_req && !pm_row) {
        // Dense tile: the tile's requests of the component, compacted in trace
        // order.  Each such lane stages its request's fields in shared memory
        // at its rank among them; the per-request loop reads them with
        // broadcast loads that do not depend on the state, so they issue
        // ahead of the dependent chain (requests outside the component are
        // never visited).  Accept iff the last departure x satisfies
        // x + tail - a <= slo, i.e. x <= lim = a + slo - tail (never when
        // slo < tail, since x >= a: hm = 0, no host).
        TileReq<T>* tq = reinterpret_cast<TileReq<T>*>(w.tile);
        const int nreq = __popc(todo);
        if ((todo >> lane) & 1u) {
          TileReq<T> q;
          q.ar = arl;
          q.hm = sll >= tll ? hml : 0u;
          q.lim = 0;
          if (sll >= tll) {  // saturating: an unbounded SLO must not wrap
            const T room = sll - tll;
            q.lim = room > (T)(TT<T>::maxv() - 1 - arl) ? (T)(TT<T>::maxv() - 1) : (T)(arl + room);
          }
          q.tl = tll;
#pragma unroll
          for (int k = 0; k < 4; ++k) q.d[k] = k < S ? w.d[ml * kSTab + k] : (T)0;
          q.m = ml;
          tq[__popc(todo & ((1u << lane) - 1u))] = q;
        }
        __syncwarp();
#pragma unroll 4
        for (int jj = 0; jj < nreq; ++jj) {
          const TileReq<T> q = tq[jj];
          T d[S];
          tile_dv<T, S>(q, w.d, d);
          T y[R];
          T val[NG];
          uint32_t oh[NG];  // one-hot winner (an index would turn the commit into local memory)
#pragma unroll
          for (int i = 0; i < NG; ++i) {
            T x = q.ar;
#pragma unroll
            for (int k = 0; k < S; ++k) {
              x = tmax(x, v[i * S + k]) + d[k];
              y[i * S + k] = x;
            }
            val[i] = (NG == 1 || ((q.hm >> i) & 1u)) ? x : TT<T>::maxv();
            oh[i] = 1u << i;
          }
          // argmin, lowest index on ties (blocks of ascending indices, C1)
#pragma unroll
          for (int st = 1; st < NG; st <<= 1)
#pragma unroll
            for (int i = 0; i + st < NG; i += 2 * st) {
              const bool p = val[i + st] < val[i];
              val[i] = p ? val[i + st] : val[i];
              oh[i] = p ? oh[i + st] : oh[i];
            }
          const bool acc = (NG > 1 || (q.hm & 1u)) && val[0] <= q.lim;
          const uint32_t win = acc ? oh[0] : 0u;
#pragma unroll
          for (int i = 0; i < NG; ++i)
#pragma unroll
            for (int k = 0; k < S; ++k)
              v[i * S + k] = (win & (1u << i)) ? y[i * S + k] : v[i * S + k];
          good += acc ? 1 : 0;
          sum += acc ? (int64_t)(val[0] - q.ar) + (int64_t)q.tl : 0;
        }
        __syncwarp();
        continue;
      }
      while (todo) {
        const int jj = __ffs(todo) - 1;
        todo &= todo - 1;
        const int m = __shfl_sync(FULL, ml, jj);
        T ar = __shfl_sync(FULL, arl, jj);
        const uint32_t hm = __shfl_sync(FULL, hml, jj);
        const T tl = __shfl_sync(FULL, tll, jj), sl = __shfl_sync(FULL, sll, jj);
        if constexpr (TT<T>::kRel) {
          if (per_req) {
            const int64_t a = __shfl_sync(FULL, al, jj);
            if (a - E > P.theta) {
              const int64_t gap = a - E;
              const T delta = gap >= 0xFFFFFFFFll ? (T)0xFFFFFFFFu : (T)gap;
#pragma unroll
              for (int r = 0; r < R; ++r) v[r] = v[r] > delta ? v[r] - delta : (T)0;
              E = a;
            }
            ar = (T)(a - E);
          }
        }
        T d[S];
#pragma unroll
        for (int k = 0; k < S; ++k) d[k] = w.d[m * kSTab + k];
        // predicted finish f of every compact group (departures y for S > 1;
        // a single stage departs at f - tail)
        T f[NG];
        T y[S > 1 ? R : 1];
#pragma unroll
        for (int i = 0; i < NG; ++i) {
          T x = ar;
#pragma unroll
          for (int k = 0; k < S; ++k) {
            x = tmax(x, v[i * S + k]) + d[k];
            if constexpr (S > 1) y[i * S + k] = x;
          }
          f[i] = ((hm >> i) & 1u) ? x + tl : TT<T>::maxv();
        }
        T fmin = f[0];
#pragma unroll
        for (int i = 1; i < NG; ++i) fmin = tmin(fmin, f[i]);
        if (fmin == TT<T>::maxv() || (T)(fmin - ar) > sl) continue;  // no host / misses the SLO
        // the lowest compact index among the minima = the lowest group id (C1)
        uint32_t eqm = 0;
#pragma unroll
        for (int i = 0; i < NG; ++i) eqm |= (f[i] == fmin ? 1u : 0u) << i;
        const int wi = __ffs(eqm) - 1;
#pragma unroll
        for (int i = 0; i < NG; ++i) {
          if constexpr (S == 1) {
            if (i == wi) v[i] = fmin - tl;
          } else {
#pragma unroll
            for (int k = 0; k < S; ++k)
              if (i == wi) v[i * S + k] = y[i * S + k];
          }
        }
        ++good;
        sum += (int64_t)(fmin - ar);
        if (pm_row && lane == 0) {
          int gw = 0;
          int64_t occ = 0;
#pragma unroll
          for (int i = 0; i < NG; ++i)
            if (i == wi) gw = cg[i];
#pragma unroll
          for (int k = 0; k < S; ++k) occ += (int64_t)d[k];
          atomicAdd(pm_row + m, 1);
          atomicAdd(reinterpret_cast<unsigned long long*>(busy_row + gw), (unsigned long long)occ);
        }
      }
    }
    // the chunk's exact correction, and equivalence with the speculative end
    if (lane == 0) {
      P.fix_good[j * cstride + (int64_t)item * 32 + cl] =
          (int32_t)(good - P.spec_good[j * cstride + (int64_t)item * 32 + cl]);
      P.fix_sum[j * cstride + (int64_t)item * 32 + cl] =
          sum - P.spec_sum[j * cstride + (int64_t)item * 32 + cl];
    }
    if (j + 1 < P.J) {
      const int64_t a_next = P.tr.arrival[i_end];
      const T* se = reinterpret_cast<const T*>(P.spec_end) + u * P.slots_max * 32;
      const int64_t Es = P.spec_epoch[u];
      bool eq = true;
#pragma unroll
      for (int i = 0; i < NG; ++i)
#pragma unroll
        for (int k = 0; k < S; ++k) {
          if (cg[i] < 0) continue;
          const int64_t t0 = (TT<T>::kRel ? E : 0) + (int64_t)v[i * S + k];
          const int64_t t1 = (TT<T>::kRel ? Es : 0) + (int64_t)se[(cg[i] * S + k) * 32 + cl];
          eq &= (t0 > a_next ? t0 : a_next) == (t1 > a_next ? t1 : a_next);
        }
      start_ok = eq;  // identical in every lane
      if (!start_ok) {  // publish column cl at the unit's canonical epoch
        const int64_t Ec = P.tr.arrival[i_end - 1];
        T* out = reinterpret_cast<T*>(P.fix_end) + u * P.slots_max * 32;
        // slots outside the component keep their start values
        for (int t = lane; t < it.slots; t += 32) {
          if ((gmask >> ((t / S) & 63)) & 1ull) continue;
          const T raw = s0[t * 32 + cl];
          if constexpr (TT<T>::kRel) {
            const int64_t r = (int64_t)raw + Ep - Ec;
            out[t * 32 + cl] = r > 0 ? (T)r : (T)0;
          } else {
            out[t * 32 + cl] = raw;
          }
        }
        if (lane == 0) {
#pragma unroll
          for (int i = 0; i < NG; ++i)
#pragma unroll
            for (int k = 0; k < S; ++k) {
              if (cg[i] < 0) continue;
              T x;
              if constexpr (TT<T>::kRel) {
                const int64_t r = (int64_t)v[i * S + k] - (Ec - E);
                x = r > 0 ? (T)r : (T)0;
              } else {
                x = v[i * S + k];
              }
              out[(cg[i] * S + k) * 32 + cl] = x;
            }
          P.fix_epoch[u] = Ec;
          atomicOr(end_src + u, 1u << cl);
        }
      }
    }
    __syncwarp();
  }
}

// Does candidate c's component fit the scalar walker (NG * S <= kScalarSlots)?
// Its per-request work grows with NG * S in every lane; larger components
// go to the cooperative walker, whose per-lane work does not.
constexpr int kScalarSlots = 16;

template <typename T, int S>
__device__ __forceinline__ bool scalar_dispatch_ng(const ChunkParams& P, const WarpMem<T>& w,
                                                   const ItemDesc& it, int item, int cl, int lane,
                                                   uint32_t* end_src, unsigned long long& walked,
                                                   unsigned long long& upd, int ng) {
  // NG = the next power of two >= ng, with NG * S <= kScalarSlots
  constexpr int K = kScalarSlots;
  if (ng <= 1) {
    scalar_candidate<T, S, 1>(P, w, it, item, cl, lane, end_src, walked, upd);
  } else if (ng <= 2 && 2 * S <= K) {
    scalar_candidate<T, S, (2 * S <= K ? 2 : 1)>(P, w, it, item, cl, lane, end_src, walked, upd);
  } else if (ng <= 4 && 4 * S <= K) {
    scalar_candidate<T, S, (4 * S <= K ? 4 : 1)>(P, w, it, item, cl, lane, end_src, walked, upd);
  } else if (ng <= 8 && 8 * S <= K) {
    scalar_candidate<T, S, (8 * S <= K ? 8 : 1)>(P, w, it, item, cl, lane, end_src, walked, upd);
  } else if (ng <= 16 && 16 * S <= K) {
    scalar_candidate<T, S, (16 * S <= K ? 16 : 1)>(P, w, it, item, cl, lane, end_src, walked, upd);
  } else {
    return false;
  }
  return true;
}

__device__ __forceinline__ bool scalar_fits(const ChunkParams& P, const ItemDesc& it, int64_t c) {
  const int ngroups = it.slots / it.S;
  const uint64_t all = ngroups >= 64 ? ~0ull : ((1ull << ngroups) - 1ull);
  const uint64_t gmask = (P.bt.cand_gmask ? P.bt.cand_gmask[c] : ~0ull) & all;
  int ng = __popcll(gmask), np2 = 1;
  while (np2 < ng) np2 <<= 1;
  return np2 * it.S <= kScalarSlots;
}

template <typename T>
__device__ __forceinline__ bool scalar_dispatch(const ChunkParams& P, const WarpMem<T>& w,
                                                const ItemDesc& it, int item, int cl, int lane,
                                                uint32_t* end_src, unsigned long long& walked,
                                                unsigned long long& upd) {
  const int64_t c = cand_of(P, it, item, cl);
  const int ngroups = it.slots / it.S;
  const uint64_t all = ngroups >= 64 ? ~0ull : ((1ull << ngroups) - 1ull);
  const uint64_t gmask = (P.bt.cand_gmask ? P.bt.cand_gmask[c] : ~0ull) & all;
  const int ng = __popcll(gmask);
  switch (it.S) {
    case 1: return scalar_dispatch_ng<T, 1>(P, w, it, item, cl, lane, end_src, walked, upd, ng);
    case 2: return scalar_dispatch_ng<T, 2>(P, w, it, item, cl, lane, end_src, walked, upd, ng);
    case 4: return scalar_dispatch_ng<T, 4>(P, w, it, item, cl, lane, end_src, walked, upd, ng);
    case 8: return scalar_dispatch_ng<T, 8>(P, w, it, item, cl, lane, end_src, walked, upd, ng);
    default: return scalar_dispatch_ng<T, 16>(P, w, it, item, cl, lane, end_src, walked, upd, ng);
  }
}

template <typename T, int S>
__device__ __forceinline__ void coop_dispatch_q(const ChunkParams& P, const WarpMem<T>& w,
                                                const ItemDesc& it, int item, int cl, int lane,
                                                uint32_t* end_src, unsigned long long& walked,
                                                unsigned long long& upd) {
  switch ((it.slots + 31) / 32) {
    case 1: coop_candidate<T, S, 1>(P, w, it, item, cl, lane, end_src, walked, upd); break;
    case 2: coop_candidate<T, S, 2>(P, w, it, item, cl, lane, end_src, walked, upd); break;
    case 3: coop_candidate<T, S, 3>(P, w, it, item, cl, lane, end_src, walked, upd); break;
    default: coop_candidate<T, S, 4>(P, w, it, item, cl, lane, end_src, walked, upd); break;
  }
}

template <typename T>
__device__ __forceinline__ void coop_dispatch(const ChunkParams& P, const WarpMem<T>& w,
                                              const ItemDesc& it, int item, int cl, int lane,
                                              uint32_t* end_src, unsigned long long& walked,
                                              unsigned long long& upd) {
  switch (it.S) {
    case 1: coop_dispatch_q<T, 1>(P, w, it, item, cl, lane, end_src, walked, upd); break;
    case 2: coop_dispatch_q<T, 2>(P, w, it, item, cl, lane, end_src, walked, upd); break;
    case 4: coop_dispatch_q<T, 4>(P, w, it, item, cl, lane, end_src, walked, upd); break;
    case 8: coop_dispatch_q<T, 8>(P, w, it, item, cl, lane, end_src, walked, upd); break;
    default: coop_dispatch_q<T, 16>(P, w, it, item, cl, lane, end_src, walked, upd); break;
  }
}

// ---------------------------------------------------------------------------
// Pass 3, components of <= 32 groups with S <= 2 stages: the group-lane
// walker.  One warp per candidate; lane i holds, in registers, the S stage free
// times of the i-th group (ascending id) of the candidate's component
// (cand_gmask).  The tile's component requests are compacted and staged in
// shared memory as in the scalar walker; per request every hosting lane runs
// its group's tandem recurrence, one warp min gives the earliest last
// departure, and the lowest lane among the minima -- the lowest group index,
// C1 -- commits.  The per-request work no longer grows with the number of
// groups (the scalar walker evaluates all of them in every lane).
template <typename T, int S>
__device__ __forceinline__ void glane_candidate(const ChunkParams& P, const WarpMem<T>& w,
                                                const ItemDesc& it, int item, int cl, int lane,
                                                uint32_t* end_src, unsigned long long& walked) {
  const int64_t c = cand_of(P, it, item, cl);
  const int my_m = P.bt.cand_model[c], my_g = P.bt.cand_group[c];
  const uint64_t kmask = P.bt.cand_kmask ? P.bt.cand_kmask[c] : ~0ull;
  const int ngroups = it.slots / S;
  const uint64_t all = ngroups >= 64 ? ~0ull : ((1ull << ngroups) - 1ull);
  const uint64_t gmask = (P.bt.cand_gmask ? P.bt.cand_gmask[c] : ~0ull) & all;
  // this lane's group: the lane-th set bit of gmask (-1: none)
  int g_l = -1;
  {
    uint64_t b = gmask;
    for (int i = 0; i < lane && b; ++i) b &= b - 1;
    g_l = b ? __ffsll((long long)b) - 1 : -1;
  }
  // compact hosting mask of every model over the component's groups (bit i =
  // lane i's group); the hosting-list region serves as scratch, as in the
  // scalar walker
  uint32_t* hmc = reinterpret_cast<uint32_t*>(w.hid);
  for (int m = lane; m < P.pr.M; m += 32) {
    const uint64_t hm = w.hmask[m] | (m == my_m ? (1ull << my_g) : 0ull);
    uint32_t x = 0;
    uint64_t b = gmask;
    for (int i = 0; b; ++i, b &= b - 1)
      if ((hm >> (__ffsll((long long)b) - 1)) & 1ull) x |= 1u << i;
    hmc[m] = x;
  }
  __syncwarp();
  const int64_t cstride = (int64_t)P.num_items * 32;
  bool start_ok = true;
  for (int j = 1; j < P.J; ++j) {
    const int64_t u = (int64_t)j * P.num_items + item;
    if (start_ok) {
      if ((P.fix_flag[u] >> cl) & 1u) {  // pass 2 exact; true end of j is its fix_end
        if (lane == 0) atomicOr(end_src + u, 1u << cl);
        start_ok = false;
      }
      continue;
    }
    ++walked;
    const int64_t i_begin = P.chunk_begin[j], i_end = P.chunk_begin[j + 1];
    int64_t E = TT<T>::kRel ? P.tr.arrival[i_begin] : 0;
    // true start: chunk j-1's true end (fix_end)
    const int64_t prev = u - P.num_items;
    const T* s0 = reinterpret_cast<const T*>(P.fix_end) + prev * P.slots_max * 32;
    const int64_t Ep = P.fix_epoch[prev];
    T v[S];
#pragma unroll
    for (int k = 0; k < S; ++k) {
      T x = 0;
      if (g_l >= 0) {
        const T raw = s0[(g_l * S + k) * 32 + cl];
        if constexpr (TT<T>::kRel) {
          const int64_t r = (int64_t)raw - (E - Ep);
          x = r > 0 ? (T)r : (T)0;
        } else {
          x = raw;
        }
      }
      v[k] = x;
    }
    int64_t good = 0, sum = 0;
    int64_t al_n = i_begin + lane < i_end ? P.tr.arrival[i_begin + lane] : 0;
    int ml_n = i_begin + lane < i_end ? (int)P.tr.model[i_begin + lane] : 0;
    for (int64_t i0 = i_begin; i0 < i_end; i0 += 32) {
      const bool valid = i0 + lane < i_end;
      const int64_t al = al_n;
      const int ml = ml_n;
      if (i0 + 32 + lane < i_end) {
        al_n = P.tr.arrival[i0 + 32 + lane];
        ml_n = (int)P.tr.model[i0 + 32 + lane];
      }
      unsigned todo = __ballot_sync(FULL, valid && ((kmask >> (ml & 63)) & 1ull));
      if (!todo) continue;
      bool per_req = false;
      if constexpr (TT<T>::kRel) {
        const int64_t a_last = __shfl_sync(FULL, al, 31 - __clz(todo));
        if (a_last - E > P.theta) {  // move the epoch to the tile's first request
          const int64_t a_first = __shfl_sync(FULL, al, __ffs(todo) - 1);
          const int64_t gap = a_first - E;
          const T delta = gap >= 0xFFFFFFFFll ? (T)0xFFFFFFFFu : (T)gap;
#pragma unroll
          for (int k = 0; k < S; ++k) v[k] = v[k] > delta ? v[k] - delta : (T)0;
          E = a_first;
          per_req = a_last - E > P.theta;
        }
      }
      // compacted component requests of the tile, staged as in the scalar walker
      TileReq<T>* tq = reinterpret_cast<TileReq<T>*>(w.tile);
      const int nreq = __popc(todo);
      if ((todo >> lane) & 1u) {
        const T arl = (T)(al - E);
        const T tll = w.tail[ml], sll = w.slo[ml];
        TileReq<T> q;
        q.ar = arl;
        q.hm = sll >= tll ? hmc[ml] : 0u;
        q.lim = 0;
        if (sll >= tll) {
          const T room = sll - tll;
          q.lim = room > (T)(TT<T>::maxv() - 1 - arl) ? (T)(TT<T>::maxv() - 1) : (T)(arl + room);
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) q.d[k] = k < S ? w.d[ml * kSTab + k] : (T)0;
        q.tl = tll;
        q.m = ml;
        tq[__popc(todo & ((1u << lane) - 1u))] = q;
      }
      __syncwarp();
      // one request: every hosting lane's tandem recurrence, the earliest last
      // departure by a warp min, the lowest lane among the minima by a second
      // one (C1; a ballot + find-first-set costs ~3x a warp min on the chain,
      // and a coarse-key variant measured slower in isolation, scripts/micro),
      // predicated commit (acceptance is warp-uniform; no host: mn = maxv > lim)
      auto request = [&](const TileReq<T>& q) {
        T d[S];
        tile_dv<T, S>(q, w.d, d);
        T x = q.ar;
        T y[S];
#pragma unroll
        for (int k = 0; k < S; ++k) {
          x = tmax(x, v[k]) + d[k];
          y[k] = x;
        }
        const T key = ((q.hm >> lane) & 1u) ? x : TT<T>::maxv();
        const T mn = warp_min<T>(key);
        const unsigned win = __reduce_min_sync(FULL, key == mn ? (unsigned)lane : 32u);
        const bool acc = mn <= q.lim;
        const bool take = acc && (unsigned)lane == win;
#pragma unroll
        for (int k = 0; k < S; ++k) v[k] = take ? y[k] : v[k];
        good += acc ? 1 : 0;
        sum += acc ? (int64_t)(mn - q.ar) + (int64_t)q.tl : 0;
      };
      if (!per_req) {
        for (int jj = 0; jj < nreq; ++jj) request(tq[jj]);
      } else if constexpr (TT<T>::kRel) {
        // sparse tiles (per-request epochs, rare): the staged relative
        // arrivals may have wrapped, so each request's absolute arrival comes
        // from its lane and its fields are recomputed at the moved epoch
        const int src = nth_set_bit(todo, lane);
        for (int jj = 0; jj < nreq; ++jj) {
          TileReq<T> q = tq[jj];
          const int64_t a_abs = __shfl_sync(FULL, al, __shfl_sync(FULL, src, jj));
          if (a_abs - E > P.theta) {
            const int64_t gap = a_abs - E;
            const T delta = gap >= 0xFFFFFFFFll ? (T)0xFFFFFFFFu : (T)gap;
#pragma unroll
            for (int k = 0; k < S; ++k) v[k] = v[k] > delta ? v[k] - delta : (T)0;
            E = a_abs;
          }
          const T ar = (T)(a_abs - E);
          const T tll = w.tail[q.m], sll = w.slo[q.m];
          q.lim = 0;
          if (sll >= tll) {
            const T room = sll - tll;
            q.lim = room > (T)(TT<T>::maxv() - 1 - ar) ? (T)(TT<T>::maxv() - 1) : (T)(ar + room);
          }
          q.ar = ar;
          request(q);
        }
      }
      __syncwarp();
    }
    // the chunk's exact correction, and equivalence with the speculative end
    if (lane == 0) {
      P.fix_good[j * cstride + (int64_t)item * 32 + cl] =
          (int32_t)(good - P.spec_good[j * cstride + (int64_t)item * 32 + cl]);
      P.fix_sum[j * cstride + (int64_t)item * 32 + cl] =
          sum - P.spec_sum[j * cstride + (int64_t)item * 32 + cl];
    }
    if (j + 1 < P.J) {
      const int64_t a_next = P.tr.arrival[i_end];
      const T* se = reinterpret_cast<const T*>(P.spec_end) + u * P.slots_max * 32;
      const int64_t Es = P.spec_epoch[u];
      bool eq = true;
      if (g_l >= 0) {
#pragma unroll
        for (int k = 0; k < S; ++k) {
          const int64_t t0 = (TT<T>::kRel ? E : 0) + (int64_t)v[k];
          const int64_t t1 = (TT<T>::kRel ? Es : 0) + (int64_t)se[(g_l * S + k) * 32 + cl];
          eq &= (t0 > a_next ? t0 : a_next) == (t1 > a_next ? t1 : a_next);
        }
      }
      start_ok = __all_sync(FULL, eq);
      if (!start_ok) {  // publish column cl at the unit's canonical epoch
        const int64_t Ec = P.tr.arrival[i_end - 1];
        T* out = reinterpret_cast<T*>(P.fix_end) + u * P.slots_max * 32;
        // slots outside the component keep their start values
        for (int t = lane; t < it.slots; t += 32) {
          if ((gmask >> ((t / S) & 63)) & 1ull) continue;
          const T raw = s0[t * 32 + cl];
          if constexpr (TT<T>::kRel) {
            const int64_t r = (int64_t)raw + Ep - Ec;
            out[t * 32 + cl] = r > 0 ? (T)r : (T)0;
          } else {
            out[t * 32 + cl] = raw;
          }
        }
        if (g_l >= 0) {
#pragma unroll
          for (int k = 0; k < S; ++k) {
            T x;
            if constexpr (TT<T>::kRel) {
              const int64_t r = (int64_t)v[k] - (Ec - E);
              x = r > 0 ? (T)r : (T)0;
            } else {
              x = v[k];
            }
            out[(g_l * S + k) * 32 + cl] = x;
          }
        }
        if (lane == 0) {
          P.fix_epoch[u] = Ec;
          atomicOr(end_src + u, 1u << cl);
        }
      }
    }
    __syncwarp();
  }
}

// Does candidate c walk with the group-lane walker?  S <= 2, <= 32 groups in
// its component, at least P.glane_walk of them, and no statistics rows.
__device__ __forceinline__ bool glane_fits(const ChunkParams& P, const ItemDesc& it, int64_t c) {
  if (P.glane_walk <= 0 || P.fix_pm || it.S > P.glane_smax) return false;
  const int ngroups = it.slots / it.S;
  const uint64_t all = ngroups >= 64 ? ~0ull : ((1ull << ngroups) - 1ull);
  const int ng = __popcll((P.bt.cand_gmask ? P.bt.cand_gmask[c] : ~0ull) & all);
  // S >= 4: the scalar walker's per-request work is NG x S >= 8 slots already at 2 groups
  return ng <= 32 && ng >= (it.S <= 2 ? P.glane_walk : 2);
}

// SCALAR = false: the cooperative walker for every candidate the scalar one
// does not take; SCALAR = true: the scalar walker (separate kernel: its
// register arrays would otherwise spill the cooperative walker).
template <typename T, bool SCALAR>
__global__ void __launch_bounds__(kWarps * 32) coop_walk_kernel(ChunkParams P, uint32_t* end_src) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const size_t wb = warp_bytes(P.slots_max, P.pr.M, P.hid_cap, sizeof(T), false);
  WarpMem<T> w = carve<T>(smem + warp * wb, P, false);
  int cur_base = -1;
  unsigned long long walked = 0, upd = 0;
  for (;;) {
    const int u = next_unit(P, lane);  // candidate slot = item * 32 + lane of the item
    if (u >= P.num_items * 32) break;
    const int item = u >> 5, cl = u & 31;
    const ItemDesc it = P.items[item];
    if (it.S == 0 || cl >= it.count || !P.bt.cand_ok[cand_of(P, it, item, cl)]) continue;
    // the scalar kernel takes the scalar walker's and the group-lane walker's
    // candidates, the cooperative kernel the rest
    const bool glane = glane_fits(P, it, cand_of(P, it, item, cl));
    const bool fits = P.scalar_walk && (glane || scalar_fits(P, it, cand_of(P, it, item, cl)));
    if (fits != SCALAR) continue;  // the other walker's candidate
    // any chunk of this candidate flagged by pass 2?  (else nothing to walk)
    bool any = false;
    for (int j = 1 + lane; j < P.J; j += 32)
      any |= (P.fix_flag[(int64_t)j * P.num_items + item] >> cl) & 1u;
    if (!__any_sync(FULL, any)) continue;
    if (it.base != cur_base) {
      load_base<T>(P, it, w, lane);
      cur_base = it.base;
    }
    const unsigned long long w0 = walked;
#ifdef ASIM_WALK_DIAGNOSTICS
    const unsigned long long u0 = upd;
    const long long t0 = clock64();
#endif
    if constexpr (SCALAR) {
      if (glane) {
        switch (it.S) {
          case 1: glane_candidate<T, 1>(P, w, it, item, cl, lane, end_src, walked); break;
          case 2: glane_candidate<T, 2>(P, w, it, item, cl, lane, end_src, walked); break;
          case 4: glane_candidate<T, 4>(P, w, it, item, cl, lane, end_src, walked); break;
          case 8: glane_candidate<T, 8>(P, w, it, item, cl, lane, end_src, walked); break;
          default: glane_candidate<T, 16>(P, w, it, item, cl, lane, end_src, walked); break;
        }
      } else {
        scalar_dispatch<T>(P, w, it, item, cl, lane, end_src, walked, upd);
      }
    } else {
      coop_dispatch<T>(P, w, it, item, cl, lane, end_src, walked, upd);
    }
    if (P.walked && lane == 0 && walked > w0) {  // statistics: walking candidates, longest walk
      atomicAdd(P.walked + 1, 1ull);
      atomicMax(P.walked + 2, walked - w0);
#ifdef ASIM_WALK_DIAGNOSTICS
      const long long cyc = clock64() - t0;
      if (P.walk_log > 0 && cyc > P.walk_log) {
        const int64_t c = cand_of(P, it, item, cl);
        printf("walk kind=%d S=%d slots=%d ng=%d models=%d chunks=%llu cycles=%lld upd=%llu\n",
               glane ? 2 : (int)SCALAR, it.S, it.slots,
               __popcll(P.bt.cand_gmask ? P.bt.cand_gmask[c] : ~0ull),
               __popcll(P.bt.cand_kmask ? P.bt.cand_kmask[c] : ~0ull), walked - w0, cyc, upd - u0);
      }
#endif
    }
  }
  if (lane == 0) {
    if (P.walked && walked) atomicAdd(P.walked, walked);
    if (P.stage_updates && upd) atomicAdd(P.stage_updates, upd);
  }
}

// Fast heuristic statistics (search.cpp run_fast): one warp per
// candidate of a uniform-config item simulates the whole trace from idle with
// the warp-cooperative recurrence and writes good, sum, per-model good and
// per-group busy.  Items hold one candidate each (cl = 0).
template <typename T, int S, int Q>
__device__ __forceinline__ void fast_candidate(const ChunkParams& P, const WarpMem<T>& w,
                                               const ItemDesc& it, int lane,
                                               const DevOut& out, unsigned long long& upd) {
  const int64_t c = it.first;
  const int slots = it.slots;
  uint64_t lastbit[Q];
  T v[Q];
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    const int t = lane + 32 * q;
    lastbit[q] = (t < slots && t % S == S - 1) ? (1ull << ((t / S) & 63)) : 0ull;
    v[q] = 0;  // idle
  }
  const int my_m = P.bt.cand_model[c], my_g = P.bt.cand_group[c];
  const uint64_t my_bit = my_m >= 0 ? (1ull << my_g) : 0ull;
  int64_t E = (TT<T>::kRel && P.tr.n > 0) ? P.tr.arrival[0] : 0;
  int64_t good = 0, sum = 0;
  const uint64_t kmask = P.bt.cand_kmask ? P.bt.cand_kmask[c] : ~0ull;  // component restriction
  const int64_t o = c - out.out_offset;
  // per-model good counts are int32 rows here; out.good_per_model is int64:
  // accumulate into the int32 scratch P.spec_pm row, copied below
  int32_t* pm_row = P.spec_pm + o * P.pr.M;
  coop_range<T, S, Q, true>(P, w, 0, P.tr.n, v, E, kmask, my_m, my_bit, lastbit, lane, good, sum,
                            upd, pm_row, out.busy + o * P.bt.G);
  __syncwarp();
  __threadfence_block();
  if (lane == 0) {
    out.good[o] = good;
    if (out.sum_latency) out.sum_latency[o] = sum;
  }
  for (int m = lane; m < P.pr.M; m += 32) out.good_per_model[o * P.pr.M + m] = pm_row[m];
}

template <typename T, int S>
__device__ __forceinline__ void fast_dispatch_q(const ChunkParams& P, const WarpMem<T>& w,
                                                const ItemDesc& it, int lane,
                                                const DevOut& out, unsigned long long& upd) {
  switch ((it.slots + 31) / 32) {
    case 1: fast_candidate<T, S, 1>(P, w, it, lane, out, upd); break;
    case 2: fast_candidate<T, S, 2>(P, w, it, lane, out, upd); break;
    case 3: fast_candidate<T, S, 3>(P, w, it, lane, out, upd); break;
    default: fast_candidate<T, S, 4>(P, w, it, lane, out, upd); break;
  }
}

template <typename T>
__global__ void __launch_bounds__(kWarps * 32) fast_stats_kernel(ChunkParams P, DevOut out) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const size_t wb = warp_bytes(P.slots_max, P.pr.M, P.hid_cap, sizeof(T), false);
  WarpMem<T> w = carve<T>(smem + warp * wb, P, false);
  const int item = blockIdx.x * kWarps + warp;
  if (item >= P.num_items) return;
  const ItemDesc it = P.items[item];
  load_base<T>(P, it, w, lane);
  unsigned long long upd = 0;
  switch (it.S) {
    case 1: fast_dispatch_q<T, 1>(P, w, it, lane, out, upd); break;
    case 2: fast_dispatch_q<T, 2>(P, w, it, lane, out, upd); break;
    case 4: fast_dispatch_q<T, 4>(P, w, it, lane, out, upd); break;
    case 8: fast_dispatch_q<T, 8>(P, w, it, lane, out, upd); break;
    default: fast_dispatch_q<T, 16>(P, w, it, lane, out, upd); break;
  }
  if (lane == 0 && P.stage_updates && upd) atomicAdd(P.stage_updates, upd);
}

// good[c] = sum_j spec_good[j][c] + sum_{j>=1} fix_good[j][c] (same for sums)
__global__ void chunk_reduce_kernel(ChunkParams P, DevOut out) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t == 0 && P.walked) {  // statistics: fold this run's longest walk (stream-ordered after it)
    P.walked[3] += P.walked[2];
    P.walked[2] = 0;
  }
  if (t >= (int64_t)P.num_items * 32) return;
  const int item = (int)(t >> 5), lane = (int)(t & 31);
  const ItemDesc it = P.items[item];
  if (lane >= it.count) return;
  const int64_t c = cand_of(P, it, item, lane);
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

// True state at every chunk boundary of chosen lanes: for each PublishItem
// (item, lane, row), out[(row * J + j) * state_stride + k] (absolute int64).
// j = 0 is idle.  Slots outside the lane's component mask (cand_gmask) were
// never simulated by that lane: they evolve exactly like the speculation
// source (the base placement), whose state at boundary j is copied instead.
template <typename T>
__global__ void publish_kernel(ChunkParams P, const uint32_t* __restrict__ end_src,
                               const PublishItem* __restrict__ pub, int32_t npub,
                               int64_t* __restrict__ out) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t total = (int64_t)npub * P.J * P.state_stride;
  if (t >= total) return;
  const int k = (int)(t % P.state_stride);
  const int j = (int)((t / P.state_stride) % P.J);
  const PublishItem pi = pub[t / ((int64_t)P.state_stride * P.J)];
  const ItemDesc it = P.items[pi.item];
  int64_t v = 0;  // j == 0: idle; slots beyond the item's: unused
  if (j > 0 && k < it.slots) {
    const int64_t c = cand_of(P, it, pi.item, pi.lane);
    bool own = true;
    if (P.bt.cand_gmask) {  // group of slot k under the base's group table
      int g = 0, off = 0;
      for (; g < P.bt.G; ++g) {
        const int cfg = P.bt.base_cfg[(int64_t)it.base * P.bt.G + g];
        if (cfg < 0) continue;
        const int s = P.pr.cfg_stages[cfg];
        if (k < off + s) break;
        off += s;
      }
      own = (P.bt.cand_gmask[c] >> g) & 1ull;
    }
    if (own || P.spec_state == nullptr) {
      const int64_t u = (int64_t)(j - 1) * P.num_items + pi.item;  // end of chunk j-1
      const bool fix = (end_src[u] >> pi.lane) & 1u;
      const T* st = reinterpret_cast<const T*>(fix ? P.fix_end : P.spec_end) + u * P.slots_max * 32;
      const T x = st[k * 32 + pi.lane];
      v = (TT<T>::kRel ? (fix ? P.fix_epoch : P.spec_epoch)[u] : 0) + (int64_t)x;
    } else {
      v = P.spec_state[((int64_t)P.spec_row[it.base] * P.J + j) * P.state_stride + k];
    }
  }
  if (j > 0) {  // canonical form: a free time below the boundary's arrival is that arrival
    const int64_t a0 = P.tr.arrival[P.chunk_begin[j]];
    v = v > a0 ? v : a0;
  }
  out[((int64_t)pi.row * P.J + j) * P.state_stride + k] = v;
}

__global__ void mix_states_kernel(int64_t C0, int64_t C1, int32_t J, int32_t stride,
                                  const int64_t* __restrict__ bcur,
                                  const int64_t* __restrict__ bprev,
                                  const int64_t* __restrict__ cprev,
                                  const MixRow* __restrict__ rows, int64_t* __restrict__ out) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t per = (int64_t)J * stride;
  if (t >= (C1 - C0) * per) return;
  const int64_t c = C0 + t / per, jk = t % per;
  const MixRow r = rows[c];
  const int64_t b = bcur[(int64_t)r.run * per + jk];
  int64_t v = b;
  if (r.prev >= 0) {
    const int64_t cp = cprev[(int64_t)r.prev * per + jk];
    if (cp != bprev[(int64_t)r.run * per + jk]) v = cp;  // the candidate's own difference
  }
  out[c * per + jk] = v;
}

template <typename K>
cudaError_t grid_for(K kernel, size_t smem, int64_t units, int sms, int64_t* blocks) {
  if (smem > 227 * 1024) return cudaErrorInvalidValue;
  int per_sm = 0;
  cudaError_t e = blocks_per_sm(reinterpret_cast<const void*>(kernel), kWarps * 32, smem, &per_sm);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  int64_t b = (int64_t)per_sm * sms;  // persistent: warps pull units from a counter
  const int64_t need = (units + kWarps - 1) / kWarps;
  if (b > need) b = need;
  *blocks = b < 1 ? 1 : b;
  return cudaSuccess;
}

template <typename T, int MODE>
cudaError_t launch_pass_t(const ChunkParams& P, cudaStream_t st, int sms) {
  constexpr int MINB = MODE == DUAL ? 3 : 5;
  const size_t smem = kWarps * warp_bytes(P.slots_max, P.pr.M, P.hid_cap, sizeof(T), MODE == DUAL, false);
  int64_t blocks = 1;
  cudaError_t e = grid_for(chunk_kernel<T, MODE, MINB>, smem, P.num_units, sms, &blocks);
  if (e != cudaSuccess) return e;
  // a split step's runs share the GPU: one unit per warp and blocks that
  // retire, so the block scheduler interleaves the two runs by stream priority
  // (persistent blocks would hold their SMs until their run's last unit)
  if (P.transient) blocks = std::max<int64_t>(1, std::min<int64_t>((P.num_units + kWarps - 1) / kWarps, 0x7FFFFFFF));
  chunk_kernel<T, MODE, MINB><<<(unsigned)blocks, kWarps * 32, smem, st>>>(P);
  return cudaGetLastError();
}

// The walkers take disjoint candidates (coop: uniform configs not taken by
// the scalar walker; scalar: small uniform components; item walker: mixed
// configs), so they run concurrently: the walk's critical path is the
// longest single walk, not the sum of the three kernels' tails.
template <typename T>
cudaError_t launch_walk_t(const ChunkParams& P, uint32_t* end_src, const WalkStreams& ws, int sms,
                          bool any_dynamic) {
  const size_t smem = kWarps * warp_bytes(P.slots_max, P.pr.M, P.hid_cap, sizeof(T), false);
  int64_t blocks = 1;
  cudaError_t e = cudaMemsetAsync(P.counter, 0, 3 * sizeof(uint32_t), ws.main);
  if (e != cudaSuccess) return e;
  const bool fork = P.scalar_walk || any_dynamic;
  if (fork && (e = cudaEventRecord(ws.fork, ws.main)) != cudaSuccess) return e;
  e = grid_for(coop_walk_kernel<T, false>, smem, (int64_t)P.num_items * 32, sms, &blocks);
  if (e != cudaSuccess) return e;
  coop_walk_kernel<T, false><<<(unsigned)blocks, kWarps * 32, smem, ws.main>>>(P, end_src);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  if (P.scalar_walk) {
    ChunkParams Q = P;
    Q.counter = P.counter + 1;
    if ((e = cudaStreamWaitEvent(ws.side[0], ws.fork, 0)) != cudaSuccess) return e;
    e = grid_for(coop_walk_kernel<T, true>, smem, (int64_t)P.num_items * 32, sms, &blocks);
    if (e != cudaSuccess) return e;
    coop_walk_kernel<T, true><<<(unsigned)blocks, kWarps * 32, smem, ws.side[0]>>>(Q, end_src);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    if ((e = cudaEventRecord(ws.join[0], ws.side[0])) != cudaSuccess) return e;
    if ((e = cudaStreamWaitEvent(ws.main, ws.join[0], 0)) != cudaSuccess) return e;
  }
  if (any_dynamic) {
    ChunkParams Q = P;
    Q.counter = P.counter + 2;
    if ((e = cudaStreamWaitEvent(ws.side[1], ws.fork, 0)) != cudaSuccess) return e;
    e = grid_for(walk_kernel<T>, smem, P.num_items, sms, &blocks);
    if (e != cudaSuccess) return e;
    walk_kernel<T><<<(unsigned)blocks, kWarps * 32, smem, ws.side[1]>>>(Q, end_src);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    if ((e = cudaEventRecord(ws.join[1], ws.side[1])) != cudaSuccess) return e;
    if ((e = cudaStreamWaitEvent(ws.main, ws.join[1], 0)) != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace

cudaError_t launch_chunk_pass(const ChunkParams& P, bool dual, bool u32, cudaStream_t st, int sms,
                              int64_t* launches) {
  if (P.num_units <= 0) return cudaSuccess;
  cudaError_t e = cudaMemsetAsync(P.counter, 0, sizeof(uint32_t), st);
  if (e != cudaSuccess) return e;
  if (u32)
    e = dual ? launch_pass_t<uint32_t, DUAL>(P, st, sms) : launch_pass_t<uint32_t, SPEC>(P, st, sms);
  else
    e = dual ? launch_pass_t<int64_t, DUAL>(P, st, sms) : launch_pass_t<int64_t, SPEC>(P, st, sms);
  if (launches) ++*launches;
  return e;
}

cudaError_t launch_chunk_walk(const ChunkParams& P, uint32_t* end_src, bool u32, bool any_dynamic,
                              const WalkStreams& ws, int sms, int64_t* launches) {
  cudaError_t e = cudaMemsetAsync(end_src, 0, (size_t)P.J * P.num_items * 4, ws.main);
  if (e != cudaSuccess) return e;
  e = u32 ? launch_walk_t<uint32_t>(P, end_src, ws, sms, any_dynamic)
          : launch_walk_t<int64_t>(P, end_src, ws, sms, any_dynamic);
  if (launches) *launches += 1 + (any_dynamic ? 1 : 0) + (P.scalar_walk ? 1 : 0);
  return e;
}

cudaError_t launch_publish_states(const ChunkParams& P, const uint32_t* end_src, bool u32,
                                  const PublishItem* pub, int32_t npub, int64_t* out,
                                  cudaStream_t st, int64_t* launches) {
  const int64_t total = (int64_t)npub * P.J * P.state_stride;
  if (total == 0) return cudaSuccess;
  const unsigned blocks = (unsigned)((total + 255) / 256);
  if (u32)
    publish_kernel<uint32_t><<<blocks, 256, 0, st>>>(P, end_src, pub, npub, out);
  else
    publish_kernel<int64_t><<<blocks, 256, 0, st>>>(P, end_src, pub, npub, out);
  if (launches) ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_mix_states(int64_t C0, int64_t C1, int32_t J, int32_t stride,
                              const int64_t* bcur, const int64_t* bprev, const int64_t* cprev,
                              const MixRow* rows, int64_t* out, cudaStream_t st,
                              int64_t* launches) {
  const int64_t n = (C1 - C0) * J * stride;
  if (n <= 0) return cudaSuccess;
  mix_states_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(C0, C1, J, stride, bcur, bprev,
                                                                 cprev, rows, out);
  if (launches) ++*launches;
  return cudaGetLastError();
}

size_t fast_stats_smem(int slots_max, int M, int hid_cap, bool u32) {
  return kWarps * warp_bytes(slots_max, M, hid_cap, u32 ? 4 : 8, false);
}

// out.good_per_model[c][m] = sum_j spec_pm[j][c][m] + sum_{j>=1} fix_pm[j][c][m];
// out.busy likewise.  One thread per (c, m) and per (c, g).
__global__ void chunk_stats_reduce_kernel(ChunkParams P, DevOut out) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t M = P.pr.M, G = P.bt.G, C = P.stat_C;
  if (t < C * M) {
    const int64_t c = t / M, m = t % M;
    int64_t v = 0;
    for (int j = 0; j < P.J; ++j) {
      v += P.spec_pm[((int64_t)j * C + c) * M + m];
      if (j > 0) v += P.fix_pm[((int64_t)j * C + c) * M + m];
    }
    out.good_per_model[(c - out.out_offset) * M + m] = v;
  } else if (t < C * M + C * G) {
    const int64_t u = t - C * M, c = u / G, g = u % G;
    int64_t v = 0;
    for (int j = 0; j < P.J; ++j) {
      v += P.spec_busy[((int64_t)j * C + c) * G + g];
      if (j > 0) v += P.fix_busy[((int64_t)j * C + c) * G + g];
    }
    out.busy[(c - out.out_offset) * G + g] = v;
  }
}

cudaError_t launch_chunk_stats_reduce(const ChunkParams& P, const DevOut& out, cudaStream_t st,
                                      int64_t* launches) {
  const int64_t n = P.stat_C * (P.pr.M + P.bt.G);
  if (n == 0) return cudaSuccess;
  chunk_stats_reduce_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(P, out);
  if (launches) ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_fast_stats(const ChunkParams& P, const DevOut& out, bool u32, cudaStream_t st,
                              int64_t* launches) {
  if (P.num_items <= 0) return cudaSuccess;
  const size_t smem = fast_stats_smem(P.slots_max, P.pr.M, P.hid_cap, u32);
  if (smem > 227 * 1024) return cudaErrorInvalidValue;
  const unsigned blocks = (unsigned)((P.num_items + kWarps - 1) / kWarps);
  cudaError_t e;
  if (u32) {
    e = allow_max_smem(reinterpret_cast<const void*>(fast_stats_kernel<uint32_t>));
    if (e == cudaSuccess) fast_stats_kernel<uint32_t><<<blocks, kWarps * 32, smem, st>>>(P, out);
  } else {
    e = allow_max_smem(reinterpret_cast<const void*>(fast_stats_kernel<int64_t>));
    if (e == cudaSuccess) fast_stats_kernel<int64_t><<<blocks, kWarps * 32, smem, st>>>(P, out);
  }
  if (e != cudaSuccess) return e;
  if (launches) ++*launches;
  return cudaGetLastError();
}

// out[c] = 1 for every candidate of the run whose trajectories pass 2 left
// unmet in some chunk (it walks), else 0 (batch-indexed; other entries kept).
__global__ void walk_flags_kernel(ChunkParams P, uint8_t* __restrict__ out) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)P.num_items * 32) return;
  const int item = (int)(t >> 5), lane = (int)(t & 31);
  const ItemDesc it = P.items[item];
  if (lane >= it.count) return;
  uint32_t f = 0;
  for (int j = 1; j + 1 < P.J && !f; ++j) f = (P.fix_flag[(int64_t)j * P.num_items + item] >> lane) & 1u;
  out[cand_of(P, it, item, lane)] = (uint8_t)f;
}

cudaError_t launch_walk_flags(const ChunkParams& P, uint8_t* out, cudaStream_t st,
                              int64_t* launches) {
  const int64_t n = (int64_t)P.num_items * 32;
  if (n == 0 || P.J < 3) return cudaSuccess;  // no chunk after a flagged one
  walk_flags_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(P, out);
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
