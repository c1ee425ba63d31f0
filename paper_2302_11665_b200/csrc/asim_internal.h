// asim_internal.h -- types shared by the host runtime (ctx.cpp, search.cpp)
// and the sm_100a kernels (sim.cu).  Not part of the public ABI.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace asim {

// Problem tables resident in HBM (copied once by asim_set_problem).
struct DevProblem {
  int32_t M, P, S;
  const int64_t* stage;     // [M][P][S]
  const int64_t* tail;      // [M][P]
  const int64_t* slo;       // [M]
  const int32_t* cfg_stages;  // [P]
};

// Trace resident in HBM (asim_set_trace).  Padded to a multiple of 32 with
// arrival = last arrival and model = 0xFFFF (never hosted).
struct DevTrace {
  int64_t n;
  const int64_t* arrival;  // [n_pad]
  const uint16_t* model;   // [n_pad]
};

// A batch of candidates in base + delta form.  Lane l of warp item w
// simulates candidate first + l.  Per-lane base: full candidates use one base
// per candidate; greedy steps share one base per run.
struct DevBatch {
  int32_t G;                    // groups per base (max_groups)
  const int32_t* base_cfg;      // [B][G]
  const uint64_t* base_mask;    // [B][M]
  const int32_t* cand_base;     // [C]
  const int32_t* cand_model;    // [C]  -1 = none
  const int32_t* cand_group;    // [C]
  const uint8_t* cand_ok;       // [C]  0 = infeasible (good = -1)
  int64_t C;
};

struct WarpItem {
  int32_t first;   // first candidate index (batch-local)
  int32_t count;   // 1..32
};

struct DevOut {
  int64_t* good;            // [C] indexed by candidate - out_offset
  int64_t* sum_latency;     // nullable
  int64_t* good_per_model;  // nullable [C][M]
  int64_t out_offset;
  unsigned long long* stage_updates;  // nullable device counter (statistics)
};

// Launchers (sim.cu).  All asynchronous on `stream`; return cudaError_t.
cudaError_t launch_simulate(const DevProblem& pr, const DevTrace& tr, const DevBatch& b,
                            const WarpItem* items, int32_t num_items, int32_t slots,
                            const DevOut& out, cudaStream_t stream, int64_t* launches);
cudaError_t launch_argmax(const int64_t* good, int64_t C, int64_t* argmax_out,
                          cudaStream_t stream, int64_t* launches);

}  // namespace asim
