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
  // stage latencies by config, padded to 16 per model (0 beyond the config's
  // stages): [P][M][16]; uint32 copy (values clipped, used only when times
  // are uint32, i.e. every latency fits) and int64 copy
  const uint32_t* dtab32;
  const int64_t* dtab64;
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
  // Component restriction (chunked path, nullable = simulate everything):
  // lane c only simulates requests of the models in cand_kmask[c] and only
  // compares the stage slots of the groups in cand_gmask[c] -- the candidate's
  // own connected component; every other component evolves exactly like the
  // base placement's (search.cpp).  Requires M <= 64.
  const uint64_t* cand_kmask;   // [C]
  const uint64_t* cand_gmask;   // [C]
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
  int64_t* busy;            // nullable [C][G]: sum of stage occupancies of accepted requests
};

// Launchers (sim.cu).  All asynchronous on `stream`; return cudaError_t.
cudaError_t launch_simulate(const DevProblem& pr, const DevTrace& tr, const DevBatch& b,
                            const WarpItem* items, int32_t num_items, int32_t slots,
                            const DevOut& out, cudaStream_t stream, int64_t* launches);
cudaError_t launch_argmax(const int64_t* good, int64_t C, int64_t* argmax_out,
                          cudaStream_t stream, int64_t* launches);

// Dynamic batching variant (batch.cu, §5.4): batch-size increments and
// the trace's per-model request lists (CSR by model, ascending trace index).
struct DevBatching {
  int64_t max_batch;       // >= 1
  const int64_t* inc;      // [M][P][S] stage increment per extra batch member
  const int32_t* moff;     // [M+1]
  const int32_t* midx;     // [n] trace indices grouped by model
  const int32_t* order;    // [C] candidate simulated by warp w (costliest first), nullable
  const uint64_t* mcum;    // [n + M] per model, running sums of its arrivals mod 2^64
                           // (entry moff[m] + m + i = sum of its first i arrivals)
};
size_t batching_smem_per_warp(int32_t slots, int32_t G, int32_t M);
cudaError_t launch_batching(const DevProblem& pr, const DevTrace& tr, const DevBatch& b,
                            const DevBatching& bp, int32_t slots, const DevOut& out,
                            cudaStream_t stream, int64_t* launches);

}  // namespace asim

namespace asim {

// ---- chunked throughput path (chunk.cu) ----------------------------------
// Work item: up to 32 consecutive candidates sharing one base placement.
struct ItemDesc {
  int32_t base;    // base index in the batch
  int32_t first;   // first candidate (batch index; ChunkParams.item_cand overrides)
  int32_t count;   // 1..32
  int32_t S;       // compile-time stage class: 1,2,4,8,16 (uniform config) or 0 (dynamic)
  int32_t cfg;     // the base's uniform config id, -1 if groups differ
  int32_t stages;  // stages of `cfg` (uniform case)
  int32_t slots;   // sum of stages over the base's groups
  int32_t pad;
};


struct ChunkParams {
  DevProblem pr;
  DevTrace tr;
  DevBatch bt;
  const ItemDesc* items;
  // nullable: [num_items][32] batch index of the candidate in each lane (-1:
  // none) when items are not runs of consecutive candidates (the host groups
  // candidates by hosting component so a warp's lanes replay the same requests)
  const int32_t* item_cand;
  int32_t num_items;
  int32_t J;                   // chunks
  const int64_t* chunk_begin;  // [J+1] request index boundaries
  int64_t theta;               // uint32 epoch threshold (see chunk.cu)
  int32_t slots_max;
  int32_t hid_cap;             // bytes of each warp's hosting-list region (host: hid_cap_for)
  int32_t num_units;
  // passes 1-2 visit items class by class (one stage count S per class) so
  // the warps in flight run the same code: class c = items
  // item_perm[class_off[c] .. class_off[c] + class_items[c]) (nullable: identity)
  const int32_t* item_perm;
  int32_t nclass;
  int32_t class_off[8], class_items[8];
  uint32_t* counter;           // dynamic work counter
  int32_t* spec_good;          // [J][items*32]
  int64_t* spec_sum;
  void* spec_end;              // [J][items][slots_max][32] of T
  int64_t* spec_epoch;         // [J][items]
  int32_t* fix_good;
  int64_t* fix_sum;
  void* fix_end;
  int64_t* fix_epoch;
  uint32_t* fix_flag;          // [J][items] lanes whose trajectories never met in the chunk
  unsigned long long* stage_updates;  // nullable statistics counter
  // Speculation source (nullable = idle): absolute int64 free times of the
  // base placement's TRUE trajectory at every chunk boundary,
  // spec_state[(spec_row[b] * J + j) * slots_max + k].  Any start state is
  // exact (the fix-up corrects it); the base's own trajectory is the one the
  // candidates (base + one replica) stay closest to.
  const int64_t* spec_state;
  const int32_t* spec_row;     // [B] row of base b in spec_state
  int32_t state_stride;        // slots per boundary row of spec_state / published states
  unsigned long long* walked;  // nullable statistics [4]: chunks walked, walking candidates, longest walk of this run, sum of longest walks
  // Per-candidate speculation rows (nullable): spec_cand[(c * J + j) * state_stride + k],
  // c = batch index; when set they replace spec_state for the candidate's own
  // trajectory (spec_state still supplies out-of-component slots when publishing).
  const int64_t* spec_cand;
  // Fast-heuristic statistics (nullable = off): per (chunk, batch candidate)
  // rows of per-model good counts [J][C][M] and per-group busy [J][C][G];
  // spec_* hold pass 1's counts, fix_* the exact corrections (pass 2 / walk),
  // summed like spec_good / fix_good.  Zeroed before pass 1.
  int32_t* spec_pm;
  int32_t* fix_pm;
  int64_t* spec_busy;
  int64_t* fix_busy;
  int64_t stat_C;
  int32_t scalar_walk;  // 1 = small components walk with the register-state scalar walker
  int32_t glane_walk;   // > 0: components of S <= 2 and glane_walk..32 groups take the group-lane walker
  int32_t glane_smax;   // largest stage count the group-lane walker takes (S >= 4: from 2 groups)
  int32_t transient;    // 1 = passes 1-2 launch one unit per warp, blocks retire (split steps)
  int64_t walk_log;     // diagnostics (ASIM_WALK_LOG=cycles): printf every walk longer than this
};

// Per-candidate speculation rows for the search (see search.cpp):
// out[c][j][k] = (cprev[kp][j][k] != bprev[r][j][k]) ? cprev[kp][j][k] : bcur[r][j][k]
// with (r, kp) = rows[c] (kp < 0: bcur).  Canonical (boundary-clamped) states.
struct MixRow {
  int32_t run, prev;
};
cudaError_t launch_mix_states(int64_t C0, int64_t C1, int32_t J, int32_t stride,
                              const int64_t* bcur, const int64_t* bprev, const int64_t* cprev,
                              const MixRow* rows, int64_t* out, cudaStream_t st,
                              int64_t* launches);

// Publish the true state at every chunk boundary of chosen lanes (item, lane)
// into out[(row * J + j) * state_stride + k] (absolute int64; j = 0 idle).
// Bit `lane` of end_src[j * items + i] = 0 if that lane's true end of chunk j
// is in spec_end, 1 if in fix_end.  Slots outside the lane's component mask
// come from spec_state.
struct PublishItem {
  int32_t item, lane, row;
};
cudaError_t launch_publish_states(const ChunkParams& P, const uint32_t* end_src, bool u32,
                                  const PublishItem* pub, int32_t npub, int64_t* out,
                                  cudaStream_t st, int64_t* launches);

cudaError_t launch_chunk_pass(const ChunkParams& P, bool dual, bool u32, cudaStream_t st, int sms,
                              int64_t* launches);
cudaError_t launch_chunk_reduce(const ChunkParams& P, const DevOut& out, cudaStream_t st,
                                int64_t* launches);
// After pass 2: out[c] = 1 if candidate c (batch index) has a chunk whose
// trajectories never met, i.e. it walks (the search's walk prediction).
cudaError_t launch_walk_flags(const ChunkParams& P, uint8_t* out, cudaStream_t st,
                              int64_t* launches);
// Fast heuristic statistics: one warp per item (one candidate each, uniform
// config, S class != 0) over the whole trace; writes good, sum, per-model good
// and per-group busy into `out`.  fast_stats_smem: dynamic shared memory.
size_t fast_stats_smem(int slots_max, int M, int hid_cap, bool u32);
// out.good_per_model[c][m] / out.busy[c][g] = sum over chunks of the spec_*
// and fix_* statistics rows (after launch_chunk_reduce).
cudaError_t launch_chunk_stats_reduce(const ChunkParams& P, const DevOut& out, cudaStream_t st,
                                      int64_t* launches);
cudaError_t launch_fast_stats(const ChunkParams& P, const DevOut& out, bool u32, cudaStream_t st,
                              int64_t* launches);
// Pass 3: re-simulate every chunk whose start state was wrong (per lane) and
// record in bit `lane` of end_src[j * items + item] whether that lane's true
// end of chunk j is in spec_end (0) or fix_end (1).
// The three walkers run concurrently: fork from `main` onto the side
// streams, join back before returning (stream-ordered for the caller).
struct WalkStreams {
  cudaStream_t main;
  cudaStream_t side[2];
  cudaEvent_t fork, join[2];
};
cudaError_t launch_chunk_walk(const ChunkParams& P, uint32_t* end_src, bool u32, bool any_dynamic,
                              const WalkStreams& ws, int sms, int64_t* launches);


}  // namespace asim
