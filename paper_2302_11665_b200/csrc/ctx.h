// ctx.h -- host-side context shared by ctx.cpp and search.cpp (private).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/asim.h"
#include "asim_internal.h"

constexpr int kSearchPool = 13;  // device scratch buffers an asim_search borrows
constexpr int kChunkSlots = 2;   // concurrent chunked runs of one step (see asim_ctx::slot)

// Grow-only device buffer.
struct DBuf {
  void* p = nullptr;
  size_t cap = 0;
  cudaError_t ensure(size_t bytes) {
    if (bytes <= cap) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    size_t want = bytes < 256 ? 256 : bytes + bytes / 4;
    cudaError_t e = cudaMalloc(&p, want);
    if (e == cudaSuccess) cap = want;
    return e;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

constexpr int kWalkedBytes = 16 * 8;  // ChunkSlot::walked

// One chunked run's device buffers, streams and bookkeeping (chunked.cpp).
struct ChunkSlot {
  DBuf items, begin, spec_good, spec_sum, fix_good, fix_sum, spec_end, fix_end, spec_epoch,
      fix_epoch, flag, counter, end_src, pub, perm, item_cand, spm, fpm, sbusy, fbusy,
      walked;  // walked: unsigned long long statistics [kWalkedBytes / 8] (profiling):
               // [0..3] walk statistics, [4..9] pass-1 warp cycles per stage class
  cudaStream_t main = nullptr;  // the run's own stream (split steps)
  cudaStream_t side[2] = {nullptr, nullptr};  // concurrent walkers
  cudaEvent_t ev_fork = nullptr, ev_join[2] = {nullptr, nullptr}, ev_done = nullptr;
  // the last run on this slot (its per-unit buffers stay valid until the next one)
  bool last_valid = false;
  bool last_u32 = false;
  uint64_t last_gen = 0;  // batch generation it ran on
  asim::ChunkParams last_params{};
  std::vector<asim::ItemDesc> last_items;
  std::vector<int32_t> last_pos;  // batch candidate -> item * 32 + lane (-1: not in the run)
  std::vector<DBuf*> bufs() {
    return {&items, &begin, &spec_good, &spec_sum, &fix_good, &fix_sum, &spec_end, &fix_end,
            &spec_epoch, &fix_epoch, &flag, &counter, &end_src, &pub, &perm, &item_cand,
            &spm, &fpm, &sbusy, &fbusy, &walked};
  }
};

struct HostProblem {
  int32_t M = 0, P = 0, S = 0;
  std::vector<int64_t> slo, stage, tail, mem;
  std::vector<int32_t> cfg_stages, cfg_devices;
  int32_t num_devices = 0;
  int64_t budget = 0;
  int64_t max_service = 0;  // max over (m,p) of sum_k stage + tail
  int64_t mem_at(int m, int p) const { return mem[(int64_t)m * P + p]; }
};

struct asim_ctx {
  int device = 0;
  std::string err;
  int64_t launches = 0;
  bool broken = false;

  bool has_problem = false;
  HostProblem hp;
  DBuf d_stage, d_tail, d_slo, d_cfg_stages, d_dtab32, d_dtab64;

  bool has_trace = false;
  int64_t n = 0;
  int64_t max_arrival = 0;
  int64_t min_arrival = 0;
  std::vector<int64_t> model_n;  // [M] requests per model in the trace
  DBuf d_arrival, d_model;
  DBuf d_moff, d_midx;  // per-model request lists (CSR) for the batching kernel
  bool has_midx = false;  // d_moff/d_midx match the current trace
  DBuf d_inc;           // batching stage increments (asim_evaluate_batching)
  DBuf d_order;         // batching launch order (costliest candidates first)
  DBuf d_mcum;          // per-model running arrival sums (batching)

  // statistics (asim_set_profiling)
  bool profiling = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> events;
  // chunked-path phases timed by their own events: 0 = pass 1, 1 = pass 2, 2 = walk
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> phase_events[3];
  double phase_ms[3] = {0.0, 0.0, 0.0};
  int64_t p1_updates = 0, p1_live = 0, p1_slots = 0;  // pass-1 work (host-counted, profiling)
  int64_t p1_class[6][2] = {};
  // phase intervals [start, end] in ms after ev_ref (profiling): with split
  // steps two runs' phases overlap, so busy time is the union of intervals
  cudaEvent_t ev_ref = nullptr;
  std::vector<std::pair<double, double>> phase_iv[3];  // per stage class (dynamic, 1, 2, 4, 8, 16): stage updates, lane slots
  int64_t walk_pred[4] = {0, 0, 0, 0};  // split-step walk prediction: hit, miss, false, neither
  int64_t sim_launches = 0;
  double sim_ms = 0.0;
  int64_t request_evals = 0;
  DBuf d_counter;  // unsigned long long stage-update counter of the kernels that count on
                   // the device (everything but pass 1; slots [1..3] unused)

  int sms = 148;
  DBuf spool[kSearchPool];  // search scratch kept across searches (search.cpp)
  // Chunked runs (chunked.cpp).  A search step may split its candidates into
  // two runs on their own streams (slot 0: the candidates predicted to walk,
  // high priority; slot 1: the rest) so that one run's sequential walks
  // overlap the other's pass 1; each slot owns its buffers and streams.
  ChunkSlot slot[kChunkSlots];
  cudaEvent_t ev_split = nullptr;  // fork point of a split step on the caller's stream
  uint64_t batch_gen = 0;          // incremented by every asim_upload_batch
  int32_t force_path = 0;  // 0 auto, 1 general kernel, 2 chunked kernel (tests)
  int64_t min_chunk = 4096;  // requests per time chunk (chunked path)
  int64_t max_chunks = 256;  // time chunks of a search (ASIM_MAX_CHUNKS; results do not depend on it)
  int64_t walk_log = 0;      // diagnostics: ASIM_WALK_LOG=<cycles> prints long walks (profiling on)
  bool split_steps = false;  // search steps run walk-prone candidates concurrently (ASIM_SPLIT=1: on;
                             // off by default: equal search time since the group-lane walker,
                             // profiles/r2l)
  bool group_cands = true;   // search steps: items group candidates by component (ASIM_GROUP_CANDIDATES=0: off)
  bool scalar_walk = true;   // register-state walker for small components (ASIM_SCALAR_WALK=0: off)
  int32_t glane_walk = 2;    // ASIM_GLANE_WALK (0: off): see ChunkParams::glane_walk
  int32_t glane_smax = 4;    // ASIM_GLANE_SMAX: see ChunkParams::glane_smax

  // scratch for evaluate()
  DBuf d_base_cfg, d_base_mask, d_cand_base, d_cand_model, d_cand_group, d_cand_ok, d_items;
  DBuf d_cand_kmask, d_cand_gmask;
  DBuf d_good, d_sum, d_pm, d_argmax, d_busy;

  asim::DevProblem dev_problem() const {
    asim::DevProblem p;
    p.M = hp.M;
    p.P = hp.P;
    p.S = hp.S;
    p.stage = d_stage.as<int64_t>();
    p.tail = d_tail.as<int64_t>();
    p.slo = d_slo.as<int64_t>();
    p.cfg_stages = d_cfg_stages.as<int32_t>();
    p.dtab32 = d_dtab32.as<uint32_t>();
    p.dtab64 = d_dtab64.as<int64_t>();
    return p;
  }
  asim::DevTrace dev_trace() const {
    asim::DevTrace t;
    t.n = n;
    t.arrival = d_arrival.as<int64_t>();
    t.model = d_model.as<uint16_t>();
    return t;
  }
};

// helpers implemented in ctx.cpp
asim_status asim_fail(asim_ctx* ctx, asim_status code, const std::string& msg);
asim_status asim_cuda(asim_ctx* ctx, cudaError_t e, const char* what);
// Validate the call order and the overflow bound (reading C20).
asim_status asim_ready(asim_ctx* ctx);
// Upload host vector to a grow-only device buffer (async on stream).
template <class T>
cudaError_t upload(DBuf& buf, const std::vector<T>& v, cudaStream_t st) {
  cudaError_t e = buf.ensure(v.size() * sizeof(T) + 8);
  if (e != cudaSuccess || v.empty()) return e;
  return cudaMemcpyAsync(buf.p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, st);
}

// Batch encoding shared by evaluate, evaluate_deltas and the search.
struct HostBatch;
struct HostBatch {
  int32_t G = 0;
  std::vector<int32_t> base_cfg;   // [B][G]
  std::vector<uint64_t> base_mask; // [B][M]
  std::vector<int32_t> cand_base, cand_model, cand_group;
  std::vector<uint8_t> cand_ok;
  std::vector<uint64_t> cand_kmask, cand_gmask;  // optional component restriction
  std::vector<int64_t> cand_key;  // optional: chunked items group candidates by this key
  int32_t slots = 1;               // max over bases of sum of stages
};
// Upload a batch and launch the simulation of candidates [0, C) writing
// good/sum/per-model at out (device pointers, indexed by candidate).
struct ChunkOptions;
// Copy a batch's bases and candidates into the context's device buffers.
asim_status asim_upload_batch(asim_ctx* ctx, const HostBatch& hb, cudaStream_t st);
asim_status asim_run_batch(asim_ctx* ctx, const HostBatch& hb, int64_t begin, int64_t end,
                           const asim::DevOut& out, cudaStream_t st,
                           const ChunkOptions* opt = nullptr, bool* took_chunked = nullptr);

// Options of the chunked path used by the search (all optional).
struct ChunkOptions {
  int64_t J = 0;                         // fixed chunk count (0 = automatic)
  const int64_t* spec_state = nullptr;   // speculation source (device), see ChunkParams
  const int32_t* spec_row = nullptr;     // [B] device
  const int64_t* spec_cand = nullptr;    // per-candidate rows (device), see ChunkParams
  int32_t state_stride = 0;
  const std::vector<uint8_t>* split = nullptr;  // search steps: walk-prone group per candidate
  uint8_t* walk_out = nullptr;  // device [C]: 1 = the candidate walked (launch_walk_flags)
};
bool asim_chunked_eligible(const asim_ctx* ctx, const HostBatch& hb, const asim::DevOut& out);
// Fast heuristic statistics (good, sum, per-model good, per-group busy) of
// every candidate of hb with the warp-cooperative whole-trace kernel; *done =
// false (nothing launched) when some base is not a gap-free uniform config of
// a supported stage count, or its tables do not fit shared memory.
asim_status asim_run_fast_stats(asim_ctx* ctx, const HostBatch& hb, const asim::DevOut& out,
                                cudaStream_t st, bool* done);
asim_status asim_run_chunked(asim_ctx* ctx, const HostBatch& hb, int64_t begin, int64_t end,
                             const asim::DevOut& out, cudaStream_t st,
                             const ChunkOptions* opt = nullptr);
// As asim_run_chunked over the candidates of [begin, end) split by `group`
// (batch-indexed, 0 or 1): two concurrent runs forked from and joined back
// into `st` (slot 0: group 0 on a high-priority stream).  A group may be empty.
asim_status asim_run_chunked_split(asim_ctx* ctx, const HostBatch& hb, int64_t begin, int64_t end,
                                   const std::vector<uint8_t>& group, const asim::DevOut& out,
                                   cudaStream_t st, const ChunkOptions* opt);
// After a chunked run: true boundary states of chosen candidates of that run
// (batch index c -> row of `out`, see publish_kernel).  Returns ASIM_ESTATE if
// a candidate was not part of the last run.
asim_status asim_publish_candidates(asim_ctx* ctx, const std::vector<int64_t>& cands,
                                    const std::vector<int32_t>& rows, int64_t* out,
                                    cudaStream_t st);
