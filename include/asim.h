/* asim.h -- C ABI of libasim.so: the batched SLO-attainment simulator that
 * AlpaServe's placement search calls for every candidate placement
 * (arXiv 2302.11665; PAPER.md cited as P:<line>).
 *
 * What it computes.  Given
 *   - a set of models with per-(model, parallel config) stage latencies and
 *     per-device memory ("parallelize(m, g, p)", Alg. 1; §4.1
 *     P:670-684),
 *   - a device cluster (device count, per-device memory budget),
 *   - a time-sorted request trace W with per-model SLOs ("we assume we know
 *     the arrival process in advance"; "SLO Scale"), and
 *   - a batch of candidate placements ("a specific cluster group partition,
 *     model selection, and parallel configuration"),
 * it returns for every candidate the number of requests that finish within
 * their SLO ("SLO attainment") plus the sum of their latencies, and the
 * argmax candidate ("pick_highest_SLO_attainment", Alg. 1).
 *
 * Runtime semantics (§4.3; readings C1-C13):
 *   - each group is a tandem of s FCFS single-server stages with unbounded
 *     buffers; a request of model m on a group with config p occupies stage k
 *     for stage_ns[m][p][k]; tail_ns[m][p] is added to its finish time only;
 *   - each request goes to the hosting group with the earliest predicted
 *     finish, ties to the lowest group index ("the group with the shortest
 *     queue length", P:791 -- reading C1);
 *   - the group rejects it at receipt if finish - arrival > slo_ns[m]
 *     ("rejects the request if it cannot", P:792 -- readings C2, C3);
 *   - equal timestamps are taken in trace order; all stages idle at t = 0.
 * Everything is int64 nanoseconds and integer counts: results are exact and
 * deterministic (bit-identical to the CPU oracle in oracle/).
 *
 * Conventions.
 *   - Every call returns asim_status: 0 = OK, < 0 = error; the message is in
 *     asim_last_error(ctx).  No call throws or aborts across the ABI.  Input
 *     errors are detected on the host before anything is launched.  After
 *     ASIM_ECUDA the context is unusable (destroy it).
 *   - ptr_kind says whether bulk arrays are host (ASIM_HOST) or device
 *     (ASIM_DEVICE, allocated on the context's device) pointers.  Device
 *     inputs/outputs are stream-ordered on `cuda_stream` (a cudaStream_t;
 *     NULL = legacy default stream); host outputs are complete on return.
 *   - Problem and trace arrays are COPIED into context-owned device memory;
 *     candidate and result arrays are BORROWED for the duration of the call.
 *   - One context per (thread, device); a context is not thread-safe.
 */
#ifndef ASIM_H
#define ASIM_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

#define ASIM_ABI_VERSION 1
#define ASIM_MAX_GROUPS 64   /* host_mask is a uint64 bit set over groups      */
#define ASIM_MAX_STAGES 64   /* per config                                      */
#define ASIM_MAX_SLOTS 128   /* sum of stages over the groups of one placement  */
#define ASIM_MAX_MODELS 65535

typedef int32_t asim_status;
enum {
  ASIM_OK = 0,
  ASIM_EINVAL = -1,    /* null required pointer, bad size or enum            */
  ASIM_EUNSORTED = -2, /* trace not non-decreasing, or a negative arrival    */
  ASIM_ERANGE = -3,    /* id / count out of range, or an int64 overflow bound */
  ASIM_ENOMEM = -4,    /* device or host allocation failed                   */
  ASIM_ECUDA = -5,     /* CUDA runtime error (context now unusable)          */
  ASIM_ESTATE = -6     /* call order: e.g. evaluate before set_problem/trace */
};
enum { ASIM_HOST = 0, ASIM_DEVICE = 1 };

typedef struct asim_ctx asim_ctx;       /* opaque */
typedef struct asim_search asim_search; /* opaque */

int32_t asim_abi_version(void);

/* Create a context on CUDA device `cuda_device` (sm_100a required).
 * *out receives the context; on error *out is NULL. */
asim_status asim_create(int32_t cuda_device, asim_ctx** out);
/* Free the context and every device buffer it owns.  NULL is a no-op. */
void asim_destroy(asim_ctx* ctx);
/* Message of the last failed call on ctx; owned by ctx, valid until its next
 * call.  NULL ctx -> message of the last failed asim_create on this thread. */
const char* asim_last_error(const asim_ctx* ctx);
/* Number of kernels this context has launched so far (for the benchmark's
 * gpu_launches count). */
int64_t asim_launch_count(const asim_ctx* ctx);

/* Kernel statistics for the benchmark's roofline (asim_set_profiling(ctx, 1)
 * records CUDA events around every simulation launch on its stream).
 *   sim_launches / sim_ms  simulation-kernel launches and their summed
 *                          device time (ms, CUDA events)
 *   stage_updates          algorithmic work: one max-plus update of one
 *                          pipeline stage of one hosting group, per request
 *                          and candidate
 *   request_evals          (request, candidate) pairs simulated
 * asim_get_stats synchronises the recorded events. */
typedef struct {
  int64_t launches;
  int64_t sim_launches;
  double sim_ms;
  int64_t stage_updates;
  int64_t request_evals;
  int64_t chunk_reruns;  /* chunks re-simulated because their start state was wrong */
  int64_t walk_candidates;      /* candidates (items for mixed configs) that walked >= 1 chunk */
  int64_t walk_critical_chunks; /* sum over walk launches of the longest single walk (chunks):
                                   the sequential critical path of the walk pass */
  double spec_ms;               /* summed device time of the chunked path's pass-1 launches */
  int64_t spec_stage_updates;   /* stage updates performed by pass 1 (part of stage_updates) */
  double pass2_ms;              /* summed device time of the chunked path's pass-2 launches */
  double walk_ms;               /* summed device time of the walk pass (all walkers) */
  int64_t spec_lane_slots;      /* pass 1: requests processed by its warps x 32 lanes */
  int64_t spec_live_lanes;      /* pass 1: (request, lane) pairs whose candidate simulates the
                                   request (live); live / slots = lane utilisation */
  int64_t walk_predicted;       /* search steps: simulated candidates that walked and had walked
                                   when last simulated (run first, split steps) */
  int64_t walk_unpredicted;     /* ... that walked but had not */
  int64_t walk_mispredicted;    /* ... that had walked but did not now */
  /* pass 1 per stage class (index 0: mixed configs, 1..5: S = 1, 2, 4, 8, 16):
   * warp cycles spent in its units (clock64), stage updates, lane slots */
  int64_t spec_class_cycles[6];
  int64_t spec_class_updates[6];
  int64_t spec_class_slots[6];
  /* busy time of each phase = length of the union of its launches' intervals
   * (ms): split steps run two chunked runs concurrently, so the summed
   * spec_ms / pass2_ms / walk_ms can exceed the wall time */
  double spec_busy_ms, pass2_busy_ms, walk_busy_ms;
} asim_stats;
asim_status asim_set_profiling(asim_ctx* ctx, int32_t on);
asim_status asim_get_stats(asim_ctx* ctx, asim_stats* out);
asim_status asim_reset_stats(asim_ctx* ctx);
/* Kernel selection (testing): 0 = automatic (default), 1 = general
 * lane-per-candidate kernel over the whole trace, 2 = chunked kernel with
 * speculative time chunks and exact fix-up whenever the batch allows it,
 * 3 = as 2 with int64 absolute times forced.
 * Results are identical for every choice. */
asim_status asim_set_path(asim_ctx* ctx, int32_t path);
/* Minimum time-chunk length in requests for the chunked kernel (default
 * 4096; small values exercise the fix-up in tests).  A search uses
 * min(256, n / min_requests) chunks (environment ASIM_MAX_CHUNKS overrides the
 * cap).  Results do not depend on either. */
asim_status asim_set_chunk_size(asim_ctx* ctx, int64_t min_requests);

/* ---------------------------------------------------------------- problem */
/* "a set of models" + "a cluster resource specification".  All
 * arrays are host pointers, row-major, and are copied.
 *   num_models M in [1, ASIM_MAX_MODELS]; num_configs P >= 1;
 *   max_stages S in [1, ASIM_MAX_STAGES]
 *   slo_ns[M]         >= 0; INT64_MAX = no deadline
 *   cfg_stages[P]     s_p in [1, S]  (inter-op degree, §4.1)
 *   cfg_devices[P]    devices used by one group of config p (s_p * n_p), >= 1
 *   stage_ns[M][P][S] occupancy of stage k (k < s_p), >= 0
 *   tail_ns[M][P]     overhead added to the finish only, >= 0
 *   mem_bytes[M][P]   bytes per device of one replica; < 0 = (m,p) not placeable
 *   num_devices       cluster size D >= 1;  device_budget_bytes >= 0
 * Bound (reading C20): sum_k stage_ns + tail_ns <= 2^60 for every (m, p).
 * A trace set earlier stays valid when M is unchanged, else it must be set
 * again (ASIM_ESTATE until then).
 * Errors: ASIM_EINVAL (null/size), ASIM_ERANGE (values out of range). */
typedef struct {
  int32_t num_models, num_configs, max_stages;
  const int64_t* slo_ns;
  const int32_t* cfg_stages;
  const int32_t* cfg_devices;
  const int64_t* stage_ns;
  const int64_t* tail_ns;
  const int64_t* mem_bytes;
  int32_t num_devices;
  int64_t device_budget_bytes;
} asim_problem;
asim_status asim_set_problem(asim_ctx* ctx, const asim_problem* problem);

/* ------------------------------------------------------------------ trace */
/* The workload W: n requests, arrival_ns[n] non-decreasing and >= 0,
 * model[n] in [0, M).  Requires asim_set_problem first (ASIM_ESTATE).
 * Copied into device memory (ptr_kind says where the inputs live).
 * n in [0, 2^31 - 1] (int32 request indices); n may be 0 (attainment 1.0,
 * reading C9).  Errors: ASIM_EUNSORTED,
 * ASIM_ERANGE (model id, arrival > 2^62, or max arrival + n * max service
 * >= 2^62), ASIM_EINVAL. */
asim_status asim_set_trace(asim_ctx* ctx, int64_t n, const int64_t* arrival_ns,
                           const int32_t* model, int32_t ptr_kind, void* cuda_stream);

/* ------------------------------------------------------------- candidates */
/* Full candidates: C placements of up to max_groups groups.
 *   group_cfg[C][max_groups]  config id of group g, -1 = no group
 *   host_mask[C][M]           bit g set <=> model m has a replica on group g
 * Candidate validity (data, not errors): a candidate that violates memory
 * ("if sel' is in memory constraint", Alg. 1; per device, sum over the
 * hosted models of mem_bytes[m][p_g] <= budget), uses more than num_devices
 * devices, or hosts m on a config with mem_bytes < 0, gets good = -1.
 * Structural errors (ASIM_ERANGE): config id out of range, a mask bit on a
 * group with cfg -1 or g >= max_groups, sum of stages > ASIM_MAX_SLOTS. */
typedef struct {
  int64_t num_candidates;
  int32_t max_groups; /* <= ASIM_MAX_GROUPS */
  const int32_t* group_cfg;
  const uint64_t* host_mask;
  int32_t ptr_kind;
} asim_candidates;

/* One greedy step in delta form: candidate c = base placement cand_base[c]
 * plus one replica of model cand_model[c] on group cand_group[c]
 * (sel.add_model_to_group(m, g), Alg. 1).  cand_model[c] = -1 means the
 * base itself.  The addition must name an existing group (ASIM_ERANGE);
 * adding a model the group already hosts leaves the base unchanged. */
typedef struct {
  int32_t num_bases, max_groups;
  const int32_t* base_group_cfg;  /* [B][max_groups] */
  const uint64_t* base_host_mask; /* [B][M] */
  int64_t num_candidates;
  const int32_t* cand_base;  /* [C] */
  const int32_t* cand_model; /* [C] */
  const int32_t* cand_group; /* [C] */
  int32_t ptr_kind;
} asim_deltas;

/* Outputs, host or device per ptr_kind.
 *   good[C]               required; requests finished within SLO; -1 infeasible
 *   sum_latency_ns[C]     optional (NULL); sum of (finish - arrival) over good
 *   good_per_model[C][M]  optional; good split by model
 *   argmax[1]             optional; index of the max good (ties -> lowest
 *                         index), -1 if no candidate is feasible
 *   busy_ns[C][max_groups] optional; per group, the sum over its accepted
 *                         requests of their stage occupancies (sum_k stage_ns)
 *                         -- the group's busy time times its stage count
 *   ptr_kind              where every output array lives
 * Requesting good_per_model or busy_ns selects the general kernel. */
typedef struct {
  int64_t* good;
  int64_t* sum_latency_ns;
  int64_t* good_per_model;
  int64_t* argmax;
  int32_t ptr_kind;
  int64_t* busy_ns;
} asim_results;

asim_status asim_evaluate(asim_ctx* ctx, const asim_candidates* cands, asim_results* out,
                          void* cuda_stream);
asim_status asim_evaluate_deltas(asim_ctx* ctx, const asim_deltas* cands, asim_results* out,
                                 void* cuda_stream);

/* ------------------------------------------------------ dynamic batching */
/* The batching variant of the simulator (§5.4 "Batching strategy", P:173:
 * "When a request arrives, it will get executed immediately if any device
 * group is available.  Otherwise, it will be put into a per-model requests
 * queue for batching.  When a device group becomes idle, it will choose a
 * model which has a replica on it and batch as many requests as possible from
 * the requests queue of the model while satisfying the SLO requirements";
 * latency "grows linearly with the batch size").  Readings C31-C37
 * (DESIGN.md):
 *   - a batch of k requests of model m occupies stage j of a group with
 *     config p for stage_ns[m][p][j] + (k-1) * stage_inc_ns[m][p][j];
 *     tail_ns is added to the finish only and does not grow with k;
 *   - a group is available when its first stage is idle;
 *   - an arrival that finds available hosting groups runs alone on the one
 *     with the earliest finish (ties -> lowest index), or is rejected if even
 *     that misses its SLO; otherwise it waits in its model's FIFO;
 *   - a group that becomes available takes, among its hosted models with
 *     waiting requests, the one whose head request is earliest in the trace;
 *     a head that misses its SLO even alone is rejected and the choice
 *     repeated; else the batch is the longest queue prefix (<= max_batch)
 *     whose members all meet the SLO;
 *   - groups available at the same time choose in ascending index, after
 *     every completion and before every arrival at that time (C6).
 * stage_inc_ns: [M][P][max_stages] int64 >= 0, HOST memory, copied.
 * Candidates as for asim_evaluate (full placements, infeasible -> good = -1).
 * Outputs: good, sum_latency_ns, good_per_model, argmax as for asim_evaluate;
 * busy_ns must be NULL (ASIM_EINVAL).
 * Errors: ASIM_ERANGE if M > 64, max_batch outside [1, 2^20], an increment
 * < 0, a first-stage latency stage_ns[m][p][0] < 1 ns, batched stages + tail
 * > 2^60 or max arrival + n * max batched service >= 2^62, or the placement's
 * state does not fit shared memory; ASIM_EINVAL for null pointers. */
typedef struct {
  int32_t max_batch;
  const int64_t* stage_inc_ns;
} asim_batching;

asim_status asim_evaluate_batching(asim_ctx* ctx, const asim_candidates* cands,
                                   const asim_batching* opt, asim_results* out,
                                   void* cuda_stream);

/* pick_highest_SLO_attainment (Alg. 1) over any vector of good counts,
 * e.g. the gathered shards of a multi-GPU evaluation: *out = index of the
 * maximum (ties -> lowest index), -1 when n == 0 or every entry is < 0
 * (infeasible).  good: n int64, host or device per ptr_kind; out: host,
 * complete on return (the call synchronises cuda_stream).  Does not need a
 * problem or trace.  Errors: ASIM_EINVAL (null / bad kind), ASIM_ERANGE (n < 0). */
asim_status asim_argmax(asim_ctx* ctx, const int64_t* good, int64_t n, int32_t ptr_kind,
                        int64_t* out, void* cuda_stream);

/* SLO attainment = good / n; n == 0 -> 1.0; good < 0 -> -1.0. */
double asim_attainment(int64_t good, int64_t n);

/* ----------------------------------------------------------------- search */
/* The placement search: Alg. 1 (simulator-guided greedy, beam k = 1,
 * P:696-737) run for every (group partition, parallel config) of Alg. 2's
 * single-bucket enumeration, all runs advanced in lockstep so one
 * launch evaluates every active run's candidates.  Readings C11-C13:
 *   - candidates of a run are its feasible additions (m, g), m-major,
 *     g-minor; a step's global candidate list concatenates the active runs in
 *     run order;
 *   - each run adds its argmax (ties -> lowest index) and keeps its best
 *     selection on strict '>'; a run stops when it has no feasible addition;
 *   - the best run (strict '>', first wins) is the result.
 * Runs: spec->num_runs = 0 enumerates Alg. 2's single bucket from the
 * problem: for every divisor `size` of num_devices (ascending) and every
 * config p with cfg_devices[p] == size (ascending id), one run of
 * num_devices/size groups of config p.  Otherwise run r has run_num_groups[r]
 * groups with configs run_group_cfg[sum_{r'<r} G_r' ...] (host arrays).
 *
 * Exactness-preserving reuse: a candidate whose connected component of the
 * (group, model) hosting graph is untouched by the previous step's winner
 * keeps its previous good shifted by the base's change (components are
 * simulated independently by construction); only the others are simulated.
 *
 * Stepwise protocol (for candidate sharding across GPUs):
 *   asim_search_prepare  -> *num_candidates = C candidates of this step that
 *                           need simulation (may be 0); -1 = search finished
 *   asim_search_evaluate -> good of global candidates [begin, end) into
 *                           good_dev[0 .. end-begin) (device, stream-ordered)
 *   (all-gather the shards into one device array of C int64)
 *   asim_search_apply    -> per-run argmax over good_all_dev[C] (NULL if C == 0)
 *                           and the memo values; apply
 * asim_search_run does the whole loop on this context's GPU.
 * The search borrows ctx (problem and trace must stay set while it lives).
 *
 * Fast heuristic (spec->fast = 1; "run the simulator only once and
 * place a model with the most unserved requests in an available group with
 * the lowest utilization"; readings C22-C24 in DESIGN.md): each iteration
 * simulates the current selection once; unserved(m) = requests of m not
 * finished within their SLO; among models with unserved > 0 and at least one
 * feasible addition, the largest unserved wins (ties -> lowest m); among its
 * feasible groups the lowest utilization busy_ns / stages wins (ties ->
 * lowest g); the run stops when no such model exists; the best selection
 * (strict '>') is kept.  Fast mode is driven by asim_search_run only.
 *
 * Model and device buckets (spec->buckets = 1; Alg. 2 as printed, P:740-785;
 * readings C25-C28 in DESIGN.md; requires num_runs = 0):
 *   get_potential_model_buckets: models sorted by (model_latency_ns, id) are
 *     cut into contiguous buckets, never between equal latencies, each with
 *     max latency <= ratio * min latency, and only where needed (no two
 *     neighbouring buckets could form one valid bucket); ordered by bucket
 *     count, then cut positions; max_buckets > 0 drops larger partitions.
 *   get_potential_device_buckets: every (H_1..H_k), H_i >= 1, sum = D, in
 *     lexicographic order; with k >= 2 kept iff max r <= bound * min r, with
 *     r_b = (demand_b / sum demand) / (capacity_b / sum capacity), demand_b =
 *     trace requests of bucket b's models, capacity_b = H_b / mean latency of
 *     its models (no demand at all: kept).
 *   each (bucket, H_i) is solved by the runs of the single-bucket
 *     enumeration over H_i devices, restricted to the bucket's models (the
 *     whole trace is simulated; other models are simply not hosted); the best
 *     run (strict '>', first wins) is plm_i*; plm* = concatenation, its good
 *     the sum of the buckets' goods; the best plm* (strict '>') is the result.
 * All runs of all buckets advance in lockstep like single-bucket runs (the
 * fast heuristic applies inside each of them when fast = 1).  The result is
 * read with asim_search_buckets_get; asim_search_result_get reports the
 * concatenated placement (best_run = -1) when it has <= ASIM_MAX_GROUPS
 * groups, else num_groups only.
 *
 * Beam search (spec->beam = k > 1; Alg. 1's beam_sels; readings
 * C29-C30): every run keeps up to k member selections; a step lists the
 * feasible additions of every member (members in beam order, then m, g); a
 * selection reached from two members counts once (its first occurrence); the
 * next members are the top-k by good (stable: ties keep list order); sel* =
 * the first of them and the run's best updates on strict '>'; the run stops
 * when no member has a feasible addition.  k = 1 is the search above.  Runs
 * (asim_search_num_runs / run_info) are Alg. 2 runs, not beam members.
 * Exact run pruning (spec->prune = 1; not in the paper): every run group r
 * gets a capacity bound UB(r) on the good of ANY selection on its groups --
 * an accepted request of model m on a group with config p occupies the
 * group's stages for sum_k d_k(m, p) within [first arrival, last arrival +
 * max SLO], so sum_m x_m * floor(min_p sum_k d_k(m, p) / s_p) <= G * H with
 * x_m <= requests of m (0 for models that fit on none of the groups or lie
 * outside the run's bucket), bounded by the floor of the fractional
 * knapsack.  Before each step, a group whose UB is below the best good some
 * group of its competition (all runs; the bucket job with buckets = 1)
 * already reached stops: it can never be the first best, so best_run,
 * best_good and the placement are exactly those of prune = 0.  A pruned
 * run's asim_search_run_info reports its best up to the step it stopped
 * (asim_search_run_pruned).
 * Exact candidate bounding (spec->cand_bound = 1; not in the paper): a step only
 * needs its argmax.  With K_c the hosting-graph component a candidate
 * changes, good(c) = good(base) - good_base(K_c) + good_c(K_c) <= good(base)
 * - good_base(K_c) + n(K_c), n(K_c) = trace requests of K_c's models.  A
 * candidate whose bound is below the best exact value known (or equal to it
 * with a later (m, g) index) is never simulated; a step simulates the
 * candidates that may gain (bound above the base's good) and the first few
 * others first, and lists the remaining undecided ones in a second round
 * (the next prepare returns them; the run does not advance meanwhile).
 * Every run's winner, and so every result, is that of cand_bound = 0; `steps`
 * counts rounds, `evaluated` only simulated candidates.
 * Errors (asim_search_create): ASIM_EINVAL null latency / bad ratio or bound;
 * fast = 1 with beam > 1;
 * ASIM_ERANGE latency outside [1, 2^60], a run with > ASIM_MAX_GROUPS groups,
 * or more than 2^20 runs in total. */
typedef struct {
  int32_t num_runs;              /* 0 = Alg. 2 single-bucket enumeration */
  const int32_t* run_num_groups; /* [num_runs] */
  const int32_t* run_group_cfg;  /* [sum run_num_groups] */
  int32_t dedup;                 /* 1 = evaluate one representative of provably
                                    identical candidates (exact) */
  int32_t fast;                  /* 1 = the fast heuristic of P:737 instead of
                                    Alg. 1 inside every run (see below) */
  int32_t buckets;               /* 1 = Alg. 2 with model / device buckets */
  int32_t max_buckets;           /* 0 = no cap on the bucket count */
  int64_t ratio_num, ratio_den;  /* bucket latency threshold (SPEC: 4 / 1) */
  int64_t bound_num, bound_den;  /* discrepancy bound (SPEC: 3 / 1) */
  const int64_t* model_latency_ns; /* [M] host; single-device latency (Table 1) */
  int32_t beam;                  /* Alg. 1 beam size k (<= 1 means 1; see below) */
  int32_t prune;                 /* 1 = exact run pruning (see below) */
  int32_t cand_bound;            /* 1 = exact candidate bounding (see below; beam = 1,
                                    not with fast) */
} asim_search_spec;

typedef struct {
  int32_t best_run;        /* -1 if no run improved on the empty placement   */
  int64_t best_good;
  int32_t num_groups;      /* of the best run                                 */
  int32_t* group_cfg;      /* [ASIM_MAX_GROUPS] caller-provided (nullable)    */
  uint64_t* host_mask;     /* [M] caller-provided (nullable)                  */
  int64_t steps;           /* lockstep iterations executed                    */
  int64_t candidates;      /* sum over steps of C (simulate() calls)          */
  int64_t evaluated;       /* candidates actually simulated (after dedup)     */
  int64_t request_evals;   /* sum over evaluated candidates of n (requests)   */
  int64_t memo_hits;       /* candidates whose good came from the component memo */
  int64_t bounded;         /* candidates never simulated (spec->cand_bound) */
} asim_search_result;

asim_status asim_search_create(asim_ctx* ctx, const asim_search_spec* spec, asim_search** out);
void asim_search_destroy(asim_search* s);
asim_status asim_search_prepare(asim_search* s, int64_t* num_candidates);
asim_status asim_search_evaluate(asim_search* s, int64_t begin, int64_t end, int64_t* good_dev,
                                 void* cuda_stream);
asim_status asim_search_apply(asim_search* s, const int64_t* good_all_dev, void* cuda_stream);
/* Work estimate of every candidate of the prepared step (shards
 * "balanced by estimated cost"): the trace requests its simulation replays
 * (those of the models of its hosting-graph component, or all n without
 * component restriction) times the stage count of the group it adds to; >= 1.
 * Identical on every rank (it depends only on the search state), so every rank
 * derives the same contiguous shard bounds from it.  Fills min(cap, C) entries
 * of the host array `cost`.  ASIM_ESTATE outside prepare ... apply. */
asim_status asim_search_costs(const asim_search* s, int64_t cap, int64_t* cost);
asim_status asim_search_run(asim_search* s, void* cuda_stream);
asim_status asim_search_result_get(const asim_search* s, asim_search_result* out);
/* Per-run outcome: best good of run r and its selection (host arrays). */
asim_status asim_search_run_info(const asim_search* s, int32_t run, int32_t* num_groups,
                                 int32_t* group_cfg, uint64_t* host_mask, int64_t* best_good,
                                 int64_t* steps);
int32_t asim_search_num_runs(const asim_search* s);
/* Step history of run r (Alg. 1's sel <- sel + (m*, g*) per iteration,
 * P:720-724): for the i-th step so far, the model and group added and the
 * good of the selection after it (the step's maximum; fast heuristic: the
 * good of its next simulation, -1 while unknown).  Beam > 1: member 0's
 * path.  Fills min(cap, steps) entries of the non-NULL arrays; *count =
 * steps.  ASIM_EINVAL for a bad run, cap < 0 or NULL count. */
asim_status asim_search_run_history(const asim_search* s, int32_t run, int64_t cap,
                                    int32_t* model, int32_t* group, int64_t* good,
                                    int64_t* count);
/* The candidate list of run r's last step (Alg. 1's new_sels):
 * every feasible addition (m, g) in (m, g) order with its good -- simulated,
 * taken from the component memo, or from its duplicate's representative;
 * INT64_MIN for a candidate removed by exact bounding (spec->cand_bound).
 * Valid between asim_search_apply and the next asim_search_prepare
 * (ASIM_ESTATE in between); empty once the run has stopped.  Beam > 1:
 * member 0's list.  Fills min(cap, count) entries; *count = list length. */
asim_status asim_search_run_candidates(const asim_search* s, int32_t run, int64_t cap,
                                       int32_t* model, int32_t* group, int64_t* good,
                                       int64_t* count);
/* Step at which run r was pruned (spec->prune), -1 if it never was or r is
 * out of range. */
int64_t asim_search_run_pruned(const asim_search* s, int32_t run);

/* Bucketed result (spec->buckets = 1), after the search finished.  Arrays are
 * caller-provided host arrays of M entries (a partition has <= M buckets).
 *   bucket_of_model[m]  bucket of model m in the best partition (-1: none)
 *   bucket_devices[i]   H_i of bucket i
 *   bucket_run[i]       run solving bucket i (asim_search_run_info), -1 when no
 *                       run of the bucket serves any request (plm_i* empty)
 * ASIM_ESTATE if the search is not bucketed or not finished. */
typedef struct {
  int64_t best_good;       /* 0 and num_buckets = 0 if nothing improved on {} */
  int32_t num_buckets;
  int64_t partitions;      /* model bucket partitions enumerated */
  int64_t considered;      /* (partition, device buckets) kept after pruning */
  int32_t* bucket_of_model;
  int32_t* bucket_devices;
  int32_t* bucket_run;
} asim_bucket_result;
asim_status asim_search_buckets_get(const asim_search* s, asim_bucket_result* out);

#ifdef __cplusplus
}
#endif
#endif /* ASIM_H */
