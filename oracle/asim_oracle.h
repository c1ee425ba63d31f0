/* asim_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct CPU discrete-event simulator of AlpaServe's
 * runtime semantics (arXiv 2302.11665 §4.3; §6 P:812-813:
 * "a continuous-time, discrete-event simulator ... maintains a global clock").
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  It shares no header, source,
 * table or helper with the product (include/asim.h, paper_2302_11665_b200/):
 * the structs below are this file's own.
 *
 * Semantics (readings C1-C13):
 *  - every group is a tandem of s FCFS single servers (one per pipeline
 *    stage), infinite buffers between stages; a request of model m occupies
 *    stage k of a group with config p for stage_ns[m][p][k] ns; tail_ns[m][p]
 *    is added to the finish time and occupies nothing (C4, C5);
 *  - the controller dispatches each arrival to the hosting group with the
 *    earliest predicted finish, ties to the lowest group index (C1);
 *    the prediction is a dry run of a deep copy of that group;
 *  - the group rejects at receipt if finish - arrival > slo (C2, C3);
 *  - events at equal time: stage completions before arrivals; arrivals in
 *    trace order (C6); idle state at t = 0 (C7).
 * All arithmetic is int64 nanoseconds.
 */
#ifndef ASIM_ORACLE_H
#define ASIM_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int32_t num_models, num_configs, max_stages;
  const int64_t* slo_ns;     /* [M] */
  const int32_t* cfg_stages; /* [P] */
  const int32_t* cfg_devices;/* [P] */
  const int64_t* stage_ns;   /* [M][P][max_stages] */
  const int64_t* tail_ns;    /* [M][P] */
  const int64_t* mem_bytes;  /* [M][P], < 0 = not placeable */
  int32_t num_devices;
  int64_t device_budget_bytes;
} asim_oracle_problem;

typedef struct {
  int64_t n;
  const int64_t* arrival_ns; /* [n] non-decreasing, >= 0 */
  const int32_t* model;      /* [n] */
} asim_oracle_trace;

/* Returns 0 on success, <0 on invalid input (message via asim_oracle_error()).
 * Outputs: *good, *sum_latency_ns; good_per_model [M] (nullable);
 * finish_ns [n] (nullable; finish time, -1 = rejected);
 * served_by [n] (nullable; group index, -1 = rejected). */
int32_t asim_oracle_simulate(const asim_oracle_problem* prob, const asim_oracle_trace* tr,
                             int32_t num_groups, const int32_t* group_cfg,
                             const uint64_t* host_mask, int64_t* good,
                             int64_t* sum_latency_ns, int64_t* good_per_model,
                             int64_t* finish_ns, int32_t* served_by);

/* Memory / device feasibility of one placement (reading C11): 1 feasible,
 * 0 infeasible, <0 invalid input. */
int32_t asim_oracle_feasible(const asim_oracle_problem* prob, int32_t num_groups,
                             const int32_t* group_cfg, const uint64_t* host_mask);

/* C placements [C][max_groups] / [C][M]; infeasible ones get good = -1.
 * num_threads <= 0 means hardware_concurrency().  Returns 0 or <0. */
int32_t asim_oracle_evaluate(const asim_oracle_problem* prob, const asim_oracle_trace* tr,
                             int64_t num_candidates, int32_t max_groups,
                             const int32_t* group_cfg, const uint64_t* host_mask,
                             int32_t num_threads, int64_t* good, int64_t* sum_latency_ns,
                             int64_t* good_per_model);

/* Dynamic batching variant (§5.4, C31-C37): same outputs as
 * above.  stage_inc_ns [M][P][max_stages] >= 0: a batch of k requests occupies
 * stage j for stage_ns + (k-1) * stage_inc_ns; max_batch >= 1; at most 64
 * models; every first-stage latency >= 1 ns. */
int32_t asim_oracle_simulate_batching(const asim_oracle_problem* prob,
                                      const asim_oracle_trace* tr, int32_t num_groups,
                                      const int32_t* group_cfg, const uint64_t* host_mask,
                                      const int64_t* stage_inc_ns, int32_t max_batch,
                                      int64_t* good, int64_t* sum_latency_ns,
                                      int64_t* good_per_model, int64_t* finish_ns,
                                      int32_t* served_by);
int32_t asim_oracle_evaluate_batching(const asim_oracle_problem* prob,
                                      const asim_oracle_trace* tr, int64_t num_candidates,
                                      int32_t max_groups, const int32_t* group_cfg,
                                      const uint64_t* host_mask, const int64_t* stage_inc_ns,
                                      int32_t max_batch, int32_t num_threads, int64_t* good,
                                      int64_t* sum_latency_ns, int64_t* good_per_model);

int32_t asim_oracle_hardware_threads(void);
const char* asim_oracle_error(void);

#ifdef __cplusplus
}
#endif
#endif
