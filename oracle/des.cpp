// des.cpp -- TEST INFRASTRUCTURE ONLY (see asim_oracle.h).
//
// An event-driven simulator written to be read against the paper, not to be
// fast.  Per candidate placement it keeps, for every group g and stage k, an
// explicit FIFO queue Q[g][k] and the request in service; a global event heap
// orders stage completions; arrivals are taken in trace order.  Dispatch
// predicts each hosting group's finish by deep-copying that group and running
// the copy alone until the new request leaves its last stage (C1).
//
// Paper passages followed:
//   §4.3  "dispatches each request to the group with the shortest
//                      queue length.  Each group manages a first-come-first-
//                      serve queue.  When a group receives a request, it
//                      checks whether it can serve the request under SLO and
//                      rejects the request if it cannot."
//   §3.2  SLO attainment = fraction of requests finished within
//                      the deadline; "drop the requests that will exceed the
//                      deadline even if we schedule it immediately".
//   §6    continuous-time discrete-event simulator, global clock.
//   Fig. 1 / P:620    pipeline timing (1.1y, 1.6y, 2.1y, 2.6y).

#include "asim_oracle.h"

#include <algorithm>
#include <cstring>
#include <deque>
#include <limits>
#include <queue>
#include <string>
#include <thread>
#include <vector>

namespace {

thread_local std::string g_err;

int32_t fail(const std::string& msg) {
  g_err = msg;
  return -1;
}

struct Problem {
  const asim_oracle_problem* p;
  int64_t stage(int m, int cfg, int k) const {
    return p->stage_ns[((int64_t)m * p->num_configs + cfg) * p->max_stages + k];
  }
  int64_t tail(int m, int cfg) const { return p->tail_ns[(int64_t)m * p->num_configs + cfg]; }
  int64_t mem(int m, int cfg) const { return p->mem_bytes[(int64_t)m * p->num_configs + cfg]; }
  int stages(int cfg) const { return p->cfg_stages[cfg]; }
};

// One pipeline stage server: FIFO queue of waiting request ids, the request in
// service (-1 = idle) and the time its service ends.
struct Stage {
  std::deque<int64_t> queue;
  int64_t busy = -1;
  int64_t busy_until = 0;
};

struct Group {
  int cfg = -1;
  std::vector<Stage> st;
};

// Event = completion of the service of `req` at stage `k` of group `g`.
struct Done {
  int64_t time;
  int64_t seq;  // push order: ties at equal time processed in push order
  int g, k;
  int64_t req;
  bool operator>(const Done& o) const {
    if (time != o.time) return time > o.time;
    return seq > o.seq;
  }
};

// Dry run (reading C1): copy group `grp`, append request `req` (model m) at its
// stage-0 queue at time t, run the copy alone and return the time `req`
// leaves the last stage plus tail[m][cfg].
int64_t dry_run(const Problem& P, const Group& grp, const std::vector<int32_t>& model_of,
                int64_t req, int m, int64_t t) {
  Group g = grp;  // deep copy: queues and services in progress
  const int s = P.stages(g.cfg);
  g.st[0].queue.push_back(req);
  std::priority_queue<Done, std::vector<Done>, std::greater<Done>> ev;
  int64_t seq = 0;
  auto try_start = [&](int k, int64_t now) {
    Stage& S = g.st[k];
    if (S.busy < 0 && !S.queue.empty()) {
      S.busy = S.queue.front();
      S.queue.pop_front();
      S.busy_until = now + P.stage(model_of[S.busy], g.cfg, k);
      ev.push(Done{S.busy_until, seq++, 0, k, S.busy});
    }
  };
  for (int k = 0; k < s; ++k)
    if (g.st[k].busy >= 0) ev.push(Done{g.st[k].busy_until, seq++, 0, k, g.st[k].busy});
  try_start(0, t);
  while (!ev.empty()) {
    Done e = ev.top();
    ev.pop();
    Stage& S = g.st[e.k];
    S.busy = -1;
    if (e.k + 1 < s) {
      g.st[e.k + 1].queue.push_back(e.req);
      try_start(e.k + 1, e.time);
    } else if (e.req == req) {
      return e.time + P.tail(m, g.cfg);
    }
    try_start(e.k, e.time);
  }
  return std::numeric_limits<int64_t>::max();  // unreachable
}

int32_t check_problem(const asim_oracle_problem* p) {
  if (!p || p->num_models <= 0 || p->num_configs <= 0 || p->max_stages <= 0)
    return fail("bad problem sizes");
  if (!p->slo_ns || !p->cfg_stages || !p->stage_ns || !p->tail_ns || !p->mem_bytes)
    return fail("null problem array");
  for (int c = 0; c < p->num_configs; ++c)
    if (p->cfg_stages[c] < 1 || p->cfg_stages[c] > p->max_stages) return fail("bad cfg_stages");
  return 0;
}

int32_t check_placement(const asim_oracle_problem* p, int32_t G, const int32_t* cfg,
                        const uint64_t* mask) {
  if (G < 0 || G > 64) return fail("num_groups must be in [0, 64]");
  for (int g = 0; g < G; ++g)
    if (cfg[g] < -1 || cfg[g] >= p->num_configs) return fail("group_cfg out of range");
  for (int m = 0; m < p->num_models; ++m)
    for (int g = 0; g < 64; ++g)
      if ((mask[m] >> g) & 1ULL)
        if (g >= G || cfg[g] < 0) return fail("host_mask names a group that does not exist");
  return 0;
}

int32_t feasible(const asim_oracle_problem* p, int32_t G, const int32_t* cfg,
                 const uint64_t* mask) {
  Problem P{p};
  int64_t devices = 0;
  for (int g = 0; g < G; ++g) {
    if (cfg[g] < 0) continue;
    devices += p->cfg_devices[cfg[g]];
    int64_t used = 0;
    for (int m = 0; m < p->num_models; ++m) {
      if (!((mask[m] >> g) & 1ULL)) continue;
      if (P.mem(m, cfg[g]) < 0) return 0;  // (m, p) not placeable
      used += P.mem(m, cfg[g]);
    }
    if (used > p->device_budget_bytes) return 0;  // "in memory constraint"
  }
  if (devices > p->num_devices) return 0;
  return 1;
}

int32_t simulate(const asim_oracle_problem* prob, const asim_oracle_trace* tr, int32_t G,
                 const int32_t* group_cfg, const uint64_t* host_mask, int64_t* good_out,
                 int64_t* sum_out, int64_t* per_model, int64_t* finish_ns, int32_t* served_by) {
  Problem P{prob};
  const int M = prob->num_models;
  std::vector<Group> groups(G);
  for (int g = 0; g < G; ++g) {
    groups[g].cfg = group_cfg[g];
    if (group_cfg[g] >= 0) groups[g].st.resize(P.stages(group_cfg[g]));
  }
  std::vector<int32_t> model_of(tr->n);
  for (int64_t i = 0; i < tr->n; ++i) model_of[i] = tr->model[i];
  std::vector<int64_t> predicted(tr->n, -1);
  std::vector<int64_t> good_m(M, 0);
  int64_t good = 0, sum_lat = 0;
  if (finish_ns)
    for (int64_t i = 0; i < tr->n; ++i) finish_ns[i] = -1;
  if (served_by)
    for (int64_t i = 0; i < tr->n; ++i) served_by[i] = -1;

  std::priority_queue<Done, std::vector<Done>, std::greater<Done>> ev;
  int64_t seq = 0;
  auto try_start = [&](int g, int k, int64_t now) {
    Stage& S = groups[g].st[k];
    if (S.busy < 0 && !S.queue.empty()) {
      S.busy = S.queue.front();
      S.queue.pop_front();
      S.busy_until = now + P.stage(model_of[S.busy], groups[g].cfg, k);
      ev.push(Done{S.busy_until, seq++, g, k, S.busy});
    }
  };
  auto on_done = [&](const Done& e) {
    Group& grp = groups[e.g];
    grp.st[e.k].busy = -1;
    const int s = (int)grp.st.size();
    if (e.k + 1 < s) {
      grp.st[e.k + 1].queue.push_back(e.req);
      try_start(e.g, e.k + 1, e.time);
    } else {
      const int m = model_of[e.req];
      const int64_t fin = e.time + P.tail(m, grp.cfg);
      if (fin != predicted[e.req]) {  // the dry run must have been exact
        g_err = "internal: dry-run prediction mismatch";
        std::abort();
      }
      const int64_t a = tr->arrival_ns[e.req];
      good += 1;
      sum_lat += fin - a;
      good_m[m] += 1;
      if (finish_ns) finish_ns[e.req] = fin;
    }
    try_start(e.g, e.k, e.time);
  };

  for (int64_t i = 0; i < tr->n; ++i) {
    const int64_t t = tr->arrival_ns[i];
    // every completion at time <= t happens before this arrival (C6)
    while (!ev.empty() && ev.top().time <= t) {
      Done e = ev.top();
      ev.pop();
      on_done(e);
    }
    const int m = model_of[i];
    int best_g = -1;
    int64_t best_f = 0;
    for (int g = 0; g < G; ++g) {  // ascending g: strict '<' keeps the lowest index on ties
      if (!((host_mask[m] >> g) & 1ULL)) continue;
      const int64_t f = dry_run(P, groups[g], model_of, i, m, t);
      if (best_g < 0 || f < best_f) {
        best_g = g;
        best_f = f;
      }
    }
    if (best_g < 0) continue;                      // hosted nowhere: rejected (C8)
    if (best_f - t > prob->slo_ns[m]) continue;    // misses its SLO: rejected at receipt (C2, C3)
    predicted[i] = best_f;
    if (served_by) served_by[i] = best_g;
    groups[best_g].st[0].queue.push_back(i);
    try_start(best_g, 0, t);
  }
  while (!ev.empty()) {  // drain: every accepted request completes
    Done e = ev.top();
    ev.pop();
    on_done(e);
  }
  *good_out = good;
  if (sum_out) *sum_out = sum_lat;
  if (per_model)
    for (int m = 0; m < M; ++m) per_model[m] = good_m[m];
  return 0;
}

// ---------------------------------------------------------------------------
// Dynamic batching variant (§5.4 "Batching strategy"; §4.3).
//
//   "When a request arrives, it will get executed immediately if any device
//    group is available.  Otherwise, it will be put into a per-model requests
//    queue for batching.  When a device group becomes idle, it will choose a
//    model which has a replica on it and batch as many requests as possible
//    from the requests queue of the model while satisfying the SLO
//    requirements."
//   "the execution latency grows linearly with the batch size"
//
// Readings (C31-C37): a batch of k requests of model m occupies
// stage j of a group with config p for stage_ns[m][p][j] + (k-1) *
// stage_inc_ns[m][p][j]; tail_ns is added to the finish only (C4) and does not
// grow with k.  A group is "available" when its first stage is idle (a
// pipeline accepts the next batch once its first stage is free).  An arrival
// that finds available hosting groups runs alone on the one with the earliest
// predicted finish (lowest index on ties) or is rejected if even that misses
// its SLO; otherwise it waits in its model's FIFO.  A group that becomes
// available picks, among its hosted models with waiting requests, the one
// whose head request came first in the trace; a head that misses its SLO even
// alone is rejected (final) and the choice is repeated; otherwise the batch is
// the longest queue prefix of size <= max_batch whose members all meet their
// SLO.  Groups that become available at the same time choose in ascending
// index order, after every stage completion at that time and before any
// arrival at that time (C6).
// ---------------------------------------------------------------------------

struct BBatch {
  int m;
  std::vector<int64_t> reqs;
  int64_t predicted = -1;
};

struct BStage {
  std::deque<int64_t> queue;  // batch ids
  int64_t busy = -1;          // batch id in service
  int64_t busy_until = 0;
};

struct BGroup {
  int cfg = -1;
  std::vector<BStage> st;
};

struct BProblem {
  Problem P;
  const int64_t* inc;
  int64_t service(int m, int cfg, int k, int64_t size) const {
    return P.stage(m, cfg, k) +
           (size - 1) * inc[((int64_t)m * P.p->num_configs + cfg) * P.p->max_stages + k];
  }
};

// Dry run: copy group `grp`, append a batch of `size` requests of model m at
// its first stage at time t, run the copy alone until that batch leaves its
// last stage; return that time + tail[m][cfg].
int64_t dry_run_batch(const BProblem& B, const BGroup& grp, const std::vector<BBatch>& batches,
                      int m, int64_t size, int64_t t) {
  BGroup g = grp;
  const int s = B.P.stages(g.cfg);
  const int64_t probe = -2;  // id of the probe batch in the copy
  auto model_of = [&](int64_t id) { return id == probe ? m : batches[id].m; };
  auto size_of = [&](int64_t id) { return id == probe ? size : (int64_t)batches[id].reqs.size(); };
  g.st[0].queue.push_back(probe);
  std::priority_queue<Done, std::vector<Done>, std::greater<Done>> ev;
  int64_t seq = 0;
  auto try_start = [&](int k, int64_t now) {
    BStage& S = g.st[k];
    if (S.busy == -1 && !S.queue.empty()) {
      S.busy = S.queue.front();
      S.queue.pop_front();
      S.busy_until = now + B.service(model_of(S.busy), g.cfg, k, size_of(S.busy));
      ev.push(Done{S.busy_until, seq++, 0, k, S.busy});
    }
  };
  for (int k = 0; k < s; ++k)
    if (g.st[k].busy != -1) ev.push(Done{g.st[k].busy_until, seq++, 0, k, g.st[k].busy});
  try_start(0, t);
  while (!ev.empty()) {
    Done e = ev.top();
    ev.pop();
    g.st[e.k].busy = -1;
    if (e.k + 1 < s) {
      g.st[e.k + 1].queue.push_back(e.req);
      try_start(e.k + 1, e.time);
    } else if (e.req == probe) {
      return e.time + B.P.tail(m, g.cfg);
    }
    try_start(e.k, e.time);
  }
  return std::numeric_limits<int64_t>::max();  // unreachable
}

int32_t simulate_batching(const asim_oracle_problem* prob, const asim_oracle_trace* tr, int32_t G,
                          const int32_t* group_cfg, const uint64_t* host_mask,
                          const int64_t* stage_inc, int32_t max_batch, int64_t* good_out,
                          int64_t* sum_out, int64_t* per_model, int64_t* finish_ns,
                          int32_t* served_by) {
  BProblem B{Problem{prob}, stage_inc};
  const int M = prob->num_models;
  std::vector<BGroup> groups(G);
  for (int g = 0; g < G; ++g) {
    groups[g].cfg = group_cfg[g];
    if (group_cfg[g] >= 0) groups[g].st.resize(B.P.stages(group_cfg[g]));
  }
  std::vector<std::deque<int64_t>> Q(M);  // per-model request queues
  std::vector<BBatch> batches;
  std::vector<int64_t> good_m(M, 0);
  int64_t good = 0, sum_lat = 0;
  if (finish_ns)
    for (int64_t i = 0; i < tr->n; ++i) finish_ns[i] = -1;
  if (served_by)
    for (int64_t i = 0; i < tr->n; ++i) served_by[i] = -1;
  auto hosts = [&](int m, int g) { return ((host_mask[m] >> g) & 1ULL) != 0; };

  std::priority_queue<Done, std::vector<Done>, std::greater<Done>> ev;
  int64_t seq = 0;
  auto try_start = [&](int g, int k, int64_t now) {
    BStage& S = groups[g].st[k];
    if (S.busy == -1 && !S.queue.empty()) {
      S.busy = S.queue.front();
      S.queue.pop_front();
      const BBatch& b = batches[S.busy];
      S.busy_until = now + B.service(b.m, groups[g].cfg, k, (int64_t)b.reqs.size());
      ev.push(Done{S.busy_until, seq++, g, k, S.busy});
    }
  };
  auto available = [&](int g) {
    return groups[g].cfg >= 0 && groups[g].st[0].busy == -1 && groups[g].st[0].queue.empty();
  };
  auto start_batch = [&](int g, int m, std::vector<int64_t> reqs, int64_t predicted, int64_t t) {
    BBatch b;
    b.m = m;
    b.reqs = std::move(reqs);
    b.predicted = predicted;
    if (served_by)
      for (int64_t r : b.reqs) served_by[r] = g;
    batches.push_back(std::move(b));
    groups[g].st[0].queue.push_back((int64_t)batches.size() - 1);
    try_start(g, 0, t);
  };
  // An available group forms one batch at time t (or rejects heads and stays idle).
  auto form_batch = [&](int g, int64_t t) {
    for (;;) {
      int bm = -1;
      for (int m = 0; m < M; ++m)  // hosted model whose head came first in the trace
        if (hosts(m, g) && !Q[m].empty() && (bm < 0 || Q[m].front() < Q[bm].front())) bm = m;
      if (bm < 0) return;
      const int64_t limit = std::min<int64_t>(max_batch, (int64_t)Q[bm].size());
      int64_t K = 0, fK = 0;
      for (int64_t k = 1; k <= limit; ++k) {  // longest prefix whose members all meet the SLO
        const int64_t f = dry_run_batch(B, groups[g], batches, bm, k, t);
        bool ok = true;
        for (int64_t j = 0; j < k; ++j)
          if (f - tr->arrival_ns[Q[bm][j]] > prob->slo_ns[bm]) ok = false;
        if (ok) {
          K = k;
          fK = f;
        }
      }
      if (K == 0) {  // the head misses its SLO even alone: rejected
        Q[bm].pop_front();
        continue;
      }
      std::vector<int64_t> reqs(Q[bm].begin(), Q[bm].begin() + K);
      Q[bm].erase(Q[bm].begin(), Q[bm].begin() + K);
      start_batch(g, bm, std::move(reqs), fK, t);
      return;
    }
  };
  auto on_done = [&](const Done& e) {
    BGroup& grp = groups[e.g];
    grp.st[e.k].busy = -1;
    const int s = (int)grp.st.size();
    if (e.k + 1 < s) {
      grp.st[e.k + 1].queue.push_back(e.req);
      try_start(e.g, e.k + 1, e.time);
    } else {
      const BBatch& b = batches[e.req];
      const int64_t fin = e.time + B.P.tail(b.m, grp.cfg);
      if (fin != b.predicted) {
        g_err = "internal: batching dry-run prediction mismatch";
        std::abort();
      }
      for (int64_t r : b.reqs) {
        good += 1;
        sum_lat += fin - tr->arrival_ns[r];
        good_m[b.m] += 1;
        if (finish_ns) finish_ns[r] = fin;
      }
    }
    try_start(e.g, e.k, e.time);
  };

  int64_t i = 0;
  for (;;) {
    const int64_t next_arrival = i < tr->n ? tr->arrival_ns[i] : INT64_MAX;
    if (!ev.empty() && ev.top().time <= next_arrival) {
      // every completion at time T, then the groups available at T in index order (C6)
      const int64_t T = ev.top().time;
      while (!ev.empty() && ev.top().time == T) {
        Done e = ev.top();
        ev.pop();
        on_done(e);
      }
      for (int g = 0; g < G; ++g)
        if (available(g)) form_batch(g, T);
      continue;
    }
    if (i >= tr->n) break;
    const int64_t t = tr->arrival_ns[i];
    const int m = tr->model[i];
    int best_g = -1;
    bool any_host = false;
    int64_t best_f = 0;
    for (int g = 0; g < G; ++g) {
      if (!hosts(m, g)) continue;
      any_host = true;
      if (!available(g)) continue;
      const int64_t f = dry_run_batch(B, groups[g], batches, m, 1, t);
      if (best_g < 0 || f < best_f) {
        best_g = g;
        best_f = f;
      }
    }
    if (!any_host) {
      // hosted nowhere: rejected (C8)
    } else if (best_g < 0) {
      Q[m].push_back(i);  // every hosting group busy: wait for batching
    } else if (best_f - t <= prob->slo_ns[m]) {
      start_batch(best_g, m, std::vector<int64_t>{i}, best_f, t);  // executed immediately
    }  // else: misses its SLO even if executed now: rejected at receipt (C2)
    ++i;
  }
  for (int m = 0; m < M; ++m)
    if (!Q[m].empty()) {
      g_err = "internal: requests left waiting at the end";
      std::abort();
    }
  *good_out = good;
  if (sum_out) *sum_out = sum_lat;
  if (per_model)
    for (int m = 0; m < M; ++m) per_model[m] = good_m[m];
  return 0;
}

int32_t check_batching(const asim_oracle_problem* p, const int64_t* inc, int32_t max_batch) {
  if (!inc) return fail("null stage_inc_ns");
  if (max_batch < 1) return fail("max_batch must be >= 1");
  if (p->num_models > 64) return fail("batching supports at most 64 models");
  const int64_t total = (int64_t)p->num_models * p->num_configs * p->max_stages;
  for (int64_t x = 0; x < total; ++x)
    if (inc[x] < 0) return fail("negative stage_inc_ns");
  for (int m = 0; m < p->num_models; ++m)
    for (int c = 0; c < p->num_configs; ++c)
      if (p->stage_ns[((int64_t)m * p->num_configs + c) * p->max_stages] < 1)
        return fail("batching needs a first-stage latency >= 1 ns");
  return 0;
}

int32_t check_trace(const asim_oracle_problem* p, const asim_oracle_trace* tr) {
  if (!tr || tr->n < 0) return fail("bad trace");
  if (tr->n > 0 && (!tr->arrival_ns || !tr->model)) return fail("null trace array");
  for (int64_t i = 0; i < tr->n; ++i) {
    if (tr->arrival_ns[i] < 0) return fail("negative arrival");
    if (i && tr->arrival_ns[i] < tr->arrival_ns[i - 1]) return fail("trace not sorted");
    if (tr->model[i] < 0 || tr->model[i] >= p->num_models) return fail("model id out of range");
  }
  return 0;
}

}  // namespace

extern "C" {

const char* asim_oracle_error(void) { return g_err.c_str(); }

int32_t asim_oracle_hardware_threads(void) {
  unsigned n = std::thread::hardware_concurrency();
  return n ? (int32_t)n : 1;
}

int32_t asim_oracle_feasible(const asim_oracle_problem* prob, int32_t G, const int32_t* cfg,
                             const uint64_t* mask) {
  if (check_problem(prob) || check_placement(prob, G, cfg, mask)) return -1;
  return feasible(prob, G, cfg, mask);
}

int32_t asim_oracle_simulate(const asim_oracle_problem* prob, const asim_oracle_trace* tr,
                             int32_t G, const int32_t* cfg, const uint64_t* mask, int64_t* good,
                             int64_t* sum_lat, int64_t* per_model, int64_t* finish_ns,
                             int32_t* served_by) {
  if (check_problem(prob) || check_trace(prob, tr) || check_placement(prob, G, cfg, mask))
    return -1;
  if (!good) return fail("null good");
  return simulate(prob, tr, G, cfg, mask, good, sum_lat, per_model, finish_ns, served_by);
}

int32_t asim_oracle_evaluate(const asim_oracle_problem* prob, const asim_oracle_trace* tr,
                             int64_t C, int32_t G, const int32_t* cfg, const uint64_t* mask,
                             int32_t nthreads, int64_t* good, int64_t* sum_lat,
                             int64_t* per_model) {
  if (check_problem(prob) || check_trace(prob, tr)) return -1;
  if (C < 0 || !good) return fail("bad candidates");
  const int M = prob->num_models;
  for (int64_t c = 0; c < C; ++c)
    if (check_placement(prob, G, cfg + c * G, mask + c * M)) return -1;
  if (nthreads <= 0) nthreads = asim_oracle_hardware_threads();
  nthreads = (int32_t)std::max<int64_t>(1, std::min<int64_t>(nthreads, C));
  auto work = [&](int64_t lo, int64_t hi) {
    for (int64_t c = lo; c < hi; ++c) {
      int64_t* pm = per_model ? per_model + c * M : nullptr;
      if (!feasible(prob, G, cfg + c * G, mask + c * M)) {
        good[c] = -1;
        if (sum_lat) sum_lat[c] = 0;
        if (pm)
          for (int m = 0; m < M; ++m) pm[m] = 0;
        continue;
      }
      int64_t s = 0;
      simulate(prob, tr, G, cfg + c * G, mask + c * M, &good[c], &s, pm, nullptr, nullptr);
      if (sum_lat) sum_lat[c] = s;
    }
  };
  std::vector<std::thread> th;
  for (int t = 0; t < nthreads; ++t) {
    int64_t lo = C * t / nthreads, hi = C * (t + 1) / nthreads;
    th.emplace_back(work, lo, hi);
  }
  for (auto& x : th) x.join();
  return 0;
}

int32_t asim_oracle_simulate_batching(const asim_oracle_problem* prob,
                                      const asim_oracle_trace* tr, int32_t G, const int32_t* cfg,
                                      const uint64_t* mask, const int64_t* stage_inc_ns,
                                      int32_t max_batch, int64_t* good, int64_t* sum_lat,
                                      int64_t* per_model, int64_t* finish_ns,
                                      int32_t* served_by) {
  if (check_problem(prob) || check_trace(prob, tr) || check_placement(prob, G, cfg, mask) ||
      check_batching(prob, stage_inc_ns, max_batch))
    return -1;
  if (!good) return fail("null good");
  return simulate_batching(prob, tr, G, cfg, mask, stage_inc_ns, max_batch, good, sum_lat,
                           per_model, finish_ns, served_by);
}

int32_t asim_oracle_evaluate_batching(const asim_oracle_problem* prob,
                                      const asim_oracle_trace* tr, int64_t C, int32_t G,
                                      const int32_t* cfg, const uint64_t* mask,
                                      const int64_t* stage_inc_ns, int32_t max_batch,
                                      int32_t nthreads, int64_t* good, int64_t* sum_lat,
                                      int64_t* per_model) {
  if (check_problem(prob) || check_trace(prob, tr) ||
      check_batching(prob, stage_inc_ns, max_batch))
    return -1;
  if (C < 0 || !good) return fail("bad candidates");
  const int M = prob->num_models;
  for (int64_t c = 0; c < C; ++c)
    if (check_placement(prob, G, cfg + c * G, mask + c * M)) return -1;
  if (nthreads <= 0) nthreads = asim_oracle_hardware_threads();
  nthreads = (int32_t)std::max<int64_t>(1, std::min<int64_t>(nthreads, C));
  auto work = [&](int64_t lo, int64_t hi) {
    for (int64_t c = lo; c < hi; ++c) {
      int64_t* pm = per_model ? per_model + c * M : nullptr;
      if (!feasible(prob, G, cfg + c * G, mask + c * M)) {
        good[c] = -1;
        if (sum_lat) sum_lat[c] = 0;
        if (pm)
          for (int m = 0; m < M; ++m) pm[m] = 0;
        continue;
      }
      int64_t s = 0;
      simulate_batching(prob, tr, G, cfg + c * G, mask + c * M, stage_inc_ns, max_batch,
                        &good[c], &s, pm, nullptr, nullptr);
      if (sum_lat) sum_lat[c] = s;
    }
  };
  std::vector<std::thread> th;
  for (int t = 0; t < nthreads; ++t) {
    int64_t lo = C * t / nthreads, hi = C * (t + 1) / nthreads;
    th.emplace_back(work, lo, hi);
  }
  for (auto& x : th) x.join();
  return 0;
}

}  // extern "C"
