// search.cpp -- the placement search driver (host, native): Alg. 1
// "Simulator-Guided Greedy Model Selection" with beam k = 1 for
// every (group partition, parallel config) of Alg. 2's single bucket
// (P:740-786), all runs advanced in lockstep so that one kernel launch
// evaluates the candidates of every active run.
//
// Per lockstep step:
//   prepare   a1: every active run lists its feasible additions (m, g),
//             m-major / g-minor ("for (m, (g, p)) in M x (G, P)", P:706;
//             "if sel' is in memory constraint"); runs without any
//             stop ("if new_sels = {} then break").
//   evaluate  the simulation kernels on a contiguous shard of the step's list.
//   apply     a7: per run, argmax (ties -> lowest index, "pick_highest",
//             P:722) and sel <- sel + (m*, g*); best_sel on strict '>'.
//
// Everything below is exact; it only decides what needs simulating.
//
// Components.  A placement's simulation splits into independent connected
// components of the bipartite (group, model) hosting graph: a request is only
// dispatched among its model's hosts, and a group's stages only see requests
// of the models it hosts.  So good(placement) = sum over components, and
// candidate c = base + (m, g) differs from its base only inside
// K_c = comp(g) u comp(m) u {m}:
//     good(c) = good(base) - good_base(comp(g)) - good_base(comp(m)) + good_c(K_c).
// The driver keeps every base component's good on the host (updated from the
// winner's total alone), and the kernels simulate only K_c's requests
// ("component restriction", chunk.cu).
//
// Memo.  Candidate (m, g) of step t whose K_c in base(t-1) is disjoint from
// the two components the step-(t-1) winner merged has
//     good_t(m, g) = good_{t-1}(m, g) + good(base(t)) - good(base(t-1)),
// so it is not simulated again.
//
// De-duplication (spec->dedup): adding model m to either of two EMPTY groups
// g1 < g2 with the same config gives the same simulation whenever g1 and g2
// sit between the same pair of m's hosting groups in index order (relabelling
// g1 <-> g2 preserves every dispatch tie-break, reading C1).  Only the lowest
// such g -- the one the argmax picks on a tie anyway -- is simulated.
//
// Speculation states.  The chunked kernels start every time chunk of a
// candidate from its base's true state at that chunk boundary.  After a step
// the new base is the winner: its boundary states are published straight
// from the winner's lane when this rank simulated it (own component from the
// lane, every other slot from the old base), else a one-lane pass simulates
// the winner's component again.  A candidate simulated in the previous step
// too starts from a mix: the new base's state, except in the slots where its
// own previous trajectory differed from the previous base -- the effect of
// its own replica, which the base cannot know.  Speculation never affects
// results; it only decides how soon the fix-up meets the true trajectory.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <functional>
#include <map>
#include <set>
#include <new>
#include <string>
#include <vector>

#include "ctx.h"

namespace {

struct Run {
  int32_t G = 0;
  std::vector<int32_t> cfg;
  std::vector<uint8_t> allowed;  // [M] selectable models (a bucket); empty = all
  std::vector<uint64_t> sel;   // [M] current selection (the base)
  std::vector<int64_t> used;   // [G] bytes per device
  std::vector<uint64_t> best;  // [M] best selection so far
  int64_t best_good = 0;
  bool active = true;
  int64_t steps = 0;
  int64_t base_good = 0;       // good of the base (the last winner)
  // components of the base: union-find over G groups + M models (node G + m)
  std::vector<int32_t> parent;
  std::vector<int64_t> cgood;  // good of the component rooted at a node
  std::vector<int64_t> cn;     // requests (in the trace) of the models of that component
  int32_t round = 0;           // candidate bounding: 1 = deferred candidates still to simulate
  // this step's full candidate list, in (m, g) order
  struct Cand {
    int32_t m, g;
    // 0 simulated in this sub-step (ref = batch index), 1 memo (value),
    // 2 duplicate (ref = rep), 3 deferred (bounding: may still be needed),
    // 4 bounded out (provably not the argmax; no value), 5 simulated in an
    // earlier round of this step (value)
    int8_t kind;
    int64_t ref;
    int64_t good;
    int32_t r1, r2;  // roots of comp(g) and comp(m) in the base
    int64_t ub = 0;  // upper bound on good (bounding)
  };
  std::vector<Cand> cands;
  // memo for the next step, flat over (m, g): good and validity
  std::vector<int64_t> memo_good;
  std::vector<uint8_t> memo_ok;
  // per-root model / group masks of the base (component restriction)
  std::vector<uint64_t> rootK, rootG;
  std::vector<std::pair<int32_t, int32_t>> history;     // winners in order
  std::vector<int64_t> history_good;                    // good of the selection after each
  // batch index of (m, g) among the candidates simulated locally in the
  // previous / current step (-1: not simulated here)
  std::vector<int32_t> prev_idx, cur_idx;
  // whether (m, g) walked (pass 2 left a chunk unmet) the last time it was
  // simulated: such candidates run first, on their own stream (split steps)
  std::vector<uint8_t> walk_prone;

  int32_t find(int32_t x) {
    while (parent[x] != x) x = parent[x] = parent[parent[x]];
    return x;
  }
  bool may_place(int32_t m) const { return allowed.empty() || allowed[m]; }
  // fast heuristic: per-model good / per-group busy of `sel`, and the root of
  // the component changed by the last addition (-1: up to date)
  std::vector<int64_t> fpm, fbusy;
  int32_t pending = -1;
};

// Alg. 2 with buckets: one job per distinct (model bucket, H)
// solved by `runs`; one combo per kept (partition, device buckets).
struct BucketJob {
  std::vector<int32_t> models;
  int32_t H = 0;
  std::vector<int32_t> runs;
};
struct BucketCombo {
  int32_t partition = 0;
  std::vector<int32_t> H;
  std::vector<int32_t> jobs;
};

// 256-bit unsigned products for the exact discrepancy test (bounded inputs:
// every product below stays under 2^230).
struct U256 {
  uint64_t w[4] = {0, 0, 0, 0};
};
U256 u256(unsigned __int128 x) {
  U256 r;
  r.w[0] = (uint64_t)x;
  r.w[1] = (uint64_t)(x >> 64);
  return r;
}
U256 mul64(const U256& a, uint64_t b) {
  U256 r;
  unsigned __int128 carry = 0;
  for (int i = 0; i < 4; ++i) {
    const unsigned __int128 t = (unsigned __int128)a.w[i] * b + carry;
    r.w[i] = (uint64_t)t;
    carry = t >> 64;
  }
  return r;
}
U256 mul128(const U256& a, unsigned __int128 b) {
  const U256 lo = mul64(a, (uint64_t)b);
  const U256 hi = mul64(a, (uint64_t)(b >> 64));
  U256 r;
  unsigned __int128 carry = 0;
  for (int i = 0; i < 4; ++i) {
    const unsigned __int128 t =
        (unsigned __int128)lo.w[i] + (i ? hi.w[i - 1] : 0) + carry;
    r.w[i] = (uint64_t)t;
    carry = t >> 64;
  }
  return r;
}
bool u256_le(const U256& a, const U256& b) {
  for (int i = 3; i >= 0; --i)
    if (a.w[i] != b.w[i]) return a.w[i] < b.w[i];
  return true;
}

}  // namespace

struct asim_search {
  asim_ctx* ctx = nullptr;
  std::vector<Run> runs;
  bool dedup = false;
  int32_t G = 0;  // max groups over runs
  // step state
  bool prepared = false;
  HostBatch hb;
  std::vector<int32_t> base_run;  // base -> run id
  std::vector<int64_t> cost;      // per candidate of the step: estimated simulation work
  std::vector<uint8_t> split;     // per candidate: 0 = predicted to walk, 1 = not
  DBuf d_walk;                    // per candidate: 1 = walked in this step's run
  std::vector<uint8_t> h_walk;
  int64_t eval_lo = 0, eval_hi = 0;  // candidates of the last local evaluate call
  DBuf d_good_all;
  std::vector<int64_t> h_good;
  // chunking / speculation states: per run, absolute free times at every chunk
  // boundary of its base (st_base); st_next receives the next base's
  bool use_states = false;
  bool restrict_k = false;  // component-restricted simulation (M <= 64)
  int64_t J = 1;
  int32_t stride = 1;
  DBuf st_base, st_next, d_rows, d_rows2, d_scratch;
  bool rows_uploaded = false;
  // candidate memory for mixed speculation (see header)
  DBuf cs_prev, cs_cur, spec_mix, d_mixrows;
  std::vector<asim::MixRow> mixrows;  // per batch candidate: (run, previous index)
  bool have_prev = false;
  // fast heuristic: per-model good and per-group busy of each base
  bool fast = false;
  DBuf d_pm, d_busy;
  // beam search (Alg. 1 with k > 1): run group gi owns slots [gi*beam, gi*beam+beam)
  int32_t beam = 1;
  int32_t ngroups = 0;
  std::vector<std::vector<uint64_t>> gbest;  // [ngroups][M] best selection (beam > 1)
  std::vector<int64_t> gbest_good, gsteps;
  // Alg. 2 with buckets
  bool bucketed = false;
  std::vector<std::vector<std::vector<int32_t>>> partitions;
  std::vector<BucketJob> jobs;
  std::vector<BucketCombo> combos;
  // exact run pruning (spec->prune): per run group a bound on the good of ANY
  // selection on its groups, and the step at which it was pruned (-1: never)
  bool prune = false;
  bool bound = false;   // exact candidate bounding (spec->cand_bound)
  int64_t bounded = 0;  // candidates never simulated thanks to it
  std::vector<int64_t> gub;
  std::vector<int64_t> gpruned;
  // statistics
  int64_t steps = 0, candidates = 0, evaluated = 0, memo_hits = 0, base_passes = 0;
  bool finished = false;
};

// candidate memory is skipped when a step's rows would exceed this
static constexpr size_t kMixBytesCap = size_t(6) << 30;

static void prune_runs(asim_search* s);
static int64_t run_capacity_bound(const asim_ctx* ctx, const Run& run);
static const Run& group_run(const asim_search* s, int32_t gi);

static asim_status sfail(asim_search* s, asim_status code, const std::string& m) {
  return asim_fail(s ? s->ctx : nullptr, code, m);
}

// Per-root model and group masks of the run's base (O(G + M) per step).
static void root_masks(Run& run, int32_t M) {
  run.rootK.assign(run.G + M, 0);
  run.rootG.assign(run.G + M, 0);
  for (int32_t x = 0; x < run.G; ++x) run.rootG[run.find(x)] |= 1ULL << x;
  for (int32_t x = 0; x < M; ++x) run.rootK[run.find(run.G + x)] |= 1ULL << x;
}

// Restriction masks of candidate (m, g): models and groups of K_c.
static void component_masks(const Run& run, int32_t m, int32_t g, int32_t r1, int32_t r2,
                            uint64_t* kmask, uint64_t* gmask) {
  *kmask = run.rootK[r1] | run.rootK[r2] | (1ULL << m);
  *gmask = run.rootG[r1] | run.rootG[r2] | (1ULL << g);
}

// Single-bucket enumeration over H devices (reading C13): for every divisor
// size of H (ascending) and config of that size (ascending id), H/size groups.
static asim_status bucket_runs(asim_ctx* ctx, int32_t H, std::vector<std::vector<int32_t>>* out) {
  const HostProblem& hp = ctx->hp;
  for (int32_t size = 1; size <= H; ++size) {
    if (H % size) continue;
    for (int32_t p = 0; p < hp.P; ++p) {
      if (hp.cfg_devices[p] != size) continue;
      const int32_t G = H / size;
      if (G > ASIM_MAX_GROUPS)
        return asim_fail(ctx, ASIM_ERANGE,
                         "Alg. 2 run with more than ASIM_MAX_GROUPS groups; pass explicit runs");
      out->emplace_back(G, p);
    }
  }
  return ASIM_OK;
}

// get_potential_model_buckets (reading C25): backtracking over cut positions
// in lexicographic order for each bucket count k.
static void model_partitions(const std::vector<int64_t>& lat, const std::vector<int32_t>& order,
                             int64_t rn, int64_t rd, int32_t max_buckets,
                             std::vector<std::vector<std::vector<int32_t>>>* out, size_t cap) {
  const int32_t M = (int32_t)order.size();
  auto ok = [&](int32_t a, int32_t b) {  // order[a, b) forms one bucket
    return (unsigned __int128)lat[order[b - 1]] * (uint64_t)rd <=
           (unsigned __int128)(uint64_t)rn * lat[order[a]];
  };
  std::vector<int32_t> cuts;
  for (int32_t k = 1; k <= M && (max_buckets <= 0 || k <= max_buckets); ++k) {
    // rec(prev_start, seg_start, left): choose the next cut > seg_start
    std::function<void(int32_t, int32_t, int32_t)> rec = [&](int32_t prev, int32_t a,
                                                              int32_t left) {
      if (out->size() > cap) return;
      if (left == 0) {
        if (!ok(a, M) || (prev >= 0 && ok(prev, M))) return;
        std::vector<std::vector<int32_t>> part;
        int32_t lo = 0;
        for (size_t i = 0; i <= cuts.size(); ++i) {
          const int32_t hi = i < cuts.size() ? cuts[i] : M;
          std::vector<int32_t> b(order.begin() + lo, order.begin() + hi);
          std::sort(b.begin(), b.end());
          part.push_back(std::move(b));
          lo = hi;
        }
        out->push_back(std::move(part));
        return;
      }
      for (int32_t c = a + 1; c < M; ++c) {
        if (lat[order[c - 1]] == lat[order[c]]) continue;  // never between equal latencies
        if (!ok(a, c)) break;                               // longer segments stay invalid
        if (prev >= 0 && ok(prev, c)) continue;             // would merge with its neighbour
        cuts.push_back(c);
        rec(a, c, left - 1);
        cuts.pop_back();
      }
    };
    rec(-1, 0, k - 1);
  }
}

// get_potential_device_buckets (reading C26), lexicographic.
static void compositions(int32_t D, int32_t k, std::vector<int32_t>& cur,
                         std::vector<std::vector<int32_t>>* out, size_t cap) {
  if (out->size() > cap) return;
  if (k == 1) {
    cur.push_back(D);
    out->push_back(cur);
    cur.pop_back();
    return;
  }
  for (int32_t h = 1; h <= D - k + 1; ++h) {
    cur.push_back(h);
    compositions(D - h, k - 1, cur, out, cap);
    cur.pop_back();
  }
}

// Discrepancy pruning (reading C26): r_b ~ demand_b * sumlat_b / (H_b * n_b).
static bool discrepancy_ok(const std::vector<std::vector<int32_t>>& part,
                           const std::vector<int32_t>& H, const std::vector<int64_t>& lat,
                           const std::vector<int64_t>& demand, int64_t bn, int64_t bd) {
  const size_t k = part.size();
  if (k == 1) return true;
  std::vector<uint64_t> dem(k, 0);
  std::vector<unsigned __int128> sl(k, 0);
  uint64_t total = 0;
  for (size_t b = 0; b < k; ++b)
    for (int32_t m : part[b]) {
      dem[b] += (uint64_t)demand[m];
      sl[b] += (unsigned __int128)lat[m];
    }
  for (uint64_t d : dem) total += d;
  if (total == 0) return true;
  for (size_t i = 0; i < k; ++i)
    for (size_t j = 0; j < k; ++j) {
      if (i == j) continue;
      // r_i <= bound * r_j
      U256 l = mul128(u256(dem[i]), sl[i]);
      l = mul64(mul64(mul64(l, (uint64_t)H[j]), (uint64_t)part[j].size()), (uint64_t)bd);
      U256 r = mul128(u256(dem[j]), sl[j]);
      r = mul64(mul64(mul64(r, (uint64_t)H[i]), (uint64_t)part[i].size()), (uint64_t)bn);
      if (!u256_le(l, r)) return false;
    }
  return true;
}

static constexpr size_t kMaxRuns = size_t(1) << 20;

// Builds the bucketed run list: groups/allowed per run, jobs and combos.
static asim_status bucket_plan(asim_ctx* ctx, const asim_search_spec* spec, asim_search* s,
                               std::vector<std::vector<int32_t>>* groups,
                               std::vector<std::vector<uint8_t>>* allowed) {
  const HostProblem& hp = ctx->hp;
  const int32_t M = hp.M;
  if (spec->num_runs != 0) return asim_fail(ctx, ASIM_EINVAL, "buckets require num_runs = 0");
  if (!spec->model_latency_ns) return asim_fail(ctx, ASIM_EINVAL, "null model_latency_ns");
  if (spec->ratio_num <= 0 || spec->ratio_den <= 0 || spec->bound_num <= 0 || spec->bound_den <= 0)
    return asim_fail(ctx, ASIM_EINVAL, "ratio and bound must be positive fractions");
  std::vector<int64_t> lat(spec->model_latency_ns, spec->model_latency_ns + M);
  for (int64_t l : lat)
    if (l < 1 || l > (int64_t(1) << 60))
      return asim_fail(ctx, ASIM_ERANGE, "model_latency_ns outside [1, 2^60]");
  std::vector<int32_t> order(M);
  for (int32_t m = 0; m < M; ++m) order[m] = m;
  std::stable_sort(order.begin(), order.end(),
                   [&](int32_t a, int32_t b) { return lat[a] < lat[b]; });
  model_partitions(lat, order, spec->ratio_num, spec->ratio_den, spec->max_buckets,
                   &s->partitions, kMaxRuns);
  if (s->partitions.size() > kMaxRuns)
    return asim_fail(ctx, ASIM_ERANGE, "too many model bucket partitions");
  std::map<std::pair<std::vector<int32_t>, int32_t>, int32_t> job_of;
  for (int32_t pi = 0; pi < (int32_t)s->partitions.size(); ++pi) {
    const auto& part = s->partitions[pi];
    std::vector<std::vector<int32_t>> splits;
    std::vector<int32_t> cur;
    compositions(hp.num_devices, (int32_t)part.size(), cur, &splits, kMaxRuns);
    if (splits.size() > kMaxRuns) return asim_fail(ctx, ASIM_ERANGE, "too many device buckets");
    for (const auto& H : splits) {
      if (!discrepancy_ok(part, H, lat, ctx->model_n, spec->bound_num, spec->bound_den)) continue;
      BucketCombo cb;
      cb.partition = pi;
      cb.H = H;
      for (size_t b = 0; b < part.size(); ++b) {
        auto key = std::make_pair(part[b], H[b]);
        auto it = job_of.find(key);
        if (it == job_of.end()) {
          BucketJob job;
          job.models = part[b];
          job.H = H[b];
          std::vector<std::vector<int32_t>> rg;
          asim_status st = bucket_runs(ctx, H[b], &rg);
          if (st) return st;
          std::vector<uint8_t> al(M, 0);
          for (int32_t m : part[b]) al[m] = 1;
          for (auto& g : rg) {
            job.runs.push_back((int32_t)groups->size());
            groups->push_back(std::move(g));
            allowed->push_back(al);
          }
          if (groups->size() > kMaxRuns) return asim_fail(ctx, ASIM_ERANGE, "more than 2^20 runs");
          it = job_of.emplace(key, (int32_t)s->jobs.size()).first;
          s->jobs.push_back(std::move(job));
        }
        cb.jobs.push_back(it->second);
      }
      s->combos.push_back(std::move(cb));
    }
  }
  s->bucketed = true;
  return ASIM_OK;
}

// The search's device scratch is lent by its context's pool (kept across
// searches, like a caching allocator: repeated searches do not pay
// cudaMalloc / cudaFree, which synchronise the device).
static void search_buffers(asim_search* s, DBuf* (&bufs)[kSearchPool]) {
  DBuf* b[kSearchPool] = {&s->d_good_all, &s->st_base, &s->st_next, &s->d_rows, &s->d_rows2,
                          &s->d_scratch, &s->cs_prev, &s->cs_cur, &s->spec_mix, &s->d_mixrows,
                          &s->d_pm, &s->d_busy, &s->d_walk};
  for (int i = 0; i < kSearchPool; ++i) bufs[i] = b[i];
}

extern "C" {

asim_status asim_search_create(asim_ctx* ctx, const asim_search_spec* spec, asim_search** out) {
  if (!ctx || !out) return ASIM_EINVAL;
  *out = nullptr;
  asim_status st = asim_ready(ctx);
  if (st) return st;
  if (!spec) return asim_fail(ctx, ASIM_EINVAL, "null spec");
  const HostProblem& hp = ctx->hp;
  std::vector<std::vector<int32_t>> groups;
  std::vector<std::vector<uint8_t>> allowed;
  asim_search* s = new (std::nothrow) asim_search();
  if (!s) return asim_fail(ctx, ASIM_ENOMEM, "host allocation failed");
  if (spec->buckets) {
    st = bucket_plan(ctx, spec, s, &groups, &allowed);
    if (st) {
      delete s;
      return st;
    }
  } else if (spec->num_runs == 0) {
    // Alg. 2 single bucket: D/size equal groups, one config each (C13)
    for (int32_t size = 1; size <= hp.num_devices; ++size) {
      if (hp.num_devices % size) continue;
      for (int32_t p = 0; p < hp.P; ++p) {
        if (hp.cfg_devices[p] != size) continue;
        const int32_t G = hp.num_devices / size;
        if (G > ASIM_MAX_GROUPS) {
          delete s;
          return asim_fail(ctx, ASIM_ERANGE,
                           "Alg. 2 run with more than ASIM_MAX_GROUPS groups; pass explicit runs");
        }
        groups.emplace_back(G, p);
      }
    }
  } else {
    if (spec->num_runs < 0 || !spec->run_num_groups || !spec->run_group_cfg) {
      delete s;
      return asim_fail(ctx, ASIM_EINVAL, "bad run list");
    }
    int64_t off = 0;
    for (int32_t r = 0; r < spec->num_runs; ++r) {
      const int32_t G = spec->run_num_groups[r];
      asim_status bad = ASIM_OK;
      const char* why = nullptr;
      if (G < 1 || G > ASIM_MAX_GROUPS) {
        bad = ASIM_ERANGE;
        why = "run_num_groups";
      } else {
        std::vector<int32_t> cfg(spec->run_group_cfg + off, spec->run_group_cfg + off + G);
        off += G;
        int32_t slots = 0;
        for (int32_t c : cfg) {
          if (c < 0 || c >= hp.P) {
            bad = ASIM_ERANGE;
            why = "run_group_cfg";
            break;
          }
          slots += hp.cfg_stages[c];
        }
        if (!bad && slots > ASIM_MAX_SLOTS) {
          bad = ASIM_ERANGE;
          why = "run exceeds ASIM_MAX_SLOTS";
        }
        if (!bad) groups.push_back(std::move(cfg));
      }
      if (bad) {
        delete s;
        return asim_fail(ctx, bad, why);
      }
    }
  }
  s->ctx = ctx;
  s->dedup = spec->dedup != 0;
  s->fast = spec->fast != 0;
  s->beam = spec->beam > 1 ? spec->beam : 1;
  if (s->fast && s->beam > 1) {
    delete s;
    return asim_fail(ctx, ASIM_EINVAL, "the fast heuristic has no beam");
  }
  if (s->beam > 4096) {
    delete s;
    return asim_fail(ctx, ASIM_ERANGE, "beam > 4096");
  }
  int32_t stride = 1;
  s->ngroups = (int32_t)groups.size();
  if (groups.size() * (size_t)s->beam > kMaxRuns) {
    delete s;
    return asim_fail(ctx, ASIM_ERANGE, "runs x beam > 2^20");
  }
  if (s->beam > 1) {
    s->gbest.assign(groups.size(), std::vector<uint64_t>(hp.M, 0));
    s->gbest_good.assign(groups.size(), 0);
    s->gsteps.assign(groups.size(), 0);
  }
  for (size_t slot = 0; slot < groups.size() * (size_t)s->beam; ++slot) {
    const size_t gi = slot / s->beam;
    auto& cfg = groups[gi];
    Run r;
    r.G = (int32_t)cfg.size();
    r.cfg = cfg;
    if (!allowed.empty()) r.allowed = allowed[gi];
    r.sel.assign(hp.M, 0);
    r.best.assign(hp.M, 0);
    r.used.assign(r.G, 0);
    r.parent.resize(r.G + hp.M);
    for (size_t i = 0; i < r.parent.size(); ++i) r.parent[i] = (int32_t)i;
    r.cgood.assign(r.G + hp.M, 0);
    r.cn.assign(r.G + hp.M, 0);
    for (int32_t m = 0; m < hp.M; ++m) r.cn[r.G + m] = ctx->model_n[m];
    r.memo_good.assign((size_t)hp.M * r.G, 0);
    r.memo_ok.assign((size_t)hp.M * r.G, 0);
    r.prev_idx.assign((size_t)hp.M * r.G, -1);
    r.walk_prone.assign((size_t)hp.M * r.G, 0);
    r.cur_idx.assign((size_t)hp.M * r.G, -1);
    int64_t devices = 0;
    int32_t slots = 0;
    for (int32_t c : cfg) {
      devices += hp.cfg_devices[c];
      slots += hp.cfg_stages[c];
    }
    stride = std::max(stride, slots);
    if (devices > hp.num_devices) r.active = false;  // the empty placement is already infeasible
    if (slot % s->beam) r.active = false;  // beam_sels = {{}}: one member to start
    s->G = std::max(s->G, r.G);
    s->runs.push_back(std::move(r));
  }
  s->stride = stride;
  {
    DBuf* bufs[kSearchPool];
    search_buffers(s, bufs);
    for (int i = 0; i < kSearchPool; ++i) std::swap(*bufs[i], ctx->spool[i]);  // borrow the pool
  }
  s->prune = spec->prune != 0;
  s->bound = spec->cand_bound != 0 && s->beam == 1 && !s->fast;
  s->gpruned.assign(s->ngroups, -1);
  s->gub.assign(s->ngroups, 0);
  if (s->prune)
    for (int32_t gi = 0; gi < s->ngroups; ++gi) s->gub[gi] = run_capacity_bound(ctx, group_run(s, gi));
  s->J = std::max<int64_t>(
      1, std::min<int64_t>(ctx->max_chunks, ctx->n / std::max<int64_t>(1, ctx->min_chunk)));
  {
    HostBatch probe_hb;
    probe_hb.slots = stride;
    asim::DevOut probe{};
    const bool eligible = asim_chunked_eligible(ctx, probe_hb, probe);
    // the general kernel has no time chunks
    s->use_states = ctx->force_path != 1 && eligible;
    s->restrict_k = s->use_states && hp.M <= 64;
  }
  if (s->use_states && !s->runs.empty()) {
    const size_t bytes = s->runs.size() * (size_t)s->J * stride * 8;
    cudaError_t e = s->st_base.ensure(bytes);
    if (e == cudaSuccess) e = s->st_next.ensure(bytes);
    if (e == cudaSuccess) e = cudaMemset(s->st_base.p, 0, bytes);  // the empty base: idle
    if (e == cudaSuccess) e = cudaMemset(s->st_next.p, 0, bytes);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      asim_search_destroy(s);
      return asim_cuda(ctx, e, "search state buffers");
    }
  }
  *out = s;
  return ASIM_OK;
}

void asim_search_destroy(asim_search* s) {
  if (!s) return;
  DBuf* bufs[kSearchPool];
  search_buffers(s, bufs);
  for (int i = 0; i < kSearchPool; ++i) {
    DBuf& pool = s->ctx ? s->ctx->spool[i] : *bufs[i];
    if (&pool != bufs[i] && pool.cap < bufs[i]->cap) std::swap(pool, *bufs[i]);  // keep the larger
    if (&pool != bufs[i]) bufs[i]->release();
  }
  if (!s->ctx) {
    for (DBuf* b : bufs) b->release();
  }
  delete s;
}

int32_t asim_search_num_runs(const asim_search* s) { return s ? s->ngroups : 0; }

asim_status asim_search_prepare(asim_search* s, int64_t* num_candidates) {
  if (!s || !num_candidates) return ASIM_EINVAL;
  asim_status st = asim_ready(s->ctx);
  if (st) return st;
  if (s->prepared) return sfail(s, ASIM_ESTATE, "prepare called twice without apply");
  if (s->fast) return sfail(s, ASIM_ESTATE, "the fast heuristic is driven by asim_search_run");
  const HostProblem& hp = s->ctx->hp;
  const int32_t M = hp.M, G = s->G;
  HostBatch& hb = s->hb;
  hb = HostBatch();
  hb.G = G;
  s->base_run.clear();
  s->cost.clear();
  s->split.clear();
  s->eval_lo = s->eval_hi = 0;
  s->rows_uploaded = false;
  s->mixrows.clear();
  prune_runs(s);
  int64_t full = 0;
  for (int32_t r = 0; r < (int32_t)s->runs.size(); ++r) {
    Run& run = s->runs[r];
    if (!run.active) continue;
    const int32_t b = (int32_t)s->base_run.size();
    // candidate c of this run goes to the batch (kind 0)
    auto emit = [&](Run::Cand& c, int32_t prev) {
      c.kind = 0;
      c.ref = (int64_t)hb.cand_base.size();
      hb.cand_base.push_back(b);
      hb.cand_model.push_back(c.m);
      hb.cand_group.push_back(c.g);
      hb.cand_ok.push_back(1);
      if (s->restrict_k) {
        uint64_t km = 0, gm = 0;
        component_masks(run, c.m, c.g, c.r1, c.r2, &km, &gm);
        hb.cand_kmask.push_back(km);
        hb.cand_gmask.push_back(gm);
      }
      if (s->restrict_k && s->ctx->group_cands) {
        // chunked items: the candidate's larger component first, so a warp's
        // lanes share the bulk of the requests they replay (ties: (m, g) order)
        const int64_t n1 = run.cn[c.r1], n2 = run.cn[c.r2];
        const int32_t dom = n2 >= n1 ? c.r2 : c.r1, oth = n2 >= n1 ? c.r1 : c.r2;
        hb.cand_key.push_back(((int64_t)dom << 32) | (uint32_t)oth);
      }
      // work estimate (sharding): requests the lane replays x stages per group
      const int64_t nreq = s->restrict_k
                               ? run.cn[c.r1] + (c.r2 != c.r1 ? run.cn[c.r2] : 0)
                               : s->ctx->n;
      s->cost.push_back(std::max<int64_t>(1, nreq) * hp.cfg_stages[run.cfg[c.g]]);
      s->split.push_back(run.walk_prone[(size_t)c.m * run.G + c.g] ? 0 : 1);
      s->mixrows.push_back(asim::MixRow{r, prev});
    };
    if (run.round == 1) {  // the same step, second round: deferred candidates
      if (s->restrict_k) root_masks(run, M);
      for (Run::Cand& c : run.cands)
        if (c.kind == 3) emit(c, -1);
    } else {
      std::vector<uint8_t> empty(run.G, 1);
      for (int32_t m = 0; m < M; ++m)
        for (int32_t g = 0; g < run.G; ++g)
          if ((run.sel[m] >> g) & 1ULL) empty[g] = 0;
      run.cands.clear();
      if (s->restrict_k) root_masks(run, M);
      for (int32_t m = 0; m < M; ++m) {
        if (!run.may_place(m)) continue;  // outside this run's bucket
        std::map<std::pair<int32_t, int32_t>, int64_t> seen;  // (cfg, rank among hosts) -> rep
        for (int32_t g = 0; g < run.G; ++g) {
          if ((run.sel[m] >> g) & 1ULL) continue;  // a model at most once per group (C11)
          const int64_t mb = hp.mem_at(m, run.cfg[g]);
          if (mb < 0 || run.used[g] + mb > hp.budget) continue;  // memory constraint
          ++full;
          Run::Cand c{m, g, 0, 0, 0, run.find(g), run.find(run.G + m)};
          const size_t mi = (size_t)m * run.G + g;
          if (run.memo_ok[mi]) {  // component untouched by the last winner
            c.kind = 1;
            c.good = run.memo_good[mi];
            ++s->memo_hits;
          } else if (s->dedup && empty[g]) {
            const uint64_t below = g ? (run.sel[m] & ((1ULL << g) - 1)) : 0ULL;
            auto key = std::make_pair(run.cfg[g], (int32_t)__builtin_popcountll(below));
            auto sit = seen.find(key);
            if (sit != seen.end()) {
              c.kind = 2;
              c.ref = sit->second;
            } else {
              seen[key] = (int64_t)run.cands.size();
            }
          }
          run.cands.push_back(c);
        }
      }
      if (run.cands.empty()) {  // no feasible addition: this run's Alg. 1 loop ends
        run.active = false;
        continue;
      }
      if (s->bound) {
        // Exact candidate bounding (not in the paper; the step's argmax is
        // unchanged).  good(c) = good(base) - good_base(K_c) + good_c(K_c)
        // and good_c(K_c) <= n(K_c), the trace's requests of K_c's models.
        // Candidates that cannot beat the best exact value known (memo) are
        // dropped; this round simulates the possible gainers (ub > good of
        // the base) and the first kFirst others in (m, g) order, the rest
        // wait for apply, which drops every one the round's best excludes.
        constexpr int kFirst = 4;
        int64_t bg = -1, bi = -1;
        for (size_t i = 0; i < run.cands.size(); ++i) {
          const Run::Cand& c = run.cands[i];
          if (c.kind == 1 && c.good > bg) {
            bg = c.good;
            bi = (int64_t)i;
          }
        }
        int first = 0;
        for (size_t i = 0; i < run.cands.size(); ++i) {
          Run::Cand& c = run.cands[i];
          if (c.kind != 0) continue;
          const bool two = c.r2 != c.r1;
          c.ub = run.base_good - run.cgood[c.r1] - (two ? run.cgood[c.r2] : 0) + run.cn[c.r1] +
                 (two ? run.cn[c.r2] : 0);
          if (c.ub < bg || (c.ub == bg && (int64_t)i > bi)) {
            c.kind = 4;
          } else if (!(c.ub > run.base_good || first < kFirst)) {
            c.kind = 3;
          } else if (c.ub <= run.base_good) {
            ++first;
          }
        }
      }
      for (Run::Cand& c : run.cands)
        if (c.kind == 0) emit(c, run.prev_idx[(size_t)c.m * run.G + c.g]);
    }
    s->base_run.push_back(r);
    for (int32_t g = 0; g < G; ++g) hb.base_cfg.push_back(g < run.G ? run.cfg[g] : -1);
    hb.base_mask.insert(hb.base_mask.end(), run.sel.begin(), run.sel.end());
    int32_t slots = 0;
    for (int32_t c : run.cfg) slots += hp.cfg_stages[c];
    hb.slots = std::max(hb.slots, slots);
  }
  if (s->base_run.empty()) {  // every run has ended: the search is finished
    s->finished = true;
    *num_candidates = -1;
    return ASIM_OK;
  }
  s->prepared = true;
  *num_candidates = (int64_t)hb.cand_base.size();
  s->candidates += full;
  s->evaluated += *num_candidates;
  ++s->steps;
  return ASIM_OK;
}

asim_status asim_search_costs(const asim_search* s, int64_t cap, int64_t* cost) {
  if (!s || cap < 0 || (cap > 0 && !cost)) return ASIM_EINVAL;
  if (!s->prepared) return asim_fail(s->ctx, ASIM_ESTATE, "costs before prepare");
  const int64_t C = (int64_t)s->cost.size();
  for (int64_t i = 0; i < C && i < cap; ++i) cost[i] = s->cost[i];
  return ASIM_OK;
}

asim_status asim_search_evaluate(asim_search* s, int64_t begin, int64_t end, int64_t* good_dev,
                                 void* cuda_stream) {
  if (!s) return ASIM_EINVAL;
  if (!s->prepared) return sfail(s, ASIM_ESTATE, "evaluate before prepare");
  const int64_t C = (int64_t)s->hb.cand_base.size();
  if (begin < 0 || end < begin || end > C) return sfail(s, ASIM_ERANGE, "shard range");
  if (end == begin) return ASIM_OK;
  if (!good_dev) return sfail(s, ASIM_EINVAL, "null good_dev");
  int prev = -1;
  cudaGetDevice(&prev);
  if (prev != s->ctx->device) cudaSetDevice(s->ctx->device);
  cudaStream_t strm = static_cast<cudaStream_t>(cuda_stream);
  asim_status st = ASIM_OK;
  ChunkOptions opt;
  ChunkOptions* popt = nullptr;
  if (s->use_states) {
    if (!s->rows_uploaded) {
      cudaError_t e = upload(s->d_rows, s->base_run, strm);
      if (e != cudaSuccess) {
        if (prev >= 0 && prev != s->ctx->device) cudaSetDevice(prev);
        return asim_cuda(s->ctx, e, "upload rows");
      }
      s->rows_uploaded = true;
    }
    opt.J = s->J;
    opt.state_stride = s->stride;
    opt.spec_state = s->st_base.as<int64_t>();
    opt.spec_row = s->d_rows.as<int32_t>();
    popt = &opt;
    // walk prediction: the candidates that walked when last simulated run
    // first, concurrently with the others (asim_run_chunked_split)
    opt.split = &s->split;
    cudaError_t ew = s->d_walk.ensure((size_t)C + 8);
    if (ew == cudaSuccess) ew = cudaMemsetAsync(s->d_walk.p, 0, (size_t)C, strm);
    if (ew != cudaSuccess) {
      if (prev >= 0 && prev != s->ctx->device) cudaSetDevice(prev);
      return asim_cuda(s->ctx, ew, "walk flags");
    }
    opt.walk_out = s->d_walk.as<uint8_t>();
    // mixed speculation rows for [begin, end) (candidate memory of the last step)
    const size_t per = (size_t)s->J * s->stride * 8;
    if (s->have_prev && (size_t)C * per <= kMixBytesCap) {
      cudaError_t e = s->spec_mix.ensure((size_t)C * per + 8);
      if (e == cudaSuccess) e = upload(s->d_mixrows, s->mixrows, strm);
      if (e == cudaSuccess)
        e = asim::launch_mix_states(begin, end, (int32_t)s->J, s->stride, s->st_base.as<int64_t>(),
                                    s->st_next.as<int64_t>(), s->cs_prev.as<int64_t>(),
                                    s->d_mixrows.as<asim::MixRow>(), s->spec_mix.as<int64_t>(),
                                    strm, &s->ctx->launches);
      if (e != cudaSuccess) {
        if (prev >= 0 && prev != s->ctx->device) cudaSetDevice(prev);
        return asim_cuda(s->ctx, e, "mix speculation");
      }
      opt.spec_cand = s->spec_mix.as<int64_t>();
    }
  }
  asim::DevOut out{};
  out.good = good_dev;
  out.out_offset = begin;
  bool chunked = false;
  st = asim_run_batch(s->ctx, s->hb, begin, end, out, strm, popt, &chunked);
  if (!st && chunked) {
    s->eval_lo = begin;  // the chunk buffers now hold these candidates' trajectories
    s->eval_hi = end;
  }
  if (prev >= 0 && prev != s->ctx->device) cudaSetDevice(prev);
  return st;
}

// New bases' boundary states into st_next, then swap: winners this rank
// simulated are published from their lanes; the others are simulated again,
// one lane each, restricted to their own component.
static asim_status update_states(asim_search* s, const std::vector<int32_t>& winner_run,
                                 const std::vector<const Run::Cand*>& winner, cudaStream_t st,
                                 const std::vector<int32_t>* target_rows = nullptr,
                                 const std::vector<int32_t>* keep_rows = nullptr) {
  // winner_run[i]: the run (old base) the winner extends; target_rows[i]: the
  // st_next row receiving the new base (default: the same run)
  asim_ctx* ctx = s->ctx;
  std::vector<int64_t> pub_c;
  std::vector<int32_t> pub_r;
  HostBatch hb;
  hb.G = s->G;
  std::vector<int32_t> rows, out_rows;
  for (size_t i = 0; i < winner_run.size(); ++i) {
    const Run::Cand& w = *winner[i];
    const int32_t target = target_rows ? (*target_rows)[i] : winner_run[i];
    if (w.kind == 0 && w.ref >= s->eval_lo && w.ref < s->eval_hi) {
      pub_c.push_back(w.ref);
      pub_r.push_back(target);
      continue;
    }
    Run& run = s->runs[winner_run[i]];  // still the old base here
    const int32_t b = (int32_t)rows.size();
    rows.push_back(winner_run[i]);
    out_rows.push_back(target);
    for (int32_t g = 0; g < s->G; ++g) hb.base_cfg.push_back(g < run.G ? run.cfg[g] : -1);
    hb.base_mask.insert(hb.base_mask.end(), run.sel.begin(), run.sel.end());
    int32_t slots = 0;
    for (int32_t c : run.cfg) slots += ctx->hp.cfg_stages[c];
    hb.slots = std::max(hb.slots, slots);
    hb.cand_base.push_back(b);
    hb.cand_model.push_back(w.m);
    hb.cand_group.push_back(w.g);
    hb.cand_ok.push_back(1);
    if (s->restrict_k) {  // rootK / rootG still describe the old base
      uint64_t km = 0, gm = 0;
      component_masks(run, w.m, w.g, w.r1, w.r2, &km, &gm);
      hb.cand_kmask.push_back(km);
      hb.cand_gmask.push_back(gm);
    }
  }
  asim_status rc = asim_publish_candidates(ctx, pub_c, pub_r, s->st_next.as<int64_t>(), st);
  if (rc) return rc;
  if (!rows.empty()) {
    ++s->base_passes;
    cudaError_t e = upload(s->d_rows2, rows, st);
    if (e == cudaSuccess) e = s->d_scratch.ensure(rows.size() * 8 + 8);
    if (e != cudaSuccess) return asim_cuda(ctx, e, "base pass buffers");
    ChunkOptions ob;
    ob.J = s->J;
    ob.state_stride = s->stride;
    ob.spec_state = s->st_base.as<int64_t>();
    ob.spec_row = s->d_rows2.as<int32_t>();
    asim::DevOut bo{};
    bo.good = s->d_scratch.as<int64_t>();
    rc = asim_upload_batch(ctx, hb, st);
    if (!rc) rc = asim_run_chunked(ctx, hb, 0, (int64_t)rows.size(), bo, st, &ob);
    if (rc) return rc;
    std::vector<int64_t> all(rows.size());
    for (size_t i = 0; i < rows.size(); ++i) all[i] = (int64_t)i;
    rc = asim_publish_candidates(ctx, all, out_rows, s->st_next.as<int64_t>(), st);
    if (rc) return rc;
  }
  if (keep_rows) {  // runs whose base did not change (a pending round): carry their rows over
    const size_t row = (size_t)s->J * s->stride * 8;
    for (int32_t r : *keep_rows) {
      cudaError_t e = cudaMemcpyAsync(s->st_next.as<char>() + (size_t)r * row,
                                      s->st_base.as<char>() + (size_t)r * row, row,
                                      cudaMemcpyDeviceToDevice, st);
      if (e != cudaSuccess) return asim_cuda(ctx, e, "carry base states");
    }
  }
  std::swap(s->st_base, s->st_next);
  return ASIM_OK;
}

}  // extern "C"

// sel <- sel + (m, g) on a run whose candidates are this step's (memo for
// the next step, merged component, selection, memory, base good).
static void apply_winner(Run& run, const Run::Cand w, const HostProblem& hp) {
  // memo for the next step: candidates whose component avoids the winner's
  const int64_t shift = w.good - run.base_good;
  std::fill(run.memo_ok.begin(), run.memo_ok.end(), 0);
  for (const Run::Cand& c : run.cands)
    if (c.kind != 3 && c.kind != 4 &&  // values only for candidates that were evaluated
        c.r1 != w.r1 && c.r1 != w.r2 && c.r2 != w.r1 && c.r2 != w.r2) {
      const size_t mi = (size_t)c.m * run.G + c.g;
      run.memo_ok[mi] = 1;
      run.memo_good[mi] = c.good + shift;
    }
  // the merged component's good, from the winner's total alone
  const int64_t merged =
      w.good - run.base_good + run.cgood[w.r1] + (w.r2 != w.r1 ? run.cgood[w.r2] : 0);
  run.parent[w.r1] = w.r2;  // unite comp(g*) and comp(m*)
  run.cgood[w.r2] = merged;
  if (w.r1 != w.r2) run.cn[w.r2] += run.cn[w.r1];
  run.round = 0;
  run.sel[w.m] |= 1ULL << w.g;
  run.used[w.g] += hp.mem_at(w.m, run.cfg[w.g]);
  run.base_good = w.good;
  run.history.emplace_back(w.m, w.g);
  run.history_good.push_back(w.good);
  ++run.steps;
}

// Alg. 1 with beam k > 1 (readings C29-C30): per run group, the
// candidates of all members in (member, m, g) order, a selection reached
// twice kept once (first occurrence), stable top-k by good; member i of the
// next step = its parent member + its addition; sel* = the first; best_sel
// on strict '>'.  Candidate memory (mixed speculation) is not used here.
static asim_status apply_beam(asim_search* s, cudaStream_t st) {
  const HostProblem& hp = s->ctx->hp;
  const int32_t K = s->beam;
  struct Pick {
    int32_t slot, ci;
    int64_t good;
  };
  std::vector<std::pair<int32_t, std::vector<Pick>>> plan;
  for (size_t b = 0; b < s->base_run.size();) {
    const int32_t gi = s->base_run[b] / K;
    std::vector<Pick> all;
    std::set<std::vector<uint64_t>> seen;
    for (; b < s->base_run.size() && s->base_run[b] / K == gi; ++b) {
      const int32_t slot = s->base_run[b];
      const Run& run = s->runs[slot];
      for (size_t i = 0; i < run.cands.size(); ++i) {
        const Run::Cand& c = run.cands[i];
        std::vector<uint64_t> key = run.sel;
        key[c.m] |= 1ULL << c.g;
        if (!seen.insert(std::move(key)).second) continue;  // reached from an earlier member
        all.push_back(Pick{slot, (int32_t)i, c.good});
      }
    }
    std::stable_sort(all.begin(), all.end(),
                     [](const Pick& a, const Pick& b) { return a.good > b.good; });
    if ((int32_t)all.size() > K) all.resize(K);
    plan.emplace_back(gi, std::move(all));
  }
  if (s->use_states) {
    std::vector<int32_t> parents, targets;
    std::vector<const Run::Cand*> cands;
    for (const auto& gp : plan)
      for (size_t i = 0; i < gp.second.size(); ++i) {
        const Pick& pk = gp.second[i];
        parents.push_back(pk.slot);
        targets.push_back(gp.first * K + (int32_t)i);
        cands.push_back(&s->runs[pk.slot].cands[pk.ci]);
      }
    s->have_prev = false;
    asim_status rc = update_states(s, parents, cands, st, &targets);
    if (rc) return rc;
  }
  for (const auto& gp : plan) {
    const int32_t gi = gp.first;
    std::map<int32_t, Run> snap;  // parents before any child overwrites a slot
    for (const Pick& pk : gp.second) snap.emplace(pk.slot, s->runs[pk.slot]);
    for (int32_t i = 0; i < K; ++i) {
      Run& dst = s->runs[gi * K + i];
      if (i >= (int32_t)gp.second.size()) {
        dst.active = false;
        continue;
      }
      const Pick& pk = gp.second[i];
      Run child = snap.at(pk.slot);
      const Run::Cand w = child.cands[pk.ci];
      apply_winner(child, w, hp);
      child.active = true;
      dst = std::move(child);
    }
    ++s->gsteps[gi];
    if (gp.second[0].good > s->gbest_good[gi]) {  // sel* = pick_highest(beam_sels)
      s->gbest_good[gi] = gp.second[0].good;
      s->gbest[gi] = s->runs[gi * K].sel;
    }
  }
  s->prepared = false;
  return ASIM_OK;
}

extern "C" {

asim_status asim_search_apply(asim_search* s, const int64_t* good_all_dev, void* cuda_stream) {
  if (!s) return ASIM_EINVAL;
  if (!s->prepared) return sfail(s, ASIM_ESTATE, "apply before prepare");
  const int64_t C = (int64_t)s->hb.cand_base.size();
  if (C > 0 && !good_all_dev) return sfail(s, ASIM_EINVAL, "null good_all_dev");
  cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
  s->h_good.resize(C);
  const bool walks = s->use_states && s->eval_hi > s->eval_lo;
  if (walks) s->h_walk.resize(C);
  if (C > 0) {
    cudaError_t e =
        cudaMemcpyAsync(s->h_good.data(), good_all_dev, C * 8, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess && walks)
      e = cudaMemcpyAsync(s->h_walk.data() + s->eval_lo, s->d_walk.as<uint8_t>() + s->eval_lo,
                          (size_t)(s->eval_hi - s->eval_lo), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return asim_cuda(s->ctx, e, "copy step results");
  }
  const HostProblem& hp = s->ctx->hp;
  const bool restricted = !s->hb.cand_kmask.empty();
  for (size_t b = 0; b < s->base_run.size(); ++b) {
    Run& run = s->runs[s->base_run[b]];
    // every candidate's good: simulated, memo, or its duplicate's representative
    for (size_t i = 0; i < run.cands.size(); ++i) {
      Run::Cand& c = run.cands[i];
      if (c.kind == 0) {
        c.good = s->h_good[c.ref];
        if (walks && c.ref >= s->eval_lo && c.ref < s->eval_hi) {
          uint8_t& wp = run.walk_prone[(size_t)c.m * run.G + c.g];
          const uint8_t w = s->h_walk[c.ref];
          // statistics of the walk prediction (split steps): walked & predicted,
          // walked & not predicted, predicted & not walked
          s->ctx->walk_pred[w && wp ? 0 : w ? 1 : wp ? 2 : 3] += 1;
          wp = w;
        }
        if (restricted)  // good(base) - good_base(comp(g)) - good_base(comp(m)) + good_c(K_c)
          c.good += run.base_good - run.cgood[c.r1] - (c.r2 != c.r1 ? run.cgood[c.r2] : 0);
      }
    }
  }
  if (s->beam > 1) {
    for (size_t b = 0; b < s->base_run.size(); ++b) {
      Run& run = s->runs[s->base_run[b]];
      for (Run::Cand& c : run.cands)
        if (c.kind == 2) c.good = run.cands[c.ref].good;
    }
    return apply_beam(s, st);
  }
  std::vector<int32_t> winner_run;
  std::vector<const Run::Cand*> winner;
  std::vector<int32_t> pending;  // runs whose step needs another round (bounding)
  for (size_t b = 0; b < s->base_run.size(); ++b) {
    Run& run = s->runs[s->base_run[b]];
    int64_t bi = -1, bg = -1;
    for (size_t i = 0; i < run.cands.size(); ++i) {
      const Run::Cand& c = run.cands[i];
      // evaluated candidates only; a duplicate never beats its representative
      // (same good, later index).  First maximum in (m, g) order: lowest
      // index on ties (C12)
      if ((c.kind == 0 || c.kind == 1 || c.kind == 5) && c.good > bg) {
        bg = c.good;
        bi = (int64_t)i;
      }
    }
    if (s->bound) {
      bool left = false;
      for (size_t i = 0; i < run.cands.size(); ++i) {
        Run::Cand& c = run.cands[i];
        if (c.kind != 3) continue;
        if (c.ub < bg || (c.ub == bg && (int64_t)i > bi)) c.kind = 4;  // cannot be the argmax
        else left = true;
      }
      if (left) {  // another round of this step: the deferred candidates that may still win
        for (Run::Cand& c : run.cands)
          if (c.kind == 0) c.kind = 5;
        run.round = 1;
        pending.push_back(s->base_run[b]);
        continue;
      }
    }
    for (Run::Cand& c : run.cands) {
      if (c.kind == 4) ++s->bounded;
      if (c.kind != 2) continue;
      const Run::Cand& rep = run.cands[c.ref];
      if (rep.kind == 4) c.kind = 4;  // no value: its representative was bounded out
      else c.good = rep.good;
    }
    if (bi < 0) return sfail(s, ASIM_ERANGE, "step results contain no feasible candidate");
    winner_run.push_back(s->base_run[b]);
    winner.push_back(&run.cands[bi]);
  }
  if (s->use_states) {
    // candidate memory: every locally simulated candidate's boundary states
    const size_t per = (size_t)s->J * s->stride * 8;
    const bool keep = s->eval_hi > s->eval_lo && (size_t)C * per <= kMixBytesCap;
    if (keep) {
      cudaError_t e = s->cs_cur.ensure((size_t)C * per + 8);
      if (e != cudaSuccess) return asim_cuda(s->ctx, e, "candidate memory");
      std::vector<int64_t> cs;
      std::vector<int32_t> rows;
      for (int64_t c = s->eval_lo; c < s->eval_hi; ++c) {
        cs.push_back(c);
        rows.push_back((int32_t)c);
      }
      asim_status rc = asim_publish_candidates(s->ctx, cs, rows, s->cs_cur.as<int64_t>(), st);
      if (rc) return rc;
    }
    for (size_t b = 0; b < s->base_run.size(); ++b) {
      Run& run = s->runs[s->base_run[b]];
      std::fill(run.cur_idx.begin(), run.cur_idx.end(), -1);
      if (keep)
        for (const Run::Cand& c : run.cands)
          if (c.kind == 0 && c.ref >= s->eval_lo && c.ref < s->eval_hi)
            run.cur_idx[(size_t)c.m * run.G + c.g] = (int32_t)c.ref;
      std::swap(run.prev_idx, run.cur_idx);
    }
    if (keep) std::swap(s->cs_prev, s->cs_cur);
    s->have_prev = keep;
    // before the bases change: the update simulates from the old ones
    asim_status rc = update_states(s, winner_run, winner, st, nullptr, &pending);
    if (rc) return rc;
  }
  for (size_t i = 0; i < winner_run.size(); ++i) {
    Run& run = s->runs[winner_run[i]];
    const Run::Cand w = *winner[i];
    apply_winner(run, w, hp);
    if (w.good > run.best_good) {  // "if sel*.slo_att > best_sel.slo_att"
      run.best_good = w.good;
      run.best = run.sel;
    }
  }
  s->prepared = false;
  return ASIM_OK;
}

}  // extern "C"

// The fast heuristic (readings C22-C24): one simulation of every active
// run's current selection per step, then a host decision per run.
static asim_status run_fast(asim_search* s, cudaStream_t st) {
  // Per run: per-model good (fpm) and per-group busy (fbusy) of the current
  // selection.  They only change inside the connected component of the
  // (group, model) hosting graph that the last addition merged, so each step
  // simulates that component alone (its models' requests; exact, as in the
  // greedy driver's component restriction) and keeps the other values.  The
  // empty selection serves nothing: the first decision needs no simulation.
  asim_ctx* ctx = s->ctx;
  const HostProblem& hp = ctx->hp;
  const int32_t M = hp.M, G = s->G;
  const bool restrict_ok = M <= 64;
  std::vector<int64_t> good, pm, busy;
  for (auto& run : s->runs) {
    run.fpm.assign(M, 0);
    run.fbusy.assign(run.G, 0);
    run.pending = -1;
  }
  for (;;) {
    asim_status rs = asim_ready(ctx);
    if (rs) return rs;
    HostBatch hb;
    hb.G = G;
    prune_runs(s);
    std::vector<int32_t> act, sim_b;
    for (int32_t r = 0; r < (int32_t)s->runs.size(); ++r) {
      Run& run = s->runs[r];
      if (!run.active) continue;
      act.push_back(r);
      if (run.pending < 0) continue;  // nothing changed since its last simulation
      const int32_t b = (int32_t)sim_b.size();
      sim_b.push_back(r);
      for (int32_t g = 0; g < G; ++g) hb.base_cfg.push_back(g < run.G ? run.cfg[g] : -1);
      hb.base_mask.insert(hb.base_mask.end(), run.sel.begin(), run.sel.end());
      hb.cand_base.push_back(b);
      hb.cand_model.push_back(-1);  // the selection itself
      hb.cand_group.push_back(0);
      hb.cand_ok.push_back(1);
      if (restrict_ok) {
        uint64_t km = 0, gm = 0;
        for (int32_t x = 0; x < run.G; ++x)
          if (run.find(x) == run.pending) gm |= 1ULL << x;
        for (int32_t x = 0; x < M; ++x)
          if (run.find(run.G + x) == run.pending) km |= 1ULL << x;
        hb.cand_kmask.push_back(km);
        hb.cand_gmask.push_back(gm);
      }
      int32_t slots = 0;
      for (int32_t c : run.cfg) slots += hp.cfg_stages[c];
      hb.slots = std::max(hb.slots, slots);
    }
    if (act.empty()) {
      s->finished = true;
      return ASIM_OK;
    }
    const int64_t C = (int64_t)sim_b.size();
    if (C > 0) {
      cudaError_t e = s->d_good_all.ensure(C * 8 + 8);
      if (e == cudaSuccess) e = s->d_pm.ensure(C * M * 8 + 8);
      if (e == cudaSuccess) e = s->d_busy.ensure(C * G * 8 + 8);
      if (e == cudaSuccess) e = cudaMemsetAsync(s->d_pm.p, 0, C * M * 8, st);
      if (e == cudaSuccess) e = cudaMemsetAsync(s->d_busy.p, 0, C * G * 8, st);
      if (e != cudaSuccess) return asim_cuda(ctx, e, "fast heuristic buffers");
      asim::DevOut out{};
      out.good = s->d_good_all.as<int64_t>();
      out.good_per_model = s->d_pm.as<int64_t>();
      out.busy = s->d_busy.as<int64_t>();
      // chunked kernels speculating from the run's previous boundary states
      // (component restricted); else the warp-cooperative whole-trace kernel
      // (uniform configs); else the general kernel over every model
      asim_status rc = asim_upload_batch(ctx, hb, st);
      if (rc) return rc;
      bool done = false;
      if (s->use_states) {
        e = upload(s->d_rows, sim_b, st);
        if (e != cudaSuccess) return asim_cuda(ctx, e, "upload rows");
        ChunkOptions opt;
        opt.J = s->J;
        opt.state_stride = s->stride;
        opt.spec_state = s->st_base.as<int64_t>();
        opt.spec_row = s->d_rows.as<int32_t>();
        asim::DevOut o2 = out;
        o2.stage_updates = ctx->profiling ? ctx->d_counter.as<unsigned long long>() : nullptr;
        cudaEvent_t ev0 = nullptr, ev1 = nullptr;
        if (ctx->profiling) {
          if (cudaEventCreate(&ev0) != cudaSuccess || cudaEventCreate(&ev1) != cudaSuccess)
            return asim_cuda(ctx, cudaGetLastError(), "event create");
          cudaEventRecord(ev0, st);
        }
        rc = asim_run_chunked(ctx, hb, 0, C, o2, st, &opt);
        if (rc) return rc;
        if (ctx->profiling) {
          cudaEventRecord(ev1, st);
          ctx->events.emplace_back(ev0, ev1);
          ++ctx->sim_launches;
          ctx->request_evals += C * ctx->n;
        }
        // the new selections' boundary states replace the old ones in place
        std::vector<int64_t> cs(C);
        for (int64_t b = 0; b < C; ++b) cs[b] = b;
        rc = asim_publish_candidates(ctx, cs, sim_b, s->st_base.as<int64_t>(), st);
        if (rc) return rc;
        done = true;
      }
      if (!done && ctx->force_path != 1) {
        rc = asim_run_fast_stats(ctx, hb, out, st, &done);
        if (rc) return rc;
      }
      if (!done) {
        hb.cand_kmask.clear();
        hb.cand_gmask.clear();
        rc = asim_run_batch(ctx, hb, 0, C, out, st);
        if (rc) return rc;
      }
      pm.resize(C * M);
      busy.resize(C * G);
      e = cudaMemcpyAsync(pm.data(), out.good_per_model, C * M * 8, cudaMemcpyDeviceToHost, st);
      if (e == cudaSuccess)
        e = cudaMemcpyAsync(busy.data(), out.busy, C * G * 8, cudaMemcpyDeviceToHost, st);
      if (e == cudaSuccess) e = cudaStreamSynchronize(st);
      if (e != cudaSuccess) return asim_cuda(ctx, e, "copy fast heuristic results");
      for (int64_t b = 0; b < C; ++b) {
        Run& run = s->runs[sim_b[b]];
        const bool part = done && restrict_ok;
        for (int32_t m = 0; m < M; ++m)
          if (!part || ((hb.cand_kmask[b] >> m) & 1ULL)) run.fpm[m] = pm[b * M + m];
        for (int32_t g = 0; g < run.G; ++g)
          if (!part || ((hb.cand_gmask[b] >> g) & 1ULL)) run.fbusy[g] = busy[b * G + g];
        run.pending = -1;
      }
    }
    ++s->steps;
    s->candidates += (int64_t)act.size();
    s->evaluated += C;
    for (int32_t r : act) {
      Run& run = s->runs[r];
      int64_t g_total = 0;
      for (int32_t m = 0; m < M; ++m) g_total += run.fpm[m];
      run.base_good = g_total;
      if (!run.history_good.empty() && run.history_good.back() < 0) run.history_good.back() = g_total;
      if (g_total > run.best_good) {  // best selection so far, strict '>' (C24)
        run.best_good = g_total;
        run.best = run.sel;
      }
      // C22: the model with the most unserved requests among those with an
      // available group; C23: its available group with the lowest mean stage
      // utilization busy_g / s_g (the common horizon cancels)
      int32_t bm = -1, bgp = -1;
      int64_t bu = 0;
      for (int32_t m = 0; m < M; ++m) {
        if (!run.may_place(m)) continue;  // outside this run's bucket
        const int64_t un = ctx->model_n[m] - run.fpm[m];
        if (un <= 0 || (bm >= 0 && un <= bu)) continue;
        int32_t gbest = -1;
        for (int32_t g = 0; g < run.G; ++g) {
          if ((run.sel[m] >> g) & 1ULL) continue;  // a model at most once per group (C11)
          const int64_t mb = hp.mem_at(m, run.cfg[g]);
          if (mb < 0 || run.used[g] + mb > hp.budget) continue;  // memory constraint
          if (gbest < 0 || (__int128)run.fbusy[g] * hp.cfg_stages[run.cfg[gbest]] <
                               (__int128)run.fbusy[gbest] * hp.cfg_stages[run.cfg[g]])
            gbest = g;
        }
        if (gbest < 0) continue;
        bm = m;
        bgp = gbest;
        bu = un;
      }
      if (bm < 0) {  // every request served, or no available pair: this run ends
        run.active = false;
        continue;
      }
      run.sel[bm] |= 1ULL << bgp;
      run.used[bgp] += hp.mem_at(bm, run.cfg[bgp]);
      run.history.emplace_back(bm, bgp);
      run.history_good.push_back(-1);  // known after the next simulation
      ++run.steps;
      const int32_t a = run.find(bgp), c = run.find(run.G + bm);
      if (a != c) run.parent[a] = c;  // unite comp(g*) and comp(m*)
      run.pending = c;
    }
  }
}

extern "C" {

asim_status asim_search_run(asim_search* s, void* cuda_stream) {
  if (!s) return ASIM_EINVAL;
  if (s->fast) return run_fast(s, static_cast<cudaStream_t>(cuda_stream));
  for (;;) {
    int64_t C = 0;
    asim_status st = asim_search_prepare(s, &C);
    if (st) return st;
    if (C < 0) return ASIM_OK;
    if (C > 0) {
      cudaError_t e = s->d_good_all.ensure(C * 8 + 8);
      if (e != cudaSuccess) return asim_cuda(s->ctx, e, "allocate step results");
      st = asim_search_evaluate(s, 0, C, s->d_good_all.as<int64_t>(), cuda_stream);
      if (st) return st;
    }
    st = asim_search_apply(s, C > 0 ? s->d_good_all.as<int64_t>() : nullptr, cuda_stream);
    if (st) return st;
  }
}

}  // extern "C"

// Outcome of run group gi (one Alg. 2 run; its beam members for beam > 1).
static void group_best(const asim_search* s, int32_t gi, int64_t* good,
                       const std::vector<uint64_t>** mask, int64_t* steps) {
  if (s->beam == 1) {
    const Run& r = s->runs[gi];
    *good = r.best_good;
    *mask = &r.best;
    *steps = r.steps;
  } else {
    *good = s->gbest_good[gi];
    *mask = &s->gbest[gi];
    *steps = s->gsteps[gi];
  }
}
static const Run& group_run(const asim_search* s, int32_t gi) { return s->runs[gi * s->beam]; }

// Capacity bound on the good of ANY selection on a run's groups (exact run
// pruning; not in the paper, results unchanged).  An accepted request of
// model m on a group with config p occupies stage k of that group for
// d_k(m, p), inside [first arrival, last arrival + max SLO] (it starts after
// its arrival and its last stage ends before its deadline).  Summing the
// per-stage constraints of a group and dividing by its stage count s:
//   sum over accepted requests of c(m, p) <= H,  c(m, p) = sum_k d_k(m, p) / s,
// so over the run's G groups sum_m x_m * min_p c(m, p) <= G * H with
// 0 <= x_m <= n_m (requests of m in the trace; models that fit on none of the
// groups, or lie outside the run's bucket, have x_m = 0).  The floor of the
// fractional-knapsack optimum (cheapest models first) bounds sum_m x_m; the
// costs are rounded down, which only loosens it.
static int64_t run_capacity_bound(const asim_ctx* ctx, const Run& run) {
  const HostProblem& hp = ctx->hp;
  if (ctx->n == 0) return 0;
  int64_t slo_max = 0;
  std::vector<std::pair<int64_t, int32_t>> cost;  // (cost, model)
  int64_t free_requests = 0;                      // models of cost 0: no capacity limit
  for (int32_t m = 0; m < hp.M; ++m) {
    if (!run.may_place(m) || ctx->model_n[m] == 0) continue;
    int64_t c = -1;
    for (int32_t p : run.cfg) {
      const int64_t mb = hp.mem_at(m, p);
      if (mb < 0 || mb > hp.budget) continue;
      const int32_t st = hp.cfg_stages[p];
      __int128 sum = 0;
      for (int32_t k = 0; k < st; ++k) sum += hp.stage[((int64_t)m * hp.P + p) * hp.S + k];
      const int64_t ck = (int64_t)(sum / st);
      c = c < 0 ? ck : std::min(c, ck);
    }
    if (c < 0) continue;  // fits on none of the run's groups
    slo_max = std::max(slo_max, hp.slo[m]);
    if (c == 0) free_requests += ctx->model_n[m];
    else cost.emplace_back(c, m);
  }
  std::sort(cost.begin(), cost.end());
  const __int128 H = (__int128)ctx->max_arrival - ctx->min_arrival + slo_max;
  __int128 cap = (__int128)run.G * H;
  __int128 ub = free_requests;
  for (const auto& cm : cost) {
    const __int128 take = std::min<__int128>(ctx->model_n[cm.second], cap / cm.first);
    ub += take;
    cap -= take * cm.first;
    if (take < ctx->model_n[cm.second]) break;
  }
  return (int64_t)std::min<__int128>(ub, ctx->n);
}

static void group_best(const asim_search* s, int32_t gi, int64_t* good,
                       const std::vector<uint64_t>** mask, int64_t* steps);

// Stop every run group whose capacity bound is below the best good another
// group of its competition (all runs, or its bucket job) already reached: it
// can never become the (first) best, so the search's result is unchanged.
static void prune_runs(asim_search* s) {
  if (!s->prune) return;
  auto sweep = [&](const std::vector<int32_t>& grp) {
    int64_t lb = 0;
    for (int32_t gi : grp) {
      int64_t g = 0, st = 0;
      const std::vector<uint64_t>* mk = nullptr;
      group_best(s, gi, &g, &mk, &st);
      lb = std::max(lb, g);
    }
    for (int32_t gi : grp) {
      if (s->gpruned[gi] >= 0 || s->gub[gi] >= lb) continue;
      bool any = false;
      for (int32_t k = 0; k < s->beam; ++k) {
        Run& r = s->runs[(size_t)gi * s->beam + k];
        any |= r.active;
        r.active = false;
      }
      if (any) s->gpruned[gi] = s->steps;
    }
  };
  if (s->bucketed) {
    for (const auto& job : s->jobs) sweep(job.runs);
  } else {
    std::vector<int32_t> all(s->ngroups);
    for (int32_t i = 0; i < s->ngroups; ++i) all[i] = i;
    sweep(all);
  }
}

// Bucketed outcome (reading C28): plm_i* per job = its first best run on
// strict '>' (none if no run serves a request); combo good = sum over its
// jobs; the first best combo on strict '>'.
static void bucket_best(const asim_search* s, int32_t* best_combo, int64_t* best_good,
                        std::vector<int32_t>* job_run) {
  job_run->assign(s->jobs.size(), -1);
  std::vector<int64_t> job_good(s->jobs.size(), 0);
  for (size_t j = 0; j < s->jobs.size(); ++j)
    for (int32_t r : s->jobs[j].runs) {
      int64_t g = 0, st = 0;
      const std::vector<uint64_t>* mk = nullptr;
      group_best(s, r, &g, &mk, &st);
      if (g > job_good[j]) {
        job_good[j] = g;
        (*job_run)[j] = r;
      }
    }
  *best_combo = -1;
  *best_good = 0;
  for (size_t c = 0; c < s->combos.size(); ++c) {
    int64_t g = 0;
    for (int32_t j : s->combos[c].jobs) g += job_good[j];
    if (g > *best_good) {
      *best_good = g;
      *best_combo = (int32_t)c;
    }
  }
}

extern "C" {

asim_status asim_search_result_get(const asim_search* s, asim_search_result* out) {
  if (!s || !out) return ASIM_EINVAL;
  const int32_t M = s->ctx->hp.M;
  out->steps = s->steps;
  out->candidates = s->candidates;
  out->evaluated = s->evaluated;
  out->request_evals = s->evaluated * s->ctx->n;
  out->memo_hits = s->memo_hits;
  out->bounded = s->bounded;
  if (s->bucketed) {  // the concatenated placement (groups of bucket 1 first)
    int32_t bc = -1;
    int64_t bg = 0;
    std::vector<int32_t> job_run;
    bucket_best(s, &bc, &bg, &job_run);
    std::vector<int32_t> cfg;
    std::vector<uint64_t> mask(M, 0);
    if (bc >= 0)
      for (int32_t j : s->combos[bc].jobs) {
        const int32_t r = job_run[j];
        if (r < 0) continue;
        const Run& run = group_run(s, r);
        int64_t g = 0, st = 0;
        const std::vector<uint64_t>* mk = nullptr;
        group_best(s, r, &g, &mk, &st);
        const int32_t off = (int32_t)cfg.size();
        for (int32_t m = 0; m < M; ++m)
          if (off < 64) mask[m] |= (*mk)[m] << off;
        cfg.insert(cfg.end(), run.cfg.begin(), run.cfg.end());
      }
    const bool fits = (int32_t)cfg.size() <= ASIM_MAX_GROUPS;
    out->best_run = -1;
    out->best_good = bg;
    out->num_groups = (int32_t)cfg.size();
    if (out->group_cfg)
      for (int32_t g = 0; g < ASIM_MAX_GROUPS; ++g)
        out->group_cfg[g] = (fits && g < (int32_t)cfg.size()) ? cfg[g] : -1;
    if (out->host_mask)
      for (int32_t m = 0; m < M; ++m) out->host_mask[m] = fits ? mask[m] : 0;
    return ASIM_OK;
  }
  int32_t best = -1;
  int64_t best_good = 0;
  const std::vector<uint64_t>* best_mask = nullptr;
  for (int32_t r = 0; r < s->ngroups; ++r) {
    int64_t g = 0, st = 0;
    const std::vector<uint64_t>* mk = nullptr;
    group_best(s, r, &g, &mk, &st);
    if (g > best_good) {  // Alg. 2: strict '>' keeps the first best run
      best_good = g;
      best = r;
      best_mask = mk;
    }
  }
  out->best_run = best;
  out->best_good = best_good;
  out->num_groups = best >= 0 ? group_run(s, best).G : 0;
  if (out->group_cfg) {
    for (int32_t g = 0; g < ASIM_MAX_GROUPS; ++g)
      out->group_cfg[g] = (best >= 0 && g < group_run(s, best).G) ? group_run(s, best).cfg[g] : -1;
  }
  if (out->host_mask)
    for (int32_t m = 0; m < M; ++m) out->host_mask[m] = best >= 0 ? (*best_mask)[m] : 0;
  return ASIM_OK;
}

int64_t asim_search_run_pruned(const asim_search* s, int32_t run) {
  if (!s || run < 0 || run >= (int32_t)s->gpruned.size()) return -1;
  return s->gpruned[run];
}

asim_status asim_search_buckets_get(const asim_search* s, asim_bucket_result* out) {
  if (!s || !out) return ASIM_EINVAL;
  if (!s->bucketed) return asim_fail(s->ctx, ASIM_ESTATE, "not a bucketed search");
  if (!s->finished) return asim_fail(s->ctx, ASIM_ESTATE, "search not finished");
  const int32_t M = s->ctx->hp.M;
  int32_t bc = -1;
  int64_t bg = 0;
  std::vector<int32_t> job_run;
  bucket_best(s, &bc, &bg, &job_run);
  out->best_good = bg;
  out->partitions = (int64_t)s->partitions.size();
  out->considered = (int64_t)s->combos.size();
  out->num_buckets = bc >= 0 ? (int32_t)s->combos[bc].jobs.size() : 0;
  if (out->bucket_of_model)
    for (int32_t m = 0; m < M; ++m) out->bucket_of_model[m] = -1;
  for (int32_t i = 0; i < out->num_buckets; ++i) {
    const int32_t j = s->combos[bc].jobs[i];
    if (out->bucket_of_model)
      for (int32_t m : s->jobs[j].models) out->bucket_of_model[m] = i;
    if (out->bucket_devices) out->bucket_devices[i] = s->combos[bc].H[i];
    if (out->bucket_run) out->bucket_run[i] = job_run[j];
  }
  return ASIM_OK;
}

asim_status asim_search_run_history(const asim_search* s, int32_t run, int64_t cap,
                                    int32_t* model, int32_t* group, int64_t* good,
                                    int64_t* count) {
  if (!s || !count || run < 0 || run >= s->ngroups || cap < 0) return ASIM_EINVAL;
  const Run& r = group_run(s, run);
  const int64_t n = (int64_t)r.history.size();
  *count = n;
  for (int64_t i = 0; i < n && i < cap; ++i) {
    if (model) model[i] = r.history[i].first;
    if (group) group[i] = r.history[i].second;
    if (good) good[i] = r.history_good[i];
  }
  return ASIM_OK;
}

asim_status asim_search_run_candidates(const asim_search* s, int32_t run, int64_t cap,
                                       int32_t* model, int32_t* group, int64_t* good,
                                       int64_t* count) {
  if (!s || !count || run < 0 || run >= s->ngroups || cap < 0) return ASIM_EINVAL;
  if (s->prepared) return asim_fail(s->ctx, ASIM_ESTATE, "candidates are read between steps");
  const Run& r = group_run(s, run);
  const int64_t n = (int64_t)r.cands.size();
  *count = n;
  for (int64_t i = 0; i < n && i < cap; ++i) {
    const Run::Cand& c = r.cands[i];
    if (model) model[i] = c.m;
    if (group) group[i] = c.g;
    // bounded out (spec->cand_bound): no value, provably not the argmax
    if (good) good[i] = c.kind == 4 ? INT64_MIN : c.good;
  }
  return ASIM_OK;
}

asim_status asim_search_run_info(const asim_search* s, int32_t run, int32_t* num_groups,
                                 int32_t* group_cfg, uint64_t* host_mask, int64_t* best_good,
                                 int64_t* steps) {
  if (!s || run < 0 || run >= s->ngroups) return ASIM_EINVAL;
  const Run& r = group_run(s, run);
  int64_t g = 0, st = 0;
  const std::vector<uint64_t>* mk = nullptr;
  group_best(s, run, &g, &mk, &st);
  if (num_groups) *num_groups = r.G;
  if (group_cfg)
    for (int32_t k = 0; k < r.G; ++k) group_cfg[k] = r.cfg[k];
  if (host_mask)
    for (int32_t m = 0; m < s->ctx->hp.M; ++m) host_mask[m] = (*mk)[m];
  if (best_good) *best_good = g;
  if (steps) *steps = st;
  return ASIM_OK;
}

}  // extern "C"
