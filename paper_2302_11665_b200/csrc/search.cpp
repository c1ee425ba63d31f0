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
//   evaluate  the simulation kernel on a contiguous shard of the step's list.
//   apply     a7: per run, argmax (ties -> lowest index, "pick_highest",
//             P:722) and sel <- sel + (m*, g*); best_sel on strict '>'.
//
// Exact component memo (always on): a placement's simulation splits into
// independent connected components of the bipartite (group, model) hosting
// graph -- a request is only ever dispatched among its model's hosts, and a
// group's stages only see requests of the models it hosts.  Candidate (m, g)
// of step t whose component K = comp(g) u comp(m) u {m} in base(t-1) is
// disjoint from the two components the step-(t-1) winner (m*, g*) merged has
// good_t(m, g) = good_{t-1}(m, g) + good(base(t)) - good(base(t-1)) exactly,
// so only the other candidates are simulated.
//
// Exact de-duplication (spec->dedup): adding model m to either of two EMPTY
// groups g1 < g2 with the same config gives the same simulation whenever g1
// and g2 sit between the same pair of m's hosting groups in index order
// (relabelling g1 <-> g2 maps one simulation onto the other and preserves
// every dispatch tie-break, reading C1).  Only the lowest such g -- the one
// the argmax would pick on a tie anyway -- is listed.
#include <cuda_runtime.h>

#include <algorithm>
#include <map>
#include <new>
#include <string>
#include <vector>

#include "ctx.h"

namespace {

struct Run {
  int32_t G = 0;
  std::vector<int32_t> cfg;
  std::vector<uint64_t> sel;   // [M] current selection
  std::vector<int64_t> used;   // [G] bytes per device
  std::vector<uint64_t> best;  // [M] best selection so far
  int64_t best_good = 0;
  bool active = true;
  int64_t steps = 0;
  int64_t base_good = 0;  // good of the current selection (the last winner)
  // this step's full candidate list, in (m, g) order
  struct Cand {
    int32_t m, g;
    int8_t kind;    // 0 simulated (ref = batch index), 1 memo (value), 2 duplicate (ref = rep)
    int64_t ref;
    int64_t good;
  };
  std::vector<Cand> cands;
  // memo carried to the next step: (m, g) -> good, valid when the winner is elsewhere
  std::map<std::pair<int32_t, int32_t>, int64_t> memo;
  std::vector<std::pair<int32_t, int32_t>> history;  // winners in order
};

// union-find over G groups + M models (node G + m) of one selection
struct Components {
  std::vector<int32_t> p;
  Components(int32_t G, int32_t M, const std::vector<uint64_t>& sel) : p(G + M) {
    for (size_t i = 0; i < p.size(); ++i) p[i] = (int32_t)i;
    for (int32_t m = 0; m < M; ++m)
      for (int32_t g = 0; g < G; ++g)
        if ((sel[m] >> g) & 1ULL) unite(g, G + m);
  }
  int32_t find(int32_t x) {
    while (p[x] != x) x = p[x] = p[p[x]];
    return x;
  }
  void unite(int32_t a, int32_t b) { p[find(a)] = find(b); }
};

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
  std::vector<int64_t> seg;       // [bases + 1] candidate offsets per base
  DBuf d_good_all;
  std::vector<int64_t> h_good;
  // Speculation from the base placement's true trajectory (chunk.cu): per run
  // the absolute free times at every chunk boundary of the current base.
  bool use_states = false;
  int64_t J = 1;
  int32_t stride = 1;       // slots per boundary row
  DBuf state_prev, state_cur, d_rows, d_base_good;
  bool base_ready = false;
  HostBatch hb_base;        // one candidate per base: the base itself
  // Component restriction: simulated candidates only replay their own
  // component; good = good(base) - good_base(K_c) + good_c(K_c).
  bool restrict_k = false;
  DBuf d_base_pm;                // [B][M] per-model good of every base (base pass)
  std::vector<int64_t> h_base_pm;
  // statistics
  int64_t steps = 0, candidates = 0, evaluated = 0, memo_hits = 0;
  bool finished = false;
};

static asim_status sfail(asim_search* s, asim_status code, const std::string& m) {
  return asim_fail(s ? s->ctx : nullptr, code, m);
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
  if (spec->num_runs == 0) {
    // Alg. 2 single bucket: D/size equal groups, one config each (C13)
    for (int32_t size = 1; size <= hp.num_devices; ++size) {
      if (hp.num_devices % size) continue;
      for (int32_t p = 0; p < hp.P; ++p) {
        if (hp.cfg_devices[p] != size) continue;
        const int32_t G = hp.num_devices / size;
        if (G > ASIM_MAX_GROUPS)
          return asim_fail(ctx, ASIM_ERANGE,
                           "Alg. 2 run with more than ASIM_MAX_GROUPS groups; pass explicit runs");
        groups.emplace_back(G, p);
      }
    }
  } else {
    if (spec->num_runs < 0 || !spec->run_num_groups || !spec->run_group_cfg)
      return asim_fail(ctx, ASIM_EINVAL, "bad run list");
    int64_t off = 0;
    for (int32_t r = 0; r < spec->num_runs; ++r) {
      const int32_t G = spec->run_num_groups[r];
      if (G < 1 || G > ASIM_MAX_GROUPS) return asim_fail(ctx, ASIM_ERANGE, "run_num_groups");
      std::vector<int32_t> cfg(spec->run_group_cfg + off, spec->run_group_cfg + off + G);
      off += G;
      int32_t slots = 0;
      for (int32_t c : cfg) {
        if (c < 0 || c >= hp.P) return asim_fail(ctx, ASIM_ERANGE, "run_group_cfg");
        slots += hp.cfg_stages[c];
      }
      if (slots > ASIM_MAX_SLOTS) return asim_fail(ctx, ASIM_ERANGE, "run exceeds ASIM_MAX_SLOTS");
      groups.push_back(std::move(cfg));
    }
  }
  asim_search* s = new (std::nothrow) asim_search();
  if (!s) return asim_fail(ctx, ASIM_ENOMEM, "host allocation failed");
  s->ctx = ctx;
  s->dedup = spec->dedup != 0;
  for (auto& cfg : groups) {
    Run r;
    r.G = (int32_t)cfg.size();
    r.cfg = cfg;
    r.sel.assign(hp.M, 0);
    r.best.assign(hp.M, 0);
    r.used.assign(r.G, 0);
    int64_t devices = 0;
    for (int32_t c : cfg) devices += hp.cfg_devices[c];
    if (devices > hp.num_devices) r.active = false;  // the empty placement is already infeasible
    s->G = std::max(s->G, r.G);
    s->runs.push_back(std::move(r));
  }
  // one chunking for the whole search; rows of idle boundary states per run
  int32_t stride = 1;
  for (auto& cfg : groups) {
    int32_t sl = 0;
    for (int32_t c : cfg) sl += hp.cfg_stages[c];
    stride = std::max(stride, sl);
  }
  s->stride = stride;
  s->J = std::max<int64_t>(1, std::min<int64_t>(1024, ctx->n / std::max<int64_t>(1, ctx->min_chunk)));
  s->use_states = ctx->force_path != 1;  // the general kernel has no time chunks
  {
    HostBatch probe_hb;
    probe_hb.slots = stride;
    asim::DevOut probe{};
    s->restrict_k = s->use_states && hp.M <= 64 && asim_chunked_eligible(ctx, probe_hb, probe);
  }
  if (s->use_states && !s->runs.empty()) {
    const size_t bytes = s->runs.size() * (size_t)s->J * stride * 8;
    cudaError_t e = s->state_prev.ensure(bytes);
    if (e == cudaSuccess) e = s->state_cur.ensure(bytes);
    if (e == cudaSuccess) e = cudaMemset(s->state_prev.p, 0, bytes);
    if (e == cudaSuccess) e = cudaMemset(s->state_cur.p, 0, bytes);
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
  s->d_good_all.release();
  s->d_base_pm.release();
  s->state_prev.release();
  s->state_cur.release();
  s->d_rows.release();
  s->d_base_good.release();
  delete s;
}

int32_t asim_search_num_runs(const asim_search* s) { return s ? (int32_t)s->runs.size() : 0; }

asim_status asim_search_prepare(asim_search* s, int64_t* num_candidates) {
  if (!s || !num_candidates) return ASIM_EINVAL;
  asim_status st = asim_ready(s->ctx);
  if (st) return st;
  if (s->prepared) return sfail(s, ASIM_ESTATE, "prepare called twice without apply");
  const HostProblem& hp = s->ctx->hp;
  const int32_t M = hp.M, G = s->G;
  HostBatch& hb = s->hb;
  hb = HostBatch();
  hb.G = G;
  s->base_run.clear();
  s->seg.assign(1, 0);
  int64_t full = 0;
  for (int32_t r = 0; r < (int32_t)s->runs.size(); ++r) {
    Run& run = s->runs[r];
    if (!run.active) continue;
    const int32_t b = (int32_t)s->base_run.size();
    std::vector<uint8_t> empty(run.G, 1);
    for (int32_t m = 0; m < M; ++m)
      for (int32_t g = 0; g < run.G; ++g)
        if ((run.sel[m] >> g) & 1ULL) empty[g] = 0;
    run.cands.clear();
    // components of the base: models / groups per root (restriction masks)
    std::vector<uint64_t> rootK, rootG;
    Components comp(run.G, M, run.sel);
    if (s->restrict_k) {
      rootK.assign(run.G + M, 0);
      rootG.assign(run.G + M, 0);
      for (int32_t g = 0; g < run.G; ++g) rootG[comp.find(g)] |= 1ULL << g;
      for (int32_t m = 0; m < M; ++m) rootK[comp.find(run.G + m)] |= 1ULL << m;
    }
    for (int32_t m = 0; m < M; ++m) {
      std::map<std::pair<int32_t, int32_t>, int64_t> seen;  // (cfg, rank among hosts) -> rep
      for (int32_t g = 0; g < run.G; ++g) {
        if ((run.sel[m] >> g) & 1ULL) continue;  // a model at most once per group (C11)
        const int64_t mb = hp.mem_at(m, run.cfg[g]);
        if (mb < 0 || run.used[g] + mb > hp.budget) continue;  // memory constraint
        ++full;
        Run::Cand c{m, g, 0, 0, 0};
        auto it = run.memo.find(std::make_pair(m, g));
        if (it != run.memo.end()) {  // component untouched by the last winner
          c.kind = 1;
          c.good = it->second;
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
        if (c.kind == 0) {
          c.ref = (int64_t)hb.cand_base.size();
          hb.cand_base.push_back(b);
          hb.cand_model.push_back(m);
          hb.cand_group.push_back(g);
          hb.cand_ok.push_back(1);
          if (s->restrict_k) {  // K_c = comp(g) u comp(m) in the base, plus m
            const int32_t r1 = comp.find(g), r2 = comp.find(run.G + m);
            hb.cand_kmask.push_back(rootK[r1] | rootK[r2] | (1ULL << m));
            hb.cand_gmask.push_back(rootG[r1] | rootG[r2] | (1ULL << g));
          }
        }
        run.cands.push_back(c);
      }
    }
    if (run.cands.empty()) {  // no feasible addition: this run's Alg. 1 loop ends
      run.active = false;
      continue;
    }
    s->base_run.push_back(r);
    for (int32_t g = 0; g < G; ++g) hb.base_cfg.push_back(g < run.G ? run.cfg[g] : -1);
    hb.base_mask.insert(hb.base_mask.end(), run.sel.begin(), run.sel.end());
    int32_t slots = 0;
    for (int32_t c : run.cfg) slots += hp.cfg_stages[c];
    hb.slots = std::max(hb.slots, slots);
    s->seg.push_back((int64_t)hb.cand_base.size());
  }
  // the bases themselves (true boundary states for speculation)
  s->base_ready = false;
  s->hb_base = HostBatch();
  s->hb_base.G = G;
  s->hb_base.base_cfg = hb.base_cfg;
  s->hb_base.base_mask = hb.base_mask;
  s->hb_base.slots = hb.slots;
  for (int32_t b = 0; b < (int32_t)s->base_run.size(); ++b) {
    s->hb_base.cand_base.push_back(b);
    s->hb_base.cand_model.push_back(-1);
    s->hb_base.cand_group.push_back(0);
    s->hb_base.cand_ok.push_back(1);
  }
  if (s->base_run.empty()) {  // every run has ended: the search is finished
    s->finished = true;
    s->prepared = false;
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
  asim::DevOut probe{};
  if (s->use_states && asim_chunked_eligible(s->ctx, s->hb, probe)) {
    const int32_t B = (int32_t)s->base_run.size();
    opt.J = s->J;
    opt.state_stride = s->stride;
    if (!s->base_ready) {
      // true boundary states of every base: simulate each base (one lane)
      // speculating from the previous base's states, publish into state_cur
      cudaError_t e = upload(s->d_rows, s->base_run, strm);
      if (e == cudaSuccess) e = s->d_base_good.ensure(B * 8 + 8);
      if (e != cudaSuccess) {
        if (prev >= 0 && prev != s->ctx->device) cudaSetDevice(prev);
        return asim_cuda(s->ctx, e, "base pass buffers");
      }
      if (s->restrict_k) {
        e = s->d_base_pm.ensure((size_t)B * s->ctx->hp.M * 8 + 8);
        if (e != cudaSuccess) {
          if (prev >= 0 && prev != s->ctx->device) cudaSetDevice(prev);
          return asim_cuda(s->ctx, e, "base per-model buffer");
        }
      }
      ChunkOptions ob = opt;
      ob.pm_out = s->restrict_k ? s->d_base_pm.as<int64_t>() : nullptr;
      ob.spec_state = s->state_prev.as<int64_t>();
      ob.spec_row = s->d_rows.as<int32_t>();
      ob.publish_out = s->state_cur.as<int64_t>();
      ob.publish_row = s->d_rows.as<int32_t>();
      asim::DevOut bo{};
      bo.good = s->d_base_good.as<int64_t>();
      bo.out_offset = 0;
      st = asim_upload_batch(s->ctx, s->hb_base, strm);
      if (!st) st = asim_run_chunked(s->ctx, s->hb_base, 0, B, bo, strm, &ob);
      if (st) {
        if (prev >= 0 && prev != s->ctx->device) cudaSetDevice(prev);
        return st;
      }
      s->base_ready = true;
    }
    opt.spec_state = s->state_cur.as<int64_t>();
    opt.spec_row = s->d_rows.as<int32_t>();
    popt = &opt;
  }
  asim::DevOut out;
  out.good = good_dev;
  out.sum_latency = nullptr;
  out.good_per_model = nullptr;
  out.out_offset = begin;
  out.stage_updates = nullptr;
  st = asim_run_batch(s->ctx, s->hb, begin, end, out, strm, popt);
  if (prev >= 0 && prev != s->ctx->device) cudaSetDevice(prev);
  return st;
}

asim_status asim_search_apply(asim_search* s, const int64_t* good_all_dev, void* cuda_stream) {
  if (!s) return ASIM_EINVAL;
  if (!s->prepared) return sfail(s, ASIM_ESTATE, "apply before prepare");
  const int64_t C = (int64_t)s->hb.cand_base.size();
  if (C > 0 && !good_all_dev) return sfail(s, ASIM_EINVAL, "null good_all_dev");
  cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
  s->h_good.resize(C);
  if (C > 0) {
    cudaError_t e =
        cudaMemcpyAsync(s->h_good.data(), good_all_dev, C * 8, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return asim_cuda(s->ctx, e, "copy step results");
  }
  const HostProblem& hp = s->ctx->hp;
  const int32_t M = hp.M;
  const bool restricted = !s->hb.cand_kmask.empty();
  if (restricted) {  // per-model good of every base (from the base pass)
    if (!s->base_ready) return sfail(s, ASIM_ESTATE, "internal: base pass missing");
    const size_t n = s->base_run.size() * (size_t)M;
    s->h_base_pm.resize(n);
    cudaError_t e = cudaMemcpyAsync(s->h_base_pm.data(), s->d_base_pm.p, n * 8,
                                    cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return asim_cuda(s->ctx, e, "copy base per-model good");
  }
  for (size_t b = 0; b < s->base_run.size(); ++b) {
    Run& run = s->runs[s->base_run[b]];
    if (restricted) {  // internal consistency: the base pass reproduces the base's good
      int64_t tot = 0;
      for (int32_t m = 0; m < M; ++m) tot += s->h_base_pm[b * M + m];
      if (tot != run.base_good)
        return sfail(s, ASIM_ERANGE, "internal: base pass disagrees with the last winner");
    }
    // every candidate's good: simulated, memo, or its duplicate's representative
    int64_t bi = -1, bg = -1;
    for (size_t i = 0; i < run.cands.size(); ++i) {
      Run::Cand& c = run.cands[i];
      if (c.kind == 0) {
        c.good = s->h_good[c.ref];
        if (restricted) {  // good(base) - good_base(K_c) + good_c(K_c)
          const uint64_t km = s->hb.cand_kmask[c.ref];
          int64_t gk = 0;
          for (int32_t m = 0; m < M; ++m)
            if ((km >> m) & 1ULL) gk += s->h_base_pm[b * M + m];
          c.good += run.base_good - gk;
        }
      } else if (c.kind == 2) {
        c.good = run.cands[c.ref].good;
      }
      if (c.good > bg) {  // first maximum in (m, g) order: lowest index on ties (C12)
        bg = c.good;
        bi = (int64_t)i;
      }
    }
    if (bi < 0) return sfail(s, ASIM_ERANGE, "step results contain no feasible candidate");
    const int32_t ms = run.cands[bi].m, gs = run.cands[bi].g;
    // memo for the next step: candidates whose component avoids the two
    // components the winner merges keep their good shifted by the base's change
    Components comp(run.G, M, run.sel);
    const int32_t w1 = comp.find(gs), w2 = comp.find(run.G + ms);
    const int64_t shift = bg - run.base_good;
    run.memo.clear();
    for (const Run::Cand& c : run.cands) {
      const int32_t a1 = comp.find(c.g), a2 = comp.find(run.G + c.m);
      if (a1 != w1 && a1 != w2 && a2 != w1 && a2 != w2)
        run.memo.emplace(std::make_pair(c.m, c.g), c.good + shift);
    }
    run.sel[ms] |= 1ULL << gs;
    run.used[gs] += hp.mem_at(ms, run.cfg[gs]);
    run.base_good = bg;
    run.history.emplace_back(ms, gs);
    ++run.steps;
    if (bg > run.best_good) {  // "if sel*.slo_att > best_sel.slo_att"
      run.best_good = bg;
      run.best = run.sel;
    }
  }
  if (s->base_ready) std::swap(s->state_prev, s->state_cur);  // next step speculates from it
  s->prepared = false;
  return ASIM_OK;
}

asim_status asim_search_run(asim_search* s, void* cuda_stream) {
  if (!s) return ASIM_EINVAL;
  for (;;) {
    int64_t C = 0;
    asim_status st = asim_search_prepare(s, &C);
    if (st) return st;
    if (C < 0) return ASIM_OK;
    cudaError_t e = s->d_good_all.ensure(C * 8 + 8);
    if (e != cudaSuccess) return asim_cuda(s->ctx, e, "allocate step results");
    st = asim_search_evaluate(s, 0, C, s->d_good_all.as<int64_t>(), cuda_stream);
    if (st) return st;
    st = asim_search_apply(s, s->d_good_all.as<int64_t>(), cuda_stream);
    if (st) return st;
  }
}

asim_status asim_search_result_get(const asim_search* s, asim_search_result* out) {
  if (!s || !out) return ASIM_EINVAL;
  int32_t best = -1;
  int64_t best_good = 0;
  for (int32_t r = 0; r < (int32_t)s->runs.size(); ++r)
    if (s->runs[r].best_good > best_good) {  // Alg. 2: strict '>' keeps the first best run
      best_good = s->runs[r].best_good;
      best = r;
    }
  out->best_run = best;
  out->best_good = best_good;
  out->num_groups = best >= 0 ? s->runs[best].G : 0;
  if (out->group_cfg) {
    for (int32_t g = 0; g < ASIM_MAX_GROUPS; ++g)
      out->group_cfg[g] = (best >= 0 && g < s->runs[best].G) ? s->runs[best].cfg[g] : -1;
  }
  if (out->host_mask)
    for (int32_t m = 0; m < s->ctx->hp.M; ++m)
      out->host_mask[m] = best >= 0 ? s->runs[best].best[m] : 0;
  out->steps = s->steps;
  out->candidates = s->candidates;
  out->evaluated = s->evaluated;
  out->request_evals = s->evaluated * s->ctx->n;
  out->memo_hits = s->memo_hits;
  return ASIM_OK;
}

asim_status asim_search_run_info(const asim_search* s, int32_t run, int32_t* num_groups,
                                 int32_t* group_cfg, uint64_t* host_mask, int64_t* best_good,
                                 int64_t* steps) {
  if (!s || run < 0 || run >= (int32_t)s->runs.size()) return ASIM_EINVAL;
  const Run& r = s->runs[run];
  if (num_groups) *num_groups = r.G;
  if (group_cfg)
    for (int32_t g = 0; g < r.G; ++g) group_cfg[g] = r.cfg[g];
  if (host_mask)
    for (int32_t m = 0; m < s->ctx->hp.M; ++m) host_mask[m] = r.best[m];
  if (best_good) *best_good = r.best_good;
  if (steps) *steps = r.steps;
  return ASIM_OK;
}

}  // extern "C"
