// chunked.cpp -- host orchestration of the chunked throughput path
// (chunk.cu): work-item construction, chunk sizing, the speculative pass,
// the fix-up passes with exact re-run chains, and the final reduction.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <vector>

#include "ctx.h"

namespace {

constexpr int kSTab = 16;

// Events around one phase of the chunked path on `st` (profiling only).
struct PhaseTimer {
  asim_ctx* ctx;
  int ph;
  cudaStream_t st;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  PhaseTimer(asim_ctx* c, int phase, cudaStream_t s, bool on) : ctx(c), ph(phase), st(s) {
    if (!on || !c->profiling) return;
    if (cudaEventCreate(&e0) != cudaSuccess || cudaEventCreate(&e1) != cudaSuccess) {
      if (e0) cudaEventDestroy(e0);
      e0 = e1 = nullptr;
      return;
    }
    cudaEventRecord(e0, st);
  }
  ~PhaseTimer() {
    if (!e0) return;
    cudaEventRecord(e1, st);
    ctx->phase_events[ph].emplace_back(e0, e1);
  }
};

int stage_class(int s) { return (s == 1 || s == 2 || s == 4 || s == 8 || s == 16) ? s : 0; }

}  // namespace

bool asim_chunked_eligible(const asim_ctx* ctx, const HostBatch& hb, const asim::DevOut& out) {
  if (out.good_per_model || out.busy) return false;  // per-model / per-group outputs: sim.cu
  if (hb.slots > ASIM_MAX_SLOTS) return false;
  const size_t M = (size_t)ctx->hp.M;
  const size_t per_warp = (size_t)hb.slots * 32 * 8 * 2 + M * (8 + 8 * (kSTab + 2)) + 256 + 1536;
  return 4 * per_warp <= 220 * 1024;
}

// Hosting-list bytes per warp: 2 bytes per (model, group) hosting of the
// largest base in the batch, at least 4 M (the scalar walker's compact
// masks), rounded.
static int32_t hid_cap_for(const asim_ctx* ctx, const HostBatch& hb) {
  const int32_t M = ctx->hp.M;
  int64_t cap = 4 * (int64_t)M;
  const size_t B = M ? hb.base_mask.size() / M : 0;
  for (size_t b = 0; b < B; ++b) {
    int64_t n = 0;
    for (int32_t m = 0; m < M; ++m) n += __builtin_popcountll(hb.base_mask[b * M + m]);
    cap = std::max(cap, 2 * n);  // uint16 entries
  }
  return (int32_t)((cap + 15) & ~int64_t(15));
}

// uint32 relative time is exact when 2^32 - 1 - max slo - max service > 0
// (chunk.cu header); require some headroom so epochs move rarely.
static int64_t theta_for(const asim_ctx* ctx) {
  int64_t slo_max = 0;
  for (int64_t s : ctx->hp.slo) slo_max = std::max(slo_max, s);
  const __int128 th = (__int128)0xFFFFFFFFll - slo_max - ctx->hp.max_service;
  if (th < 100000000) return -1;  // < 0.1 s of headroom: use int64
  return (int64_t)th;
}

asim_status asim_run_fast_stats(asim_ctx* ctx, const HostBatch& hb, const asim::DevOut& out,
                                cudaStream_t st, bool* done) {
  *done = false;
  const HostProblem& hp = ctx->hp;
  const int64_t C = (int64_t)hb.cand_base.size();
  if (C == 0) {
    *done = true;
    return ASIM_OK;
  }
  std::vector<asim::ItemDesc> items;
  int32_t slots_max = 1;
  for (int64_t c = 0; c < C; ++c) {
    const int32_t b = hb.cand_base[c];
    int32_t u = -2, slots = 0;
    bool hole = false;
    for (int32_t g = 0; g < hb.G; ++g) {
      const int32_t k = hb.base_cfg[(int64_t)b * hb.G + g];
      if (k < 0) {
        hole = true;
        continue;
      }
      slots += hp.cfg_stages[k];
      u = (!hole && (u == -2 || u == k)) ? k : -1;
    }
    if (u < 0 || !hb.cand_ok[c] || hb.cand_model[c] >= 0) return ASIM_OK;
    asim::ItemDesc it{};
    it.base = b;
    it.first = (int32_t)c;
    it.count = 1;
    it.cfg = u;
    it.stages = hp.cfg_stages[u];
    it.S = stage_class(it.stages);
    it.slots = slots;
    if (it.S == 0 || slots > ASIM_MAX_SLOTS) return ASIM_OK;
    slots_max = std::max(slots_max, slots);
    items.push_back(it);
  }
  const int64_t theta = ctx->force_path == 3 ? -1 : theta_for(ctx);
  const bool u32 = theta > 0;
  const int32_t hid_cap = hid_cap_for(ctx, hb);
  if (asim::fast_stats_smem(slots_max, hp.M, hid_cap, u32) > 227 * 1024) return ASIM_OK;
  ChunkSlot& cs = ctx->slot[0];
  cs.last_valid = false;  // its chunk buffers are reused below
  cudaError_t e = upload(cs.items, items, st);
  if (e == cudaSuccess) e = cs.spm.ensure((size_t)C * hp.M * 4 + 8);  // int32 count rows
  if (e == cudaSuccess) e = cudaMemsetAsync(cs.spm.p, 0, (size_t)C * hp.M * 4, st);
  if (e != cudaSuccess) return asim_cuda(ctx, e, "upload fast items");
  asim::ChunkParams P{};
  P.pr = ctx->dev_problem();
  P.tr = ctx->dev_trace();
  P.bt.G = hb.G;
  P.bt.base_cfg = ctx->d_base_cfg.as<int32_t>();
  P.bt.base_mask = ctx->d_base_mask.as<uint64_t>();
  P.bt.cand_base = ctx->d_cand_base.as<int32_t>();
  P.bt.cand_model = ctx->d_cand_model.as<int32_t>();
  P.bt.cand_group = ctx->d_cand_group.as<int32_t>();
  P.bt.cand_ok = ctx->d_cand_ok.as<uint8_t>();
  P.bt.cand_kmask = hb.cand_kmask.empty() ? nullptr : ctx->d_cand_kmask.as<uint64_t>();
  P.bt.C = C;
  P.items = cs.items.as<asim::ItemDesc>();
  P.num_items = (int32_t)items.size();
  P.J = 1;
  P.theta = theta;
  P.slots_max = slots_max;
  P.hid_cap = hid_cap;
  P.spec_pm = cs.spm.as<int32_t>();
  P.stat_C = C;
  P.stage_updates = ctx->profiling ? ctx->d_counter.as<unsigned long long>() : nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  if (ctx->profiling) {
    if (cudaEventCreate(&ev0) != cudaSuccess || cudaEventCreate(&ev1) != cudaSuccess)
      return asim_cuda(ctx, cudaGetLastError(), "event create");
    cudaEventRecord(ev0, st);
  }
  e = asim::launch_fast_stats(P, out, u32, st, &ctx->launches);
  if (e != cudaSuccess) return asim_cuda(ctx, e, "fast statistics kernel");
  if (ctx->profiling) {
    cudaEventRecord(ev1, st);
    ctx->events.emplace_back(ev0, ev1);
    ++ctx->sim_launches;
    ctx->request_evals += C * ctx->n;
  }
  *done = true;
  return ASIM_OK;
}

// Pass 1's algorithmic work, fixed by the candidates alone (profiling): every
// (item, chunk) unit replays the chunk's requests of the models some active
// lane simulates (the union of the lanes' components), and a live lane
// performs, for each request of a model m of its component, one max-plus
// update per stage of every group hosting m.  Summed over
// the J chunks that is the whole trace's per-model counts n(m):
//   stage updates  = sum_lanes sum_{m in K_c} n(m) * sum_{g hosts m} s_g
//   live lane-reqs = sum_lanes sum_{m in K_c} n(m)
//   lane slots     = 32 * sum_items sum_{m in union of the lanes' K_c} n(m)
static void pass1_work(asim_ctx* ctx, const HostBatch& hb,
                       const std::vector<asim::ItemDesc>& items,
                       const std::vector<int32_t>& item_cand, bool grouped) {
  const HostProblem& hp = ctx->hp;
  const int32_t M = hp.M;
  const bool restricted = !hb.cand_kmask.empty();
  unsigned long long upd = 0, live = 0, slots = 0;
  std::vector<int64_t> hs(M);  // sum of host stage counts of m in the base
  std::vector<uint8_t> rel(M);
  for (size_t i = 0; i < items.size(); ++i) {
    const asim::ItemDesc& it = items[i];
    const int32_t b = it.base;
    const unsigned long long upd_i = upd, slots_i = slots;
    for (int32_t m = 0; m < M; ++m) {
      const uint64_t mk = hb.base_mask[(size_t)b * M + m];
      int64_t x = 0;
      for (uint64_t r = mk; r; r &= r - 1) {
        const int g = __builtin_ctzll(r);
        x += hp.cfg_stages[hb.base_cfg[(size_t)b * hb.G + g]];
      }
      hs[m] = x;
      rel[m] = 0;
    }
    for (int32_t l = 0; l < it.count; ++l) {
      const int32_t c = grouped ? item_cand[i * 32 + l] : it.first + l;
      if (!hb.cand_ok[c]) continue;
      const int32_t mm = hb.cand_model[c], gg = hb.cand_group[c];
      const uint64_t km = restricted ? hb.cand_kmask[c] : ~0ull;
      for (int32_t m = 0; m < M; ++m) {
        const bool in = restricted ? (m < 64 && ((km >> m) & 1ull))
                                   : (hs[m] > 0 || m == mm);
        if (!in) continue;
        rel[m] = 1;
        const int64_t n = ctx->model_n[m];
        live += (unsigned long long)n;
        int64_t h = hs[m];
        if (m == mm) h += hp.cfg_stages[hb.base_cfg[(size_t)b * hb.G + gg]];
        upd += (unsigned long long)(n * h);
      }
    }
    int64_t u = 0;
    for (int32_t m = 0; m < M; ++m)
      if (rel[m]) u += ctx->model_n[m];
    slots += 32ull * (unsigned long long)u;
    const int cls = it.S == 1 ? 1 : it.S == 2 ? 2 : it.S == 4 ? 3 : it.S == 8 ? 4 : it.S == 16 ? 5 : 0;
    ctx->p1_class[cls][0] += (int64_t)(upd - upd_i);
    ctx->p1_class[cls][1] += (int64_t)(slots - slots_i);
  }
  ctx->p1_updates += (int64_t)upd;
  ctx->p1_live += (int64_t)live;
  ctx->p1_slots += (int64_t)slots;
}

// One chunked run of the candidates `cand` (batch indices) on slot `cs`,
// stream-ordered on `st`.
static asim_status run_slot(asim_ctx* ctx, ChunkSlot& cs, const HostBatch& hb,
                            std::vector<int32_t> ord, const asim::DevOut& out, cudaStream_t st,
                            const ChunkOptions* opt, bool transient = false) {
  const int64_t N = ctx->n;
  const HostProblem& hp = ctx->hp;
  // ---- work items: <= 32 consecutive candidates of one base
  std::vector<asim::ItemDesc> items;
  std::vector<int32_t> base_cfg_uniform, base_slots;
  const int32_t B = hb.G ? (int32_t)(hb.base_cfg.size() / hb.G) : (int32_t)(hb.base_mask.size() / hp.M);
  base_cfg_uniform.assign(B, -1);
  base_slots.assign(B, 0);
  for (int32_t b = 0; b < B; ++b) {
    int32_t u = -2, slots = 0;
    bool hole = false;
    for (int32_t g = 0; g < hb.G; ++g) {
      const int32_t c = hb.base_cfg[(int64_t)b * hb.G + g];
      if (c < 0) {
        hole = true;
        continue;
      }
      slots += hp.cfg_stages[c];
      // uniform kernels address group g's stages at g * S: no gaps allowed
      u = (!hole && (u == -2 || u == c)) ? c : -1;
    }
    base_cfg_uniform[b] = u >= 0 ? u : -1;
    base_slots[b] = slots;
  }
  int32_t slots_max = 1;
  // Candidate order inside the range: the batch's, or grouped by hosting
  // component (hb.cand_key, the search's): a warp replays the union of its
  // lanes' requests, so lanes sharing their components keep every lane busy.
  const bool by_key = !hb.cand_key.empty();
  // items list their candidates explicitly (item_cand) unless they are runs of
  // consecutive batch indices: when regrouped, or when the run takes a subset
  // of the range (a split step)
  bool grouped = by_key;
  for (size_t i = 1; i < ord.size() && !grouped; ++i) grouped = ord[i] != ord[i - 1] + 1;
  if (by_key)
    std::stable_sort(ord.begin(), ord.end(), [&](int32_t a, int32_t b) {
      if (hb.cand_base[a] != hb.cand_base[b]) return hb.cand_base[a] < hb.cand_base[b];
      return hb.cand_key[a] < hb.cand_key[b];
    });
  std::vector<int32_t> item_cand;
  for (size_t pos = 0; pos < ord.size();) {
    const int32_t b = hb.cand_base[ord[pos]];
    int32_t cnt = 1;
    while (pos + cnt < ord.size() && cnt < 32 && hb.cand_base[ord[pos + cnt]] == b) ++cnt;
    asim::ItemDesc it{};
    it.base = b;
    it.first = ord[pos];
    it.count = cnt;
    it.cfg = base_cfg_uniform[b];
    it.stages = it.cfg >= 0 ? hp.cfg_stages[it.cfg] : 0;
    it.S = it.cfg >= 0 ? stage_class(it.stages) : 0;
    if (it.S == 0) it.cfg = -1;
    it.slots = base_slots[b];
    slots_max = std::max(slots_max, it.slots);
    items.push_back(it);
    if (grouped)
      for (int32_t l = 0; l < 32; ++l) item_cand.push_back(l < cnt ? ord[pos + l] : -1);
    pos += cnt;
  }
  const int32_t I = (int32_t)items.size();
  if (I == 0) return ASIM_OK;
  // ---- chunks: enough (item, chunk) units to fill the GPU, chunks >= kMinChunk
  const int64_t target_units = (int64_t)ctx->sms * 16 * 4;
  int64_t J = (target_units + I - 1) / I;
  J = std::min<int64_t>(J, std::max<int64_t>(1, N / std::max<int64_t>(1, ctx->min_chunk)));
  J = std::max<int64_t>(1, std::min<int64_t>(J, 1 << 16));
  if (N == 0) J = 1;
  if (opt && opt->J > 0) J = opt->J;  // the search keeps one chunking for all its steps
  std::vector<int64_t> cb(J + 1);
  for (int64_t j = 0; j <= J; ++j) cb[j] = N * j / J;
  const int64_t theta = ctx->force_path == 3 ? -1 : theta_for(ctx);
  const bool u32 = theta > 0;
  const size_t tsz = u32 ? 4 : 8;

  // ---- device buffers (grow-only)
  const int64_t per_chunk = (int64_t)I * 32;
  cudaError_t e = upload(cs.items, items, st);
  if (e == cudaSuccess && grouped) e = upload(cs.item_cand, item_cand, st);
  if (e == cudaSuccess) e = upload(cs.begin, cb, st);
  if (e == cudaSuccess) e = cs.spec_good.ensure(J * per_chunk * 4);
  if (e == cudaSuccess) e = cs.spec_sum.ensure(J * per_chunk * 8);
  if (e == cudaSuccess) e = cs.fix_good.ensure(J * per_chunk * 4);
  if (e == cudaSuccess) e = cs.fix_sum.ensure(J * per_chunk * 8);
  if (e == cudaSuccess) e = cs.spec_end.ensure(J * I * (int64_t)slots_max * 32 * tsz);
  if (e == cudaSuccess) e = cs.fix_end.ensure(J * I * (int64_t)slots_max * 32 * tsz);
  if (e == cudaSuccess) e = cs.spec_epoch.ensure(J * I * 8);
  if (e == cudaSuccess) e = cs.fix_epoch.ensure(J * I * 8);
  if (e == cudaSuccess) e = cs.flag.ensure(J * I * 4 + 8);
  if (e == cudaSuccess) e = cs.counter.ensure(16);
  if (e != cudaSuccess) return asim_cuda(ctx, e, "chunk buffers");

  asim::ChunkParams P{};
  P.pr = ctx->dev_problem();
  P.tr = ctx->dev_trace();
  P.bt.G = hb.G;
  P.bt.base_cfg = ctx->d_base_cfg.as<int32_t>();
  P.bt.base_mask = ctx->d_base_mask.as<uint64_t>();
  P.bt.cand_base = ctx->d_cand_base.as<int32_t>();
  P.bt.cand_model = ctx->d_cand_model.as<int32_t>();
  P.bt.cand_group = ctx->d_cand_group.as<int32_t>();
  P.bt.cand_ok = ctx->d_cand_ok.as<uint8_t>();
  P.bt.cand_kmask = hb.cand_kmask.empty() ? nullptr : ctx->d_cand_kmask.as<uint64_t>();
  P.bt.cand_gmask = hb.cand_gmask.empty() ? nullptr : ctx->d_cand_gmask.as<uint64_t>();
  P.bt.C = (int64_t)hb.cand_base.size();
  P.items = cs.items.as<asim::ItemDesc>();
  P.item_cand = grouped ? cs.item_cand.as<int32_t>() : nullptr;
  P.num_items = I;
  P.J = (int32_t)J;
  P.chunk_begin = cs.begin.as<int64_t>();
  P.theta = theta;
  P.slots_max = slots_max;
  P.hid_cap = hid_cap_for(ctx, hb);
  P.counter = cs.counter.as<uint32_t>();
  P.spec_good = cs.spec_good.as<int32_t>();
  P.spec_sum = cs.spec_sum.as<int64_t>();
  P.spec_end = cs.spec_end.p;
  P.spec_epoch = cs.spec_epoch.as<int64_t>();
  P.fix_good = cs.fix_good.as<int32_t>();
  P.fix_sum = cs.fix_sum.as<int64_t>();
  P.fix_end = cs.fix_end.p;
  P.fix_epoch = cs.fix_epoch.as<int64_t>();
  P.fix_flag = cs.flag.as<uint32_t>();
  P.stage_updates = out.stage_updates;
  P.walked = ctx->profiling ? cs.walked.as<unsigned long long>() : nullptr;
  P.scalar_walk = ctx->scalar_walk ? 1 : 0;
  P.glane_walk = ctx->glane_walk;
  P.glane_smax = ctx->glane_smax;
  P.transient = transient ? 1 : 0;
  P.walk_log = ctx->walk_log;
  P.spec_state = opt ? opt->spec_state : nullptr;
  P.spec_row = opt ? opt->spec_row : nullptr;
  P.spec_cand = opt ? opt->spec_cand : nullptr;
  P.state_stride = (opt && opt->state_stride > 0) ? opt->state_stride : slots_max;
  if (P.spec_state && P.state_stride < slots_max)
    return asim_fail(ctx, ASIM_ERANGE, "internal: state stride below slots");
  // fast-heuristic statistics (per-model good, per-group busy) of every candidate
  const bool stats = out.good_per_model != nullptr || out.busy != nullptr;
  if (stats) {
    if (!out.good_per_model || !out.busy || (int64_t)ord.size() != P.bt.C)
      return asim_fail(ctx, ASIM_ESTATE, "internal: statistics need both outputs, whole batch");
    const int64_t C = P.bt.C;
    const size_t npm = (size_t)J * C * hp.M, nb = (size_t)J * C * std::max(hb.G, 1);
    e = cs.spm.ensure(npm * 4 + 8);
    if (e == cudaSuccess) e = cs.fpm.ensure(npm * 4 + 8);
    if (e == cudaSuccess) e = cs.sbusy.ensure(nb * 8 + 8);
    if (e == cudaSuccess) e = cs.fbusy.ensure(nb * 8 + 8);
    if (e == cudaSuccess) e = cudaMemsetAsync(cs.spm.p, 0, npm * 4, st);
    if (e == cudaSuccess) e = cudaMemsetAsync(cs.fpm.p, 0, npm * 4, st);
    if (e == cudaSuccess) e = cudaMemsetAsync(cs.sbusy.p, 0, nb * 8, st);
    if (e == cudaSuccess) e = cudaMemsetAsync(cs.fbusy.p, 0, nb * 8, st);
    if (e != cudaSuccess) return asim_cuda(ctx, e, "statistics buffers");
    P.spec_pm = cs.spm.as<int32_t>();
    P.fix_pm = cs.fpm.as<int32_t>();
    P.spec_busy = cs.sbusy.as<int64_t>();
    P.fix_busy = cs.fbusy.as<int64_t>();
    P.stat_C = C;
  }

  // ---- item classes by stage count (passes 1-2 run one class after another)
  {
    const int order[6] = {1, 2, 4, 8, 16, 0};
    std::vector<int32_t> perm;
    P.nclass = 0;
    for (int S : order) {
      const int32_t off = (int32_t)perm.size();
      for (int32_t i = 0; i < I; ++i)
        if (items[i].S == S) perm.push_back(i);
      if ((int32_t)perm.size() > off) {
        P.class_off[P.nclass] = off;
        P.class_items[P.nclass] = (int32_t)perm.size() - off;
        ++P.nclass;
      }
    }
    e = upload(cs.perm, perm, st);
    if (e != cudaSuccess) return asim_cuda(ctx, e, "item classes");
    P.item_perm = cs.perm.as<int32_t>();
  }
  // ---- pass 1: every (item, chunk) from the speculative start
  P.num_units = (int32_t)(J * I);
  {
    // profiling: pass 1 alone (the dominant kernel) gets its own events and
    // work counter (d_counter[1]; the total is d_counter[0] + d_counter[1])
    asim::ChunkParams P1 = P;
    if (ctx->profiling && P.stage_updates) pass1_work(ctx, hb, items, item_cand, grouped);
    PhaseTimer t(ctx, 0, st, P.stage_updates != nullptr);
    e = asim::launch_chunk_pass(P1, false, u32, st, ctx->sms, &ctx->launches);
    if (e != cudaSuccess) return asim_cuda(ctx, e, "chunk pass 1");
  }

  e = cs.end_src.ensure(J * I * 4 + 8);
  if (e != cudaSuccess) return asim_cuda(ctx, e, "end_src buffer");
  uint32_t* end_src = cs.end_src.as<uint32_t>();
  bool any_dynamic = false;
  for (const auto& it : items) any_dynamic |= it.S == 0;
  if (J > 1) {
    // ---- pass 2: fix-up of every chunk j >= 1 from chunk j-1's speculative end
    P.num_units = (int32_t)((J - 1) * I);
    {
      PhaseTimer t(ctx, 1, st, P.stage_updates != nullptr);
      e = asim::launch_chunk_pass(P, true, u32, st, ctx->sms, &ctx->launches);
    }
    if (e != cudaSuccess) return asim_cuda(ctx, e, "chunk pass 2");
    if (opt && opt->walk_out) {
      e = asim::launch_walk_flags(P, opt->walk_out, st, &ctx->launches);
      if (e != cudaSuccess) return asim_cuda(ctx, e, "walk flags");
    }
    // ---- pass 3: walk the chunks whose start state was wrong (exact chains)
    const asim::WalkStreams ws{st, {cs.side[0], cs.side[1]}, cs.ev_fork,
                               {cs.ev_join[0], cs.ev_join[1]}};
    {
      PhaseTimer t(ctx, 2, st, P.stage_updates != nullptr);
      e = asim::launch_chunk_walk(P, end_src, u32, any_dynamic, ws, ctx->sms, &ctx->launches);
    }
    if (e != cudaSuccess) return asim_cuda(ctx, e, "chunk walk");
  } else {
    e = cudaMemsetAsync(end_src, 0, J * I * 4, st);
    if (e != cudaSuccess) return asim_cuda(ctx, e, "end_src");
  }
  e = asim::launch_chunk_reduce(P, out, st, &ctx->launches);
  if (e != cudaSuccess) return asim_cuda(ctx, e, "chunk reduce");
  if (stats) {
    e = asim::launch_chunk_stats_reduce(P, out, st, &ctx->launches);
    if (e != cudaSuccess) return asim_cuda(ctx, e, "statistics reduce");
  }
  cs.last_valid = true;
  cs.last_u32 = u32;
  cs.last_gen = ctx->batch_gen;
  cs.last_params = P;
  cs.last_items = std::move(items);
  cs.last_pos.assign(P.bt.C, -1);  // candidate -> item * 32 + lane of this run
  for (size_t i = 0, pos = 0; i < cs.last_items.size(); ++i)
    for (int32_t l = 0; l < cs.last_items[i].count; ++l, ++pos)
      cs.last_pos[ord[pos]] = (int32_t)(i * 32 + l);
  return ASIM_OK;
}

asim_status asim_run_chunked(asim_ctx* ctx, const HostBatch& hb, int64_t begin, int64_t end,
                             const asim::DevOut& out, cudaStream_t st, const ChunkOptions* opt) {
  std::vector<int32_t> ord;
  ord.reserve(end > begin ? end - begin : 0);
  for (int64_t c = begin; c < end; ++c) ord.push_back((int32_t)c);
  ctx->slot[1].last_valid = false;  // only slot 0 holds this batch's run
  return run_slot(ctx, ctx->slot[0], hb, std::move(ord), out, st, opt);
}

asim_status asim_run_chunked_split(asim_ctx* ctx, const HostBatch& hb, int64_t begin, int64_t end,
                                   const std::vector<uint8_t>& group, const asim::DevOut& out,
                                   cudaStream_t st, const ChunkOptions* opt) {
  std::vector<int32_t> ord[kChunkSlots];
  for (int64_t c = begin; c < end; ++c) ord[group[c] ? 1 : 0].push_back((int32_t)c);
  if (ord[0].empty() || ord[1].empty())
    return asim_run_chunked(ctx, hb, begin, end, out, st, opt);
  // fork both runs from the caller's stream (after the batch upload), join back
  cudaError_t e = cudaEventRecord(ctx->ev_split, st);
  if (e != cudaSuccess) return asim_cuda(ctx, e, "split fork");
  for (int k = 0; k < kChunkSlots; ++k) {
    ChunkSlot& cs = ctx->slot[k];
    e = cudaStreamWaitEvent(cs.main, ctx->ev_split, 0);
    if (e != cudaSuccess) return asim_cuda(ctx, e, "split fork");
    asim_status rc = run_slot(ctx, cs, hb, std::move(ord[k]), out, cs.main, opt, true);
    if (rc) return rc;
    e = cudaEventRecord(cs.ev_done, cs.main);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(st, cs.ev_done, 0);
    if (e != cudaSuccess) return asim_cuda(ctx, e, "split join");
  }
  return ASIM_OK;
}

asim_status asim_publish_candidates(asim_ctx* ctx, const std::vector<int64_t>& cands,
                                    const std::vector<int32_t>& rows, int64_t* out,
                                    cudaStream_t st) {
  if (cands.empty()) return ASIM_OK;
  // the runs of the current batch (one, or two for a split step)
  std::vector<asim::PublishItem> pub[kChunkSlots];
  for (size_t i = 0; i < cands.size(); ++i) {
    const int64_t c = cands[i];
    bool found = false;
    for (int k = 0; k < kChunkSlots && !found; ++k) {
      const ChunkSlot& cs = ctx->slot[k];
      if (!cs.last_valid || cs.last_gen != ctx->batch_gen) continue;
      const int32_t pos = (c >= 0 && c < (int64_t)cs.last_pos.size()) ? cs.last_pos[c] : -1;
      if (pos < 0) continue;
      pub[k].push_back(asim::PublishItem{pos >> 5, pos & 31, rows[i]});
      found = true;
    }
    if (!found)
      return asim_fail(ctx, ASIM_ESTATE, "internal: candidate not in the last chunked run");
  }
  for (int k = 0; k < kChunkSlots; ++k) {
    if (pub[k].empty()) continue;
    ChunkSlot& cs = ctx->slot[k];
    cudaError_t e = upload(cs.pub, pub[k], st);
    if (e == cudaSuccess)
      e = asim::launch_publish_states(cs.last_params, cs.end_src.as<uint32_t>(), cs.last_u32,
                                      cs.pub.as<asim::PublishItem>(), (int32_t)pub[k].size(), out,
                                      st, &ctx->launches);
    if (e != cudaSuccess) return asim_cuda(ctx, e, "publish states");
  }
  return ASIM_OK;
}
