// ctx.cpp -- context, input validation, encoding and evaluate entry points of
// libasim.so (see include/asim.h for the contract).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <climits>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "ctx.h"

namespace {

thread_local std::string g_create_err;

constexpr int64_t kMaxService = int64_t(1) << 60;  // reading C20
constexpr int64_t kMaxTime = int64_t(1) << 62;

// Make ctx's device current for the duration of a call; restore afterwards.
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

template <class T>
asim_status fetch(asim_ctx* ctx, std::vector<T>& dst, const T* src, int64_t count, int32_t kind,
                  cudaStream_t st, const char* what) {
  if (count == 0) {
    dst.clear();
    return ASIM_OK;
  }
  if (!src) return asim_fail(ctx, ASIM_EINVAL, std::string("null ") + what);
  try {
    dst.resize((size_t)count);
  } catch (const std::bad_alloc&) {
    return asim_fail(ctx, ASIM_ENOMEM, "host allocation failed");
  }
  if (kind == ASIM_HOST) {
    std::memcpy(dst.data(), src, (size_t)count * sizeof(T));
    return ASIM_OK;
  }
  if (kind != ASIM_DEVICE) return asim_fail(ctx, ASIM_EINVAL, "ptr_kind must be ASIM_HOST or ASIM_DEVICE");
  cudaError_t e = cudaMemcpyAsync(dst.data(), src, (size_t)count * sizeof(T),
                                  cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  return asim_cuda(ctx, e, what);
}

// Per-base structural check + memory/device feasibility (reading C11).
// Fills used[G] (bytes per device on each group); returns ASIM_OK and sets
// *feasible, or an error status for structural problems.
asim_status check_base(asim_ctx* ctx, const int32_t* cfg, const uint64_t* mask, int32_t G,
                       std::vector<int64_t>& used, bool* feasible, int32_t* slots) {
  const HostProblem& hp = ctx->hp;
  used.assign(G, 0);
  int64_t devices = 0;
  int32_t nslots = 0;
  bool ok = true;
  for (int g = 0; g < G; ++g) {
    if (cfg[g] < -1 || cfg[g] >= hp.P)
      return asim_fail(ctx, ASIM_ERANGE, "group_cfg out of range");
    if (cfg[g] >= 0) {
      devices += hp.cfg_devices[cfg[g]];
      nslots += hp.cfg_stages[cfg[g]];
    }
  }
  if (nslots > ASIM_MAX_SLOTS)
    return asim_fail(ctx, ASIM_ERANGE, "sum of stages over groups exceeds ASIM_MAX_SLOTS");
  for (int m = 0; m < hp.M; ++m) {
    const uint64_t bits = mask[m];
    if (!bits) continue;
    if (G < 64 && (bits >> G))
      return asim_fail(ctx, ASIM_ERANGE, "host_mask bit beyond max_groups");
    for (int g = 0; g < G; ++g) {
      if (!((bits >> g) & 1ULL)) continue;
      if (cfg[g] < 0) return asim_fail(ctx, ASIM_ERANGE, "host_mask names a group with cfg -1");
      const int64_t mb = hp.mem_at(m, cfg[g]);
      if (mb < 0) ok = false;  // (m, p) not placeable
      else used[g] += mb;
    }
  }
  for (int g = 0; g < G; ++g)
    if (used[g] > hp.budget) ok = false;  // "if sel' is in memory constraint"
  if (devices > hp.num_devices) ok = false;
  *feasible = ok;
  *slots = std::max(*slots, nslots);
  return ASIM_OK;
}

asim_status finish_outputs(asim_ctx* ctx, asim_results* out, int64_t C, int32_t G, bool want_sum,
                           bool want_pm, bool want_busy, bool want_arg, cudaStream_t st) {
  const int64_t M = ctx->hp.M;
  cudaError_t e = cudaSuccess;
  if (out->ptr_kind == ASIM_HOST) {
    if (C > 0) e = cudaMemcpyAsync(out->good, ctx->d_good.p, C * 8, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess && want_sum && C > 0)
      e = cudaMemcpyAsync(out->sum_latency_ns, ctx->d_sum.p, C * 8, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess && want_pm && C > 0)
      e = cudaMemcpyAsync(out->good_per_model, ctx->d_pm.p, C * M * 8, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess && want_busy && C * G > 0)
      e = cudaMemcpyAsync(out->busy_ns, ctx->d_busy.p, C * G * 8, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess && want_arg)
      e = cudaMemcpyAsync(out->argmax, ctx->d_argmax.p, 8, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  }
  return asim_cuda(ctx, e, "copy results");
}

}  // namespace

asim_status asim_fail(asim_ctx* ctx, asim_status code, const std::string& msg) {
  if (ctx) ctx->err = msg;
  else g_create_err = msg;
  return code;
}

asim_status asim_cuda(asim_ctx* ctx, cudaError_t e, const char* what) {
  if (e == cudaSuccess) return ASIM_OK;
  if (ctx) ctx->broken = true;
  return asim_fail(ctx, ASIM_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

asim_status asim_ready(asim_ctx* ctx) {
  if (!ctx) return ASIM_EINVAL;
  if (ctx->broken) return asim_fail(ctx, ASIM_ECUDA, "context unusable after a CUDA error");
  if (!ctx->has_problem) return asim_fail(ctx, ASIM_ESTATE, "asim_set_problem not called");
  if (!ctx->has_trace) return asim_fail(ctx, ASIM_ESTATE, "asim_set_trace not called");
  // reading C20: every time the kernels form stays below 2^62
  const __int128 bound = (__int128)ctx->max_arrival + (__int128)ctx->n * ctx->hp.max_service;
  if (bound >= (__int128)kMaxTime)
    return asim_fail(ctx, ASIM_ERANGE, "max arrival + n * max service must stay below 2^62");
  return ASIM_OK;
}

asim_status asim_upload_batch(asim_ctx* ctx, const HostBatch& hb, cudaStream_t st) {
  ++ctx->batch_gen;  // chunked runs of earlier batches can no longer publish
  cudaError_t e = upload(ctx->d_base_cfg, hb.base_cfg, st);
  if (e == cudaSuccess) e = upload(ctx->d_base_mask, hb.base_mask, st);
  if (e == cudaSuccess) e = upload(ctx->d_cand_base, hb.cand_base, st);
  if (e == cudaSuccess) e = upload(ctx->d_cand_model, hb.cand_model, st);
  if (e == cudaSuccess) e = upload(ctx->d_cand_group, hb.cand_group, st);
  if (e == cudaSuccess) e = upload(ctx->d_cand_ok, hb.cand_ok, st);
  if (e == cudaSuccess && !hb.cand_kmask.empty()) e = upload(ctx->d_cand_kmask, hb.cand_kmask, st);
  if (e == cudaSuccess && !hb.cand_gmask.empty()) e = upload(ctx->d_cand_gmask, hb.cand_gmask, st);
  return asim_cuda(ctx, e, "upload batch");
}

asim_status asim_run_batch(asim_ctx* ctx, const HostBatch& hb, int64_t begin, int64_t end,
                           const asim::DevOut& out, cudaStream_t st, const ChunkOptions* opt,
                           bool* took_chunked) {
  const int64_t C = (int64_t)hb.cand_base.size();
  if (took_chunked) *took_chunked = false;
  if (end <= begin) return ASIM_OK;
  if (begin < 0 || end > C) return asim_fail(ctx, ASIM_ERANGE, "candidate range");
  asim_status us = asim_upload_batch(ctx, hb, st);
  if (us) return us;
  cudaError_t e = cudaSuccess;
  // Throughput path: candidates sharing a base placement, no per-model
  // counts -> chunked kernel (chunk.cu); otherwise the general kernel below.
  const bool shared_bases = (int64_t)(hb.base_cfg.size() / std::max<int32_t>(hb.G, 1)) < C ||
                            hb.G == 0;
  bool chunked = ctx->force_path >= 2 ||
                 (ctx->force_path == 0 && shared_bases && asim_chunked_eligible(ctx, hb, out));
  if (ctx->force_path >= 2 && !asim_chunked_eligible(ctx, hb, out)) chunked = false;
  // Component-restricted batches only exist on the chunked path, and a caller
  // passing ChunkOptions (the search) relies on the chunked run's boundary
  // states afterwards (candidate memory, publishing), so both force it.
  if (!hb.cand_kmask.empty() || (opt && ctx->force_path != 1)) {
    if (!asim_chunked_eligible(ctx, hb, out))
      return asim_fail(ctx, ASIM_ESTATE, "internal: restricted batch not chunk-eligible");
    chunked = true;
  }
  if (chunked) {
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    if (ctx->profiling) {
      if (cudaEventCreate(&ev0) != cudaSuccess || cudaEventCreate(&ev1) != cudaSuccess)
        return asim_cuda(ctx, cudaGetLastError(), "event create");
      cudaEventRecord(ev0, st);
    }
    asim::DevOut o2 = out;
    o2.stage_updates = ctx->profiling ? ctx->d_counter.as<unsigned long long>() : nullptr;
    asim_status s = (opt && opt->split && ctx->split_steps)
                        ? asim_run_chunked_split(ctx, hb, begin, end, *opt->split, o2, st, opt)
                        : asim_run_chunked(ctx, hb, begin, end, o2, st, opt);
    if (took_chunked) *took_chunked = s == ASIM_OK;
    if (ctx->profiling) {
      cudaEventRecord(ev1, st);
      ctx->events.emplace_back(ev0, ev1);
      ++ctx->sim_launches;
      int64_t ok = 0;
      for (int64_t i = begin; i < end; ++i) ok += hb.cand_ok[i];
      ctx->request_evals += ok * ctx->n;
    }
    return s;
  }
  // warp items: 32 consecutive candidates, cut where the base changes so a
  // warp shares one base placement (uniform hosting lists)
  std::vector<asim::WarpItem> items;
  int64_t c = begin;
  while (c < end) {
    int32_t cnt = 1;
    while (c + cnt < end && cnt < 32 && hb.cand_base[c + cnt] == hb.cand_base[c]) ++cnt;
    // full candidates (one base each): pack 32 per warp anyway
    if (cnt == 1) {
      while (c + cnt < end && cnt < 32 && hb.cand_base[c + cnt] != hb.cand_base[c + cnt - 1]) ++cnt;
    }
    items.push_back(asim::WarpItem{(int32_t)c, cnt});
    c += cnt;
  }
  e = upload(ctx->d_items, items, st);
  if (e != cudaSuccess) return asim_cuda(ctx, e, "upload items");
  asim::DevBatch b;
  b.G = hb.G;
  b.base_cfg = ctx->d_base_cfg.as<int32_t>();
  b.base_mask = ctx->d_base_mask.as<uint64_t>();
  b.cand_base = ctx->d_cand_base.as<int32_t>();
  b.cand_model = ctx->d_cand_model.as<int32_t>();
  b.cand_group = ctx->d_cand_group.as<int32_t>();
  b.cand_ok = ctx->d_cand_ok.as<uint8_t>();
  b.cand_kmask = nullptr;  // the general kernel simulates whole placements
  b.cand_gmask = nullptr;
  b.C = C;
  asim::DevOut o = out;
  o.stage_updates = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  if (ctx->profiling) {
    o.stage_updates = ctx->d_counter.as<unsigned long long>();
    if (cudaEventCreate(&ev0) != cudaSuccess || cudaEventCreate(&ev1) != cudaSuccess)
      return asim_cuda(ctx, cudaGetLastError(), "event create");
    cudaEventRecord(ev0, st);
  }
  e = asim::launch_simulate(ctx->dev_problem(), ctx->dev_trace(), b,
                            ctx->d_items.as<asim::WarpItem>(), (int32_t)items.size(), hb.slots,
                            o, st, &ctx->launches);
  if (ctx->profiling) {
    cudaEventRecord(ev1, st);
    ctx->events.emplace_back(ev0, ev1);
    ++ctx->sim_launches;
    int64_t ok = 0;
    for (int64_t i = begin; i < end; ++i) ok += hb.cand_ok[i];
    ctx->request_evals += ok * ctx->n;
  }
  return asim_cuda(ctx, e, "simulate kernel");
}

extern "C" {

int32_t asim_abi_version(void) { return ASIM_ABI_VERSION; }

asim_status asim_create(int32_t cuda_device, asim_ctx** out) {
  if (!out) return asim_fail(nullptr, ASIM_EINVAL, "null out");
  *out = nullptr;
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0)
    return asim_fail(nullptr, ASIM_ECUDA,
                     std::string("no CUDA device: ") + cudaGetErrorString(e));
  if (cuda_device < 0 || cuda_device >= count)
    return asim_fail(nullptr, ASIM_EINVAL, "cuda_device out of range");
  cudaDeviceProp prop;
  e = cudaGetDeviceProperties(&prop, cuda_device);
  if (e != cudaSuccess)
    return asim_fail(nullptr, ASIM_ECUDA, std::string("cudaGetDeviceProperties: ") +
                                              cudaGetErrorString(e));
  if (prop.major != 10 || prop.minor != 0)
    return asim_fail(nullptr, ASIM_EINVAL, "libasim.so is built for sm_100a (B200) only");
  asim_ctx* ctx = new (std::nothrow) asim_ctx();
  if (!ctx) return asim_fail(nullptr, ASIM_ENOMEM, "host allocation failed");
  ctx->device = cuda_device;
  ctx->sms = prop.multiProcessorCount;
  if (const char* sw = getenv("ASIM_SCALAR_WALK")) ctx->scalar_walk = sw[0] != '0';
  if (const char* wl = getenv("ASIM_WALK_LOG")) ctx->walk_log = atoll(wl);
  if (const char* gw = getenv("ASIM_GLANE_WALK")) ctx->glane_walk = atoi(gw);
  if (const char* gs = getenv("ASIM_GLANE_SMAX")) ctx->glane_smax = atoi(gs);
  if (const char* gc = getenv("ASIM_GROUP_CANDIDATES")) ctx->group_cands = gc[0] != '0';
  if (const char* sp = getenv("ASIM_SPLIT")) ctx->split_steps = sp[0] != '0';
  if (const char* mc = getenv("ASIM_MAX_CHUNKS")) ctx->max_chunks = std::max(1ll, atoll(mc));
  {
    DeviceGuard dg(cuda_device);
    int lo = 0, hi = 0;  // stream priorities: `hi` is the most urgent
    e = cudaDeviceGetStreamPriorityRange(&lo, &hi);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->ev_split, cudaEventDisableTiming);
    for (int k = 0; k < kChunkSlots && e == cudaSuccess; ++k) {
      ChunkSlot& cs = ctx->slot[k];
      const int prio = k == 0 ? hi : lo;  // slot 0 carries the walk-prone candidates
      e = cudaStreamCreateWithPriority(&cs.main, cudaStreamNonBlocking, prio);
      for (int i = 0; i < 2 && e == cudaSuccess; ++i) {
        e = cudaStreamCreateWithPriority(&cs.side[i], cudaStreamNonBlocking, prio);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&cs.ev_join[i], cudaEventDisableTiming);
      }
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&cs.ev_fork, cudaEventDisableTiming);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&cs.ev_done, cudaEventDisableTiming);
    }
    if (e != cudaSuccess) {
      asim_destroy(ctx);
      return asim_fail(nullptr, ASIM_ECUDA, std::string("side streams: ") + cudaGetErrorString(e));
    }
  }
  *out = ctx;
  return ASIM_OK;
}

void asim_destroy(asim_ctx* ctx) {
  if (!ctx) return;
  asim_reset_stats(ctx);
  {
    DeviceGuard dg(ctx->device);
    DBuf* bufs[] = {&ctx->d_stage, &ctx->d_tail, &ctx->d_slo, &ctx->d_cfg_stages,
                    &ctx->d_dtab32, &ctx->d_dtab64,
                    &ctx->d_arrival, &ctx->d_model, &ctx->d_moff, &ctx->d_midx, &ctx->d_inc,
                    &ctx->d_order, &ctx->d_mcum, &ctx->d_base_cfg, &ctx->d_base_mask,
                    &ctx->d_cand_base, &ctx->d_cand_model, &ctx->d_cand_group, &ctx->d_cand_ok,
                    &ctx->d_items, &ctx->d_good, &ctx->d_sum, &ctx->d_pm, &ctx->d_busy,
                    &ctx->d_argmax, &ctx->d_counter, &ctx->d_cand_kmask, &ctx->d_cand_gmask};
    for (DBuf* b : bufs) b->release();
    for (DBuf& b : ctx->spool) b.release();
    auto sdestroy = [](cudaStream_t& x) { if (x) cudaStreamDestroy(x); x = nullptr; };
    auto edestroy = [](cudaEvent_t& x) { if (x) cudaEventDestroy(x); x = nullptr; };
    for (ChunkSlot& cs : ctx->slot) {
      for (DBuf* b : cs.bufs()) b->release();
      sdestroy(cs.main);
      for (int i = 0; i < 2; ++i) {
        sdestroy(cs.side[i]);
        edestroy(cs.ev_join[i]);
      }
      edestroy(cs.ev_fork);
      edestroy(cs.ev_done);
    }
    edestroy(ctx->ev_split);
    edestroy(ctx->ev_ref);
  }
  delete ctx;
}

const char* asim_last_error(const asim_ctx* ctx) {
  return ctx ? ctx->err.c_str() : g_create_err.c_str();
}

int64_t asim_launch_count(const asim_ctx* ctx) { return ctx ? ctx->launches : 0; }

// Reference event for the phase intervals: recorded, then the device drained,
// so every later event's elapsed time from it is >= 0.
static cudaError_t record_ref(asim_ctx* ctx) {
  cudaError_t e = ctx->ev_ref ? cudaSuccess : cudaEventCreate(&ctx->ev_ref);
  if (e == cudaSuccess) e = cudaEventRecord(ctx->ev_ref, 0);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  return e;
}

// Length of the union of intervals (ms).
static double union_ms(std::vector<std::pair<double, double>> iv) {
  std::sort(iv.begin(), iv.end());
  double total = 0.0, a = 0.0, b = -1.0;
  for (const auto& x : iv) {
    if (x.first > b) {
      if (b > a) total += b - a;
      a = x.first;
      b = x.second;
    } else if (x.second > b) {
      b = x.second;
    }
  }
  if (b > a) total += b - a;
  return total;
}

asim_status asim_reset_stats(asim_ctx* ctx) {
  if (!ctx) return ASIM_EINVAL;
  DeviceGuard dg(ctx->device);
  for (auto* evs : {&ctx->events, &ctx->phase_events[0], &ctx->phase_events[1],
                    &ctx->phase_events[2]}) {
    for (auto& ev : *evs) {
      cudaEventSynchronize(ev.second);
      cudaEventDestroy(ev.first);
      cudaEventDestroy(ev.second);
    }
    evs->clear();
  }
  ctx->sim_launches = 0;
  ctx->sim_ms = 0.0;
  for (double& x : ctx->phase_ms) x = 0.0;
  for (auto& v : ctx->phase_iv) v.clear();
  ctx->p1_updates = ctx->p1_live = ctx->p1_slots = 0;
  for (auto& r : ctx->p1_class) r[0] = r[1] = 0;
  for (int64_t& x : ctx->walk_pred) x = 0;
  ctx->request_evals = 0;
  if (ctx->d_counter.p) {
    cudaError_t e = cudaMemset(ctx->d_counter.p, 0, 32);
    for (ChunkSlot& cs : ctx->slot)
      if (e == cudaSuccess) e = cudaMemset(cs.walked.p, 0, kWalkedBytes);
    if (e == cudaSuccess) e = record_ref(ctx);
    if (e != cudaSuccess) return asim_cuda(ctx, e, "reset stats");
  }
  return ASIM_OK;
}

asim_status asim_set_path(asim_ctx* ctx, int32_t path) {
  if (!ctx) return ASIM_EINVAL;
  if (path < 0 || path > 3) return asim_fail(ctx, ASIM_EINVAL, "path must be 0..3");
  ctx->force_path = path;
  return ASIM_OK;
}

asim_status asim_set_chunk_size(asim_ctx* ctx, int64_t min_requests) {
  if (!ctx) return ASIM_EINVAL;
  if (min_requests < 1) return asim_fail(ctx, ASIM_ERANGE, "min_requests must be >= 1");
  ctx->min_chunk = min_requests;
  return ASIM_OK;
}

asim_status asim_set_profiling(asim_ctx* ctx, int32_t on) {
  if (!ctx) return ASIM_EINVAL;
  DeviceGuard dg(ctx->device);
  if (on && !ctx->d_counter.p) {
    cudaError_t e = ctx->d_counter.ensure(32);
    if (e == cudaSuccess) e = cudaMemset(ctx->d_counter.p, 0, 32);
    for (ChunkSlot& cs : ctx->slot) {
      if (e == cudaSuccess) e = cs.walked.ensure(kWalkedBytes);
      if (e == cudaSuccess) e = cudaMemset(cs.walked.p, 0, kWalkedBytes);
    }
    if (e == cudaSuccess) e = record_ref(ctx);
    if (e != cudaSuccess) return asim_cuda(ctx, e, "profiling counter");
  }
  ctx->profiling = on != 0;
  return ASIM_OK;
}

asim_status asim_get_stats(asim_ctx* ctx, asim_stats* out) {
  if (!ctx || !out) return ASIM_EINVAL;
  DeviceGuard dg(ctx->device);
  for (auto& ev : ctx->events) {
    cudaError_t e = cudaEventSynchronize(ev.second);
    float ms = 0.f;
    if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, ev.first, ev.second);
    if (e != cudaSuccess) return asim_cuda(ctx, e, "stats events");
    ctx->sim_ms += ms;
    cudaEventDestroy(ev.first);
    cudaEventDestroy(ev.second);
  }
  ctx->events.clear();
  for (int ph = 0; ph < 3; ++ph) {
    for (auto& ev : ctx->phase_events[ph]) {
      cudaError_t e = cudaEventSynchronize(ev.second);
      float ms = 0.f;
      if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, ev.first, ev.second);
      if (e != cudaSuccess) return asim_cuda(ctx, e, "stats events");
      ctx->phase_ms[ph] += ms;
      float t0 = 0.f, t1 = 0.f;
      if (ctx->ev_ref && cudaEventElapsedTime(&t0, ctx->ev_ref, ev.first) == cudaSuccess &&
          cudaEventElapsedTime(&t1, ctx->ev_ref, ev.second) == cudaSuccess)
        ctx->phase_iv[ph].emplace_back(t0, t1);
      cudaEventDestroy(ev.first);
      cudaEventDestroy(ev.second);
    }
    ctx->phase_events[ph].clear();
  }
  constexpr int kW = kWalkedBytes / 8;
  unsigned long long upd2[4] = {0, 0, 0, 0}, walked[kW] = {};
  if (ctx->d_counter.p) {
    cudaError_t e = cudaMemcpy(upd2, ctx->d_counter.p, 32, cudaMemcpyDeviceToHost);
    for (ChunkSlot& cs : ctx->slot) {
      unsigned long long w[kW] = {};
      if (e == cudaSuccess && cs.walked.p)
        e = cudaMemcpy(w, cs.walked.p, kWalkedBytes, cudaMemcpyDeviceToHost);
      for (int i = 0; i < kW; ++i) walked[i] += w[i];
    }
    if (e != cudaSuccess) return asim_cuda(ctx, e, "stats counter");
  }
  out->launches = ctx->launches;
  out->sim_launches = ctx->sim_launches;
  out->sim_ms = ctx->sim_ms;
  out->stage_updates = (int64_t)upd2[0] + ctx->p1_updates;
  out->spec_stage_updates = ctx->p1_updates;
  out->spec_ms = ctx->phase_ms[0];
  out->pass2_ms = ctx->phase_ms[1];
  out->walk_ms = ctx->phase_ms[2];
  out->spec_busy_ms = union_ms(ctx->phase_iv[0]);
  out->pass2_busy_ms = union_ms(ctx->phase_iv[1]);
  out->walk_busy_ms = union_ms(ctx->phase_iv[2]);
  out->spec_lane_slots = ctx->p1_slots;
  out->spec_live_lanes = ctx->p1_live;
  out->walk_predicted = ctx->walk_pred[0];
  out->walk_unpredicted = ctx->walk_pred[1];
  out->walk_mispredicted = ctx->walk_pred[2];
  out->request_evals = ctx->request_evals;
  out->chunk_reruns = (int64_t)walked[0];
  out->walk_candidates = (int64_t)walked[1];
  out->walk_critical_chunks = (int64_t)walked[3];
  for (int i = 0; i < 6; ++i) {
    out->spec_class_cycles[i] = (int64_t)walked[4 + i];
    out->spec_class_updates[i] = ctx->p1_class[i][0];
    out->spec_class_slots[i] = ctx->p1_class[i][1];
  }
  return ASIM_OK;
}

double asim_attainment(int64_t good, int64_t n) {
  if (good < 0) return -1.0;
  if (n == 0) return 1.0;
  return (double)good / (double)n;
}

asim_status asim_argmax(asim_ctx* ctx, const int64_t* good, int64_t n, int32_t ptr_kind,
                        int64_t* out, void* cuda_stream) {
  if (!ctx) return ASIM_EINVAL;
  if (ctx->broken) return asim_fail(ctx, ASIM_ECUDA, "context unusable after a CUDA error");
  if (!out || (n > 0 && !good)) return asim_fail(ctx, ASIM_EINVAL, "null good / out");
  if (n < 0) return asim_fail(ctx, ASIM_ERANGE, "n < 0");
  if (ptr_kind != ASIM_HOST && ptr_kind != ASIM_DEVICE)
    return asim_fail(ctx, ASIM_EINVAL, "bad ptr_kind");
  DeviceGuard dg(ctx->device);
  cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
  const int64_t* g = good;
  cudaError_t e = ctx->d_argmax.ensure(8);
  if (e == cudaSuccess && ptr_kind == ASIM_HOST && n > 0) {
    e = ctx->d_good.ensure((size_t)n * 8);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(ctx->d_good.p, good, (size_t)n * 8, cudaMemcpyHostToDevice, st);
    g = ctx->d_good.as<int64_t>();
  }
  if (e == cudaSuccess) e = asim::launch_argmax(g, n, ctx->d_argmax.as<int64_t>(), st, &ctx->launches);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(out, ctx->d_argmax.p, 8, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  return asim_cuda(ctx, e, "argmax");
}

asim_status asim_set_problem(asim_ctx* ctx, const asim_problem* p) {
  if (!ctx) return ASIM_EINVAL;
  if (ctx->broken) return asim_fail(ctx, ASIM_ECUDA, "context unusable after a CUDA error");
  if (!p) return asim_fail(ctx, ASIM_EINVAL, "null problem");
  if (p->num_models < 1 || p->num_models > ASIM_MAX_MODELS)
    return asim_fail(ctx, ASIM_ERANGE, "num_models out of range");
  if (p->num_configs < 1 || p->num_configs > 65535)
    return asim_fail(ctx, ASIM_ERANGE, "num_configs out of range");
  if (p->max_stages < 1 || p->max_stages > ASIM_MAX_STAGES)
    return asim_fail(ctx, ASIM_ERANGE, "max_stages out of range");
  if (!p->slo_ns || !p->cfg_stages || !p->cfg_devices || !p->stage_ns || !p->tail_ns ||
      !p->mem_bytes)
    return asim_fail(ctx, ASIM_EINVAL, "null problem array");
  if (p->num_devices < 1 || p->device_budget_bytes < 0)
    return asim_fail(ctx, ASIM_ERANGE, "num_devices / budget out of range");
  HostProblem hp;
  hp.M = p->num_models;
  hp.P = p->num_configs;
  hp.S = p->max_stages;
  const int64_t M = hp.M, P = hp.P, S = hp.S;
  hp.slo.assign(p->slo_ns, p->slo_ns + M);
  hp.cfg_stages.assign(p->cfg_stages, p->cfg_stages + P);
  hp.cfg_devices.assign(p->cfg_devices, p->cfg_devices + P);
  hp.stage.assign(p->stage_ns, p->stage_ns + M * P * S);
  hp.tail.assign(p->tail_ns, p->tail_ns + M * P);
  hp.mem.assign(p->mem_bytes, p->mem_bytes + M * P);
  hp.num_devices = p->num_devices;
  hp.budget = p->device_budget_bytes;
  for (int64_t m = 0; m < M; ++m)
    if (hp.slo[m] < 0) return asim_fail(ctx, ASIM_ERANGE, "slo_ns must be >= 0");
  for (int64_t c = 0; c < P; ++c) {
    if (hp.cfg_stages[c] < 1 || hp.cfg_stages[c] > S)
      return asim_fail(ctx, ASIM_ERANGE, "cfg_stages out of range");
    if (hp.cfg_devices[c] < 1) return asim_fail(ctx, ASIM_ERANGE, "cfg_devices must be >= 1");
  }
  hp.max_service = 0;
  for (int64_t m = 0; m < M; ++m)
    for (int64_t c = 0; c < P; ++c) {
      __int128 tot = hp.tail[m * P + c];
      if (hp.tail[m * P + c] < 0) return asim_fail(ctx, ASIM_ERANGE, "tail_ns must be >= 0");
      for (int64_t k = 0; k < S; ++k) {
        const int64_t d = hp.stage[(m * P + c) * S + k];
        if (d < 0) return asim_fail(ctx, ASIM_ERANGE, "stage_ns must be >= 0");
        if (k < hp.cfg_stages[c]) tot += d;
      }
      if (tot > kMaxService)
        return asim_fail(ctx, ASIM_ERANGE, "sum of stages + tail must be <= 2^60");
      hp.max_service = std::max<int64_t>(hp.max_service, (int64_t)tot);
    }
  DeviceGuard dg(ctx->device);
  cudaError_t e = upload(ctx->d_stage, hp.stage, 0);
  if (e == cudaSuccess) e = upload(ctx->d_tail, hp.tail, 0);
  if (e == cudaSuccess) e = upload(ctx->d_slo, hp.slo, 0);
  if (e == cudaSuccess) e = upload(ctx->d_cfg_stages, hp.cfg_stages, 0);
  {
    // per-config stage-latency rows for the passes (read through L1)
    std::vector<uint32_t> t32((size_t)P * M * 16, 0u);
    std::vector<int64_t> t64((size_t)P * M * 16, 0);
    for (int64_t c = 0; c < P; ++c)
      for (int64_t m = 0; m < M; ++m)
        for (int64_t k = 0; k < std::min<int64_t>(S, 16); ++k) {
          if (k >= hp.cfg_stages[c]) continue;
          const int64_t d = hp.stage[(m * P + c) * S + k];
          t64[(c * M + m) * 16 + k] = d;
          t32[(c * M + m) * 16 + k] = d >= 0xFFFFFFFFll ? 0xFFFFFFFFu : (uint32_t)d;
        }
    if (e == cudaSuccess) e = upload(ctx->d_dtab32, t32, 0);
    if (e == cudaSuccess) e = upload(ctx->d_dtab64, t64, 0);
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(0);
  if (e != cudaSuccess) return asim_cuda(ctx, e, "upload problem");
  // a trace set for another model count must be set again
  if (ctx->has_trace && hp.M != ctx->hp.M) ctx->has_trace = false;
  ctx->hp = std::move(hp);
  ctx->has_problem = true;
  return ASIM_OK;
}

asim_status asim_set_trace(asim_ctx* ctx, int64_t n, const int64_t* arrival_ns,
                           const int32_t* model, int32_t ptr_kind, void* cuda_stream) {
  if (!ctx) return ASIM_EINVAL;
  if (ctx->broken) return asim_fail(ctx, ASIM_ECUDA, "context unusable after a CUDA error");
  if (!ctx->has_problem) return asim_fail(ctx, ASIM_ESTATE, "asim_set_problem not called");
  if (n < 0 || n > (int64_t(1) << 31) - 1) return asim_fail(ctx, ASIM_ERANGE, "n out of range");
  DeviceGuard dg(ctx->device);
  cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
  std::vector<int64_t> a;
  std::vector<int32_t> m;
  asim_status s = fetch(ctx, a, arrival_ns, n, ptr_kind, st, "arrival_ns");
  if (s) return s;
  s = fetch(ctx, m, model, n, ptr_kind, st, "model");
  if (s) return s;
  for (int64_t i = 0; i < n; ++i) {
    if (a[i] < 0) return asim_fail(ctx, ASIM_EUNSORTED, "negative arrival");
    if (i && a[i] < a[i - 1]) return asim_fail(ctx, ASIM_EUNSORTED, "trace not sorted by arrival");
    if (m[i] < 0 || m[i] >= ctx->hp.M) return asim_fail(ctx, ASIM_ERANGE, "model id out of range");
  }
  if (n && a[n - 1] > kMaxTime) return asim_fail(ctx, ASIM_ERANGE, "arrival > 2^62");
  // pad to a multiple of 32 requests plus a look-ahead margin of 256 records
  // (chunk.cu prefetches 4 tiles ahead); sentinel model 0xFFFF is never hosted
  const int64_t npad = (n + 31) / 32 * 32 + 256;
  std::vector<int64_t> ap(npad, n ? a[n - 1] : 0);
  std::vector<uint16_t> mp(npad, 0xFFFF);
  for (int64_t i = 0; i < n; ++i) {
    ap[i] = a[i];
    mp[i] = (uint16_t)m[i];
  }
  cudaError_t e = upload(ctx->d_arrival, ap, st);
  if (e == cudaSuccess) e = upload(ctx->d_model, mp, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return asim_cuda(ctx, e, "upload trace");
  ctx->n = n;
  ctx->max_arrival = n ? a[n - 1] : 0;
  ctx->min_arrival = n ? a[0] : 0;
  ctx->model_n.assign(ctx->hp.M, 0);
  for (int64_t i = 0; i < n; ++i) ++ctx->model_n[m[i]];
  ctx->has_midx = false;  // built on the first batching call
  ctx->has_trace = true;
  return ASIM_OK;
}

static asim_status evaluate_batch(asim_ctx* ctx, HostBatch& hb, asim_results* out,
                                  cudaStream_t st) {
  if (!out || !out->good) return asim_fail(ctx, ASIM_EINVAL, "null results / good");
  if (out->ptr_kind != ASIM_HOST && out->ptr_kind != ASIM_DEVICE)
    return asim_fail(ctx, ASIM_EINVAL, "bad results ptr_kind");
  const int64_t C = (int64_t)hb.cand_base.size();
  const int64_t M = ctx->hp.M;
  const bool want_sum = out->sum_latency_ns != nullptr;
  const bool want_pm = out->good_per_model != nullptr;
  const bool want_arg = out->argmax != nullptr;
  const bool want_busy = out->busy_ns != nullptr;
  const int32_t G = hb.G;
  asim::DevOut dout{};
  dout.out_offset = 0;
  dout.stage_updates = nullptr;
  cudaError_t e = cudaSuccess;
  if (out->ptr_kind == ASIM_DEVICE) {
    dout.good = out->good;
    dout.sum_latency = out->sum_latency_ns;
    dout.good_per_model = out->good_per_model;
    dout.busy = out->busy_ns;
  } else {
    e = ctx->d_good.ensure(C * 8 + 8);
    if (e == cudaSuccess && want_sum) e = ctx->d_sum.ensure(C * 8 + 8);
    if (e == cudaSuccess && want_pm) e = ctx->d_pm.ensure(C * M * 8 + 8);
    if (e == cudaSuccess && want_busy) e = ctx->d_busy.ensure(C * G * 8 + 8);
    if (e != cudaSuccess) return asim_cuda(ctx, e, "allocate results");
    dout.good = ctx->d_good.as<int64_t>();
    dout.sum_latency = want_sum ? ctx->d_sum.as<int64_t>() : nullptr;
    dout.good_per_model = want_pm ? ctx->d_pm.as<int64_t>() : nullptr;
    dout.busy = want_busy ? ctx->d_busy.as<int64_t>() : nullptr;
  }
  if (want_pm && C > 0) {
    e = cudaMemsetAsync(dout.good_per_model, 0, C * M * 8, st);
    if (e != cudaSuccess) return asim_cuda(ctx, e, "memset per-model");
  }
  if (want_busy && C * G > 0) {
    e = cudaMemsetAsync(dout.busy, 0, C * G * 8, st);
    if (e != cudaSuccess) return asim_cuda(ctx, e, "memset busy");
  }
  asim_status s = asim_run_batch(ctx, hb, 0, C, dout, st);
  if (s) return s;
  if (want_arg) {
    e = ctx->d_argmax.ensure(8);
    int64_t* arg_dev = out->ptr_kind == ASIM_DEVICE ? out->argmax : ctx->d_argmax.as<int64_t>();
    if (e == cudaSuccess) e = asim::launch_argmax(dout.good, C, arg_dev, st, &ctx->launches);
    if (e != cudaSuccess) return asim_cuda(ctx, e, "argmax kernel");
  }
  return finish_outputs(ctx, out, C, G, want_sum, want_pm, want_busy, want_arg, st);
}

asim_status asim_evaluate(asim_ctx* ctx, const asim_candidates* cands, asim_results* out,
                          void* cuda_stream) {
  asim_status s = asim_ready(ctx);
  if (s) return s;
  if (!cands) return asim_fail(ctx, ASIM_EINVAL, "null candidates");
  const int64_t C = cands->num_candidates;
  const int32_t G = cands->max_groups;
  const int64_t M = ctx->hp.M;
  if (C < 0 || C > (int64_t(1) << 31) - 64) return asim_fail(ctx, ASIM_ERANGE, "num_candidates");
  if (G < 0 || G > ASIM_MAX_GROUPS) return asim_fail(ctx, ASIM_ERANGE, "max_groups out of range");
  DeviceGuard dg(ctx->device);
  cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
  HostBatch hb;
  hb.G = G;
  s = fetch(ctx, hb.base_cfg, cands->group_cfg, C * G, cands->ptr_kind, st, "group_cfg");
  if (s) return s;
  s = fetch(ctx, hb.base_mask, cands->host_mask, C * M, cands->ptr_kind, st, "host_mask");
  if (s) return s;
  hb.cand_base.resize(C);
  hb.cand_model.assign(C, -1);
  hb.cand_group.assign(C, 0);
  hb.cand_ok.resize(C);
  std::vector<int64_t> used;
  for (int64_t c = 0; c < C; ++c) {
    bool ok = false;
    s = check_base(ctx, hb.base_cfg.data() + c * G, hb.base_mask.data() + c * M, G, used, &ok,
                   &hb.slots);
    if (s) return s;
    hb.cand_base[c] = (int32_t)c;
    hb.cand_ok[c] = ok ? 1 : 0;
  }
  return evaluate_batch(ctx, hb, out, st);
}

asim_status asim_evaluate_batching(asim_ctx* ctx, const asim_candidates* cands,
                                   const asim_batching* opt, asim_results* out,
                                   void* cuda_stream) {
  asim_status s = asim_ready(ctx);
  if (s) return s;
  if (!cands || !opt) return asim_fail(ctx, ASIM_EINVAL, "null candidates / batching options");
  if (!opt->stage_inc_ns) return asim_fail(ctx, ASIM_EINVAL, "null stage_inc_ns");
  if (!out || !out->good) return asim_fail(ctx, ASIM_EINVAL, "null results / good");
  if (out->busy_ns) return asim_fail(ctx, ASIM_EINVAL, "busy_ns is not produced with batching");
  if (out->ptr_kind != ASIM_HOST && out->ptr_kind != ASIM_DEVICE)
    return asim_fail(ctx, ASIM_EINVAL, "bad results ptr_kind");
  const HostProblem& hp = ctx->hp;
  const int64_t M = hp.M, P = hp.P, S = hp.S;
  if (M > 64) return asim_fail(ctx, ASIM_ERANGE, "batching supports at most 64 models");
  if (opt->max_batch < 1 || opt->max_batch > (1 << 20))
    return asim_fail(ctx, ASIM_ERANGE, "max_batch must be in [1, 2^20]");
  const int64_t C = cands->num_candidates;
  const int32_t G = cands->max_groups;
  if (C < 0 || C > (int64_t(1) << 31) - 64) return asim_fail(ctx, ASIM_ERANGE, "num_candidates");
  if (G < 0 || G > ASIM_MAX_GROUPS) return asim_fail(ctx, ASIM_ERANGE, "max_groups out of range");
  // increments, first-stage latency >= 1 ns (C33), and the time bound of
  // reading C20 with every service at its largest batch
  std::vector<int64_t> inc(opt->stage_inc_ns, opt->stage_inc_ns + M * P * S);
  int64_t max_service = 0;
  for (int64_t m = 0; m < M; ++m)
    for (int64_t p = 0; p < P; ++p) {
      if (hp.stage[(m * P + p) * S] < 1)
        return asim_fail(ctx, ASIM_ERANGE, "batching needs a first-stage latency >= 1 ns");
      __int128 tot = hp.tail[m * P + p];
      for (int64_t k = 0; k < S; ++k) {
        const int64_t x = inc[(m * P + p) * S + k];
        if (x < 0) return asim_fail(ctx, ASIM_ERANGE, "stage_inc_ns must be >= 0");
        if (k < hp.cfg_stages[p])
          tot += (__int128)hp.stage[(m * P + p) * S + k] + (__int128)(opt->max_batch - 1) * x;
      }
      if (tot > kMaxService)
        return asim_fail(ctx, ASIM_ERANGE, "batched stages + tail must be <= 2^60");
      max_service = std::max<int64_t>(max_service, (int64_t)tot);
    }
  if ((__int128)ctx->max_arrival + (__int128)ctx->n * max_service >= (__int128)kMaxTime)
    return asim_fail(ctx, ASIM_ERANGE, "max arrival + n * max batched service must stay below 2^62");
  DeviceGuard dg(ctx->device);
  cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
  HostBatch hb;
  hb.G = G;
  s = fetch(ctx, hb.base_cfg, cands->group_cfg, C * G, cands->ptr_kind, st, "group_cfg");
  if (s) return s;
  s = fetch(ctx, hb.base_mask, cands->host_mask, C * M, cands->ptr_kind, st, "host_mask");
  if (s) return s;
  hb.cand_base.resize(C);
  hb.cand_model.assign(C, -1);
  hb.cand_group.assign(C, 0);
  hb.cand_ok.resize(C);
  std::vector<int64_t> used;
  for (int64_t c = 0; c < C; ++c) {
    bool ok = false;
    s = check_base(ctx, hb.base_cfg.data() + c * G, hb.base_mask.data() + c * M, G, used, &ok,
                   &hb.slots);
    if (s) return s;
    hb.cand_base[c] = (int32_t)c;
    hb.cand_ok[c] = ok ? 1 : 0;
  }
  const size_t smem = 4 * asim::batching_smem_per_warp(hb.slots, G, (int32_t)M);
  if (smem > 227 * 1024) return asim_fail(ctx, ASIM_ERANGE, "placement too large for batching");
  const bool want_sum = out->sum_latency_ns != nullptr;
  const bool want_pm = out->good_per_model != nullptr;
  const bool want_arg = out->argmax != nullptr;
  asim::DevOut dout{};
  cudaError_t e = upload(ctx->d_inc, inc, st);
  if (e != cudaSuccess) return asim_cuda(ctx, e, "upload increments");
  if (!ctx->has_midx) {  // per-model request lists (CSR, ascending trace index)
    const int64_t n = ctx->n;
    std::vector<uint16_t> mh(n > 0 ? n : 1);
    if (n > 0) e = cudaMemcpy(mh.data(), ctx->d_model.p, n * 2, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return asim_cuda(ctx, e, "download trace models");
    std::vector<int32_t> moff(M + 1, 0), midx(n > 0 ? n : 1, 0);
    for (int64_t i = 0; i < n; ++i) ++moff[mh[i] + 1];
    for (int64_t k = 0; k < M; ++k) moff[k + 1] += moff[k];
    std::vector<int32_t> fill(moff.begin(), moff.end() - 1);
    for (int64_t i = 0; i < n; ++i) midx[fill[mh[i]]++] = (int32_t)i;
    // running arrival sums per model (mod 2^64): model m's block starts at
    // moff[m] + m and has moff[m+1] - moff[m] + 1 entries
    std::vector<int64_t> arr(n > 0 ? n : 1);
    if (n > 0) e = cudaMemcpy(arr.data(), ctx->d_arrival.p, n * 8, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return asim_cuda(ctx, e, "download trace arrivals");
    std::vector<uint64_t> mcum(n + M, 0);
    for (int64_t k = 0; k < M; ++k) {
      uint64_t acc = 0;
      const int64_t b0 = moff[k] + k;
      mcum[b0] = 0;
      for (int64_t i = moff[k]; i < moff[k + 1]; ++i) {
        acc += (uint64_t)arr[midx[i]];
        mcum[b0 + (i - moff[k]) + 1] = acc;
      }
    }
    e = upload(ctx->d_moff, moff, st);
    if (e == cudaSuccess) e = upload(ctx->d_midx, midx, st);
    if (e == cudaSuccess) e = upload(ctx->d_mcum, mcum, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return asim_cuda(ctx, e, "upload per-model request lists");
    ctx->has_midx = true;
  }
  if (out->ptr_kind == ASIM_DEVICE) {
    dout.good = out->good;
    dout.sum_latency = out->sum_latency_ns;
    dout.good_per_model = out->good_per_model;
  } else {
    e = ctx->d_good.ensure(C * 8 + 8);
    if (e == cudaSuccess && want_sum) e = ctx->d_sum.ensure(C * 8 + 8);
    if (e == cudaSuccess && want_pm) e = ctx->d_pm.ensure(C * M * 8 + 8);
    if (e != cudaSuccess) return asim_cuda(ctx, e, "allocate results");
    dout.good = ctx->d_good.as<int64_t>();
    dout.sum_latency = want_sum ? ctx->d_sum.as<int64_t>() : nullptr;
    dout.good_per_model = want_pm ? ctx->d_pm.as<int64_t>() : nullptr;
  }
  if (want_pm && C > 0) {
    e = cudaMemsetAsync(dout.good_per_model, 0, C * M * 8, st);
    if (e != cudaSuccess) return asim_cuda(ctx, e, "memset per-model");
  }
  s = asim_upload_batch(ctx, hb, st);
  if (s) return s;
  asim::DevBatch b;
  b.G = G;
  b.base_cfg = ctx->d_base_cfg.as<int32_t>();
  b.base_mask = ctx->d_base_mask.as<uint64_t>();
  b.cand_base = ctx->d_cand_base.as<int32_t>();
  b.cand_model = ctx->d_cand_model.as<int32_t>();
  b.cand_group = ctx->d_cand_group.as<int32_t>();
  b.cand_ok = ctx->d_cand_ok.as<uint8_t>();
  b.cand_kmask = nullptr;
  b.cand_gmask = nullptr;
  b.C = C;
  // launch order: longest-processing-time first, so the second wave of
  // warps fills in behind the slow candidates instead of leaving a tail;
  // estimated cost = sum over hosted models of requests x stages of the group
  {
    std::vector<int64_t> cost(C, 0);
    for (int64_t c = 0; c < C; ++c) {
      if (!hb.cand_ok[c]) continue;
      for (int64_t m = 0; m < M; ++m) {
        uint64_t w = hb.base_mask[c * M + m];
        while (w) {
          const int g = __builtin_ctzll(w);
          w &= w - 1;
          cost[c] += ctx->model_n[m] * hp.cfg_stages[hb.base_cfg[c * G + g]];
        }
      }
    }
    std::vector<int32_t> order(C);
    for (int64_t c = 0; c < C; ++c) order[c] = (int32_t)c;
    std::stable_sort(order.begin(), order.end(),
                     [&](int32_t x, int32_t y) { return cost[x] > cost[y]; });
    e = upload(ctx->d_order, order, st);
    if (e != cudaSuccess) return asim_cuda(ctx, e, "upload launch order");
  }
  asim::DevBatching bp;
  bp.order = ctx->d_order.as<int32_t>();
  bp.mcum = ctx->d_mcum.as<uint64_t>();
  bp.max_batch = opt->max_batch;
  bp.inc = ctx->d_inc.as<int64_t>();
  bp.moff = ctx->d_moff.as<int32_t>();
  bp.midx = ctx->d_midx.as<int32_t>();
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  if (ctx->profiling) {
    dout.stage_updates = ctx->d_counter.as<unsigned long long>();
    if (cudaEventCreate(&ev0) != cudaSuccess || cudaEventCreate(&ev1) != cudaSuccess)
      return asim_cuda(ctx, cudaGetLastError(), "event create");
    cudaEventRecord(ev0, st);
  }
  e = asim::launch_batching(ctx->dev_problem(), ctx->dev_trace(), b, bp, hb.slots, dout, st,
                            &ctx->launches);
  if (e != cudaSuccess) return asim_cuda(ctx, e, "batching kernel");
  if (ctx->profiling) {
    cudaEventRecord(ev1, st);
    ctx->events.emplace_back(ev0, ev1);
    ++ctx->sim_launches;
    int64_t ok = 0;
    for (int64_t i = 0; i < C; ++i) ok += hb.cand_ok[i];
    ctx->request_evals += ok * ctx->n;
  }
  if (want_arg) {
    e = ctx->d_argmax.ensure(8);
    int64_t* arg_dev = out->ptr_kind == ASIM_DEVICE ? out->argmax : ctx->d_argmax.as<int64_t>();
    if (e == cudaSuccess) e = asim::launch_argmax(dout.good, C, arg_dev, st, &ctx->launches);
    if (e != cudaSuccess) return asim_cuda(ctx, e, "argmax kernel");
  }
  return finish_outputs(ctx, out, C, G, want_sum, want_pm, false, want_arg, st);
}

asim_status asim_evaluate_deltas(asim_ctx* ctx, const asim_deltas* d, asim_results* out,
                                 void* cuda_stream) {
  asim_status s = asim_ready(ctx);
  if (s) return s;
  if (!d) return asim_fail(ctx, ASIM_EINVAL, "null deltas");
  const int64_t C = d->num_candidates;
  const int32_t B = d->num_bases, G = d->max_groups;
  const int64_t M = ctx->hp.M;
  if (C < 0 || C > (int64_t(1) << 31) - 64) return asim_fail(ctx, ASIM_ERANGE, "num_candidates");
  if (B < 0 || (C > 0 && B < 1)) return asim_fail(ctx, ASIM_ERANGE, "num_bases");
  if (G < 0 || G > ASIM_MAX_GROUPS) return asim_fail(ctx, ASIM_ERANGE, "max_groups out of range");
  DeviceGuard dg(ctx->device);
  cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
  HostBatch hb;
  hb.G = G;
  s = fetch(ctx, hb.base_cfg, d->base_group_cfg, (int64_t)B * G, d->ptr_kind, st, "base_group_cfg");
  if (s) return s;
  s = fetch(ctx, hb.base_mask, d->base_host_mask, (int64_t)B * M, d->ptr_kind, st, "base_host_mask");
  if (s) return s;
  s = fetch(ctx, hb.cand_base, d->cand_base, C, d->ptr_kind, st, "cand_base");
  if (s) return s;
  s = fetch(ctx, hb.cand_model, d->cand_model, C, d->ptr_kind, st, "cand_model");
  if (s) return s;
  s = fetch(ctx, hb.cand_group, d->cand_group, C, d->ptr_kind, st, "cand_group");
  if (s) return s;
  std::vector<std::vector<int64_t>> used(B);
  std::vector<uint8_t> base_ok(B);
  for (int32_t b = 0; b < B; ++b) {
    bool ok = false;
    s = check_base(ctx, hb.base_cfg.data() + (int64_t)b * G, hb.base_mask.data() + (int64_t)b * M,
                   G, used[b], &ok, &hb.slots);
    if (s) return s;
    base_ok[b] = ok;
  }
  hb.cand_ok.resize(C);
  for (int64_t c = 0; c < C; ++c) {
    const int32_t b = hb.cand_base[c], m = hb.cand_model[c], g = hb.cand_group[c];
    if (b < 0 || b >= B) return asim_fail(ctx, ASIM_ERANGE, "cand_base out of range");
    if (m < -1 || m >= M) return asim_fail(ctx, ASIM_ERANGE, "cand_model out of range");
    bool ok = base_ok[b];
    if (m >= 0) {
      if (g < 0 || g >= G) return asim_fail(ctx, ASIM_ERANGE, "cand_group out of range");
      const int32_t cfg = hb.base_cfg[(int64_t)b * G + g];
      if (cfg < 0) return asim_fail(ctx, ASIM_ERANGE, "cand_group names a group with cfg -1");
      const bool already = (hb.base_mask[(int64_t)b * M + m] >> g) & 1ULL;
      if (!already) {
        const int64_t mb = ctx->hp.mem_at(m, cfg);
        if (mb < 0 || used[b][g] + mb > ctx->hp.budget) ok = false;
      }
    } else {
      hb.cand_group[c] = 0;
    }
    hb.cand_ok[c] = ok ? 1 : 0;
  }
  return evaluate_batch(ctx, hb, out, st);
}

}  // extern "C"
