// extern "C" ABI of libcmgb (include/cmgb.h).
//
// Host responsibilities (all C++, none of them on the hot path): config
// validation, mesh ingest, SDF program validation/packing, surface build
// checks (src/surface.cpp:9-44), per-device geometry upload, manifold layout,
// kernel-parameter assembly and launch. No exception crosses the boundary.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <mutex>
#include <unordered_map>
#include <vector>

#include "host.h"
#include "../kernels/launch_util.cuh"

namespace cmgb {
int manifold_max_threads(int k1, int k2);
size_t compact_workspace_bytes(int64_t n_env, int C);
int launch_compact(const float* contacts, const int32_t* src, int64_t n_env, int C, float thr, int64_t capacity,
                   float* out_contacts, int32_t* out_slot, int32_t* out_src, int64_t* env_offset,
                   int32_t* env_count, int64_t* total, void* workspace, cudaStream_t s);
size_t compact_masked_workspace_bytes(int64_t n_env);
int launch_compact_masked(const float* contacts, const int32_t* src, int64_t n_env, int C, const uint32_t* mask,
                          const int32_t* count, int64_t capacity, float* out_contacts, int32_t* out_slot,
                          int32_t* out_src, int64_t* env_offset, int32_t* env_count, int64_t* total,
                          void* workspace, cudaStream_t s);
}

using namespace cmgb;

namespace {

thread_local std::string g_error;

int set_error(int status, const std::string& msg) {
  g_error = msg;
  return status;
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return CMGB_OK;
  } catch (const Error& e) {
    return set_error(e.status, e.what());
  } catch (const std::bad_alloc&) {
    return set_error(CMGB_ERR_INVALID_ARGUMENT, "out of host memory");
  } catch (const std::exception& e) {
    return set_error(CMGB_ERR_INVALID_ARGUMENT, e.what());
  }
}

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw Error(e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver ? CMGB_ERR_NO_DEVICE
                                                                          : CMGB_ERR_CUDA,
                std::string(what) + ": " + cudaGetErrorString(e));
}

void validate_config(const cmgb_config* c) {
  if (!c) invalid("config: null pointer");
  auto positive = [](double v, const char* name) {
    if (!(v > 0.0)) invalid(std::string("smoothing: ") + name + " must be > 0");
  };
  positive(c->lambda, "lambda");
  positive(c->tau_clip, "tau_clip");
  positive(c->tau_min, "tau_min");
  positive(c->tau_comp, "tau_comp");
  positive(c->tau_sign, "tau_sign");
  positive(c->tau_pen, "tau_pen");
  positive(c->tau_nn, "tau_nn");
  positive(c->tau_clash, "tau_clash");
  positive(c->tau_cont, "tau_cont");
  positive(c->tau_topk_verts, "tau_topk_verts");
  positive(c->tau_topk_edges, "tau_topk_edges");
  positive(c->tau_normal, "tau_normal");
  positive(c->tau_union, "tau_union");
  if (c->sphere_trace_iters < 0) invalid("smoothing: sphere_trace_iters >= 0");
  if (c->mode < CMGB_MODE_FULL || c->mode > CMGB_MODE_ONE_SIDED) invalid("config: unknown mode");
}

DevCfg device_config(const cmgb_config* c) {
  DevCfg d{};
  d.lambda = c->lambda;
  d.tau_clip = c->tau_clip;
  d.inv_tau_clip = 1.0 / c->tau_clip;
  d.inv_tau_min = 1.0 / c->tau_min;
  d.inv_tau_comp = 1.0 / c->tau_comp;
  d.inv_tau_sign = 1.0 / c->tau_sign;
  d.inv_tau_pen = 1.0 / c->tau_pen;
  d.inv_tau_nn = 1.0 / c->tau_nn;
  d.inv_tau_clash = 1.0 / c->tau_clash;
  d.inv_tau_cont = 1.0 / c->tau_cont;
  d.inv_tau_topk_v = 1.0 / c->tau_topk_verts;
  d.inv_tau_topk_e = 1.0 / c->tau_topk_edges;
  d.tau_normal = c->tau_normal;
  d.clip_C = std::exp(-1.0 / c->tau_clip);
  d.comp_C = std::exp(-1.0 / c->tau_comp);
  d.inv_clip_C = 1.0 / d.clip_C;
  d.inv_comp_C = 1.0 / d.comp_C;
  d.pair_exp = (1.0 / c->tau_clip < 700.0 && 1.0 / c->tau_comp < 700.0) ? 1 : 0;
  d.hard_ops = c->hard_ops ? 1 : 0;
  d.trace_iters = (c->sphere_trace && c->sphere_trace_iters > 0) ? c->sphere_trace_iters : 0;
  d.containment = c->containment_safeguard ? 1 : 0;
  d.mode = c->mode;
  return d;
}

cmgb_layout layout_of(const cmgb_surface_s* s1, const cmgb_surface_s* s2, const cmgb_config* c) {
  cmgb_layout L{};
  L.mode = c->mode;
  L.n1 = s1->effective_vertex_topk();
  const bool two = c->mode != CMGB_MODE_ONE_SIDED;
  const bool full = c->mode == CMGB_MODE_FULL;
  L.n2 = two ? s2->effective_vertex_topk() : 0;
  L.m1 = full ? s1->effective_edge_topk() : 0;
  L.m2 = full ? s2->effective_edge_topk() : 0;
  L.n_contacts = L.n1 + L.n2 + 2 * L.m1 * L.m2;
  L.dynamic_src = (L.n1 < s1->mesh.nv()) || (two && L.n2 < s2->mesh.nv()) ||
                  (full && (L.m1 < s1->mesh.ne() || L.m2 < s2->mesh.ne()));
  return L;
}

DeviceSurface& device_image(cmgb_surface_s* s) {
  int dev = 0;
  cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
  std::lock_guard<std::mutex> lock(s->mu);
  auto it = s->device.find(dev);
  if (it != s->device.end()) return it->second;
  DeviceSurface d;
  std::vector<double4> pool;
  std::vector<DevNode> ext;
  d.sdf = pack_program(s->program, &pool, &ext);
  if (!ext.empty()) {  // programs above kMaxNodes: the generic interpreter reads the nodes from here
    cuda_check(cudaMalloc(&d.ext, sizeof(DevNode) * ext.size()), "cudaMalloc");
    cuda_check(cudaMemcpy(d.ext, ext.data(), sizeof(DevNode) * ext.size(), cudaMemcpyHostToDevice), "cudaMemcpy");
  }
  d.sdf.ext = d.ext;
  cuda_check(cudaMalloc(&d.verts, sizeof(double) * s->mesh.vertices.size()), "cudaMalloc");
  cuda_check(cudaMemcpy(d.verts, s->mesh.vertices.data(), sizeof(double) * s->mesh.vertices.size(),
                        cudaMemcpyHostToDevice), "cudaMemcpy");
  cuda_check(cudaMalloc(&d.edges, sizeof(int32_t) * s->mesh.edges.size()), "cudaMalloc");
  cuda_check(cudaMemcpy(d.edges, s->mesh.edges.data(), sizeof(int32_t) * s->mesh.edges.size(),
                        cudaMemcpyHostToDevice), "cudaMemcpy");
  {
    std::vector<double> eb(6 * (size_t)s->mesh.ne());
    for (int e = 0; e < s->mesh.ne(); ++e)
      for (int k = 0; k < 2; ++k)
        for (int c = 0; c < 3; ++c) eb[6 * e + 3 * k + c] = s->mesh.vertices[3 * s->mesh.edges[2 * e + k] + c];
    cuda_check(cudaMalloc(&d.edge_body, sizeof(double) * std::max<size_t>(eb.size(), 1)), "cudaMalloc");
    cuda_check(cudaMemcpy(d.edge_body, eb.data(), sizeof(double) * eb.size(), cudaMemcpyHostToDevice), "cudaMemcpy");
  }
  if (!pool.empty()) {
    cuda_check(cudaMalloc(&d.pool, sizeof(double4) * pool.size()), "cudaMalloc");
    cuda_check(cudaMemcpy(d.pool, pool.data(), sizeof(double4) * pool.size(), cudaMemcpyHostToDevice),
               "cudaMemcpy");
  }
  d.sdf.pool = d.pool;
  return s->device.emplace(dev, d).first->second;
}

int align16(int x) { return (x + 15) & ~15; }

struct LaunchPlan {
  ManifoldParams p{};
  int threads = 0, grid = 0;
  size_t smem = 0;
  bool pairs_global = false;  // pair records in a global workspace (large pass-through pair sets)
};

LaunchPlan plan_manifold(cmgb_surface_s* s1, cmgb_surface_s* s2, const double* poses1, int st1,
                         const double* poses2, int st2, int64_t n_env, const cmgb_config* cfg,
                         const cmgb_manifold_out* out) {
  validate_config(cfg);
  if (!s1 || !s2) invalid("manifold: null surface");
  if (n_env < 0) invalid("manifold: n_env >= 0");
  if (!out) invalid("manifold: null output descriptor");
  if (n_env > 0 && !out->contacts) invalid("manifold: contacts output is required");
  if (n_env > 0 && (!poses1 || !poses2)) invalid("manifold: null poses");
  if ((st1 != 0 && st1 != 1) || (st2 != 0 && st2 != 1)) invalid("manifold: pose stride must be 0 or 1");
  const cmgb_layout L = layout_of(s1, s2, cfg);
  LaunchPlan plan;
  ManifoldParams& p = plan.p;
  cmgb_surface_s* ss[2] = {s1, s2};
  const int nsel[2] = {L.n1, L.mode == CMGB_MODE_ONE_SIDED ? 0 : L.n2};
  const int msel[2] = {L.m1, L.m2};
  for (int k = 0; k < 2; ++k) {
    DeviceSurface& d = device_image(ss[k]);
    DevSide& side = p.side[k];
    side.verts = d.verts;
    side.edges = d.edges;
    side.edge_body = d.edge_body;
    side.nv = ss[k]->mesh.nv();
    side.ne = ss[k]->mesh.ne();
    side.n_sel = nsel[k];
    side.m_sel = msel[k];
    // Selection stages only run for slots that are actually emitted.
    side.topk_v = (nsel[k] > 0 && nsel[k] < side.nv) ? 1 : 0;
    side.topk_e = (msel[k] > 0 && msel[k] < side.ne) ? 1 : 0;
    side.sdf = d.sdf;
  }
  p.cfg = device_config(cfg);
  p.poses1 = poses1;
  p.poses2 = poses2;
  p.stride1 = st1;
  p.stride2 = st2;
  p.pose_stride1 = 6 * st1;
  p.pose_stride2 = 6 * st2;
  p.n_env = n_env;
  p.n1 = L.n1;
  p.n2 = nsel[1];
  p.m1 = L.m1;
  p.m2 = L.m2;
  p.n_contacts = L.n_contacts;
  p.frames1 = nullptr;  // bound by the caller (workspace)
  p.frames2 = nullptr;
  p.contacts = out->contacts;
  p.src = out->src;
  p.ee = (L.m1 > 0 && L.m2 > 0) ? out->ee : nullptr;
  p.mean_dist = out->mean_dist;
  p.act_mask = out->active_mask;
  p.act_count = out->active_count;
  p.act_thr = out->active_threshold;
  p.mask_words = (L.n_contacts + 31) / 32;
  if (p.act_mask && !p.act_count) invalid("manifold: active_mask needs active_count");
  if (p.act_mask && !(out->active_threshold == out->active_threshold)) invalid("manifold: active_threshold is NaN");

  // Shared-memory carve-up per env.
  const int P = L.m1 * L.m2;
  const int nslot_v = p.n1 + p.n2, nslot_e = L.m1 + L.m2;
  const bool topk = p.side[0].topk_v || p.side[1].topk_v || p.side[0].topk_e || p.side[1].topk_e;
  const int nscore = topk ? (p.side[0].nv + p.side[1].nv + p.side[0].ne + p.side[1].ne) : 0;
  SmemLayout& S = p.smem;
  // pairs_in_smem: the per-pair records live in shared memory unless the env's
  // working set would exceed the per-CTA budget; then they move to a global
  // workspace (L2-resident per chunk of envs, launch_with_workspace).
  auto carve = [&](bool pairs_in_smem) {
    int off = 0;
    S.frames = off; off = align16(off + 24 * 8);
    S.vslots = off; off = align16(off + nslot_v * 3 * 8);
    S.eslots = off; off = align16(off + nslot_e * 13 * 8);
    S.prov = off; off = align16(off + (nslot_v + nslot_e) * 4);
    S.scores = off; off = align16(off + nscore * 8);
    S.sorted = off; off = align16(off + nscore * 4);
    S.tkw = off; off = align16(off + nscore * 8);
    S.pairs = off; off = align16(off + (pairs_in_smem ? P * kPairRec * 4 : 0));
    S.vsdist = off; off = align16(off + nslot_v * 4);
    S.nnstat = off; off = align16(off + nslot_e * 3 * 8);
    S.hpart = off; off = align16(off + 10 * 8);  // one partial per warp (<= 320-thread CTAs)
    S.amask = off; off = align16(off + (out->active_mask ? 4 * ((L.n_contacts + 31) / 32) : 0));
    S.bytes = off;
  };
  const size_t kSmemMax = (size_t)smem_optin_per_block();  // device attribute (227 KB on B200)
  carve(true);
  p.pairs_gmem = nullptr;
  p.pair_stride = 0;
  plan.pairs_global = (size_t)S.bytes > kSmemMax;
  if (plan.pairs_global) {
    carve(false);
    p.pair_stride = (int64_t)P * (kPairRec / 2);
    if ((size_t)S.bytes > kSmemMax)
      throw Error(CMGB_ERR_UNSUPPORTED, "manifold: per-env working set exceeds shared memory");
  }

  // Envs per block: about one CTA's worth of E-E pairs (2 box-box envs per
  // 320-thread CTA), shared memory capped so the kernel's resident-CTA target fits.
  // the global-record path runs the generic instantiation (manifold.cu)
  const int k1 = plan.pairs_global ? (int)kGeneric : p.side[0].sdf.kind;
  const int k2 = plan.pairs_global ? (int)kGeneric : p.side[1].sdf.kind;
  const int maxt = manifold_max_threads(k1, k2);
  const int per_env = std::max({P, nslot_v, 1});
  int epb = std::max(1, maxt / per_env);
  // shared memory per CTA such that the kernel's resident-CTA target fits the SM
  const size_t smem_cap =
      (size_t)(smem_per_sm() - manifold_min_blocks(k1, k2) * kSmemReservedPerCta) / manifold_min_blocks(k1, k2);
  while (epb > 1 && (size_t)epb * S.bytes > smem_cap) --epb;
  const int threads = maxt;
  p.envs_per_block = epb;
  auto fd = [](int d) {
    FastDiv f;
    f.d = (uint32_t)std::max(d, 1);
    f.mul = ((1ULL << 32) + f.d - 1) / f.d;
    f.pad = 0;
    return f;
  };
  p.div_pairs = fd(P);
  p.div_m2 = fd(L.m2);
  p.div_nvs = fd(nslot_v);
  p.div_nslots = fd(nslot_v + nslot_e);
  p.div_nrc = fd(nslot_e);
  p.div_nv_all = fd(p.side[0].nv + p.side[1].nv);
  p.div_ne_all = fd(p.side[0].ne + p.side[1].ne);
  p.div_scores = fd(p.side[0].nv + p.side[1].nv + p.side[0].ne + p.side[1].ne);
  plan.threads = threads;
  plan.grid = static_cast<int>((n_env + epb - 1) / epb);
  plan.smem = (size_t)epb * S.bytes;
  if (std::getenv("CMGB_DEBUG_PLAN"))  // developer instrumentation
    std::fprintf(stderr, "cmgb plan: kinds %d/%d threads %d envs/CTA %d smem/env %d B (scores %d) P %d\n", k1, k2,
                 threads, epb, S.bytes, nscore, P);
  return plan;
}

// Scratch for the end-to-end host API, per (device, thread) reuse.
struct HostScratch {
  double* poses1 = nullptr;
  double* poses2 = nullptr;
  float* contacts = nullptr;
  float* mean = nullptr;
  double* frames = nullptr;
  int32_t* src = nullptr;
  float* ee = nullptr;
  size_t cap_poses1 = 0, cap_poses2 = 0, cap_contacts = 0, cap_mean = 0, cap_frames = 0, cap_src = 0, cap_ee = 0;
  cudaStream_t q[2] = {nullptr, nullptr};  // pipeline streams of the host-buffer API
  cudaEvent_t ev[2] = {nullptr, nullptr};
  cudaEvent_t ev_start = nullptr;
};

// Smallest env chunk worth its own pipeline stage of the host-buffer API.
constexpr int64_t kHostChunkMin = 2048;

size_t workspace_doubles(int64_t n_env, int st1, int st2) {
  return 12 * (size_t)((st1 ? n_env : 1) + (st2 ? n_env : 1));
}

// Binds the frames workspace (caller's, or a stream-ordered pool block) and
// launches frames_kernel + manifold_kernel on the stream.
// Stream-ordered scratch (cudaMallocAsync) from the device's default memory
// pool, which by default returns freed blocks to the driver at every
// synchronisation: a synchronous caller (one call, then a stream sync) would
// pay a fresh driver allocation per call. The pool keeps up to 2 GB cached.
cudaError_t scratch_alloc(void** p, size_t bytes, cudaStream_t s) {
  static PerDeviceOnce retain;
  retain([] {
    int dev = 0;
    cudaMemPool_t pool;
    if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t keep = 2ull << 30;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
  });
  return cudaMallocAsync(p, bytes, s);
}

// One planned launch whose frame pointers are set: the pass-through kernels, or
// (pair records in global memory) env chunks whose records fit a 512 MB
// stream-ordered block, one launch each (frames land in the caller's slots).
void launch_planned(LaunchPlan& plan, int64_t n_env, cudaStream_t stream) {
  int rc = 0;
  if (!plan.pairs_global) {
    rc = launch_manifold(plan.p, plan.threads, plan.grid, plan.smem, stream);
  } else {
    const size_t rec_bytes = sizeof(double) * (size_t)plan.p.pair_stride;
    const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(n_env, (512ll << 20) / (int64_t)rec_bytes));
    double* rec = nullptr;
    cuda_check(scratch_alloc(reinterpret_cast<void**>(&rec), rec_bytes * chunk, stream),
               "cudaMallocAsync(pair records)");
    const int C = plan.p.n_contacts, P = plan.p.m1 * plan.p.m2;
    for (int64_t c0 = 0; c0 < n_env && rc == 0; c0 += chunk) {
      const int64_t cn = std::min(chunk, n_env - c0);
      ManifoldParams q = plan.p;
      q.n_env = cn;
      q.poses1 += q.pose_stride1 * c0;
      q.poses2 += q.pose_stride2 * c0;
      q.frames1 += 12 * c0 * q.stride1;
      q.frames2 += 12 * c0 * q.stride2;
      q.contacts += c0 * C * 8;
      if (q.src) q.src += c0 * C * 2;
      if (q.ee) q.ee += c0 * 9 * P;
      if (q.mean_dist) q.mean_dist += c0;
      if (q.act_mask) {
        q.act_mask += c0 * q.mask_words;
        q.act_count += c0;
      }
      q.pairs_gmem = rec;
      const int grid = (int)((cn + q.envs_per_block - 1) / q.envs_per_block);
      rc = launch_manifold(q, plan.threads, grid, plan.smem, stream);
    }
    cudaFreeAsync(rec, stream);
  }
  if (rc != 0)
    throw Error(CMGB_ERR_CUDA, std::string("manifold launch: ") + cudaGetErrorString(cudaGetLastError()));
}

void launch_with_workspace(LaunchPlan& plan, int64_t n_env, int st1, int st2, void* ws, size_t ws_bytes,
                           cudaStream_t stream) {
  const size_t need = workspace_doubles(n_env, st1, st2) * sizeof(double);
  void* buf = ws;
  const bool pooled = ws == nullptr || ws_bytes < need;
  if (pooled) cuda_check(scratch_alloc(&buf, need, stream), "cudaMallocAsync(workspace)");
  double* f = static_cast<double*>(buf);
  plan.p.frames1 = f;
  plan.p.frames2 = f + 12 * (st1 ? n_env : 1);
  try {
    launch_planned(plan, n_env, stream);
  } catch (...) {
    if (pooled) cudaFreeAsync(buf, stream);
    throw;
  }
  if (pooled) cudaFreeAsync(buf, stream);
}

// Independent launches of one call spread over a device's side streams: fork
// from the caller's stream, join back into it (events), so a scene's pairs
// overlap each other's tails; the caller sees one stream-ordered operation.
struct SideStreams {
  static constexpr int kN = 4;
  cudaStream_t s[kN] = {};
};
SideStreams& side_streams() {
  static std::mutex mu;
  static std::unordered_map<int, SideStreams> per_dev;
  int dev = 0;
  cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
  std::lock_guard<std::mutex> lock(mu);
  SideStreams& ss = per_dev[dev];
  if (!ss.s[0])
    for (auto& x : ss.s) cuda_check(cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking), "cudaStreamCreate");
  return ss;
}
struct ForkEvents {  // per host thread and device: reused, so a call creates no events
  cudaEvent_t start = nullptr, done[SideStreams::kN] = {};
  ForkEvents() = default;
  ForkEvents(const ForkEvents&) = delete;
  ForkEvents& operator=(const ForkEvents&) = delete;
  ~ForkEvents() {  // at thread exit (harmless error codes if the context is already gone)
    if (start) cudaEventDestroy(start);
    for (auto& d : done)
      if (d) cudaEventDestroy(d);
  }
};
ForkEvents& fork_events() {
  thread_local std::unordered_map<int, ForkEvents> per_dev;
  int dev = 0;
  cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
  ForkEvents& e = per_dev[dev];
  if (!e.start) {
    cuda_check(cudaEventCreateWithFlags(&e.start, cudaEventDisableTiming), "cudaEventCreate");
    for (auto& d : e.done) cuda_check(cudaEventCreateWithFlags(&d, cudaEventDisableTiming), "cudaEventCreate");
  }
  return e;
}
struct StreamFork {
  cudaStream_t base;
  int n;
  SideStreams& ss;
  ForkEvents& ev;
  StreamFork(cudaStream_t b, int want)
      : base(b), n(std::max(1, std::min(want, SideStreams::kN))), ss(side_streams()), ev(fork_events()) {
    cuda_check(cudaEventRecord(ev.start, base), "cudaEventRecord");
    for (int k = 0; k < n; ++k) cuda_check(cudaStreamWaitEvent(ss.s[k], ev.start, 0), "cudaStreamWaitEvent");
  }
  cudaStream_t stream(int q) const { return ss.s[q % n]; }
  ~StreamFork() {  // join (also on the error path: the caller's stream must cover every launch)
    for (int k = 0; k < n; ++k)
      if (cudaEventRecord(ev.done[k], ss.s[k]) == cudaSuccess) cudaStreamWaitEvent(base, ev.done[k], 0);
  }
};

template <class T>
void ensure(T** ptr, size_t* cap, size_t n) {
  if (*cap >= n) return;
  if (*ptr) cudaFree(*ptr);
  *ptr = nullptr;
  cuda_check(cudaMalloc(ptr, sizeof(T) * std::max<size_t>(n, 1)), "cudaMalloc");
  *cap = n;
}

// Host-buffer API scratch: a pool per device from which each call leases its
// own HostScratch for its duration, so concurrent host threads never share
// device buffers or pipeline streams (the lock covers only check-out/return).
struct ScratchPool {
  std::mutex mu;
  std::unordered_map<int, std::vector<HostScratch*>> idle;
};
ScratchPool g_scratch_pool;

// The two pipeline streams (and their events) of a host scratch, created once.
void ensure_pipeline(HostScratch& sc) {
  if (sc.q[0]) return;
  for (int k = 0; k < 2; ++k) {
    cuda_check(cudaStreamCreateWithFlags(&sc.q[k], cudaStreamNonBlocking), "cudaStreamCreate");
    cuda_check(cudaEventCreateWithFlags(&sc.ev[k], cudaEventDisableTiming), "cudaEventCreate");
  }
  cuda_check(cudaEventCreateWithFlags(&sc.ev_start, cudaEventDisableTiming), "cudaEventCreate");
}

struct ScratchLease {
  int dev;
  HostScratch* sc;
  explicit ScratchLease(int d) : dev(d), sc(nullptr) {
    std::lock_guard<std::mutex> lock(g_scratch_pool.mu);
    auto& v = g_scratch_pool.idle[d];
    if (!v.empty()) {
      sc = v.back();
      v.pop_back();
    }
    if (!sc) sc = new HostScratch();
  }
  // Also on the error path: copies into the caller's host buffers may already be
  // queued on the pipeline streams; they must finish before the call returns.
  ~ScratchLease() {
    for (cudaStream_t q : sc->q)
      if (q) cudaStreamSynchronize(q);
    std::lock_guard<std::mutex> lock(g_scratch_pool.mu);
    g_scratch_pool.idle[dev].push_back(sc);
  }
  ScratchLease(const ScratchLease&) = delete;
  ScratchLease& operator=(const ScratchLease&) = delete;
};

}  // namespace

int cmgb_surface_s::effective_vertex_topk() const {
  const int v = mesh.nv();
  return vertex_topk <= 0 ? v : std::min(vertex_topk, v);
}

int cmgb_surface_s::effective_edge_topk() const {
  const int e = mesh.ne();
  return edge_topk <= 0 ? std::min(program.leaf_count, e) : std::min(edge_topk, e);
}

extern "C" {

const char* cmgb_last_error(void) { return g_error.c_str(); }
int32_t cmgb_abi_version(void) { return CMGB_ABI_VERSION; }

void cmgb_config_default(cmgb_config* c) {
  if (!c) return;
  *c = cmgb_config{};
  c->lambda = 0.01;
  c->tau_clip = c->tau_min = c->tau_comp = 0.1;
  c->tau_sign = 0.1;
  c->tau_pen = 0.01;
  c->tau_nn = 0.01;
  c->tau_clash = 0.1;
  c->tau_cont = 0.01;
  c->tau_topk_verts = c->tau_topk_edges = 0.01;
  c->tau_normal = 1e-9;
  c->tau_union = 0.01;
  c->hard_ops = 0;
  c->sphere_trace = 1;
  c->sphere_trace_iters = 5;
  c->containment_safeguard = 0;
  c->mode = CMGB_MODE_FULL;
}

void cmgb_config_no_smoothing(cmgb_config* c) {
  cmgb_config_default(c);
  if (!c) return;
  c->lambda = 1e-6;
  c->hard_ops = 1;
}

int cmgb_config_validate(const cmgb_config* c) {
  return guarded([&] { validate_config(c); });
}

int cmgb_config_for_variant(const char* variant, const cmgb_config* base, cmgb_config* out) {
  return guarded([&] {
    if (!variant || !base || !out) invalid("config_for_variant: null argument");
    cmgb_config c = *base;
    const std::string v(variant);
    if (v == "ours") {
      c.hard_ops = 0;
      c.mode = CMGB_MODE_FULL;
    } else if (v == "ours_ns") {
      c.hard_ops = 1;
      c.lambda = 1e-6;
      c.mode = CMGB_MODE_FULL;
    } else if (v == "ours_ne") {
      c.hard_ops = 0;
      c.mode = CMGB_MODE_NO_EE;
    } else if (v == "ours_ne_s") {
      c.hard_ops = 0;
      c.mode = CMGB_MODE_ONE_SIDED;
    } else {
      invalid("unknown variant: " + v + " (expected ours|ours_ns|ours_ne|ours_ne_s)");
    }
    *out = c;
  });
}

// ---- meshes ---------------------------------------------------------------
int cmgb_mesh_box(const double half[3], int32_t subdivisions, int32_t quad_edges, cmgb_mesh* out) {
  return guarded([&] {
    if (!half || !out) invalid("mesh_box: null argument");
    auto* m = new cmgb_mesh_s{make_box_mesh(half, subdivisions, quad_edges != 0)};
    *out = m;
  });
}

int cmgb_mesh_parse_obj(const char* text, size_t length, cmgb_mesh* out, int32_t* error_line) {
  return guarded([&] {
    if (!text || !out) invalid("parse_obj: null argument");
    try {
      auto* m = new cmgb_mesh_s{parse_obj_text(std::string(text, length))};
      *out = m;
    } catch (const Error& e) {
      if (error_line) *error_line = e.line;
      throw;
    }
  });
}

int cmgb_mesh_from_arrays(const double* vertices, int32_t n_vertices, const int32_t* faces,
                          int32_t n_faces, const int32_t* edges, int32_t n_edges, cmgb_mesh* out) {
  return guarded([&] {
    if (!out || n_vertices < 0 || n_faces < 0 || n_edges < 0) invalid("mesh_from_arrays: bad argument");
    if ((n_vertices && !vertices) || (n_faces && !faces) || (n_edges && !edges))
      invalid("mesh_from_arrays: null array");
    auto* m = new cmgb_mesh_s;
    m->mesh.vertices.assign(vertices, vertices + 3 * (size_t)n_vertices);
    if (n_faces) m->mesh.faces.assign(faces, faces + 3 * (size_t)n_faces);
    if (n_edges) m->mesh.edges.assign(edges, edges + 2 * (size_t)n_edges);
    *out = m;
  });
}

int cmgb_mesh_sizes(cmgb_mesh mesh, int32_t* nv, int32_t* nf, int32_t* ne, int32_t* nw) {
  return guarded([&] {
    if (!mesh) invalid("mesh_sizes: null mesh");
    if (nv) *nv = mesh->mesh.nv();
    if (nf) *nf = mesh->mesh.nf();
    if (ne) *ne = mesh->mesh.ne();
    if (nw) *nw = static_cast<int32_t>(mesh->mesh.warnings.size());
  });
}

int cmgb_mesh_read(cmgb_mesh mesh, double* vertices, int32_t* faces, int32_t* edges) {
  return guarded([&] {
    if (!mesh) invalid("mesh_read: null mesh");
    const Mesh& m = mesh->mesh;
    if (vertices) std::memcpy(vertices, m.vertices.data(), sizeof(double) * m.vertices.size());
    if (faces) std::memcpy(faces, m.faces.data(), sizeof(int32_t) * m.faces.size());
    if (edges) std::memcpy(edges, m.edges.data(), sizeof(int32_t) * m.edges.size());
  });
}

const char* cmgb_mesh_warning(cmgb_mesh mesh, int32_t i) {
  if (!mesh || i < 0 || i >= (int32_t)mesh->mesh.warnings.size()) return nullptr;
  return mesh->mesh.warnings[i].c_str();
}

void cmgb_mesh_destroy(cmgb_mesh mesh) { delete mesh; }

// ---- surfaces ---------------------------------------------------------------
int cmgb_surface_create(cmgb_mesh mesh, const cmgb_sdf_node* sdf, int32_t n_nodes,
                        int32_t vertex_topk, int32_t edge_topk, double tolerance_fraction,
                        cmgb_surface* out) {
  return guarded([&] {
    if (!mesh || !out) invalid("surface_create: null argument");
    Program prog = make_program(sdf, n_nodes);
    const Mesh& m = mesh->mesh;
    // build_surface validation (src/surface.cpp:11-24), same messages.
    if (m.nv() == 0 || m.ne() == 0) invalid("surface: mesh needs vertices and edges");
    if (vertex_topk < 0 || vertex_topk > m.nv())
      invalid("surface: vertex_topk must lie in [1, V] (or 0 for all)");
    if (edge_topk < 0 || edge_topk > m.ne())
      invalid("surface: edge_topk must lie in [1, E] (or 0 for default)");
    for (int32_t idx : m.edges)
      if (idx < 0 || idx >= m.nv()) invalid("surface: edge index out of range");
    for (int32_t idx : m.faces)
      if (idx < 0 || idx >= m.nv()) invalid("surface: face index out of range");
    auto* s = new cmgb_surface_s;
    s->mesh = m;
    s->program = std::move(prog);
    s->vertex_topk = vertex_topk;
    s->edge_topk = edge_topk;
    s->warnings = m.warnings;
    // Mesh/SDF discrepancy is a warning (src/surface.cpp:31-42).
    double worst = 0.0;
    for (int i = 0; i < m.nv(); ++i) worst = std::max(worst, std::abs(s->program.value(&m.vertices[3 * i])));
    const double tol = tolerance_fraction * m.bounding_diagonal();
    if (worst > tol)
      s->warnings.push_back("mesh/SDF discrepancy: max |phi(vertex)| = " + std::to_string(worst) +
                            " exceeds tolerance " + std::to_string(tol) +
                            "; witness projection and activity indicators may drift");
    *out = s;
  });
}

void cmgb_surface_destroy(cmgb_surface s) {
  if (!s) return;
  int prev = -1;
  cudaGetDevice(&prev);
  for (auto& [dev, d] : s->device) {
    cudaSetDevice(dev);
    cudaFree(d.verts);
    cudaFree(d.edge_body);
    cudaFree(d.edges);
    if (d.pool) cudaFree(d.pool);
    if (d.ext) cudaFree(d.ext);
  }
  if (prev >= 0) cudaSetDevice(prev);
  delete s;
}

int cmgb_surface_get_info(cmgb_surface s, cmgb_surface_info* out) {
  return guarded([&] {
    if (!s || !out) invalid("surface_get_info: null argument");
    out->n_vertices = s->mesh.nv();
    out->n_edges = s->mesh.ne();
    out->n_faces = s->mesh.nf();
    out->leaf_count = s->program.leaf_count;
    out->vertex_topk = s->vertex_topk;
    out->edge_topk = s->edge_topk;
    out->effective_vertex_topk = s->effective_vertex_topk();
    out->effective_edge_topk = s->effective_edge_topk();
    out->n_warnings = static_cast<int32_t>(s->warnings.size());
    out->n_nodes = static_cast<int32_t>(s->program.nodes.size());
  });
}

const char* cmgb_surface_warning(cmgb_surface s, int32_t i) {
  if (!s || i < 0 || i >= (int32_t)s->warnings.size()) return nullptr;
  return s->warnings[i].c_str();
}

// ---- layout -------------------------------------------------------------------
int cmgb_layout_query(cmgb_surface s1, cmgb_surface s2, const cmgb_config* cfg, cmgb_layout* out) {
  return guarded([&] {
    if (!s1 || !s2 || !out) invalid("layout_query: null argument");
    validate_config(cfg);
    *out = layout_of(s1, s2, cfg);
  });
}

int cmgb_layout_metadata(cmgb_surface s1, cmgb_surface s2, const cmgb_config* cfg, int32_t* kind,
                         int32_t* side, int32_t* src_a, int32_t* src_b) {
  return guarded([&] {
    if (!s1 || !s2) invalid("layout_metadata: null surface");
    validate_config(cfg);
    const cmgb_layout L = layout_of(s1, s2, cfg);
    const bool sel_v1 = L.n1 < s1->mesh.nv(), sel_v2 = L.n2 < s2->mesh.nv();
    const bool sel_e1 = L.m1 < s1->mesh.ne(), sel_e2 = L.m2 < s2->mesh.ne();
    int q = 0;
    auto put = [&](int k, int sd, int a, int b) {
      if (kind) kind[q] = k;
      if (side) side[q] = sd;
      if (src_a) src_a[q] = a;
      if (src_b) src_b[q] = b;
      ++q;
    };
    for (int i = 0; i < L.n1; ++i) put(0, 1, sel_v1 ? -1 : i, -1);
    for (int i = 0; i < L.n2; ++i) put(0, 2, sel_v2 ? -1 : i, -1);
    for (int k = 0; k < L.m1; ++k)
      for (int l = 0; l < L.m2; ++l) {
        put(1, 1, sel_e1 ? -1 : k, sel_e2 ? -1 : l);
        put(1, 2, sel_e1 ? -1 : k, sel_e2 ? -1 : l);
      }
  });
}

// ---- batched manifold ------------------------------------------------------------
int cmgb_manifold_batch(cmgb_surface s1, cmgb_surface s2, const double* poses1, int32_t st1,
                        const double* poses2, int32_t st2, int64_t n_env, const cmgb_config* cfg,
                        const cmgb_manifold_out* out, void* stream) {
  return guarded([&] {
    LaunchPlan plan = plan_manifold(s1, s2, poses1, st1, poses2, st2, n_env, cfg, out);
    if (n_env == 0 || plan.p.n_contacts == 0) return;
    launch_with_workspace(plan, n_env, st1, st2, out->workspace, out->workspace_bytes,
                          static_cast<cudaStream_t>(stream));
  });
}

int cmgb_manifold_batch_host_ex(cmgb_surface s1, cmgb_surface s2, const double* poses1_host,
                                int32_t st1, const double* poses2_host, int32_t st2, int64_t n_env,
                                const cmgb_config* cfg, const cmgb_manifold_out* host_out, void* stream) {
  return guarded([&] {
    if (!host_out) invalid("manifold_batch_host: null output descriptor");
    float* mean_dist_host = host_out->mean_dist;
    float* contacts_host = host_out->contacts;
    int32_t* src_host = host_out->src;
    float* ee_host = host_out->ee;
    if (!s1 || !s2) invalid("manifold_batch_host: null surface");
    validate_config(cfg);
    if ((st1 != 0 && st1 != 1) || (st2 != 0 && st2 != 1)) invalid("manifold: pose stride must be 0 or 1");
    if (n_env == 0) return;
    if (!poses1_host || !poses2_host) invalid("manifold_batch_host: null poses");
    const cmgb_layout L = layout_of(s1, s2, cfg);
    int dev = 0;
    cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
    ScratchLease lease(dev);
    HostScratch& sc = *lease.sc;
    const size_t np1 = (st1 ? n_env : 1) * 6, np2 = (st2 ? n_env : 1) * 6;
    ensure(&sc.poses1, &sc.cap_poses1, np1);
    ensure(&sc.poses2, &sc.cap_poses2, np2);
    ensure(&sc.contacts, &sc.cap_contacts, (size_t)n_env * L.n_contacts * 8);
    ensure(&sc.mean, &sc.cap_mean, (size_t)n_env);
    const size_t P = (size_t)L.m1 * L.m2;
    if (!(L.m1 > 0 && L.m2 > 0)) ee_host = nullptr;  // EeIndicatorMatrices exist in full mode only
    if (src_host) ensure(&sc.src, &sc.cap_src, (size_t)n_env * L.n_contacts * 2);
    if (ee_host) ensure(&sc.ee, &sc.cap_ee, (size_t)n_env * 9 * P);
    // Pipelined over env chunks on two internal streams: chunk c+1's pose
    // upload overlaps chunk c's kernels, and each chunk's results stream back
    // as soon as it is done. Ordered after the caller's stream and joined back
    // into it (then synchronised: the outputs are host memory).
    ensure_pipeline(sc);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    // Two chunks: a small lead chunk whose pose upload is the only exposed
    // copy, then the rest, uploaded while the lead chunk computes (equal
    // chunks pay a wave-quantisation tail and launch gaps per chunk: measured
    // box-box 65,536 envs, 8 equal chunks 48.8 M/s, 4 50.3; lead 1/16, 1/8,
    // 1/4 of the envs: 51.3, 51.4, 50.9).
    // With the full contacts coming back (9.7 KB/env box-box, D2H-bound) the
    // batch runs as up to kHostChunksFull equal chunks alternating between the
    // streams, so each chunk's D2H overlaps the next chunk's kernels.
    constexpr int64_t lead_div = 8;
    constexpr int kHostChunksFull = 8;
    std::vector<int64_t> bounds = {0, n_env};
    if ((contacts_host || src_host || ee_host) && n_env >= 2 * kHostChunkMin) {
      const int64_t k = std::min<int64_t>(kHostChunksFull, n_env / kHostChunkMin);
      bounds.clear();
      for (int64_t c = 0; c <= k; ++c) bounds.push_back(n_env * c / k);
    } else if (n_env >= 2 * kHostChunkMin) {
      bounds = {0, std::max(kHostChunkMin, n_env / lead_div), n_env};
    }
    const int nchunk = (int)bounds.size() - 1;
    int64_t per = 0;
    for (int c = 0; c < nchunk; ++c) per = std::max(per, bounds[c + 1] - bounds[c]);
    ensure(&sc.frames, &sc.cap_frames, 2 * workspace_doubles(per, st1, st2));
    cuda_check(cudaEventRecord(sc.ev_start, s), "cudaEventRecord");
    for (int k = 0; k < 2; ++k) cuda_check(cudaStreamWaitEvent(sc.q[k], sc.ev_start, 0), "cudaStreamWaitEvent");
    // shared (stride-0) poses: uploaded once, before either stream uses them
    for (int b = 0; b < 2; ++b) {
      const bool shared = b == 0 ? !st1 : !st2;
      if (!shared) continue;
      cuda_check(cudaMemcpyAsync(b == 0 ? sc.poses1 : sc.poses2, b == 0 ? poses1_host : poses2_host,
                                 sizeof(double) * 6, cudaMemcpyHostToDevice, sc.q[0]),
                 "H2D shared pose");
    }
    cuda_check(cudaEventRecord(sc.ev[0], sc.q[0]), "cudaEventRecord");
    cuda_check(cudaStreamWaitEvent(sc.q[1], sc.ev[0], 0), "cudaStreamWaitEvent");
    const size_t C = (size_t)L.n_contacts;
    for (int c = 0; c < nchunk; ++c) {
      const int64_t e0 = bounds[c], ne = bounds[c + 1] - e0;
      if (ne <= 0) break;
      cudaStream_t q = sc.q[c & 1];
      double* p1 = sc.poses1 + (st1 ? 6 * e0 : 0);
      double* p2 = sc.poses2 + (st2 ? 6 * e0 : 0);
      if (st1)
        cuda_check(cudaMemcpyAsync(p1, poses1_host + 6 * e0, sizeof(double) * 6 * ne, cudaMemcpyHostToDevice, q),
                   "H2D poses1");
      if (st2)
        cuda_check(cudaMemcpyAsync(p2, poses2_host + 6 * e0, sizeof(double) * 6 * ne, cudaMemcpyHostToDevice, q),
                   "H2D poses2");
      // n == 1 chunks keep stride semantics: a single-env chunk with st = 1 is one pose
      cmgb_manifold_out out{sc.contacts + e0 * C * 8, src_host ? sc.src + e0 * C * 2 : nullptr,
                            ee_host ? sc.ee + e0 * 9 * P : nullptr, sc.mean + e0,
                            sc.frames + (c & 1) * workspace_doubles(per, st1, st2),
                            workspace_doubles(per, st1, st2) * sizeof(double), nullptr, nullptr, 0.0f, 0};
      LaunchPlan plan = plan_manifold(s1, s2, p1, st1, p2, st2, ne, cfg, &out);
      launch_with_workspace(plan, ne, st1, st2, out.workspace, out.workspace_bytes, q);
      if (mean_dist_host)
        cuda_check(cudaMemcpyAsync(mean_dist_host + e0, sc.mean + e0, sizeof(float) * ne, cudaMemcpyDeviceToHost, q),
                   "D2H mean");
      if (contacts_host)
        cuda_check(cudaMemcpyAsync(contacts_host + e0 * C * 8, sc.contacts + e0 * C * 8, sizeof(float) * ne * C * 8,
                                   cudaMemcpyDeviceToHost, q),
                   "D2H contacts");
      if (src_host)
        cuda_check(cudaMemcpyAsync(src_host + e0 * C * 2, sc.src + e0 * C * 2, sizeof(int32_t) * ne * C * 2,
                                   cudaMemcpyDeviceToHost, q),
                   "D2H src");
      if (ee_host)
        cuda_check(cudaMemcpyAsync(ee_host + e0 * 9 * P, sc.ee + e0 * 9 * P, sizeof(float) * ne * 9 * P,
                                   cudaMemcpyDeviceToHost, q),
                   "D2H ee");
    }
    for (int k = 0; k < 2; ++k) {
      cuda_check(cudaEventRecord(sc.ev[k], sc.q[k]), "cudaEventRecord");
      cuda_check(cudaStreamWaitEvent(s, sc.ev[k], 0), "cudaStreamWaitEvent");
    }
    cuda_check(cudaStreamSynchronize(s), "cudaStreamSynchronize");
  });
}

int cmgb_manifold_batch_host(cmgb_surface s1, cmgb_surface s2, const double* poses1_host,
                             int32_t st1, const double* poses2_host, int32_t st2, int64_t n_env,
                             const cmgb_config* cfg, float* mean_dist_host, float* contacts_host,
                             void* stream) {
  const cmgb_manifold_out o{contacts_host, nullptr, nullptr, mean_dist_host, nullptr, 0, nullptr, nullptr, 0.0f, 0};
  return cmgb_manifold_batch_host_ex(s1, s2, poses1_host, st1, poses2_host, st2, n_env, cfg, &o, stream);
}

// ---- active-contact compaction -----------------------------------------------------
size_t cmgb_compact_workspace_bytes(int64_t n_env, int32_t n_contacts) {
  return n_env > 0 && n_contacts > 0 ? compact_workspace_bytes(n_env, n_contacts) : 0;
}

int cmgb_compact_contacts(const float* contacts, const int32_t* src, int64_t n_env, int32_t n_contacts,
                          float thr, const cmgb_compact_out* out, void* stream) {
  return guarded([&] {
    if (!out) invalid("compact: null output descriptor");
    if (n_env < 0 || n_contacts < 0) invalid("compact: n_env >= 0 and n_contacts >= 0");
    if (out->capacity < 0) invalid("compact: capacity >= 0");
    if (!(thr == thr)) invalid("compact: activity_threshold must not be NaN");
    if (out->src && !src) invalid("compact: src output needs the batch's src input");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (n_env == 0 || n_contacts == 0) {
      if (out->total) cuda_check(cudaMemsetAsync(out->total, 0, sizeof(int64_t), s), "cudaMemsetAsync");
      if (out->env_offset)
        cuda_check(cudaMemsetAsync(out->env_offset, 0, sizeof(int64_t) * (n_env + 1), s), "cudaMemsetAsync");
      if (out->env_count) cuda_check(cudaMemsetAsync(out->env_count, 0, sizeof(int32_t) * n_env, s), "cudaMemsetAsync");
      return;
    }
    if (!contacts) invalid("compact: null contacts");
    if (!out->contacts && out->capacity > 0) invalid("compact: null output contacts");
    // the fixed layout is staged by cp.async.bulk: 16-byte aligned source
    if (reinterpret_cast<uintptr_t>(contacts) % 16 != 0) invalid("compact: contacts must be 16-byte aligned");
    const size_t need = compact_workspace_bytes(n_env, n_contacts);
    void* ws = out->workspace;
    const bool pooled = !ws || out->workspace_bytes < need;
    if (pooled) cuda_check(scratch_alloc(&ws, need, s), "cudaMallocAsync(compact workspace)");
    const int rc = launch_compact(contacts, src, n_env, n_contacts, thr, out->capacity, out->contacts, out->slot,
                                  out->src, out->env_offset, out->env_count, out->total, ws, s);
    if (pooled) cudaFreeAsync(ws, s);
    if (rc != 0)
      throw Error(CMGB_ERR_CUDA, std::string("compact launch: ") + cudaGetErrorString(cudaGetLastError()));
  });
}

size_t cmgb_compact_masked_workspace_bytes(int64_t n_env) {
  return n_env > 0 ? compact_masked_workspace_bytes(n_env) : 0;
}

int cmgb_compact_masked(const float* contacts, const int32_t* src, int64_t n_env, int32_t n_contacts,
                        const uint32_t* mask, const int32_t* count, const cmgb_compact_out* out, void* stream) {
  return guarded([&] {
    if (!out) invalid("compact: null output descriptor");
    if (n_env < 0 || n_contacts < 0) invalid("compact: n_env >= 0 and n_contacts >= 0");
    if (out->capacity < 0) invalid("compact: capacity >= 0");
    if (out->src && !src) invalid("compact: src output needs the batch's src input");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (n_env == 0 || n_contacts == 0) {
      if (out->total) cuda_check(cudaMemsetAsync(out->total, 0, sizeof(int64_t), s), "cudaMemsetAsync");
      if (out->env_offset)
        cuda_check(cudaMemsetAsync(out->env_offset, 0, sizeof(int64_t) * (n_env + 1), s), "cudaMemsetAsync");
      if (out->env_count) cuda_check(cudaMemsetAsync(out->env_count, 0, sizeof(int32_t) * n_env, s), "cudaMemsetAsync");
      return;
    }
    if (!contacts || !mask || !count) invalid("compact: null contacts / mask / count");
    if (!out->contacts && out->capacity > 0) invalid("compact: null output contacts");
    if (reinterpret_cast<uintptr_t>(contacts) % 16 != 0) invalid("compact: contacts must be 16-byte aligned");
    const size_t need = compact_masked_workspace_bytes(n_env);
    void* ws = out->workspace;
    const bool pooled = !ws || out->workspace_bytes < need;
    if (pooled) cuda_check(scratch_alloc(&ws, need, s), "cudaMallocAsync(compact workspace)");
    const int rc = launch_compact_masked(contacts, src, n_env, n_contacts, mask, count, out->capacity, out->contacts,
                                         out->slot, out->src, out->env_offset, out->env_count, out->total, ws, s);
    if (pooled) cudaFreeAsync(ws, s);
    if (rc != 0)
      throw Error(CMGB_ERR_CUDA, std::string("compact launch: ") + cudaGetErrorString(cudaGetLastError()));
  });
}

// ---- pose Jacobians (Dual12 forward mode) -------------------------------------------
namespace {

void validate_jvp(const cmgb_config* cfg, const cmgb_manifold_jvp_out* out) {
  if (!out) invalid("manifold_jvp: null output descriptor");
  validate_config(cfg);
  if (cfg->hard_ops)
    throw Error(CMGB_ERR_UNSUPPORTED,
                "manifold_jvp: hard_ops has no derivative path (the reference's hard operators are double-only)");
}

// JVP launch plan on top of a value plan: per-unit dual working set and units
// per CTA (~one CTA's worth of E-E pairs, within the kernel's shared-memory
// budget per CTA).
JvpParams plan_jvp(const LaunchPlan& plan, const cmgb_manifold_jvp_out* out) {
  JvpParams j{};
  j.m = plan.p;
  j.tangents = out->tangents;
  j.mean_grad = out->mean_dist_grad;
  j.mean_f64 = out->mean_dist_f64;
  j.mean_grad_f64 = out->mean_dist_grad_f64;
  // One unit = one env carrying all 12 pose directions (manifold_jvp.cu).
  // Tangent records: FP64 primal + 12 FP32 tangents (56 B). The top-K scores /
  // order / row weights are dead after the slot phase and share their bytes
  // with the pair side-Jacobian / QP records (E1 -> E2).
  j.nd = jvp_directions();
  j.groups = 1;
  const ManifoldParams& m = j.m;
  const int T = 8 + 12 * 4;                  // bytes per tangent record
  const int SJ = 33 * 8, QP = 19 * 8, AUX = 16, VS = 19 * 8, PR = 17 * 8;  // manifold_jvp.cuh records
  const int FRAMES = 2 * 12 * 8 + 12 * 7 * 8;  // 2 x Frame + 12 x Vel
  const int P = m.m1 * m.m2, nslot_v = m.n1 + m.n2, nslot_e = m.m1 + m.m2, nsl = nslot_v + nslot_e;
  const bool topk = m.side[0].topk_v || m.side[1].topk_v || m.side[0].topk_e || m.side[1].topk_e;
  const int nscore = topk ? (m.side[0].nv + m.side[1].nv + m.side[0].ne + m.side[1].ne) : 0;
  int dmax = 0;
  for (int k = 0; k < 2; ++k) {
    if (m.side[k].topk_v) dmax = std::max(dmax, m.side[k].nv);
    if (m.side[k].topk_e) dmax = std::max(dmax, m.side[k].ne);
  }
  j.ebuf_stride = dmax;
  int off = 0;
  j.o_frames = off; off = align16(off + FRAMES);
  j.o_vslots = off; off = align16(off + nslot_v * 3 * T);
  j.o_eslots = off; off = align16(off + nslot_e * (48 + 6 * T + 8));  // ESlot
  j.o_prov = off; off = align16(off + nsl * 4);
  j.o_pairs = off; off = align16(off + P * (4 * T + 8));  // 4 records + 8 B: odd 8-byte stride per pair
  j.o_vsdist = off; off = align16(off + nslot_v * T);
  j.o_nnstat = off; off = align16(off + nslot_e * 2 * T);
  const int u0 = off;
  j.o_scores = off; off = align16(off + nscore * T);
  j.o_sorted = off; off = align16(off + nscore * 4);
  j.o_aux = off; off = align16(off + (topk ? nsl * AUX : 0));
  j.o_ebuf = off; off = align16(off + nsl * dmax * 4);
  const int end_topk = off;
  off = u0;
  j.o_sj = off; off = align16(off + 2 * P * SJ);
  j.o_qp = off; off = align16(off + P * QP);
  j.o_vsrec = off; off = align16(off + nslot_v * VS);
  j.o_prec = off; off = align16(off + P * PR);
  j.bytes = std::max(off, end_topk);
  if (j.bytes > smem_optin_per_block())
    throw Error(CMGB_ERR_UNSUPPORTED, "manifold_jvp: per-env dual working set exceeds shared memory");
  // E1 items: 2 sides + 1 QP per pair, 1 per V-S contact; as many envs per CTA
  // as its shared-memory budget holds (about 2 passes of items)
  const int per_unit = std::max(3 * P + nslot_v, 1);
  j.geom_bytes = align16(8 * (3 * (m.side[0].nv + m.side[1].nv) + 6 * (m.side[0].ne + m.side[1].ne)));
  if (j.bytes + j.geom_bytes > smem_optin_per_block())
    throw Error(CMGB_ERR_UNSUPPORTED, "manifold_jvp: per-env dual working set exceeds shared memory");
  int upb = std::max(1, (2 * jvp_max_threads() + per_unit - 1) / per_unit);
  while (upb > 1 && (size_t)upb * j.bytes + j.geom_bytes > (size_t)jvp_smem_cap()) --upb;
  j.units_per_block = upb;
  if ((m.n_env + upb - 1) / upb > 0x7fffffffLL) invalid("manifold_jvp: n_env too large for one launch");
  return j;
}

void launch_jvp(const JvpParams& j, cudaStream_t s) {
  if (launch_manifold_jvp(j, 0, s) != 0)
    throw Error(CMGB_ERR_CUDA, std::string("manifold_jvp launch: ") + cudaGetErrorString(cudaGetLastError()));
}

}  // namespace

int cmgb_manifold_jvp_batch(cmgb_surface s1, cmgb_surface s2, const double* poses1, int32_t st1,
                            const double* poses2, int32_t st2, int64_t n_env, const cmgb_config* cfg,
                            const cmgb_manifold_jvp_out* out, void* stream) {
  return guarded([&] {
    validate_jvp(cfg, out);
    cmgb_manifold_out mo{out->contacts, out->src, nullptr, out->mean_dist, nullptr, 0, nullptr, nullptr, 0.0f, 0};
    LaunchPlan plan = plan_manifold(s1, s2, poses1, st1, poses2, st2, n_env, cfg, &mo);
    if (n_env == 0 || plan.p.n_contacts == 0) return;
    if (!out->contacts || !out->tangents) invalid("manifold_jvp: contacts and tangents outputs are required");
    launch_jvp(plan_jvp(plan, out), static_cast<cudaStream_t>(stream));
  });
}

// Host-buffer form of the pose-Jacobian batch: device buffers from the stream-
// ordered pool for the duration of the call, synchronised before returning.
namespace {

struct PoolBuffers {  // cudaMallocAsync blocks released in order on the stream (also on error)
  cudaStream_t s;
  std::vector<void*> bufs;
  explicit PoolBuffers(cudaStream_t st) : s(st) {}
  void* get(size_t bytes) {
    void* p = nullptr;
    cuda_check(scratch_alloc(&p, std::max<size_t>(bytes, 16), s), "cudaMallocAsync");
    bufs.push_back(p);
    return p;
  }
  ~PoolBuffers() {
    for (void* p : bufs) cudaFreeAsync(p, s);
    cudaStreamSynchronize(s);
  }
};

void h2d(void* dst, const void* src, size_t bytes, cudaStream_t s) {
  cuda_check(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s), "H2D");
}
void d2h(void* dst, const void* src, size_t bytes, cudaStream_t s) {
  if (dst) cuda_check(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s), "D2H");
}

// Host-buffer witness batches with reference-precision outputs (run_ee_batch /
// run_vf_batch, src/batch.cpp:53-98, return doubles): E-E through the FP64
// solver; V-F through the FP32-output solver, widened on the device. Both run
// as a two-stream pipeline over pair chunks: chunk c+1's upload overlaps chunk
// c's kernel and download (one copy engine per direction), joined back into the
// caller's stream. The pairs are PCIe-bound (96 B in per pair): with pinned
// host buffers the outputs' download hides behind the uploads.
constexpr int kWitnessChunks = 8;
constexpr int64_t kWitnessChunkMin = 65536;

extern "C++" {  // a template inside the extern "C" block
// chunk(e0, ne, stream) for each [bounds[c], bounds[c + 1]) on the two
// pipeline streams alternately, ordered after s and joined back into it
template <class Chunk>
void host_pipeline(const std::vector<int64_t>& bounds, cudaStream_t s, Chunk&& chunk) {
  int dev = 0;
  cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
  ScratchLease lease(dev);
  HostScratch& sc = *lease.sc;
  ensure_pipeline(sc);
  cuda_check(cudaEventRecord(sc.ev_start, s), "cudaEventRecord");
  for (int q = 0; q < 2; ++q) cuda_check(cudaStreamWaitEvent(sc.q[q], sc.ev_start, 0), "cudaStreamWaitEvent");
  for (size_t c = 0; c + 1 < bounds.size(); ++c) {
    const int64_t e0 = bounds[c], ne = bounds[c + 1] - e0;
    if (ne > 0) chunk(e0, ne, sc.q[c & 1]);
  }
  for (int q = 0; q < 2; ++q) {
    cuda_check(cudaEventRecord(sc.ev[q], sc.q[q]), "cudaEventRecord");
    cuda_check(cudaStreamWaitEvent(s, sc.ev[q], 0), "cudaStreamWaitEvent");
  }
}
template <class Chunk>
void witness_pipeline(int64_t n, cudaStream_t s, Chunk&& chunk) {
  const int64_t k = std::max<int64_t>(1, std::min<int64_t>(kWitnessChunks, n / kWitnessChunkMin));
  std::vector<int64_t> bounds;
  for (int64_t c = 0; c <= k; ++c) bounds.push_back(n * c / k);
  host_pipeline(bounds, s, chunk);
}
}  // extern "C++"

}  // namespace

int cmgb_manifold_jvp_batch_host(cmgb_surface s1, cmgb_surface s2, const double* poses1_host, int32_t st1,
                                 const double* poses2_host, int32_t st2, int64_t n_env, const cmgb_config* cfg,
                                 const cmgb_manifold_jvp_out* host_out, void* stream) {
  return guarded([&] {
    validate_jvp(cfg, host_out);
    if (!s1 || !s2) invalid("manifold_jvp_batch_host: null surface");
    if ((st1 != 0 && st1 != 1) || (st2 != 0 && st2 != 1)) invalid("manifold: pose stride must be 0 or 1");
    if (n_env == 0) return;
    if (n_env < 0) invalid("manifold: n_env >= 0");
    if (!poses1_host || !poses2_host) invalid("manifold_jvp_batch_host: null poses");
    if (!host_out->contacts || !host_out->tangents)
      invalid("manifold_jvp: contacts and tangents outputs are required");
    const cmgb_layout L = layout_of(s1, s2, cfg);
    const size_t n = (size_t)n_env, C = (size_t)L.n_contacts;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    PoolBuffers pb(s);
    const size_t np1 = (st1 ? n : 1) * 6, np2 = (st2 ? n : 1) * 6;
    double* p1 = static_cast<double*>(pb.get(sizeof(double) * (np1)));
    double* p2 = static_cast<double*>(pb.get(sizeof(double) * (np2)));
    h2d(p1, poses1_host, sizeof(double) * np1, s);
    h2d(p2, poses2_host, sizeof(double) * np2, s);
    cmgb_manifold_jvp_out d{};
    d.contacts = static_cast<float*>(pb.get(sizeof(float) * (n * C * 8)));
    d.tangents = static_cast<float*>(pb.get(sizeof(float) * (n * C * 96)));
    d.src = host_out->src ? static_cast<int32_t*>(pb.get(sizeof(int32_t) * (n * C * 2))) : nullptr;
    d.mean_dist = host_out->mean_dist ? static_cast<float*>(pb.get(sizeof(float) * (n))) : nullptr;
    d.mean_dist_grad = host_out->mean_dist_grad ? static_cast<float*>(pb.get(sizeof(float) * (n * 12))) : nullptr;
    d.mean_dist_f64 = host_out->mean_dist_f64 ? static_cast<double*>(pb.get(sizeof(double) * (n))) : nullptr;
    d.mean_dist_grad_f64 = host_out->mean_dist_grad_f64 ? static_cast<double*>(pb.get(sizeof(double) * (n * 12))) : nullptr;
    cmgb_manifold_out mo{d.contacts, d.src, nullptr, d.mean_dist, nullptr, 0, nullptr, nullptr, 0.0f, 0};
    LaunchPlan plan = plan_manifold(s1, s2, p1, st1, p2, st2, n_env, cfg, &mo);
    if (plan.p.n_contacts == 0) return;
    launch_jvp(plan_jvp(plan, &d), s);
    d2h(host_out->contacts, d.contacts, sizeof(float) * n * C * 8, s);
    d2h(host_out->tangents, d.tangents, sizeof(float) * n * C * 96, s);
    if (d.src) d2h(host_out->src, d.src, sizeof(int32_t) * n * C * 2, s);
    if (d.mean_dist) d2h(host_out->mean_dist, d.mean_dist, sizeof(float) * n, s);
    if (d.mean_dist_grad) d2h(host_out->mean_dist_grad, d.mean_dist_grad, sizeof(float) * n * 12, s);
    if (d.mean_dist_f64) d2h(host_out->mean_dist_f64, d.mean_dist_f64, sizeof(double) * n, s);
    if (d.mean_dist_grad_f64)
      d2h(host_out->mean_dist_grad_f64, d.mean_dist_grad_f64, sizeof(double) * n * 12, s);
  });
}

int cmgb_ee_witness_batch_host(const double* pairs_host, int64_t n, const cmgb_config* cfg, double* out_host,
                               int32_t* labels_host, void* stream) {
  return guarded([&] {
    validate_config(cfg);
    if (n < 0) invalid("ee_witness_batch_host: n >= 0");
    if (n == 0) return;
    if (!pairs_host || !out_host) invalid("ee_witness_batch_host: null buffer");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    PoolBuffers pb(s);  // freed after the join, then synchronised
    double* pairs = static_cast<double*>(pb.get(sizeof(double) * ((size_t)n * 12)));
    double* out = static_cast<double*>(pb.get(sizeof(double) * ((size_t)n * 6)));
    int32_t* labels = labels_host ? static_cast<int32_t*>(pb.get(sizeof(int32_t) * ((size_t)n))) : nullptr;
    const DevCfg dc = device_config(cfg);
    witness_pipeline(n, s, [&](int64_t e0, int64_t ne, cudaStream_t q) {
      h2d(pairs + 12 * e0, pairs_host + 12 * e0, sizeof(double) * 12 * ne, q);
      WitnessParams p{pairs + 12 * e0, 1, ne, dc, out + 6 * e0, nullptr, labels ? labels + e0 : nullptr, nullptr};
      if (launch_ee_witness_f64(p, q) != 0)
        throw Error(CMGB_ERR_CUDA, std::string("ee_witness_f64 launch: ") + cudaGetErrorString(cudaGetLastError()));
      d2h(out_host + 6 * e0, out + 6 * e0, sizeof(double) * 6 * ne, q);
      if (labels) d2h(labels_host + e0, labels + e0, sizeof(int32_t) * ne, q);
    });
  });
}

int cmgb_vf_witness_batch_host(const double* pairs_host, int64_t n, const cmgb_config* cfg, double* out_host,
                               int32_t* labels_host, void* stream) {
  return guarded([&] {
    validate_config(cfg);
    if (n < 0) invalid("vf_witness_batch_host: n >= 0");
    if (n == 0) return;
    if (!pairs_host || !out_host) invalid("vf_witness_batch_host: null buffer");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    PoolBuffers pb(s);
    double* pairs = static_cast<double*>(pb.get(sizeof(double) * ((size_t)n * 12)));
    float* out = static_cast<float*>(pb.get(sizeof(float) * ((size_t)n * 3)));
    double* wide = static_cast<double*>(pb.get(sizeof(double) * ((size_t)n * 3)));
    int32_t* labels = labels_host ? static_cast<int32_t*>(pb.get(sizeof(int32_t) * ((size_t)n))) : nullptr;
    const DevCfg dc = device_config(cfg);
    witness_pipeline(n, s, [&](int64_t e0, int64_t ne, cudaStream_t q) {
      h2d(pairs + 12 * e0, pairs_host + 12 * e0, sizeof(double) * 12 * ne, q);
      WitnessParams p{pairs + 12 * e0, 1, ne, dc, out + 3 * e0, nullptr, labels ? labels + e0 : nullptr, nullptr};
      if (launch_vf_witness(p, q) != 0)
        throw Error(CMGB_ERR_CUDA, std::string("vf_witness launch: ") + cudaGetErrorString(cudaGetLastError()));
      if (launch_widen(out + 3 * e0, wide + 3 * e0, 3 * ne, q) != 0)
        throw Error(CMGB_ERR_CUDA, std::string("widen launch: ") + cudaGetErrorString(cudaGetLastError()));
      d2h(out_host + 3 * e0, wide + 3 * e0, sizeof(double) * 3 * ne, q);
      if (labels) d2h(labels_host + e0, labels + e0, sizeof(int32_t) * ne, q);
    });
  });
}

int cmgb_manifold_scene_jvp_batch(const cmgb_surface* bodies, int32_t n_bodies, const int32_t* pairs,
                                  int32_t n_pairs, const double* poses, int64_t n_env,
                                  const cmgb_config* cfg, const cmgb_manifold_jvp_out* outs, void* stream) {
  return guarded([&] {
    if (!bodies || !outs || n_bodies < 1 || n_pairs < 0 || n_env < 0 || (n_pairs > 0 && !pairs) ||
        (n_env > 0 && !poses))
      invalid("manifold_scene_jvp_batch: bad argument");
    std::vector<JvpParams> plans;
    for (int q = 0; q < n_pairs; ++q) {
      const int i = pairs[2 * q], j = pairs[2 * q + 1];
      if (i < 0 || j < 0 || i >= n_bodies || j >= n_bodies || i == j)
        invalid("manifold_scene_jvp_batch: pair index out of range");
      const cmgb_manifold_jvp_out& o = outs[q];
      validate_jvp(cfg, &o);
      cmgb_manifold_out mo{o.contacts, o.src, nullptr, o.mean_dist, nullptr, 0, nullptr, nullptr, 0.0f, 0};
      LaunchPlan plan = plan_manifold(bodies[i], bodies[j], poses + 6 * i, 1, poses + 6 * j, 1, n_env, cfg, &mo);
      if (n_env == 0 || plan.p.n_contacts == 0) continue;
      if (!o.contacts || !o.tangents) invalid("manifold_jvp: contacts and tangents outputs are required");
      plan.p.pose_stride1 = plan.p.pose_stride2 = 6 * (int64_t)n_bodies;
      plans.push_back(plan_jvp(plan, &o));
    }
    // (one stream: measured, concurrent JVP pairs on side streams run 0.5% slower)
    for (const JvpParams& j : plans) launch_jvp(j, static_cast<cudaStream_t>(stream));
  });
}

// ---- SDF queries / sphere tracing ---------------------------------------------------
int cmgb_sdf_query(cmgb_surface s, int32_t flavor, const double* points, int64_t n, double* out, void* stream) {
  return guarded([&] {
    if (!s) invalid("sdf_query: null surface");
    if (flavor < 0 || flavor > 2) invalid("sdf_query: flavor must be 0 (value), 1 (gradient) or 2 (normal source)");
    if (n < 0) invalid("sdf_query: n >= 0");
    if (n == 0) return;
    if (!points || !out) invalid("sdf_query: null buffer");
    SdfQueryParams q{};
    q.sdf = device_image(s).sdf;
    q.points = points;
    q.n = n;
    q.out = out;
    if (launch_sdf_query(q, flavor, stream) != 0)
      throw Error(CMGB_ERR_CUDA, std::string("sdf_query launch: ") + cudaGetErrorString(cudaGetLastError()));
  });
}

int cmgb_sphere_trace(cmgb_surface s, const double* pose_host, const double* points, int64_t n, int32_t iters,
                      double tau, double* out, void* stream) {
  return guarded([&] {
    if (!s || !pose_host) invalid("sphere_trace: null surface or pose");
    if (n < 0 || iters < 0) invalid("sphere_trace: n >= 0 and iters >= 0");
    if (n == 0) return;
    if (!points || !out) invalid("sphere_trace: null buffer");
    SdfQueryParams q{};
    q.sdf = device_image(s).sdf;
    q.points = points;
    q.n = n;
    q.out = out;
    q.iters = iters;
    q.tau = tau;
    se3_exp_host(pose_host, q.R, q.t);
    if (launch_sdf_query(q, 3, stream) != 0)
      throw Error(CMGB_ERR_CUDA, std::string("sphere_trace launch: ") + cudaGetErrorString(cudaGetLastError()));
  });
}

// ---- witness batches --------------------------------------------------------------
int cmgb_ee_witness_batch(const void* pairs, int32_t fp64, int64_t n, const cmgb_config* cfg,
                          float* out, float* alpha_gamma, int32_t* labels, void* stream) {
  return guarded([&] {
    validate_config(cfg);
    if (n < 0) invalid("ee_witness_batch: n >= 0");
    if (n == 0) return;
    if (!pairs || !out) invalid("ee_witness_batch: null buffer");
    // input tiles arrive by cp.async.bulk, which needs a 16-byte aligned source
    if (reinterpret_cast<uintptr_t>(pairs) % 16 != 0) invalid("ee_witness_batch: pairs must be 16-byte aligned");
    WitnessParams p{pairs, fp64 ? 1 : 0, n, device_config(cfg), out, alpha_gamma, labels, nullptr};
    if (launch_ee_witness(p, stream) != 0)
      throw Error(CMGB_ERR_CUDA, std::string("ee_witness launch: ") + cudaGetErrorString(cudaGetLastError()));
  });
}

int cmgb_ee_witness_batch_f64(const double* pairs, int64_t n, const cmgb_config* cfg, double* out,
                              double* alpha_gamma, int32_t* labels, void* stream) {
  return guarded([&] {
    validate_config(cfg);
    if (n < 0) invalid("ee_witness_batch_f64: n >= 0");
    if (n == 0) return;
    if (!pairs || !out) invalid("ee_witness_batch_f64: null buffer");
    if (reinterpret_cast<uintptr_t>(pairs) % 16 != 0) invalid("ee_witness_batch_f64: pairs must be 16-byte aligned");
    WitnessParams p{pairs, 1, n, device_config(cfg), out, nullptr, labels, alpha_gamma};
    if (launch_ee_witness_f64(p, stream) != 0)
      throw Error(CMGB_ERR_CUDA, std::string("ee_witness_f64 launch: ") + cudaGetErrorString(cudaGetLastError()));
  });
}

// Rotating-edge sweep (src/sweep.cpp:17-56): edge 1 = +/-(sin t, cos t, 0), edge 2
// = x in [-2, 2] at y = -1.2; witness p1 and its central difference (h = 1e-7)
// for n_samples angles over [0, pi], all 3 n_samples QPs in one FP64 launch.
int cmgb_rotating_edge_sweep(int32_t variant, int32_t n_samples, double* out_host) {
  return guarded([&] {
    if (variant < 0 || variant > 2) invalid("rotating_edge_sweep: variant must be 0 (no smoothing), 1 (l2), 2 (smooth)");
    if (n_samples < 2 || !out_host) invalid("rotating_edge_sweep: n_samples >= 2 and an output buffer");
    cmgb_config cfg;
    cmgb_config_default(&cfg);
    if (variant == 0) {
      cmgb_config_no_smoothing(&cfg);
    } else if (variant == 1) {
      cmgb_config_no_smoothing(&cfg);
      cfg.lambda = 0.01;
    } else {
      cfg.lambda = 0.01;
      cfg.tau_clip = cfg.tau_min = cfg.tau_comp = 0.1;
    }
    const double h = 1e-7;
    const double pi = 3.14159265358979323846;
    std::vector<double> pairs((size_t)n_samples * 3 * 12);
    std::vector<double> theta(n_samples);
    for (int i = 0; i < n_samples; ++i) {
      theta[i] = pi * i / (n_samples - 1);
      const double th3[3] = {theta[i], theta[i] + h, theta[i] - h};
      for (int k = 0; k < 3; ++k) {
        double* q = pairs.data() + ((size_t)i * 3 + k) * 12;
        const double sx = std::sin(th3[k]), cy = std::cos(th3[k]);
        q[0] = -sx; q[1] = -cy; q[2] = -0.0;
        q[3] = sx; q[4] = cy; q[5] = 0.0;
        q[6] = -2.0; q[7] = -1.2; q[8] = 0.0;
        q[9] = 2.0; q[10] = -1.2; q[11] = 0.0;
      }
    }
    const size_t np = pairs.size() / 12;
    double *d_pairs = nullptr, *d_out = nullptr;
    cuda_check(cudaMalloc(&d_pairs, sizeof(double) * pairs.size()), "cudaMalloc");
    cuda_check(cudaMalloc(&d_out, sizeof(double) * np * 6), "cudaMalloc");
    std::vector<double> res(np * 6);
    int rc = cudaMemcpy(d_pairs, pairs.data(), sizeof(double) * pairs.size(), cudaMemcpyHostToDevice);
    WitnessParams p{d_pairs, 1, (int64_t)np, device_config(&cfg), d_out, nullptr, nullptr, nullptr};
    if (rc == cudaSuccess) rc = launch_ee_witness_f64(p, nullptr) == 0 ? cudaSuccess : cudaErrorLaunchFailure;
    if (rc == cudaSuccess) rc = cudaMemcpy(res.data(), d_out, sizeof(double) * np * 6, cudaMemcpyDeviceToHost);
    cudaFree(d_pairs);
    cudaFree(d_out);
    if (rc != cudaSuccess) throw Error(CMGB_ERR_CUDA, "rotating_edge_sweep: CUDA failure");
    for (int i = 0; i < n_samples; ++i) {
      const double* c = res.data() + (size_t)i * 18;
      double* o = out_host + (size_t)i * 7;
      o[0] = theta[i];
      for (int k = 0; k < 3; ++k) {
        o[1 + k] = c[k];                                  // p1(theta)
        o[4 + k] = (c[6 + k] - c[12 + k]) / (2.0 * h);    // (p1(t+h) - p1(t-h)) / 2h
      }
    }
  });
}

int cmgb_vf_witness_batch(const void* pairs, int32_t fp64, int64_t n, const cmgb_config* cfg,
                          float* out, int32_t* labels, void* stream) {
  return guarded([&] {
    validate_config(cfg);
    if (n < 0) invalid("vf_witness_batch: n >= 0");
    if (n == 0) return;
    if (!pairs || !out) invalid("vf_witness_batch: null buffer");
    // input tiles arrive by cp.async.bulk, which needs a 16-byte aligned source
    if (reinterpret_cast<uintptr_t>(pairs) % 16 != 0) invalid("vf_witness_batch: pairs must be 16-byte aligned");
    WitnessParams p{pairs, fp64 ? 1 : 0, n, device_config(cfg), out, nullptr, labels, nullptr};
    if (launch_vf_witness(p, stream) != 0)
      throw Error(CMGB_ERR_CUDA, std::string("vf_witness launch: ") + cudaGetErrorString(cudaGetLastError()));
  });
}

int cmgb_scene_pairs(const int32_t* is_static, int32_t n_bodies, int32_t* pairs, int32_t* n_pairs) {
  return guarded([&] {
    if (n_bodies < 0 || !n_pairs) invalid("scene_pairs: bad argument");
    int32_t k = 0;
    for (int i = 0; i < n_bodies; ++i)
      for (int j = i + 1; j < n_bodies; ++j) {
        if (is_static && is_static[i] && is_static[j]) continue;  // demosim.cpp:90
        if (pairs) {
          pairs[2 * k] = i;
          pairs[2 * k + 1] = j;
        }
        ++k;
      }
    *n_pairs = k;
  });
}

namespace {

// every (env, body) frame once (the pairs share bodies), then the pairs on the
// device's side streams, joined back into s (throws)
void scene_batch(const cmgb_surface* bodies, int32_t n_bodies, const int32_t* pairs, int32_t n_pairs,
                 const double* poses, int64_t n_env, const cmgb_config* cfg, const cmgb_manifold_out* outs,
                 cudaStream_t s) {
  if (!bodies || !outs || n_bodies < 1 || n_pairs < 0 || n_env < 0 || (n_pairs > 0 && !pairs) ||
      (n_env > 0 && !poses))
    invalid("manifold_scene_batch: bad argument");
  std::vector<LaunchPlan> plans;
  std::vector<std::pair<int, int>> ij;
  for (int q = 0; q < n_pairs; ++q) {
    const int i = pairs[2 * q], j = pairs[2 * q + 1];
    if (i < 0 || j < 0 || i >= n_bodies || j >= n_bodies || i == j)
      invalid("manifold_scene_batch: pair index out of range");
    LaunchPlan plan = plan_manifold(bodies[i], bodies[j], poses + 6 * i, 1, poses + 6 * j, 1, n_env, cfg, &outs[q]);
    if (n_env == 0 || plan.p.n_contacts == 0) continue;
    plans.push_back(plan);
    ij.emplace_back(i, j);
  }
  if (plans.empty()) return;
  double* frames = nullptr;
  cuda_check(scratch_alloc(reinterpret_cast<void**>(&frames), sizeof(double) * 12 * (size_t)n_env * n_bodies, s),
             "cudaMallocAsync(scene frames)");
  if (launch_scene_frames(poses, n_env * n_bodies, frames, s) != 0) {
    cudaFreeAsync(frames, s);
    throw Error(CMGB_ERR_CUDA, std::string("frames launch: ") + cudaGetErrorString(cudaGetLastError()));
  }
  try {
    StreamFork fork(s, (int)plans.size());  // the pairs overlap each other's tails
    for (size_t k = 0; k < plans.size(); ++k) {
      LaunchPlan& plan = plans[k];
      plan.p.pose_stride1 = plan.p.pose_stride2 = 6 * (int64_t)n_bodies;
      plan.p.frames1 = frames + 12 * ij[k].first;
      plan.p.frames2 = frames + 12 * ij[k].second;
      plan.p.stride1 = plan.p.stride2 = n_bodies;
      plan.p.frames_ready = 1;
      launch_planned(plan, n_env, fork.stream((int)k));
    }
  } catch (...) {
    cudaFreeAsync(frames, s);
    throw;
  }
  cudaFreeAsync(frames, s);  // after the fork's join
}

}  // namespace

int cmgb_manifold_scene_batch(const cmgb_surface* bodies, int32_t n_bodies, const int32_t* pairs,
                              int32_t n_pairs, const double* poses, int64_t n_env,
                              const cmgb_config* cfg, const cmgb_manifold_out* outs, void* stream) {
  return guarded([&] {
    scene_batch(bodies, n_bodies, pairs, n_pairs, poses, n_env, cfg, outs, static_cast<cudaStream_t>(stream));
  });
}

// Host-buffer scene batch: HOST poses [n_env][n_bodies][6] in, each pair's
// per-env mean distance [n_pairs][n_env] out. A lead chunk of the envs, then
// the rest, on the two pipeline streams: the rest's pose upload overlaps the
// lead chunk's kernels (as cmgb_manifold_batch_host).
int cmgb_manifold_scene_batch_host(const cmgb_surface* bodies, int32_t n_bodies, const int32_t* pairs,
                                   int32_t n_pairs, const double* poses_host, int64_t n_env,
                                   const cmgb_config* cfg, float* mean_dist_host, void* stream) {
  return guarded([&] {
    if (!bodies || n_bodies < 1 || n_pairs < 0 || n_env < 0 || (n_pairs > 0 && !pairs) ||
        (n_env > 0 && n_pairs > 0 && (!poses_host || !mean_dist_host)))
      invalid("manifold_scene_batch_host: bad argument");
    if (n_env == 0 || n_pairs == 0) return;
    validate_config(cfg);
    std::vector<size_t> C(n_pairs);
    for (int q = 0; q < n_pairs; ++q) {
      const int i = pairs[2 * q], j = pairs[2 * q + 1];
      if (i < 0 || j < 0 || i >= n_bodies || j >= n_bodies || i == j || !bodies[i] || !bodies[j])
        invalid("manifold_scene_batch: pair index out of range");
      C[q] = (size_t)layout_of(bodies[i], bodies[j], cfg).n_contacts;
    }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    PoolBuffers pb(s);  // freed after the join, then synchronised
    const size_t row = 6 * (size_t)n_bodies, n = (size_t)n_env;
    double* P = static_cast<double*>(pb.get(sizeof(double) * row * n));
    float* mean = static_cast<float*>(pb.get(sizeof(float) * n * n_pairs));
    std::vector<float*> contacts(n_pairs);
    for (int q = 0; q < n_pairs; ++q) contacts[q] = static_cast<float*>(pb.get(sizeof(float) * n * C[q] * 8));
    std::vector<int64_t> bounds = {0, n_env};
    if (n_env >= 2 * kHostChunkMin) bounds = {0, std::max(kHostChunkMin, n_env / 8), n_env};
    for (int q = 0; q < n_pairs; ++q)  // an empty layout's mean is 0 / 0 in the reference (manifold.hpp:379-384)
      if (C[q] == 0)
        cuda_check(cudaMemsetAsync(mean + (size_t)q * n, 0xFF, sizeof(float) * n, s), "cudaMemsetAsync");
    std::vector<cmgb_manifold_out> outs(n_pairs);
    host_pipeline(bounds, s, [&](int64_t e0, int64_t ne, cudaStream_t st) {
      h2d(P + row * e0, poses_host + row * e0, sizeof(double) * row * ne, st);
      for (int q = 0; q < n_pairs; ++q) {
        outs[q] = cmgb_manifold_out{};
        outs[q].contacts = contacts[q] + (size_t)e0 * C[q] * 8;
        outs[q].mean_dist = mean + (size_t)q * n + e0;
      }
      scene_batch(bodies, n_bodies, pairs, n_pairs, P + row * e0, ne, cfg, outs.data(), st);
      for (int q = 0; q < n_pairs; ++q)
        d2h(mean_dist_host + (size_t)q * n + e0, mean + (size_t)q * n + e0, sizeof(float) * ne, st);
    });
  });
}

// ---- batched demo integrator (DemoSim::step) -------------------------------------
void cmgb_demo_params_default(cmgb_demo_params* p) {
  if (!p) return;
  // PenaltyParams{} (include/cmg/demosim.hpp:24-31)
  p->stiffness = 1e4;
  p->damping = 100.0;
  p->friction = 0.5;
  p->friction_viscous = 100.0;
  p->tau_force = 1e-4;
  p->gravity[0] = 0.0;
  p->gravity[1] = 0.0;
  p->gravity[2] = -9.81;
}

namespace {

struct DemoPlan {
  std::vector<std::pair<int, int>> pairs;
  std::vector<int> C;              // contacts per pair
  std::vector<size_t> off_contacts, off_frames;
  size_t off_wrench = 0, off_deep = 0, bytes = 0;
};

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

DemoPlan plan_demo(const cmgb_demo_body* bodies, int32_t nb, const cmgb_config* cfg, int64_t n_env) {
  if (!bodies || nb < 1) invalid("demo: bodies required");
  if (nb > kDemoMaxBodies) invalid("demo: at most 16 bodies per scene");
  validate_config(cfg);
  if (n_env < 0) invalid("demo: n_env >= 0");
  DemoPlan d;
  for (int i = 0; i < nb; ++i) {
    if (!bodies[i].surface) invalid("demo: null surface");
    if (!(bodies[i].mass > 0.0)) invalid("demo: body mass must be > 0");
  }
  for (int i = 0; i < nb; ++i)
    for (int j = i + 1; j < nb; ++j)
      if (!(bodies[i].is_static && bodies[j].is_static)) d.pairs.emplace_back(i, j);
  size_t off = 0;
  for (const auto& [i, j] : d.pairs) {
    const cmgb_layout L = layout_of(bodies[i].surface, bodies[j].surface, cfg);
    d.C.push_back(L.n_contacts);
    d.off_contacts.push_back(off);
    off = align256(off + sizeof(float) * (size_t)n_env * L.n_contacts * 8);
    d.off_frames.push_back(off);
    off = align256(off + sizeof(double) * workspace_doubles(n_env, 1, 1));
  }
  d.off_wrench = off;
  off = align256(off + sizeof(double) * d.pairs.size() * (size_t)n_env * 12);
  d.off_deep = off;
  off = align256(off + sizeof(double) * d.pairs.size() * (size_t)n_env);
  d.bytes = std::max<size_t>(off, 256);
  return d;
}

}  // namespace

size_t cmgb_demo_workspace_bytes(const cmgb_demo_body* bodies, int32_t n_bodies, const cmgb_config* cfg,
                                 int64_t n_env) {
  try {
    return plan_demo(bodies, n_bodies, cfg, n_env).bytes;
  } catch (...) {
    return 0;
  }
}

int cmgb_demo_step_batch(const cmgb_demo_body* bodies, int32_t nb, const cmgb_config* cfg,
                         const cmgb_demo_params* prm, double dt, int64_t n_env, double* poses,
                         double* velocities, double* deepest, int32_t* ok, void* workspace,
                         size_t workspace_bytes, void* stream) {
  return guarded([&] {
    if (!prm) invalid("demo: null params");
    const DemoPlan d = plan_demo(bodies, nb, cfg, n_env);
    if (n_env == 0) return;
    if (!poses || !velocities) invalid("demo: poses and velocities are required");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    void* buf = workspace;
    const bool pooled = workspace == nullptr || workspace_bytes < d.bytes;
    if (pooled) cuda_check(scratch_alloc(&buf, d.bytes, s), "cudaMallocAsync(demo workspace)");
    unsigned char* base = static_cast<unsigned char*>(buf);
    DemoParamsDev P{prm->stiffness, prm->damping, prm->friction, prm->friction_viscous, prm->tau_force,
                    {prm->gravity[0], prm->gravity[1], prm->gravity[2]}};
    double* wrench = reinterpret_cast<double*>(base + d.off_wrench);
    double* pdeep = reinterpret_cast<double*>(base + d.off_deep);
    int rc = 0;
    {
    // the pairs (manifold + penalty each) on the device's side streams, joined
    // before the integrator
    StreamFork fork(s, (int)d.pairs.size());
    for (size_t q = 0; q < d.pairs.size() && rc == 0; ++q) {
      const cudaStream_t ps = fork.stream((int)q);
      const auto [i, j] = d.pairs[q];
      float* contacts = reinterpret_cast<float*>(base + d.off_contacts[q]);
      double* frames = reinterpret_cast<double*>(base + d.off_frames[q]);
      cmgb_manifold_out out{contacts, nullptr, nullptr, nullptr, frames, sizeof(double) * workspace_doubles(n_env, 1, 1),
                            nullptr, nullptr, 0.0f, 0};
      LaunchPlan plan = plan_manifold(bodies[i].surface, bodies[j].surface, poses + 6 * i, 1, poses + 6 * j, 1,
                                      n_env, cfg, &out);
      if (plan.p.n_contacts == 0) {  // no contacts: zero wrench / deepest for this pair
        cuda_check(cudaMemsetAsync(wrench + q * n_env * 12, 0, sizeof(double) * n_env * 12, ps), "memset");
        cuda_check(cudaMemsetAsync(pdeep + q * n_env, 0, sizeof(double) * n_env, ps), "memset");
        continue;
      }
      plan.p.pose_stride1 = plan.p.pose_stride2 = 6 * (int64_t)nb;
      launch_with_workspace(plan, n_env, 1, 1, frames, out.workspace_bytes, ps);
      PenaltyArgs a{};
      a.contacts = contacts;
      a.frames1 = frames;
      a.frames2 = frames + 12 * n_env;
      a.vel = velocities;
      a.nb = nb;
      a.bi = i;
      a.bj = j;
      a.C = plan.p.n_contacts;
      a.n1 = plan.p.n1;
      a.n2 = plan.p.n2;
      a.n_env = n_env;
      a.prm = P;
      a.wrench = wrench + q * n_env * 12;
      a.deepest = pdeep + q * n_env;
      rc = launch_penalty(a, ps);
    }
    }  // join
    if (rc == 0) {
      IntegrateArgs g{};
      g.poses = poses;
      g.vel = velocities;
      g.wrench = wrench;
      g.pair_deepest = pdeep;
      g.deepest = deepest;
      g.ok = ok;
      g.n_env = n_env;
      g.nb = nb;
      g.n_pairs = (int32_t)d.pairs.size();
      g.dt = dt;
      for (int k = 0; k < 3; ++k) g.gravity[k] = prm->gravity[k];
      for (int b = 0; b < nb; ++b) {
        g.mass[b] = bodies[b].mass;
        g.is_static[b] = bodies[b].is_static ? 1 : 0;
        const double* I = bodies[b].inertia_diag;
        if (I[0] > 0.0 && I[1] > 0.0 && I[2] > 0.0) {
          for (int k = 0; k < 3; ++k) g.inertia[3 * b + k] = I[k];
        } else {  // box_inertia_diag over the mesh AABB (demosim.cpp:17-23)
          const Mesh& M = bodies[b].surface->mesh;
          double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
          for (int v = 0; v < M.nv(); ++v)
            for (int k = 0; k < 3; ++k) {
              lo[k] = std::min(lo[k], M.vertices[3 * v + k]);
              hi[k] = std::max(hi[k], M.vertices[3 * v + k]);
            }
          const double sx = hi[0] - lo[0], sy = hi[1] - lo[1], sz = hi[2] - lo[2], m = bodies[b].mass;
          g.inertia[3 * b] = m / 12.0 * (sy * sy + sz * sz);
          g.inertia[3 * b + 1] = m / 12.0 * (sx * sx + sz * sz);
          g.inertia[3 * b + 2] = m / 12.0 * (sx * sx + sy * sy);
        }
      }
      for (size_t q = 0; q < d.pairs.size(); ++q) {
        g.pair_i[q] = d.pairs[q].first;
        g.pair_j[q] = d.pairs[q].second;
      }
      rc = launch_integrate(g, s);
    }
    if (pooled) cudaFreeAsync(buf, s);
    if (rc != 0)
      throw Error(CMGB_ERR_CUDA, std::string("demo launch: ") + cudaGetErrorString(cudaGetLastError()));
  });
}

size_t cmgb_manifold_workspace_bytes(int64_t n_env, int32_t st1, int32_t st2) {
  return n_env > 0 ? workspace_doubles(n_env, st1, st2) * sizeof(double) : 0;
}

int cmgb_device_count(int32_t* count) {
  return guarded([&] {
    int n = 0;
    cuda_check(cudaGetDeviceCount(&n), "cudaGetDeviceCount");
    if (count) *count = n;
  });
}

}  // extern "C"
