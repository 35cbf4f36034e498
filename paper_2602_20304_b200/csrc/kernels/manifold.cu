// Fused batched contact-manifold kernel (K1-K5 of SURVEY.md §2):
//   generate_manifold<T> (include/cmg/manifold.hpp:336-377) for every env of
//   a batch, + mean_contact_distance (379-384), in ONE launch.
//
// Mapping: a CTA owns `envs_per_block` consecutive envs (all envs share the
// same two surfaces, so every branch on geometry / config is warp-uniform).
// Phases, separated by __syncthreads():
//   A  pose -> (R, t)                         se3_exp            pose.hpp:78-91
//   B  opposing-SDF vertex scores (top-K)     vertex/edge_penetrations 77-94
//   C  rank sort of scores (top-K)            soft_topk sort     smooth_ops.hpp:180-185
//   D  selected vertex / edge slots           select_topk_*      manifold.hpp:128-181
//   E  V-S contacts | E-E pair stage          vs_contacts 185-204, ee_contacts 237-287
//   F  row / column NN softmin statistics     ee_contacts 289-301
//   G  activity product + fixed-layout store  ee_contacts 303-330
//   H  per-env mean contact distance          mean_contact_distance 379-384
// Per-env state lives in shared memory (SmemLayout); the only HBM traffic is
// the poses in (96 B/env), mesh/SDF reads (L1/L2-resident) and the contacts
// out (C x 32 B/env).
#include <cuda_runtime.h>

#include "../common.h"
#include "../device/dmath.cuh"
#include "../device/sdf.cuh"
#include "../device/witness.cuh"

namespace cmgb {

namespace {

constexpr int kMaxThreads = 512;

struct EnvView {
  unsigned char* base;
  const SmemLayout* L;
  __device__ double* R(int s) const { return reinterpret_cast<double*>(base + L->frames) + 12 * s; }
  __device__ double* t(int s) const { return R(s) + 9; }
  __device__ double* vslot(int i) const { return reinterpret_cast<double*>(base + L->vslots) + 3 * i; }
  __device__ double* eslot(int i) const { return reinterpret_cast<double*>(base + L->eslots) + 12 * i; }
  __device__ int* prov() const { return reinterpret_cast<int*>(base + L->prov); }
  __device__ float* scores() const { return reinterpret_cast<float*>(base + L->scores); }
  __device__ float* sorted() const { return reinterpret_cast<float*>(base + L->sorted); }
  __device__ float* pair(int i) const { return reinterpret_cast<float*>(base + L->pairs) + kPairRec * i; }
  __device__ float* vsdist() const { return reinterpret_cast<float*>(base + L->vsdist); }
  __device__ float* nnstat() const { return reinterpret_cast<float*>(base + L->nnstat); }
};

__device__ __forceinline__ double3 ld_vert(const double* v, int i) {
  return d3(__ldg(v + 3 * i), __ldg(v + 3 * i + 1), __ldg(v + 3 * i + 2));
}

__device__ __forceinline__ double3 to_world(const double* R, const double* t, double3 pb) {
  return mul_R(R, pb) + d3(t[0], t[1], t[2]);
}
__device__ __forceinline__ double3 to_body(const double* R, const double* t, double3 pw) {
  return mul_Rt(R, pw - d3(t[0], t[1], t[2]));
}

// Score-set index helpers: sets 0 = V1, 1 = V2, 2 = E1, 3 = E2.
struct Sets {
  int off[5];
  __device__ Sets(const ManifoldParams& p) {
    off[0] = 0;
    off[1] = p.side[0].nv;
    off[2] = off[1] + p.side[1].nv;
    off[3] = off[2] + p.side[0].ne;
    off[4] = off[3] + p.side[1].ne;
  }
};

__device__ __forceinline__ void store_contact(float* dst, float px, float py, float pz, float d,
                                              float nx, float ny, float nz, float a) {
  float4* o = reinterpret_cast<float4*>(dst);
  o[0] = make_float4(px, py, pz, d);
  o[1] = make_float4(nx, ny, nz, a);
}

// V-S contact for a selected vertex (world) against the opposing posed SDF
// (vs_contacts, manifold.hpp:185-204).
__device__ __forceinline__ void vs_contact(const DevSdf& opp, const double* Ro, const double* to,
                                           double3 pw, const DevCfg& c, float* out_dist,
                                           float* dst) {
  const float3 pb = to_f3(to_body(Ro, to, pw));
  const SdfOut s = sdf_eval<kNormalSource>(opp, pb);
  const float inv = rsqf(c.tau_normal + fdot(s.g, s.g));  // normalize_smooth (vec3.hpp:56-62)
  const float3 n = mul_R_f(Ro, f3(s.g.x * inv, s.g.y * inv, s.g.z * inv));
  const float act = sigmoidf(-s.v * c.inv_tau_pen);  // sigma_greater(-phi, 0, tau_pen)
  *out_dist = s.v;
  store_contact(dst, (float)pw.x, (float)pw.y, (float)pw.z, s.v, n.x, n.y, n.z, act);
}

// sphere_trace_project (sdf.hpp:318-326) in the body frame, FP64 position.
__device__ __forceinline__ double3 trace(const DevSdf& sdf, double3 p, const DevCfg& c) {
#pragma unroll 1
  for (int k = 0; k < c.trace_iters; ++k) {
    const SdfOut s = sdf_eval<kGrad>(sdf, to_f3(p));
    const float sc = s.v * rsqf(c.tau_normal + fdot(s.g, s.g));
    p = p - d3((double)(s.g.x * sc), (double)(s.g.y * sc), (double)(s.g.z * sc));
  }
  return p;
}

// E-E pair stage (ee_contacts loop body, manifold.hpp:237-287). Writes the
// pair record consumed by the NN / activity phases.
__device__ __forceinline__ void ee_pair(const ManifoldParams& p, const EnvView& ev, int k, int l,
                                        float* rec) {
  const DevCfg& c = p.cfg;
  const double* s1 = ev.eslot(k);
  const double* s2 = ev.eslot(p.m1 + l);
  const double3 a1w = d3(s1[0], s1[1], s1[2]), b1w = d3(s1[3], s1[4], s1[5]);
  const double3 a2w = d3(s2[0], s2[1], s2[2]), b2w = d3(s2[3], s2[4], s2[5]);
  const QpSol w = ee_qp(a1w, b1w, a2w, b2w, c);
  // Witness points in their own body frames (edge_point, witness.hpp:130-133).
  const double3 a1b = d3(s1[6], s1[7], s1[8]), b1b = d3(s1[9], s1[10], s1[11]);
  const double3 a2b = d3(s2[6], s2[7], s2[8]), b2b = d3(s2[9], s2[10], s2[11]);
  double3 p1b = a1b + (b1b - a1b) * w.a1;
  double3 p2b = a2b + (b2b - a2b) * w.a2;
  if (c.trace_iters > 0) {
    p1b = trace(p.side[0].sdf, p1b, c);
    p2b = trace(p.side[1].sdf, p2b, c);
  }
  const double* R1 = ev.R(0);
  const double* t1 = ev.t(0);
  const double* R2 = ev.R(1);
  const double* t2 = ev.t(1);
  const double3 p1w = to_world(R1, t1, p1b);
  const double3 p2w = to_world(R2, t2, p2b);
  const double3 de = p1w - p2w;
  const double dg = sqrt(ddot(de, de) + 1e-12);  // kEdgeNormalEps
  const double inv_dg = 1.0 / dg;
  const float3 nb = f3((float)(de.x * inv_dg), (float)(de.y * inv_dg), (float)(de.z * inv_dg));
  SdfOut o1, o2;
  if (c.containment) {
    o1 = sdf_eval<kNormalSource>(p.side[0].sdf, to_f3(p1b));
    o2 = sdf_eval<kNormalSource>(p.side[1].sdf, to_f3(p2b));
  } else {
    o1 = sdf_eval<kNormalOnly>(p.side[0].sdf, to_f3(p1b));
    o2 = sdf_eval<kNormalOnly>(p.side[1].sdf, to_f3(p2b));
  }
  const float i1 = rsqf(c.tau_normal + fdot(o1.g, o1.g));
  const float i2 = rsqf(c.tau_normal + fdot(o2.g, o2.g));
  const float3 n1 = mul_R_f(R1, f3(o1.g.x * i1, o1.g.y * i1, o1.g.z * i1));
  const float3 n2 = mul_R_f(R2, f3(o2.g.x * i2, o2.g.y * i2, o2.g.z * i2));
  float g1, g2;
  const float d2 = fdot(n2, nb), d1 = fdot(n1, nb);
  if (c.hard_ops) {  // sign_hard (smooth_ops.hpp:208)
    g1 = d2 < 0.f ? -1.f : (d2 > 0.f ? 1.f : 0.f);
    g2 = d1 < 0.f ? -1.f : (d1 > 0.f ? 1.f : 0.f);
  } else {
    g1 = tanh_acc(d2 * c.inv_tau_sign);
    g2 = tanh_acc(d1 * c.inv_tau_sign);
  }
  // Penetration of each witness point into the opposing surface.
  const float v12 = sdf_eval<kValue>(p.side[1].sdf, to_f3(to_body(R2, t2, p1w))).v;
  const float v21 = sdf_eval<kValue>(p.side[0].sdf, to_f3(to_body(R1, t1, p2w))).v;
  rec[0] = (float)p1w.x; rec[1] = (float)p1w.y; rec[2] = (float)p1w.z;
  rec[3] = (float)p2w.x; rec[4] = (float)p2w.y; rec[5] = (float)p2w.z;
  rec[6] = nb.x; rec[7] = nb.y; rec[8] = nb.z;
  rec[9] = g1;
  rec[10] = g2;
  rec[11] = (float)dg;
  rec[12] = w.gamma;
  rec[13] = sigmoidf(-v12 * c.inv_tau_pen);
  rec[14] = sigmoidf(-v21 * c.inv_tau_pen);
  rec[15] = sigmoidf(-fdot(n1, n2) * c.inv_tau_clash);
  rec[16] = c.containment ? sigmoidf(-o1.v * c.inv_tau_cont) * sigmoidf(-o2.v * c.inv_tau_cont)
                          : 1.0f;
}

__global__ void __launch_bounds__(kMaxThreads, 1)
    manifold_kernel(const __grid_constant__ ManifoldParams p) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int epb = p.envs_per_block;
  const int64_t env0 = (int64_t)blockIdx.x * epb;
  const int n_here = (int)(p.n_env - env0 < epb ? p.n_env - env0 : epb);
  const int tid = threadIdx.x, nth = blockDim.x;
  const DevCfg& c = p.cfg;
  const DevSide& S1 = p.side[0];
  const DevSide& S2 = p.side[1];
  const int n1 = p.n1, n2 = p.n2, m1 = p.m1, m2 = p.m2, P = m1 * m2;
  const bool full = m1 > 0 && m2 > 0;
  auto env = [&](int e) { return EnvView{smem + (size_t)e * p.smem.bytes, &p.smem}; };

  // ---- A: poses -> frames ------------------------------------------------
  for (int i = tid; i < 2 * n_here; i += nth) {
    const int e = i >> 1, s = i & 1;
    const double* pose = s == 0 ? p.poses1 + 6 * (env0 + e) * p.stride1
                                : p.poses2 + 6 * (env0 + e) * p.stride2;
    double xi[6];
#pragma unroll
    for (int k = 0; k < 6; ++k) xi[k] = __ldg(pose + k);
    const EnvView ev = env(e);
    se3_exp_d(xi, ev.R(s), ev.t(s));
  }
  __syncthreads();

  const bool topk_any = S1.topk_v | S2.topk_v | S1.topk_e | S2.topk_e;
  const Sets sets(p);
  if (topk_any) {
    // ---- B: vertex penetration scores (opposing posed SDF value) ----------
    const int nv_all = S1.nv + S2.nv;
    for (int it = tid; it < n_here * nv_all; it += nth) {
      const int e = it / nv_all, i = it % nv_all;
      const int s = i < S1.nv ? 0 : 1;
      const int vi = s == 0 ? i : i - S1.nv;
      const EnvView ev = env(e);
      const double3 pw = to_world(ev.R(s), ev.t(s), ld_vert(s == 0 ? S1.verts : S2.verts, vi));
      const double3 pb = to_body(ev.R(1 - s), ev.t(1 - s), pw);
      const float pen = s == 0 ? sdf_eval<kValue>(S2.sdf, to_f3(pb)).v
                               : sdf_eval<kValue>(S1.sdf, to_f3(pb)).v;
      ev.scores()[i] = -pen;  // scores = negated penetrations (manifold.hpp:142-143)
    }
    __syncthreads();
    // edge scores: -(mean of endpoint penetrations) (edge_penetrations, 86-94)
    const int ne_all = S1.ne + S2.ne;
    for (int it = tid; it < n_here * ne_all; it += nth) {
      const int e = it / ne_all, i = it % ne_all;
      const int s = i < S1.ne ? 0 : 1;
      const int ei = s == 0 ? i : i - S1.ne;
      const int32_t* E = s == 0 ? S1.edges : S2.edges;
      const int va = __ldg(E + 2 * ei), vb = __ldg(E + 2 * ei + 1);
      float* sc = env(e).scores();
      const int voff = s == 0 ? 0 : S1.nv;
      const float pa = -sc[voff + va], pb = -sc[voff + vb];
      sc[sets.off[2] + i] = -((pa + pb) * 0.5f);
    }
    __syncthreads();
    // ---- C: descending rank sort (values only matter; smooth_ops.hpp:180-185)
    const int total = sets.off[4];
    for (int it = tid; it < n_here * total; it += nth) {
      const int e = it / total, i = it % total;
      const int set = i < sets.off[1] ? 0 : i < sets.off[2] ? 1 : i < sets.off[3] ? 2 : 3;
      const bool active = set == 0 ? S1.topk_v : set == 1 ? S2.topk_v : set == 2 ? S1.topk_e : S2.topk_e;
      if (!active) continue;
      const float* sc = env(e).scores();
      const float x = sc[i];
      int rank = 0;
      for (int j = sets.off[set]; j < sets.off[set + 1]; ++j) {
        const float y = sc[j];
        rank += (y > x) || (y == x && j < i);
      }
      env(e).sorted()[sets.off[set] + rank] = x;
    }
    __syncthreads();
  }

  // ---- D: selected slots (pass-through or soft top-K rows) --------------
  {
    const int nsl = n1 + n2 + m1 + m2;
    for (int it = tid; it < n_here * nsl; it += nth) {
      const int e = it / nsl, r0 = it % nsl;
      const EnvView ev = env(e);
      const bool is_edge = r0 >= n1 + n2;
      const int s = is_edge ? (r0 - n1 - n2 < m1 ? 0 : 1) : (r0 < n1 ? 0 : 1);
      const int r = is_edge ? (s == 0 ? r0 - n1 - n2 : r0 - n1 - n2 - m1) : (s == 0 ? r0 : r0 - n1);
      const DevSide& S = s == 0 ? S1 : S2;
      const double* R = ev.R(s);
      const double* t = ev.t(s);
      const bool sel = is_edge ? S.topk_e : S.topk_v;
      double3 a = d3(0, 0, 0), b = d3(0, 0, 0);
      int prov = r;
      if (!sel) {  // K == D pass-through (manifold.hpp:135-140, 158-167)
        if (is_edge) {
          a = ld_vert(S.verts, __ldg(S.edges + 2 * r));
          b = ld_vert(S.verts, __ldg(S.edges + 2 * r + 1));
        } else {
          a = ld_vert(S.verts, r);
        }
      } else {  // soft top-K row r (smooth_ops.hpp:191-196, manifold.hpp:141-148, 168-180)
        const int set = (is_edge ? 2 : 0) + s;
        const float* x = ev.scores() + sets.off[set];
        const int D = sets.off[set + 1] - sets.off[set];
        const float sr = ev.sorted()[sets.off[set] + r];
        const float inv_tau = is_edge ? c.inv_tau_topk_e : c.inv_tau_topk_v;
        float tot = 0.f;
        prov = -1;
        for (int i = 0; i < D; ++i) {
          const float dist = fabsf(sr - x[i]);
          tot += __expf(-dist * inv_tau);
          if (prov < 0 && dist == 0.0f) prov = i;  // first argmax (hard_attribution, 110-121)
        }
        const float inv = rcpf(tot);
        for (int i = 0; i < D; ++i) {
          const double wi = (double)(__expf(-fabsf(sr - x[i]) * inv_tau) * inv);
          if (is_edge) {
            a = a + ld_vert(S.verts, __ldg(S.edges + 2 * i)) * wi;
            b = b + ld_vert(S.verts, __ldg(S.edges + 2 * i + 1)) * wi;
          } else {
            a = a + ld_vert(S.verts, i) * wi;
          }
        }
      }
      ev.prov()[r0] = prov;
      if (is_edge) {
        double* q = ev.eslot(r0 - n1 - n2);
        const double3 aw = to_world(R, t, a), bw = to_world(R, t, b);
        q[0] = aw.x; q[1] = aw.y; q[2] = aw.z;
        q[3] = bw.x; q[4] = bw.y; q[5] = bw.z;
        q[6] = a.x; q[7] = a.y; q[8] = a.z;
        q[9] = b.x; q[10] = b.y; q[11] = b.z;
      } else {
        double* q = ev.vslot(r0);
        const double3 aw = to_world(R, t, a);
        q[0] = aw.x; q[1] = aw.y; q[2] = aw.z;
      }
    }
  }
  __syncthreads();

  // ---- E: V-S contacts, then E-E pair stage ------------------------------
  const int C = p.n_contacts;
  {
    const int nvs = n1 + n2;
    for (int it = tid; it < n_here * nvs; it += nth) {
      const int e = it / nvs, r = it % nvs;
      const EnvView ev = env(e);
      const double* q = ev.vslot(r);
      float* dst = p.contacts + ((env0 + e) * C + r) * 8;
      if (r < n1) vs_contact(S2.sdf, ev.R(1), ev.t(1), d3(q[0], q[1], q[2]), c, ev.vsdist() + r, dst);
      else vs_contact(S1.sdf, ev.R(0), ev.t(0), d3(q[0], q[1], q[2]), c, ev.vsdist() + r, dst);
      if (p.src) {
        int* sp = p.src + ((env0 + e) * C + r) * 2;
        sp[0] = ev.prov()[r];
        sp[1] = -1;
      }
    }
    if (full) {
      for (int it = tid; it < n_here * P; it += nth) {
        const int e = it / P, i = it % P;
        ee_pair(p, env(e), i / m2, i % m2, env(e).pair(i));
      }
    }
  }
  __syncthreads();

  if (full) {
    // ---- F: NN softmin statistics: rows (side 1) and columns (side 2) -------
    const int nrc = m1 + m2;
    for (int it = tid; it < n_here * nrc; it += nth) {
      const int e = it / nrc, r = it % nrc;
      const EnvView ev = env(e);
      const bool row = r < m1;
      const int n = row ? m2 : m1;
      float m = INFINITY;
      for (int j = 0; j < n; ++j) {
        const int i = row ? r * m2 + j : j * m2 + (r - m1);
        m = fminf(m, ev.pair(i)[11]);
      }
      float tot = 0.f;
      for (int j = 0; j < n; ++j) {
        const int i = row ? r * m2 + j : j * m2 + (r - m1);
        tot += __expf((m - ev.pair(i)[11]) * c.inv_tau_nn);
      }
      ev.nnstat()[2 * r] = m;
      ev.nnstat()[2 * r + 1] = rcpf(tot);
    }
    __syncthreads();
    // ---- G: activity product + fixed-layout E-E output (303-330) -----------
    for (int it = tid; it < n_here * P; it += nth) {
      const int e = it / P, i = it % P;
      const int k = i / m2, l = i % m2;
      const EnvView ev = env(e);
      const float* rec = ev.pair(i);
      const float* ns = ev.nnstat();
      const float dgf = rec[11];
      const float nn1 = __expf((ns[2 * k] - dgf) * c.inv_tau_nn) * ns[2 * k + 1];
      const float nn2 = __expf((ns[2 * (m1 + l)] - dgf) * c.inv_tau_nn) * ns[2 * (m1 + l) + 1];
      const float con = rec[12], pen1 = rec[13], pen2 = rec[14], clash = rec[15], cont = rec[16];
      const float act1 = con * pen1 * nn1 * clash * cont;
      const float act2 = con * pen2 * nn2 * clash * cont;
      const float g1 = rec[9], g2 = rec[10];
      const int64_t row = (env0 + e) * C + n1 + n2 + 2 * i;
      float* dst = p.contacts + row * 8;
      store_contact(dst, rec[0], rec[1], rec[2], g1 * dgf, rec[6] * g1, rec[7] * g1, rec[8] * g1, act1);
      store_contact(dst + 8, rec[3], rec[4], rec[5], g2 * dgf, rec[6] * g2, rec[7] * g2, rec[8] * g2, act2);
      if (p.src) {
        int* sp = p.src + row * 2;
        const int sa = ev.prov()[n1 + n2 + k], sb = ev.prov()[n1 + n2 + m1 + l];
        sp[0] = sa; sp[1] = sb; sp[2] = sa; sp[3] = sb;
      }
      if (p.ee) {
        float* E = p.ee + (env0 + e) * 9 * P;
        E[i] = dgf;
        E[P + i] = con;
        E[2 * P + i] = pen1;
        E[3 * P + i] = pen2;
        E[4 * P + i] = nn1;
        E[5 * P + i] = nn2;
        E[6 * P + i] = clash;
        E[7 * P + i] = act1;
        E[8 * P + i] = act2;
      }
      // keep the signed distances for the mean reduction
      float* w = const_cast<float*>(rec);
      w[17] = g1 * dgf;
      w[18] = g2 * dgf;
    }
    __syncthreads();
  }

  // ---- H: mean contact distance, one warp per env, fixed reduction order --
  if (p.mean_dist) {
    const int warp = tid >> 5, lane = tid & 31, nwarps = nth >> 5;
    for (int e = warp; e < n_here; e += nwarps) {
      const EnvView ev = env(e);
      double acc = 0.0;
      for (int r = lane; r < n1 + n2; r += 32) acc += (double)ev.vsdist()[r];
      if (full)
        for (int i = lane; i < P; i += 32) acc += (double)ev.pair(i)[17] + (double)ev.pair(i)[18];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (lane == 0) p.mean_dist[env0 + e] = (float)(acc / (double)C);
    }
  }
}

}  // namespace

int launch_manifold(const ManifoldParams& p, int block_threads, int grid, size_t smem_bytes,
                    void* stream) {
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(manifold_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    configured = true;
  }
  manifold_kernel<<<grid, block_threads, smem_bytes, static_cast<cudaStream_t>(stream)>>>(p);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

int manifold_max_threads() { return kMaxThreads; }

}  // namespace cmgb
