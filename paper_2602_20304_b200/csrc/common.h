// Structures shared by the host C++ layer and the sm_100a kernels.
//
// Device layout: geometry is FP64 in HBM (a few hundred bytes
// per surface, read through L1/L2), SDF programs are packed into the kernel's
// __grid_constant__ parameter block (constant bank: warp-uniform broadcast
// loads), large primitive tables (CP planes, OPC points) live in a double4 pool
// in HBM. Poses are FP64 [n_env][6]; contacts are FP32 [n_env][C][8].
#pragma once

#include <cstdint>

#include <vector_types.h>  // double4 (CUDA toolkit header, host-safe)

namespace cmgb {

constexpr int kMaxNodes = 16;      // SDF program nodes per surface held in the param block
constexpr int kMaxNodesExt = 4096; // larger programs: the node array in device memory (DevSdf::ext)
constexpr int kMaxStack = 8;       // generic interpreter stack depth (wide unions are chained to fit)
constexpr int kPairRec = 38;    // floats per E-E pair record in shared memory (19 doubles:
                                 // an odd stride keeps per-lane FP64 accesses bank-conflict free)

// kSqE01: a lone superquadric with eps1 = eps2 = 0.1 (the box-box benchmark
// body), whose exponents (n1, n2, n3, n4) = (10, 1, 10, 20) are compiled in.
// kBoxCp: a lone convex polyhedron whose 6 planes are the axis-aligned box
// pattern of box_planes (scene.cpp:49-62: +x, -x, +y, -y, +z, -z unit
// normals): plane distances are +-p_i - w_i (bit-identical to the FMA dot).
enum SdfKind : int32_t {
  kSingleSq = 0, kSingleCp = 1, kGeneric = 2, kSqE01 = 3, kBoxCp = 4,
  // more lone superquadrics with compile-time exponents (n1, n2, n3, n4):
  kSqE02 = 5,   // eps1 = eps2 = 0.2  (5, 1, 5, 10): rounded box (config C), box-box eps 0.2
  kSqE025 = 6,  // eps1 = eps2 = 0.25 (4, 1, 4, 8)
  kSqE05 = 7,   // eps1 = eps2 = 0.5  (2, 1, 2, 4)
  kSqEll = 8,   // eps1 = eps2 = 1    (1, 1, 1, 2): ellipsoid / sphere
  kSqCyl = 9,   // eps1 = 0.1, eps2 = 1 (1, 10, 10, 20): cylinder (config C)
  // a recognised composition: union(kSqCyl cylinder, kSqEll cap, kSqEll cap) --
  // the capsule of config C, leaves in registers
  kCapsule = 10
};

// Exponents of the compile-time superquadric kinds (0: not such a kind).
struct SqExpTuple {
  int n1, n2, n3, n4;
};
__host__ __device__ constexpr SqExpTuple sq_exps(int k) {
  return k == kSqE01    ? SqExpTuple{10, 1, 10, 20}
         : k == kSqE02  ? SqExpTuple{5, 1, 5, 10}
         : k == kSqE025 ? SqExpTuple{4, 1, 4, 8}
         : k == kSqE05  ? SqExpTuple{2, 1, 2, 4}
         : k == kSqEll  ? SqExpTuple{1, 1, 1, 2}
         : k == kSqCyl  ? SqExpTuple{1, 10, 10, 20}
                        : SqExpTuple{0, 0, 0, 0};
}
__host__ __device__ constexpr bool ct_sq(int k) { return sq_exps(k).n1 > 0; }
enum Flavor : int32_t { kValue = 0, kGrad = 1, kNormalSource = 2, kNormalOnly = 3 };

// Superquadric leaf, pre-digested on the host (sdf.hpp:85-108):
//   f = (x2^p1 + y2^p1)^p2 + z2^p3, phi = (1 - f^p4) / |x~|.
// n1..n3 > 0 when the exponent is an exact small integer in double precision
// (then powers are repeated products: no SFU work).
struct DevSq {
  double inv_ax[3];
  double ax[3];          // axes (the normalised-coordinate sphere trace maps back with them)
  double p1, p2, p3;     // 1/e2, e2/e1, 1/e1 (general-exponent path)
  double c_xy, c_z;      // 2 p1 p2, 2 p3 (grad f prefactors)
  double R[9], t[3];     // body_from_prim (sdf.cpp:9)
  double p4;             // -e1/2
  int32_t n1, n2, n3;    // integer exponents (1..64) or 0
  int32_t has_frame;     // 0 identity pose, 1 rotated, 2 translation only (R = I exactly)
  int32_t n4;            // -1/p4 = 2/e1 when an exact integer (1..64): f^p4 = 1 / f^(1/n4)
};

struct DevNode {
  int32_t op;      // cmgb_sdf_op
  int32_t count;   // planes | points | children
  int32_t offset;  // into the double4 pool (CP: 1 per plane, OPC: 2 per point)
  int32_t pad;
  double tau_d;
  double inv_tau_d;
  DevSq sq;
  double box_w[6];  // kBoxCp: plane offsets n . point in the +x, -x, +y, -y, +z, -z order
};

struct DevSdf {
  int32_t n_nodes;
  int32_t kind;        // SdfKind
  int32_t leaf_count;
  int32_t max_stack;
  DevNode nodes[kMaxNodes];
  const double4* pool;  // CP: (n, n.p) per plane; OPC: (p, -1/2th^2), (n, 1/th^2)
  const DevNode* ext;   // all n_nodes nodes in device memory when n_nodes > kMaxNodes (generic kind), else null
};

// One side of a surface pair as the kernel sees it.
struct DevSide {
  const double* verts;  // [nv][3] body frame
  const int32_t* edges; // [ne][2]
  const double* edge_body;  // [ne][6] endpoints a, b of every edge (body frame)
  int32_t nv, ne;
  int32_t n_sel;        // V-S contacts of this side (effective vertex top-K, or 0)
  int32_t m_sel;        // selected edges of this side (effective edge top-K, or 0)
  int32_t topk_v;       // 1: soft top-K over vertices active (n_sel < nv)
  int32_t topk_e;       // 1: soft top-K over edges active (m_sel < ne)
  DevSdf sdf;
};

// SmoothingConfig on the device (config.hpp:17-46), FP64 (temperatures as
// reciprocals: x / tau -> x * inv_tau, within 1 ulp of the reference).
struct DevCfg {
  double lambda;
  double tau_clip, inv_tau_clip, inv_tau_min, inv_tau_comp;
  double inv_tau_sign, inv_tau_pen, inv_tau_nn, inv_tau_clash, inv_tau_cont;
  double inv_tau_topk_v, inv_tau_topk_e;
  double tau_normal;
  double clip_C, comp_C;  // exp(-1/tau_clip), exp(-1/tau_comp): one exp per softplus / sigmoid pair
  double inv_clip_C, inv_comp_C;
  int32_t pair_exp;       // 1 when both C are normal doubles (1/tau < 700)
  int32_t hard_ops, trace_iters, containment, mode;
  int32_t pad;
};

// Per-env shared-memory carve-up (bytes from the env's base), host-computed.
struct SmemLayout {
  int32_t frames;    // 2 x (R[9], t[3]) doubles
  int32_t vslots;    // (n1+n2) x 3 doubles: selected vertex payload, WORLD frame
  int32_t eslots;    // (m1+m2) x 12 doubles: a_world, b_world, a_body, b_body
  int32_t prov;      // (n1+n2+m1+m2) int32 provenance
  int32_t scores;    // (V1+V2+E1+E2) floats: top-K scores (-penetration), top-K only
  int32_t sorted;    // (V1+V2+E1+E2) int32: set-local index of the score of each rank < K (top-K rows)
  int32_t tkw;       // (V1+V2+E1+E2) doubles: soft top-K weight factors P_i (manifold.cuh C2), top-K only
  int32_t pairs;     // P x kPairRec floats: per E-E pair record
  int32_t vsdist;    // (n1+n2) floats
  int32_t nnstat;    // (m1+m2) x 2 floats: min, 1/sum
  int32_t hpart;     // (warps per CTA) doubles: per-warp partial sums of the E-E distances (G)
  int32_t amask;     // mask_words uint32: activity > threshold bit per contact (compaction extra)
  int32_t bytes;     // per env, 16-byte aligned
};

// n / d for 0 <= n < 2^32 / d: q = (n * mul) >> 32, mul = ceil(2^32 / d)
// (64-bit: d = 1 needs mul = 2^32).
struct FastDiv {
  uint64_t mul;
  uint32_t d, pad;
};

struct ManifoldParams {
  DevSide side[2];
  DevCfg cfg;
  const double* poses1;
  const double* poses2;
  const double* frames1;  // [n1][12] R (row-major), t: device workspace filled by frames_kernel
  const double* frames2;
  int32_t stride1, stride2;            // frames: env e's frame at 12 e stride (1 = one per env, 0 = shared,
                                       //   n_bodies = a scene's [env][body] frame array)
  int64_t pose_stride1, pose_stride2;  // poses: doubles between consecutive envs (0 = shared)
  int64_t n_env;
  int32_t n1, n2, m1, m2, n_contacts;
  int32_t envs_per_block;
  FastDiv div_pairs, div_m2, div_nvs, div_nslots, div_nrc, div_nv_all, div_ne_all, div_scores;
  SmemLayout smem;
  float* contacts;
  int32_t* src;
  float* ee;
  float* mean_dist;
  int32_t vs_ext;       // 1: V-S contacts (and their share of mean_dist) come from vs_kernel, launched first
  double* pairs_gmem;   // pair records in global memory ([n_env][pair_stride] doubles), or null = shared
  int64_t pair_stride;  // doubles per env in pairs_gmem
  uint32_t* act_mask;   // optional [n_env][mask_words]: bit c = (activity of contact c > act_thr)
  int32_t* act_count;   // optional [n_env]: set bits
  float act_thr;
  int32_t mask_words;   // ceil(n_contacts / 32)
  int32_t frames_ready; // 1: frames1 / frames2 already hold every env's frames (a scene's shared pass)
};

// Pose-Jacobian (forward-mode, Dual12) batch: the geometry / config / slot
// counts of a ManifoldParams plan; one unit = one env with all 12 pose tangent
// directions (dual.hpp:249-263), `units_per_block` envs per CTA. Shared-memory
// offsets are in bytes from the env's base (host-computed; tangent records
// are an FP64 primal + 12 FP32 tangents, 56 bytes).
struct JvpParams {
  ManifoldParams m;
  float* tangents;   // [n_env][C][8][12]
  float* mean_grad;  // [n_env][12]
  double* mean_f64;       // [n_env] or null
  double* mean_grad_f64;  // [n_env][12] or null
  int32_t nd, groups;
  int32_t units_per_block;
  int32_t o_frames, o_scores, o_sorted, o_vslots, o_eslots, o_prov, o_pairs, o_vsdist, o_nnstat;
  int32_t o_sj, o_qp;  // per-pair side Jacobian / witness QP records (E1 -> E2)
  int32_t o_ebuf, o_aux, ebuf_stride;
  int32_t o_vsrec, o_prec;  // V-S / E-E pair primal records (E1 -> E2)
  int32_t geom_bytes;       // per CTA after the envs: both meshes' vertices + edge endpoints (FP64)  // soft top-K row weights (FP32, stride per slot) / row totals
  int32_t bytes;  // per unit
};

// Demo integrator (kernels/demo.cu). PenaltyParams (demosim.hpp:24-31).
constexpr int kDemoMaxBodies = 16;
constexpr int kDemoMaxPairs = kDemoMaxBodies * (kDemoMaxBodies - 1) / 2;

struct DemoParamsDev {
  double stiffness, damping, friction, friction_viscous, tau_force;
  double gravity[3];
};

struct PenaltyArgs {
  const float* contacts;  // [n_env][C][8] of pair (bi, bj)
  const double* frames1;  // [n_env][12] R, t of body bi (the pair's frames workspace)
  const double* frames2;
  const double* vel;      // [n_env][nb][6]
  int32_t nb, bi, bj;
  int32_t C, n1, n2;      // layout: V-S rows of side 1 / side 2, then E-E rows alternating sides
  int64_t n_env;
  DemoParamsDev prm;
  double* wrench;         // [n_env][12]: force1, torque1, force2, torque2
  double* deepest;        // [n_env]
};

struct IntegrateArgs {
  double* poses;                // [n_env][nb][6]
  double* vel;                  // [n_env][nb][6]
  const double* wrench;         // [n_pairs][n_env][12]
  const double* pair_deepest;   // [n_pairs][n_env]
  double* deepest;              // [n_env] or null
  int32_t* ok;                  // [n_env] or null
  int64_t n_env;
  int32_t nb, n_pairs;
  double dt;
  double gravity[3];
  double mass[kDemoMaxBodies];
  double inertia[3 * kDemoMaxBodies];
  int32_t is_static[kDemoMaxBodies];
  int32_t pair_i[kDemoMaxPairs], pair_j[kDemoMaxPairs];
};

// Batched SDF queries / sphere traces on one surface (kernels/sdf_query.cu).
struct SdfQueryParams {
  DevSdf sdf;
  const double* points;  // [n][3]
  int64_t n;
  double* out;           // [n][4] value, gradient | [n][3] traced points
  double R[9], t[3];     // trace: posed surface
  int32_t iters;
  double tau;
};

struct WitnessParams {
  const void* pairs;
  int32_t fp64;
  int64_t n;
  DevCfg cfg;
  void* out_any;          // float [n][W], or double for the FP64-output solver
  float* alpha_gamma;
  int32_t* labels;
  void* alpha_gamma_f64;  // double [n][3] (FP64-output solver)
};

}  // namespace cmgb

// Launchers implemented in the .cu files (host-callable, stream-ordered).
namespace cmgb {
int launch_manifold(const ManifoldParams& p, int block_threads, int grid, size_t smem_bytes,
                    void* stream);
// se3_exp of n_poses contiguous [6] poses into [12] frames (a scene's bodies x envs, once per call)
int launch_scene_frames(const double* poses, int64_t n_poses, double* frames, void* stream);
int manifold_min_blocks(int k1, int k2);  // resident CTAs / SM the kernel for this kind pair is built for
int launch_manifold_jvp(const JvpParams& p, int block_threads, void* stream);
int jvp_directions();    // tangent directions per thread of the compiled JVP kernel
int jvp_max_threads();   // CTA size of the JVP kernel
int jvp_smem_cap();      // shared-memory bytes per JVP CTA the host may plan for
int launch_ee_witness(const WitnessParams& p, void* stream);
int launch_ee_witness_f64(const WitnessParams& p, void* stream);
int launch_penalty(const PenaltyArgs& a, void* stream);
int launch_sdf_query(const SdfQueryParams& q, int mode, void* stream);
int launch_integrate(const IntegrateArgs& a, void* stream);
int launch_vf_witness(const WitnessParams& p, void* stream);
int launch_widen(const float* src, double* dst, int64_t n, void* stream);
const char* last_cuda_error_string();
}  // namespace cmgb
