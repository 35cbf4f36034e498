/*
 * cmgb.h — C ABI of the B200-native batched contact-manifold path.
 *
 * Drop-in boundary for the reference C++ collision API of arXiv 2602.20304
 * (/root/reference/proj, namespace cmg). The reference exposes header-only
 * templates and has no FFI of its own; every entry point below names the
 * reference interface it replaces (file:line, relative to
 * /root/reference/proj). Plain pointers and sizes only; no C++ or torch types
 * cross this boundary, and no exception escapes it: every call returns a
 * cmgb_status and cmgb_last_error() holds the message (thread-local).
 *
 * Memory conventions
 *   - Descriptor inputs (meshes, SDF programs, configs) are HOST memory and are
 *     copied at create time; handles are immutable afterwards and may be shared
 *     between host threads (reference: SurfaceModel value semantics,
 *     include/cmg/surface.hpp:16-33; sdf.cpp:52-67 deep copy).
 *   - Batch entry points named *_batch take DEVICE pointers and a cudaStream_t
 *     passed as void*; they are stream-ordered and allocate nothing on the hot
 *     call when the caller supplies the workspace (cmgb_manifold_out). The
 *     *_batch_host variants take HOST pointers and perform the H2D/D2H copies
 *     inside the call (the end-to-end path).
 *   - Scalars follow the reference: poses and witness inputs are FP64 exactly
 *     as the reference receives them; contact outputs are FP32.
 */
#ifndef CMGB_H_
#define CMGB_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CMGB_ABI_VERSION 2  /* 2: cmgb_manifold_out gained the activity-mask fields */

typedef enum cmgb_status {
  CMGB_OK = 0,
  CMGB_ERR_INVALID_ARGUMENT = 1, /* reference: std::invalid_argument */
  CMGB_ERR_PARSE = 2,            /* reference: MeshParseError (mesh.hpp:19-23) */
  CMGB_ERR_CUDA = 3,             /* launch / runtime failure on the device */
  CMGB_ERR_NO_DEVICE = 4,        /* no CUDA device: there is no CPU fallback */
  CMGB_ERR_UNSUPPORTED = 5       /* valid in the reference, not supported here (message says why) */
} cmgb_status;

/* Thread-local message of the last failing call on this thread. */
const char* cmgb_last_error(void);
int32_t cmgb_abi_version(void);

/* ---------------------------------------------------------------------------
 * Smoothing configuration — mirrors cmg::SmoothingConfig
 * (include/cmg/config.hpp:17-46) field for field.
 * ------------------------------------------------------------------------- */
typedef enum cmgb_mode {
  CMGB_MODE_FULL = 0,      /* ContactMode::kFull     (config.hpp:9)  */
  CMGB_MODE_NO_EE = 1,     /* ContactMode::kNoEe     (config.hpp:10) */
  CMGB_MODE_ONE_SIDED = 2  /* ContactMode::kOneSided (config.hpp:11) */
} cmgb_mode;

typedef struct cmgb_config {
  double lambda, tau_clip, tau_min, tau_comp;          /* witness solver     */
  double tau_sign, tau_pen, tau_nn, tau_clash, tau_cont; /* contact indicators */
  double tau_topk_verts, tau_topk_edges, tau_normal, tau_union;
  int32_t hard_ops;               /* bool */
  int32_t sphere_trace;           /* bool */
  int32_t sphere_trace_iters;
  int32_t containment_safeguard;  /* bool */
  int32_t mode;                   /* cmgb_mode */
  int32_t reserved;
} cmgb_config;

/* SmoothingConfig{} defaults (config.hpp:17-46). */
void cmgb_config_default(cmgb_config* out);
/* SmoothingConfig::no_smoothing() (config.hpp:48-53). */
void cmgb_config_no_smoothing(cmgb_config* out);
/* SmoothingConfig::validate() (config.hpp:55-73). */
int cmgb_config_validate(const cmgb_config* cfg);
/* config_for_variant(): ours | ours_ns | ours_ne | ours_ne_s (src/batch.cpp:131-150). */
int cmgb_config_for_variant(const char* variant, const cmgb_config* base, cmgb_config* out);

/* ---------------------------------------------------------------------------
 * SDF program — public, flattened form of the private cmg::SmoothSdf tree
 * (include/cmg/sdf.hpp:138-202). Nodes are listed in POSTFIX order: a UNION
 * node with `count` children pops the `count` most recent subtrees (in
 * order), a SUBTRACTION pops (positive, negative). The last node is the root.
 * Device limits: up to 4,096 nodes (above 16 the node array lives in device
 * memory); unions of any width (wide ones are evaluated as chains of binary
 * unions with the same temperature: the same smooth minimum); nesting up to 8
 * levels deep -- deeper programs fail with CMGB_ERR_UNSUPPORTED on first use.
 * ------------------------------------------------------------------------- */
typedef enum cmgb_sdf_op {
  CMGB_SDF_SUPERQUADRIC = 0,        /* SuperquadricParams        sdf.hpp:35-47  */
  CMGB_SDF_CONVEX_POLYHEDRON = 1,   /* ConvexPolyhedronParams    sdf.hpp:49-62  */
  CMGB_SDF_ORIENTED_POINTCLOUD = 2, /* OrientedPointcloudParams  sdf.hpp:64-79  */
  CMGB_SDF_UNION = 3,               /* SdfUnion                  sdf.hpp:143-146 */
  CMGB_SDF_SUBTRACTION = 4          /* SdfSubtraction            sdf.hpp:148-152 */
} cmgb_sdf_op;

typedef struct cmgb_sdf_node {
  int32_t op;                 /* cmgb_sdf_op */
  int32_t count;              /* CP planes | OPC points | UNION children | SUB: 2 */
  double tau;                 /* CP logsumexp tau (default 1e-3) | UNION/SUB tau */
  double eps1, eps2;          /* SQ boxiness, (0, 2] */
  double axes[3];             /* SQ axis lengths > 0 */
  double pose[6];             /* SQ primitive pose in the body frame [t; axis-angle] */
  const double* normals;      /* CP / OPC: count x 3, unit */
  const double* points;       /* CP / OPC: count x 3 */
  const double* lengthscales; /* OPC: count, > 0 */
} cmgb_sdf_node;

/* ---------------------------------------------------------------------------
 * Collision mesh — cmg::CollisionMesh (include/cmg/mesh.hpp:25-34).
 * Vertex order and (lexicographic, lo<hi) edge order are preserved exactly:
 * they define the candidate indices src_a / src_b of every contact.
 * ------------------------------------------------------------------------- */
typedef struct cmgb_mesh_s* cmgb_mesh;

/* make_box_mesh(half, subdivisions, quad_edges) (src/mesh.cpp:123-173). */
int cmgb_mesh_box(const double half_extents[3], int32_t subdivisions, int32_t quad_edges,
                  cmgb_mesh* out);
/* parse_obj(istream) on an in-memory OBJ text (src/mesh.cpp:60-115). On
 * CMGB_ERR_PARSE, *error_line receives the OBJ line number (MeshParseError). */
int cmgb_mesh_parse_obj(const char* text, size_t length, cmgb_mesh* out, int32_t* error_line);
/* Raw arrays (faces/edges as given; edges must be unique lo<hi pairs). */
int cmgb_mesh_from_arrays(const double* vertices, int32_t n_vertices, const int32_t* faces,
                          int32_t n_faces, const int32_t* edges, int32_t n_edges, cmgb_mesh* out);
int cmgb_mesh_sizes(cmgb_mesh mesh, int32_t* n_vertices, int32_t* n_faces, int32_t* n_edges,
                    int32_t* n_warnings);
int cmgb_mesh_read(cmgb_mesh mesh, double* vertices, int32_t* faces, int32_t* edges);
const char* cmgb_mesh_warning(cmgb_mesh mesh, int32_t index);
void cmgb_mesh_destroy(cmgb_mesh mesh);

/* ---------------------------------------------------------------------------
 * Surface — cmg::SurfaceModel + build_surface (include/cmg/surface.hpp:16-40,
 * src/surface.cpp:9-44): mesh + SDF program + top-K budgets, validated at
 * create time with the reference's messages; the mesh/SDF discrepancy check is
 * a warning. Device copies are made lazily, once per device.
 * ------------------------------------------------------------------------- */
typedef struct cmgb_surface_s* cmgb_surface;

int cmgb_surface_create(cmgb_mesh mesh, const cmgb_sdf_node* sdf_postfix, int32_t n_nodes,
                        int32_t vertex_topk, int32_t edge_topk, double tolerance_fraction,
                        cmgb_surface* out);
void cmgb_surface_destroy(cmgb_surface surface);

typedef struct cmgb_surface_info {
  int32_t n_vertices, n_edges, n_faces, leaf_count;
  int32_t vertex_topk, edge_topk;                     /* as given (0 = default) */
  int32_t effective_vertex_topk, effective_edge_topk; /* surface.hpp:24-32 */
  int32_t n_warnings;
  int32_t n_nodes;
} cmgb_surface_info;
int cmgb_surface_get_info(cmgb_surface surface, cmgb_surface_info* out);
const char* cmgb_surface_warning(cmgb_surface surface, int32_t index);

/* ---------------------------------------------------------------------------
 * Manifold layout — ContactManifold::expected_size and the fixed ordering
 * (include/cmg/manifold.hpp:14-17, 62-72): [V-S side 1: n1][V-S side 2: n2]
 * [E-E (k,l) row-major; side 1 then side 2].
 * ------------------------------------------------------------------------- */
typedef struct cmgb_layout {
  int32_t n1, n2, m1, m2;
  int32_t mode;
  int32_t n_contacts;     /* expected_size() */
  int32_t dynamic_src;    /* 1 if top-K selection is active on any side (src is data-dependent) */
  int32_t reserved;
} cmgb_layout;

int cmgb_layout_query(cmgb_surface s1, cmgb_surface s2, const cmgb_config* cfg, cmgb_layout* out);
/* Static per-contact metadata, each array n_contacts long (host memory):
 * kind (0 = VS, 1 = EE), side (1|2), src_a, src_b. For selected (top-K) slots
 * src_* hold -1 here; the batch call writes the data-dependent provenance. */
int cmgb_layout_metadata(cmgb_surface s1, cmgb_surface s2, const cmgb_config* cfg,
                         int32_t* kind, int32_t* side, int32_t* src_a, int32_t* src_b);

/* ---------------------------------------------------------------------------
 * Batched manifold generation — replaces the per-env loop body of
 * bench_manifold (src/batch.cpp:207-215): generate_manifold<double>
 * (include/cmg/manifold.hpp:336-377) + mean_contact_distance (379-384) for
 * every env, in one launch sequence.
 * ------------------------------------------------------------------------- */
typedef struct cmgb_manifold_out {
  float* contacts;   /* required: [n_env][n_contacts][8] = px,py,pz,dist,nx,ny,nz,activity */
  int32_t* src;      /* optional: [n_env][n_contacts][2] = src_a, src_b (provenance)       */
  float* ee;         /* optional: [n_env][9][m1*m2] dist,con,pen1,pen2,nn1,nn2,clash,act1,act2
                        (EeIndicatorMatrices, manifold.hpp:41-52); full mode only          */
  float* mean_dist;  /* optional: [n_env] mean_contact_distance (manifold.hpp:379-384)      */
  void* workspace;   /* optional device scratch of cmgb_manifold_workspace_bytes(); when null
                        the call takes it from the stream-ordered pool (cudaMallocAsync)     */
  size_t workspace_bytes;
  uint32_t* active_mask;   /* optional: [n_env][ceil(n_contacts / 32)] bit c of an env's row =
                              (activity of contact c > active_threshold), produced by the
                              kernels beside the fixed layout (input of cmgb_compact_masked)   */
  int32_t* active_count;   /* optional (with active_mask): [n_env] set bits per env               */
  float active_threshold;
  int32_t reserved;
} cmgb_manifold_out;

/* Device scratch one cmgb_manifold_batch call needs (per-env pose frames). */
size_t cmgb_manifold_workspace_bytes(int64_t n_env, int32_t pose1_stride, int32_t pose2_stride);

/* poses*: DEVICE [n][6] FP64 (Pose6d = [t; axis-angle], pose.hpp:16-18).
 * pose1_stride / pose2_stride: 1 = one pose per env, 0 = the same pose for
 * every env (bench_manifold keeps body 1 fixed, batch.cpp:196-203). */
int cmgb_manifold_batch(cmgb_surface s1, cmgb_surface s2, const double* poses1,
                        int32_t pose1_stride, const double* poses2, int32_t pose2_stride,
                        int64_t n_env, const cmgb_config* cfg, const cmgb_manifold_out* out,
                        void* cuda_stream);

/* End-to-end variant: HOST poses in, HOST mean distances (and optionally HOST
 * contacts) out; copies happen inside the call on the given stream, which is
 * synchronised before returning (also when the call fails). Device scratch comes
 * from a per-device pool: each call leases its own buffers and pipeline
 * streams, so concurrent host threads do not serialise on each other. When
 * contacts_host is given the batch is pipelined in equal chunks so each chunk's
 * D2H overlaps the next chunk's kernels (host buffers should be pinned). */
int cmgb_manifold_batch_host(cmgb_surface s1, cmgb_surface s2, const double* poses1_host,
                             int32_t pose1_stride, const double* poses2_host,
                             int32_t pose2_stride, int64_t n_env, const cmgb_config* cfg,
                             float* mean_dist_host, float* contacts_host, void* cuda_stream);

/* General host-buffer form: every field of host_out is a HOST pointer (or
 * null): contacts [n_env][n_contacts][8], src [n_env][n_contacts][2], ee
 * [n_env][9][m1*m2] (full mode), mean_dist [n_env]; workspace fields ignored.
 * Replaces generate_manifold<double> returning ContactManifold by value
 * (manifold.hpp:336-377); used by the C++ drop-in header (cmgb_cmg.hpp). */
int cmgb_manifold_batch_host_ex(cmgb_surface s1, cmgb_surface s2, const double* poses1_host,
                                int32_t pose1_stride, const double* poses2_host, int32_t pose2_stride,
                                int64_t n_env, const cmgb_config* cfg, const cmgb_manifold_out* host_out,
                                void* cuda_stream);

/* ---------------------------------------------------------------------------
 * Active-contact compaction — an EXTRA output beside the fixed layout (which it
 * never replaces; manifold.hpp:62-72, 303-330): the contacts of a batch with
 * activity > activity_threshold, in fixed-layout order, packed env after env
 * (one TMA-staged pass over the fixed layout, warp ballots, decoupled
 * look-back scan across env tiles). All buffers are DEVICE memory.
 * ------------------------------------------------------------------------- */
typedef struct cmgb_compact_out {
  float* contacts;      /* required: [capacity][8] kept contacts (px,py,pz,dist,nx,ny,nz,activity) */
  int32_t* slot;        /* optional: [capacity] slot of each kept contact in its env's fixed layout
                           (kind / side / static provenance: cmgb_layout_metadata)               */
  int32_t* src;         /* optional: [capacity][2] provenance (needs the batch's src output)     */
  int64_t* env_offset;  /* optional: [n_env + 1] first kept row of each env; [n_env] = total     */
  int32_t* env_count;   /* optional: [n_env] kept contacts per env                               */
  int64_t* total;       /* optional: [1] kept contacts in the batch (rows beyond capacity are
                           counted but not written)                                               */
  int64_t capacity;     /* rows available in contacts / slot / src (n_env * n_contacts never overflows) */
  void* workspace;      /* optional: cmgb_compact_workspace_bytes() of device scratch, else pooled */
  size_t workspace_bytes;
} cmgb_compact_out;

size_t cmgb_compact_workspace_bytes(int64_t n_env, int32_t n_contacts);

/* Compaction from the activity masks / counts a cmgb_manifold_batch call
 * produced (cmgb_manifold_out.active_mask / active_count): a scan of the
 * counts, then only the kept contacts are read. Same outputs as
 * cmgb_compact_contacts with activity_threshold = the batch's active_threshold. */
size_t cmgb_compact_masked_workspace_bytes(int64_t n_env);
int cmgb_compact_masked(const float* contacts, const int32_t* src, int64_t n_env, int32_t n_contacts,
                        const uint32_t* active_mask, const int32_t* active_count, const cmgb_compact_out* out,
                        void* cuda_stream);

/* contacts: DEVICE [n_env][n_contacts][8] (a cmgb_manifold_batch output, 16-byte
 * aligned); src: optional DEVICE [n_env][n_contacts][2]. Stream-ordered. */
int cmgb_compact_contacts(const float* contacts, const int32_t* src, int64_t n_env, int32_t n_contacts,
                          float activity_threshold, const cmgb_compact_out* out, void* cuda_stream);

/* ---------------------------------------------------------------------------
 * Pose Jacobians — generate_manifold<Dual12> with seed_pose_tangents
 * (include/cmg/dual.hpp:249-263; tests/test_dual.cpp gradchecks) for every
 * env: each output scalar's derivative w.r.t. the 12 pose coordinates
 * (pose1[0..5], pose2[0..5]). Smooth mode only: hard_ops != 0 returns
 * CMGB_ERR_UNSUPPORTED (the reference's hard operators are double-only,
 * smooth_ops.hpp:199).
 * ------------------------------------------------------------------------- */
typedef struct cmgb_manifold_jvp_out {
  float* contacts;        /* required: [n_env][n_contacts][8] primal, as cmgb_manifold_out */
  float* tangents;        /* required: [n_env][n_contacts][8][12] d(field)/d(pose coord)    */
  int32_t* src;           /* optional: [n_env][n_contacts][2] provenance                     */
  float* mean_dist;       /* optional: [n_env]                                               */
  float* mean_dist_grad;  /* optional: [n_env][12] tangents of mean_contact_distance         */
  double* mean_dist_f64;       /* optional: [n_env] FP64 mean (as accumulated on the device)  */
  double* mean_dist_grad_f64;  /* optional: [n_env][12] FP64 mean tangents (gradcheck)       */
} cmgb_manifold_jvp_out;

/* poses*: DEVICE [n][6] FP64, strides as cmgb_manifold_batch. */
int cmgb_manifold_jvp_batch(cmgb_surface s1, cmgb_surface s2, const double* poses1,
                            int32_t pose1_stride, const double* poses2, int32_t pose2_stride,
                            int64_t n_env, const cmgb_config* cfg, const cmgb_manifold_jvp_out* out,
                            void* cuda_stream);

/* Host-buffer form: poses and every output field of host_out are HOST memory
 * (generate_manifold<Dual12> by value, main.cpp:202-205). Synchronous. */
int cmgb_manifold_jvp_batch_host(cmgb_surface s1, cmgb_surface s2, const double* poses1_host,
                                 int32_t pose1_stride, const double* poses2_host, int32_t pose2_stride,
                                 int64_t n_env, const cmgb_config* cfg, const cmgb_manifold_jvp_out* host_out,
                                 void* cuda_stream);

/* ---------------------------------------------------------------------------
 * Batched demo integrator — DemoSim::step (src/demosim.cpp:81-138) for every
 * env of a batch: all-pairs manifolds -> penalty_forces (31-66) -> semi-
 * implicit Euler on SE(3) with se3_log bookkeeping (108-133).
 * ------------------------------------------------------------------------- */
typedef struct cmgb_demo_params { /* PenaltyParams (include/cmg/demosim.hpp:24-31) */
  double stiffness;         /* N/m */
  double damping;           /* N s/m along the normal */
  double friction;          /* Coulomb coefficient */
  double friction_viscous;  /* N s/m tangential, capped by friction |Fn| */
  double tau_force;         /* softplus temperature of max_s(-dist, 0) (m) */
  double gravity[3];
} cmgb_demo_params;

typedef struct cmgb_demo_body { /* SceneBody's dynamics fields (include/cmg/scene.hpp:15-22) */
  cmgb_surface surface;
  double mass;
  double inertia_diag[3]; /* all > 0, else derived from the mesh AABB (demosim.cpp:17-23) */
  int32_t is_static;
  int32_t reserved;
} cmgb_demo_body;

void cmgb_demo_params_default(cmgb_demo_params* p);

/* Device scratch one cmgb_demo_step_batch call needs. */
size_t cmgb_demo_workspace_bytes(const cmgb_demo_body* bodies, int32_t n_bodies, const cmgb_config* cfg,
                                 int64_t n_env);

/* One DemoSim::step(dt) for every env. poses / velocities: DEVICE
 * [n_env][n_bodies][6] FP64, updated in place (velocity = world [linear;
 * angular]). deepest: optional DEVICE [n_env] FP64 deepest_penetration();
 * ok: optional DEVICE [n_env] int32, 0 where the state went non-finite (the
 * reference's step() == false; that env's state is then undefined). workspace:
 * optional (cmgb_demo_workspace_bytes), else taken from the stream-ordered pool. */
int cmgb_demo_step_batch(const cmgb_demo_body* bodies, int32_t n_bodies, const cmgb_config* cfg,
                         const cmgb_demo_params* params, double dt, int64_t n_env, double* poses,
                         double* velocities, double* deepest, int32_t* ok, void* workspace,
                         size_t workspace_bytes, void* cuda_stream);

/* ---------------------------------------------------------------------------
 * Multi-body scenes — the all-pairs loop of DemoSim::step (src/demosim.cpp:
 * 88-104): every body pair (i < j) except static-static, for every env.
 * ------------------------------------------------------------------------- */
/* Enumerate the pairs in (i, j) lexicographic order; pairs may be null to
 * query the count. is_static: [n_bodies] 0/1 (nullable = all dynamic). */
int cmgb_scene_pairs(const int32_t* is_static, int32_t n_bodies, int32_t* pairs, int32_t* n_pairs);
/* poses: DEVICE [n_env][n_bodies][6]; outs[q] receives pair q's manifolds
 * (layout of cmgb_layout_query(bodies[i], bodies[j])). */
int cmgb_manifold_scene_batch(const cmgb_surface* bodies, int32_t n_bodies, const int32_t* pairs,
                              int32_t n_pairs, const double* poses, int64_t n_env,
                              const cmgb_config* cfg, const cmgb_manifold_out* outs,
                              void* cuda_stream);
/* The same with HOST buffers: poses_host [n_env][n_bodies][6] in, each pair's
 * per-env mean contact distance mean_dist_host [n_pairs][n_env] out (copies
 * inside; a lead env chunk, then the rest, so the rest's upload overlaps the
 * lead chunk's kernels). Synchronous. */
int cmgb_manifold_scene_batch_host(const cmgb_surface* bodies, int32_t n_bodies, const int32_t* pairs,
                                   int32_t n_pairs, const double* poses_host, int64_t n_env,
                                   const cmgb_config* cfg, float* mean_dist_host, void* cuda_stream);
/* Config D's "forward + 12-tangent JVP per pair": pair q's primal contacts and
 * pose Jacobians (w.r.t. the poses of bodies[pairs[2q]] and bodies[pairs[2q+1]])
 * into outs[q], as cmgb_manifold_jvp_batch. */
int cmgb_manifold_scene_jvp_batch(const cmgb_surface* bodies, int32_t n_bodies, const int32_t* pairs,
                                  int32_t n_pairs, const double* poses, int64_t n_env,
                                  const cmgb_config* cfg, const cmgb_manifold_jvp_out* outs,
                                  void* cuda_stream);

/* ---------------------------------------------------------------------------
 * Witness batches — run_ee_batch / run_vf_batch (src/batch.cpp:53-98) over
 * ee_witness / vf_witness (include/cmg/witness.hpp:137-158, 163-227).
 * pairs: DEVICE [n][12] (e1a,e1b,e2a,e2b | v,t0,t1,t2), FP64 if pairs_fp64
 * else FP32. out: DEVICE FP32 [n][6] (p1,p2) | [n][3] (closest point).
 * alpha_gamma (optional, E-E): [n][3] = alpha1, alpha2, gamma_con.
 * labels (optional): active-set label per pair = argmax candidate weight
 * (0..3 E-E, 0..2 V-F) | (inside-indicator >= 0.5) << 2.
 * ------------------------------------------------------------------------- */
int cmgb_ee_witness_batch(const void* pairs, int32_t pairs_fp64, int64_t n,
                          const cmgb_config* cfg, float* out, float* alpha_gamma,
                          int32_t* labels, void* cuda_stream);
/* SDF queries on one surface (SmoothSdf::value / value_and_gradient /
 * value_and_normal_source, include/cmg/sdf.hpp:177-195): points DEVICE [n][3]
 * in the body frame; out DEVICE [n][4] = value, gradient (flavor 1) or normal
 * source (flavor 2; zeros for flavor 0). */
int cmgb_sdf_query(cmgb_surface s, int32_t flavor, const double* points, int64_t n, double* out,
                   void* cuda_stream);

/* sphere_trace_project against the posed SDF (sdf.hpp:318-326): world points
 * DEVICE [n][3], pose HOST [6], iters steps with normalisation tau; out DEVICE
 * [n][3] world points. */
int cmgb_sphere_trace(cmgb_surface s, const double* pose, const double* points, int64_t n, int32_t iters,
                      double tau, double* out, void* cuda_stream);

/* Reference-precision E-E witnesses: FP64 pairs in, FP64 soft indicators,
 * FP64 outputs out [n][6] (alpha_gamma [n][3] FP64, labels optional): what
 * ee_witness<double> returns (witness.hpp:137-158). */
int cmgb_ee_witness_batch_f64(const double* pairs, int64_t n, const cmgb_config* cfg, double* out,
                              double* alpha_gamma, int32_t* labels, void* cuda_stream);

/* rotating_edge_sweep (src/sweep.cpp:17-56, Fig. 4): variant 0 = no smoothing,
 * 1 = regularised only (hard, lambda 0.01), 2 = smooth (tau 0.1, lambda 0.01);
 * out_host [n_samples][7] = theta, p1 (3), dp1/dtheta (3, central difference
 * h = 1e-7), theta over [0, pi]. Synchronous (host buffers). */
int cmgb_rotating_edge_sweep(int32_t variant, int32_t n_samples, double* out_host);

int cmgb_vf_witness_batch(const void* pairs, int32_t pairs_fp64, int64_t n,
                          const cmgb_config* cfg, float* out, int32_t* labels,
                          void* cuda_stream);

/* Host-buffer witness batches with the reference's output precision
 * (run_ee_batch / run_vf_batch write doubles, src/batch.cpp:53-98): pairs_host
 * [n][12] FP64; out_host [n][6] (E-E: the FP64 solver of
 * cmgb_ee_witness_batch_f64) / [n][3] (V-F: FP32 solver, widened on the
 * device); labels optional. Synchronous. Batches of >= 131,072 pairs run as a
 * two-stream pipeline over up to 8 pair chunks (a chunk's upload overlaps the
 * previous chunk's kernel and download); page-locked host buffers let the
 * copies run asynchronously. Results are bit-identical to the device-buffer
 * calls. */
int cmgb_ee_witness_batch_host(const double* pairs_host, int64_t n, const cmgb_config* cfg, double* out_host,
                               int32_t* labels_host, void* cuda_stream);
int cmgb_vf_witness_batch_host(const double* pairs_host, int64_t n, const cmgb_config* cfg, double* out_host,
                               int32_t* labels_host, void* cuda_stream);

/* ---------------------------------------------------------------------------
 * Device info (SM count etc. queried, never hard-coded).
 * ------------------------------------------------------------------------- */
int cmgb_device_count(int32_t* count);

#ifdef __cplusplus
}  /* extern "C" */
#endif

#endif /* CMGB_H_ */
