/*
 * TEST INFRASTRUCTURE — CPU oracle for the batched contact-manifold path.
 *
 * A plain-C (C11, double precision) restatement of the reference algorithm
 * (/root/reference/proj, arXiv 2602.20304). Used only by tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg as the CHECKER;
 * never linked into or called by the product library.
 *
 * Pinning: tests/test_oracle_golden.py checks this restatement against golden
 * vectors produced by the compiled reference itself (oracle/_ref, see
 * tests/golden/make_golden.py) and against SPEC.md's known-answer examples.
 */
#ifndef CMG_ORACLE_H_
#define CMG_ORACLE_H_

#include <stdint.h>

#include "../include/cmgb.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct orc_surface orc_surface;

/* Surface = mesh (vertices, edges) + SDF program + budgets (surface.hpp:16-33). */
orc_surface* orc_surface_create(const double* vertices, int32_t n_vertices, const int32_t* edges,
                                int32_t n_edges, const cmgb_sdf_node* nodes, int32_t n_nodes,
                                int32_t vertex_topk, int32_t edge_topk);
void orc_surface_destroy(orc_surface* s);
/* out: effective vertex top-K, effective edge top-K, leaf count. */
void orc_surface_budgets(const orc_surface* s, int32_t* out3);

/* flavor 0 value | 1 value_and_gradient | 2 value_and_normal_source; body frame.
 * out: n x 4 (value, gx, gy, gz). */
void orc_sdf_query(const orc_surface* s, int32_t flavor, const double* p, int64_t n, double* out);
void orc_sphere_trace(const orc_surface* s, const double* pose, const double* p, int64_t n,
                      int32_t iters, double tau, double* out);

/* generate_manifold<double> for one env. layout out: n1, n2, m1, m2, n_contacts.
 * contacts: C x 8; meta: C x 4 (kind, side, src_a, src_b); ee: 9 x m1m2 (nullable). */
int orc_manifold(const orc_surface* s1, const orc_surface* s2, const double* pose1,
                 const double* pose2, const cmgb_config* cfg, double* contacts, int32_t* meta,
                 double* ee, int32_t* layout);
/* Many envs, `threads` pthreads; outputs per env (contacts/meta/ee nullable). */
int orc_manifold_batch(const orc_surface* s1, const orc_surface* s2, const double* poses1,
                       int32_t pose1_stride, const double* poses2, int32_t pose2_stride,
                       int64_t n_env, const cmgb_config* cfg, int32_t threads, double* contacts,
                       int32_t* meta, double* ee, double* mean_dist);

/* ee_witness over n pairs (n x 12): out n x 9 (p1, p2, alpha1, alpha2, gamma).
 * labels (nullable): argmax of pick_min weights | (gamma_con >= 0.5) << 2. */
void orc_ee_witness(const double* pairs, int64_t n, const cmgb_config* cfg, double* out,
                    int32_t* labels);
/* vf_witness over n pairs: out n x 3, labels as above over 3 candidates. */
void orc_vf_witness(const double* pairs, int64_t n, const cmgb_config* cfg, double* out,
                    int32_t* labels);
/* solve_box_qp_2: qp n x 5 (q11, q12, q22, c1, c2) -> n x 3 (alpha1, alpha2, gamma). */
void orc_box_qp(const double* qp, int64_t n, const cmgb_config* cfg, double* out);

void orc_se3_exp(const double* pose, double* R, double* t);
int orc_soft_topk(const double* xs, int32_t d, int32_t k, double tau, double* w);
void orc_mt19937_64_uniform(uint64_t seed, int64_t n, double lo, double hi, double* out);

#ifdef __cplusplus
}
#endif
#endif
