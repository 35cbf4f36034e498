// A C++ caller written against the REFERENCE's API (namespace cmg,
// /root/reference/proj/include/cmg). The same source builds two ways:
//   -DUSE_REFERENCE -I/root/reference/proj/include  + the reference library
//   -I<repo>/include                                + libcmgb.so (B200 path)
// tests/test_cpp_dropin.py builds both; the reference build's output is the
// golden (tests/golden/dropin_ref.json) the B200 build is compared with.
//
// Exercises: make_box_mesh / parse_obj / build_surface / SmoothSdf factories,
// SmoothingConfig + config_for_variant, generate_manifold<double> (box-box and
// box-on-plane, smooth and hard), ContactManifold fields incl. EeIndicatorMatrices,
// generate_manifold<Dual12> via seed_pose_tangents + mean_contact_distance,
// make_random_*_pairs + run_*_batch checksums, bench_manifold / write_bench_csv.
#include <cstdio>
#include <fstream>
#include <random>
#include <sstream>
#include <string>
#include <vector>

#include "cmg/batch.hpp"
#include "cmg/dual.hpp"
#include "cmg/manifold.hpp"
#include "cmg/manifold_io.hpp"
#include "cmg/mesh.hpp"
#include "cmg/scene.hpp"
#include "cmg/surface.hpp"

using namespace cmg;

static void print_manifold(const char* name, const ContactManifold<double>& m, bool last = false) {
  std::printf("\"%s\": {\"n1\": %d, \"n2\": %d, \"m1\": %d, \"m2\": %d, \"size\": %zu, \"contacts\": [", name, m.n1,
              m.n2, m.m1, m.m2, m.expected_size());
  for (size_t i = 0; i < m.contacts.size(); ++i) {
    const auto& c = m.contacts[i];
    std::printf("%s[%.17g, %.17g, %.17g, %.17g, %.17g, %.17g, %.17g, %.17g, %d, %d, %d, %d]", i ? ", " : "",
                c.point.x, c.point.y, c.point.z, c.dist, c.normal.x, c.normal.y, c.normal.z, c.activity,
                c.kind == ContactKind::kEdgeEdge ? 1 : 0, c.side, c.src_a, c.src_b);
  }
  std::printf("], \"ee_act1\": [");
  for (size_t i = 0; i < m.ee.act1.size(); ++i) std::printf("%s%.17g", i ? ", " : "", m.ee.act1[i]);
  std::printf("], \"ee_dist\": [");
  for (size_t i = 0; i < m.ee.dist.size(); ++i) std::printf("%s%.17g", i ? ", " : "", m.ee.dist[i]);
  std::printf("], \"mean\": %.17g}%s\n", mean_contact_distance(m), last ? "" : ",");
}

int main(int argc, char** argv) {
  if (argc == 4) {  // scene file -> manifold of bodies 0 and 1 -> CSV + JSON (cmd_manifold, main.cpp:124-148)
    const Scene scene = load_scene(argv[1]);
    const auto m = generate_manifold(scene.bodies[0].surface, scene.bodies[1].surface, scene.bodies[0].pose,
                                     scene.bodies[1].pose, scene.smoothing);
    std::ofstream csv(argv[2]);
    write_manifold_csv(csv, m);
    std::ofstream js(argv[3]);
    js << manifold_to_json(m);
    return 0;
  }
  SuperquadricParams sq;
  sq.eps1 = sq.eps2 = 0.1;
  sq.axes = {0.5, 0.5, 0.5};
  SurfaceModel box = build_surface(make_box_mesh({0.5, 0.5, 0.5}, 1, true), SmoothSdf::superquadric(sq), 0, 12);

  ConvexPolyhedronParams planes;
  const double h[3] = {2.0, 2.0, 0.1};
  for (int k = 0; k < 3; ++k)
    for (int s = 0; s < 2; ++s) {
      Vec3d n{0, 0, 0}, p{0, 0, 0};
      n[k] = s ? -1.0 : 1.0;
      p[k] = s ? -h[k] : h[k];
      planes.normals.push_back(n);
      planes.points.push_back(p);
    }
  SurfaceModel ground =
      build_surface(make_box_mesh({2.0, 2.0, 0.1}), SmoothSdf::convex_polyhedron(planes), 0, 0);

  // an OBJ-ingested tetrahedron with a capsule-like union SDF (parse_obj + smooth_union)
  std::istringstream obj("v 0 0 0\nv 0.3 0 0\nv 0 0.3 0\nv 0 0 0.3\nf 1 3 2\nf 1 2 4\nf 1 4 3\nf 2 3 4\n");
  SuperquadricParams s1, s2;
  s1.eps1 = s1.eps2 = 1.0;
  s1.axes = {0.15, 0.15, 0.15};
  s2 = s1;
  s2.pose = {0.1, 0.1, 0.1, 0, 0, 0};
  SurfaceModel tet = build_surface(parse_obj(obj),
                                   SmoothSdf::smooth_union({SmoothSdf::superquadric(s1), SmoothSdf::superquadric(s2)},
                                                           0.01),
                                   0, 3);

  SmoothingConfig cfg;
  const Pose6d pb{0, 0, 0.5, 0, 0, 0};
  const Pose6d pt{0.02, 0.035, 1.46, 0, 0, 0.7853981633974483};
  std::printf("{\n");
  print_manifold("box_box_ours", generate_manifold(box, box, pb, pt, cfg));
  print_manifold("box_box_ours_ns", generate_manifold(box, box, pb, pt, config_for_variant("ours_ns", cfg)));
  print_manifold("box_box_ours_ne", generate_manifold(box, box, pb, pt, config_for_variant("ours_ne", cfg)));
  print_manifold("box_on_plane", generate_manifold(box, ground, Pose6d{0, 0, 0.49, 0, 0, 0},
                                                   Pose6d{0, 0, -0.1, 0, 0, 0}, cfg));
  SurfaceModel box4 = box;
  box4.vertex_topk = 4;  // budget override after build_surface, as the reference CLI does
  print_manifold("box_on_plane_topk", generate_manifold(box4, ground, Pose6d{0.01, 0, 0.49, 0, 0, 0.1},
                                                        Pose6d{0, 0, -0.1, 0, 0, 0}, cfg));
  print_manifold("tet_vs_box", generate_manifold(tet, box, Pose6d{0.1, 0.05, 0.95, 0.1, 0.2, 0.3}, pb, cfg));

  // pose gradient as the reference's gradcheck does (main.cpp:202-205)
  const auto seeded = seed_pose_tangents(pb, pt);
  const auto md = generate_manifold(box, box, seeded.first, seeded.second, cfg);
  const Dual12 mean = mean_contact_distance(md);
  std::printf("\"grad_mean\": [%.17g", primal(mean));
  for (int k = 0; k < 12; ++k) std::printf(", %.17g", mean.d[k]);
  std::printf("],\n");

  // witness batches: make_random_*_pairs + run_*_batch checksums and outputs
  const EeProblemSet ee = make_random_ee_pairs(2000, 0);
  const VfProblemSet vf = make_random_vf_pairs(2000, 0);
  std::vector<double> ee_out, vf_out;
  const double cs_ee = run_ee_batch(ee, SmoothingConfig{}, 4, &ee_out);
  const double cs_ee_ns = run_ee_batch(ee, config_for_variant("ours_ns", SmoothingConfig{}), 4, nullptr);
  const double cs_vf = run_vf_batch(vf, SmoothingConfig{}, 4, &vf_out);
  std::printf("\"checksums\": [%.17g, %.17g, %.17g],\n\"ee_out\": [", cs_ee, cs_ee_ns, cs_vf);
  for (size_t i = 0; i < 60; ++i) std::printf("%s%.17g", i ? ", " : "", ee_out[i]);
  std::printf("],\n\"vf_out\": [");
  for (size_t i = 0; i < 30; ++i) std::printf("%s%.17g", i ? ", " : "", vf_out[i]);
  std::printf("],\n");

  // bench_manifold over a two-body scene + the CSV writer
  Scene scene;
  SceneBody b1, b2;
  b1.surface = box;
  b1.pose = pb;
  b2.surface = box;
  b2.pose = pt;
  scene.bodies = {b1, b2};
  const auto recs = bench_manifold(scene, {1024}, {"ours", "ours_ne"}, 0, 2, 4);
  std::ostringstream csv;
  write_bench_csv(csv, recs);
  std::string line0 = csv.str().substr(0, csv.str().find('\n'));
  std::printf("\"bench\": {\"records\": %zu, \"csv_header\": \"%s\", \"kinds\": [\"%s\", \"%s\"], \"qps_positive\": %d}\n",
              recs.size(), line0.c_str(), recs[0].variant.c_str(), recs[1].variant.c_str(),
              recs[0].throughput_qps > 0 && recs[1].throughput_qps > 0 ? 1 : 0);
  std::printf("}\n");
  return 0;
}
