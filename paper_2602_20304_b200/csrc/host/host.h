// Host-side internals of libcmgb (not part of the ABI).
#pragma once

#include <array>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include <vector_functions.h>

#include "../../../include/cmgb.h"
#include "../common.h"

namespace cmgb {

// Error carrying a cmgb_status across the C++ layer; converted at the ABI.
struct Error : std::runtime_error {
  Error(int st, const std::string& msg, int line = 0) : std::runtime_error(msg), status(st), line(line) {}
  int status;
  int line;
};

[[noreturn]] inline void invalid(const std::string& msg) { throw Error(CMGB_ERR_INVALID_ARGUMENT, msg); }

struct Mesh {
  std::vector<double> vertices;     // V x 3
  std::vector<int32_t> faces;       // F x 3
  std::vector<int32_t> edges;       // E x 2 (lo < hi, lexicographic for generated meshes)
  std::vector<std::string> warnings;
  int nv() const { return static_cast<int>(vertices.size() / 3); }
  int nf() const { return static_cast<int>(faces.size() / 3); }
  int ne() const { return static_cast<int>(edges.size() / 2); }
  double bounding_diagonal() const;
};

Mesh make_box_mesh(const double half[3], int subdivisions, bool quad_edges);
Mesh parse_obj_text(const std::string& text);

// Validated, owned copy of a postfix SDF program.
struct ProgramNode {
  int op = 0;
  int count = 0;
  double tau = 0.0;
  double eps1 = 1.0, eps2 = 1.0;
  double axes[3] = {1, 1, 1};
  double pose[6] = {0, 0, 0, 0, 0, 0};
  double R[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1}, t[3] = {0, 0, 0};  // body_from_prim
  std::vector<double> normals, points, lengthscales;
  std::vector<int> children;  // node indices
};

struct Program {
  std::vector<ProgramNode> nodes;
  int root = -1;
  int leaf_count = 0;
  int max_stack = 0;
  double value(const double p[3]) const;  // host phi (build-time validation only)
  double node_value(int i, const double p[3]) const;
};

Program make_program(const cmgb_sdf_node* nodes, int n);
void se3_exp_host(const double xi[6], double R[9], double t[3]);

// Device image of a program + geometry, one per CUDA device.
struct DeviceSurface {
  double* verts = nullptr;
  int32_t* edges = nullptr;
  double* edge_body = nullptr;  // [ne][6]: both endpoints of every edge (body frame), no index chase
  double4* pool = nullptr;
  DevNode* ext = nullptr;  // program nodes in device memory (programs above kMaxNodes)
  DevSdf sdf{};
};

// Packs a program into the kernels' image; programs above kMaxNodes nodes also
// return every node in *ext (the caller uploads it and sets DevSdf::ext).
DevSdf pack_program(const Program& prog, std::vector<double4>* pool, std::vector<DevNode>* ext);

}  // namespace cmgb

struct cmgb_mesh_s {
  cmgb::Mesh mesh;
};

struct cmgb_surface_s {
  cmgb::Mesh mesh;
  cmgb::Program program;
  int vertex_topk = 0, edge_topk = 0;
  std::vector<std::string> warnings;
  std::mutex mu;
  std::map<int, cmgb::DeviceSurface> device;  // per CUDA device ordinal
  int effective_vertex_topk() const;
  int effective_edge_topk() const;
};
