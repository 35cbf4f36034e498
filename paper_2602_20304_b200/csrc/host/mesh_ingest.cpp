// Collision-mesh ingest for the C ABI (host only).
//
// Semantics follow the reference so that candidate indices (vertex order,
// edge order) are identical:
//   box generator   src/mesh.cpp:123-173  (face grids +z,-z,+x,-x,+y,-y; lattice
//                                          welding at 1e-9; edges in lexicographic
//                                          (lo, hi) order; quads drop diagonals)
//   OBJ subset      src/mesh.cpp:60-115   (v / f lines, tri or quad, "i/j/k" and
//                                          negative indices, quad diagonals removed
//                                          from the edge set, non-manifold warning)
#include <cmath>
#include <set>
#include <sstream>

#include "host.h"

namespace cmgb {

double Mesh::bounding_diagonal() const {
  if (vertices.empty()) return 0.0;
  double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
  for (size_t i = 0; i < vertices.size(); i += 3)
    for (int k = 0; k < 3; ++k) {
      lo[k] = std::min(lo[k], vertices[i + k]);
      hi[k] = std::max(hi[k], vertices[i + k]);
    }
  const double dx = hi[0] - lo[0], dy = hi[1] - lo[1], dz = hi[2] - lo[2];
  return std::sqrt(dx * dx + dy * dy + dz * dz);
}

namespace {

using EdgeKey = std::array<int, 2>;
EdgeKey ordered(int a, int b) { return a < b ? EdgeKey{a, b} : EdgeKey{b, a}; }

void emit_edges(const std::set<EdgeKey>& set, Mesh* m) {
  m->edges.clear();
  m->edges.reserve(set.size() * 2);
  for (const EdgeKey& e : set) {
    m->edges.push_back(e[0]);
    m->edges.push_back(e[1]);
  }
}

}  // namespace

Mesh make_box_mesh(const double half[3], int subdivisions, bool quad_edges) {
  if (subdivisions < 1) invalid("make_box_mesh: subdivisions >= 1");
  Mesh m;
  std::map<std::array<long long, 3>, int> lattice;
  auto vertex_at = [&](double u, double v, double w) {
    const std::array<long long, 3> key{std::llround(u * 1e9), std::llround(v * 1e9),
                                       std::llround(w * 1e9)};
    const auto found = lattice.find(key);
    if (found != lattice.end()) return found->second;
    const int id = m.nv();
    m.vertices.insert(m.vertices.end(), {u * half[0], v * half[1], w * half[2]});
    lattice.emplace(key, id);
    return id;
  };
  std::set<EdgeKey> edges;
  const int n = subdivisions;
  // (origin, du, dv) per face grid, in the generator's order.
  const double grids[6][9] = {
      {0, 0, 1, 1, 0, 0, 0, 1, 0},  {0, 0, -1, 1, 0, 0, 0, 1, 0}, {1, 0, 0, 0, 1, 0, 0, 0, 1},
      {-1, 0, 0, 0, 1, 0, 0, 0, 1}, {0, 1, 0, 1, 0, 0, 0, 0, 1},  {0, -1, 0, 1, 0, 0, 0, 0, 1},
  };
  for (const auto& g : grids) {
    auto corner = [&](double u, double v) {
      const double q[3] = {g[0] + g[3] * u + g[6] * v, g[1] + g[4] * u + g[7] * v,
                           g[2] + g[5] * u + g[8] * v};
      return vertex_at(q[0], q[1], q[2]);
    };
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) {
        const double u0 = -1.0 + 2.0 * i / n, u1 = -1.0 + 2.0 * (i + 1) / n;
        const double v0 = -1.0 + 2.0 * j / n, v1 = -1.0 + 2.0 * (j + 1) / n;
        const int a = corner(u0, v0);
        const int b = corner(u1, v0);
        const int c = corner(u1, v1);
        const int d = corner(u0, v1);
        m.faces.insert(m.faces.end(), {a, b, c, a, c, d});
        edges.insert(ordered(a, b));
        edges.insert(ordered(b, c));
        edges.insert(ordered(c, d));
        edges.insert(ordered(d, a));
        if (!quad_edges) edges.insert(ordered(a, c));
      }
  }
  emit_edges(edges, &m);
  return m;
}

namespace {

// "7", "7/2", "7/2/3", "7//3" -> zero-based vertex index (negative = relative).
int face_index(const std::string& tok, int nv, int line) {
  const std::string head = tok.substr(0, tok.find('/'));
  long v = 0;
  try {
    size_t used = 0;
    v = std::stol(head, &used);
  } catch (const std::exception&) {
    throw Error(CMGB_ERR_PARSE, "bad face index '" + tok + "' (line " + std::to_string(line) + ")",
                line);
  }
  if (v < 0) v = nv + 1 + v;
  if (v < 1 || v > nv)
    throw Error(CMGB_ERR_PARSE, "face index out of range (line " + std::to_string(line) + ")", line);
  return static_cast<int>(v - 1);
}

}  // namespace

Mesh parse_obj_text(const std::string& text) {
  Mesh m;
  std::set<EdgeKey> boundary, diagonals;
  std::istringstream in(text);
  std::string raw;
  int line = 0;
  while (std::getline(in, raw)) {
    ++line;
    std::istringstream ls(raw);
    std::string tag;
    if (!(ls >> tag) || tag[0] == '#') continue;
    if (tag == "v") {
      double x, y, z;
      if (!(ls >> x >> y >> z))
        throw Error(CMGB_ERR_PARSE, "bad vertex line (line " + std::to_string(line) + ")", line);
      m.vertices.insert(m.vertices.end(), {x, y, z});
    } else if (tag == "f") {
      std::vector<int> ids;
      std::string tok;
      while (ls >> tok) ids.push_back(face_index(tok, m.nv(), line));
      const size_t k = ids.size();
      if (k != 3 && k != 4)
        throw Error(CMGB_ERR_PARSE,
                    "only triangle and quad faces are supported (line " + std::to_string(line) + ")",
                    line);
      m.faces.insert(m.faces.end(), {ids[0], ids[1], ids[2]});
      if (k == 4) {
        m.faces.insert(m.faces.end(), {ids[0], ids[2], ids[3]});
        diagonals.insert(ordered(ids[0], ids[2]));
      }
      for (size_t q = 0; q < k; ++q) boundary.insert(ordered(ids[q], ids[(q + 1) % k]));
    }
  }
  if (m.vertices.empty() || m.faces.empty())
    throw Error(CMGB_ERR_PARSE, "no geometry found (line " + std::to_string(line) + ")", line);
  // Quad diagonals leave the edge set (the reference removes them unconditionally).
  for (const EdgeKey& d : diagonals) boundary.erase(d);
  std::map<EdgeKey, int> uses;
  for (size_t f = 0; f < m.faces.size(); f += 3)
    for (int q = 0; q < 3; ++q) {
      const EdgeKey e = ordered(m.faces[f + q], m.faces[f + (q + 1) % 3]);
      if (boundary.count(e)) ++uses[e];
    }
  emit_edges(boundary, &m);
  for (const auto& [e, count] : uses)
    if (count > 2)
      m.warnings.push_back("non-manifold edge (" + std::to_string(e[0]) + "," +
                           std::to_string(e[1]) + ") shared by " + std::to_string(count) + " faces");
  return m;
}

}  // namespace cmgb
