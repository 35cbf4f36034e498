// SDF programs on the host: validation with the reference's messages
// (sdf.hpp:41-77, sdf.cpp:33-43), a double-precision value evaluator used
// only by the build-time mesh/SDF discrepancy check (surface.cpp:31-42), and
// packing into the kernels' DevSdf parameter image.
#include <cmath>

#include "host.h"

namespace cmgb {

void se3_exp_host(const double xi[6], double R[9], double t[3]) {
  const double wx = xi[3], wy = xi[4], wz = xi[5];
  const double th2 = wx * wx + wy * wy + wz * wz;
  double a, b, c;
  if (th2 < 1e-8) {
    a = 1.0 - th2 / 6.0 + th2 * th2 / 120.0;
    b = 0.5 - th2 / 24.0 + th2 * th2 / 720.0;
    c = 1.0 / 6.0 - th2 / 120.0 + th2 * th2 / 5040.0;
  } else {
    const double th = std::sqrt(th2);
    a = std::sin(th) / th;
    b = (1.0 - std::cos(th)) / th2;
    c = (1.0 - a) / th2;
  }
  const double W[9] = {0, -wz, wy, wz, 0, -wx, -wy, wx, 0};
  double W2[9];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      W2[3 * i + j] = W[3 * i] * W[j] + W[3 * i + 1] * W[3 + j] + W[3 * i + 2] * W[6 + j];
  double V[9];
  for (int i = 0; i < 9; ++i) {
    const double id = (i % 4 == 0) ? 1.0 : 0.0;
    R[i] = (id + W[i] * a) + W2[i] * b;
    V[i] = (id + W[i] * b) + W2[i] * c;
  }
  for (int r = 0; r < 3; ++r) t[r] = V[3 * r] * xi[0] + V[3 * r + 1] * xi[1] + V[3 * r + 2] * xi[2];
}

namespace {

void check_unit(const std::vector<double>& n, const char* what) {
  for (size_t i = 0; i < n.size(); i += 3) {
    const double len = std::sqrt(n[i] * n[i] + n[i + 1] * n[i + 1] + n[i + 2] * n[i + 2]);
    if (std::abs(len - 1.0) > 1e-9) invalid(std::string(what) + ": normals must be unit length");
  }
}

}  // namespace

Program make_program(const cmgb_sdf_node* in, int n) {
  if (!in || n < 1) invalid("sdf: program needs at least one node");
  Program prog;
  prog.nodes.resize(n);
  std::vector<int> stack;
  std::vector<int> leaves;  // per node: leaf count of its subtree
  leaves.resize(n, 0);
  for (int i = 0; i < n; ++i) {
    const cmgb_sdf_node& s = in[i];
    ProgramNode& d = prog.nodes[i];
    d.op = s.op;
    d.count = s.count;
    d.tau = s.tau;
    switch (s.op) {
      case CMGB_SDF_SUPERQUADRIC:
        if (!(s.eps1 > 0.0 && s.eps1 <= 2.0 && s.eps2 > 0.0 && s.eps2 <= 2.0))
          invalid("superquadric: eps1, eps2 must lie in (0, 2]");
        if (!(s.axes[0] > 0.0 && s.axes[1] > 0.0 && s.axes[2] > 0.0))
          invalid("superquadric: axis lengths must be positive");
        d.eps1 = s.eps1;
        d.eps2 = s.eps2;
        for (int k = 0; k < 3; ++k) d.axes[k] = s.axes[k];
        for (int k = 0; k < 6; ++k) d.pose[k] = s.pose[k];
        se3_exp_host(d.pose, d.R, d.t);
        leaves[i] = 1;
        stack.push_back(i);
        break;
      case CMGB_SDF_CONVEX_POLYHEDRON:
        if (s.count < 1 || !s.normals || !s.points)
          invalid("convex polyhedron: need matching normals/points, N >= 1");
        d.normals.assign(s.normals, s.normals + 3 * s.count);
        d.points.assign(s.points, s.points + 3 * s.count);
        check_unit(d.normals, "convex polyhedron");
        if (!(s.tau > 0.0)) invalid("convex polyhedron: tau > 0");
        leaves[i] = 1;
        stack.push_back(i);
        break;
      case CMGB_SDF_ORIENTED_POINTCLOUD:
        if (s.count < 1 || !s.normals || !s.points || !s.lengthscales)
          invalid("oriented pointcloud: need matching arrays, N >= 1");
        d.normals.assign(s.normals, s.normals + 3 * s.count);
        d.points.assign(s.points, s.points + 3 * s.count);
        d.lengthscales.assign(s.lengthscales, s.lengthscales + s.count);
        check_unit(d.normals, "oriented pointcloud");
        for (double th : d.lengthscales)
          if (!(th > 0.0)) invalid("oriented pointcloud: lengthscales > 0");
        leaves[i] = 1;
        stack.push_back(i);
        break;
      case CMGB_SDF_UNION:
        if (s.count < 1) invalid("smooth_union: need at least one child");
        if (!(s.tau > 0.0)) invalid("smooth_union: tau > 0");
        if (static_cast<size_t>(s.count) > stack.size()) invalid("sdf: union pops more children than exist");
        d.children.assign(stack.end() - s.count, stack.end());
        stack.resize(stack.size() - s.count);
        for (int ch : d.children) leaves[i] += leaves[ch];
        stack.push_back(i);
        break;
      case CMGB_SDF_SUBTRACTION:
        if (!(s.tau > 0.0)) invalid("subtraction: tau > 0");
        if (stack.size() < 2) invalid("sdf: subtraction needs two operands");
        d.count = 2;
        d.children.assign(stack.end() - 2, stack.end());
        stack.resize(stack.size() - 2);
        leaves[i] = leaves[d.children[0]] + leaves[d.children[1]];
        stack.push_back(i);
        break;
      default:
        invalid("sdf: unknown node op " + std::to_string(s.op));
    }
    prog.max_stack = std::max<int>(prog.max_stack, static_cast<int>(stack.size()));
  }
  if (stack.size() != 1) invalid("sdf: postfix program must leave exactly one root");
  prog.root = stack[0];
  prog.leaf_count = leaves[prog.root];
  return prog;
}

double Program::value(const double p[3]) const { return node_value(root, p); }

// phi in double (sdf.hpp:85-132, 204-231); validation-time use only.
double Program::node_value(int i, const double p[3]) const {
  const ProgramNode& d = nodes[i];
  switch (d.op) {
    case CMGB_SDF_SUPERQUADRIC: {
      const double q[3] = {p[0] - d.t[0], p[1] - d.t[1], p[2] - d.t[2]};
      double l[3];
      for (int r = 0; r < 3; ++r) l[r] = d.R[r] * q[0] + d.R[3 + r] * q[1] + d.R[6 + r] * q[2];
      const double xn = l[0] / d.axes[0], yn = l[1] / d.axes[1], zn = l[2] / d.axes[2];
      const double g = std::pow(xn * xn + 1e-30, 1.0 / d.eps2) + std::pow(yn * yn + 1e-30, 1.0 / d.eps2);
      const double f = std::pow(g, d.eps2 / d.eps1) + std::pow(zn * zn + 1e-30, 1.0 / d.eps1);
      const double r = std::sqrt(xn * xn + yn * yn + zn * zn + 1e-20);
      return (1.0 - std::pow(f, -d.eps1 / 2.0)) / r;
    }
    case CMGB_SDF_CONVEX_POLYHEDRON: {
      std::vector<double> dist(d.count);
      double m = -1e300;
      for (int k = 0; k < d.count; ++k) {
        const double* n = &d.normals[3 * k];
        const double* o = &d.points[3 * k];
        dist[k] = n[0] * (p[0] - o[0]) + n[1] * (p[1] - o[1]) + n[2] * (p[2] - o[2]);
        m = std::max(m, dist[k]);
      }
      double acc = 0.0;
      for (double x : dist) acc += std::exp((x - m) / d.tau);
      return m + d.tau * std::log(acc);
    }
    case CMGB_SDF_ORIENTED_POINTCLOUD: {
      double num = 0.0, den = 1e-30;
      for (int k = 0; k < d.count; ++k) {
        const double r[3] = {p[0] - d.points[3 * k], p[1] - d.points[3 * k + 1], p[2] - d.points[3 * k + 2]};
        const double th = d.lengthscales[k];
        const double w = std::exp(-(r[0] * r[0] + r[1] * r[1] + r[2] * r[2]) / (2.0 * th * th));
        num += w * (d.normals[3 * k] * r[0] + d.normals[3 * k + 1] * r[1] + d.normals[3 * k + 2] * r[2]);
        den += w;
      }
      return num / den;
    }
    case CMGB_SDF_UNION: {
      std::vector<double> v;
      for (int ch : d.children) v.push_back(node_value(ch, p));
      double m = v[0];
      for (double x : v) m = std::min(m, x);
      double acc = 0.0;
      for (double x : v) acc += std::exp((m - x) / d.tau);
      return m - d.tau * std::log(acc);
    }
    default: {
      const double a = node_value(d.children[0], p), b = -node_value(d.children[1], p);
      const double m = std::max(a, b);
      return m + d.tau * std::log(std::exp((a - m) / d.tau) + std::exp((b - m) / d.tau));
    }
  }
}

namespace {

// Exact small positive integer (double) -> n, else 0.
int exact_int(double x) {
  if (!(x >= 1.0 && x <= 64.0)) return 0;
  const double r = std::nearbyint(x);
  return r == x ? static_cast<int>(r) : 0;
}

}  // namespace

namespace {

// Postfix order of the device program, from the tree. Unions wider than the
// interpreter's stack allows are emitted as left-deep chains of binary unions
// with the same temperature: -tau log sum exp(-phi_i / tau) is associative,
// and the blended gradient / normal source weights compose, so the chain is the
// same smooth minimum (rounding aside). Only programs that would not otherwise
// fit are rewritten; the others keep the reference's n-ary order exactly.
struct Emit {
  int src;    // program node
  int count;  // union arity of this emission (-1: the node's own)
};

int emit(const Program& prog, int i, bool chain, std::vector<Emit>* out) {  // returns the stack depth used
  const ProgramNode& d = prog.nodes[i];
  if (d.op != CMGB_SDF_UNION && d.op != CMGB_SDF_SUBTRACTION) {
    out->push_back({i, -1});
    return 1;
  }
  if (d.op == CMGB_SDF_SUBTRACTION || !chain || d.children.size() <= 2) {
    int depth = 0, k = 0;
    for (int ch : d.children) depth = std::max(depth, k++ + emit(prog, ch, chain, out));
    out->push_back({i, -1});
    return depth;
  }
  int depth = emit(prog, d.children[0], chain, out);
  for (size_t k = 1; k < d.children.size(); ++k) {
    depth = std::max(depth, 1 + emit(prog, d.children[k], chain, out));
    out->push_back({i, 2});
  }
  return depth;
}

}  // namespace

DevSdf pack_program(const Program& prog, std::vector<double4>* pool, std::vector<DevNode>* ext) {
  DevSdf s{};
  std::vector<Emit> order;
  int depth = emit(prog, prog.root, false, &order);
  if (depth > kMaxStack) {  // wide unions: binary chains
    order.clear();
    depth = emit(prog, prog.root, true, &order);
  }
  if (depth > kMaxStack)
    throw Error(CMGB_ERR_UNSUPPORTED, "sdf: composition nesting exceeds " + std::to_string(kMaxStack) + " levels");
  const int n = static_cast<int>(order.size());
  if (n > kMaxNodesExt)
    throw Error(CMGB_ERR_UNSUPPORTED, "sdf: programs are limited to " + std::to_string(kMaxNodesExt) +
                                          " nodes per surface");
  std::vector<DevNode> all(n);
  s.n_nodes = n;
  s.leaf_count = prog.leaf_count;
  s.max_stack = depth;
  s.kind = kGeneric;
  if (n == 1 && prog.nodes[0].op == CMGB_SDF_SUPERQUADRIC) s.kind = kSingleSq;
  if (n == 1 && prog.nodes[0].op == CMGB_SDF_CONVEX_POLYHEDRON) s.kind = kSingleCp;
  for (int i = 0; i < n; ++i) {
    const ProgramNode& d = prog.nodes[order[i].src];
    DevNode& o = all[i];
    o.op = d.op;
    o.count = order[i].count >= 0 ? order[i].count : d.count;
    o.tau_d = d.tau;
    o.inv_tau_d = d.tau > 0.0 ? 1.0 / d.tau : 0.0;
    o.offset = static_cast<int32_t>(pool->size());
    if (d.op == CMGB_SDF_SUPERQUADRIC) {
      DevSq& q = o.sq;
      for (int k = 0; k < 3; ++k) q.inv_ax[k] = 1.0 / d.axes[k];
      for (int k = 0; k < 3; ++k) q.ax[k] = d.axes[k];
      const double p1 = 1.0 / d.eps2, p2 = d.eps2 / d.eps1, p3 = 1.0 / d.eps1, p4 = -d.eps1 / 2.0;
      q.p1 = p1;
      q.p2 = p2;
      q.p3 = p3;
      q.c_xy = 2.0 * p1 * p2;
      q.c_z = 2.0 * p3;
      q.p4 = p4;
      q.n1 = exact_int(p1);
      q.n2 = exact_int(p2);
      q.n3 = exact_int(p3);
      q.n4 = exact_int(-1.0 / p4);
      bool ident = true, no_rot = true;
      for (int k = 0; k < 6; ++k) ident = ident && d.pose[k] == 0.0;
      for (int k = 3; k < 6; ++k) no_rot = no_rot && d.pose[k] == 0.0;
      // 2: translation only -- se3_exp of a zero rotation is I exactly, so
      // R^T (p - t) = p - t bit for bit (the capsule's caps)
      q.has_frame = ident ? 0 : (no_rot ? 2 : 1);
      for (int k = 0; k < 9; ++k) q.R[k] = d.R[k];
      for (int k = 0; k < 3; ++k) q.t[k] = d.t[k];
    } else if (d.op == CMGB_SDF_CONVEX_POLYHEDRON) {
      for (int k = 0; k < d.count; ++k) {
        const double* nn = &d.normals[3 * k];
        const double* pp = &d.points[3 * k];
        const double off = nn[0] * pp[0] + nn[1] * pp[1] + nn[2] * pp[2];
        pool->push_back(make_double4(nn[0], nn[1], nn[2], off));
      }
    } else if (d.op == CMGB_SDF_ORIENTED_POINTCLOUD) {
      for (int k = 0; k < d.count; ++k) {
        const double th = d.lengthscales[k];
        pool->push_back(make_double4(d.points[3 * k], d.points[3 * k + 1], d.points[3 * k + 2],
                                     -1.0 / (2.0 * th * th)));
        pool->push_back(make_double4(d.normals[3 * k], d.normals[3 * k + 1], d.normals[3 * k + 2],
                                     1.0 / (th * th)));
      }
    }
  }
  for (int i = 0; i < n && i < kMaxNodes; ++i) s.nodes[i] = all[i];
  if (n > kMaxNodes) *ext = std::move(all);

  if (s.kind == kSingleSq) {
    const DevSq& q = s.nodes[0].sq;
    for (int k : {kSqE01, kSqE02, kSqE025, kSqE05, kSqEll, kSqCyl}) {
      const SqExpTuple e = sq_exps(k);
      if (q.n1 == e.n1 && q.n2 == e.n2 && q.n3 == e.n3 && q.n4 == e.n4) s.kind = k;
    }
  }
  if (n == 4 && prog.nodes[3].op == CMGB_SDF_UNION && prog.nodes[3].count == 3) {
    auto sq_kind = [&](int i) {
      if (prog.nodes[i].op != CMGB_SDF_SUPERQUADRIC) return -1;
      const DevSq& q = s.nodes[i].sq;
      for (int k : {kSqCyl, kSqEll}) {
        const SqExpTuple e = sq_exps(k);
        if (q.n1 == e.n1 && q.n2 == e.n2 && q.n3 == e.n3 && q.n4 == e.n4) return k;
      }
      return -1;
    };
    // (the kernel evaluates the caps as translation-only leaves)
    if (sq_kind(0) == kSqCyl && sq_kind(1) == kSqEll && sq_kind(2) == kSqEll && s.nodes[1].sq.has_frame != 1 &&
        s.nodes[2].sq.has_frame != 1)
      s.kind = kCapsule;
  }
  if (s.kind == kSingleCp && prog.nodes[0].count == 6) {
    // the box_planes pattern: unit normals +x, -x, +y, -y, +z, -z in this order
    const ProgramNode& d = prog.nodes[0];
    bool box = true;
    for (int k = 0; k < 6 && box; ++k)
      for (int a = 0; a < 3; ++a) {
        const double want = a == k / 2 ? (k % 2 == 0 ? 1.0 : -1.0) : 0.0;
        box = box && d.normals[3 * k + a] == want;
      }
    if (box) {
      s.kind = kBoxCp;
      for (int k = 0; k < 6; ++k) s.nodes[0].box_w[k] = (*pool)[s.nodes[0].offset + k].w;
    }
  }
  return s;
}

}  // namespace cmgb
