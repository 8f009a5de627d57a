// geometry.cpp — level set + background mesh classification (TEST INFRASTRUCTURE).
// Restates /root/reference/proj/src/core/levelset.cpp and mesh.cpp semantics.
#include <algorithm>
#include <atomic>
#include <cmath>

#include "oracle.hpp"

namespace oracle {

namespace {
std::atomic<int> g_threads{1};
}
int thread_count() { return g_threads.load(); }
void set_thread_count(int n) { g_threads.store(n < 1 ? 1 : n); }

// levelset.cpp:27-31: d = x - c; return d.norm() - r. Eigen's norm() of a
// Vector3d is sqrt((dx*dx + dy*dy) + dz*dz) (no FMA: built -ffp-contract=off).
// Union: levelset.cpp:129-133 pattern, v = phi_0; v = min(v, phi_i).
double phi(const Geometry& g, double x, double y, double z) {
  double v = 0;
  for (size_t i = 0; i < g.balls.size(); ++i) {
    const Ball& b = g.balls[i];
    const double dx = x - b.cx, dy = y - b.cy, dz = z - b.cz;
    const double s = std::sqrt(dx * dx + dy * dy + dz * dz) - b.r;
    v = i == 0 ? s : std::min(v, s);
  }
  return v;
}

// mesh.cpp:46-53
void Mesh::node_coords(std::int64_t node, int out[3]) const {
  const std::int64_t nz = n[2] + 1;
  out[2] = (int)(node % nz);
  const std::int64_t rest = node / nz;
  out[1] = (int)(rest % (n[1] + 1));
  out[0] = (int)(rest / (n[1] + 1));
}

// mesh.cpp:32-39
void Mesh::cell_coords(std::int64_t cell, int out[3]) const {
  out[2] = (int)(cell % n[2]);
  const std::int64_t rest = cell / n[2];
  out[1] = (int)(rest % n[1]);
  out[0] = (int)(rest / n[1]);
}

// mesh.cpp:65-72: local node l uses bit l = lx + 2*ly + 4*lz (mesh.hpp:52).
void Mesh::cell_nodes(std::int64_t cell, std::int64_t out[8]) const {
  int c[3];
  cell_coords(cell, c);
  for (int l = 0; l < 8; ++l) out[l] = node_id(c[0] + (l & 1), c[1] + ((l >> 1) & 1), c[2] + ((l >> 2) & 1));
}

// mesh.cpp:74-108 (3-D branch): the lattice edge is active when any of the
// (up to 4) cells sharing it is non-exterior.
bool Mesh::edge_active(std::int64_t na, std::int64_t nb) const {
  int a[3], b[3];
  node_coords(na, a);
  node_coords(nb, b);
  int axis = -1;
  for (int d = 0; d < 3; ++d) {
    if (a[d] != b[d]) {
      if (axis != -1 || std::abs(a[d] - b[d]) != 1) return false;
      axis = d;
    }
  }
  if (axis < 0) return false;
  const int i0 = std::min(a[0], b[0]), j0 = std::min(a[1], b[1]), k0 = std::min(a[2], b[2]);
  for (int da = -1; da <= 0; ++da) {
    for (int db = -1; db <= 0; ++db) {
      int ci = i0, cj = j0, ck = k0;
      if (axis == 0) {
        cj += da;
        ck += db;
      } else if (axis == 1) {
        ci += da;
        ck += db;
      } else {
        ci += da;
        cj += db;
      }
      if (ci < 0 || cj < 0 || ck < 0 || ci >= n[0] || cj >= n[1] || ck >= n[2]) continue;
      if (cls[(size_t)cell_id(ci, cj, ck)] != kExterior) return true;
    }
  }
  return false;
}

// mesh.cpp:114-169
Mesh classify(const MeshParams& p, const Geometry& g) {
  Mesh m;
  for (int d = 0; d < 3; ++d) {
    m.n[d] = p.cells[d];
    if (m.n[d] < 1) fail(ErrorCode::InvalidArgument, "mesh: needs at least one cell per axis");
  }
  for (int d = 0; d < 3; ++d) m.origin[d] = p.lo[d] + p.translation[d];                 // :122
  for (int d = 0; d < 3; ++d) m.h[d] = (p.hi[d] - p.lo[d]) / m.n[d];                     // :123
  double hmin = std::min(m.h[0], std::min(m.h[1], m.h[2]));
  if (!(hmin > 0)) fail(ErrorCode::InvalidArgument, "mesh: non-positive cell size");
  m.tol = 1e-12 * hmin;                                                                    // :128
  const std::int64_t nn = m.n_nodes();
  m.phi.resize((size_t)nn);
  parallel_for(nn, [&](std::int64_t node) {                                                // :132-136
    int c[3];
    m.node_coords(node, c);
    // mesh.cpp:55-58: origin_ + Vec3(i*h0, j*h1, k*h2), component-wise.
    const double x = m.origin[0] + c[0] * m.h[0];
    const double y = m.origin[1] + c[1] * m.h[1];
    const double z = m.origin[2] + c[2] * m.h[2];
    double v = phi(g, x, y, z);
    if (std::abs(v) <= m.tol) v = -m.tol;
    m.phi[(size_t)node] = v;
  });
  const std::int64_t nc = m.n_cells();
  m.cls.resize((size_t)nc);
  parallel_for(nc, [&](std::int64_t cell) {                                                // :141-149
    std::int64_t nodes[8];
    m.cell_nodes(cell, nodes);
    int neg = 0;
    for (int l = 0; l < 8; ++l)
      if (m.phi[(size_t)nodes[l]] < 0) ++neg;
    m.cls[(size_t)cell] = neg == 8 ? kInterior : (neg == 0 ? kExterior : kCut);
  });
  for (std::int64_t c = 0; c < nc; ++c)                                                    // :151-153
    if (m.cls[(size_t)c] != kExterior) m.active.push_back(c);
  if (m.active.empty()) fail(ErrorCode::InvalidArgument, "mesh: empty active mesh");
  m.dof_of_node.assign((size_t)nn, -1);                                                    // :155-167
  for (std::int64_t c : m.active) {
    std::int64_t nodes[8];
    m.cell_nodes(c, nodes);
    for (int l = 0; l < 8; ++l) m.dof_of_node[(size_t)nodes[l]] = 0;
  }
  for (std::int64_t node = 0; node < nn; ++node) {
    if (m.dof_of_node[(size_t)node] == 0) {
      m.dof_of_node[(size_t)node] = m.n_dof++;
      m.node_of_dof.push_back(node);
    }
  }
  return m;
}

}  // namespace oracle
