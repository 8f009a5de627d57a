// quadrature.cpp — sub-simplex cut-cell quadrature (TEST INFRASTRUCTURE).
// SPEC.md:139-184 (build_cut_quadrature :150-158, full_cell_quadrature
// :159-167, design decisions :172-175). Pins:
//   * Kuhn split along the v0-v7 diagonal in the local bit order of
//     mesh.hpp:52 (l = lx + 2ly + 4lz): for each axis permutation (a,b,c) in
//     lexicographic order the tet is v0, v0+e_a, v0+e_a+e_b, v7.
//   * edge point X_uv = P_u + t (P_v - P_u), t = q_u / (q_u - q_v).
//   * 1 negative vertex a: tet (a, X_ab, X_ac, X_ad); facet (X_ab, X_ac, X_ad).
//     3 negative (d positive): prism (a,b,c | X_ad,X_bd,X_cd); facet (X_ad,X_bd,X_cd).
//     2 negative (a,b): prism (a, X_ac, X_ad | b, X_bc, X_bd);
//       facets (X_ac, X_ad, X_bd), (X_ac, X_bd, X_bc).
//     prism (A,B,C | A',B',C') -> tets (A,B,C,A'), (B,C,A',B'), (C,A',B',C').
//   * 4-point degree-2 tet rule, 3-point degree-2 triangle rule.
//   * pieces with volume < 1e-14 |e| (facets with area < 1e-14 |e|^(2/3)) dropped.
//   * normal = gradient of the tet's linear interpolant, normalised.
// All in reference coordinates of the unit cell; the physical cell is x_lo + h*xi.
#include <cmath>

#include "oracle.hpp"

namespace oracle {

namespace {

struct P3 {
  double x, y, z;
};
inline P3 sub(P3 a, P3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
inline P3 lerp_edge(P3 pu, P3 pv, double qu, double qv) {
  const double t = qu / (qu - qv);
  return {pu.x + t * (pv.x - pu.x), pu.y + t * (pv.y - pu.y), pu.z + t * (pv.z - pu.z)};
}
inline P3 cross(P3 a, P3 b) { return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x}; }
inline double dot3(P3 a, P3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }

constexpr double kTetA = 0.5854101966249685;
constexpr double kTetB = 0.1381966011250105;
constexpr double kDrop = 1e-14;

void add_tet(CutRule& r, P3 a, P3 b, P3 c, P3 d) {
  const double vol = std::fabs(dot3(sub(b, a), cross(sub(c, a), sub(d, a)))) / 6.0;
  if (vol < kDrop) {
    ++r.dropped;
    return;
  }
  const P3 v[4] = {a, b, c, d};
  for (int i = 0; i < 4; ++i) {
    double x = kTetA * v[i].x, y = kTetA * v[i].y, z = kTetA * v[i].z;
    for (int j = 0; j < 4; ++j) {
      if (j == i) continue;
      x += kTetB * v[j].x;
      y += kTetB * v[j].y;
      z += kTetB * v[j].z;
    }
    r.vol.push_back({x, y, z, vol / 4.0});
  }
}

void add_tri(CutRule& r, P3 a, P3 b, P3 c, P3 n) {
  const P3 cr = cross(sub(b, a), sub(c, a));
  const double area = std::sqrt(dot3(cr, cr)) / 2.0;
  if (area < kDrop) {
    ++r.dropped;
    return;
  }
  const P3 v[3] = {a, b, c};
  for (int i = 0; i < 3; ++i) {
    const P3& p = v[i];
    const P3& q = v[(i + 1) % 3];
    const P3& s = v[(i + 2) % 3];
    const double x = (2.0 / 3.0) * p.x + (1.0 / 6.0) * q.x + (1.0 / 6.0) * s.x;
    const double y = (2.0 / 3.0) * p.y + (1.0 / 6.0) * q.y + (1.0 / 6.0) * s.y;
    const double z = (2.0 / 3.0) * p.z + (1.0 / 6.0) * q.z + (1.0 / 6.0) * s.z;
    r.surf.push_back({x, y, z, area / 3.0, n.x, n.y, n.z});
  }
}

void add_prism(CutRule& r, P3 A, P3 B, P3 C, P3 A2, P3 B2, P3 C2) {
  add_tet(r, A, B, C, A2);
  add_tet(r, B, C, A2, B2);
  add_tet(r, C, A2, B2, C2);
}

}  // namespace

CutRule cut_quadrature_ref(const double phiv[8]) {
  static const int perms[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
  CutRule rule;
  for (int t = 0; t < 6; ++t) {
    const int a = perms[t][0], b = perms[t][1];
    const int vid[4] = {0, 1 << a, (1 << a) | (1 << b), 7};
    P3 P[4];
    double q[4];
    for (int i = 0; i < 4; ++i) {
      P[i] = {(double)(vid[i] & 1), (double)((vid[i] >> 1) & 1), (double)((vid[i] >> 2) & 1)};
      q[i] = phiv[vid[i]];
    }
    // gradient of the linear interpolant: edges of the Kuhn path are e_a, e_b, e_c.
    double g[3];
    const int c = perms[t][2];
    g[a] = q[1] - q[0];
    g[b] = q[2] - q[1];
    g[c] = q[3] - q[2];
    const double gn = std::sqrt(g[0] * g[0] + g[1] * g[1] + g[2] * g[2]);
    const P3 nrm = gn > 0 ? P3{g[0] / gn, g[1] / gn, g[2] / gn} : P3{0, 0, 0};
    int neg[4], pos[4], nn = 0, np = 0;
    for (int i = 0; i < 4; ++i) {
      if (q[i] < 0)
        neg[nn++] = i;
      else
        pos[np++] = i;
    }
    if (nn == 4) {
      add_tet(rule, P[0], P[1], P[2], P[3]);
    } else if (nn == 1) {
      const int ia = neg[0], ib = pos[0], ic = pos[1], id = pos[2];
      const P3 xab = lerp_edge(P[ia], P[ib], q[ia], q[ib]);
      const P3 xac = lerp_edge(P[ia], P[ic], q[ia], q[ic]);
      const P3 xad = lerp_edge(P[ia], P[id], q[ia], q[id]);
      add_tet(rule, P[ia], xab, xac, xad);
      add_tri(rule, xab, xac, xad, nrm);
    } else if (nn == 3) {
      const int ia = neg[0], ib = neg[1], ic = neg[2], id = pos[0];
      const P3 xad = lerp_edge(P[ia], P[id], q[ia], q[id]);
      const P3 xbd = lerp_edge(P[ib], P[id], q[ib], q[id]);
      const P3 xcd = lerp_edge(P[ic], P[id], q[ic], q[id]);
      add_prism(rule, P[ia], P[ib], P[ic], xad, xbd, xcd);
      add_tri(rule, xad, xbd, xcd, nrm);
    } else if (nn == 2) {
      const int ia = neg[0], ib = neg[1], ic = pos[0], id = pos[1];
      const P3 xac = lerp_edge(P[ia], P[ic], q[ia], q[ic]);
      const P3 xad = lerp_edge(P[ia], P[id], q[ia], q[id]);
      const P3 xbc = lerp_edge(P[ib], P[ic], q[ib], q[ic]);
      const P3 xbd = lerp_edge(P[ib], P[id], q[ib], q[id]);
      add_prism(rule, P[ia], xac, xad, P[ib], xbc, xbd);
      add_tri(rule, xac, xad, xbd, nrm);
      add_tri(rule, xac, xbd, xbc, nrm);
    }
  }
  return rule;
}

// 2x2x2 tensor Gauss rule (order 2) on the unit cell.
CutRule full_quadrature_ref() {
  CutRule r;
  const double g0 = 0.5 - 0.5 / std::sqrt(3.0), g1 = 0.5 + 0.5 / std::sqrt(3.0);
  const double gp[2] = {g0, g1};
  for (int l = 0; l < 8; ++l) r.vol.push_back({gp[l & 1], gp[(l >> 1) & 1], gp[(l >> 2) & 1], 0.125});
  return r;
}

}  // namespace oracle
