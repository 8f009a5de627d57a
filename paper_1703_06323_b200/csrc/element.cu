// element.cu — cut-cell quadrature, beta_e and Nitsche element matrices (K2).
//
// One thread per cut cell. The cut rule depends only on the 8 snapped vertex
// phi values cached by the classification (mesh.hpp:26-29),
// so no level-set callback is needed. Pinned rule (SPEC.md:150-158,
// :172-175): Kuhn 6-tet split along v0-v7, linear-interpolant cut
// per tet, 4-point degree-2 tet rule, 3-point degree-2 triangle rule, pieces
// below 1e-14 |e| dropped; beta_e = 2 lambda_max of the deflated pencil
// (linalg.cpp:108-136) by cyclic Jacobi; K_e = D_e + beta M_e - N_e - N_e^T
// (PAPER.md:315), f = 1, g = 0. A cut cell whose retained volume rule is
// empty contributes nothing.
// Compiled with -fmad=false: identical op order to the CPU restatement.
#include <cub/cub.cuh>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "handle.cuh"
#include "mms.cuh"

#ifndef CB_HD
#define CB_HD __host__ __device__
#endif

namespace cutbddc_b200 {
namespace {

struct P3 {
  double x, y, z;
};
CB_HD inline P3 sub(P3 a, P3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
CB_HD inline P3 cross(P3 a, P3 b) { return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x}; }
CB_HD inline double dot3(P3 a, P3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
CB_HD inline P3 lerp_edge(P3 pu, P3 pv, double qu, double qv) {
  const double t = qu / (qu - qv);
  return {pu.x + t * (pv.x - pu.x), pu.y + t * (pv.y - pu.y), pu.z + t * (pv.z - pu.z)};
}

constexpr double kTetA = 0.5854101966249685;
constexpr double kTetB = 0.1381966011250105;
constexpr double kDrop = 1e-14;

struct Acc {
  double dr[64], br[64], mr[64], nr[64], fr[8];
  int nvol, nsurf;
};

CB_HD inline void q1_eval(double x, double y, double z, double val[8], double grad[8][3]) {
  const double xi[3] = {x, y, z};
#pragma unroll
  for (int l = 0; l < 8; ++l) {
    double f[3], df[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      const bool bit = (l >> d) & 1;
      f[d] = bit ? xi[d] : 1.0 - xi[d];
      df[d] = bit ? 1.0 : -1.0;
    }
    val[l] = f[0] * f[1] * f[2];
    grad[l][0] = df[0] * f[1] * f[2];
    grad[l][1] = f[0] * df[1] * f[2];
    grad[l][2] = f[0] * f[1] * df[2];
  }
}

CB_HD void vol_point(Acc& a, double x, double y, double z, double w) {
  double val[8], grad[8][3];
  q1_eval(x, y, z, val, grad);
  for (int i = 0; i < 8; ++i) {
    a.fr[i] += w * val[i];
    for (int j = 0; j < 8; ++j)
      a.dr[i * 8 + j] += w * (grad[i][0] * grad[j][0] + grad[i][1] * grad[j][1] + grad[i][2] * grad[j][2]);
  }
  a.nvol++;
}

CB_HD void surf_point(Acc& a, double x, double y, double z, double w, P3 n) {
  double val[8], grad[8][3], gn[8];
  q1_eval(x, y, z, val, grad);
  for (int i = 0; i < 8; ++i) gn[i] = n.x * grad[i][0] + n.y * grad[i][1] + n.z * grad[i][2];
  for (int i = 0; i < 8; ++i)
    for (int j = 0; j < 8; ++j) {
      a.br[i * 8 + j] += w * (gn[i] * gn[j]);
      a.mr[i * 8 + j] += w * (val[i] * val[j]);
      a.nr[i * 8 + j] += w * (val[j] * gn[i]);
    }
  a.nsurf++;
}

CB_HD void add_tet(Acc& a, P3 p0, P3 p1, P3 p2, P3 p3) {
  const double vol = fabs(dot3(sub(p1, p0), cross(sub(p2, p0), sub(p3, p0)))) / 6.0;
  if (vol < kDrop) return;
  const P3 v[4] = {p0, p1, p2, p3};
  for (int i = 0; i < 4; ++i) {
    double x = kTetA * v[i].x, y = kTetA * v[i].y, z = kTetA * v[i].z;
    for (int j = 0; j < 4; ++j) {
      if (j == i) continue;
      x += kTetB * v[j].x;
      y += kTetB * v[j].y;
      z += kTetB * v[j].z;
    }
    vol_point(a, x, y, z, vol / 4.0);
  }
}

CB_HD void add_tri(Acc& a, P3 p0, P3 p1, P3 p2, P3 n) {
  const P3 cr = cross(sub(p1, p0), sub(p2, p0));
  const double area = sqrt(dot3(cr, cr)) / 2.0;
  if (area < kDrop) return;
  const P3 v[3] = {p0, p1, p2};
  for (int i = 0; i < 3; ++i) {
    const P3 p = v[i], q = v[(i + 1) % 3], s = v[(i + 2) % 3];
    const double x = (2.0 / 3.0) * p.x + (1.0 / 6.0) * q.x + (1.0 / 6.0) * s.x;
    const double y = (2.0 / 3.0) * p.y + (1.0 / 6.0) * q.y + (1.0 / 6.0) * s.y;
    const double z = (2.0 / 3.0) * p.z + (1.0 / 6.0) * q.z + (1.0 / 6.0) * s.z;
    surf_point(a, x, y, z, area / 3.0, n);
  }
}

CB_HD inline void add_prism(Acc& a, P3 A, P3 B, P3 C, P3 A2, P3 B2, P3 C2) {
  add_tet(a, A, B, C, A2);
  add_tet(a, B, C, A2, B2);
  add_tet(a, C, A2, B2, C2);
}

// Jacobi rotation (c, s) from h = a_qq - a_pp, g = 2 a_pq (oracle/element.cpp
// jacobi_rotation, the same operations).
CB_HD inline void jacobi_rotation(double h, double g, double& c, double& s) {
  const double sgn = (h == 0.0 || (h > 0.0) == (g > 0.0)) ? 1.0 : -1.0;
  const double rho = sqrt(h * h + g * g);
  const double d = fabs(h) + rho;
  const double w = sqrt(d * d + g * g);
  if (w > 0.0 && w <= 1.7976931348623157e308) {
    c = d / w;
    s = sgn * fabs(g) / w;
    return;
  }
  const double theta = h / g;
  const double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
  c = 1.0 / sqrt(t * t + 1.0);
  s = t * c;
}

// Parallel-order cyclic Jacobi (n <= 8): round-robin rounds of four disjoint
// pairs, per round A <- A J, A <- J^T A, V <- V J with the rotations taken
// from the matrix at the start of the round; same order / thresholds as the
// CPU restatement (oracle/element.cpp jacobi_eigs).
CB_HD void jacobi(int n, double* a, double* v, double* ev) {
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) v[i * n + j] = i == j ? 1.0 : 0.0;
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0, diag = 0.0;
    for (int i = 0; i < n; ++i) {
      diag += a[i * n + i] * a[i * n + i];
      for (int j = i + 1; j < n; ++j) off += a[i * n + j] * a[i * n + j];
    }
    if (off <= 1e-32 * diag || off < 1e-300) break;
    for (int r = 0; r < 7; ++r) {
      int P[4], Q[4];
      double C[4], S[4];
      bool act[4];
      for (int k = 0; k < 4; ++k) {
        const int x = k == 0 ? 7 : (r + k) % 7;
        const int y = k == 0 ? r : (r - k + 7) % 7;
        P[k] = x < y ? x : y;
        Q[k] = x < y ? y : x;
        act[k] = Q[k] < n && a[P[k] * n + Q[k]] != 0.0;
        C[k] = 1.0;
        S[k] = 0.0;
        if (act[k])
          jacobi_rotation(a[Q[k] * n + Q[k]] - a[P[k] * n + P[k]], 2.0 * a[P[k] * n + Q[k]], C[k], S[k]);
      }
      for (int k = 0; k < 4; ++k) {
        if (!act[k]) continue;
        const int p = P[k], q = Q[k];
        const double c = C[k], s = S[k];
        for (int i = 0; i < n; ++i) {
          const double aip = a[i * n + p], aiq = a[i * n + q];
          a[i * n + p] = c * aip - s * aiq;
          a[i * n + q] = s * aip + c * aiq;
          const double vip = v[i * n + p], viq = v[i * n + q];
          v[i * n + p] = c * vip - s * viq;
          v[i * n + q] = s * vip + c * viq;
        }
      }
      for (int k = 0; k < 4; ++k) {
        if (!act[k]) continue;
        const int p = P[k], q = Q[k];
        const double c = C[k], s = S[k];
        for (int j = 0; j < n; ++j) {
          const double apj = a[p * n + j], aqj = a[q * n + j];
          a[p * n + j] = c * apj - s * aqj;
          a[q * n + j] = s * apj + c * aqj;
        }
      }
      for (int k = 0; k < 4; ++k)
        if (act[k]) a[P[k] * n + Q[k]] = a[Q[k] * n + P[k]] = 0.0;
    }
  }
  for (int i = 0; i < n; ++i) ev[i] = a[i * n + i];
}

// dense_generalized_eigs_max (linalg.cpp:108-136), kernel_tol 1e-12. Returns
// -1 for a degenerate pencil (lambda_max(D) <= 0).
CB_HD double gen_eigs_max(const double* b, const double* d) {
  double a[64], v[64], ev[8];
  for (int i = 0; i < 64; ++i) a[i] = d[i];
  jacobi(8, a, v, ev);
  double lmax = ev[0];
  for (int i = 1; i < 8; ++i) lmax = fmax(lmax, ev[i]);
  if (!(lmax > 0.0)) return -1.0;
  int keep[8], m = 0;
  for (int k = 0; k < 8; ++k)
    if (ev[k] >= 1e-12 * lmax) keep[m++] = k;
  double bq[64];
  for (int i = 0; i < 8; ++i)
    for (int k = 0; k < m; ++k) {
      double s = 0;
      for (int j = 0; j < 8; ++j) s += b[i * 8 + j] * v[j * 8 + keep[k]];
      bq[i * m + k] = s;
    }
  double c[64], cv[64], cev[8];
  for (int k = 0; k < m; ++k)
    for (int l = 0; l < m; ++l) {
      double s = 0;
      for (int i = 0; i < 8; ++i) s += v[i * 8 + keep[k]] * bq[i * m + l];
      c[k * m + l] = s / (sqrt(ev[keep[k]]) * sqrt(ev[keep[l]]));
    }
  for (int k = 0; k < m; ++k)
    for (int l = k + 1; l < m; ++l) {
      const double s = 0.5 * (c[k * m + l] + c[l * m + k]);
      c[k * m + l] = s;
      c[l * m + k] = s;
    }
  jacobi(m, c, cv, cev);
  double best = cev[0];
  for (int k = 1; k < m; ++k) best = fmax(best, cev[k]);
  return best;
}

// One cut cell from its 8 vertex phi values. Returns 1 for a degenerate
// pencil (D numerically zero), else 0.
CB_HD int cut_element(const double q8[8], double h, double* K, double* F, double* beta_out, uint8_t* empty_out) {
  Acc a;
  for (int t = 0; t < 64; ++t) a.dr[t] = a.br[t] = a.mr[t] = a.nr[t] = 0.0;
  for (int t = 0; t < 8; ++t) a.fr[t] = 0.0;
  a.nvol = a.nsurf = 0;
  // Fully unrolled so every vertex index is a compile-time constant (no
  // dynamically indexed local arrays on the device).
#pragma unroll
  for (int t = 0; t < 6; ++t) {
    const int pa = t < 2 ? 0 : (t < 4 ? 1 : 2);
    const int pb = (t == 0 || t == 5) ? 1 : ((t == 1 || t == 3) ? 2 : 0);
    const int pc = 3 - pa - pb;
    const int vid[4] = {0, 1 << pa, (1 << pa) | (1 << pb), 7};
    P3 P[4];
    double q[4];
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      P[v] = {(double)(vid[v] & 1), (double)((vid[v] >> 1) & 1), (double)((vid[v] >> 2) & 1)};
      q[v] = q8[vid[v]];
    }
    double g[3];
    g[pa] = q[1] - q[0];
    g[pb] = q[2] - q[1];
    g[pc] = q[3] - q[2];
    const double gn = sqrt(g[0] * g[0] + g[1] * g[1] + g[2] * g[2]);
    const P3 nrm = gn > 0 ? P3{g[0] / gn, g[1] / gn, g[2] / gn} : P3{0, 0, 0};
    int neg[4], pos[4], nn = 0, np = 0;
    for (int v = 0; v < 4; ++v) {
      if (q[v] < 0)
        neg[nn++] = v;
      else
        pos[np++] = v;
    }
    if (nn == 4) {
      add_tet(a, P[0], P[1], P[2], P[3]);
    } else if (nn == 1) {
      const int ia = neg[0], ib = pos[0], ic = pos[1], id = pos[2];
      const P3 xab = lerp_edge(P[ia], P[ib], q[ia], q[ib]);
      const P3 xac = lerp_edge(P[ia], P[ic], q[ia], q[ic]);
      const P3 xad = lerp_edge(P[ia], P[id], q[ia], q[id]);
      add_tet(a, P[ia], xab, xac, xad);
      add_tri(a, xab, xac, xad, nrm);
    } else if (nn == 3) {
      const int ia = neg[0], ib = neg[1], ic = neg[2], id = pos[0];
      const P3 xad = lerp_edge(P[ia], P[id], q[ia], q[id]);
      const P3 xbd = lerp_edge(P[ib], P[id], q[ib], q[id]);
      const P3 xcd = lerp_edge(P[ic], P[id], q[ic], q[id]);
      add_prism(a, P[ia], P[ib], P[ic], xad, xbd, xcd);
      add_tri(a, xad, xbd, xcd, nrm);
    } else if (nn == 2) {
      const int ia = neg[0], ib = neg[1], ic = pos[0], id = pos[1];
      const P3 xac = lerp_edge(P[ia], P[ic], q[ia], q[ic]);
      const P3 xad = lerp_edge(P[ia], P[id], q[ia], q[id]);
      const P3 xbc = lerp_edge(P[ib], P[ic], q[ib], q[ic]);
      const P3 xbd = lerp_edge(P[ib], P[id], q[ib], q[id]);
      add_prism(a, P[ia], xac, xad, P[ib], xbc, xbd);
      add_tri(a, xac, xad, xbd, nrm);
      add_tri(a, xac, xbd, xbc, nrm);
    }
  }
  if (a.nvol == 0) {
    for (int t = 0; t < 64; ++t) K[t] = 0.0;
    for (int t = 0; t < 8; ++t) F[t] = 0.0;
    *beta_out = 0.0;
    *empty_out = 1;
    return 0;
  }
  double lambda = 0.0;
  int degenerate = 0;
  if (a.nsurf > 0) {
    lambda = gen_eigs_max(a.br, a.dr);
    if (lambda < 0) {
      degenerate = 1;
      lambda = 0.0;
    }
  }
  const double betar = 2.0 * lambda;
  for (int x = 0; x < 8; ++x)
    for (int y = 0; y < 8; ++y) K[x * 8 + y] = h * (a.dr[x * 8 + y] + betar * a.mr[x * 8 + y] - (a.nr[x * 8 + y] + a.nr[y * 8 + x]));
  for (int x = 0; x < 8; ++x) F[x] = h * h * h * a.fr[x];
  *beta_out = betar / h;
  *empty_out = 0;
  return degenerate;
}

// ---------------------------------------------------------------------------
// Two-kernel form of cut_element (same arithmetic, bit for bit).
//
// k_cut_acc, one warp per cut cell: lanes 0-5 cut one Kuhn tet each and
// write its quadrature points to shared memory; then every accumulator of
// the sequential code (D, F, B, M, N: 180 unique entries) is owned by one
// lane, which sums it over the points in the sequential order (tet, piece,
// point), so every sum sees the same operands in the same order. The Q1
// factors are rebuilt per point from f_d in {x_d, 1 - x_d}: grad[l][0] =
// (+-1 * f1) * f2 = +-(f1 f2) exactly, so no product differs from q1_eval.
// The 180 sums go to global memory.
//
// k_cut_pencil, eight lanes per cell: beta_e from the deflated pencil
// (gen_eigs_max) with the 8x8 matrices held in registers, lane k owning row
// k (Jacobi rotations exchange rows by shuffles: no shared memory, so many
// cells are in flight), then K_e and F_e.
constexpr int kVolPts = 12;   // per tet: up to three sub-tets x 4 points
constexpr int kSurfPts = 6;   // per tet: up to two triangles x 3 points
constexpr int kAccCells = 4;  // cells (warps) per CTA of k_cut_acc
constexpr int kAcc = 196;     // accumulators per cell: 0-35 D (i <= j), 36-43 F, 44-79 B, 80-115 M (i <= j), 116-179 N,
                              // manufactured problem only: 180-187 G1 = sum g phi_a, 188-195 G2 = sum g n.grad phi_a
constexpr int kAccBase = 180; // the accumulators of every problem

struct PointSmem {
  double vp[6][kVolPts][4];
  double sp[6][kSurfPts][7];
  int nv[6], ns[6];
};

struct PtList {
  double (*vp)[4];
  double (*sp)[7];
  int nv, ns;
};

__device__ void pl_tet(PtList& L, P3 p0, P3 p1, P3 p2, P3 p3) {
  const double vol = fabs(dot3(sub(p1, p0), cross(sub(p2, p0), sub(p3, p0)))) / 6.0;
  if (vol < kDrop) return;
  const P3 v[4] = {p0, p1, p2, p3};
  for (int i = 0; i < 4; ++i) {
    double x = kTetA * v[i].x, y = kTetA * v[i].y, z = kTetA * v[i].z;
    for (int j = 0; j < 4; ++j) {
      if (j == i) continue;
      x += kTetB * v[j].x;
      y += kTetB * v[j].y;
      z += kTetB * v[j].z;
    }
    double* o = L.vp[L.nv++];
    o[0] = x;
    o[1] = y;
    o[2] = z;
    o[3] = vol / 4.0;
  }
}

__device__ void pl_tri(PtList& L, P3 p0, P3 p1, P3 p2, P3 n) {
  const P3 cr = cross(sub(p1, p0), sub(p2, p0));
  const double area = sqrt(dot3(cr, cr)) / 2.0;
  if (area < kDrop) return;
  const P3 v[3] = {p0, p1, p2};
  for (int i = 0; i < 3; ++i) {
    const P3 p = v[i], q = v[(i + 1) % 3], s = v[(i + 2) % 3];
    double* o = L.sp[L.ns++];
    o[0] = (2.0 / 3.0) * p.x + (1.0 / 6.0) * q.x + (1.0 / 6.0) * s.x;
    o[1] = (2.0 / 3.0) * p.y + (1.0 / 6.0) * q.y + (1.0 / 6.0) * s.y;
    o[2] = (2.0 / 3.0) * p.z + (1.0 / 6.0) * q.z + (1.0 / 6.0) * s.z;
    o[3] = area / 3.0;
    o[4] = n.x;
    o[5] = n.y;
    o[6] = n.z;
  }
}

// the points of Kuhn tet t (the body of cut_element's tet loop)
__device__ void tet_points(int t, const double* q8, PtList& L) {
  const int pa = t < 2 ? 0 : (t < 4 ? 1 : 2);
  const int pb = (t == 0 || t == 5) ? 1 : ((t == 1 || t == 3) ? 2 : 0);
  const int pc = 3 - pa - pb;
  const int vid[4] = {0, 1 << pa, (1 << pa) | (1 << pb), 7};
  P3 P[4];
  double q[4];
  for (int v = 0; v < 4; ++v) {
    P[v] = {(double)(vid[v] & 1), (double)((vid[v] >> 1) & 1), (double)((vid[v] >> 2) & 1)};
    q[v] = q8[vid[v]];
  }
  double g[3];
  g[pa] = q[1] - q[0];
  g[pb] = q[2] - q[1];
  g[pc] = q[3] - q[2];
  const double gn = sqrt(g[0] * g[0] + g[1] * g[1] + g[2] * g[2]);
  const P3 nrm = gn > 0 ? P3{g[0] / gn, g[1] / gn, g[2] / gn} : P3{0, 0, 0};
  int neg[4], pos[4], nn = 0, np = 0;
  for (int v = 0; v < 4; ++v) {
    if (q[v] < 0)
      neg[nn++] = v;
    else
      pos[np++] = v;
  }
  if (nn == 4) {
    pl_tet(L, P[0], P[1], P[2], P[3]);
  } else if (nn == 1) {
    const int ia = neg[0], ib = pos[0], ic = pos[1], id = pos[2];
    const P3 xab = lerp_edge(P[ia], P[ib], q[ia], q[ib]);
    const P3 xac = lerp_edge(P[ia], P[ic], q[ia], q[ic]);
    const P3 xad = lerp_edge(P[ia], P[id], q[ia], q[id]);
    pl_tet(L, P[ia], xab, xac, xad);
    pl_tri(L, xab, xac, xad, nrm);
  } else if (nn == 3) {
    const int ia = neg[0], ib = neg[1], ic = neg[2], id = pos[0];
    const P3 xad = lerp_edge(P[ia], P[id], q[ia], q[id]);
    const P3 xbd = lerp_edge(P[ib], P[id], q[ib], q[id]);
    const P3 xcd = lerp_edge(P[ic], P[id], q[ic], q[id]);
    pl_tet(L, P[ia], P[ib], P[ic], xad);
    pl_tet(L, P[ib], P[ic], xad, xbd);
    pl_tet(L, P[ic], xad, xbd, xcd);
    pl_tri(L, xad, xbd, xcd, nrm);
  } else if (nn == 2) {
    const int ia = neg[0], ib = neg[1], ic = pos[0], id = pos[1];
    const P3 xac = lerp_edge(P[ia], P[ic], q[ia], q[ic]);
    const P3 xad = lerp_edge(P[ia], P[id], q[ia], q[id]);
    const P3 xbc = lerp_edge(P[ib], P[ic], q[ib], q[ic]);
    const P3 xbd = lerp_edge(P[ib], P[id], q[ib], q[id]);
    pl_tet(L, P[ia], xac, xad, P[ib]);
    pl_tet(L, xac, xad, P[ib], xbc);
    pl_tet(L, xad, P[ib], xbc, xbd);
    pl_tri(L, xac, xad, xbd, nrm);
    pl_tri(L, xac, xbd, xbc, nrm);
  }
}

// q1_eval's grad[l][0..2] at x (exact same values, see above): f_d = bit_d(l)
// ? x_d : 1 - x_d, grad = (+-f1 f2, +-f0 f2, +-f0 f1), val = (f0 f1) f2
__device__ __forceinline__ void q1_gv(const double* x, int l, double g[3], double* val) {
  const bool b0 = l & 1, b1 = (l >> 1) & 1, b2 = (l >> 2) & 1;
  const double f0 = b0 ? x[0] : 1.0 - x[0];
  const double f1 = b1 ? x[1] : 1.0 - x[1];
  const double f2 = b2 ? x[2] : 1.0 - x[2];
  const double g0 = f1 * f2, g1 = f0 * f2, f01 = f0 * f1;
  g[0] = b0 ? g0 : -g0;
  g[1] = b1 ? g1 : -g1;
  g[2] = b2 ? f01 : -f01;
  if (val) *val = f01 * f2;
}

// accumulator `it` -> (kind, i, j): 0 D, 1 F, 2 B, 3 M, 4 N
__device__ __forceinline__ void acc_index(int it, int& kind, int& i, int& j) {
  if (it < 36 || (it >= 44 && it < 116)) {
    int u = it < 36 ? it : (it - 44) % 36;
    kind = it < 36 ? 0 : (it < 80 ? 2 : 3);
    i = 0;
    while (u >= 8 - i) {
      u -= 8 - i;
      ++i;
    }
    j = i + u;
  } else if (it < 44) {
    kind = 1;
    i = it - 36;
    j = i;
  } else {
    kind = 4;
    i = (it - 116) / 8;
    j = (it - 116) % 8;
  }
}

// Problem data of the load vector: f = 1, g = 0, or the manufactured u
// evaluated at the physical point origin + (cell + xi) h (mms.cuh).
struct LoadArgs {
  int problem, n;
  const int64_t* cells;  // cut cell ids
  double ox, oy, oz, h;
};

// Per-warp staging of one batch of kBatch quadrature points: the Q1 factors
// of every (point, node) pair are evaluated once by the warp and shared by
// the accumulators (they were rebuilt per accumulator before: ~3x the FP64
// instructions). Node stride 5 doubles: the eight nodes fall in distinct
// shared-memory banks.
constexpr int kBatch = 8;
struct BatchSmem {
  double gv[kBatch][8][5];  // volume points: grad (3), val; surface points: n.grad, val
  double px[kBatch];        // weight of the point
  double pf[kBatch];        // manufactured problem: f (volume) or g (surface) at the point
  unsigned char vmap[6 * kVolPts], smap[6 * kSurfPts];  // flat point order -> (tet, point)
};

#ifndef CB_ACC_MINB
#define CB_ACC_MINB 6
#endif
__global__ void __launch_bounds__(32 * kAccCells, CB_ACC_MINB) k_cut_acc(int64_t ncut, const double* __restrict__ q8all,
                                                             double* __restrict__ accs, int* __restrict__ nvs,
                                                             LoadArgs la) {
  __shared__ PointSmem smem[kAccCells];
  __shared__ BatchSmem bsm[kAccCells];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t e = (int64_t)blockIdx.x * kAccCells + wid;
  if (e >= ncut) return;
  PointSmem& S = smem[wid];
  BatchSmem& Bt = bsm[wid];
  int mynv = 0, myns = 0;
  if (lane < 6) {
    PtList L{S.vp[lane], S.sp[lane], 0, 0};
    double q[8];
    for (int i = 0; i < 8; ++i) q[i] = q8all[e * 8 + i];
    tet_points(lane, q, L);
    S.nv[lane] = mynv = L.nv;
    S.ns[lane] = myns = L.ns;
  }
  // flat point order (tet, then point): offsets by a warp prefix sum
  int voff = mynv, soff = myns;
#pragma unroll
  for (int d = 1; d < 8; d <<= 1) {
    const int a = __shfl_up_sync(0xffffffffu, voff, d), b2 = __shfl_up_sync(0xffffffffu, soff, d);
    if (lane >= d) voff += a, soff += b2;
  }
  const int nvol = __shfl_sync(0xffffffffu, voff, 5), nsurf = __shfl_sync(0xffffffffu, soff, 5);
  if (lane < 6) {
    for (int k = 0; k < mynv; ++k) Bt.vmap[voff - mynv + k] = (unsigned char)(lane * kVolPts + k);
    for (int k = 0; k < myns; ++k) Bt.smap[soff - myns + k] = (unsigned char)(lane * kSurfPts + k);
  }
  __syncwarp();
  if (lane == 0) {
    nvs[2 * e] = nvol;
    nvs[2 * e + 1] = nsurf;
  }
  if (nvol == 0) return;
  const bool mms = la.problem == kProblemManufactured;
  double cx = 0, cy = 0, cz = 0;  // the cell's lattice coordinates
  if (mms) {
    const int64_t cell = la.cells[e], n = la.n;
    cz = (double)(cell % n);
    cy = (double)((cell / n) % n);
    cx = (double)(cell / n / n);
  }
  const int spt = lane >> 2, sn0 = (lane & 3) * 2;  // staging: this lane's point of the batch and its two nodes

  // ---- volume accumulators: 0-35 D (i <= j), 36-43 F
  {
    int kind[2], ai[2], aj[2];
    double acc[2] = {0.0, 0.0};
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int it = lane + 32 * k;
      kind[k] = -1;
      ai[k] = aj[k] = 0;
      if (it < 44) acc_index(it, kind[k], ai[k], aj[k]);
    }
    const double* vp = &S.vp[0][0][0];
    for (int p0 = 0; p0 < nvol; p0 += kBatch) {
      const int cnt = min(kBatch, nvol - p0);
      if (spt < cnt) {
        const double* P = vp + 4 * Bt.vmap[p0 + spt];
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          double g[3], val;
          q1_gv(P, sn0 + q, g, &val);
          Bt.gv[spt][sn0 + q][0] = g[0];
          Bt.gv[spt][sn0 + q][1] = g[1];
          Bt.gv[spt][sn0 + q][2] = g[2];
          Bt.gv[spt][sn0 + q][3] = val;
        }
        if (sn0 == 0) {
          Bt.px[spt] = P[3];
          if (mms) Bt.pf[spt] = mms_f(la.ox + (cx + P[0]) * la.h, la.oy + (cy + P[1]) * la.h, la.oz + (cz + P[2]) * la.h);
        }
      }
      __syncwarp();
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        if (kind[k] == 0) {
          for (int pp = 0; pp < cnt; ++pp) {
            const double* gi = Bt.gv[pp][ai[k]];
            const double* gj = Bt.gv[pp][aj[k]];
            acc[k] += Bt.px[pp] * (gi[0] * gj[0] + gi[1] * gj[1] + gi[2] * gj[2]);
          }
        } else if (kind[k] == 1) {
          for (int pp = 0; pp < cnt; ++pp) {
            const double vi = Bt.gv[pp][ai[k]][3];
            if (mms)
              acc[k] += Bt.px[pp] * (Bt.pf[pp] * vi);
            else
              acc[k] += Bt.px[pp] * vi;
          }
        }
      }
      __syncwarp();
    }
#pragma unroll
    for (int k = 0; k < 2; ++k)
      if (kind[k] >= 0) accs[e * kAcc + lane + 32 * k] = acc[k];
  }

  // ---- surface accumulators: 44-79 B (i <= j), 80-115 M (i <= j), 116-179 N; manufactured: 180-187 G1, 188-195 G2
  {
    constexpr int kS = 5;  // (196 - 44) / 32 rounded up
    const int nacc = (mms ? kAcc : kAccBase) - 44;
    int kind[kS], ai[kS], aj[kS];
    double acc[kS];
#pragma unroll
    for (int k = 0; k < kS; ++k) {
      const int it = 44 + lane + 32 * k;
      kind[k] = -1;
      ai[k] = aj[k] = 0;
      acc[k] = 0.0;
      if (lane + 32 * k < nacc) {
        if (it >= kAccBase) {
          kind[k] = it >= kAccBase + 8 ? 6 : 5;  // G2 / G1
          ai[k] = (it - kAccBase) & 7;
        } else {
          acc_index(it, kind[k], ai[k], aj[k]);
        }
      }
    }
    const double* sp = &S.sp[0][0][0];
    for (int p0 = 0; p0 < nsurf; p0 += kBatch) {
      const int cnt = min(kBatch, nsurf - p0);
      if (spt < cnt) {
        const double* P = sp + 7 * Bt.smap[p0 + spt];
        const double nx = P[4], ny = P[5], nz = P[6];
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          double g[3], val;
          q1_gv(P, sn0 + q, g, &val);
          Bt.gv[spt][sn0 + q][0] = nx * g[0] + ny * g[1] + nz * g[2];
          Bt.gv[spt][sn0 + q][1] = val;
        }
        if (sn0 == 0) {
          Bt.px[spt] = P[3];
          if (mms) Bt.pf[spt] = mms_u(la.ox + (cx + P[0]) * la.h, la.oy + (cy + P[1]) * la.h, la.oz + (cz + P[2]) * la.h);
        }
      }
      __syncwarp();
#pragma unroll
      for (int k = 0; k < kS; ++k) {
        if (kind[k] < 0) continue;
        for (int pp = 0; pp < cnt; ++pp) {
          const double w = Bt.px[pp];
          const double ni = Bt.gv[pp][ai[k]][0], vi = Bt.gv[pp][ai[k]][1];
          const double nj = Bt.gv[pp][aj[k]][0], vj = Bt.gv[pp][aj[k]][1];
          if (kind[k] == 2)
            acc[k] += w * (ni * nj);
          else if (kind[k] == 3)
            acc[k] += w * (vi * vj);
          else if (kind[k] == 4)
            acc[k] += w * (vj * ni);
          else if (kind[k] == 5)
            acc[k] += w * (Bt.pf[pp] * vi);
          else
            acc[k] += w * (Bt.pf[pp] * ni);
        }
      }
      __syncwarp();
    }
#pragma unroll
    for (int k = 0; k < kS; ++k)
      if (kind[k] >= 0) accs[e * kAcc + 44 + lane + 32 * k] = acc[k];
  }
}

__device__ __forceinline__ double gsh(double v, int src, unsigned gm) { return __shfl_sync(gm, v, src, 8); }
// r[idx] with a runtime idx (no local-memory array)
__device__ __forceinline__ double sel8(const double (&r)[8], int idx) {
  double x = r[0];
#pragma unroll
  for (int j = 1; j < 8; ++j) x = idx == j ? r[j] : x;
  return x;
}
// packed-upper index of (i, j), i <= j, in the D / B / M accumulator blocks
__device__ __forceinline__ int tri(int i, int j) { return i * 8 - i * (i - 1) / 2 + (j - i); }

// The round-robin pair (p < q) number k of round r over 8 players (the order
// of jacobi above).
__host__ __device__ constexpr int rr_x(int r, int k) { return k == 0 ? 7 : (r + k) % 7; }
__host__ __device__ constexpr int rr_y(int r, int k) { return k == 0 ? r : (r - k + 7) % 7; }
__host__ __device__ constexpr int rr_p(int r, int k) { return rr_x(r, k) < rr_y(r, k) ? rr_x(r, k) : rr_y(r, k); }
__host__ __device__ constexpr int rr_q(int r, int k) { return rr_x(r, k) < rr_y(r, k) ? rr_y(r, k) : rr_x(r, k); }

// jacobi(n, a, v, ev) by the 8 lanes of a group, lane k holding row k of a
// and of v in registers. Per round: lane l computes the rotation of pair
// l & 3 (the sqrt / div chains of the four pairs run side by side in
// different lanes) and the (c, s) are broadcast; A <- A J and V <- V J are
// lane-local (four disjoint column pairs of the lane's row); A <- J^T A
// exchanges the lane's row with its partner's by one round of shuffles.
// Every entry sees jacobi's operations on the same operands, so the result
// is bit-identical. Rounds and pairs are unrolled: every register index is a
// compile-time constant.
__device__ void reg_jacobi(int n, double (&a)[8], double (&v)[8], int gl, unsigned gm) {
#pragma unroll
  for (int j = 0; j < 8; ++j) v[j] = j == gl ? 1.0 : 0.0;
  const int k4 = gl & 3;
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0, diag = 0.0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const double aii = gsh(a[i], i, gm);
      if (i < n) diag += aii * aii;
#pragma unroll
      for (int j = i + 1; j < 8; ++j) {
        const double aij = gsh(a[j], i, gm);
        if (j < n) off += aij * aij;
      }
    }
    if (off <= 1e-32 * diag || off < 1e-300) break;
#pragma unroll
    for (int r = 0; r < 7; ++r) {
      // the pair whose rotation this lane computes (mp, mq); this lane's own
      // pair number, partner and side
      int mp = rr_p(r, 0), mq = rr_q(r, 0), mate = 0, mypair = 0;
      bool is_p = false;
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        if (k4 == kk) {
          mp = rr_p(r, kk);
          mq = rr_q(r, kk);
        }
        if (gl == rr_p(r, kk)) {
          mate = rr_q(r, kk);
          mypair = kk;
          is_p = true;
        }
        if (gl == rr_q(r, kk)) {
          mate = rr_p(r, kk);
          mypair = kk;
        }
      }
      const double dg = sel8(a, gl);    // A[gl][gl]
      const double om = sel8(a, mate);  // A[gl][mate]
      const double app = gsh(dg, mp, gm), aqq = gsh(dg, mq, gm), apq = gsh(om, mp, gm);
      const bool act = mq < n && apq != 0.0;
      double c = 1.0, s = 0.0;
      if (act) jacobi_rotation(aqq - app, 2.0 * apq, c, s);
      double C[4], S[4];
      bool A[4];
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        C[kk] = gsh(c, kk, gm);
        S[kk] = gsh(s, kk, gm);
        A[kk] = __shfl_sync(gm, (int)act, kk, 8) != 0;
      }
      // A <- A J, V <- V J: this lane's row, four disjoint column pairs
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const int p = rr_p(r, kk), q = rr_q(r, kk);
        if (A[kk] && gl < n) {
          const double aip = a[p], aiq = a[q];
          a[p] = C[kk] * aip - S[kk] * aiq;
          a[q] = S[kk] * aip + C[kk] * aiq;
          const double vip = v[p], viq = v[q];
          v[p] = C[kk] * vip - S[kk] * viq;
          v[q] = S[kk] * vip + C[kk] * viq;
        }
      }
      // A <- J^T A: row p = c row p - s row q, row q = s row p + c row q
      double other[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) other[j] = gsh(a[j], mate, gm);
      bool mine = false;
      double cm = 1.0, sm = 0.0;
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)
        if (mypair == kk) {
          mine = A[kk];
          cm = C[kk];
          sm = S[kk];
        }
      if (mine) {
        if (is_p) {
#pragma unroll
          for (int j = 0; j < 8; ++j)
            if (j < n) a[j] = cm * a[j] - sm * other[j];
        } else {
#pragma unroll
          for (int j = 0; j < 8; ++j)
            if (j < n) a[j] = sm * other[j] + cm * a[j];
        }
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (j == mate) a[j] = 0.0;
      }
    }
  }
}

// gen_eigs_max (linalg.cpp:108-136) by a lane group with register rows: the
// same operations as the sequential function above. d, b: row gl.
__device__ double reg_gen_eigs_max(const double (&d)[8], const double (&b)[8], int gl, unsigned gm) {
  double a[8], v[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = d[j];
  reg_jacobi(8, a, v, gl, gm);
  double ev[8];
  const double evk = sel8(a, gl);
#pragma unroll
  for (int i = 0; i < 8; ++i) ev[i] = gsh(evk, i, gm);
  double lmax = ev[0];
#pragma unroll
  for (int i = 1; i < 8; ++i) lmax = fmax(lmax, ev[i]);
  if (!(lmax > 0.0)) return -1.0;
  int keep[8], m = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k)
    if (ev[k] >= 1e-12 * lmax) keep[m++] = k;
  // bq row gl: bq[gl][k] = sum_j b[gl][j] v[j][keep[k]]
  double bq[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int kk = k < m ? keep[k] : 0;
    const double mine = sel8(v, kk);  // v[gl][keep[k]], sent to every lane below
    double s = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += b[j] * gsh(mine, j, gm);
    bq[k] = s;
  }
  // c row gl (gl < m): c[gl][l] = sum_i v[i][keep[gl]] bq[i][l] / (sqrt(ev[keep[gl]]) sqrt(ev[keep[l]]))
  const int kg = gl < m ? keep[gl] : 0;
  double cs[8];
#pragma unroll
  for (int l = 0; l < 8; ++l) cs[l] = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    double vi[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) vi[j] = gsh(v[j], i, gm);
    const double vik = sel8(vi, kg);
#pragma unroll
    for (int l = 0; l < 8; ++l) cs[l] += vik * gsh(bq[l], i, gm);
  }
  const double ek = sel8(ev, kg);
  double c[8];
#pragma unroll
  for (int l = 0; l < 8; ++l) c[l] = cs[l] / (sqrt(ek) * sqrt(ev[l < m ? keep[l] : 0]));
  // symmetrise: (k, l), k != l: 0.5 (c[min][max] + c[max][min])
  double a2[8];
#pragma unroll
  for (int l = 0; l < 8; ++l) {
    double crow[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) crow[j] = gsh(c[j], l, gm);
    const double clk = sel8(crow, gl);  // c[l][gl]
    a2[l] = l == gl ? c[l] : (gl < l ? 0.5 * (c[l] + clk) : 0.5 * (clk + c[l]));
  }
  double cv[8];
  reg_jacobi(m, a2, cv, gl, gm);
  const double ck = sel8(a2, gl);
  double best = gsh(ck, 0, gm);
#pragma unroll
  for (int k = 1; k < 8; ++k) {
    const double x = gsh(ck, k, gm);
    if (k < m) best = fmax(best, x);
  }
  return best;
}

// eight lanes per cut cell: beta_e, K_e = h (D + beta M - N - N^T), F_e = h^3 F
#ifndef CB_PENCIL_MINB
#define CB_PENCIL_MINB 2  // 128 registers (28 bytes spilled): two CTAs per SM hide the rotation chains (B200: assembly 1.32 -> 1.20 ms)
#endif
#ifndef CB_PENCIL_THREADS
#define CB_PENCIL_THREADS 256
#endif
__global__ void __launch_bounds__(CB_PENCIL_THREADS, CB_PENCIL_MINB) k_cut_pencil(double h, int64_t ncut, int problem, const double* __restrict__ accs,
                                                     const int* __restrict__ nvs, double* __restrict__ ke,
                                                     double* __restrict__ fe, double* __restrict__ beta,
                                                     uint8_t* __restrict__ empty, int* __restrict__ degenerate) {
  const int lane = threadIdx.x & 31, g = lane >> 3, gl = lane & 7;
  const unsigned gm = 0xffu << (8 * g);
  const int64_t e = (int64_t)(blockIdx.x * blockDim.x + threadIdx.x) / 8;
  if (e >= ncut) return;  // whole groups: ncut cells x 8 lanes
  const int nvol = nvs[2 * e], nsurf = nvs[2 * e + 1];
  if (nvol == 0) {
    for (int t = gl; t < 64; t += 8) ke[e * 64 + t] = 0.0;
    fe[e * 8 + gl] = 0.0;
    if (gl == 0) {
      beta[e] = 0.0;
      empty[e] = 1;
    }
    return;
  }
  const double* A = accs + e * kAcc;
  double d[8], b[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int i0 = gl < j ? gl : j, j0 = gl < j ? j : gl;
    d[j] = A[tri(i0, j0)];
    b[j] = A[44 + tri(i0, j0)];
  }
  double lambda = 0.0;
  if (nsurf > 0) {
    lambda = reg_gen_eigs_max(d, b, gl, gm);
    if (lambda < 0) {
      if (gl == 0) atomicExch(degenerate, 1);
      lambda = 0.0;
    }
  }
  const double betar = 2.0 * lambda;
#pragma unroll
  for (int y = 0; y < 8; ++y) {
    const int i0 = gl < y ? gl : y, j0 = gl < y ? y : gl;
    const double mxy = A[80 + tri(i0, j0)];
    ke[e * 64 + gl * 8 + y] = h * (d[y] + betar * mxy - (A[116 + gl * 8 + y] + A[116 + y * 8 + gl]));
  }
  fe[e * 8 + gl] = problem == kProblemManufactured
                      ? h * h * h * A[36 + gl] + h * (betar * A[kAccBase + gl] - A[kAccBase + 8 + gl])
                      : h * h * h * A[36 + gl];
  if (gl == 0) {
    beta[e] = betar / h;
    empty[e] = 0;
  }
}

#ifndef CB_CUT_LB
#define CB_CUT_LB 64
#endif
__global__ void __launch_bounds__(CB_CUT_LB) k_cut_elements(double h, int64_t ncut, const double* __restrict__ q8all,
                                                     double* __restrict__ ke,
                                                     double* __restrict__ fe, double* __restrict__ beta,
                                                     uint8_t* __restrict__ empty, int* __restrict__ degenerate) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= ncut) return;
  // vertex phi gathered by k_gather_q8 into global memory: passing a
  // thread-local array into cut_element produced wrong results on sm_100a
  // (nvcc 12.9, ~5.6 KB stack frame); the global-pointer form is verified
  // bit-exact against the host build of the same function.
  if (cut_element(q8all + e * 8, h, ke + e * 64, fe + e * 8, beta + e, empty + e)) atomicExch(degenerate, 1);
}

__global__ void k_gather_q8(int n, int64_t ncut, const int64_t* __restrict__ cut_cells, const double* __restrict__ phi,
                            double* __restrict__ q8all) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= ncut) return;
  const int64_t cell = cut_cells[e];
  const int k = (int)(cell % n), j = (int)((cell / n) % n), i = (int)(cell / n / n);
#pragma unroll
  for (int l = 0; l < 8; ++l)
    q8all[e * 8 + l] = phi[((int64_t)(i + (l & 1)) * (n + 1) + j + ((l >> 1) & 1)) * (n + 1) + k + ((l >> 2) & 1)];
}

// Interior cells: the same volume accumulation with the 2x2x2 Gauss rule
// (SPEC.md:159-167); one constant matrix for every interior cell.
__global__ void k_interior_element(double h, double* __restrict__ kint, double* __restrict__ fint) {
  Acc a;
  for (int t = 0; t < 64; ++t) a.dr[t] = 0.0;
  for (int t = 0; t < 8; ++t) a.fr[t] = 0.0;
  a.nvol = 0;
  const double g0 = 0.5 - 0.5 / sqrt(3.0), g1 = 0.5 + 0.5 / sqrt(3.0);
  const double gp[2] = {g0, g1};
  for (int l = 0; l < 8; ++l) vol_point(a, gp[l & 1], gp[(l >> 1) & 1], gp[(l >> 2) & 1], 0.125);
  for (int t = 0; t < 64; ++t) kint[t] = h * (a.dr[t] + 0.0 * 0.0 - (0.0 + 0.0));
  for (int t = 0; t < 8; ++t) fint[t] = h * h * h * a.fr[t];
}

// error_norms: per active cell of this rank, the volume
// integrals of (u_h - u)^2 and |grad u_h - grad u|^2 over the cell's rule
// (the cut rule of the element kernel, 2x2x2 Gauss for interior cells),
// u_h from the local solution vector. One thread per cell, the oracle's
// operation order (oracle/element.cpp error_norms).
__global__ void k_error_cells(int64_t na, const int64_t* __restrict__ cells, int n, double ox, double oy, double oz,
                              double h, const double* __restrict__ phi, const uint8_t* __restrict__ cls,
                              const int32_t* __restrict__ dof_of_node, const int32_t* __restrict__ loc_of_dof,
                              const double* __restrict__ x, double* __restrict__ out) {
  const int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (a >= na) return;
  const int64_t cell = cells[a];
  const int k = (int)(cell % n), j = (int)((cell / n) % n), i = (int)(cell / n / n);
  double q[8], uh[8];
  for (int l = 0; l < 8; ++l) {
    const int64_t v = ((int64_t)(i + (l & 1)) * (n + 1) + j + ((l >> 1) & 1)) * (n + 1) + k + ((l >> 2) & 1);
    q[l] = phi[v];
    const int32_t d = dof_of_node[v];
    const int32_t lo = d >= 0 ? loc_of_dof[d] : -1;
    uh[l] = lo >= 0 ? x[lo] : 0.0;
  }
  double vp[6][kVolPts][4], sp[6][kSurfPts][7];
  int nv[6];
  const bool cut = cls[cell] == CUTBDDC_CUT;
  if (cut) {
    for (int t = 0; t < 6; ++t) {
      PtList L{vp[t], sp[t], 0, 0};
      tet_points(t, q, L);
      nv[t] = L.nv;
    }
  } else {  // full_quadrature_ref: 2x2x2 Gauss, weight 1/8 (in tet slot 0)
    const double g0 = 0.5 - 0.5 / sqrt(3.0), g1 = 0.5 + 0.5 / sqrt(3.0);
    for (int l = 0; l < 8; ++l) {
      vp[0][l][0] = (l & 1) ? g1 : g0;
      vp[0][l][1] = ((l >> 1) & 1) ? g1 : g0;
      vp[0][l][2] = ((l >> 2) & 1) ? g1 : g0;
      vp[0][l][3] = 0.125;
    }
    nv[0] = 8;
    for (int t = 1; t < 6; ++t) nv[t] = 0;
  }
  double el2 = 0.0, eh1 = 0.0;
  for (int t = 0; t < 6; ++t)
    for (int p = 0; p < nv[t]; ++p) {
      const double* P = vp[t][p];
      double v = 0.0, g[3] = {0.0, 0.0, 0.0};
      for (int l = 0; l < 8; ++l) {
        double gl[3], vl;
        q1_gv(P, l, gl, &vl);
        v += uh[l] * vl;
        for (int d = 0; d < 3; ++d) g[d] += uh[l] * gl[d];
      }
      const double xp = ox + ((double)i + P[0]) * h, yp = oy + ((double)j + P[1]) * h, zp = oz + ((double)k + P[2]) * h;
      double gu[3];
      mms_grad(xp, yp, zp, gu);
      const double e = v - mms_u(xp, yp, zp);
      const double w = P[3] * (h * h * h);
      el2 += w * (e * e);
      double s = 0.0;
      for (int d = 0; d < 3; ++d) {
        const double ed = g[d] / h - gu[d];
        s += ed * ed;
      }
      eh1 += w * s;
    }
  out[2 * a] = el2;
  out[2 * a + 1] = eh1;
}

__global__ void k_local_active(int64_t nc, int n, int B, int nb, const int64_t* __restrict__ active,
                               const int32_t* __restrict__ sd_of_block, uint8_t* __restrict__ flag) {
  const int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (a >= nc) return;
  const int64_t c = active[a];
  const int64_t k = c % n, j = (c / n) % n, i = c / n / n;
  flag[a] = sd_of_block[((i / B) * nb + j / B) * nb + k / B] >= 0;
}

}  // namespace

// sum over this rank's active cells, ascending cell id (the oracle's order)
void error_norms_device(cutbddc_gpu* h, const double* xloc, double* l2sq, double* h1sq) {
  cudaStream_t s = h->stream;
  const int64_t na = h->n_active;
  DevBuf<uint8_t>& flag = h->ws_tmp2;
  DevBuf<int64_t>& cells = h->ws_cells;
  DevBuf<int64_t>& cnt = h->ws_cnt;
  flag.alloc((size_t)std::max<int64_t>(1, na));
  cells.alloc((size_t)std::max<int64_t>(1, na));
  cnt.alloc(2);
  k_local_active<<<grid_for(std::max<int64_t>(1, na), 256), 256, 0, s>>>(na, h->n, h->block, h->nb, h->active_cells.p,
                                                                        h->sd_of_block.p, flag.p);
  CB_LAUNCH();
  size_t tb = 0;
  CB_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, h->active_cells.p, flag.p, cells.p, cnt.p, na, s));
  DevBuf<uint8_t>& tmp = h->ws_tmp;
  tmp.alloc(std::max(tmp.n, tb));
  CB_CUDA(cub::DeviceSelect::Flagged(tmp.p, tb, h->active_cells.p, flag.p, cells.p, cnt.p, na, s));
  int64_t nl = 0;
  CB_CUDA(cudaMemcpyAsync(&nl, cnt.p, 8, cudaMemcpyDeviceToHost, s));
  CB_CUDA(cudaStreamSynchronize(s));
  DevBuf<double> per;
  per.alloc((size_t)std::max<int64_t>(1, 2 * nl));
  if (nl > 0) {
    k_error_cells<<<grid_for(nl, 64), 64, 0, s>>>(nl, cells.p, h->n, h->origin[0], h->origin[1], h->origin[2], h->h,
                                                  h->phi.p, h->cls.p, h->dof_of_node.p, h->loc_of_dof.p, xloc, per.p);
    CB_LAUNCH();
  }
  std::vector<double> hv = per.to_host(s);
  double a = 0.0, b = 0.0;
  for (int64_t c = 0; c < nl; ++c) {
    a += hv[(size_t)(2 * c)];
    b += hv[(size_t)(2 * c + 1)];
  }
  *l2sq = a;
  *h1sq = b;
}

void interior_element_device(cutbddc_gpu* h, double* kint, double* fint) {
  k_interior_element<<<1, 1, 0, h->stream>>>(h->h, kint, fint);
  CB_LAUNCH();
}

void cut_elements_device(cutbddc_gpu* h) {
  DevBuf<int>& degen = h->ws_flag;
  degen.alloc(1);
  degen.zero(h->stream);
  h->ke.alloc((size_t)std::max<int64_t>(1, h->n_cut) * 64);
  h->fe.alloc((size_t)std::max<int64_t>(1, h->n_cut) * 8);
  h->beta.alloc((size_t)std::max<int64_t>(1, h->n_cut));
  h->empty.alloc((size_t)std::max<int64_t>(1, h->n_cut));
  if (h->n_cut > 0) {
    DevBuf<double>& q8all = h->ws_q8;
    q8all.alloc((size_t)h->n_cut * 8);

    k_gather_q8<<<grid_for(h->n_cut, 256), 256, 0, h->stream>>>(h->n, h->n_cut, h->cut_cells.p, h->phi.p, q8all.p);
    CB_LAUNCH();
    if (std::getenv("CUTBDDC_CUT_THREAD")) {  // the thread-per-cell form (A/B reference, f = 1 only)
      if (h->problem != kProblemUnitLoad) throw Failure(CUTBDDC_CONFIG, "CUTBDDC_CUT_THREAD: unit load only");
      k_cut_elements<<<grid_for(h->n_cut, 64), 64, 0, h->stream>>>(h->h, h->n_cut, q8all.p, h->ke.p, h->fe.p,
                                                                    h->beta.p, h->empty.p, degen.p);
      CB_LAUNCH();
    } else {
      DevBuf<double>& accs = h->ws_acc;
      DevBuf<int>& nvs = h->ws_nvs;
      accs.alloc((size_t)h->n_cut * kAcc);
      nvs.alloc((size_t)h->n_cut * 2);
      const LoadArgs la{h->problem, h->n, h->cut_cells.p, h->origin[0], h->origin[1], h->origin[2], h->h};
      k_cut_acc<<<(unsigned)((h->n_cut + kAccCells - 1) / kAccCells), 32 * kAccCells, 0, h->stream>>>(
          h->n_cut, q8all.p, accs.p, nvs.p, la);
      CB_LAUNCH();
      k_cut_pencil<<<(unsigned)((h->n_cut * 8 + CB_PENCIL_THREADS - 1) / CB_PENCIL_THREADS), CB_PENCIL_THREADS, 0,
                     h->stream>>>(
          h->h, h->n_cut, h->problem, accs.p, nvs.p, h->ke.p, h->fe.p, h->beta.p, h->empty.p, degen.p);
      CB_LAUNCH();
    }
  }
  int dg = 0;
  CB_CUDA(cudaMemcpyAsync(&dg, degen.p, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
  CB_CUDA(cudaStreamSynchronize(h->stream));
  if (dg) throw Failure(CUTBDDC_DEGENERATE, "generalized eigs: D is numerically zero (degenerate element)");
}

}  // namespace cutbddc_b200
