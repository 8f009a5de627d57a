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
#include <cstdlib>

#include "handle.cuh"

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

// Cyclic Jacobi, same sweep order / thresholds as the CPU restatement.
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
    for (int p = 0; p < n; ++p) {
      for (int q = p + 1; q < n; ++q) {
        const double apq = a[p * n + q];
        if (apq == 0.0) continue;
        const double app = a[p * n + p], aqq = a[q * n + q];
        const double theta = (aqq - app) / (2.0 * apq);
        const double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
        const double c = 1.0 / sqrt(t * t + 1.0);
        const double s = t * c;
        for (int k = 0; k < n; ++k) {
          const double akp = a[k * n + p], akq = a[k * n + q];
          a[k * n + p] = c * akp - s * akq;
          a[k * n + q] = s * akp + c * akq;
        }
        for (int k = 0; k < n; ++k) {
          const double apk = a[p * n + k], aqk = a[q * n + k];
          a[p * n + k] = c * apk - s * aqk;
          a[q * n + k] = s * apk + c * aqk;
        }
        a[p * n + q] = 0.0;
        a[q * n + p] = 0.0;
        for (int k = 0; k < n; ++k) {
          const double vkp = v[k * n + p], vkq = v[k * n + q];
          v[k * n + p] = c * vkp - s * vkq;
          v[k * n + q] = s * vkp + c * vkq;
        }
      }
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
// Lane-group form of cut_element (same arithmetic, bit for bit): four cut
// cells per warp, eight lanes per cell.
//
// Lanes 0-5 of a group cut one Kuhn tet each and write its quadrature points
// to shared memory (volume: x, y, z, w; surface: x, y, z, w, n). Every
// accumulator of the sequential code (D, F, B, M, N: 180 unique entries) is
// then owned by one lane, which sums its entry over the points in the
// sequential order (tet, piece, point), so every sum sees the same operands
// in the same order. The Q1 factors are rebuilt per point from f_d in {x_d,
// 1 - x_d}: grad[l][0] = (+-1 * f1) * f2 = +-(f1 f2) exactly, so no product
// differs from q1_eval. The Jacobi rotations of the 8x8 pencil run
// lane-parallel over k (each k touches only its own row / column entries,
// as in the sequential loops).
constexpr int kVolPts = 12;   // per tet: up to three sub-tets x 4 points
constexpr int kSurfPts = 6;   // per tet: up to two triangles x 3 points
constexpr int kCellWarps = 1; // warps per CTA (four cut cells per warp; shared memory bound)

struct CellSmem {
  union {
    struct {  // quadrature points (dead after the accumulation)
      double vp[6][kVolPts][4];
      double sp[6][kSurfPts][7];
    };
    struct {  // pencil scratch (gen_eigs_max)
      double a[64], v[64], ev[8], bq[64], c[64], cv[64], cev[8];
    };
  };
  double dr[64], br[64], mr[64], nr[64], fr[8];
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

// jacobi(n, a, v, ev) by a group of 8 lanes (gl = index within the group):
// lane k owns index k of each rotation's row / column updates
__device__ void grp_jacobi(int n, double* a, double* v, double* ev, int gl, unsigned gm) {
  for (int k = gl; k < n * n; k += 8) v[k] = (k / n) == (k % n) ? 1.0 : 0.0;
  __syncwarp(gm);
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0, diag = 0.0;
    for (int i = 0; i < n; ++i) {
      diag += a[i * n + i] * a[i * n + i];
      for (int j = i + 1; j < n; ++j) off += a[i * n + j] * a[i * n + j];
    }
    if (off <= 1e-32 * diag || off < 1e-300) break;
    for (int p = 0; p < n; ++p) {
      for (int q = p + 1; q < n; ++q) {
        const double apq = a[p * n + q];
        if (apq == 0.0) continue;
        const double app = a[p * n + p], aqq = a[q * n + q];
        const double theta = (aqq - app) / (2.0 * apq);
        const double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
        const double c = 1.0 / sqrt(t * t + 1.0);
        const double s = t * c;
        __syncwarp(gm);
        const int k = gl;
        if (k < n) {
          const double akp = a[k * n + p], akq = a[k * n + q];
          a[k * n + p] = c * akp - s * akq;
          a[k * n + q] = s * akp + c * akq;
        }
        __syncwarp(gm);
        if (k < n) {
          const double apk = a[p * n + k], aqk = a[q * n + k];
          a[p * n + k] = c * apk - s * aqk;
          a[q * n + k] = s * apk + c * aqk;
          const double vkp = v[k * n + p], vkq = v[k * n + q];
          v[k * n + p] = c * vkp - s * vkq;
          v[k * n + q] = s * vkp + c * vkq;
        }
        __syncwarp(gm);
        if (gl == 0) {
          a[p * n + q] = 0.0;
          a[q * n + p] = 0.0;
        }
        __syncwarp(gm);
      }
    }
  }
  for (int i = gl; i < n; i += 8) ev[i] = a[i * n + i];
  __syncwarp(gm);
}

// gen_eigs_max (linalg.cpp:108-136) by a lane group: the same operations as
// the sequential function above
__device__ double grp_gen_eigs_max(CellSmem& S, int gl, unsigned gm) {
  for (int i = gl; i < 64; i += 8) S.a[i] = S.dr[i];
  __syncwarp(gm);
  grp_jacobi(8, S.a, S.v, S.ev, gl, gm);
  double lmax = S.ev[0];
  for (int i = 1; i < 8; ++i) lmax = fmax(lmax, S.ev[i]);
  if (!(lmax > 0.0)) return -1.0;
  int m = 0;
  int keep[8];
  for (int k = 0; k < 8; ++k)
    if (S.ev[k] >= 1e-12 * lmax) keep[m++] = k;
  for (int e = gl; e < 8 * m; e += 8) {
    const int i = e / m, k = e % m;
    double s = 0;
    for (int j = 0; j < 8; ++j) s += S.br[i * 8 + j] * S.v[j * 8 + keep[k]];
    S.bq[i * m + k] = s;
  }
  __syncwarp(gm);
  for (int e = gl; e < m * m; e += 8) {
    const int k = e / m, l = e % m;
    double s = 0;
    for (int i = 0; i < 8; ++i) s += S.v[i * 8 + keep[k]] * S.bq[i * m + l];
    S.c[k * m + l] = s / (sqrt(S.ev[keep[k]]) * sqrt(S.ev[keep[l]]));
  }
  __syncwarp(gm);
  for (int e = gl; e < m * m; e += 8) {
    const int k = e / m, l = e % m;
    S.a[k * m + l] = l == k ? S.c[k * m + k] : 0.5 * (S.c[min(k, l) * m + max(k, l)] + S.c[max(k, l) * m + min(k, l)]);
  }
  __syncwarp(gm);
  grp_jacobi(m, S.a, S.cv, S.cev, gl, gm);
  double best = S.cev[0];
  for (int k = 1; k < m; ++k) best = fmax(best, S.cev[k]);
  return best;
}

// four cut cells per warp, eight lanes per cell
__global__ void __launch_bounds__(32 * kCellWarps) k_cut_elements_warp(double h, int64_t ncut,
                                                                       const double* __restrict__ q8all,
                                                                       double* __restrict__ ke, double* __restrict__ fe,
                                                                       double* __restrict__ beta,
                                                                       uint8_t* __restrict__ empty,
                                                                       int* __restrict__ degenerate) {
  __shared__ CellSmem smem[4 * kCellWarps];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, g = lane >> 3, gl = lane & 7;
  const unsigned gm = 0xffu << (8 * g);
  const int64_t e = ((int64_t)blockIdx.x * kCellWarps + wid) * 4 + g;
  if (e >= ncut) return;
  CellSmem& S = smem[4 * wid + g];
  const double* q8 = q8all + e * 8;
  if (gl < 6) {
    PtList L{S.vp[gl], S.sp[gl], 0, 0};
    double q[8];
    for (int i = 0; i < 8; ++i) q[i] = q8[i];
    tet_points(gl, q, L);
    S.nv[gl] = L.nv;
    S.ns[gl] = L.ns;
  }
  __syncwarp(gm);
  int nvol = 0, nsurf = 0;
  for (int t = 0; t < 6; ++t) {
    nvol += S.nv[t];
    nsurf += S.ns[t];
  }
  if (nvol == 0) {
    for (int t = gl; t < 64; t += 8) ke[e * 64 + t] = 0.0;
    fe[e * 8 + gl] = 0.0;
    if (gl == 0) {
      beta[e] = 0.0;
      empty[e] = 1;
    }
    return;
  }
  // accumulators: 0-35 D (i <= j), 36-43 F, 44-79 B (i <= j), 80-115 M (i <= j), 116-179 N
  for (int it = gl; it < 180; it += 8) {
    int kind, i, j;
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
    double acc = 0.0;
    if (kind <= 1) {
      for (int t = 0; t < 6; ++t)
        for (int pnt = 0; pnt < S.nv[t]; ++pnt) {
          const double* P = S.vp[t][pnt];
          const double w = P[3];
          double gi[3], gj[3], vi;
          q1_gv(P, i, gi, &vi);
          if (kind == 1) {
            acc += w * vi;
          } else {
            q1_gv(P, j, gj, nullptr);
            acc += w * (gi[0] * gj[0] + gi[1] * gj[1] + gi[2] * gj[2]);
          }
        }
    } else {
      for (int t = 0; t < 6; ++t)
        for (int pnt = 0; pnt < S.ns[t]; ++pnt) {
          const double* P = S.sp[t][pnt];
          const double w = P[3], nx = P[4], ny = P[5], nz = P[6];
          double gi[3], gj[3], vi, vj;
          q1_gv(P, i, gi, &vi);
          q1_gv(P, j, gj, &vj);
          if (kind == 2) {
            const double ni = nx * gi[0] + ny * gi[1] + nz * gi[2];
            const double nj = nx * gj[0] + ny * gj[1] + nz * gj[2];
            acc += w * (ni * nj);
          } else if (kind == 3) {
            acc += w * (vi * vj);
          } else {
            const double ni = nx * gi[0] + ny * gi[1] + nz * gi[2];
            acc += w * (vj * ni);
          }
        }
    }
    if (kind == 0) {
      S.dr[i * 8 + j] = acc;
      S.dr[j * 8 + i] = acc;
    } else if (kind == 1) {
      S.fr[i] = acc;
    } else if (kind == 2) {
      S.br[i * 8 + j] = acc;
      S.br[j * 8 + i] = acc;
    } else if (kind == 3) {
      S.mr[i * 8 + j] = acc;
      S.mr[j * 8 + i] = acc;
    } else {
      S.nr[i * 8 + j] = acc;
    }
  }
  __syncwarp(gm);
  double lambda = 0.0;
  if (nsurf > 0) {
    lambda = grp_gen_eigs_max(S, gl, gm);
    if (lambda < 0) {
      if (gl == 0) atomicExch(degenerate, 1);
      lambda = 0.0;
    }
  }
  const double betar = 2.0 * lambda;
  for (int t = gl; t < 64; t += 8) {
    const int x = t / 8, y = t % 8;
    ke[e * 64 + t] = h * (S.dr[x * 8 + y] + betar * S.mr[x * 8 + y] - (S.nr[x * 8 + y] + S.nr[y * 8 + x]));
  }
  fe[e * 8 + gl] = h * h * h * S.fr[gl];
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

}  // namespace

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
    if (std::getenv("CUTBDDC_CUT_THREAD"))  // the thread-per-cell form (A/B reference)
      k_cut_elements<<<grid_for(h->n_cut, 64), 64, 0, h->stream>>>(h->h, h->n_cut, q8all.p, h->ke.p, h->fe.p,
                                                                    h->beta.p, h->empty.p, degen.p);
    else
      k_cut_elements_warp<<<(unsigned)((h->n_cut + 4 * kCellWarps - 1) / (4 * kCellWarps)), 32 * kCellWarps, 0,
                            h->stream>>>(
          h->h, h->n_cut, q8all.p, h->ke.p, h->fe.p, h->beta.p, h->empty.p, degen.p);
    CB_LAUNCH();
  }
  int dg = 0;
  CB_CUDA(cudaMemcpyAsync(&dg, degen.p, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
  CB_CUDA(cudaStreamSynchronize(h->stream));
  if (dg) throw Failure(CUTBDDC_DEGENERATE, "generalized eigs: D is numerically zero (degenerate element)");
}

}  // namespace cutbddc_b200
