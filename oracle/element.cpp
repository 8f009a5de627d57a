// element.cpp — Q1 Nitsche element matrices and beta_e (TEST INFRASTRUCTURE).
// SPEC.md:205-222 (nitsche_beta, assemble_element); PAPER.md:314-348 (forms
// A_e, l_e, beta_e = 2 lambda_max of B_e x = lambda D_e x).
// dense_generalized_eigs_max follows linalg.cpp:108-136 (eigendecompose D,
// keep eigenvalues >= kernel_tol * lambda_max(D), project B, largest
// eigenvalue of the deflated pencil) with a cyclic Jacobi eigensolver in
// place of Eigen's SelfAdjointEigenSolver.
//
// Everything is computed on the reference cell [0,1]^3 and scaled:
//   D = h Dr, B = Br, M_gamma = h^2 Mr, N = h Nr, beta = 2 lambda(Br, Dr) / h,
//   K_e = h (Dr + 2 lambda Mr - Nr - Nr^T), f_e = h^3 int_ref phi_b  (f = 1, g = 0).
// Pin: a cut cell whose retained volume rule is
// empty contributes nothing (no volume and no Nitsche term).
#include <cmath>
#include <cstring>

#include "oracle.hpp"

namespace oracle {

// Jacobi rotation (c, s) annihilating a_pq from h = a_qq - a_pp, g = 2 a_pq
// (g != 0): t = tan = sgn / (|theta| + sqrt(theta^2 + 1)) with theta = h / g,
// c = 1 / sqrt(t^2 + 1), s = t c, evaluated without theta as c = d / w,
// s = sgn |g| / w with d = |h| + sqrt(h^2 + g^2), w = sqrt(d^2 + g^2) (two
// square roots and one division deep instead of two and three); the theta
// form is the fallback when the squares under- or overflow.
void jacobi_rotation(double h, double g, double* c, double* s) {
  const double sgn = (h == 0.0 || (h > 0.0) == (g > 0.0)) ? 1.0 : -1.0;
  const double rho = std::sqrt(h * h + g * g);
  const double d = std::fabs(h) + rho;
  const double w = std::sqrt(d * d + g * g);
  if (w > 0.0 && w <= 1.7976931348623157e308) {
    *c = d / w;
    *s = sgn * std::fabs(g) / w;
    return;
  }
  const double theta = h / g;
  const double t = (theta >= 0 ? 1.0 : -1.0) / (std::fabs(theta) + std::sqrt(theta * theta + 1.0));
  *c = 1.0 / std::sqrt(t * t + 1.0);
  *s = t * *c;
}

// Parallel-order cyclic Jacobi: a (n x n row-major, destroyed) -> eigenvalues
// ev, vectors v (columns, row-major storage v[i*n+k]). A sweep visits every
// pair (p, q), p < q, once, in round-robin (tournament) rounds of disjoint
// pairs: N = 8 players for n <= 8, else 16 (indices >= n sit out); round
// r = 0 .. N-2 pairs player N-1 with r and (r + k) mod (N-1) with (r - k) mod
// (N-1), k = 1 .. N/2-1. A round takes its rotations J_k from the matrix at
// the start of the round (the pairs are disjoint, so the angles do not depend
// on one another: the device computes them side by side), then A <- A J
// (column rotations, pairs in order), A <- J^T A (row rotations), a_pq =
// a_qp = 0, V <- V J. A pair whose a_pq is exactly zero is skipped. Stop when
// the off-diagonal Frobenius norm is <= 1e-16 of the diagonal's (or <= 1e-150)
// or after 100 sweeps.
void jacobi_eigs(int n, double* a, double* v, double* ev) {
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) v[i * n + j] = i == j ? 1.0 : 0.0;
  const int N = n <= 8 ? 8 : 16;
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0, diag = 0.0;
    for (int i = 0; i < n; ++i) {
      diag += a[i * n + i] * a[i * n + i];
      for (int j = i + 1; j < n; ++j) off += a[i * n + j] * a[i * n + j];
    }
    if (off <= 1e-32 * diag || off < 1e-300) break;
    for (int r = 0; r < N - 1; ++r) {
      int P[8], Q[8];
      double C[8], S[8];
      bool act[8];
      for (int k = 0; k < N / 2; ++k) {
        const int x = k == 0 ? N - 1 : (r + k) % (N - 1);
        const int y = k == 0 ? r : (r - k + (N - 1)) % (N - 1);
        P[k] = x < y ? x : y;
        Q[k] = x < y ? y : x;
        act[k] = Q[k] < n && a[P[k] * n + Q[k]] != 0.0;
        if (act[k])
          jacobi_rotation(a[Q[k] * n + Q[k]] - a[P[k] * n + P[k]], 2.0 * a[P[k] * n + Q[k]], &C[k], &S[k]);
      }
      for (int k = 0; k < N / 2; ++k) {  // A <- A J, V <- V J
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
      for (int k = 0; k < N / 2; ++k) {  // A <- J^T A
        if (!act[k]) continue;
        const int p = P[k], q = Q[k];
        const double c = C[k], s = S[k];
        for (int j = 0; j < n; ++j) {
          const double apj = a[p * n + j], aqj = a[q * n + j];
          a[p * n + j] = c * apj - s * aqj;
          a[q * n + j] = s * apj + c * aqj;
        }
      }
      for (int k = 0; k < N / 2; ++k)
        if (act[k]) a[P[k] * n + Q[k]] = a[Q[k] * n + P[k]] = 0.0;
    }
  }
  for (int i = 0; i < n; ++i) ev[i] = a[i * n + i];
}

double dense_generalized_eigs_max(const double* b, const double* d, int n, double kernel_tol) {
  if (n <= 0 || n > 16) fail(ErrorCode::InvalidArgument, "generalized eigs: dimension mismatch");
  double a[256], v[256], ev[16];
  std::memcpy(a, d, sizeof(double) * n * n);
  jacobi_eigs(n, a, v, ev);
  double lmax = ev[0];
  for (int i = 1; i < n; ++i) lmax = std::max(lmax, ev[i]);
  if (!(lmax > 0.0)) fail(ErrorCode::Degenerate, "generalized eigs: D is numerically zero (degenerate element)");
  int keep[16], m = 0;
  for (int k = 0; k < n; ++k)
    if (ev[k] >= kernel_tol * lmax) keep[m++] = k;
  if (m == 0) fail(ErrorCode::Degenerate, "generalized eigs: all directions deflated (degenerate element)");
  // C = Dk^{-1/2} Q^T B Q Dk^{-1/2}
  double bq[256];  // B Q : n x m
  for (int i = 0; i < n; ++i)
    for (int k = 0; k < m; ++k) {
      double s = 0;
      for (int j = 0; j < n; ++j) s += b[i * n + j] * v[j * n + keep[k]];
      bq[i * m + k] = s;
    }
  double c[256], cv[256], cev[16];
  for (int k = 0; k < m; ++k)
    for (int l = 0; l < m; ++l) {
      double s = 0;
      for (int i = 0; i < n; ++i) s += v[i * n + keep[k]] * bq[i * m + l];
      c[k * m + l] = s / (std::sqrt(ev[keep[k]]) * std::sqrt(ev[keep[l]]));
    }
  for (int k = 0; k < m; ++k)
    for (int l = k + 1; l < m; ++l) {
      const double s = 0.5 * (c[k * m + l] + c[l * m + k]);
      c[k * m + l] = s;
      c[l * m + k] = s;
    }
  jacobi_eigs(m, c, cv, cev);
  double best = cev[0];
  for (int k = 1; k < m; ++k) best = std::max(best, cev[k]);
  return best;
}

namespace {

inline void q1_eval(const double xi[3], double val[8], double grad[8][3]) {
  for (int l = 0; l < 8; ++l) {
    double f[3], df[3];
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

}  // namespace

Element element_matrix(const Mesh& m, std::int64_t cell) {
  Element e{};
  const double h = m.h[0];
  const bool cut = m.cls[(size_t)cell] == kCut;
  std::int64_t nodes[8];
  m.cell_nodes(cell, nodes);
  double phiv[8];
  for (int l = 0; l < 8; ++l) phiv[l] = m.phi[(size_t)nodes[l]];
  const CutRule rule = cut ? cut_quadrature_ref(phiv) : full_quadrature_ref();
  if (rule.vol.empty()) {
    e.empty = true;
    return e;
  }
  double dr[64] = {0}, br[64] = {0}, mr[64] = {0}, nr[64] = {0}, fr[8] = {0}, g1[8] = {0}, g2[8] = {0};
  double val[8], grad[8][3];
  const bool mms = m.problem == kProblemManufactured;
  int cc[3];
  m.cell_coords(cell, cc);
  auto phys = [&](const double* xi, double x[3]) {  // origin + (cell + xi) h
    for (int d = 0; d < 3; ++d) x[d] = m.origin[d] + ((double)cc[d] + xi[d]) * h;
  };
  for (const auto& p : rule.vol) {
    const double xi[3] = {p[0], p[1], p[2]};
    q1_eval(xi, val, grad);
    double fx = 1.0;
    if (mms) {
      double x[3];
      phys(xi, x);
      fx = Manufactured::f(x);
    }
    for (int a = 0; a < 8; ++a) {
      fr[a] += mms ? p[3] * (fx * val[a]) : p[3] * val[a];
      for (int b = 0; b < 8; ++b)
        dr[a * 8 + b] += p[3] * (grad[a][0] * grad[b][0] + grad[a][1] * grad[b][1] + grad[a][2] * grad[b][2]);
    }
  }
  double lambda = 0.0;
  if (!rule.surf.empty()) {
    for (const auto& p : rule.surf) {
      const double xi[3] = {p[0], p[1], p[2]};
      q1_eval(xi, val, grad);
      double gn[8];
      for (int a = 0; a < 8; ++a) gn[a] = p[4] * grad[a][0] + p[5] * grad[a][1] + p[6] * grad[a][2];
      if (mms) {  // Nitsche load: beta g phi_a - g n.grad phi_a, g = u on the boundary
        double x[3];
        phys(xi, x);
        const double gx = Manufactured::u(x);
        for (int a = 0; a < 8; ++a) {
          g1[a] += p[3] * (gx * val[a]);
          g2[a] += p[3] * (gx * gn[a]);
        }
      }
      for (int a = 0; a < 8; ++a)
        for (int b = 0; b < 8; ++b) {
          br[a * 8 + b] += p[3] * (gn[a] * gn[b]);
          mr[a * 8 + b] += p[3] * (val[a] * val[b]);
          nr[a * 8 + b] += p[3] * (val[b] * gn[a]);
        }
    }
    lambda = dense_generalized_eigs_max(br, dr, 8, 1e-12);
  }
  const double betar = 2.0 * lambda;
  for (int a = 0; a < 8; ++a)
    for (int b = 0; b < 8; ++b)
      e.k[a * 8 + b] = h * (dr[a * 8 + b] + betar * mr[a * 8 + b] - (nr[a * 8 + b] + nr[b * 8 + a]));
  for (int a = 0; a < 8; ++a) e.f[a] = mms ? h * h * h * fr[a] + h * (betar * g1[a] - g2[a]) : h * h * h * fr[a];
  e.beta = betar / h;
  e.empty = false;
  return e;
}

void error_norms(const Mesh& m, const double* x, double* l2, double* h1) {
  const double h = m.h[0];
  double el2 = 0.0, eh1 = 0.0;
  for (std::int64_t cell : m.active) {  // ascending cell id, sequential sums
    std::int64_t nodes[8];
    m.cell_nodes(cell, nodes);
    double phiv[8], uh[8];
    for (int l = 0; l < 8; ++l) {
      phiv[l] = m.phi[(size_t)nodes[l]];
      const std::int32_t d = m.dof_of_node[(size_t)nodes[l]];
      uh[l] = d >= 0 ? x[d] : 0.0;
    }
    const CutRule rule = m.cls[(size_t)cell] == kCut ? cut_quadrature_ref(phiv) : full_quadrature_ref();
    int cc[3];
    m.cell_coords(cell, cc);
    double val[8], grad[8][3];
    for (const auto& p : rule.vol) {
      const double xi[3] = {p[0], p[1], p[2]};
      q1_eval(xi, val, grad);
      double xp[3];
      for (int d = 0; d < 3; ++d) xp[d] = m.origin[d] + ((double)cc[d] + xi[d]) * h;
      double v = 0.0, g[3] = {0.0, 0.0, 0.0}, gu[3];
      for (int l = 0; l < 8; ++l) {
        v += uh[l] * val[l];
        for (int d = 0; d < 3; ++d) g[d] += uh[l] * grad[l][d];
      }
      Manufactured::grad(xp, gu);
      const double e = v - Manufactured::u(xp);
      const double w = p[3] * (h * h * h);
      el2 += w * (e * e);
      double s = 0.0;
      for (int d = 0; d < 3; ++d) {
        const double ed = g[d] / h - gu[d];
        s += ed * ed;
      }
      eh1 += w * s;
    }
  }
  *l2 = std::sqrt(el2);
  *h1 = std::sqrt(eh1);
}

}  // namespace oracle
