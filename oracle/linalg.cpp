// linalg.cpp — sparse/dense Cholesky without Eigen (TEST INFRASTRUCTURE).
// Replaces SparseCholesky (linalg.cpp:34-62: Eigen SimplicialLDLT + AMD) by a
// left-looking simplicial LL^T with a geometric nested-dissection ordering of
// the lattice coordinates. Pivot rule of linalg.cpp:42-54: a non-positive
// pivot raises Singular carrying the ORIGINAL index of the offending row.
#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <functional>

#include "oracle.hpp"

namespace oracle {

namespace {

// Recursive coordinate bisection: split the longest axis at the midpoint
// plane; order = ND(left) ND(right) separator.
// ND leaf size: 16 by default. ORACLE_ND_LEAF overrides it (perturbation
// experiments of tests/test_oracle_sensitivity.py: the elimination order is
// not part of SparseCholesky's contract, linalg.hpp:55-67).
size_t nd_leaf() {
  const char* e = std::getenv("ORACLE_ND_LEAF");
  return e && e[0] ? (size_t)std::max(1, std::atoi(e)) : 16;
}

void nd_order(std::vector<int>& ids, const std::vector<std::array<int, 3>>& xyz, std::vector<int>& out) {
  if (ids.size() <= nd_leaf()) {
    out.insert(out.end(), ids.begin(), ids.end());
    return;
  }
  int lo[3], hi[3];
  for (int d = 0; d < 3; ++d) {
    lo[d] = 1 << 30;
    hi[d] = -(1 << 30);
  }
  for (int i : ids)
    for (int d = 0; d < 3; ++d) {
      lo[d] = std::min(lo[d], xyz[(size_t)i][(size_t)d]);
      hi[d] = std::max(hi[d], xyz[(size_t)i][(size_t)d]);
    }
  int ax = 0;
  for (int d = 1; d < 3; ++d)
    if (hi[d] - lo[d] > hi[ax] - lo[ax]) ax = d;
  if (hi[ax] == lo[ax]) {
    out.insert(out.end(), ids.begin(), ids.end());
    return;
  }
  const int mid = (lo[ax] + hi[ax]) / 2;
  std::vector<int> l, r, s;
  for (int i : ids) {
    const int c = xyz[(size_t)i][(size_t)ax];
    (c < mid ? l : (c > mid ? r : s)).push_back(i);
  }
  nd_order(l, xyz, out);
  nd_order(r, xyz, out);
  out.insert(out.end(), s.begin(), s.end());
}

}  // namespace

void SparseCholesky::factor(const Csr& a, const std::vector<std::array<int, 3>>& coords) {
  n = a.n;
  std::vector<int> ids((size_t)n);
  for (int i = 0; i < n; ++i) ids[(size_t)i] = i;
  perm.clear();
  perm.reserve((size_t)n);
  nd_order(ids, coords, perm);
  iperm.assign((size_t)n, 0);
  for (int k = 0; k < n; ++k) iperm[(size_t)perm[(size_t)k]] = k;
  // columns of L, dynamic
  std::vector<std::vector<int>> rows((size_t)n);
  std::vector<std::vector<double>> vals((size_t)n);
  std::vector<int> head((size_t)n, -1), link((size_t)n, -1), next((size_t)n, 0);
  std::vector<double> w((size_t)n, 0.0);
  std::vector<char> mark((size_t)n, 0);
  std::vector<int> pat;
  for (int j = 0; j < n; ++j) {
    pat.clear();
    const int oj = perm[(size_t)j];
    for (int p = a.ptr[(size_t)oj]; p < a.ptr[(size_t)oj + 1]; ++p) {
      const int i = iperm[(size_t)a.col[(size_t)p]];
      if (i < j) continue;
      w[(size_t)i] += a.val[(size_t)p];
      if (!mark[(size_t)i]) {
        mark[(size_t)i] = 1;
        pat.push_back(i);
      }
    }
    if (!mark[(size_t)j]) {
      mark[(size_t)j] = 1;
      pat.push_back(j);
    }
    int k = head[(size_t)j];
    while (k != -1) {
      const int nk = link[(size_t)k];
      int p = next[(size_t)k];
      const auto& rk = rows[(size_t)k];
      const auto& vk = vals[(size_t)k];
      const double ljk = vk[(size_t)p];
      for (size_t q = (size_t)p; q < rk.size(); ++q) {
        const int i = rk[q];
        w[(size_t)i] -= vk[q] * ljk;
        if (!mark[(size_t)i]) {
          mark[(size_t)i] = 1;
          pat.push_back(i);
        }
      }
      ++p;
      next[(size_t)k] = p;
      if ((size_t)p < rk.size()) {
        const int r = rk[(size_t)p];
        link[(size_t)k] = head[(size_t)r];
        head[(size_t)r] = k;
      }
      k = nk;
    }
    const double d = w[(size_t)j];
    if (!(d > 0.0)) {
      for (int i : pat) {
        w[(size_t)i] = 0;
        mark[(size_t)i] = 0;
      }
      fail(ErrorCode::Singular,
           "cholesky: matrix is not positive definite (pivot index " + std::to_string(oj) + ")");
    }
    const double ljj = std::sqrt(d);
    std::sort(pat.begin(), pat.end());
    auto& rj = rows[(size_t)j];
    auto& vj = vals[(size_t)j];
    rj.reserve(pat.size());
    vj.reserve(pat.size());
    for (int i : pat) {
      rj.push_back(i);
      vj.push_back(i == j ? ljj : w[(size_t)i] / ljj);
      w[(size_t)i] = 0;
      mark[(size_t)i] = 0;
    }
    next[(size_t)j] = 1;
    if (rj.size() > 1) {
      const int r = rj[1];
      link[(size_t)j] = head[(size_t)r];
      head[(size_t)r] = j;
    }
  }
  lp.assign((size_t)n + 1, 0);
  for (int j = 0; j < n; ++j) lp[(size_t)j + 1] = lp[(size_t)j] + (int)rows[(size_t)j].size();
  li.resize((size_t)lp[(size_t)n]);
  lx.resize((size_t)lp[(size_t)n]);
  for (int j = 0; j < n; ++j) {
    std::copy(rows[(size_t)j].begin(), rows[(size_t)j].end(), li.begin() + lp[(size_t)j]);
    std::copy(vals[(size_t)j].begin(), vals[(size_t)j].end(), lx.begin() + lp[(size_t)j]);
  }
}

void SparseCholesky::solve(double* x) const {
  std::vector<double> y((size_t)n);
  for (int k = 0; k < n; ++k) y[(size_t)k] = x[perm[(size_t)k]];
  for (int j = 0; j < n; ++j) {  // L y = b (column oriented)
    const double yj = y[(size_t)j] / lx[(size_t)lp[(size_t)j]];
    y[(size_t)j] = yj;
    for (int p = lp[(size_t)j] + 1; p < lp[(size_t)j + 1]; ++p) y[(size_t)li[(size_t)p]] -= lx[(size_t)p] * yj;
  }
  for (int j = n - 1; j >= 0; --j) {  // L^T x = y
    double s = y[(size_t)j];
    for (int p = lp[(size_t)j] + 1; p < lp[(size_t)j + 1]; ++p) s -= lx[(size_t)p] * y[(size_t)li[(size_t)p]];
    y[(size_t)j] = s / lx[(size_t)lp[(size_t)j]];
  }
  for (int k = 0; k < n; ++k) x[perm[(size_t)k]] = y[(size_t)k];
}

void DenseCholesky::factor(const std::vector<double>& a, int nn, const std::string& ctx) {
  n = nn;
  l = a;
  for (int j = 0; j < n; ++j) {
    double d = l[(size_t)j * n + j];
    for (int k = 0; k < j; ++k) d -= l[(size_t)j * n + k] * l[(size_t)j * n + k];
    if (!(d > 0.0))
      fail(ErrorCode::Singular, "dense cholesky: not positive definite (pivot index " + std::to_string(j) + ")" +
                                    (ctx.empty() ? "" : " (" + ctx + ")"));
    const double ljj = std::sqrt(d);
    l[(size_t)j * n + j] = ljj;
    for (int i = j + 1; i < n; ++i) {
      double s = l[(size_t)i * n + j];
      for (int k = 0; k < j; ++k) s -= l[(size_t)i * n + k] * l[(size_t)j * n + k];
      l[(size_t)i * n + j] = s / ljj;
    }
  }
  for (int i = 0; i < n; ++i)
    for (int j = i + 1; j < n; ++j) l[(size_t)i * n + j] = 0.0;
}

void DenseCholesky::solve(double* x) const {
  for (int i = 0; i < n; ++i) {
    double s = x[i];
    for (int k = 0; k < i; ++k) s -= l[(size_t)i * n + k] * x[k];
    x[i] = s / l[(size_t)i * n + i];
  }
  for (int i = n - 1; i >= 0; --i) {
    double s = x[i];
    for (int k = i + 1; k < n; ++k) s -= l[(size_t)k * n + i] * x[k];
    x[i] = s / l[(size_t)i * n + i];
  }
}

}  // namespace oracle
