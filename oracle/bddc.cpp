// bddc.cpp — BDDC preconditioner (TEST INFRASTRUCTURE).
// SPEC.md:351-418 (build_weighting :370-378, build_coarse_space :379-387,
// apply :388-396); PAPER.md:387-473 (Eq. (bddc) M = I0 A0^{-1} I0^T + Q A~^{-1} Q^T).
// Pins:
//   * constraint rows C_w: corner -> e_xi; edge/face -> (1/|lambda|) sum e_xi
//     (SPEC.md:404, :406); rows in global coarse order.
//   * constrained Neumann solve by augmented Lagrangian:
//     K = A_w + rho C^T C, rho = mean(diag A_w); W = K^{-1} C^T; S = C W;
//     Phi = W S^{-1} (solves [A C^T; C 0][Phi; .] = [0; I]);
//     saddle solve with zero constraints: z = y - Phi (C y), y = K^{-1} r.
//   * A_c,w = Phi^T A_w Phi, assembled in subdomain order, dense Cholesky.
//   * r1 = r - Abar z0 with r1 := 0 exactly on interior dofs (App. B.12).
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "oracle.hpp"

namespace oracle {

namespace {

std::vector<std::array<int, 3>> local_coords(const Problem& pb, const Subdomain& S, const std::vector<int>& locals) {
  std::vector<std::array<int, 3>> xyz;
  xyz.reserve(locals.size());
  for (int li : locals) {
    int c[3];
    pb.mesh.node_coords(pb.mesh.node_of_dof[(size_t)S.l2g[(size_t)li]], c);
    xyz.push_back({c[0], c[1], c[2]});
  }
  return xyz;
}

}  // namespace

void build_bddc(const Problem& pb, Bddc& bd, int objects, int weighting, int variant) {
  bd.objects = objects;
  bd.weighting = weighting;
  bd.variant = variant;
  bd.w = build_weighting(pb, weighting);
  std::vector<Object> objs = pb.objects;
  if (variant == kVariantV1) objs = split_edges_v1(pb, objs);
  if (variant == kVariantV2) {
    const auto ws = weighting == kWeightStiffness ? bd.w : build_weighting(pb, kWeightStiffness);
    objs = split_edges_v2(pb, objs, ws);
  }
  bd.coarse_objects.clear();
  for (auto& o : objs) {
    const bool sel = o.kind == kCorner || (o.kind == kEdge && objects >= kObjCE) || (o.kind == kFace && objects >= kObjCEF);
    if (sel) bd.coarse_objects.push_back(o);
  }
  bd.n_coarse = (int)bd.coarse_objects.size();
  const int nsd = (int)pb.sd.size();
  // constraint rows per subdomain
  bd.loc.assign((size_t)nsd, LocalBddc{});
  for (auto& L : bd.loc) L.c_ptr = {0};
  for (int c = 0; c < bd.n_coarse; ++c) {
    const Object& o = bd.coarse_objects[(size_t)c];
    for (int s : o.neigh) {
      auto& L = bd.loc[(size_t)s];
      const auto& l2g = pb.sd[(size_t)s].l2g;
      const double coef = 1.0 / (double)o.dofs.size();
      for (int g : o.dofs) {
        L.c_col.push_back((int)(std::lower_bound(l2g.begin(), l2g.end(), g) - l2g.begin()));
        L.c_val.push_back(o.kind == kCorner ? 1.0 : coef);
      }
      L.c_ptr.push_back((int)L.c_col.size());
      L.coarse_ids.push_back(c);
    }
  }
  parallel_for(nsd, [&](std::int64_t s) {
    const Subdomain& S = pb.sd[(size_t)s];
    LocalBddc& L = bd.loc[(size_t)s];
    const int n = (int)S.l2g.size();
    const int m = (int)L.coarse_ids.size();
    // interior problem A_II
    L.interior_local.clear();
    for (int i = 0; i < n; ++i)
      if (S.interior[(size_t)i]) L.interior_local.push_back(i);
    L.has_interior = !L.interior_local.empty();
    if (L.has_interior) {
      const int ni = (int)L.interior_local.size();
      std::vector<int> g2i((size_t)n, -1);
      for (int k = 0; k < ni; ++k) g2i[(size_t)L.interior_local[(size_t)k]] = k;
      Csr aii;
      aii.n = ni;
      aii.ptr.assign((size_t)ni + 1, 0);
      for (int k = 0; k < ni; ++k) {
        const int i = L.interior_local[(size_t)k];
        for (int p = S.a.ptr[(size_t)i]; p < S.a.ptr[(size_t)i + 1]; ++p) {
          const int j = g2i[(size_t)S.a.col[(size_t)p]];
          if (j < 0) continue;
          aii.col.push_back(j);
          aii.val.push_back(S.a.val[(size_t)p]);
        }
        aii.ptr[(size_t)k + 1] = (int)aii.col.size();
      }
      try {
        L.a_ii.factor(aii, local_coords(pb, S, L.interior_local));
      } catch (const Error& e) {
        fail(e.code, std::string(e.what()) + " (interior problem of subdomain " + std::to_string(s) + ")");
      }
    }
    // K = A + rho C^T C
    double dsum = 0;
    for (int i = 0; i < n; ++i) dsum += S.a.at(i, i);
    L.rho = dsum / (double)n;
    // ORACLE_RHO_ULPS=k moves rho by k ulps (perturbation experiments only;
    // any rho > 0 gives the same saddle solution in exact arithmetic)
    if (const char* e = std::getenv("ORACLE_RHO_ULPS"))
      for (int k = std::atoi(e); k != 0; k += k > 0 ? -1 : 1)
        L.rho = std::nextafter(L.rho, k > 0 ? HUGE_VAL : 0.0);
    std::vector<std::vector<std::pair<int, double>>> rows((size_t)n);
    for (int i = 0; i < n; ++i)
      for (int p = S.a.ptr[(size_t)i]; p < S.a.ptr[(size_t)i + 1]; ++p)
        rows[(size_t)i].emplace_back(S.a.col[(size_t)p], S.a.val[(size_t)p]);
    // ORACLE_K_CORNERS=1: augment with the corner rows only (K_c = A + rho
    // C_c^T C_c, the GPU's corner formulation; same saddle solutions in exact
    // arithmetic -- used to compare the GPU's K_c solves factor for factor)
    const bool corners_only = std::getenv("ORACLE_K_CORNERS") != nullptr;
    for (int r = 0; r < m; ++r)
      if (!corners_only || bd.coarse_objects[(size_t)L.coarse_ids[(size_t)r]].kind == kCorner)
      for (int p = L.c_ptr[(size_t)r]; p < L.c_ptr[(size_t)r + 1]; ++p)
        for (int q = L.c_ptr[(size_t)r]; q < L.c_ptr[(size_t)r + 1]; ++q) {
          const int i = L.c_col[(size_t)p], j = L.c_col[(size_t)q];
          const double v = L.rho * L.c_val[(size_t)p] * L.c_val[(size_t)q];
          bool found = false;
          for (auto& e : rows[(size_t)i])
            if (e.first == j) {
              e.second += v;
              found = true;
              break;
            }
          if (!found) rows[(size_t)i].emplace_back(j, v);
        }
    Csr kmat;
    kmat.n = n;
    kmat.ptr.assign((size_t)n + 1, 0);
    for (int i = 0; i < n; ++i) {
      std::sort(rows[(size_t)i].begin(), rows[(size_t)i].end());
      for (auto& e : rows[(size_t)i]) {
        kmat.col.push_back(e.first);
        kmat.val.push_back(e.second);
      }
      kmat.ptr[(size_t)i + 1] = (int)kmat.col.size();
    }
    std::vector<int> all((size_t)n);
    for (int i = 0; i < n; ++i) all[(size_t)i] = i;
    try {
      L.k.factor(kmat, local_coords(pb, S, all));
    } catch (const Error& e) {
      fail(ErrorCode::Singular, std::string("saddle: singular augmented system (subdomain ") + std::to_string(s) +
                                    "); constraints do not control the operator kernel: " + e.what());
    }
    // W = K^{-1} C^T, S = C W, Phi = W S^{-1}, A_c = Phi^T A Phi
    std::vector<double> wmat((size_t)n * m, 0.0);
    for (int r = 0; r < m; ++r) {
      double* col = &wmat[(size_t)r * n];
      for (int p = L.c_ptr[(size_t)r]; p < L.c_ptr[(size_t)r + 1]; ++p) col[L.c_col[(size_t)p]] += L.c_val[(size_t)p];
      L.k.solve(col);
    }
    std::vector<double> smat((size_t)m * m, 0.0);
    for (int r = 0; r < m; ++r)
      for (int c = 0; c < m; ++c) {
        double v = 0;
        for (int p = L.c_ptr[(size_t)r]; p < L.c_ptr[(size_t)r + 1]; ++p)
          v += L.c_val[(size_t)p] * wmat[(size_t)c * n + L.c_col[(size_t)p]];
        smat[(size_t)r * m + c] = v;
      }
    for (int r = 0; r < m; ++r)
      for (int c = r + 1; c < m; ++c) {
        const double v = 0.5 * (smat[(size_t)r * m + c] + smat[(size_t)c * m + r]);
        smat[(size_t)r * m + c] = v;
        smat[(size_t)c * m + r] = v;
      }
    L.phi.assign((size_t)n * m, 0.0);
    if (m > 0) {
      DenseCholesky sc;
      sc.factor(smat, m, "constraint Schur complement of subdomain " + std::to_string(s));
      std::vector<double> row((size_t)m);
      for (int i = 0; i < n; ++i) {
        for (int c = 0; c < m; ++c) row[(size_t)c] = wmat[(size_t)c * n + i];
        sc.solve(row.data());
        for (int c = 0; c < m; ++c) L.phi[(size_t)c * n + i] = row[(size_t)c];
      }
    }
    std::vector<double> aphi((size_t)n);
    L.ac.assign((size_t)m * m, 0.0);
    for (int c = 0; c < m; ++c) {
      S.a.spmv(&L.phi[(size_t)c * n], aphi.data());
      for (int r = 0; r < m; ++r) L.ac[(size_t)r * m + c] = dot(n, &L.phi[(size_t)r * n], aphi.data());
    }
    for (int r = 0; r < m; ++r)
      for (int c = r + 1; c < m; ++c) {
        const double v = 0.5 * (L.ac[(size_t)r * m + c] + L.ac[(size_t)c * m + r]);
        L.ac[(size_t)r * m + c] = v;
        L.ac[(size_t)c * m + r] = v;
      }
  });
  // coarse matrix
  const int nc = bd.n_coarse;
  bd.acoarse.assign((size_t)nc * nc, 0.0);
  for (int s = 0; s < nsd; ++s) {
    const auto& L = bd.loc[(size_t)s];
    const int m = (int)L.coarse_ids.size();
    for (int r = 0; r < m; ++r)
      for (int c = 0; c < m; ++c)
        bd.acoarse[(size_t)L.coarse_ids[(size_t)r] * nc + L.coarse_ids[(size_t)c]] += L.ac[(size_t)r * m + c];
  }
  if (nc > 0) bd.acoarse_chol.factor(bd.acoarse, nc, "coarse matrix");
}

void bddc_apply(const Problem& pb, const Bddc& bd, const double* r, double* z) {
  const int n = pb.mesh.n_dof;
  const int nsd = (int)pb.sd.size();
  // z0 = I0 A0^{-1} I0^T r
  std::vector<double> z0((size_t)n, 0.0);
  parallel_for(nsd, [&](std::int64_t s) {
    const auto& S = pb.sd[(size_t)s];
    const auto& L = bd.loc[(size_t)s];
    if (!L.has_interior) return;
    std::vector<double> t(L.interior_local.size());
    for (size_t k = 0; k < t.size(); ++k) t[k] = r[S.l2g[(size_t)L.interior_local[k]]];
    L.a_ii.solve(t.data());
    for (size_t k = 0; k < t.size(); ++k) z0[(size_t)S.l2g[(size_t)L.interior_local[k]]] = t[k];
  });
  // r1 = r - Abar z0 on interface rows, 0 on interior rows
  std::vector<double> r1((size_t)n, 0.0);
  for (int i = 0; i < n; ++i) {
    if (pb.neigh[(size_t)i].size() < 2) continue;
    double s = 0;
    for (int p = pb.abar.ptr[(size_t)i]; p < pb.abar.ptr[(size_t)i + 1]; ++p)
      s += pb.abar.val[(size_t)p] * z0[(size_t)pb.abar.col[(size_t)p]];
    r1[(size_t)i] = r[i] - s;
  }
  // local saddle solves + coarse rhs
  std::vector<std::vector<double>> zt((size_t)nsd), gl((size_t)nsd), yl((size_t)nsd);
  parallel_for(nsd, [&](std::int64_t s) {
    const auto& S = pb.sd[(size_t)s];
    const auto& L = bd.loc[(size_t)s];
    const int nl = (int)S.l2g.size();
    const int m = (int)L.coarse_ids.size();
    std::vector<double> rl((size_t)nl);
    for (int i = 0; i < nl; ++i) rl[(size_t)i] = bd.w[(size_t)s][(size_t)i] * r1[(size_t)S.l2g[(size_t)i]];
    gl[(size_t)s].assign((size_t)m, 0.0);
    for (int c = 0; c < m; ++c) gl[(size_t)s][(size_t)c] = dot(nl, &L.phi[(size_t)c * nl], rl.data());
    std::vector<double> y = rl;
    L.k.solve(y.data());
    std::vector<double> cy((size_t)m, 0.0);
    for (int c = 0; c < m; ++c)
      for (int p = L.c_ptr[(size_t)c]; p < L.c_ptr[(size_t)c + 1]; ++p)
        cy[(size_t)c] += L.c_val[(size_t)p] * y[(size_t)L.c_col[(size_t)p]];
    yl[(size_t)s] = std::move(y);
    zt[(size_t)s] = std::move(cy);
  });
  std::vector<double> zc((size_t)bd.n_coarse, 0.0);
  for (int s = 0; s < nsd; ++s) {
    const auto& L = bd.loc[(size_t)s];
    for (size_t c = 0; c < L.coarse_ids.size(); ++c) zc[(size_t)L.coarse_ids[c]] += gl[(size_t)s][c];
  }
  if (bd.n_coarse > 0) bd.acoarse_chol.solve(zc.data());
  // z~ = y + Phi (R_c z_c - C y); v = sum R^T (w . z~)
  std::vector<double> v((size_t)n, 0.0);
  for (int s = 0; s < nsd; ++s) {
    const auto& S = pb.sd[(size_t)s];
    const auto& L = bd.loc[(size_t)s];
    const int nl = (int)S.l2g.size();
    const int m = (int)L.coarse_ids.size();
    std::vector<double>& y = yl[(size_t)s];
    for (int c = 0; c < m; ++c) {
      const double coef = zc[(size_t)L.coarse_ids[(size_t)c]] - zt[(size_t)s][(size_t)c];
      const double* ph = &L.phi[(size_t)c * nl];
      for (int i = 0; i < nl; ++i) y[(size_t)i] += ph[i] * coef;
    }
    for (int i = 0; i < nl; ++i) v[(size_t)S.l2g[(size_t)i]] += bd.w[(size_t)s][(size_t)i] * y[(size_t)i];
  }
  // harmonic extension: v -= I0 A0^{-1} I0^T (Abar v)
  std::vector<double> av((size_t)n, 0.0);
  for (int i = 0; i < n; ++i) {
    if (pb.neigh[(size_t)i].size() != 1) continue;
    double s = 0;
    for (int p = pb.abar.ptr[(size_t)i]; p < pb.abar.ptr[(size_t)i + 1]; ++p)
      s += pb.abar.val[(size_t)p] * v[(size_t)pb.abar.col[(size_t)p]];
    av[(size_t)i] = s;
  }
  parallel_for(nsd, [&](std::int64_t s) {
    const auto& S = pb.sd[(size_t)s];
    const auto& L = bd.loc[(size_t)s];
    if (!L.has_interior) return;
    std::vector<double> t(L.interior_local.size());
    for (size_t k = 0; k < t.size(); ++k) t[k] = av[(size_t)S.l2g[(size_t)L.interior_local[k]]];
    L.a_ii.solve(t.data());
    for (size_t k = 0; k < t.size(); ++k) v[(size_t)S.l2g[(size_t)L.interior_local[k]]] -= t[k];
  });
  for (int i = 0; i < n; ++i) z[i] = z0[(size_t)i] + v[(size_t)i];
}

// extreme eigenvalues of the CG Lanczos tridiagonal
// T_ii = 1/alpha_i + beta_{i-1}/alpha_{i-1}, T_{i,i+1} = sqrt(beta_i)/alpha_i,
// by Sturm-sequence bisection.
bool condition_estimate(const std::vector<double>& alpha, const std::vector<double>& beta, double& lmin,
                        double& lmax) {
  const int k = (int)alpha.size();
  if (k < 2) return false;
  std::vector<double> d((size_t)k), e((size_t)k, 0.0);
  for (int i = 0; i < k; ++i) {
    d[(size_t)i] = 1.0 / alpha[(size_t)i] + (i > 0 ? beta[(size_t)i - 1] / alpha[(size_t)i - 1] : 0.0);
    if (i + 1 < k) e[(size_t)i] = std::sqrt(beta[(size_t)i]) / alpha[(size_t)i];
  }
  double lo = 1e300, hi = -1e300;
  for (int i = 0; i < k; ++i) {
    const double r = (i > 0 ? std::fabs(e[(size_t)i - 1]) : 0.0) + (i + 1 < k ? std::fabs(e[(size_t)i]) : 0.0);
    lo = std::min(lo, d[(size_t)i] - r);
    hi = std::max(hi, d[(size_t)i] + r);
  }
  auto count_below = [&](double x) {
    int c = 0;
    double q = d[0] - x;
    if (q < 0) ++c;
    for (int i = 1; i < k; ++i) {
      const double qq = q == 0.0 ? 1e-300 : q;
      q = d[(size_t)i] - x - e[(size_t)i - 1] * e[(size_t)i - 1] / qq;
      if (q < 0) ++c;
    }
    return c;
  };
  auto kth = [&](int idx) {
    double a = lo, b = hi;
    for (int it = 0; it < 200; ++it) {
      const double mid = 0.5 * (a + b);
      if (count_below(mid) > idx)
        b = mid;
      else
        a = mid;
    }
    return 0.5 * (a + b);
  };
  lmin = kth(0);
  lmax = kth(k - 1);
  return true;
}

}  // namespace oracle
