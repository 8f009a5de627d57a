// capi.cpp — flat C entry points of the oracle for the ctypes harness
// (TEST INFRASTRUCTURE; loaded only by tests/, smoke() and bench.py's CPU legs).
#include <chrono>
#include <cstring>
#include <memory>
#include <string>

#include "oracle.hpp"

using namespace oracle;

namespace {
thread_local std::string g_err;

struct Handle {
  Problem pb;
  Bddc bd;
  bool has_bddc = false;
  double t_classify = 0, t_assembly = 0, t_setup = 0, t_pcg = 0;
};

double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

template <typename F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const Error& e) {
    g_err = e.what();
    return (int)e.code;
  } catch (const std::exception& e) {
    g_err = e.what();
    return (int)ErrorCode::Internal;
  }
}
}  // namespace

extern "C" {

struct orc_config {
  int cells[3];
  double lo[3], hi[3], translation[3];
  int block;
  int n_balls;
  const double* balls;  // 4 doubles per ball: cx, cy, cz, r
  int threads;
  int problem;          // 0: f = 1, g = 0; 1: manufactured u = sin(5 pi |x|)
};

const char* orc_last_error() { return g_err.c_str(); }

int orc_create(const orc_config* cfg, void** out) {
  return guard([&] {
    auto h = std::make_unique<Handle>();
    set_thread_count(cfg->threads);
    for (int d = 0; d < 3; ++d) {
      h->pb.params.cells[d] = cfg->cells[d];
      h->pb.params.lo[d] = cfg->lo[d];
      h->pb.params.hi[d] = cfg->hi[d];
      h->pb.params.translation[d] = cfg->translation[d];
    }
    for (int i = 0; i < cfg->n_balls; ++i)
      h->pb.geom.balls.push_back({cfg->balls[4 * i], cfg->balls[4 * i + 1], cfg->balls[4 * i + 2], cfg->balls[4 * i + 3]});
    double t0 = now();
    h->pb.mesh = classify(h->pb.params, h->pb.geom);
    h->pb.mesh.problem = cfg->problem;
    double t1 = now();
    h->t_classify = t1 - t0;
    if (cfg->block > 0) {
      build_problem(h->pb, cfg->block);
      h->pb.objects = classify_objects(h->pb);
    }
    h->t_assembly = now() - t1;
    *out = h.release();
  });
}

void orc_destroy(void* h) { delete static_cast<Handle*>(h); }

// info[0..]: n_dof, n_active, n_cut, n_interior_cells, n_sd, n_objects, n_corner,
// n_edge, n_face, n_dirichlet, n_void_cells, n_coarse, sum_local_dofs, max_local
int orc_info(void* hv, long long* info) {
  return guard([&] {
    auto* h = static_cast<Handle*>(hv);
    const auto& m = h->pb.mesh;
    long long ncut = 0, nint = 0;
    for (auto c : m.active) (m.cls[(size_t)c] == kCut ? ncut : nint)++;
    long long kinds[3] = {0, 0, 0};
    for (auto& o : h->pb.objects) kinds[o.kind]++;
    long long ndir = 0, nvoid = 0, sum = 0, mx = 0;
    for (char c : h->pb.dirichlet) ndir += c;
    for (char c : h->pb.void_cell) nvoid += c;
    for (auto& s : h->pb.sd) {
      sum += (long long)s.l2g.size();
      mx = std::max(mx, (long long)s.l2g.size());
    }
    info[0] = m.n_dof;
    info[1] = (long long)m.active.size();
    info[2] = ncut;
    info[3] = nint;
    info[4] = (long long)h->pb.sd.size();
    info[5] = (long long)h->pb.objects.size();
    info[6] = kinds[kCorner];
    info[7] = kinds[kEdge];
    info[8] = kinds[kFace];
    info[9] = ndir;
    info[10] = nvoid;
    info[11] = h->has_bddc ? h->bd.n_coarse : -1;
    info[12] = sum;
    info[13] = mx;
  });
}

int orc_times(void* hv, double* t) {
  auto* h = static_cast<Handle*>(hv);
  t[0] = h->t_classify;
  t[1] = h->t_assembly;
  t[2] = h->t_setup;
  t[3] = h->t_pcg;
  return 0;
}

int orc_mesh(void* hv, double* phi, unsigned char* cls, int* dof_of_node) {
  return guard([&] {
    auto* h = static_cast<Handle*>(hv);
    const auto& m = h->pb.mesh;
    if (phi) std::memcpy(phi, m.phi.data(), m.phi.size() * sizeof(double));
    if (cls) std::memcpy(cls, m.cls.data(), m.cls.size());
    if (dof_of_node) std::memcpy(dof_of_node, m.dof_of_node.data(), m.dof_of_node.size() * sizeof(int));
  });
}

// per active cell: beta and void flag
int orc_cells(void* hv, double* beta, unsigned char* void_cell) {
  return guard([&] {
    auto* h = static_cast<Handle*>(hv);
    for (size_t a = 0; a < h->pb.beta.size(); ++a) {
      if (beta) beta[a] = h->pb.beta[a];
      if (void_cell) void_cell[a] = (unsigned char)h->pb.void_cell[a];
    }
  });
}

int orc_dirichlet(void* hv, unsigned char* mask) {
  return guard([&] {
    auto* h = static_cast<Handle*>(hv);
    for (size_t i = 0; i < h->pb.dirichlet.size(); ++i) mask[i] = (unsigned char)h->pb.dirichlet[i];
  });
}

int orc_element(void* hv, long long cell, double* k, double* f, double* beta, int* empty) {
  return guard([&] {
    auto* h = static_cast<Handle*>(hv);
    Element e = element_matrix(h->pb.mesh, cell);
    std::memcpy(k, e.k, sizeof(e.k));
    std::memcpy(f, e.f, sizeof(e.f));
    *beta = e.beta;
    *empty = e.empty;
  });
}

// cut rule on the reference cell: returns counts, fills up to cap points.
int orc_cut_rule(const double* phiv, int full, double* vol, int vol_cap, double* surf, int surf_cap, int* counts) {
  return guard([&] {
    CutRule r = full ? full_quadrature_ref() : cut_quadrature_ref(phiv);
    counts[0] = (int)r.vol.size();
    counts[1] = (int)r.surf.size();
    counts[2] = r.dropped;
    for (int i = 0; i < (int)r.vol.size() && i < vol_cap; ++i) std::memcpy(vol + 4 * i, r.vol[(size_t)i].data(), 32);
    for (int i = 0; i < (int)r.surf.size() && i < surf_cap; ++i)
      std::memcpy(surf + 7 * i, r.surf[(size_t)i].data(), 56);
  });
}

int orc_gen_eigs(const double* b, const double* d, int n, double tol, double* out) {
  return guard([&] { *out = dense_generalized_eigs_max(b, d, n, tol); });
}

int orc_error_norms(void* hv, const double* x, double* out) {
  return guard([&] {
    auto* h = static_cast<Handle*>(hv);
    error_norms(h->pb.mesh, x, out, out + 1);
  });
}

int orc_rhs(void* hv, double* b) {
  return guard([&] {
    auto* h = static_cast<Handle*>(hv);
    std::memcpy(b, h->pb.b.data(), h->pb.b.size() * sizeof(double));
  });
}

int orc_spmv(void* hv, const double* x, double* y) {
  return guard([&] { static_cast<Handle*>(hv)->pb.abar.spmv(x, y); });
}

// global matrix in CSR
int orc_abar(void* hv, int* ptr, int* col, double* val, long long* nnz) {
  return guard([&] {
    auto* h = static_cast<Handle*>(hv);
    const auto& a = h->pb.abar;
    *nnz = (long long)a.val.size();
    if (ptr) std::memcpy(ptr, a.ptr.data(), a.ptr.size() * sizeof(int));
    if (col) std::memcpy(col, a.col.data(), a.col.size() * sizeof(int));
    if (val) std::memcpy(val, a.val.data(), a.val.size() * sizeof(double));
  });
}

// subdomain s: info[0]=n_local, info[1]=nnz, info[2..4]=block coords, info[5]=block id
int orc_subdomain_info(void* hv, int s, long long* info) {
  return guard([&] {
    auto* h = static_cast<Handle*>(hv);
    const auto& S = h->pb.sd.at((size_t)s);
    info[0] = (long long)S.l2g.size();
    info[1] = (long long)S.a.val.size();
    info[2] = S.block[0];
    info[3] = S.block[1];
    info[4] = S.block[2];
    info[5] = S.block_id;
  });
}

int orc_subdomain(void* hv, int s, int* l2g, int* ptr, int* col, double* val, double* f) {
  return guard([&] {
    auto* h = static_cast<Handle*>(hv);
    const auto& S = h->pb.sd.at((size_t)s);
    if (l2g) std::memcpy(l2g, S.l2g.data(), S.l2g.size() * sizeof(int));
    if (ptr) std::memcpy(ptr, S.a.ptr.data(), S.a.ptr.size() * sizeof(int));
    if (col) std::memcpy(col, S.a.col.data(), S.a.col.size() * sizeof(int));
    if (val) std::memcpy(val, S.a.val.data(), S.a.val.size() * sizeof(double));
    if (f) std::memcpy(f, S.f.data(), S.f.size() * sizeof(double));
  });
}

// objects flattened: kinds[n_obj], dof_ptr[n_obj+1], dofs[], neigh_ptr[n_obj+1], neigh[]
// which: 0 = standard objects, 1 = coarse (selected, post-variant) objects of the bddc
int orc_objects(void* hv, int which, int* n_obj, int* kinds, int* dof_ptr, int* dofs, int* neigh_ptr, int* neigh) {
  return guard([&] {
    auto* h = static_cast<Handle*>(hv);
    const auto& objs = which == 0 ? h->pb.objects : h->bd.coarse_objects;
    *n_obj = (int)objs.size();
    if (!kinds) return;
    int pd = 0, pn = 0;
    dof_ptr[0] = 0;
    neigh_ptr[0] = 0;
    for (size_t i = 0; i < objs.size(); ++i) {
      kinds[i] = objs[i].kind;
      for (int d : objs[i].dofs) dofs[pd++] = d;
      for (int s : objs[i].neigh) neigh[pn++] = s;
      dof_ptr[i + 1] = pd;
      neigh_ptr[i + 1] = pn;
    }
  });
}

int orc_setup(void* hv, int objects, int weighting, int variant) {
  return guard([&] {
    auto* h = static_cast<Handle*>(hv);
    double t0 = now();
    build_bddc(h->pb, h->bd, objects, weighting, variant);
    h->t_setup = now() - t0;
    h->has_bddc = true;
  });
}

// weights per subdomain concatenated in subdomain order
int orc_weights(void* hv, double* w) {
  return guard([&] {
    auto* h = static_cast<Handle*>(hv);
    size_t p = 0;
    for (auto& ws : h->bd.w)
      for (double v : ws) w[p++] = v;
  });
}

int orc_coarse_matrix(void* hv, double* ac) {
  return guard([&] {
    auto* h = static_cast<Handle*>(hv);
    std::memcpy(ac, h->bd.acoarse.data(), h->bd.acoarse.size() * sizeof(double));
  });
}

int orc_apply(void* hv, const double* r, double* z) {
  return guard([&] {
    auto* h = static_cast<Handle*>(hv);
    bddc_apply(h->pb, h->bd, r, z);
  });
}

// PCG with Abar and (precond ? BDDC : identity). out_i[0]=iterations,
// out_i[1]=converged; out_d[0]=cond, [1]=lmin, [2]=lmax; resid has
// max_iter+1 slots.
int orc_pcg(void* hv, const double* b, double rtol, int max_iter, int precond, double* x, double* resid, int* out_i,
            double* out_d) {
  return guard([&] {
    auto* h = static_cast<Handle*>(hv);
    const int n = h->pb.mesh.n_dof;
    SolveReport rep;
    double t0 = now();
    auto aapply = [&](const double* xx, double* yy) { h->pb.abar.spmv(xx, yy); };
    if (precond) {
      pcg(n, aapply, [&](const double* r, double* z) { bddc_apply(h->pb, h->bd, r, z); }, b, x, rtol, max_iter, rep);
    } else {
      pcg(n, aapply, [&](const double* r, double* z) { std::memcpy(z, r, sizeof(double) * n); }, b, x, rtol,
          max_iter, rep);
    }
    h->t_pcg = now() - t0;
    out_i[0] = rep.iterations;
    out_i[1] = rep.converged;
    out_d[0] = rep.cond;
    out_d[1] = rep.lmin;
    out_d[2] = rep.lmax;
    for (size_t i = 0; i < rep.residuals.size(); ++i) resid[i] = rep.residuals[i];
  });
}

// Local solve of subdomain s in its local dof order (ascending global dof):
// which = 0: A_II^{-1} on the interior dofs (x has n_local entries; only the
// interior ones are read and written, the rest are zeroed); which = 1: K^{-1}
// with K = A + rho C^T C (SparseCholesky::solve, linalg.cpp:58).
int orc_local_solve(void* hv, int s, int which, double* x) {
  return guard([&] {
    auto* h = static_cast<Handle*>(hv);
    if (!h->has_bddc) fail(ErrorCode::InvalidArgument, "setup first");
    const auto& L = h->bd.loc.at((size_t)s);
    const size_t n = h->pb.sd.at((size_t)s).l2g.size();
    if (which == 1) {
      L.k.solve(x);
      return;
    }
    std::vector<double> t(L.interior_local.size());
    for (size_t k = 0; k < t.size(); ++k) t[k] = x[L.interior_local[k]];
    if (L.has_interior) L.a_ii.solve(t.data());
    std::fill(x, x + n, 0.0);
    for (size_t k = 0; k < t.size(); ++k) x[L.interior_local[k]] = t[k];
  });
}

// standalone sparse Cholesky on a CSR matrix (for linalg known-answer tests)
int orc_cholesky_solve(int n, const int* ptr, const int* col, const double* val, double* x) {
  return guard([&] {
    Csr a;
    a.n = n;
    a.ptr.assign(ptr, ptr + n + 1);
    a.col.assign(col, col + ptr[n]);
    a.val.assign(val, val + ptr[n]);
    std::vector<std::array<int, 3>> xyz((size_t)n);
    for (int i = 0; i < n; ++i) xyz[(size_t)i] = {i, 0, 0};
    SparseCholesky c;
    c.factor(a, xyz);
    c.solve(x);
  });
}

int orc_condition_estimate(const double* alpha, const double* beta, int k, double* out) {
  return guard([&] {
    std::vector<double> a(alpha, alpha + k), b(beta, beta + (k > 0 ? k - 1 : 0));
    if (!condition_estimate(a, b, out[0], out[1])) fail(ErrorCode::InvalidArgument, "fewer than 2 iterations");
  });
}

}  // extern "C"
