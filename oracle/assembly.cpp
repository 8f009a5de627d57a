// assembly.cpp — global and sub-assembled operators (TEST INFRASTRUCTURE).
// SPEC.md:223-240 (assemble_global, assemble_subassembled); storage semantics
// of SparseSymMatrix::add/finalize (linalg.cpp:12-32: exact-zero adds skipped,
// duplicates merged, explicit zeros pruned, full symmetric copy kept).
// Partition: SPEC.md:295-303 (block aggregation, empty blocks dropped).
// Pins: subdomain ids = nonempty blocks in ascending block id
// ((bi*nby+bj)*nbz+bk); local dofs in ascending global dof; strong-Dirichlet
// ("orphan") dofs = dofs all of whose active cells are empty (Appendix B.1):
// Abar row/col -> identity, rhs 0; in every subdomain holding the dof the
// local diagonal is 1/|neigh|.
#include <algorithm>
#include <cmath>
#include <map>

#include "oracle.hpp"

namespace oracle {

void Csr::spmv(const double* x, double* y) const {
  for (int i = 0; i < n; ++i) {
    double s = 0;
    for (int p = ptr[i]; p < ptr[i + 1]; ++p) s += val[p] * x[col[p]];
    y[i] = s;
  }
}

double Csr::at(int i, int j) const {
  for (int p = ptr[i]; p < ptr[i + 1]; ++p)
    if (col[p] == j) return val[p];
  return 0.0;
}

namespace {

// Row-wise triplet accumulator (both mirror entries stored = full storage).
struct RowAcc {
  std::vector<std::vector<std::pair<int, double>>> rows;
  explicit RowAcc(int n) : rows((size_t)n) {}
  void add(int i, int j, double v) {
    if (v == 0.0) return;  // linalg.cpp:16
    auto& r = rows[(size_t)i];
    for (auto& e : r)
      if (e.first == j) {
        e.second += v;
        return;
      }
    r.emplace_back(j, v);
  }
  Csr finalize() {
    Csr c;
    c.n = (int)rows.size();
    c.ptr.assign((size_t)c.n + 1, 0);
    for (int i = 0; i < c.n; ++i) {
      auto& r = rows[(size_t)i];
      std::sort(r.begin(), r.end());
      for (auto& e : r)
        if (e.second != 0.0) {  // prune(0,0), linalg.cpp:27
          c.col.push_back(e.first);
          c.val.push_back(e.second);
        }
      c.ptr[(size_t)i + 1] = (int)c.col.size();
    }
    rows.clear();
    return c;
  }
};

}  // namespace

void build_problem(Problem& pb, int block) {
  const Mesh& m = pb.mesh;
  pb.block = block;
  for (int d = 0; d < 3; ++d) {
    if (block < 1 || m.n[d] % block != 0)
      fail(ErrorCode::InvalidArgument, "partition: mesh dims not divisible by H/h");
    pb.nb[d] = m.n[d] / block;
  }
  const std::int64_t na = (std::int64_t)m.active.size();
  // element contributions (parallel map)
  std::vector<Element> el((size_t)na);
  parallel_for(na, [&](std::int64_t a) { el[(size_t)a] = element_matrix(m, m.active[(size_t)a]); });
  pb.void_cell.assign((size_t)na, 0);
  pb.beta.assign((size_t)na, 0.0);
  for (std::int64_t a = 0; a < na; ++a) {
    pb.void_cell[(size_t)a] = el[(size_t)a].empty;
    pb.beta[(size_t)a] = el[(size_t)a].beta;
  }
  // blocks
  std::map<std::int64_t, int> block_to_sd;
  std::vector<std::int64_t> cell_block((size_t)na);
  for (std::int64_t a = 0; a < na; ++a) {
    int c[3];
    m.cell_coords(m.active[(size_t)a], c);
    const std::int64_t bid = ((std::int64_t)(c[0] / block) * pb.nb[1] + c[1] / block) * pb.nb[2] + c[2] / block;
    cell_block[(size_t)a] = bid;
    block_to_sd[bid] = 0;
  }
  pb.sd.clear();
  for (auto& kv : block_to_sd) {
    kv.second = (int)pb.sd.size();
    Subdomain s;
    s.block_id = kv.first;
    s.block[2] = (int)(kv.first % pb.nb[2]);
    s.block[1] = (int)((kv.first / pb.nb[2]) % pb.nb[1]);
    s.block[0] = (int)(kv.first / pb.nb[2] / pb.nb[1]);
    pb.sd.push_back(std::move(s));
  }
  std::vector<int> cell_sd((size_t)na);
  for (std::int64_t a = 0; a < na; ++a) {
    cell_sd[(size_t)a] = block_to_sd[cell_block[(size_t)a]];
    pb.sd[(size_t)cell_sd[(size_t)a]].cells.push_back(a);  // store active index
  }
  const int nsd = (int)pb.sd.size();
  // local dofs + neigh
  pb.neigh.assign((size_t)m.n_dof, {});
  std::vector<int> nonvoid_count((size_t)m.n_dof, 0);
  for (int s = 0; s < nsd; ++s) {
    auto& S = pb.sd[(size_t)s];
    std::vector<int> dofs;
    for (std::int64_t a : S.cells) {
      std::int64_t nodes[8];
      m.cell_nodes(m.active[(size_t)a], nodes);
      for (int l = 0; l < 8; ++l) {
        const int d = m.dof_of_node[(size_t)nodes[l]];
        dofs.push_back(d);
        if (!el[(size_t)a].empty) nonvoid_count[(size_t)d]++;
      }
    }
    std::sort(dofs.begin(), dofs.end());
    dofs.erase(std::unique(dofs.begin(), dofs.end()), dofs.end());
    S.l2g = dofs;
    for (int d : dofs) pb.neigh[(size_t)d].push_back(s);
  }
  pb.dirichlet.assign((size_t)m.n_dof, 0);
  for (int d = 0; d < m.n_dof; ++d) pb.dirichlet[(size_t)d] = nonvoid_count[(size_t)d] == 0;
  // sub-assembled matrices
  parallel_for(nsd, [&](std::int64_t s) {
    auto& S = pb.sd[(size_t)s];
    const int n = (int)S.l2g.size();
    RowAcc acc(n);
    S.f.assign((size_t)n, 0.0);
    auto loc = [&](int g) { return (int)(std::lower_bound(S.l2g.begin(), S.l2g.end(), g) - S.l2g.begin()); };
    for (std::int64_t a : S.cells) {
      const Element& e = el[(size_t)a];
      if (e.empty) continue;
      std::int64_t nodes[8];
      m.cell_nodes(m.active[(size_t)a], nodes);
      int li[8];
      for (int l = 0; l < 8; ++l) li[l] = loc(m.dof_of_node[(size_t)nodes[l]]);
      for (int x = 0; x < 8; ++x) {
        S.f[(size_t)li[x]] += e.f[x];
        for (int y = 0; y < 8; ++y) acc.add(li[x], li[y], e.k[x * 8 + y]);
      }
    }
    S.interior.assign((size_t)n, 0);
    for (int i = 0; i < n; ++i) {
      const int g = S.l2g[(size_t)i];
      S.interior[(size_t)i] = pb.neigh[(size_t)g].size() == 1;
      if (pb.dirichlet[(size_t)g]) acc.add(i, i, 1.0 / (double)pb.neigh[(size_t)g].size());
    }
    S.a = acc.finalize();
  });
  // global matrix straight from the elements
  RowAcc acc(m.n_dof);
  pb.b.assign((size_t)m.n_dof, 0.0);
  for (std::int64_t a = 0; a < na; ++a) {
    const Element& e = el[(size_t)a];
    if (e.empty) continue;
    std::int64_t nodes[8];
    m.cell_nodes(m.active[(size_t)a], nodes);
    int gi[8];
    for (int l = 0; l < 8; ++l) gi[l] = m.dof_of_node[(size_t)nodes[l]];
    for (int x = 0; x < 8; ++x) {
      pb.b[(size_t)gi[x]] += e.f[x];
      for (int y = 0; y < 8; ++y) acc.add(gi[x], gi[y], e.k[x * 8 + y]);
    }
  }
  for (int d = 0; d < m.n_dof; ++d)
    if (pb.dirichlet[(size_t)d]) acc.add(d, d, 1.0);  // symmetric elimination, g = 0
  pb.abar = acc.finalize();
}

}  // namespace oracle
