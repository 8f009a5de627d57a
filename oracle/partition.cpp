// partition.cpp — interface objects, edge-splitting variants, weighting
// (TEST INFRASTRUCTURE).
// SPEC.md:304-330 (classify_objects, split_edges_v1, split_edges_v2),
// SPEC.md:370-378 (build_weighting).
// Pins: node adjacency = lattice edge of an active
// cell (BackgroundMesh::edge_active, mesh.cpp:74-108);
// |neigh| = 2 multi-node component -> Face, |neigh| > 2 multi-node -> Edge,
// singletons -> Corner; objects ordered by smallest global dof, nodes
// ascending; strong-Dirichlet dofs excluded. Variant split
// components of >= 2 nodes -> Edge, singletons -> Corner.
#include <algorithm>
#include <cmath>
#include <functional>
#include <map>
#include <numeric>

#include "oracle.hpp"

namespace oracle {

namespace {

struct Dsu {
  std::vector<int> p;
  explicit Dsu(int n) : p((size_t)n) { std::iota(p.begin(), p.end(), 0); }
  int find(int x) {
    while (p[(size_t)x] != x) x = p[(size_t)x] = p[(size_t)p[(size_t)x]];
    return x;
  }
  void unite(int a, int b) {
    a = find(a);
    b = find(b);
    if (a != b) p[(size_t)std::max(a, b)] = std::min(a, b);
  }
};

// Lattice neighbours (6) of a dof's node that are dofs in `members` and share
// an active FE edge; `pred(a, b)` filters the pair further.
std::vector<std::vector<int>> components(const Problem& pb, const std::vector<int>& members,
                                         const std::function<bool(int, int)>& pred) {
  const Mesh& m = pb.mesh;
  std::map<int, int> idx;
  for (size_t i = 0; i < members.size(); ++i) idx[members[i]] = (int)i;
  Dsu dsu((int)members.size());
  for (size_t i = 0; i < members.size(); ++i) {
    const std::int64_t node = m.node_of_dof[(size_t)members[i]];
    int c[3];
    m.node_coords(node, c);
    for (int d = 0; d < 3; ++d) {
      int cc[3] = {c[0], c[1], c[2]};
      cc[d] += 1;
      if (cc[d] > m.n[d]) continue;
      const std::int64_t nb = m.node_id(cc[0], cc[1], cc[2]);
      const int dn = m.dof_of_node[(size_t)nb];
      if (dn < 0) continue;
      auto it = idx.find(dn);
      if (it == idx.end()) continue;
      if (!m.edge_active(node, nb)) continue;
      if (!pred(members[i], dn)) continue;
      dsu.unite((int)i, it->second);
    }
  }
  std::map<int, std::vector<int>> comp;
  for (size_t i = 0; i < members.size(); ++i) comp[dsu.find((int)i)].push_back(members[i]);
  std::vector<std::vector<int>> out;
  for (auto& kv : comp) {
    std::sort(kv.second.begin(), kv.second.end());
    out.push_back(kv.second);
  }
  return out;
}

void sort_objects(std::vector<Object>& objs) {
  std::sort(objs.begin(), objs.end(), [](const Object& a, const Object& b) { return a.dofs[0] < b.dofs[0]; });
}

}  // namespace

std::vector<Object> classify_objects(const Problem& pb) {
  std::map<std::vector<int>, std::vector<int>> groups;
  for (int d = 0; d < pb.mesh.n_dof; ++d) {
    if (pb.neigh[(size_t)d].size() < 2 || pb.dirichlet[(size_t)d]) continue;
    groups[pb.neigh[(size_t)d]].push_back(d);
  }
  std::vector<Object> objs;
  for (auto& kv : groups) {
    for (auto& comp : components(pb, kv.second, [](int, int) { return true; })) {
      Object o;
      o.neigh = kv.first;
      o.dofs = comp;
      if (comp.size() == 1)
        o.kind = kCorner;
      else
        o.kind = kv.first.size() == 2 ? kFace : kEdge;
      objs.push_back(std::move(o));
    }
  }
  sort_objects(objs);
  return objs;
}

// dofs on cut FE edges of a coarse edge
// become corners; the remaining nodes are aggregated into connected subedges
// over the uncut FE edges.
std::vector<Object> split_edges_v1(const Problem& pb, const std::vector<Object>& objs) {
  const Mesh& m = pb.mesh;
  auto phi_of = [&](int dof) { return m.phi[(size_t)m.node_of_dof[(size_t)dof]]; };
  std::vector<Object> out;
  for (const Object& o : objs) {
    if (o.kind != kEdge) {
      out.push_back(o);
      continue;
    }
    std::map<int, bool> on_cut;
    for (int d : o.dofs) on_cut[d] = false;
    // FE edges inside the object
    for (auto& comp : components(pb, o.dofs, [&](int a, int b) {
           const bool cut = (phi_of(a) < 0) != (phi_of(b) < 0);
           if (cut) {
             on_cut[a] = true;
             on_cut[b] = true;
           }
           return true;
         })) {
      (void)comp;
    }
    std::vector<int> rest;
    for (int d : o.dofs) {
      if (on_cut[d]) {
        Object c;
        c.kind = kCorner;
        c.dofs = {d};
        c.neigh = o.neigh;
        out.push_back(c);
      } else {
        rest.push_back(d);
      }
    }
    if (!rest.empty()) {
      for (auto& comp : components(pb, rest, [](int, int) { return true; })) {
        Object e;
        e.kind = comp.size() >= 2 ? kEdge : kCorner;
        e.dofs = comp;
        e.neigh = o.neigh;
        out.push_back(e);
      }
    }
  }
  sort_objects(out);
  return out;
}

// aggregate neighbour nodes on a coarse
// edge whose weight tuples (ordered by subdomain id) agree within rel_tol;
// un-aggregated nodes become corners.
std::vector<Object> split_edges_v2(const Problem& pb, const std::vector<Object>& objs,
                                   const std::vector<std::vector<double>>& w, double rel_tol) {
  auto tuple = [&](int dof) {
    std::vector<double> t;
    for (int s : pb.neigh[(size_t)dof]) {
      const auto& l2g = pb.sd[(size_t)s].l2g;
      const int li = (int)(std::lower_bound(l2g.begin(), l2g.end(), dof) - l2g.begin());
      t.push_back(w[(size_t)s][(size_t)li]);
    }
    return t;
  };
  std::vector<Object> out;
  for (const Object& o : objs) {
    if (o.kind != kEdge) {
      out.push_back(o);
      continue;
    }
    auto same = [&](int a, int b) {
      const auto ta = tuple(a), tb = tuple(b);
      for (size_t k = 0; k < ta.size(); ++k) {
        const double scale = std::max(1.0, std::max(std::fabs(ta[k]), std::fabs(tb[k])));
        if (std::fabs(ta[k] - tb[k]) > rel_tol * scale) return false;
      }
      return true;
    };
    for (auto& comp : components(pb, o.dofs, same)) {
      Object e;
      e.kind = comp.size() >= 2 ? kEdge : kCorner;
      e.dofs = comp;
      e.neigh = o.neigh;
      out.push_back(e);
    }
  }
  sort_objects(out);
  return out;
}

// SPEC.md:370-378; PAPER.md:420-423 (topological), :550-553 (stiffness).
std::vector<std::vector<double>> build_weighting(const Problem& pb, int mode) {
  const int nsd = (int)pb.sd.size();
  std::vector<double> total((size_t)pb.mesh.n_dof, 0.0);
  if (mode == kWeightStiffness) {
    for (int s = 0; s < nsd; ++s) {
      const auto& S = pb.sd[(size_t)s];
      for (size_t i = 0; i < S.l2g.size(); ++i) total[(size_t)S.l2g[i]] += S.a.at((int)i, (int)i);
    }
  }
  std::vector<std::vector<double>> w((size_t)nsd);
  for (int s = 0; s < nsd; ++s) {
    const auto& S = pb.sd[(size_t)s];
    w[(size_t)s].resize(S.l2g.size());
    for (size_t i = 0; i < S.l2g.size(); ++i) {
      const int g = S.l2g[i];
      const size_t k = pb.neigh[(size_t)g].size();
      if (k == 1) {
        w[(size_t)s][i] = 1.0;
      } else if (mode == kWeightTopological) {
        w[(size_t)s][i] = 1.0 / (double)k;
      } else {
        if (!(total[(size_t)g] != 0.0))
          fail(ErrorCode::Degenerate, "weighting: zero total diagonal at dof " + std::to_string(g));
        w[(size_t)s][i] = S.a.at((int)i, (int)i) / total[(size_t)g];
      }
    }
  }
  return w;
}

}  // namespace oracle
