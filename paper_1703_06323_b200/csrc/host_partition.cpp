// host_partition.cpp — caller-side partition and interface objects.
//
// The reference computes these once on the host ("Object
// classification single-threaded (cheap, runs once)"); the GPU path only
// consumes the resulting index maps. Reference ops:
//   build_partition   SPEC.md:295-303 (block aggregation, empty blocks dropped)
//   classify_objects  SPEC.md:304-312 (exact neigh set + connected components
//                     over active FE edges, BackgroundMesh::edge_active
//                     mesh.cpp:74-108; Corner/Edge/Face)
//   split_edges_v1
//   split_edges_v2
// Pinned rules shared with the oracle: objects
// ordered by smallest global dof, nodes ascending; singletons -> Corner;
// strong-Dirichlet (orphan) dofs excluded.
#include <algorithm>
#include <array>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <mutex>
#include <numeric>
#include <thread>
#include <string>
#include <vector>

#include "cutbddc.h"
#include "status.hpp"

namespace cutbddc_b200 {
namespace {

struct Lattice {
  int n;
  const uint8_t* cls;
  const int32_t* dof_of_node;
  int64_t node(int i, int j, int k) const { return ((int64_t)i * (n + 1) + j) * (n + 1) + k; }
  int64_t cell(int i, int j, int k) const { return ((int64_t)i * n + j) * n + k; }
  void node_ijk(int64_t v, int c[3]) const {
    c[2] = (int)(v % (n + 1));
    c[1] = (int)((v / (n + 1)) % (n + 1));
    c[0] = (int)(v / (n + 1) / (n + 1));
  }
  // mesh.cpp:74-108 for axis-aligned unit lattice edges from node c along +axis.
  bool edge_active(const int c[3], int axis) const {
    const int o1 = axis == 0 ? 1 : 0, o2 = axis == 2 ? 1 : 2;
    for (int da = -1; da <= 0; ++da)
      for (int db = -1; db <= 0; ++db) {
        int cc[3] = {c[0], c[1], c[2]};
        cc[o1] += da;
        cc[o2] += db;
        bool ok = true;
        for (int d = 0; d < 3; ++d) ok = ok && cc[d] >= 0 && cc[d] < n;
        if (ok && cls[cell(cc[0], cc[1], cc[2])] != CUTBDDC_EXTERIOR) return true;
      }
    return false;
  }
};

// Static partition of [0, n) over up to 16 host threads (results do not
// depend on the thread count: every index writes only its own outputs).
template <typename F>
void parallel_for(int64_t n, F&& f) {
  static const int hw = [] {
    const char* e = std::getenv("CUTBDDC_HOST_THREADS");
    const int v = e ? std::atoi(e) : 0;
    return v > 0 ? v : (int)std::min<unsigned>(16u, std::max(1u, std::thread::hardware_concurrency()));
  }();
  const int nt = (int)std::min<int64_t>(hw, std::max<int64_t>(1, n / 4));
  if (nt <= 1) {
    for (int64_t i = 0; i < n; ++i) f(i);
    return;
  }
  std::vector<std::thread> th;
  std::exception_ptr err;
  std::mutex mu;
  for (int t = 0; t < nt; ++t)
    th.emplace_back([&, t] {
      try {
        for (int64_t i = n * t / nt; i < n * (t + 1) / nt; ++i) f(i);
      } catch (...) {
        std::lock_guard<std::mutex> g(mu);
        if (!err) err = std::current_exception();
      }
    });
  for (auto& x : th) x.join();
  if (err) std::rethrow_exception(err);
}

struct Obj {
  int kind;
  std::vector<int32_t> dofs;
  std::vector<int32_t> neigh;
};

// Union-find over positions 0..n-1.
struct UF {
  std::vector<int> p;
  explicit UF(int n) : p((size_t)n) { std::iota(p.begin(), p.end(), 0); }
  int f(int x) {
    while (p[(size_t)x] != x) x = p[(size_t)x] = p[(size_t)p[(size_t)x]];
    return x;
  }
  void u(int a, int b) {
    a = f(a);
    b = f(b);
    if (a != b) p[(size_t)std::max(a, b)] = std::min(a, b);
  }
};

// Connected components of `members` (sorted dofs) over active +axis lattice
// edges accepted by `join`. Components sorted internally; returned in order
// of their smallest member.
template <typename J>
std::vector<std::vector<int32_t>> components(const Lattice& L, const std::vector<int64_t>& node_of_dof,
                                             const std::vector<int32_t>& members, J&& join) {
  UF uf((int)members.size());
  for (size_t i = 0; i < members.size(); ++i) {
    int c[3];
    L.node_ijk(node_of_dof[(size_t)members[i]], c);
    for (int ax = 0; ax < 3; ++ax) {
      if (c[ax] + 1 > L.n) continue;
      int cc[3] = {c[0], c[1], c[2]};
      cc[ax] += 1;
      const int32_t d2 = L.dof_of_node[L.node(cc[0], cc[1], cc[2])];
      if (d2 < 0) continue;
      auto it = std::lower_bound(members.begin(), members.end(), d2);
      if (it == members.end() || *it != d2) continue;
      if (!L.edge_active(c, ax)) continue;
      if (!join(members[i], d2)) continue;
      uf.u((int)i, (int)(it - members.begin()));
    }
  }
  std::vector<std::vector<int32_t>> comps;
  std::vector<int> root_slot(members.size(), -1);
  for (size_t i = 0; i < members.size(); ++i) {  // members ascending -> components by smallest member
    const int r = uf.f((int)i);
    if (root_slot[(size_t)r] < 0) {
      root_slot[(size_t)r] = (int)comps.size();
      comps.emplace_back();
    }
    comps[(size_t)root_slot[(size_t)r]].push_back(members[i]);
  }
  return comps;
}

void check_mesh(const cutbddc_mesh_view* m) {
  if (!m || !m->cls || !m->dof_of_node) throw Failure(CUTBDDC_INVALID_ARGUMENT, "mesh view: null arrays");
  if (m->cells[0] != m->cells[1] || m->cells[1] != m->cells[2])
    throw Failure(CUTBDDC_INVALID_ARGUMENT, "mesh view: only cubic cell counts are supported");
}

}  // namespace
}  // namespace cutbddc_b200

using namespace cutbddc_b200;

extern "C" cutbddc_status cutbddc_build_partition(const cutbddc_mesh_view* mesh, int block, int64_t* n_sd,
                                                  int64_t* block_ids) {
  return guard([&] {
    check_mesh(mesh);
    const int n = mesh->cells[0];
    if (block < 1 || n % block != 0) throw Failure(CUTBDDC_INVALID_ARGUMENT, "partition: mesh dims not divisible by H/h");
    const int nb = n / block;
    std::vector<uint8_t> used((size_t)nb * nb * nb, 0);
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j)
        for (int k = 0; k < n; ++k)
          if (mesh->cls[((int64_t)i * n + j) * n + k] != CUTBDDC_EXTERIOR)
            used[((size_t)(i / block) * nb + j / block) * nb + k / block] = 1;
    int64_t c = 0;
    for (size_t b = 0; b < used.size(); ++b)
      if (used[b]) {
        if (block_ids) block_ids[c] = (int64_t)b;
        ++c;
      }
    *n_sd = c;
  });
}

extern "C" cutbddc_status cutbddc_classify_objects(const cutbddc_mesh_view* mesh, const cutbddc_partition_view* part,
                                                   const uint8_t* dirichlet, int objects, int variant,
                                                   const double* local_diag, cutbddc_objects** out) {
  return guard([&] {
    check_mesh(mesh);
    const int n = mesh->cells[0];
    const int B = part->block;
    const int nb = n / B;
    const int64_t ndof = mesh->n_dof;
    Lattice L{n, mesh->cls, mesh->dof_of_node};
    // local dofs of every subdomain (in parallel): nodes of its active
    // cells, ascending global dof (mark the 8 nodes of every active cell,
    // then scan the lattice; lexicographic slot order == ascending dof)
    std::vector<int64_t> node_of_dof((size_t)ndof, -1);
    std::vector<std::vector<int32_t>> sd_dofs((size_t)part->n_sd);
    std::vector<std::vector<int64_t>> sd_nodes((size_t)part->n_sd);
    const int b1 = B + 1;
    parallel_for(part->n_sd, [&](int64_t s) {
      std::vector<uint8_t> act((size_t)b1 * b1 * b1, 0);
      const int64_t b = part->block_ids[s];
      const int bi = (int)(b / nb / nb), bj = (int)((b / nb) % nb), bk = (int)(b % nb);
      auto& dl = sd_dofs[(size_t)s];
      auto& nl = sd_nodes[(size_t)s];
      for (int ci = 0; ci < B; ++ci)
        for (int cj = 0; cj < B; ++cj) {
          const uint8_t* row = mesh->cls + L.cell(bi * B + ci, bj * B + cj, bk * B);
          for (int ck = 0; ck < B; ++ck) {
            if (row[ck] == CUTBDDC_EXTERIOR) continue;
            uint8_t* a = act.data() + ((size_t)ci * b1 + cj) * b1 + ck;
            a[0] = a[1] = a[b1] = a[b1 + 1] = 1;
            a[b1 * b1] = a[b1 * b1 + 1] = a[b1 * b1 + b1] = a[b1 * b1 + b1 + 1] = 1;
          }
        }
      for (int li = 0; li <= B; ++li)
        for (int lj = 0; lj <= B; ++lj) {
          const uint8_t* a = act.data() + ((size_t)li * b1 + lj) * b1;
          const int64_t v0 = L.node(bi * B + li, bj * B + lj, bk * B);
          for (int lk = 0; lk <= B; ++lk)
            if (a[lk]) {
              const int32_t d = mesh->dof_of_node[v0 + lk];
              if (d < 0 || d >= ndof) throw Failure(CUTBDDC_INVALID_ARGUMENT, "mesh view: active node without a dof");
              dl.push_back(d);
              nl.push_back(v0 + lk);
            }
        }
    });
    // neigh sets: subdomains (ascending) holding each dof; local copies in
    // (subdomain, ascending dof) order for the weights.
    std::vector<uint8_t> nn_count((size_t)ndof, 0);
    std::vector<int32_t> neigh8((size_t)ndof * 8, -1);
    std::vector<int64_t> copy_off((size_t)part->n_sd + 1, 0);   // copies per subdomain
    for (int s = 0; s < part->n_sd; ++s) {
      const auto& dl = sd_dofs[(size_t)s];
      for (size_t q = 0; q < dl.size(); ++q) {
        const int32_t d = dl[q];
        node_of_dof[(size_t)d] = sd_nodes[(size_t)s][q];
        const uint8_t k = nn_count[(size_t)d]++;
        if (k >= 8) throw Failure(CUTBDDC_INTERNAL, "partition: node in more than 8 subdomains");
        neigh8[(size_t)d * 8 + k] = s;
      }
      copy_off[(size_t)s + 1] = copy_off[(size_t)s] + (int64_t)sd_dofs[(size_t)s].size();
    }
    // group interface dofs by exact neigh set (hash-sorted; objects are
    // ordered by their smallest dof below, so group order does not matter)
    auto same_key = [&](int32_t a, int32_t b) {
      const int k = nn_count[(size_t)a];
      return nn_count[(size_t)b] == k &&
             std::memcmp(&neigh8[(size_t)a * 8], &neigh8[(size_t)b * 8], sizeof(int32_t) * (size_t)k) == 0;
    };
    std::vector<std::pair<uint64_t, int32_t>> hk;  // (hash of the neigh set, dof)
    for (int64_t d = 0; d < ndof; ++d) {
      const int k = nn_count[(size_t)d];
      if (k < 2 || (dirichlet && dirichlet[d])) continue;
      uint64_t h = 1469598103934665603ull ^ (uint64_t)k;
      for (int q = 0; q < k; ++q) h = (h ^ (uint64_t)(uint32_t)neigh8[(size_t)d * 8 + q]) * 1099511628211ull;
      hk.emplace_back(h, (int32_t)d);
    }
    std::sort(hk.begin(), hk.end());
    std::vector<std::vector<int32_t>> group_dofs, group_key;
    for (size_t q0 = 0; q0 < hk.size();) {
      size_t q1 = q0 + 1;
      while (q1 < hk.size() && hk[q1].first == hk[q0].first) ++q1;
      // one hash run: split by exact key (a collision yields several groups)
      const size_t g0 = group_dofs.size();
      for (size_t q = q0; q < q1; ++q) {
        const int32_t d = hk[q].second;
        size_t g = g0;
        while (g < group_dofs.size() && !same_key(group_dofs[g][0], d)) ++g;
        if (g == group_dofs.size()) {
          group_dofs.emplace_back();
          group_key.emplace_back(neigh8.begin() + (int64_t)d * 8, neigh8.begin() + (int64_t)d * 8 + nn_count[(size_t)d]);
        }
        group_dofs[g].push_back(d);  // ascending dof within a group
      }
      q0 = q1;
    }
    std::vector<std::vector<std::vector<int32_t>>> gcomp(group_dofs.size());
    parallel_for((int64_t)group_dofs.size(), [&](int64_t g) {
      gcomp[(size_t)g] = components(L, node_of_dof, group_dofs[(size_t)g], [](int32_t, int32_t) { return true; });
    });
    std::vector<Obj> objs;
    for (size_t g = 0; g < group_dofs.size(); ++g) {
      for (auto& comp : gcomp[g]) {
        Obj o;
        o.kind = comp.size() == 1 ? CUTBDDC_CORNER : (group_key[g].size() == 2 ? CUTBDDC_FACE : CUTBDDC_EDGE);
        o.dofs = std::move(comp);
        o.neigh = group_key[g];
        objs.push_back(std::move(o));
      }
    }
    // variants split coarse edges only
    if (variant == CUTBDDC_VARIANT_V1 || variant == CUTBDDC_VARIANT_V2) {
      if (variant == CUTBDDC_VARIANT_V1 && !mesh->phi)
        throw Failure(CUTBDDC_INVALID_ARGUMENT, "split_edges_v1 needs node phi");
      if (variant == CUTBDDC_VARIANT_V2 && !local_diag)
        throw Failure(CUTBDDC_INVALID_ARGUMENT, "split_edges_v2 needs the local diagonals");
      // stiffness weight tuple of a dof: A^w_xixi / sum over its subdomains
      auto local_index = [&](int32_t s, int32_t d) {
        const auto& dl = sd_dofs[(size_t)s];
        return copy_off[(size_t)s] + (std::lower_bound(dl.begin(), dl.end(), d) - dl.begin());
      };
      auto weights = [&](int32_t d, double* w) {
        const int k = nn_count[(size_t)d];
        double tot = 0;
        for (int q = 0; q < k; ++q) tot += local_diag[local_index(neigh8[(size_t)d * 8 + q], d)];
        for (int q = 0; q < k; ++q) w[q] = local_diag[local_index(neigh8[(size_t)d * 8 + q], d)] / tot;
      };
      std::vector<Obj> split;
      for (auto& o : objs) {
        if (o.kind != CUTBDDC_EDGE) {
          split.push_back(std::move(o));
          continue;
        }
        std::vector<std::vector<int32_t>> parts;
        if (variant == CUTBDDC_VARIANT_V1) {
          auto phi_of = [&](int32_t d) { return mesh->phi[node_of_dof[(size_t)d]]; };
          std::vector<int32_t> cutnodes;
          components(L, node_of_dof, o.dofs, [&](int32_t a, int32_t b) {
            if ((phi_of(a) < 0) != (phi_of(b) < 0)) {
              cutnodes.push_back(a);
              cutnodes.push_back(b);
            }
            return true;
          });
          std::sort(cutnodes.begin(), cutnodes.end());
          cutnodes.erase(std::unique(cutnodes.begin(), cutnodes.end()), cutnodes.end());
          std::vector<int32_t> rest;
          for (int32_t d : o.dofs)
            if (!std::binary_search(cutnodes.begin(), cutnodes.end(), d))
              rest.push_back(d);
            else
              parts.push_back({d});
          if (!rest.empty())
            for (auto& c : components(L, node_of_dof, rest, [](int32_t, int32_t) { return true; })) parts.push_back(c);
        } else {
          const double tol = 1e-8;
          for (auto& c : components(L, node_of_dof, o.dofs, [&](int32_t a, int32_t b) {
                 double wa[8], wb[8];
                 weights(a, wa);
                 weights(b, wb);
                 for (int q = 0; q < nn_count[(size_t)a]; ++q) {
                   const double scale = std::max(1.0, std::max(std::fabs(wa[q]), std::fabs(wb[q])));
                   if (std::fabs(wa[q] - wb[q]) > tol * scale) return false;
                 }
                 return true;
               }))
            parts.push_back(c);
        }
        for (auto& p : parts) {
          Obj e;
          e.kind = p.size() >= 2 ? CUTBDDC_EDGE : CUTBDDC_CORNER;
          e.dofs = std::move(p);
          e.neigh = o.neigh;
          split.push_back(std::move(e));
        }
      }
      objs = std::move(split);
    }
    std::vector<Obj> sel;
    for (auto& o : objs) {
      const bool keep = o.kind == CUTBDDC_CORNER || (o.kind == CUTBDDC_EDGE && objects >= CUTBDDC_OBJECTS_CE) ||
                        (o.kind == CUTBDDC_FACE && objects >= CUTBDDC_OBJECTS_CEF);
      if (keep) sel.push_back(std::move(o));
    }
    std::sort(sel.begin(), sel.end(), [](const Obj& a, const Obj& b) { return a.dofs[0] < b.dofs[0]; });
    auto* r = new cutbddc_objects{};
    r->n_sd = part->n_sd;
    r->block_ids = new int64_t[(size_t)part->n_sd];
    std::memcpy(r->block_ids, part->block_ids, sizeof(int64_t) * (size_t)part->n_sd);
    r->n_objects = (int)sel.size();
    r->kinds = new int32_t[sel.size()];
    r->dof_ptr = new int64_t[sel.size() + 1];
    r->neigh_ptr = new int64_t[sel.size() + 1];
    int64_t nd = 0, nn = 0;
    for (auto& o : sel) {
      nd += (int64_t)o.dofs.size();
      nn += (int64_t)o.neigh.size();
    }
    r->dofs = new int32_t[(size_t)nd + 1];
    r->neigh = new int32_t[(size_t)nn + 1];
    r->dof_ptr[0] = r->neigh_ptr[0] = 0;
    for (size_t i = 0; i < sel.size(); ++i) {
      r->kinds[i] = sel[i].kind;
      std::copy(sel[i].dofs.begin(), sel[i].dofs.end(), r->dofs + r->dof_ptr[i]);
      std::copy(sel[i].neigh.begin(), sel[i].neigh.end(), r->neigh + r->neigh_ptr[i]);
      r->dof_ptr[i + 1] = r->dof_ptr[i] + (int64_t)sel[i].dofs.size();
      r->neigh_ptr[i + 1] = r->neigh_ptr[i] + (int64_t)sel[i].neigh.size();
    }
    *out = r;
  });
}

extern "C" void cutbddc_objects_free(cutbddc_objects* o) {
  if (!o) return;
  delete[] o->block_ids;
  delete[] o->kinds;
  delete[] o->dof_ptr;
  delete[] o->dofs;
  delete[] o->neigh_ptr;
  delete[] o->neigh;
  delete o;
}

// Multi-GPU assignment: nonempty subdomains ordered
// along a Morton curve over their block coordinates, cut into `world`
// contiguous chunks of (nearly) equal estimated cost. cost[s] may be NULL
// (unit cost). rank_of_sd[s] receives the rank of global subdomain s.
extern "C" cutbddc_status cutbddc_assign_subdomains(const cutbddc_partition_view* part, int cells, int world,
                                                    const double* cost, int32_t* rank_of_sd) {
  return guard([&] {
    if (!part || part->n_sd < 1 || world < 1) throw Failure(CUTBDDC_INVALID_ARGUMENT, "assign: empty partition");
    const int nb = cells / part->block;
    auto morton = [](uint32_t x, uint32_t y, uint32_t z) {
      uint64_t key = 0;
      for (int b = 0; b < 21; ++b) {
        key |= (uint64_t)((x >> b) & 1) << (3 * b + 2);
        key |= (uint64_t)((y >> b) & 1) << (3 * b + 1);
        key |= (uint64_t)((z >> b) & 1) << (3 * b);
      }
      return key;
    };
    std::vector<std::pair<uint64_t, int>> order;
    for (int s = 0; s < part->n_sd; ++s) {
      const int64_t b = part->block_ids[s];
      order.emplace_back(morton((uint32_t)(b / nb / nb), (uint32_t)((b / nb) % nb), (uint32_t)(b % nb)), s);
    }
    std::sort(order.begin(), order.end());
    double total = 0;
    for (int s = 0; s < part->n_sd; ++s) total += cost ? cost[s] : 1.0;
    double acc = 0;
    for (auto& [key, s] : order) {
      const double c = cost ? cost[s] : 1.0;
      // rank by the midpoint of this subdomain's cost interval
      int r = (int)((acc + 0.5 * c) / total * world);
      rank_of_sd[s] = std::min(world - 1, std::max(0, r));
      acc += c;
    }
  });
}

// Interface exchange plan of one rank, on the host: the same arrays, in the
// same order, as the device plan (dist.cu build_plan_device; compared entry
// for entry by tests/test_gpu_dist.py). Used by the multi-process CPU tests
// (tests/test_multigpu_gloo.py) to drive real exchanges with product lists.
extern "C" cutbddc_status cutbddc_build_exchange_plan(const cutbddc_mesh_view* mesh, const cutbddc_partition_view* part,
                                                      const int32_t* rank_of_sd, int rank, int world,
                                                      cutbddc_exchange_plan** out) {
  using namespace cutbddc_b200;
  return guard([&] {
    check_mesh(mesh);
    if (!part || !part->block_ids || part->n_sd < 1 || !rank_of_sd || !out)
      throw Failure(CUTBDDC_INVALID_ARGUMENT, "exchange plan: null argument");
    if (world < 1 || world > 32 || rank < 0 || rank >= world)
      throw Failure(CUTBDDC_INVALID_ARGUMENT, "exchange plan: rank / world out of range");
    const int n = mesh->cells[0], B = part->block;
    if (B < 1 || n % B) throw Failure(CUTBDDC_INVALID_ARGUMENT, "partition: mesh dims not divisible by H/h");
    const int nb = n / B, b1 = B + 1, T = b1 * b1 * b1, nsd_g = part->n_sd;
    Lattice L{n, mesh->cls, mesh->dof_of_node};
    std::vector<int32_t> gsd_of_block((size_t)nb * nb * nb, -1), lsd((size_t)nsd_g, -1);
    int nsd = 0;
    for (int g = 0; g < nsd_g; ++g) {
      gsd_of_block[(size_t)part->block_ids[g]] = g;
      if (rank_of_sd[g] < 0 || rank_of_sd[g] >= world) throw Failure(CUTBDDC_INVALID_ARGUMENT, "exchange plan: bad rank_of_sd");
      if (rank_of_sd[g] == rank) lsd[(size_t)g] = nsd++;
    }
    const int64_t nd = mesh->n_dof;
    std::vector<int64_t> node_of_dof((size_t)nd);
    for (int64_t v = 0; v < (int64_t)(n + 1) * (n + 1) * (n + 1); ++v)
      if (mesh->dof_of_node[v] >= 0) node_of_dof[(size_t)mesh->dof_of_node[v]] = v;
    // subdomains of every dof (ascending), local dofs
    std::vector<std::array<int32_t, 8>> sds((size_t)nd);
    std::vector<uint8_t> ns((size_t)nd);
    std::vector<int32_t> glist;
    for (int64_t d = 0; d < nd; ++d) {
      int c[3];
      L.node_ijk(node_of_dof[(size_t)d], c);
      int m = 0;
      std::array<int32_t, 8>& s = sds[(size_t)d];
      for (int dx = 0; dx < 2; ++dx)
        for (int dy = 0; dy < 2; ++dy)
          for (int dz = 0; dz < 2; ++dz) {
            const int ci = c[0] - 1 + dx, cj = c[1] - 1 + dy, ck = c[2] - 1 + dz;
            if (ci < 0 || cj < 0 || ck < 0 || ci >= n || cj >= n || ck >= n) continue;
            if (mesh->cls[L.cell(ci, cj, ck)] == CUTBDDC_EXTERIOR) continue;
            const int32_t g = gsd_of_block[((size_t)(ci / B) * nb + cj / B) * nb + ck / B];
            if (std::find(s.begin(), s.begin() + m, g) == s.begin() + m) s[(size_t)m++] = g;
          }
      std::sort(s.begin(), s.begin() + m);
      ns[(size_t)d] = (uint8_t)m;
      bool loc = false;
      for (int q = 0; q < m; ++q) loc |= rank_of_sd[s[(size_t)q]] == rank;
      if (loc) glist.push_back((int32_t)d);
    }
    const int64_t nloc = (int64_t)glist.size();
    auto seg = [&](int32_t d) {
      const int32_t g0 = sds[(size_t)d][0];
      return rank_of_sd[g0] == rank ? lsd[(size_t)g0] : nsd;
    };
    std::vector<int32_t> loc_glob(glist);
    std::stable_sort(loc_glob.begin(), loc_glob.end(), [&](int32_t a, int32_t b) { return seg(a) < seg(b); });
    std::vector<int32_t> seg_ptr((size_t)nsd + 1, 0), loc_of_dof((size_t)nd, -1);
    for (int64_t i = 0; i < nloc; ++i) loc_of_dof[(size_t)loc_glob[(size_t)i]] = (int32_t)i;
    for (int s2 = 0; s2 <= nsd; ++s2)
      seg_ptr[(size_t)s2] = (int32_t)(std::lower_bound(loc_glob.begin(), loc_glob.end(), s2,
                                                       [&](int32_t d, int key) { return seg(d) < key; }) -
                                      loc_glob.begin());
    auto count_rank = [&](int32_t d, int q) {
      int c = 0;
      for (int x = 0; x < ns[(size_t)d]; ++x) c += rank_of_sd[sds[(size_t)d][(size_t)x]] == q;
      return c;
    };
    std::vector<int32_t> nbr;
    std::vector<int> nbr_of_rank((size_t)world, -1);
    {
      std::vector<uint8_t> seen((size_t)world, 0);
      for (int32_t d : glist)
        for (int x = 0; x < ns[(size_t)d]; ++x) seen[(size_t)rank_of_sd[sds[(size_t)d][(size_t)x]]] = 1;
      for (int q = 0; q < world; ++q)
        if (q != rank && seen[(size_t)q]) {
          nbr_of_rank[(size_t)q] = (int)nbr.size();
          nbr.push_back(q);
        }
    }
    const int nn = (int)nbr.size();
    // message offsets of every dof (ascending global order)
    std::vector<int64_t> send_ptr(1, 0), recv_ptr(1, 0);
    std::vector<std::vector<int64_t>> roff((size_t)nn, std::vector<int64_t>((size_t)nloc)),
        soff((size_t)nn, std::vector<int64_t>((size_t)nloc));
    for (int k = 0; k < nn; ++k) {
      int64_t r = 0, sacc = 0;
      for (int64_t j = 0; j < nloc; ++j) {
        const int32_t d = glist[(size_t)j];
        const int cq = count_rank(d, nbr[(size_t)k]);
        roff[(size_t)k][(size_t)j] = r;
        soff[(size_t)k][(size_t)j] = sacc;
        r += cq;
        sacc += cq > 0 ? count_rank(d, rank) : 0;
      }
      recv_ptr.push_back(recv_ptr.back() + r);
      send_ptr.push_back(send_ptr.back() + sacc);
    }
    std::vector<int32_t> copy_ptr((size_t)nloc + 1, 0);
    for (int64_t i = 0; i < nloc; ++i) copy_ptr[(size_t)i + 1] = copy_ptr[(size_t)i] + ns[(size_t)loc_glob[(size_t)i]];
    std::vector<int32_t> copy_src((size_t)copy_ptr[(size_t)nloc]), send_src((size_t)send_ptr.back());
    for (int64_t j = 0; j < nloc; ++j) {
      const int32_t d = glist[(size_t)j];
      const int32_t i = loc_of_dof[(size_t)d];
      int c[3];
      L.node_ijk(node_of_dof[(size_t)d], c);
      std::vector<int> pos_q((size_t)world, 0);
      int32_t p = copy_ptr[(size_t)i];
      int mloc = 0;
      for (int x = 0; x < ns[(size_t)d]; ++x) {
        const int32_t g = sds[(size_t)d][(size_t)x];
        const int q = rank_of_sd[g];
        if (q == rank) {
          const int64_t bid = part->block_ids[g];
          const int bi = (int)(bid / nb / nb), bj = (int)((bid / nb) % nb), bk = (int)(bid % nb);
          const int32_t src = lsd[(size_t)g] * T + ((c[0] - bi * B) * b1 + (c[1] - bj * B)) * b1 + (c[2] - bk * B);
          copy_src[(size_t)p++] = src;
          for (int k = 0; k < nn; ++k)
            if (count_rank(d, nbr[(size_t)k]) > 0) send_src[(size_t)(send_ptr[(size_t)k] + soff[(size_t)k][(size_t)j] + mloc)] = src;
          ++mloc;
        } else {
          const int k = nbr_of_rank[(size_t)q];
          copy_src[(size_t)p++] = -1 - (int32_t)(recv_ptr[(size_t)k] + roff[(size_t)k][(size_t)j] + pos_q[(size_t)q]++);
        }
      }
    }
    auto* r = new cutbddc_exchange_plan();
    r->n_loc = nloc;
    r->n_own = seg_ptr[(size_t)nsd];
    r->n_sd_local = nsd;
    r->n_nbr = nn;
    auto dup32 = [](const std::vector<int32_t>& v) {
      auto* a = new int32_t[v.size() + 1];
      std::copy(v.begin(), v.end(), a);
      return a;
    };
    auto dup64 = [](const std::vector<int64_t>& v) {
      auto* a = new int64_t[v.size() + 1];
      std::copy(v.begin(), v.end(), a);
      return a;
    };
    r->loc_glob = dup32(loc_glob);
    r->seg_ptr = dup32(seg_ptr);
    r->copy_ptr = dup32(copy_ptr);
    r->copy_src = dup32(copy_src);
    r->nbr = dup32(nbr);
    r->send_ptr = dup64(send_ptr);
    r->send_src = dup32(send_src);
    r->recv_ptr = dup64(recv_ptr);
    *out = r;
  });
}
