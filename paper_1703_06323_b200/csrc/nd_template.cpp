// nd_template.cpp — see nd_template.hpp.
#include "nd_template.hpp"

#include <algorithm>
#include <stdexcept>

namespace cutbddc_b200 {
namespace {

struct Box {
  int lo[3], hi[3];  // half-open
  int count() const { return (hi[0] - lo[0]) * (hi[1] - lo[1]) * (hi[2] - lo[2]); }
};

struct Builder {
  Template& t;
  std::vector<std::vector<int32_t>> cols_of;  // temp per supernode
  std::vector<Box> box_of;
  explicit Builder(Template& tt) : t(tt) {}

  int slot(int x, int y, int z) const { return (x * t.b1 + y) * t.b1 + z; }

  // returns supernode id (postorder assigned on creation after children)
  int build(const Box& b, int level) {
    std::vector<int32_t> cols;
    int kids[2] = {-1, -1}, nk = 0;
    if (b.count() <= t.leaf_max) {
      for (int x = b.lo[0]; x < b.hi[0]; ++x)
        for (int y = b.lo[1]; y < b.hi[1]; ++y)
          for (int z = b.lo[2]; z < b.hi[2]; ++z) cols.push_back(slot(x, y, z));
    } else {
      int ax = 0;
      for (int d = 1; d < 3; ++d)
        if (b.hi[d] - b.lo[d] > b.hi[ax] - b.lo[ax]) ax = d;
      const int mid = b.lo[ax] + (b.hi[ax] - b.lo[ax]) / 2;
      Box l = b, r = b;
      l.hi[ax] = mid;
      r.lo[ax] = mid + 1;
      if (l.count() > 0) kids[nk++] = build(l, level + 1);
      if (r.count() > 0) kids[nk++] = build(r, level + 1);
      Box s = b;
      s.lo[ax] = mid;
      s.hi[ax] = mid + 1;
      for (int x = s.lo[0]; x < s.hi[0]; ++x)
        for (int y = s.lo[1]; y < s.hi[1]; ++y)
          for (int z = s.lo[2]; z < s.hi[2]; ++z) cols.push_back(slot(x, y, z));
    }
    Supernode sn;
    sn.level = level;
    sn.ncols = (int)cols.size();
    sn.nchild = nk;
    sn.child[0] = kids[0];
    sn.child[1] = kids[1];
    const int id = (int)t.sn.size();
    for (int k = 0; k < nk; ++k) t.sn[(size_t)kids[k]].parent = id;
    t.sn.push_back(sn);
    cols_of.push_back(cols);
    box_of.push_back(b);
    return id;
  }
};

}  // namespace

Template build_template(int block, int leaf_max, bool shell_root) {
  Template t;
  t.b1 = block + 1;
  t.slots = t.b1 * t.b1 * t.b1;
  t.leaf_max = leaf_max;
  t.shell_root = shell_root;
  Builder bld(t);
  Box root{{0, 0, 0}, {t.b1, t.b1, t.b1}};
  if (!shell_root || t.b1 < 3) {
    bld.build(root, 0);
  } else {
    Box inner{{1, 1, 1}, {t.b1 - 1, t.b1 - 1, t.b1 - 1}};
    const int kid = bld.build(inner, 1);
    std::vector<int32_t> shell;
    for (int x = 0; x < t.b1; ++x)
      for (int y = 0; y < t.b1; ++y)
        for (int z = 0; z < t.b1; ++z)
          if (x == 0 || y == 0 || z == 0 || x == t.b1 - 1 || y == t.b1 - 1 || z == t.b1 - 1)
            shell.push_back(bld.slot(x, y, z));
    Supernode sn;
    sn.level = 0;
    sn.ncols = (int)shell.size();
    sn.nchild = 1;
    sn.child[0] = kid;
    const int id = (int)t.sn.size();
    t.sn[(size_t)kid].parent = id;
    t.sn.push_back(sn);
    bld.cols_of.push_back(shell);
    bld.box_of.push_back(root);
  }
  const int ns = (int)t.sn.size();
  // elimination order = postorder, cols in order
  t.elim.assign((size_t)t.slots, -1);
  int pos = 0;
  for (int s = 0; s < ns; ++s)
    for (int32_t u : bld.cols_of[(size_t)s]) t.elim[(size_t)u] = pos++;
  if (pos != t.slots) throw std::logic_error("nd template: slots not covered");
  // rows = cols + halo(box)
  std::vector<int32_t> posmark((size_t)t.slots, -1);
  for (int s = 0; s < ns; ++s) {
    Supernode& sn = t.sn[(size_t)s];
    const Box& b = bld.box_of[(size_t)s];
    std::vector<int32_t> halo;
    for (int x = std::max(0, b.lo[0] - 1); x < std::min(t.b1, b.hi[0] + 1); ++x)
      for (int y = std::max(0, b.lo[1] - 1); y < std::min(t.b1, b.hi[1] + 1); ++y)
        for (int z = std::max(0, b.lo[2] - 1); z < std::min(t.b1, b.hi[2] + 1); ++z) {
          const bool inside = x >= b.lo[0] && x < b.hi[0] && y >= b.lo[1] && y < b.hi[1] && z >= b.lo[2] && z < b.hi[2];
          if (!inside) halo.push_back(bld.slot(x, y, z));
        }
    sn.rows_off = (int64_t)t.rows.size();
    for (int32_t u : bld.cols_of[(size_t)s]) t.rows.push_back(u);
    for (int32_t u : halo) t.rows.push_back(u);
    sn.nrows = sn.ncols + (int)halo.size();
    t.max_rows = std::max(t.max_rows, sn.nrows);
    t.max_cols = std::max(t.max_cols, sn.ncols);
  }
  // offsets
  int64_t po = 0, fo = 0, uo = 0;
  for (int s = 0; s < ns; ++s) {
    Supernode& sn = t.sn[(size_t)s];
    sn.panel_off = po;
    po += (int64_t)sn.nrows * sn.ncols;
    sn.front_off = fo;
    fo += (int64_t)sn.nrows * sn.nrows;
    sn.upd_off = uo;
    uo += sn.nrows - sn.ncols;
    const double c = sn.ncols, r = sn.nrows;
    t.flops += c * c * c / 3.0 + (r - c) * c * c + (r - c) * (r - c) * c;
  }
  t.panel_total = po;
  t.front_total = fo;
  t.upd_total = uo;
  // assembly map + extend-add maps
  for (int s = 0; s < ns; ++s) {
    Supernode& sn = t.sn[(size_t)s];
    for (int i = 0; i < sn.nrows; ++i) posmark[(size_t)t.rows[(size_t)(sn.rows_off + i)]] = i;
    sn.amap_off = (int64_t)t.amap.size();
    for (int c = 0; c < sn.ncols; ++c) {
      const int u = t.rows[(size_t)(sn.rows_off + c)];
      const int ux = u / (t.b1 * t.b1), uy = (u / t.b1) % t.b1, uz = u % t.b1;
      for (int k = 0; k < 27; ++k) {
        const int vx = ux + k / 9 - 1, vy = uy + (k / 3) % 3 - 1, vz = uz + k % 3 - 1;
        if (vx < 0 || vy < 0 || vz < 0 || vx >= t.b1 || vy >= t.b1 || vz >= t.b1) continue;
        const int v = (vx * t.b1 + vy) * t.b1 + vz;
        if (t.elim[(size_t)v] < t.elim[(size_t)u]) continue;
        const int r = posmark[(size_t)v];
        if (r < 0 || r < c) throw std::logic_error("nd template: stencil entry outside front");
        t.amap.push_back({r + c * sn.nrows, u, k, 0});
      }
    }
    sn.amap_len = (int)(t.amap.size() - (size_t)sn.amap_off);
    for (int k = 0; k < sn.nchild; ++k) {
      Supernode& ch = t.sn[(size_t)sn.child[k]];
      ch.emap_off = (int64_t)t.emap.size();
      for (int i = ch.ncols; i < ch.nrows; ++i) {
        const int p = posmark[(size_t)t.rows[(size_t)(ch.rows_off + i)]];
        if (p < 0) throw std::logic_error("nd template: child update outside parent front");
        t.emap.push_back(p);
      }
    }
    for (int i = 0; i < sn.nrows; ++i) posmark[(size_t)t.rows[(size_t)(sn.rows_off + i)]] = -1;
  }
  t.root_pos.assign((size_t)t.slots, -1);
  {
    const Supernode& root_sn = t.sn.back();
    for (int i = 0; i < root_sn.ncols; ++i) t.root_pos[(size_t)t.rows[(size_t)(root_sn.rows_off + i)]] = i;
  }
  int maxlev = 0;
  for (auto& sn : t.sn) maxlev = std::max(maxlev, sn.level);
  t.levels.assign((size_t)maxlev + 1, {});
  for (int s = 0; s < ns; ++s) t.levels[(size_t)t.sn[(size_t)s].level].push_back(s);
  return t;
}

}  // namespace cutbddc_b200
