// coarse_sparse.cu — the coarse problem A_c z = g as a sparse multifrontal
// Cholesky when n_c is large (n_c > kCoarseInverseMax; cfg5: 8946 coarse dofs).
//
// Replaces, for the coarse matrix, the dense Cholesky + explicit inverse
// (A_c^{-1} = X^T X, bddc.cu) that SPEC.md:386 ("factorise A_c") allows but
// does not require: A_c couples two coarse dofs only when they share a
// subdomain, so it is a 3-D lattice-like sparse matrix and a nested-dissection
// factorisation costs O(n_c^2) flops instead of O(n_c^3) (cfg5: ~1e9 against
// 7e11) and its solve streams the factor (tens of MB) instead of X (640 MB).
//
// Ordering: nested dissection on the subdomain lattice. A coarse object's
// position along an axis is lo + hi + 1 in doubled block coordinates (lo, hi:
// the extreme block indices of its neighbour subdomains): odd inside a block
// layer, even on the plane between two layers. The objects on a plane x = 2k
// separate those with x < 2k (all their subdomains in layers < k) from those
// with x > 2k (layers >= k): no subdomain touches both sides. Recursive
// bisection at the plane nearest the median, longest extent first; leaves of
// at most kLeaf objects. Post-order elimination; the row structure of each
// front is the usual multifrontal union (its columns' neighbours and its
// children's structures, minus what is eliminated).
//
// Numeric: per tree level (leaves first) one assembly kernel (A_c entries of
// the front's columns + the children's update matrices, extend-add in fixed
// order) and one dense-DAG launch (dense_dag_fronts: the partial Cholesky and
// the panel [L11^{-1}; L21 L11^{-1}] on the DMMA tile kernel). Solve: a
// forward level sweep (y_c = P11 v_c, u = v_r - P21 v_c, children's updates
// gathered in fixed order) and a backward one (x_c = P11^T y_c - P21^T x_r).
// Deterministic: every sum has a fixed order.
#include <algorithm>
#include <cstdio>
#include <numeric>
#include <vector>

#include "factor.cuh"

namespace cutbddc_b200 {
namespace {

constexpr int kLeaf = 96;

struct CsNode {
  std::vector<int> cols;  // objects eliminated here (ascending elimination order)
  std::vector<int> rows;  // row structure (ancestors' objects, ascending elimination order)
  int ch[2] = {-1, -1};
  int parent = -1;
  int level = 0;          // 0: leaves ... (height in the tree)
};

// position of every object (doubled block coordinates per axis)
struct ObjPos {
  std::vector<int> x[3];
};

void nd_split(const ObjPos& pos, std::vector<int>& set, std::vector<CsNode>& nodes, int& root) {
  // returns (in root) the node index of this set's subtree; post-order push
  if ((int)set.size() <= kLeaf) {
    CsNode n;
    n.cols = set;
    nodes.push_back(std::move(n));
    root = (int)nodes.size() - 1;
    return;
  }
  // axes by decreasing extent; the even plane nearest the median that leaves
  // both sides non-empty
  int ext[3], lo[3], hi[3];
  for (int a = 0; a < 3; ++a) {
    lo[a] = 1 << 30;
    hi[a] = -(1 << 30);
    for (int o : set) {
      lo[a] = std::min(lo[a], pos.x[a][(size_t)o]);
      hi[a] = std::max(hi[a], pos.x[a][(size_t)o]);
    }
    ext[a] = hi[a] - lo[a];
  }
  int order[3] = {0, 1, 2};
  std::stable_sort(order, order + 3, [&](int p, int q) { return ext[p] > ext[q]; });
  for (int oa = 0; oa < 3; ++oa) {
    const int a = order[oa];
    if (ext[a] < 2) break;
    std::vector<int> xs;
    xs.reserve(set.size());
    for (int o : set) xs.push_back(pos.x[a][(size_t)o]);
    std::nth_element(xs.begin(), xs.begin() + xs.size() / 2, xs.end());
    const int med = xs[xs.size() / 2];
    // candidate even planes strictly inside (lo, hi), nearest the median first
    int best = -1, bestd = 1 << 30;
    for (int X = (lo[a] + 1) & ~1; X < hi[a]; X += 2) {
      if (X <= lo[a]) continue;
      const int dd = std::abs(X - med);
      if (dd < bestd) {
        bestd = dd;
        best = X;
      }
    }
    if (best < 0) continue;
    std::vector<int> L, R, S;
    for (int o : set) {
      const int v = pos.x[a][(size_t)o];
      (v < best ? L : (v > best ? R : S)).push_back(o);
    }
    if (L.empty() || R.empty()) continue;
    int rl = -1, rr = -1;
    nd_split(pos, L, nodes, rl);
    nd_split(pos, R, nodes, rr);
    CsNode n;
    n.cols = S;
    n.ch[0] = rl;
    n.ch[1] = rr;
    nodes.push_back(std::move(n));
    root = (int)nodes.size() - 1;
    nodes[(size_t)rl].parent = root;
    nodes[(size_t)rr].parent = root;
    return;
  }
  CsNode n;  // no separating plane: one dense leaf
  n.cols = set;
  nodes.push_back(std::move(n));
  root = (int)nodes.size() - 1;
}

// device record of one front
struct CsFront {
  long long fo, po, ioff, voff, uoff;  // front, panel, index list, y (c) and update (rt - c) vector offsets
  long long moff[2];                   // children's extend-add maps (cmap offsets)
  int rt, c, ch[2];
};

// F = A_c entries of the front's columns (lower part) + the children's update
// matrices (extend-add, child 0 then child 1). One block per front.
__global__ void k_cs_assemble(const int* __restrict__ fl, const CsFront* __restrict__ fr, const int32_t* __restrict__ idx,
                              const int32_t* __restrict__ cmap, const double* __restrict__ Ac, int nc,
                              double* __restrict__ F) {
  const CsFront d = fr[fl[blockIdx.x]];
  double* f = F + d.fo;
  const int rt = d.rt, c = d.c;
  const int32_t* id = idx + d.ioff;
  const int64_t n2 = (int64_t)rt * rt;
  for (int64_t e = threadIdx.x; e < n2; e += blockDim.x) {
    const int i = (int)(e % rt), j = (int)(e / rt);
    f[e] = (j < c && i >= j) ? Ac[(int64_t)id[i] * nc + id[j]] : 0.0;
  }
  for (int k = 0; k < 2; ++k) {
    if (d.ch[k] < 0) continue;
    __syncthreads();
    const CsFront cd = fr[d.ch[k]];
    const int r = cd.rt - cd.c;
    const double* u = F + cd.fo + cd.c + (int64_t)cd.c * cd.rt;
    const int32_t* mp = cmap + d.moff[k];
    const int64_t m2 = (int64_t)r * r;
    for (int64_t e = threadIdx.x; e < m2; e += blockDim.x) {
      const int a = (int)(e % r), b = (int)(e / r);
      if (a < b) continue;
      f[mp[a] + (int64_t)mp[b] * rt] += u[a + (int64_t)b * cd.rt];
    }
  }
}

// forward: v = [g(cols); 0] + children's update vectors, y = P11 v_c,
// u = v_r - P21 v_c. Blocks (front, 32-row chunk): every block stages the
// whole v in shared memory, thread (row, slice) sums the columns j = slice
// mod 8 (32 consecutive rows per j: coalesced), the 8 partials of a row are
// added in slice order.
constexpr int kCsRows = 32, kCsSlices = 8;
__global__ void __launch_bounds__(kCsRows * kCsSlices) k_cs_fwd(const int* __restrict__ fl, const CsFront* __restrict__ fr,
                                                              const int32_t* __restrict__ idx, const int32_t* __restrict__ cmap,
                                                              const double* __restrict__ P, const double* __restrict__ g,
                                                              double* __restrict__ ybuf, double* __restrict__ ubuf,
                                                              const int* __restrict__ skip) {
  if (skip && *skip) return;
  extern __shared__ double v[];
  __shared__ double part[kCsSlices][kCsRows];
  const CsFront d = fr[fl[blockIdx.x]];
  const int rt = d.rt, c = d.c, i0 = blockIdx.y * kCsRows;
  if (i0 >= rt) return;
  const int32_t* id = idx + d.ioff;
  for (int i = threadIdx.x; i < rt; i += blockDim.x) v[i] = i < c ? g[id[i]] : 0.0;
  for (int k = 0; k < 2; ++k) {
    if (d.ch[k] < 0) continue;
    __syncthreads();
    const CsFront cd = fr[d.ch[k]];
    const int r = cd.rt - cd.c;
    const int32_t* mp = cmap + d.moff[k];
    const double* u = ubuf + cd.uoff;
    for (int a = threadIdx.x; a < r; a += blockDim.x) v[mp[a]] += u[a];
  }
  __syncthreads();
  const double* p = P + d.po;
  const int rr = threadIdx.x & (kCsRows - 1), sl = threadIdx.x / kCsRows, i = i0 + rr;
  double sacc = 0.0;
  if (i < rt) {
    const int jn = i < c ? i + 1 : c;  // P11 lower; P21 all c columns
    for (int j = sl; j < jn; j += kCsSlices) sacc += p[i + (int64_t)j * rt] * v[j];
  }
  part[sl][rr] = sacc;
  __syncthreads();
  if (sl == 0 && i < rt) {
    double t = part[0][rr];
#pragma unroll
    for (int q = 1; q < kCsSlices; ++q) t += part[q][rr];
    if (i < c)
      ybuf[d.voff + i] = t;
    else
      ubuf[d.uoff + i - c] = v[i] - t;
  }
}

// backward: x_c = P11^T y_c - P21^T x_r (x_r: the ancestors' final values).
// Blocks (front, 32-column chunk), a warp per column (coalesced down the
// panel column, fixed-order warp sum).
__global__ void k_cs_bwd(const int* __restrict__ fl, const CsFront* __restrict__ fr, const int32_t* __restrict__ idx,
                         const double* __restrict__ P, const double* __restrict__ ybuf, double* __restrict__ z,
                         const int* __restrict__ skip) {
  if (skip && *skip) return;
  extern __shared__ double w[];  // [y_c; -x_r]
  const CsFront d = fr[fl[blockIdx.x]];
  const int rt = d.rt, c = d.c, j0 = blockIdx.y * kCsRows;
  if (j0 >= c) return;
  const int32_t* id = idx + d.ioff;
  for (int i = j0 + threadIdx.x; i < rt; i += blockDim.x) w[i] = i < c ? ybuf[d.voff + i] : -z[id[i]];
  __syncthreads();
  const double* p = P + d.po;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int j = j0 + wid; j < min(c, j0 + kCsRows); j += nw) {
    double s = 0.0;
    for (int i = j + lane; i < rt; i += 32) s += p[i + (int64_t)j * rt] * w[i];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if (lane == 0) z[id[j]] = s;
  }
}

}  // namespace

void coarse_sparse_setup(cutbddc_gpu* h, int nc, const std::vector<std::vector<int>>& obj_of_gsd) {
  CoarseSparse& cs = h->csparse;
  cudaStream_t s = h->stream;
  ProfScope ps(h->prof, s, "coarse sparse symbolic");
  // ---- positions from the neighbour subdomains' block coordinates
  const int nb = h->nb, nsd_g = h->nsd_g;
  ObjPos pos;
  std::vector<int> lo[3], hi[3];
  for (int a = 0; a < 3; ++a) {
    lo[a].assign((size_t)nc, 1 << 30);
    hi[a].assign((size_t)nc, -1);
  }
  std::vector<std::vector<int>> sd_of_obj((size_t)nc);
  for (int g = 0; g < nsd_g; ++g) {
    const int64_t bid = h->g_block_ids[(size_t)g];
    const int bc[3] = {(int)(bid / nb / nb), (int)((bid / nb) % nb), (int)(bid % nb)};
    for (int o : obj_of_gsd[(size_t)g]) {
      sd_of_obj[(size_t)o].push_back(g);
      for (int a = 0; a < 3; ++a) {
        lo[a][(size_t)o] = std::min(lo[a][(size_t)o], bc[a]);
        hi[a][(size_t)o] = std::max(hi[a][(size_t)o], bc[a]);
      }
    }
  }
  for (int a = 0; a < 3; ++a) {
    pos.x[a].resize((size_t)nc);
    for (int o = 0; o < nc; ++o) {
      if (hi[a][(size_t)o] < 0) throw Failure(CUTBDDC_INVALID_ARGUMENT, "coarse object without a neighbour subdomain");
      pos.x[a][(size_t)o] = lo[a][(size_t)o] + hi[a][(size_t)o] + 1;
    }
  }
  // ---- nested dissection, post-order
  std::vector<CsNode> nodes;
  std::vector<int> all((size_t)nc);
  std::iota(all.begin(), all.end(), 0);
  int root = -1;
  nd_split(pos, all, nodes, root);
  const int nn = (int)nodes.size();
  std::vector<int> elim((size_t)nc, -1);  // elimination position of every object
  {
    int k = 0;
    for (CsNode& n : nodes)
      for (int o : n.cols) elim[(size_t)o] = k++;
    if (k != nc) throw Failure(CUTBDDC_INTERNAL, "coarse nested dissection lost objects");
  }
  // ---- row structures (post-order: children before parents)
  std::vector<int> mark((size_t)nc, -1);
  for (int q = 0; q < nn; ++q) {
    CsNode& n = nodes[(size_t)q];
    int last = -1;
    for (int o : n.cols) last = std::max(last, elim[(size_t)o]);
    std::vector<int> rows;
    auto add = [&](int o) {
      if (elim[(size_t)o] > last && mark[(size_t)o] != q) {
        mark[(size_t)o] = q;
        rows.push_back(o);
      }
    };
    for (int o : n.cols)
      for (int g : sd_of_obj[(size_t)o])
        for (int o2 : obj_of_gsd[(size_t)g]) add(o2);
    for (int k = 0; k < 2; ++k)
      if (n.ch[k] >= 0)
        for (int o : nodes[(size_t)n.ch[k]].rows) add(o);
    std::sort(rows.begin(), rows.end(), [&](int p, int r) { return elim[(size_t)p] < elim[(size_t)r]; });
    n.rows = std::move(rows);
    n.level = 0;
    for (int k = 0; k < 2; ++k)
      if (n.ch[k] >= 0) n.level = std::max(n.level, nodes[(size_t)n.ch[k]].level + 1);
  }
  // ---- device records, level lists, extend-add maps
  std::vector<CsFront> fr((size_t)nn);
  std::vector<int32_t> idx, cmap;
  long long fo = 0, po = 0, vo = 0, uo = 0;
  int nlev = 0, rt_max = 0;
  for (int q = 0; q < nn; ++q) {
    const CsNode& n = nodes[(size_t)q];
    CsFront& d = fr[(size_t)q];
    d.c = (int)n.cols.size();
    d.rt = d.c + (int)n.rows.size();
    d.ch[0] = n.ch[0];
    d.ch[1] = n.ch[1];
    d.fo = fo;
    d.po = po;
    d.voff = vo;
    d.uoff = uo;
    d.ioff = (long long)idx.size();
    fo += (long long)d.rt * d.rt;
    po += (long long)d.rt * d.c;
    vo += d.c;
    uo += d.rt - d.c;
    for (int o : n.cols) idx.push_back(o);
    for (int o : n.rows) idx.push_back(o);
    nlev = std::max(nlev, n.level + 1);
    rt_max = std::max(rt_max, d.rt);
  }
  for (int q = 0; q < nn; ++q) {
    CsFront& d = fr[(size_t)q];
    for (int k = 0; k < 2; ++k) {
      d.moff[k] = (long long)cmap.size();
      if (d.ch[k] < 0) continue;
      // position of each of the child's structure rows in this front's list
      for (int o : nodes[(size_t)d.ch[k]].rows) {
        const int32_t* b = idx.data() + d.ioff;
        const int32_t* e = b + d.rt;
        // the list is sorted by elimination order
        const int32_t* it = std::lower_bound(b, e, o, [&](int32_t x, int y) { return elim[(size_t)x] < elim[(size_t)y]; });
        if (it == e || *it != o) throw Failure(CUTBDDC_INTERNAL, "coarse front: child row not in the parent");
        cmap.push_back((int32_t)(it - b));
      }
    }
  }
  std::vector<int> level_ptr((size_t)nlev + 1, 0), flist((size_t)nn);
  for (const CsNode& n : nodes) ++level_ptr[(size_t)n.level + 1];
  for (int l = 0; l < nlev; ++l) level_ptr[(size_t)l + 1] += level_ptr[(size_t)l];
  {
    std::vector<int> at(level_ptr.begin(), level_ptr.end() - 1);
    for (int q = 0; q < nn; ++q) flist[(size_t)at[(size_t)nodes[(size_t)q].level]++] = q;
  }
  if ((size_t)rt_max * sizeof(double) > 48 * 1024)
    throw Failure(CUTBDDC_CONFIG, "coarse sparse: front larger than the solve kernels' shared staging");
  cs.level_rt.assign((size_t)nlev, 0);
  cs.level_c.assign((size_t)nlev, 0);
  for (int q = 0; q < nn; ++q) {
    const int l = nodes[(size_t)q].level;
    cs.level_rt[(size_t)l] = std::max(cs.level_rt[(size_t)l], fr[(size_t)q].rt);
    cs.level_c[(size_t)l] = std::max(cs.level_c[(size_t)l], fr[(size_t)q].c);
  }
  cs.level_ptr = level_ptr;
  cs.nlev = nlev;
  cs.rt_max = rt_max;
  cs.n_fronts = nn;
  static_assert(sizeof(CsFront) % 8 == 0, "CsFront layout");
  cs.fronts.upload(reinterpret_cast<const long long*>(fr.data()), fr.size() * (sizeof(CsFront) / 8), s);
  cs.idx.upload(idx, s);
  cs.cmap.upload(cmap.empty() ? std::vector<int32_t>{0} : cmap, s);
  cs.flist.upload(flist, s);
  cs.F.alloc((size_t)std::max(1ll, fo));
  cs.P.alloc((size_t)std::max(1ll, po));
  cs.ybuf.alloc((size_t)std::max(1ll, vo));
  cs.ubuf.alloc((size_t)std::max(1ll, uo));
  while (cs.plans.size() < (size_t)nlev) cs.plans.push_back(std::make_unique<DagPlan>());
  cs.dense.assign((size_t)nlev, {});
  double flops = 0.0;
  for (int l = 0; l < nlev; ++l)
    for (int t = level_ptr[(size_t)l]; t < level_ptr[(size_t)l + 1]; ++t) {
      const CsFront& d = fr[(size_t)flist[(size_t)t]];
      cs.dense[(size_t)l].push_back(DenseFront{d.fo, d.po, d.rt, d.c});
      const double c = d.c, r = d.rt - d.c;
      flops += c * c * c / 3.0 + c * c * r + c * r * r;
    }
  cs.flops = flops;
  cs.ready = true;
  if (std::getenv("CUTBDDC_COARSE_STATS"))
    std::fprintf(stderr, "[cutbddc] coarse sparse: n_c %d fronts %d levels %d max front %d, factor %.3g flops, L %.3g doubles\n",
                 nc, nn, nlev, rt_max, flops, (double)po);
}

void coarse_sparse_factor(cutbddc_gpu* h, const double* Ac, int nc, unsigned long long* fail) {
  CoarseSparse& cs = h->csparse;
  cudaStream_t s = h->stream;
  ProfScope ps(h->prof, s, "coarse sparse factor");
  const CsFront* fr = reinterpret_cast<const CsFront*>(cs.fronts.p);
  for (int l = 0; l < cs.nlev; ++l) {
    const int f0 = cs.level_ptr[(size_t)l], nf = cs.level_ptr[(size_t)l + 1] - f0;
    k_cs_assemble<<<nf, 256, 0, s>>>(cs.flist.p + f0, fr, cs.idx.p, cs.cmap.p, Ac, nc, cs.F.p);
    CB_LAUNCH();
    dense_dag_fronts(h, *cs.plans[(size_t)l], cs.F.p, cs.P.p, cs.dense[(size_t)l], fail);
  }
}

void coarse_sparse_solve(cutbddc_gpu* h, const double* g, double* z, const int* skip) {
  CoarseSparse& cs = h->csparse;
  cudaStream_t s = h->stream;
  const CsFront* fr = reinterpret_cast<const CsFront*>(cs.fronts.p);
  const size_t shm = sizeof(double) * (size_t)cs.rt_max;
  for (int l = 0; l < cs.nlev; ++l) {
    const int f0 = cs.level_ptr[(size_t)l], nf = cs.level_ptr[(size_t)l + 1] - f0;
    const dim3 grid(nf, (cs.level_rt[(size_t)l] + kCsRows - 1) / kCsRows);
    k_cs_fwd<<<grid, kCsRows * kCsSlices, shm, s>>>(cs.flist.p + f0, fr, cs.idx.p, cs.cmap.p, cs.P.p, g, cs.ybuf.p,
                                                    cs.ubuf.p, skip);
    CB_LAUNCH();
  }
  for (int l = cs.nlev; l-- > 0;) {
    const int f0 = cs.level_ptr[(size_t)l], nf = cs.level_ptr[(size_t)l + 1] - f0;
    const dim3 grid(nf, (cs.level_c[(size_t)l] + kCsRows - 1) / kCsRows);
    k_cs_bwd<<<grid, 256, shm, s>>>(cs.flist.p + f0, fr, cs.idx.p, cs.P.p, cs.ybuf.p, z, skip);
    CB_LAUNCH();
  }
}

}  // namespace cutbddc_b200
