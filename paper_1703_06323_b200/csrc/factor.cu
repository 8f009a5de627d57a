// factor.cu — batched multifrontal Cholesky over the ND template (K6) and
// the level-scheduled triangular solves (K7).
//
// Replaces SparseCholesky (linalg.cpp:34-62) for the interior problems A_II
// and the augmented Neumann matrices K = A + rho C^T C used by the
// constrained solves (linalg.cpp:64-106 / SPEC.md:379-396).
//
// All subdomains share one elimination tree (the (B+1)^3 lattice template,
// nd_template.cpp); each front is compacted per subdomain to the slots the
// matrix actually has (interior dofs for A_II, local dofs for K), so a cut
// subdomain pays only for its own dofs. One launch per tree level covers
// (every supernode of the level) x (every subdomain); a CTA owns one
// compact front. Fronts are dense column-major in an HBM workspace; the
// parent gathers its children's update matrices (extend-add in fixed child
// order: deterministic, no atomics).
//
// Factor storage per (subdomain, supernode): the Cholesky panel [L11; L21]
// (r' x c', column-major, lower part). Solves use blocked substitution
// (subst.cuh). Non-positive pivots are reported with the offending
// (subdomain, slot) — the pivot rule of linalg.cpp:42-54.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "factor.cuh"
#include "subst.cuh"

namespace cutbddc_b200 {
namespace {

constexpr int kThreads = 256;

// Compact row index of template row q of supernode s in subdomain sd.
__device__ inline int pfx_at(const FactorDev& f, const TplDev& t, int sd, const Supernode& s, int q) {
  return f.pfx[(int64_t)sd * t.rows_total + s.rows_off + q];
}

// ---------------------------------------------------------------- symbolic
// CTA per (supernode, subdomain): prefix-count the masked template rows.
__global__ void __launch_bounds__(kThreads) k_symbolic(TplDev t, int nsd, const uint8_t* __restrict__ mask,
                                                       int32_t* __restrict__ pfx, int32_t* __restrict__ tpos,
                                                       int2* __restrict__ rc) {
  const int sid = blockIdx.x, sd = blockIdx.y;
  const Supernode s = t.sn[sid];
  const int r = s.nrows;
  const int per = (r + kThreads - 1) / kThreads;
  const int q0 = threadIdx.x * per, q1 = min(r, q0 + per);
  int cnt = 0;
  for (int q = q0; q < q1; ++q) cnt += mask[(int64_t)sd * t.T + t.rows[s.rows_off + q]] != 0;
  __shared__ int sc[kThreads + 1];
  sc[threadIdx.x] = cnt;
  __syncthreads();
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int i = 0; i < kThreads; ++i) {
      const int v = sc[i];
      sc[i] = acc;
      acc += v;
    }
    sc[kThreads] = acc;
  }
  __syncthreads();
  int run = sc[threadIdx.x];
  int32_t* out = pfx + (int64_t)sd * t.rows_total + s.rows_off;
  int ccount = 0;
  int32_t* inv = tpos + (int64_t)sd * t.rows_total + s.rows_off;
  for (int q = q0; q < q1; ++q) {
    const bool p = mask[(int64_t)sd * t.T + t.rows[s.rows_off + q]] != 0;
    out[q] = p ? run : -1;
    if (p) inv[run] = q;  // compact row -> template row position
    run += p;
  }
  // compact cols = present rows among the first ncols template rows
  __shared__ int ncols_present;
  if (threadIdx.x == 0) ncols_present = 0;
  __syncthreads();
  for (int q = threadIdx.x; q < s.ncols; q += blockDim.x) ccount += mask[(int64_t)sd * t.T + t.rows[s.rows_off + q]] != 0;
  atomicAdd(&ncols_present, ccount);
  __syncthreads();
  if (threadIdx.x == 0) rc[(int64_t)sd * t.nsn + sid] = make_int2(sc[kThreads], ncols_present);
}

// ---------------------------------------------------------------- numeric
// The numeric factorisation is one dataflow launch over every front
// (dense_dag.cu). Split fronts are cut into 64 x 64 tile tasks shared by many
// CTAs; the others are factorised whole by one CTA (W task). A front is split
// from kSplitRows template rows (cfg4: against 600 / 250 / 150) or
// kSplitMflop template MFLOP of partial Cholesky (a dense root: one CTA would
// run it alone for ~0.5 ms). CUTBDDC_SPLIT_ROWS / CUTBDDC_SPLIT_MFLOP
// override, for measurements.
static const int kSplitRows = [] {
  const char* e = std::getenv("CUTBDDC_SPLIT_ROWS");
  return e ? std::max(64, std::atoi(e)) : 400;
}();
static const double kSplitMflop = [] {
  const char* e = std::getenv("CUTBDDC_SPLIT_MFLOP");
  return e ? std::atof(e) : 7.0;
}();
static bool is_split_front(const Supernode& sn) {
  const double r = sn.nrows, c = sn.ncols;
  const double mflop = (c * c * c / 3.0 + (r - c) * c * c + (r - c) * (r - c) * c) * 1e-6;
  return sn.nrows >= kSplitRows || mflop >= kSplitMflop;
}

// ---------------------------------------------------------------- solves
// forward elimination: X holds b on entry (slot vectors), y on exit at the
// front's columns; v_rest - L21 y goes to the parent through `upd`.
__global__ void __launch_bounds__(256) k_fwd_level(TplDev t, FactorDev f, const int32_t* __restrict__ level_sn, int nsd,
                                                   const double* __restrict__ panel, double* __restrict__ X,
                                                   double* __restrict__ upd, const int* __restrict__ skip) {
  if (skip && *skip) return;
  extern __shared__ double v[];
  const int sid = level_sn[blockIdx.x];
  const Supernode s = t.sn[sid];
  const int sd = blockIdx.y, rhs = blockIdx.z;
  const int2 rc = f.rc[(int64_t)sd * t.nsn + sid];
  const int r = rc.x, c = rc.y;
  if (r == 0) return;
  double* x = X + ((int64_t)rhs * nsd + sd) * t.T;
  double* ub = upd + (int64_t)rhs * f.upd_total;
  const int32_t* rows = t.rows + s.rows_off;
  for (int q = threadIdx.x; q < s.nrows; q += blockDim.x) {
    const int p = pfx_at(f, t, sd, s, q);
    if (p >= 0) v[p] = q < s.ncols ? x[rows[q]] : 0.0;
  }
  __syncthreads();
  for (int ch = 0; ch < s.nchild; ++ch) {
    const int cid = s.child[ch];
    const Supernode cs = t.sn[cid];
    const int ccc = f.rc[(int64_t)sd * t.nsn + cid].y;
    const double* cu = ub + f.upd_off[(int64_t)sd * t.nsn + cid];
    for (int a = threadIdx.x; a < cs.nrows - cs.ncols; a += blockDim.x) {
      const int ia = pfx_at(f, t, sd, cs, cs.ncols + a);
      if (ia >= 0) v[pfx_at(f, t, sd, s, t.emap[cs.emap_off + a])] += cu[ia - ccc];
    }
    __syncthreads();
  }
  panel_forward(panel + f.panel_off[(int64_t)sd * t.nsn + sid], r, c, v);
  double* uo = ub + f.upd_off[(int64_t)sd * t.nsn + sid];
  for (int q = threadIdx.x; q < s.nrows; q += blockDim.x) {
    const int p = pfx_at(f, t, sd, s, q);
    if (p < 0) continue;
    if (q < s.ncols)
      x[rows[q]] = v[p];
    else
      uo[p - c] = v[p];
  }
}

// backward substitution: X holds y at this level's columns and the final x
// at ancestors; x_c = L11^{-T} (y - L21^T x_rest).
__global__ void __launch_bounds__(256) k_bwd_level(TplDev t, FactorDev f, const int32_t* __restrict__ level_sn, int nsd,
                                                   const double* __restrict__ panel, double* __restrict__ X,
                                                   const int* __restrict__ skip) {
  if (skip && *skip) return;
  extern __shared__ double w[];
  __shared__ double tile[32][33];
  const int sid = level_sn[blockIdx.x];
  const Supernode s = t.sn[sid];
  const int sd = blockIdx.y, rhs = blockIdx.z;
  const int2 rc = f.rc[(int64_t)sd * t.nsn + sid];
  const int r = rc.x, c = rc.y;
  if (c == 0) return;
  double* x = X + ((int64_t)rhs * nsd + sd) * t.T;
  const int32_t* rows = t.rows + s.rows_off;
  for (int q = threadIdx.x; q < s.nrows; q += blockDim.x) {
    const int p = pfx_at(f, t, sd, s, q);
    if (p >= 0) w[p] = x[rows[q]];
  }
  __syncthreads();
  panel_backward(panel + f.panel_off[(int64_t)sd * t.nsn + sid], r, c, w, tile);
  for (int q = threadIdx.x; q < s.ncols; q += blockDim.x) {
    const int p = pfx_at(f, t, sd, s, q);
    if (p >= 0) x[rows[q]] = w[p];
  }
}

// Big fronts, forward: [y; t] = G v_c as a GEMV split into 128-row chunks
// (one CTA each). Every chunk rebuilds the full front vector (gather +
// children's updates) in shared memory; y goes to `ysave` (x keeps b at the
// columns until the backward sweep, so concurrent chunks never race).
// Fronts with at least kBigMinCols template columns get explicit-inverse
// panels and multi-CTA GEMV sweeps; all fronts do (measured: the blocked
// substitution path was latency-bound at every level).
constexpr int kBigMinCols = 1;
// ND leaf size: boxes of at most this many lattice nodes are leaf fronts
// (CUTBDDC_LEAF overrides, for measurements).
constexpr int kLeafMax = 216;  // cfg4: 27 -> 125 cut the apply's solve time 744 -> 668 us; 125 -> 216: 3.49 -> 3.72 M DOF/s (profiles/r01_tune_leaf.txt)
constexpr int kBigRows = 32;   // forward: rows per CTA (one row per lane)
constexpr int kBigCols = 16;   // backward: columns per CTA (two per warp)

__global__ void __launch_bounds__(256) k_fwd_big(TplDev t, FactorDev f, const int2* __restrict__ items, int nsd,
                                                 const double* __restrict__ panel, const double* __restrict__ X,
                                                 double* __restrict__ ysave, double* __restrict__ upd,
                                                 const int* __restrict__ skip) {
  if (skip && *skip) return;
  extern __shared__ double v[];
  int* slot_of = reinterpret_cast<int*>(v + 2048);
  const int2 it = items[blockIdx.x];
  const int sid = it.x;
  const Supernode s = t.sn[sid];
  const int sd = blockIdx.y, rhs = blockIdx.z;
  const int2 rc = f.rc[(int64_t)sd * t.nsn + sid];
  const int r = rc.x, c = rc.y;
  const int i0 = it.y * kBigRows;
  if (i0 >= r) return;
  const int i1 = min(r, i0 + kBigRows);
  const double* x = X + ((int64_t)rhs * nsd + sd) * t.T;
  double* ys = ysave + ((int64_t)rhs * nsd + sd) * t.T;
  double* ub = upd + (int64_t)rhs * f.upd_total;
  const int32_t* rows = t.rows + s.rows_off;
  for (int q = threadIdx.x; q < s.nrows; q += blockDim.x) {
    const int p = pfx_at(f, t, sd, s, q);
    if (p >= 0) {
      v[p] = q < s.ncols ? x[rows[q]] : 0.0;
      slot_of[p] = rows[q];
    }
  }
  __syncthreads();
  for (int ch = 0; ch < s.nchild; ++ch) {
    const int cid = s.child[ch];
    const Supernode cs = t.sn[cid];
    const int ccc = f.rc[(int64_t)sd * t.nsn + cid].y;
    const double* cu = ub + f.upd_off[(int64_t)sd * t.nsn + cid];
    for (int a = threadIdx.x; a < cs.nrows - cs.ncols; a += blockDim.x) {
      const int ia = pfx_at(f, t, sd, cs, cs.ncols + a);
      if (ia >= 0) v[pfx_at(f, t, sd, s, t.emap[cs.emap_off + a])] += cu[ia - ccc];
    }
    __syncthreads();
  }
  const double* G = panel + f.panel_off[(int64_t)sd * t.nsn + sid];
  double* uo = ub + f.upd_off[(int64_t)sd * t.nsn + sid];
  // lane = row of the 32-row chunk, warp = contiguous column range; four
  // independent accumulators keep 4 coalesced 256-B loads per warp in flight.
  // (G's strict upper triangle is stored as zeros, so rows need no mask.)
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int jend = min(c, i1);
  const int cw = (jend + nw - 1) / nw;
  const int ja = min(jend, wid * cw), jb = min(jend, ja + cw);
  const int i = i0 + lane;
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  if (i < i1) {
    const double* gi = G + i;
    int j = ja;
    for (; j + 4 <= jb; j += 4) {
      s0 += gi[(int64_t)j * r] * v[j];
      s1 += gi[(int64_t)(j + 1) * r] * v[j + 1];
      s2 += gi[(int64_t)(j + 2) * r] * v[j + 2];
      s3 += gi[(int64_t)(j + 3) * r] * v[j + 3];
    }
    for (; j < jb; ++j) s0 += gi[(int64_t)j * r] * v[j];
  }
  __shared__ double part[8][33];
  part[wid][lane] = (s0 + s1) + (s2 + s3);
  __syncthreads();
  if (wid == 0 && i < i1) {
    double o = 0.0;
    for (int q = 0; q < nw; ++q) o += part[q][lane];
    if (i < c)
      ys[slot_of[i]] = o;
    else
      uo[i - c] = v[i] - o;
  }
}

// Big fronts, backward: x_c = G^T [y; -x_rest], 32 columns per CTA, one warp
// per column reducing over the rows.
__global__ void __launch_bounds__(256) k_bwd_big(TplDev t, FactorDev f, const int2* __restrict__ items, int nsd,
                                                 const double* __restrict__ panel, double* __restrict__ X,
                                                 const double* __restrict__ ysave, const int* __restrict__ skip) {
  if (skip && *skip) return;
  extern __shared__ double w[];
  int* slot_of = reinterpret_cast<int*>(w + 2048);
  const int2 it = items[blockIdx.x];
  const int sid = it.x;
  const Supernode s = t.sn[sid];
  const int sd = blockIdx.y, rhs = blockIdx.z;
  const int2 rc = f.rc[(int64_t)sd * t.nsn + sid];
  const int r = rc.x, c = rc.y;
  const int j0 = it.y * kBigCols;
  if (j0 >= c) return;
  const int j1 = min(c, j0 + kBigCols);
  double* x = X + ((int64_t)rhs * nsd + sd) * t.T;
  const double* ys = ysave + ((int64_t)rhs * nsd + sd) * t.T;
  const int32_t* rows = t.rows + s.rows_off;
  for (int q = threadIdx.x; q < s.nrows; q += blockDim.x) {
    const int p = pfx_at(f, t, sd, s, q);
    if (p >= 0) {
      w[p] = p < c ? ys[rows[q]] : -x[rows[q]];
      slot_of[p] = rows[q];
    }
  }
  __syncthreads();
  const double* G = panel + f.panel_off[(int64_t)sd * t.nsn + sid];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int j = j0 + wid; j < j1; j += nw) {
    const double* col = G + (int64_t)j * r;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    int i = j + lane;
    for (; i + 96 < r; i += 128) {
      s0 += col[i] * w[i];
      s1 += col[i + 32] * w[i + 32];
      s2 += col[i + 64] * w[i + 64];
      s3 += col[i + 96] * w[i + 96];
    }
    for (; i < r; i += 32) s0 += col[i] * w[i];
    const double sum = warp_sum((s0 + s1) + (s2 + s3));
    if (lane == 0) x[slot_of[j]] = sum;
  }
}

}  // namespace

TplDev tpl_dev(const TplSet& ts, int slots) {
  TplDev t;
  t.sn = ts.sn.p;
  t.rows = ts.rows.p;
  t.amap = ts.amap.p;
  t.emap = ts.emap.p;
  t.root_pos = ts.root_pos.p;
  t.is_big = ts.big_flag.p;
  t.T = slots;
  t.nsn = (int)ts.tpl.sn.size();
  t.root = t.nsn - 1;
  t.rows_total = (int64_t)ts.tpl.rows.size();
  return t;
}

FactorDev factor_dev(const FactorSet& f) {
  return FactorDev{f.pfx.p,     f.tpos.p,
                   f.rc.p,      f.panel_off.p,
                   f.upd_off.p, f.upd_total,
                   reinterpret_cast<const FrontDesc*>(f.desc.p), reinterpret_cast<const int2*>(f.gmap.p),
                   f.cslot.p};
}

void upload_template(cutbddc_gpu* h, TplSet& ts, bool shell_root) {
  cudaStream_t s = h->stream;
  static const int leaf = [] {
    const char* e = std::getenv("CUTBDDC_LEAF");
    return e ? std::max(8, std::atoi(e)) : kLeafMax;
  }();
  ts.tpl = build_template(h->block, leaf, shell_root);
  if (ts.tpl.max_rows > 2048) throw Failure(CUTBDDC_CONFIG, "nd template: front larger than 2048 rows");
  ts.sn.upload(ts.tpl.sn, s);
  ts.rows.upload(ts.tpl.rows, s);
  ts.amap.upload(ts.tpl.amap, s);
  ts.emap.upload(ts.tpl.emap.empty() ? std::vector<int32_t>{0} : ts.tpl.emap, s);
  ts.root_pos.upload(ts.tpl.root_pos, s);
  std::vector<int32_t> lv, small, big;
  std::vector<int2> fwd, bwd;
  ts.level_first.clear();
  ts.level_count.clear();
  ts.small_first.clear();
  ts.small_count.clear();
  ts.big_first.clear();
  ts.big_count.clear();
  ts.fwd_first.clear();
  ts.fwd_count.clear();
  ts.bwd_first.clear();
  ts.bwd_count.clear();
  ts.is_big.assign(ts.tpl.sn.size(), 0);
  ts.is_split.assign(ts.tpl.sn.size(), 0);
  for (size_t sid = 0; sid < ts.tpl.sn.size(); ++sid) ts.is_split[sid] = is_split_front(ts.tpl.sn[sid]);
  for (auto& L : ts.tpl.levels) {
    ts.level_first.push_back((int)lv.size());
    ts.level_count.push_back((int)L.size());
    lv.insert(lv.end(), L.begin(), L.end());
    ts.small_first.push_back((int)small.size());
    ts.big_first.push_back((int)big.size());
    ts.fwd_first.push_back((int)fwd.size());
    ts.bwd_first.push_back((int)bwd.size());
    for (int sid : L) {
      const Supernode& sn = ts.tpl.sn[(size_t)sid];
      // big: explicit-inverse panel swept by many CTAs
      const bool is_big = sn.ncols >= kBigMinCols;
      ts.is_big[(size_t)sid] = is_big;
      if (!is_big) {
        small.push_back(sid);
        continue;
      }
      big.push_back(sid);
      for (int ch = 0; ch < (sn.nrows + kBigRows - 1) / kBigRows; ++ch) fwd.push_back(make_int2(sid, ch));
      for (int ch = 0; ch < (sn.ncols + kBigCols - 1) / kBigCols; ++ch) bwd.push_back(make_int2(sid, ch));
    }
    ts.small_count.push_back((int)small.size() - ts.small_first.back());
    ts.big_count.push_back((int)big.size() - ts.big_first.back());
    ts.fwd_count.push_back((int)fwd.size() - ts.fwd_first.back());
    ts.bwd_count.push_back((int)bwd.size() - ts.bwd_first.back());
  }
  auto nz32 = [](std::vector<int32_t> v) { return v.empty() ? std::vector<int32_t>{0} : v; };
  auto nz2 = [](std::vector<int2> v) { return v.empty() ? std::vector<int2>{make_int2(0, 0)} : v; };
  ts.level_sn.upload(lv, s);
  ts.small_sn.upload(nz32(small), s);
  ts.big_sn.upload(nz32(big), s);
  ts.fwd_items.upload(nz2(fwd), s);
  ts.bwd_items.upload(nz2(bwd), s);
  ts.big_flag.upload(ts.is_big, s);
  ts.ready = true;
}

double sweep_bytes(const FactorSet& f) { return f.bytes_per_sweep; }

// device bytes of the (grow-only, reusable) front workspace already held
static int64_t front_bytes_held(const cutbddc_gpu* h) { return (int64_t)h->ws_front.cap * (int64_t)sizeof(double); }

static const char* tag_of(const cutbddc_gpu* h, const FactorSet& f) { return &f == &h->fI ? "I" : "K"; }

// Symbolic phase: compact rows per (sd, supernode), offsets, sweep plan.
void factor_symbolic(cutbddc_gpu* h, const TplSet& ts, const FactorInput& in, FactorSet& f) {
  cudaStream_t s = h->stream;
  const TplDev t = tpl_dev(ts, h->slots);
  const int nsd = h->nsd, nsn = t.nsn;
  f.pfx.alloc((size_t)nsd * t.rows_total);
  f.tpos.alloc((size_t)nsd * t.rows_total);
  f.rc.alloc((size_t)nsd * nsn);
  ProfScope pplan(h->prof, s, std::string("factor") + tag_of(h, f) + " symbolic+plan");
  k_symbolic<<<dim3(nsn, nsd), kThreads, 0, s>>>(t, nsd, in.mask, f.pfx.p, f.tpos.p, f.rc.p);
  CB_LAUNCH();
  f.h_rc = f.rc.to_host(s);
  std::vector<int64_t> poff((size_t)nsd * nsn), uoff((size_t)nsd * nsn), foff((size_t)nsd * nsn);
  f.h_front_base.assign((size_t)nsd + 1, 0);
  int64_t pt = 0, ut = 0;
  double bytes = 0, flops = 0, flops_inv = 0;
  for (int sd = 0; sd < nsd; ++sd) {
    int64_t fo = 0;
    for (int q = 0; q < nsn; ++q) {
      const int2 v = f.h_rc[(size_t)sd * nsn + q];
      const double r = v.x, c = v.y;
      poff[(size_t)sd * nsn + q] = pt;
      pt += (int64_t)v.x * v.y;
      uoff[(size_t)sd * nsn + q] = ut;
      ut += v.x - v.y;
      foff[(size_t)sd * nsn + q] = fo;
      fo += (int64_t)v.x * v.x;
      bytes += 2.0 * 8.0 * (r * c - c * (c - 1) / 2.0) + 2.0 * 2.0 * 8.0 * r;
      flops += c * c * c / 3.0 + (r - c) * c * c + (r - c) * (r - c) * c;
      flops_inv += c * c * c / 3.0 + (r - c) * c * c;
    }
    f.h_front_base[(size_t)sd + 1] = f.h_front_base[(size_t)sd] + fo;
  }
  f.panel_total = pt;
  f.upd_total = ut;
  f.bytes_per_sweep = bytes;
  f.flops = flops;
  f.flops_inv = flops_inv;
  f.panel_off.upload(poff, s);
  f.h_panel_off = poff;
  f.h_front_off = foff;
  f.upd_off.upload(uoff, s);
  f.panel.alloc((size_t)pt + 2);  // +2: the sweeps' 16-byte aligned bulk copies may read one double past the end
  build_sweep_plan(h, ts, f, poff, uoff);
}

// Numeric phase. The factorisations share one dataflow launch (the interior
// problems' fronts fill the SMs the K root's POTRF chain leaves idle) when
// all their fronts fit a workspace budget of half the free device memory;
// otherwise each runs alone in subdomain chunks bounded by the budget (every
// chunk repeats the tree's critical path).
void factor_numeric(cutbddc_gpu* h, const std::vector<FactorJob>& jobs) {
  cudaStream_t s = h->stream;
  const int nsd = h->nsd;
  DevBuf<unsigned long long>& fail = h->ws_fail;
  fail.alloc(jobs.size());
  CB_CUDA(cudaMemsetAsync(fail.p, 0xff, 8 * jobs.size(), s));
  DevBuf<double>& front = h->ws_front;
  for (cudaEvent_t e : h->dag_ev) cudaEventDestroy(e);
  h->dag_ev.clear();
  ProfScope pnum(h->prof, s, "factor numeric");
  int64_t all = 0;
  for (const FactorJob& j : jobs) all += j.f->h_front_base[(size_t)nsd];
  // front workspace budget: what is held, plus half the free memory. The
  // memory query (slow, and it can stall behind other driver work: up to
  // ~90 ms seen) only when the held workspace is too small.
  int64_t budget = (int64_t)front.cap;
  if (all > budget) {
    size_t free_b = 0, total_b = 0;
    CB_CUDA(cudaMemGetInfo(&free_b, &total_b));
    budget = std::max<int64_t>((1ll << 30) / 8, (int64_t)(free_b / 2 + front_bytes_held(h)) / 8);
  }
  if (all <= budget) {
    std::vector<FactorSpan> spans;
    int64_t off = 0;
    for (size_t g = 0; g < jobs.size(); ++g) {
      spans.push_back(FactorSpan{jobs[g].ts, jobs[g].in, jobs[g].f, 0, nsd, off, fail.p + g});
      off += jobs[g].f->h_front_base[(size_t)nsd];
    }
    if ((int64_t)front.n < all) front.alloc((size_t)std::max<int64_t>(1, all));
    dense_dag_factor(h, spans, front.p);
  } else {
    for (size_t g = 0; g < jobs.size(); ++g) {
      const FactorSet& f = *jobs[g].f;
      int sd0 = 0;
      while (sd0 < nsd) {
        int sd1 = sd0 + 1;
        while (sd1 < nsd && f.h_front_base[(size_t)sd1 + 1] - f.h_front_base[(size_t)sd0] <= budget) ++sd1;
        const int64_t need = f.h_front_base[(size_t)sd1] - f.h_front_base[(size_t)sd0];
        if ((int64_t)front.n < need) front.alloc((size_t)need);
        dense_dag_factor(h, {FactorSpan{jobs[g].ts, jobs[g].in, jobs[g].f, sd0, sd1, 0, fail.p + g}}, front.p);
        sd0 = sd1;
      }
    }
  }
  pnum.close();
  std::vector<unsigned long long> fl(jobs.size());
  CB_CUDA(cudaMemcpyAsync(fl.data(), fail.p, 8 * jobs.size(), cudaMemcpyDeviceToHost, s));
  CB_CUDA(cudaStreamSynchronize(s));
  for (size_t g = 0; g < jobs.size(); ++g)
    if (jobs[g].failed) {
      *jobs[g].failed = fl[g] != ~0ull;
      if (fl[g] != ~0ull && std::getenv("CUTBDDC_K_STATS"))
        std::fprintf(stderr, "[cutbddc] %s: non-positive pivot at subdomain %lld slot %lld\n", jobs[g].what,
                     (long long)(fl[g] / (unsigned long long)h->slots), (long long)(fl[g] % (unsigned long long)h->slots));
    }
  for (size_t g = 0; g < jobs.size(); ++g)
    if (fl[g] != ~0ull && !jobs[g].failed) {
      const int64_t sd = (int64_t)(fl[g] / (unsigned long long)h->slots);
      const int64_t slot = (int64_t)(fl[g] % (unsigned long long)h->slots);
      throw Failure(CUTBDDC_SINGULAR, std::string(jobs[g].what) + ": matrix is not positive definite (subdomain " +
                                          std::to_string(sd) + ", pivot slot " + std::to_string(slot) + ")");
    }
}

// CUTBDDC_LEVEL_SWEEPS=1 selects the level-synchronous sweeps for single
// right-hand sides too (A/B measurement of the dataflow sweeps).
static bool level_sweeps() {
  static const bool v = [] {
    const char* e = std::getenv("CUTBDDC_LEVEL_SWEEPS");
    return e && e[0] == '1';
  }();
  return v;
}

// In-place solve of nrhs x nsd slot vectors X ([rhs][sd][T]); masked-out
// slots are left untouched. upd must hold nrhs * f.upd_total doubles.
void solve_device(cutbddc_gpu* h, const TplSet& ts, const FactorSet& f, double* X, int nrhs, double* upd,
                  double* ysave, const int* skip, bool rhs_root_only) {
  if (nrhs == 1 && !rhs_root_only && !level_sweeps()) {
    sweep_solve(h, ts, f, X, ysave, upd, skip);
    return;
  }
  cudaStream_t s = h->stream;
  const TplDev t = tpl_dev(ts, h->slots);
  const FactorDev fd = factor_dev(f);
  const int nlev = (int)ts.level_first.size();
  const size_t shm = sizeof(double) * (size_t)ts.tpl.max_rows;
  const size_t shm_big = (sizeof(double) + sizeof(int)) * 2048;
  if (rhs_root_only) {
    // right-hand sides supported on the root columns only (C^T of the shell
    // template): every lower forward step is zero, so only the root is swept.
    CB_CUDA(cudaMemsetAsync(upd, 0, sizeof(double) * (size_t)nrhs * f.upd_total, s));
    CB_CUDA(cudaMemsetAsync(ysave, 0, sizeof(double) * (size_t)nrhs * h->nsd * h->slots, s));
  }
  const std::string tag = std::string("solve") + (&f == &h->fI ? "I" : "K") + (nrhs > 1 ? "m " : " ");
  for (int L = nlev - 1; L >= 0; --L) {
    if (rhs_root_only && L > 0) continue;
    ProfScope ps(h->prof, s, tag + "fwd L" + std::to_string(L));
    if (ts.small_count[(size_t)L] > 0) {
      dim3 grid(ts.small_count[(size_t)L], h->nsd, nrhs);
      k_fwd_level<<<grid, 256, shm, s>>>(t, fd, ts.small_sn.p + ts.small_first[(size_t)L], h->nsd, f.panel.p, X, upd,
                                         skip);
      CB_LAUNCH();
    }
    if (ts.fwd_count[(size_t)L] > 0) {
      dim3 grid(ts.fwd_count[(size_t)L], h->nsd, nrhs);
      k_fwd_big<<<grid, 256, shm_big, s>>>(t, fd, ts.fwd_items.p + ts.fwd_first[(size_t)L], h->nsd, f.panel.p, X, ysave,
                                           upd, skip);
      CB_LAUNCH();
    }
  }
  for (int L = 0; L < nlev; ++L) {
    ProfScope ps(h->prof, s, tag + "bwd L" + std::to_string(L));
    if (ts.bwd_count[(size_t)L] > 0) {
      dim3 grid(ts.bwd_count[(size_t)L], h->nsd, nrhs);
      k_bwd_big<<<grid, 256, shm_big, s>>>(t, fd, ts.bwd_items.p + ts.bwd_first[(size_t)L], h->nsd, f.panel.p, X, ysave,
                                           skip);
      CB_LAUNCH();
    }
    if (ts.small_count[(size_t)L] > 0) {
      dim3 grid(ts.small_count[(size_t)L], h->nsd, nrhs);
      k_bwd_level<<<grid, 256, shm, s>>>(t, fd, ts.small_sn.p + ts.small_first[(size_t)L], h->nsd, f.panel.p, X, skip);
      CB_LAUNCH();
    }
  }
}

}  // namespace cutbddc_b200
