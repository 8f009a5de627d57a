// factor.cu — batched multifrontal Cholesky over the ND template (K6) and
// the symbolic phase of the dataflow triangular solves (sweep.cu).
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
// from kSplitRows template rows or
// kSplitMflop template MFLOP of partial Cholesky (a dense root: one CTA would
// run it alone for ~0.5 ms). CUTBDDC_SPLIT_ROWS / CUTBDDC_SPLIT_MFLOP
// override, for measurements.
static const int kSplitRows = [] {
  const char* e = std::getenv("CUTBDDC_SPLIT_ROWS");
  return e ? std::max(64, std::atoi(e)) : 400;
}();
// Split threshold in MFLOP: few subdomains (cfg4: 51) leave most SMs idle
// unless the leaves are tiled too (7 -> 1 MFLOP: setup 4.8 -> 4.4 ms); many
// (cfg5: 1 960) fill the GPU with whole fronts, where tiling only adds task
// overhead (1 MFLOP: setup 607 -> 662 ms). profiles/r02_tune_split.txt.
static double split_mflop(int nsd) {
  static const char* e = std::getenv("CUTBDDC_SPLIT_MFLOP");
  return e ? std::atof(e) : (nsd >= 256 ? 7.0 : 1.0);
}
static bool is_split_front(const Supernode& sn, int nsd) {
  const double r = sn.nrows, c = sn.ncols;
  const double mflop = (c * c * c / 3.0 + (r - c) * c * c + (r - c) * (r - c) * c) * 1e-6;
  return sn.nrows >= kSplitRows || mflop >= split_mflop(nsd);
}


}  // namespace

void set_split_flags(TplSet& ts, int nsd) {
  ts.is_split.assign(ts.tpl.sn.size(), 0);
  for (size_t sid = 0; sid < ts.tpl.sn.size(); ++sid) ts.is_split[sid] = is_split_front(ts.tpl.sn[sid], nsd);
}

TplDev tpl_dev(const TplSet& ts, int slots) {
  TplDev t;
  t.sn = ts.sn.p;
  t.rows = ts.rows.p;
  t.amap = ts.amap.p;
  t.emap = ts.emap.p;
  t.root_pos = ts.root_pos.p;
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

constexpr int kLeafMax = 216;  // cfg4: 27 -> 125 cut the apply's solve time 744 -> 668 us; 125 -> 216: 3.49 -> 3.72 M DOF/s (profiles/r01_tune_leaf.txt)

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
  set_split_flags(ts, h->nsd);
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
  pplan.next(std::string("factor") + tag_of(h, f) + " symbolic host");
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
  pplan.next(std::string("factor") + tag_of(h, f) + " sweep plan");
  build_sweep_plan(h, ts, f, poff, uoff);
}

// Numeric phase. The factorisations share one dataflow launch (the interior
// problems' fronts fill the SMs the K root's POTRF chain leaves idle) when
// all their fronts fit a workspace budget of half the free device memory;
// otherwise each runs alone in subdomain chunks bounded by the budget (every
// chunk repeats the tree's critical path).
void factor_numeric(cutbddc_gpu* h, const std::vector<FactorJob>& jobs, const std::function<void()>& overlap,
                    bool append_events) {
  cudaStream_t s = h->stream;
  const int nsd = h->nsd;
  DevBuf<unsigned long long>& fail = h->ws_fail;
  fail.alloc(jobs.size());
  CB_CUDA(cudaMemsetAsync(fail.p, 0xff, 8 * jobs.size(), s));
  DevBuf<double>& front = h->ws_front;
  if (!append_events) {
    for (cudaEvent_t e : h->dag_ev) cudaEventDestroy(e);
    h->dag_ev.clear();
  }
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
      spans.push_back(FactorSpan{jobs[g].ts, jobs[g].in, jobs[g].f, 0, nsd, off, fail.p + g, jobs[g].fail_sd});
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
        dense_dag_factor(h, {FactorSpan{jobs[g].ts, jobs[g].in, jobs[g].f, sd0, sd1, 0, fail.p + g, jobs[g].fail_sd}},
                         front.p);
        sd0 = sd1;
      }
    }
  }
  pnum.close();
  if (overlap) overlap();
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

// In-place solve of the nsd slot vectors X ([sd][T]) by the dataflow sweeps
// (sweep.cu); masked-out slots are left untouched.
void solve_device(cutbddc_gpu* h, const TplSet& ts, const FactorSet& f, double* X, double* upd, double* ysave,
                  const int* skip) {
  sweep_solve(h, ts, f, X, ysave, upd, skip);
}

// The constrained Neumann solve of every subdomain: K_c (corner
// formulation) or K (shell root); a mixed K takes each subdomain's own.
void solve_k_device(cutbddc_gpu* h, double* X, const int* skip) {
  solve_device(h, h->tplK(), h->fK, X, h->upd.p, h->ysave.p, skip);
  if (h->k_mixed) solve_device(h, h->tK, h->fKs, X, h->upd.p, h->ysave.p, skip);
}

}  // namespace cutbddc_b200
