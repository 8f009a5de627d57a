// factor.cu — batched multifrontal Cholesky over the ND template (K6) and
// the level-scheduled triangular solves (K7).
//
// Replaces SparseCholesky (linalg.cpp:34-62) for the interior problems A_II
// and the augmented Neumann matrices K = A + rho C^T C used by the
// constrained solves (linalg.cpp:64-106 / SPEC.md:379-396). One launch per
// elimination-tree level covers (every supernode of the level) x (every
// subdomain): all subdomains share the template, so front shapes are uniform
// across the batch. Fronts are dense (column-major) in an HBM workspace; the
// parent gathers its children's update matrices (extend-add, fixed child
// order: deterministic, no atomics).
//
// Factor storage per supernode s (rows r, pivots c): the Cholesky panel
// [L11; L21] (r x c, column-major, lower part only). Solves use blocked
// substitution on it (32-column diagonal blocks solved by one warp from
// registers, the rest of the panel applied as coalesced GEMV updates), which
// keeps the backward stability of the CPU restatement's triangular solves
// (explicit L11^{-1} panels lost ~1e-9 on ill-conditioned cut subdomains).
// Non-positive pivots are reported with the offending (subdomain, slot), the
// pivot rule of linalg.cpp:42-54.
#include <algorithm>

#include "factor.cuh"
#include "subst.cuh"

namespace cutbddc_b200 {
namespace {

constexpr int kFactorThreads = 256;

__device__ inline double entry_value(const FactorInput& in, int64_t sdT, int u, int k) {
  // value of A(v, u), v = u + offset(k), in the masked/augmented matrix
  const int b1 = in.b1;
  const int ux = u / (b1 * b1), uy = (u / b1) % b1, uz = u % b1;
  const int v = ((ux + k / 9 - 1) * b1 + (uy + (k / 3) % 3 - 1)) * b1 + (uz + k % 3 - 1);
  const bool mu = in.mask[sdT + u], mv = in.mask[sdT + v];
  if (!(mu && mv)) return k == 13 ? 1.0 : 0.0;
  double a = in.As[(sdT / in.T) * 27 * in.T + (int64_t)k * in.T + u];
  if (k == 13 && in.diag_add) a += in.diag_add[sdT + u];
  return a;
}

__global__ void __launch_bounds__(kFactorThreads) k_factor_level(TplDev t, const int32_t* __restrict__ level_sn,
                                                                 FactorInput in, int sd0, double* __restrict__ front,
                                                                 double* __restrict__ G, unsigned long long* fail) {
  const int sid = level_sn[blockIdx.x];
  const Supernode sn = t.sn[sid];
  const int sdl = blockIdx.y;          // within chunk
  const int sd = sd0 + sdl;
  const int64_t sdT = (int64_t)sd * t.T;
  const int r = sn.nrows, c = sn.ncols;
  double* F = front + (int64_t)sdl * t.front_total + sn.front_off;
  const int tid = threadIdx.x;
  for (int64_t q = tid; q < (int64_t)r * r; q += blockDim.x) F[q] = 0.0;
  __syncthreads();
  for (int q = tid; q < sn.amap_len; q += blockDim.x) {
    const AmapEntry e = t.amap[sn.amap_off + q];
    F[e.pos] = entry_value(in, sdT, e.slot, e.k);
  }
  __syncthreads();
  if (sid == t.root && in.c_ptr) {
    // rho c c^T of every edge/face constraint row; objects are disjoint, so
    // every (p, q) pair of a row hits a distinct front entry.
    const double rho = in.rho[sd];
    for (int64_t row = in.m_off[sd]; row < in.m_off[sd + 1]; ++row) {
      if (in.corner[row]) continue;
      const int64_t p0 = in.c_ptr[row];
      const int len = (int)(in.c_ptr[row + 1] - p0);
      for (int q = tid; q < len * len; q += blockDim.x) {
        const int a = q / len, b = q % len;
        const int pa = t.root_pos[in.c_slot[p0 + a]], pb = t.root_pos[in.c_slot[p0 + b]];
        if (pa < pb) continue;
        F[pa + (int64_t)pb * r] += rho * in.c_val[p0 + a] * in.c_val[p0 + b];
      }
    }
    __syncthreads();
  }
  for (int ch = 0; ch < sn.nchild; ++ch) {
    const Supernode cs = t.sn[sn.child[ch]];
    const int rc = cs.nrows, cc = cs.ncols, nu = rc - cc;
    const double* U = front + (int64_t)sdl * t.front_total + cs.front_off;
    const int32_t* em = t.emap + cs.emap_off;
    for (int64_t q = tid; q < (int64_t)nu * nu; q += blockDim.x) {
      const int a = (int)(q % nu), b = (int)(q / nu);
      if (a < b) continue;
      const int pa = em[a], pb = em[b];
      const int row = max(pa, pb), col = min(pa, pb);
      F[row + (int64_t)col * r] += U[(cc + a) + (int64_t)(cc + b) * rc];
    }
    __syncthreads();
  }
  // right-looking partial Cholesky of the c pivot columns
  __shared__ double s_ljj;
  for (int j = 0; j < c; ++j) {
    if (tid == 0) {
      double d = F[j + (int64_t)j * r];
      if (!(d > 0.0)) {
        atomicMin(fail, (unsigned long long)(sdT + t.rows[sn.rows_off + j]));
        d = 1.0;
      }
      s_ljj = sqrt(d);
      F[j + (int64_t)j * r] = s_ljj;
    }
    __syncthreads();
    const double inv = 1.0 / s_ljj;
    for (int i = j + 1 + tid; i < r; i += blockDim.x) F[i + (int64_t)j * r] *= inv;
    __syncthreads();
    for (int k = j + 1; k < r; ++k) {
      const double lkj = F[k + (int64_t)j * r];
      if (lkj == 0.0) continue;
      for (int i = k + tid; i < r; i += blockDim.x) F[i + (int64_t)k * r] -= F[i + (int64_t)j * r] * lkj;
    }
    __syncthreads();
  }
  // panel [L11; L21] (lower part; the strict upper triangle of L11 is never read)
  double* P = G + (int64_t)sd * t.panel_total + sn.panel_off;
  for (int j = 0; j < c; ++j)
    for (int i = j + tid; i < r; i += blockDim.x) P[i + (int64_t)j * r] = F[i + (int64_t)j * r];
}

// forward elimination step: X holds b on entry (slot vectors), y on exit at
// cols; the update v_rest - L21 y goes to the parent through `upd`.
__global__ void __launch_bounds__(256) k_fwd_level(TplDev t, const int32_t* __restrict__ level_sn, int nsd,
                                                   const double* __restrict__ G, double* __restrict__ X,
                                                   double* __restrict__ upd, const int* __restrict__ skip) {
  if (skip && *skip) return;
  extern __shared__ double v[];
  const Supernode sn = t.sn[level_sn[blockIdx.x]];
  const int sd = blockIdx.y, rhs = blockIdx.z;
  const int r = sn.nrows, c = sn.ncols;
  double* x = X + ((int64_t)rhs * nsd + sd) * t.T;
  double* ub = upd + ((int64_t)rhs * nsd + sd) * t.upd_total;
  const int32_t* rows = t.rows + sn.rows_off;
  for (int i = threadIdx.x; i < r; i += blockDim.x) v[i] = i < c ? x[rows[i]] : 0.0;
  __syncthreads();
  for (int ch = 0; ch < sn.nchild; ++ch) {
    const Supernode cs = t.sn[sn.child[ch]];
    const int nu = cs.nrows - cs.ncols;
    const int32_t* em = t.emap + cs.emap_off;
    const double* cu = ub + cs.upd_off;
    for (int a = threadIdx.x; a < nu; a += blockDim.x) v[em[a]] += cu[a];
    __syncthreads();
  }
  panel_forward(G + (int64_t)sd * t.panel_total + sn.panel_off, r, c, v);
  for (int i = threadIdx.x; i < r; i += blockDim.x) {
    if (i < c)
      x[rows[i]] = v[i];
    else
      ub[sn.upd_off + (i - c)] = v[i];
  }
}

// backward substitution step: X holds y at cols of this level, final x at
// ancestors (rest rows). x_c = L11^{-T} (y - L21^T x_rest).
__global__ void __launch_bounds__(256) k_bwd_level(TplDev t, const int32_t* __restrict__ level_sn, int nsd,
                                                   const double* __restrict__ G, double* __restrict__ X,
                                                   const int* __restrict__ skip) {
  if (skip && *skip) return;
  extern __shared__ double w[];
  __shared__ double tile[32][33];
  const Supernode sn = t.sn[level_sn[blockIdx.x]];
  const int sd = blockIdx.y, rhs = blockIdx.z;
  const int r = sn.nrows, c = sn.ncols;
  double* x = X + ((int64_t)rhs * nsd + sd) * t.T;
  const int32_t* rows = t.rows + sn.rows_off;
  for (int i = threadIdx.x; i < r; i += blockDim.x) w[i] = x[rows[i]];
  __syncthreads();
  panel_backward(G + (int64_t)sd * t.panel_total + sn.panel_off, r, c, w, tile);
  for (int j = threadIdx.x; j < c; j += blockDim.x) x[rows[j]] = w[j];
}

}  // namespace

TplDev tpl_dev(const TplSet& ts, int slots) {
  TplDev t;
  t.sn = ts.sn.p;
  t.rows = ts.rows.p;
  t.amap = ts.amap.p;
  t.emap = ts.emap.p;
  t.root_pos = ts.root_pos.p;
  t.T = slots;
  t.root = (int)ts.tpl.sn.size() - 1;
  t.panel_total = ts.tpl.panel_total;
  t.front_total = ts.tpl.front_total;
  t.upd_total = ts.tpl.upd_total;
  return t;
}

void upload_template(cutbddc_gpu* h, TplSet& ts, bool shell_root) {
  cudaStream_t s = h->stream;
  ts.tpl = build_template(h->block, 27, shell_root);
  ts.sn.upload(ts.tpl.sn, s);
  ts.rows.upload(ts.tpl.rows, s);
  ts.amap.upload(ts.tpl.amap, s);
  ts.emap.upload(ts.tpl.emap.empty() ? std::vector<int32_t>{0} : ts.tpl.emap, s);
  ts.root_pos.upload(ts.tpl.root_pos, s);
  std::vector<int32_t> lv;
  ts.level_first.clear();
  ts.level_count.clear();
  for (auto& L : ts.tpl.levels) {
    ts.level_first.push_back((int)lv.size());
    ts.level_count.push_back((int)L.size());
    lv.insert(lv.end(), L.begin(), L.end());
  }
  ts.level_sn.upload(lv, s);
  ts.ready = true;
}

// Factor every subdomain's masked/augmented matrix into G (nsd * panel_total).
void factor_device(cutbddc_gpu* h, const TplSet& ts, const FactorInput& in, DevBuf<double>& G, const char* what) {
  cudaStream_t s = h->stream;
  const TplDev t = tpl_dev(ts, h->slots);
  G.alloc((size_t)h->nsd * ts.tpl.panel_total);
  // subdomain chunks bounded by a front-workspace budget (~4 GiB)
  const int64_t per = ts.tpl.front_total;
  int chunk = (int)std::max<int64_t>(1, std::min<int64_t>(h->nsd, (4ll << 30) / 8 / per));
  DevBuf<double> front;
  front.alloc((size_t)chunk * per);
  DevBuf<unsigned long long> fail;
  fail.alloc(1);
  CB_CUDA(cudaMemsetAsync(fail.p, 0xff, 8, s));
  const int nlev = (int)ts.level_first.size();
  for (int sd0 = 0; sd0 < h->nsd; sd0 += chunk) {
    const int nc = std::min(chunk, h->nsd - sd0);
    for (int L = nlev - 1; L >= 0; --L) {
      dim3 grid(ts.level_count[(size_t)L], nc);
      k_factor_level<<<grid, kFactorThreads, 0, s>>>(t, ts.level_sn.p + ts.level_first[(size_t)L], in, sd0, front.p,
                                                     G.p, fail.p);
      CB_LAUNCH();
    }
  }
  unsigned long long f = 0;
  CB_CUDA(cudaMemcpyAsync(&f, fail.p, 8, cudaMemcpyDeviceToHost, s));
  CB_CUDA(cudaStreamSynchronize(s));
  if (f != ~0ull) {
    const int64_t sd = (int64_t)(f / (unsigned long long)h->slots), slot = (int64_t)(f % (unsigned long long)h->slots);
    throw Failure(CUTBDDC_SINGULAR, std::string(what) + ": matrix is not positive definite (subdomain " +
                                        std::to_string(sd) + ", pivot slot " + std::to_string(slot) + ")");
  }
}

// In-place solve of nrhs x nsd slot vectors X ([rhs][sd][T]) with factor G.
void solve_device(cutbddc_gpu* h, const TplSet& ts, const DevBuf<double>& G, double* X, int nrhs, double* upd,
                  const int* skip) {
  cudaStream_t s = h->stream;
  const TplDev t = tpl_dev(ts, h->slots);
  const int nlev = (int)ts.level_first.size();
  const size_t shm = sizeof(double) * (size_t)ts.tpl.max_rows;
  for (int L = nlev - 1; L >= 0; --L) {
    dim3 grid(ts.level_count[(size_t)L], h->nsd, nrhs);
    k_fwd_level<<<grid, 256, shm, s>>>(t, ts.level_sn.p + ts.level_first[(size_t)L], h->nsd, G.p, X, upd, skip);
    CB_LAUNCH();
  }
  for (int L = 0; L < nlev; ++L) {
    dim3 grid(ts.level_count[(size_t)L], h->nsd, nrhs);
    k_bwd_level<<<grid, 256, shm, s>>>(t, ts.level_sn.p + ts.level_first[(size_t)L], h->nsd, G.p, X, skip);
    CB_LAUNCH();
  }
}

}  // namespace cutbddc_b200
