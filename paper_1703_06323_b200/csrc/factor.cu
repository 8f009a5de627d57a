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
#include <cstdlib>
#include <vector>

#include "dense_chol.cuh"
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
__device__ inline double stencil_value(const FactorInput& in, int sd, int u, int k) {
  double a = in.As[(int64_t)sd * 27 * in.T + (int64_t)k * in.T + u];
  if (k == 13 && in.diag_add) a += in.diag_add[(int64_t)sd * in.T + u];
  return a;
}

__global__ void __launch_bounds__(kThreads) k_factor_level(TplDev t, FactorDev f, const int32_t* __restrict__ level_sn,
                                                           FactorInput in, int sd0, const int64_t* __restrict__ front_off,
                                                           int64_t front_base0, const int64_t* __restrict__ front_base,
                                                           double* __restrict__ front, double* __restrict__ panel,
                                                           unsigned long long* fail) {
  const int sid = level_sn[blockIdx.x];
  if (t.is_split[sid]) return;  // large fronts: multi-CTA assembly + panel steps
  const Supernode s = t.sn[sid];
  const int sd = sd0 + blockIdx.y;
  const int2 rc = f.rc[(int64_t)sd * t.nsn + sid];
  const int r = rc.x, c = rc.y;
  if (r == 0) return;
  const int tid = threadIdx.x;
  double* F = front + (front_base[sd] - front_base0) + front_off[(int64_t)sd * t.nsn + sid];
  for (int64_t q = tid; q < (int64_t)r * r; q += blockDim.x) F[q] = 0.0;
  __syncthreads();
  // original entries: template (row, col) positions -> compact
  for (int q = tid; q < s.amap_len; q += blockDim.x) {
    const AmapEntry e = t.amap[s.amap_off + q];
    const int qr = e.pos % s.nrows, qc = e.pos / s.nrows;
    const int pr = pfx_at(f, t, sd, s, qr), pc = pfx_at(f, t, sd, s, qc);
    if (pr < 0 || pc < 0) continue;
    F[pr + (int64_t)pc * r] = stencil_value(in, sd, e.slot, e.k);
  }
  __syncthreads();
  if (sid == t.root && in.c_ptr) {
    // rho c c^T of every edge/face constraint row (objects are disjoint:
    // every (p, q) pair of a row hits a distinct entry)
    const double rho = in.rho[sd];
    for (int64_t row = in.m_off[sd]; row < in.m_off[sd + 1]; ++row) {
      if (in.corner[row]) continue;
      const int64_t p0 = in.c_ptr[row];
      const int len = (int)(in.c_ptr[row + 1] - p0);
      for (int q = tid; q < len * len; q += blockDim.x) {
        const int a = q / len, b = q % len;
        const int pa = pfx_at(f, t, sd, s, t.root_pos[in.c_slot[p0 + a]]);
        const int pb = pfx_at(f, t, sd, s, t.root_pos[in.c_slot[p0 + b]]);
        if (pa < pb || pa < 0 || pb < 0) continue;
        F[pa + (int64_t)pb * r] += rho * in.c_val[p0 + a] * in.c_val[p0 + b];
      }
    }
    __syncthreads();
  }
  // extend-add of the children's update matrices (the child-row map reuses
  // the shared memory of the Cholesky phase)
  __shared__ __align__(16) unsigned char smraw[sizeof(CholSmem)];
  static_assert(sizeof(CholSmem) >= 2048 * sizeof(int), "cmap does not fit");
  int* cmap = reinterpret_cast<int*>(smraw);
  for (int ch = 0; ch < s.nchild; ++ch) {
    const int cid = s.child[ch];
    const Supernode cs = t.sn[cid];
    const int2 crc = f.rc[(int64_t)sd * t.nsn + cid];
    const int rcc = crc.x, ccc = crc.y, nu = rcc - ccc;
    if (nu <= 0) continue;
    // compact child rest row -> compact parent row
    for (int a = tid; a < cs.nrows - cs.ncols; a += blockDim.x) {
      const int ia = pfx_at(f, t, sd, cs, cs.ncols + a);
      if (ia >= 0) cmap[ia - ccc] = pfx_at(f, t, sd, s, t.emap[cs.emap_off + a]);
    }
    __syncthreads();
    const double* U = front + (front_base[sd] - front_base0) + front_off[(int64_t)sd * t.nsn + cid];
    for (int64_t q = tid; q < (int64_t)nu * nu; q += blockDim.x) {
      const int a = (int)(q % nu), b = (int)(q / nu);
      if (a < b) continue;
      const int pa = cmap[a], pb = cmap[b];
      const int row = max(pa, pb), col = min(pa, pb);
      F[row + (int64_t)col * r] += U[(ccc + a) + (int64_t)(ccc + b) * rcc];
    }
    __syncthreads();
  }
  // blocked right-looking partial Cholesky of the c pivot columns
  CholSmem& sm = *reinterpret_cast<CholSmem*>(smraw);
  front_partial_cholesky(F, r, c, sm, [&](int j) {
    // report the template slot of compact column j
    for (int q = 0; q < s.ncols; ++q)
      if (pfx_at(f, t, sd, s, q) == j) {
        atomicMin(fail, (unsigned long long)((int64_t)sd * t.T + t.rows[s.rows_off + q]));
        break;
      }
  });
  __syncthreads();
  if (t.is_big[sid]) return;  // big fronts: G panel written by k_trinv / k_gemm_m
  double* P = panel + f.panel_off[(int64_t)sd * t.nsn + sid];
  for (int j = 0; j < c; ++j)
    for (int i = j + tid; i < r; i += blockDim.x) P[i + (int64_t)j * r] = F[i + (int64_t)j * r];
}

// ---------------------------------------------------------------- split fronts
// Large fronts (template rows >= kSplitRows) are factorised by three
// launches per 32-column panel step so that many CTAs share one front:
// (1) the diagonal block, (2) the panel rows below it in 128-row chunks,
// (3) the rank-32 update of the trailing lower triangle in 64x64 tiles.
// (CUTBDDC_SPLIT_ROWS overrides, for measurements)
static const int kSplitRows = [] {
  const char* e = std::getenv("CUTBDDC_SPLIT_ROWS");
  return e ? std::max(64, std::atoi(e)) : 600;
}();

struct SplitArgs {
  const int32_t* sn;          // split supernodes of this level
  int sd0;
  const int64_t* front_off;
  int64_t front_base0;
  const int64_t* front_base;
  double* front;
  unsigned long long* fail;
};

__device__ inline double* split_front(const TplDev& t, const FactorDev& f, const SplitArgs& a, int sid, int sd) {
  return a.front + (a.front_base[sd] - a.front_base0) + a.front_off[(int64_t)sd * t.nsn + sid];
}

// Multi-CTA assembly of split fronts: zero, original entries, rho c c^T
// (root), then each child's update matrix (one launch per child; the entries
// of one child map to distinct parent entries).
__global__ void __launch_bounds__(256) k_split_zero(TplDev t, FactorDev f, SplitArgs a) {
  const int sid = a.sn[blockIdx.y];
  const int sd = a.sd0 + blockIdx.z;
  const int r = f.rc[(int64_t)sd * t.nsn + sid].x;
  double* F = split_front(t, f, a, sid, sd);
  // lower triangle only (nothing reads the strict upper part of a split front)
  for (int j = blockIdx.x; j < r; j += gridDim.x)
    for (int i = j + threadIdx.x; i < r; i += blockDim.x) F[i + (int64_t)j * r] = 0.0;
}

__global__ void __launch_bounds__(256) k_split_amap(TplDev t, FactorDev f, SplitArgs a, FactorInput in) {
  const int sid = a.sn[blockIdx.y];
  const int sd = a.sd0 + blockIdx.z;
  const Supernode s = t.sn[sid];
  const int r = f.rc[(int64_t)sd * t.nsn + sid].x;
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= s.amap_len || r == 0) return;
  const AmapEntry e = t.amap[s.amap_off + q];
  const int pr = pfx_at(f, t, sd, s, e.pos % s.nrows), pc = pfx_at(f, t, sd, s, e.pos / s.nrows);
  if (pr < 0 || pc < 0) return;
  split_front(t, f, a, sid, sd)[pr + (int64_t)pc * r] = stencil_value(in, sd, e.slot, e.k);
}

__global__ void __launch_bounds__(256) k_split_penalty(TplDev t, FactorDev f, SplitArgs a, FactorInput in) {
  const int sid = a.sn[blockIdx.y];
  if (sid != t.root || !in.c_ptr) return;
  const int sd = a.sd0 + blockIdx.z;
  const int64_t row = in.m_off[sd] + blockIdx.x;
  if (row >= in.m_off[sd + 1] || in.corner[row]) return;
  const Supernode s = t.sn[sid];
  const int r = f.rc[(int64_t)sd * t.nsn + sid].x;
  double* F = split_front(t, f, a, sid, sd);
  const double rho = in.rho[sd];
  const int64_t p0 = in.c_ptr[row];
  const int len = (int)(in.c_ptr[row + 1] - p0);
  for (int q = threadIdx.x; q < len * len; q += blockDim.x) {
    const int x = q / len, y = q % len;
    const int pa = pfx_at(f, t, sd, s, t.root_pos[in.c_slot[p0 + x]]);
    const int pb = pfx_at(f, t, sd, s, t.root_pos[in.c_slot[p0 + y]]);
    if (pa < pb || pa < 0 || pb < 0) continue;
    F[pa + (int64_t)pb * r] += rho * in.c_val[p0 + x] * in.c_val[p0 + y];
  }
}

// umap (sweep.cu: parent compact row of every update entry) places the
// child's update matrix; one CTA per update column, threads down the column.
__global__ void __launch_bounds__(256) k_split_extend(TplDev t, FactorDev f, SplitArgs a, int ch,
                                                      const int32_t* __restrict__ umap) {
  const int sid = a.sn[blockIdx.y];
  const int sd = a.sd0 + blockIdx.z;
  const Supernode s = t.sn[sid];
  if (ch >= s.nchild) return;
  const int cid = s.child[ch];
  const int64_t cf = (int64_t)sd * t.nsn + cid;
  const int2 crc = f.rc[cf];
  const int rcc = crc.x, ccc = crc.y, nu = rcc - ccc;
  if (nu <= 0) return;
  const int r = f.rc[(int64_t)sd * t.nsn + sid].x;
  double* F = split_front(t, f, a, sid, sd);
  const double* U = split_front(t, f, a, cid, sd);
  const int32_t* um = umap + f.upd_off[cf];
  for (int y = blockIdx.x; y < nu; y += gridDim.x) {
    const int py = um[y];
    const double* uc = U + ccc + (int64_t)(ccc + y) * rcc;
    for (int x = y + threadIdx.x; x < nu; x += blockDim.x) {
      const int px = um[x];
      const int row = max(px, py), col = min(px, py);
      F[row + (int64_t)col * r] += uc[x];
    }
  }
}

__global__ void __launch_bounds__(32) k_split_diag(TplDev t, FactorDev f, SplitArgs a, int k) {
  const int sid = a.sn[blockIdx.x];
  const int sd = a.sd0 + blockIdx.y;
  const int2 rc = f.rc[(int64_t)sd * t.nsn + sid];
  const int r = rc.x, c = rc.y;
  if (k >= c) return;
  const int nb = min(32, c - k);
  double* F = split_front(t, f, a, sid, sd);
  __shared__ double d[32][33];
  const int lane = threadIdx.x;
  for (int j = 0; j < nb; ++j) d[lane][j] = (lane < nb && lane >= j) ? F[(k + lane) + (int64_t)(k + j) * r] : 0.0;
  __syncwarp();
  for (int j = 0; j < nb; ++j) {
    double djj = d[j][j];
    if (lane == 0 && !(djj > 0.0)) {
      const Supernode s = t.sn[sid];
      for (int q = 0; q < s.ncols; ++q)
        if (f.pfx[(int64_t)sd * t.rows_total + s.rows_off + q] == k + j) {
          atomicMin(a.fail, (unsigned long long)((int64_t)sd * t.T + t.rows[s.rows_off + q]));
          break;
        }
    }
    if (!(djj > 0.0)) djj = 1.0;
    const double l = sqrt(djj);
    __syncwarp();
    if (lane == j) d[j][j] = l;
    if (lane > j && lane < nb) d[lane][j] /= l;
    __syncwarp();
    if (lane > j && lane < nb) {
      const double lij = d[lane][j];
      for (int q = j + 1; q <= lane; ++q) d[lane][q] -= lij * d[q][j];
    }
    __syncwarp();
  }
  for (int j = 0; j < nb; ++j)
    if (lane < nb && lane >= j) F[(k + lane) + (int64_t)(k + j) * r] = d[lane][j];
}

__global__ void __launch_bounds__(128) k_split_trsm(TplDev t, FactorDev f, SplitArgs a, int k) {
  const int sid = a.sn[blockIdx.y];
  const int sd = a.sd0 + blockIdx.z;
  const int2 rc = f.rc[(int64_t)sd * t.nsn + sid];
  const int r = rc.x, c = rc.y;
  if (k >= c) return;
  const int nb = min(32, c - k);
  const int i = k + nb + blockIdx.x * 128 + threadIdx.x;
  double* F = split_front(t, f, a, sid, sd);
  __shared__ double d[32][33];
  __shared__ double inv[32];
  for (int q = threadIdx.x; q < 32 * 32; q += blockDim.x) {
    const int ii = q & 31, jj = q >> 5;
    d[ii][jj] = (ii < nb && jj < nb && ii >= jj) ? F[(k + ii) + (int64_t)(k + jj) * r] : 0.0;
  }
  __syncthreads();
  if (threadIdx.x < 32) inv[threadIdx.x] = threadIdx.x < nb ? 1.0 / d[threadIdx.x][threadIdx.x] : 0.0;
  __syncthreads();
  if (i >= r) return;
  double x[32];
#pragma unroll
  for (int q = 0; q < 32; ++q) x[q] = q < nb ? F[i + (int64_t)(k + q) * r] : 0.0;
#pragma unroll
  for (int q = 0; q < 32; ++q) {
    if (q < nb) {
      double s = x[q];
#pragma unroll
      for (int u = 0; u < q; ++u) s -= x[u] * d[q][u];
      x[q] = s * inv[q];
    }
  }
#pragma unroll
  for (int q = 0; q < 32; ++q)
    if (q < nb) F[i + (int64_t)(k + q) * r] = x[q];
}

__global__ void __launch_bounds__(256) k_split_syrk(TplDev t, FactorDev f, SplitArgs a, int k) {
  const int sid = a.sn[blockIdx.y];
  const int sd = a.sd0 + blockIdx.z;
  const int2 rc = f.rc[(int64_t)sd * t.nsn + sid];
  const int r = rc.x, c = rc.y;
  if (k >= c) return;
  const int nb = min(32, c - k);
  const int m0 = k + nb;
  // tile pair (ti >= tj) from the linear index
  const int q = blockIdx.x;
  int ti = (int)((sqrt(8.0 * q + 1.0) - 1.0) * 0.5);
  while ((ti + 1) * (ti + 2) / 2 <= q) ++ti;
  while (ti * (ti + 1) / 2 > q) --ti;
  const int tj = q - ti * (ti + 1) / 2;
  const int i0 = m0 + ti * 64, j0 = m0 + tj * 64;
  if (i0 >= r) return;
  double* F = split_front(t, f, a, sid, sd);
  __shared__ double pi[32][64], pj[32][64];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  for (int e = tid; e < 32 * 64; e += blockDim.x) {
    const int rr = e & 63, kk = e >> 6;
    const int i = i0 + rr, j = j0 + rr;
    pi[kk][rr] = (kk < nb && i < r) ? F[i + (int64_t)(k + kk) * r] : 0.0;
    pj[kk][rr] = (kk < nb && j < r) ? F[j + (int64_t)(k + kk) * r] : 0.0;
  }
  __syncthreads();
  double acc[4][4];
#pragma unroll
  for (int x = 0; x < 4; ++x)
#pragma unroll
    for (int y = 0; y < 4; ++y) acc[x][y] = 0.0;
  for (int kk = 0; kk < nb; ++kk) {
    double pa[4], pb[4];
#pragma unroll
    for (int x = 0; x < 4; ++x) pa[x] = pi[kk][tx + 16 * x];
#pragma unroll
    for (int y = 0; y < 4; ++y) pb[y] = pj[kk][ty + 16 * y];
#pragma unroll
    for (int x = 0; x < 4; ++x)
#pragma unroll
      for (int y = 0; y < 4; ++y) acc[x][y] += pa[x] * pb[y];
  }
#pragma unroll
  for (int y = 0; y < 4; ++y) {
    const int j = j0 + ty + 16 * y;
    if (j >= r) continue;
#pragma unroll
    for (int x = 0; x < 4; ++x) {
      const int i = i0 + tx + 16 * x;
      if (i >= r || i < j) continue;
      F[i + (int64_t)j * r] -= acc[x][y];
    }
  }
}

// Big fronts: X = L11^{-1} into the top c x c block of the G panel, one CTA
// per (32-column right-hand-side block, front). Left-looking over 32-row
// blocks: acc = E - sum_k L[ib,kb] X[kb,:] (32^3 tiles in shared memory),
// then a 32x32 triangular solve with 32 right-hand sides.
__global__ void __launch_bounds__(256) k_trinv(TplDev t, FactorDev f, const int2* __restrict__ items, int sd0,
                                               const int64_t* __restrict__ front_off, int64_t front_base0,
                                               const int64_t* __restrict__ front_base, const double* __restrict__ front,
                                               double* __restrict__ panel, int skip_split) {
  const int2 it = items[blockIdx.x];
  const int sid = it.x, jb = it.y;
  if (skip_split && t.is_split[sid]) return;  // G written by the dense DAG (dense_dag.cu)
  const int sd = sd0 + blockIdx.y;
  const int2 rc = f.rc[(int64_t)sd * t.nsn + sid];
  const int r = rc.x, c = rc.y;
  const int j0 = jb * 32;
  if (j0 >= c) return;
  const int nb = min(32, c - j0);
  const double* L = front + (front_base[sd] - front_base0) + front_off[(int64_t)sd * t.nsn + sid];
  double* X = panel + f.panel_off[(int64_t)sd * t.nsn + sid];
  __shared__ double lt[32][33], xt[32][33], ab[32][33];
  const int tid = threadIdx.x, ti = tid & 31, tj = tid >> 5;  // 8 groups of 4 rhs columns
  // zero the strictly upper part of this column block (rows < j0)
  for (int q = tid; q < j0 * nb; q += blockDim.x) X[(q % j0) + (int64_t)(j0 + q / j0) * r] = 0.0;
  for (int i0 = j0; i0 < c; i0 += 32) {
    const int mb = min(32, c - i0);
    double acc[4];
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      const int j = tj + 8 * a;
      acc[a] = (i0 + ti == j0 + j) ? 1.0 : 0.0;
    }
    for (int k0 = j0; k0 < i0; k0 += 32) {
      for (int q = tid; q < 32 * 32; q += blockDim.x) {
        const int i = q & 31, k = q >> 5;
        lt[i][k] = (i < mb) ? L[(i0 + i) + (int64_t)(k0 + k) * r] : 0.0;
        xt[i][k] = (k < nb) ? X[(k0 + i) + (int64_t)(j0 + k) * r] : 0.0;  // xt[row k0+i][rhs k]
      }
      __syncthreads();
#pragma unroll 8
      for (int k = 0; k < 32; ++k) {
        const double l = lt[ti][k];
#pragma unroll
        for (int a = 0; a < 4; ++a) acc[a] -= l * xt[k][tj + 8 * a];
      }
      __syncthreads();
    }
#pragma unroll
    for (int a = 0; a < 4; ++a) ab[ti][tj + 8 * a] = acc[a];
    for (int q = tid; q < 32 * 32; q += blockDim.x) {
      const int i = q & 31, k = q >> 5;
      lt[i][k] = (i < mb && k < mb) ? L[(i0 + i) + (int64_t)(i0 + k) * r] : 0.0;
    }
    __syncthreads();
    if (tid < nb) {
      const int j = tid;
      for (int i = 0; i < mb; ++i) {
        double s = ab[i][j];
        for (int k = 0; k < i; ++k) s -= lt[i][k] * ab[k][j];
        ab[i][j] = s / lt[i][i];
      }
      for (int i = 0; i < mb; ++i) X[(i0 + i) + (int64_t)(j0 + j) * r] = ab[i][j];
    }
    __syncthreads();
  }
}

// Big fronts: M = L21 X into rows c..r of the G panel (64x64 output tiles,
// k loop from the tile's first column: X is lower triangular).
__global__ void __launch_bounds__(256) k_gemm_m(TplDev t, FactorDev f, const int2* __restrict__ items, int sd0,
                                                const int64_t* __restrict__ front_off, int64_t front_base0,
                                                const int64_t* __restrict__ front_base, const double* __restrict__ front,
                                                double* __restrict__ panel, int skip_split) {
  const int2 it = items[blockIdx.x];
  const int sid = it.x;
  if (skip_split && t.is_split[sid]) return;  // G written by the dense DAG (dense_dag.cu)
  const int sd = sd0 + blockIdx.y;
  const int2 rc = f.rc[(int64_t)sd * t.nsn + sid];
  const int r = rc.x, c = rc.y, m = r - c;
  const int ncb = (c + 63) / 64;
  if (ncb == 0) return;
  const int tiI = it.y / ncb, tiJ = it.y % ncb;
  const int i0 = c + tiI * 64, j0 = tiJ * 64;
  if (tiI * 64 >= m || j0 >= c) return;
  const double* L = front + (front_base[sd] - front_base0) + front_off[(int64_t)sd * t.nsn + sid];
  double* G = panel + f.panel_off[(int64_t)sd * t.nsn + sid];
  __shared__ double la[32][64];  // [k][row]
  __shared__ double xb[32][64];  // [k][col]
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  double acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
  for (int k0 = j0; k0 < c; k0 += 32) {
    for (int q = tid; q < 32 * 64; q += blockDim.x) {
      const int ii = q & 63, k = q >> 6;
      const int i = i0 + ii, kk = k0 + k, j = j0 + ii;
      la[k][ii] = (i < r && kk < c) ? L[i + (int64_t)kk * r] : 0.0;
      xb[k][ii] = (j < c && kk < c && kk >= j) ? G[kk + (int64_t)j * r] : 0.0;
    }
    __syncthreads();
#pragma unroll 4
    for (int k = 0; k < 32; ++k) {
      double pa[4], pb[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) pa[a] = la[k][tx + 16 * a];
#pragma unroll
      for (int b = 0; b < 4; ++b) pb[b] = xb[k][ty + 16 * b];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] += pa[a] * pb[b];
    }
    __syncthreads();
  }
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const int i = i0 + tx + 16 * a;
    if (i >= r) continue;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int j = j0 + ty + 16 * b;
      if (j < c) G[i + (int64_t)j * r] = acc[a][b];
    }
  }
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
constexpr int kLeafMax = 125;  // cfg4: 27 -> 125 cut the apply's solve time 744 -> 668 us
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
  t.is_split = ts.split_flag.p;
  t.T = slots;
  t.nsn = (int)ts.tpl.sn.size();
  t.root = t.nsn - 1;
  t.rows_total = (int64_t)ts.tpl.rows.size();
  return t;
}

FactorDev factor_dev(const FactorSet& f) {
  return FactorDev{f.pfx.p, f.tpos.p, f.rc.p, f.panel_off.p, f.upd_off.p, f.upd_total};
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
  std::vector<int2> fwd, bwd, inv, gem;
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
  ts.inv_first.clear();
  ts.inv_count.clear();
  ts.gemm_first.clear();
  ts.gemm_count.clear();
  ts.is_big.assign(ts.tpl.sn.size(), 0);
  std::vector<uint8_t> is_split(ts.tpl.sn.size(), 0);
  std::vector<int32_t> split;
  ts.split_first.clear();
  ts.split_count.clear();
  ts.split_maxc.clear();
  ts.split_maxr.clear();
  for (auto& L : ts.tpl.levels) {
    ts.split_first.push_back((int)split.size());
    int maxc = 0, maxr = 0;
    for (int sid : L) {
      const Supernode& sn = ts.tpl.sn[(size_t)sid];
      if (sn.nrows >= kSplitRows) {
        is_split[(size_t)sid] = 1;
        split.push_back(sid);
        maxc = std::max(maxc, sn.ncols);
        maxr = std::max(maxr, sn.nrows);
      }
    }
    ts.split_count.push_back((int)split.size() - ts.split_first.back());
    ts.split_maxc.push_back(maxc);
    ts.split_maxr.push_back(maxr);
  }
  for (auto& L : ts.tpl.levels) {
    ts.level_first.push_back((int)lv.size());
    ts.level_count.push_back((int)L.size());
    lv.insert(lv.end(), L.begin(), L.end());
    ts.small_first.push_back((int)small.size());
    ts.big_first.push_back((int)big.size());
    ts.fwd_first.push_back((int)fwd.size());
    ts.bwd_first.push_back((int)bwd.size());
    ts.inv_first.push_back((int)inv.size());
    ts.gemm_first.push_back((int)gem.size());
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
      for (int ch = 0; ch < (sn.ncols + 31) / 32; ++ch) inv.push_back(make_int2(sid, ch));
      const int tiles = ((sn.nrows - sn.ncols + 63) / 64) * ((sn.ncols + 63) / 64);
      for (int ch = 0; ch < tiles; ++ch) gem.push_back(make_int2(sid, ch));
    }
    ts.small_count.push_back((int)small.size() - ts.small_first.back());
    ts.big_count.push_back((int)big.size() - ts.big_first.back());
    ts.fwd_count.push_back((int)fwd.size() - ts.fwd_first.back());
    ts.bwd_count.push_back((int)bwd.size() - ts.bwd_first.back());
    ts.inv_count.push_back((int)inv.size() - ts.inv_first.back());
    ts.gemm_count.push_back((int)gem.size() - ts.gemm_first.back());
  }
  auto nz32 = [](std::vector<int32_t> v) { return v.empty() ? std::vector<int32_t>{0} : v; };
  auto nz2 = [](std::vector<int2> v) { return v.empty() ? std::vector<int2>{make_int2(0, 0)} : v; };
  ts.level_sn.upload(lv, s);
  ts.small_sn.upload(nz32(small), s);
  ts.big_sn.upload(nz32(big), s);
  ts.fwd_items.upload(nz2(fwd), s);
  ts.bwd_items.upload(nz2(bwd), s);
  ts.inv_items.upload(nz2(inv), s);
  ts.gemm_items.upload(nz2(gem), s);
  ts.big_flag.upload(ts.is_big, s);
  ts.split_flag.upload(is_split, s);
  ts.split_sn.upload(nz32(split), s);
  ts.ready = true;
}

double sweep_bytes(const FactorSet& f) { return f.bytes_per_sweep; }

// device bytes of the (grow-only, reusable) front workspace already held
static int64_t front_bytes_held(const cutbddc_gpu* h) { return (int64_t)h->ws_front.cap * (int64_t)sizeof(double); }

// Symbolic (compact structure) + numeric factorisation of every subdomain.
void factor_device(cutbddc_gpu* h, const TplSet& ts, const FactorInput& in, FactorSet& f, const char* what) {
  cudaStream_t s = h->stream;
  const TplDev t = tpl_dev(ts, h->slots);
  const int nsd = h->nsd, nsn = t.nsn;
  // symbolic: compact rows per (sd, supernode)
  f.pfx.alloc((size_t)nsd * t.rows_total);
  f.tpos.alloc((size_t)nsd * t.rows_total);
  f.rc.alloc((size_t)nsd * nsn);
  ProfScope psym(h->prof, s, std::string("factor") + (&ts == &h->tI ? "I" : "K") + " total");
  ProfScope pplan(h->prof, s, std::string("factor") + (&ts == &h->tI ? "I" : "K") + " symbolic+plan");
  k_symbolic<<<dim3(nsn, nsd), kThreads, 0, s>>>(t, nsd, in.mask, f.pfx.p, f.tpos.p, f.rc.p);
  CB_LAUNCH();
  f.h_rc = f.rc.to_host(s);
  std::vector<int64_t> poff((size_t)nsd * nsn), uoff((size_t)nsd * nsn), foff((size_t)nsd * nsn);
  f.h_front_base.assign((size_t)nsd + 1, 0);
  int64_t pt = 0, ut = 0;
  double bytes = 0, flops = 0;
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
    }
    f.h_front_base[(size_t)sd + 1] = f.h_front_base[(size_t)sd] + fo;
  }
  f.panel_total = pt;
  f.upd_total = ut;
  f.bytes_per_sweep = bytes;
  f.flops = flops;
  f.panel_off.upload(poff, s);
  f.h_panel_off = poff;
  f.upd_off.upload(uoff, s);
  f.front_off.upload(foff, s);
  DevBuf<int64_t>& fbase = h->ws_fbase;
  fbase.upload(f.h_front_base, s);
  f.panel.alloc((size_t)std::max<int64_t>(1, pt));
  build_sweep_plan(h, ts, f, poff, uoff);
  pplan.close();
  const FactorDev fd = factor_dev(f);
  // numeric, in subdomain chunks bounded by a front-workspace budget: half
  // of the free device memory (every chunk repeats the levels' critical paths)
  size_t free_b = 0, total_b = 0;
  CB_CUDA(cudaMemGetInfo(&free_b, &total_b));
  const int64_t budget = std::max<int64_t>((1ll << 30) / 8, (int64_t)(free_b / 2 + front_bytes_held(h)) / 8);
  DevBuf<unsigned long long>& fail = h->ws_fail;
  fail.alloc(1);
  CB_CUDA(cudaMemsetAsync(fail.p, 0xff, 8, s));
  DevBuf<double>& front = h->ws_front;
  const int nlev = (int)ts.level_first.size();
  static const int use_dag = [] {  // CUTBDDC_SPLIT_STEPS=1: the 32-column panel steps (A/B measurement)
    const char* e = std::getenv("CUTBDDC_SPLIT_STEPS");
    return e && e[0] == '1' ? 0 : 1;
  }();
  int sd0 = 0;
  while (sd0 < nsd) {
    int sd1 = sd0 + 1;
    while (sd1 < nsd && f.h_front_base[(size_t)sd1 + 1] - f.h_front_base[(size_t)sd0] <= budget) ++sd1;
    const int64_t need = f.h_front_base[(size_t)sd1] - f.h_front_base[(size_t)sd0];
    if ((int64_t)front.n < need) front.alloc((size_t)need);
    const std::string tag = std::string("factor") + (&ts == &h->tI ? "I" : "K") + " L";
    for (int L = nlev - 1; L >= 0; --L) {
      dim3 grid(ts.level_count[(size_t)L], sd1 - sd0);
      ProfScope ps0(h->prof, s, tag + std::to_string(L) + " all");
      k_factor_level<<<grid, kThreads, 0, s>>>(t, fd, ts.level_sn.p + ts.level_first[(size_t)L], in, sd0,
                                               f.front_off.p, f.h_front_base[(size_t)sd0], fbase.p, front.p, f.panel.p,
                                               fail.p);
      CB_LAUNCH();
      if (ts.split_count[(size_t)L] > 0) {
        ProfScope ps1(h->prof, s, tag + std::to_string(L) + " split");
        SplitArgs sa{ts.split_sn.p + ts.split_first[(size_t)L], sd0, f.front_off.p, f.h_front_base[(size_t)sd0],
                     fbase.p, front.p, fail.p};
        const int ns_ = ts.split_count[(size_t)L], nc_ = sd1 - sd0;
        const int maxc = ts.split_maxc[(size_t)L], maxr = ts.split_maxr[(size_t)L];
        int max_amap = 0, max_child_nu = 0;
        for (int sid : ts.tpl.levels[(size_t)L]) {
          const Supernode& sn = ts.tpl.sn[(size_t)sid];
          if (sn.nrows < kSplitRows) continue;
          max_amap = std::max(max_amap, sn.amap_len);
          for (int c2 = 0; c2 < sn.nchild; ++c2) {
            const Supernode& cs = ts.tpl.sn[(size_t)sn.child[c2]];
            max_child_nu = std::max(max_child_nu, cs.nrows - cs.ncols);
          }
        }
        k_split_zero<<<dim3(std::min(maxr, 512), ns_, nc_), 256, 0, s>>>(t, fd, sa);
        CB_LAUNCH();
        k_split_amap<<<dim3((max_amap + 255) / 256, ns_, nc_), 256, 0, s>>>(t, fd, sa, in);
        CB_LAUNCH();
        if (in.c_ptr && h->m_max > 0) {
          k_split_penalty<<<dim3(h->m_max, ns_, nc_), 256, 0, s>>>(t, fd, sa, in);
          CB_LAUNCH();
        }
        for (int c2 = 0; c2 < 2; ++c2) {
          k_split_extend<<<dim3(std::max(1, std::min(max_child_nu, 1024)), ns_, nc_), 256, 0, s>>>(t, fd, sa, c2,
                                                                                                   f.umap.p);
          CB_LAUNCH();
        }
        if (use_dag) {
          // tiled Cholesky + inverse panel of every split front (dense_dag.cu)
          std::vector<int> sids;
          for (int sid : ts.tpl.levels[(size_t)L])
            if (ts.tpl.sn[(size_t)sid].nrows >= kSplitRows) sids.push_back(sid);
          dense_dag_level(h, ts, f, sids, sd0, sd1, foff, poff, front.p, fail.p);
        } else {
          for (int k = 0; k < maxc; k += 32) {
            k_split_diag<<<dim3(ns_, nc_), 32, 0, s>>>(t, fd, sa, k);
            CB_LAUNCH();
            const int rows_below = maxr - k - 1;
            if (rows_below <= 0) continue;
            k_split_trsm<<<dim3((rows_below + 127) / 128, ns_, nc_), 128, 0, s>>>(t, fd, sa, k);
            CB_LAUNCH();
            const int nt = (rows_below + 63) / 64;
            k_split_syrk<<<dim3(nt * (nt + 1) / 2, ns_, nc_), 256, 0, s>>>(t, fd, sa, k);
            CB_LAUNCH();
          }
        }
      }
      if (ts.inv_count[(size_t)L] > 0) {
        ProfScope ps2(h->prof, s, tag + std::to_string(L) + " trinv");
        dim3 gi(ts.inv_count[(size_t)L], sd1 - sd0);
        k_trinv<<<gi, 256, 0, s>>>(t, fd, ts.inv_items.p + ts.inv_first[(size_t)L], sd0, f.front_off.p,
                                   f.h_front_base[(size_t)sd0], fbase.p, front.p, f.panel.p, use_dag);
        CB_LAUNCH();
      }
      if (ts.gemm_count[(size_t)L] > 0) {
        ProfScope ps3(h->prof, s, tag + std::to_string(L) + " gemm");
        dim3 gg(ts.gemm_count[(size_t)L], sd1 - sd0);
        k_gemm_m<<<gg, 256, 0, s>>>(t, fd, ts.gemm_items.p + ts.gemm_first[(size_t)L], sd0, f.front_off.p,
                                    f.h_front_base[(size_t)sd0], fbase.p, front.p, f.panel.p, use_dag);
        CB_LAUNCH();
      }
    }
    sd0 = sd1;
  }
  unsigned long long fl = 0;
  CB_CUDA(cudaMemcpyAsync(&fl, fail.p, 8, cudaMemcpyDeviceToHost, s));
  CB_CUDA(cudaStreamSynchronize(s));
  if (fl != ~0ull) {
    const int64_t sd = (int64_t)(fl / (unsigned long long)h->slots), slot = (int64_t)(fl % (unsigned long long)h->slots);
    throw Failure(CUTBDDC_SINGULAR, std::string(what) + ": matrix is not positive definite (subdomain " +
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
  const std::string tag = std::string("solve") + (&ts == &h->tI ? "I" : "K") + (nrhs > 1 ? "m " : " ");
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
