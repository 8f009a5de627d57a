// dist.cu — subdomains over ranks: the local dof space, the
// interface exchange plan and the exchange itself, segment partials, and the
// matrix-free sub-assembled operator (one constant Q1
// stencil for interior cells plus the stored 8x8 matrix of each cut cell;
// no assembled global matrix anywhere).
//
// Reference: the sum over subdomain copies is SPEC.md:393 ("sum the weighted
// subdomain corrections") and Abar = Σ_w R_w^T A_w R_w; the
// parallel contract is "independent parallel tasks joined by global
// reductions". The plan is built on the device from the mesh
// and the global partition every rank holds; host_partition.cpp has the same
// plan as host C++ (cutbddc_build_exchange_plan) for the CPU multi-process
// tests, and tests/test_gpu_dist.py checks the two agree entry for entry.
#include <cub/cub.cuh>

#include <algorithm>

#include "comm.cuh"
#include "dist.cuh"

namespace cutbddc_b200 {
namespace {

constexpr int kMaxRanks = 32;  // rank masks are 32-bit

// ---------------------------------------------------------------- plan kernels
struct PlanArgs {
  int n, B, nb, b1, T, rank;
  const uint8_t* cls;
  const int64_t* node_of_dof;
  const int32_t* gsd_of_block;   // nb^3: global subdomain or -1
  const int32_t* rank_of_gsd;
  const int32_t* lsd_of_gsd;     // local subdomain index or -1
  const int64_t* gblock;         // nsd_g: block id of each global subdomain
};

// per global dof: subdomains of its active cells (global ids ascending,
// padded with -1), whether this rank has a copy, its segment (local index of
// its lowest subdomain, or nsd for the ghost segment) and the rank mask
__global__ void k_dof_sds(int64_t nd, PlanArgs a, int nsd, int32_t* __restrict__ sds, uint8_t* __restrict__ nsds,
                          uint8_t* __restrict__ local, int32_t* __restrict__ seg, uint32_t* __restrict__ rmask) {
  const int64_t d = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (d >= nd) return;
  const int n = a.n;
  const int64_t v = a.node_of_dof[d];
  const int k = (int)(v % (n + 1)), j = (int)((v / (n + 1)) % (n + 1)), i = (int)(v / (n + 1) / (n + 1));
  int32_t s[8];
  int m = 0;
  for (int dx = 0; dx < 2; ++dx)
    for (int dy = 0; dy < 2; ++dy)
      for (int dz = 0; dz < 2; ++dz) {
        const int ci = i - 1 + dx, cj = j - 1 + dy, ck = k - 1 + dz;
        if (ci < 0 || cj < 0 || ck < 0 || ci >= n || cj >= n || ck >= n) continue;
        if (a.cls[((int64_t)ci * n + cj) * n + ck] == CUTBDDC_EXTERIOR) continue;
        const int32_t g = a.gsd_of_block[((int64_t)(ci / a.B) * a.nb + cj / a.B) * a.nb + ck / a.B];
        bool seen = false;
        for (int q = 0; q < m; ++q) seen |= s[q] == g;
        if (!seen) s[m++] = g;
      }
  for (int x = 1; x < m; ++x)  // ascending block id == ascending global subdomain
    for (int y = x; y > 0 && s[y - 1] > s[y]; --y) {
      const int32_t t = s[y];
      s[y] = s[y - 1];
      s[y - 1] = t;
    }
  uint32_t mask = 0;
  for (int q = 0; q < m; ++q) mask |= 1u << a.rank_of_gsd[s[q]];
  for (int q = 0; q < 8; ++q) sds[d * 8 + q] = q < m ? s[q] : -1;
  nsds[d] = (uint8_t)m;
  const bool loc = (mask >> a.rank) & 1u;
  local[d] = loc;
  seg[d] = m > 0 && a.rank_of_gsd[s[0]] == a.rank ? a.lsd_of_gsd[s[0]] : nsd;
  rmask[d] = loc ? mask : 0u;
}

__global__ void k_gather_i32(int64_t n, const int32_t* __restrict__ idx, const int32_t* __restrict__ src,
                             int32_t* __restrict__ dst) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) dst[i] = src[idx[i]];
}

__global__ void k_scatter_pos(int64_t n, const int32_t* __restrict__ idx, int32_t* __restrict__ pos) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) pos[idx[i]] = (int32_t)i;
}

// seg_ptr[s] = first position with key >= s (keys sorted)
__global__ void k_seg_ptr(int nseg, int64_t n, const int32_t* __restrict__ keys, int32_t* __restrict__ seg_ptr) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s > nseg) return;
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (keys[mid] < s) lo = mid + 1;
    else hi = mid;
  }
  seg_ptr[s] = (int32_t)lo;
}

__global__ void k_or_mask(int64_t nd, const uint32_t* __restrict__ rmask, unsigned int* __restrict__ out) {
  __shared__ unsigned int sm;
  if (threadIdx.x == 0) sm = 0;
  __syncthreads();
  unsigned int m = 0;
  for (int64_t d = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; d < nd; d += (int64_t)gridDim.x * blockDim.x)
    m |= rmask[d];
  atomicOr(&sm, m);
  __syncthreads();
  if (threadIdx.x == 0) atomicOr(out, sm);
}

__device__ inline int count_rank(const int32_t* s, const int32_t* rank_of_gsd, int q) {
  int c = 0;
  for (int x = 0; x < 8 && s[x] >= 0; ++x) c += rank_of_gsd[s[x]] == q;
  return c;
}

// per neighbour k, in ascending-global order j of the local dofs:
//   rc = copies on q (message q -> rank), sc = copies here if q has a copy (message rank -> q)
__global__ void k_nbr_counts(int64_t nloc, int nnbr, const int32_t* __restrict__ glist, const int32_t* __restrict__ sds,
                             const int32_t* __restrict__ rank_of_gsd, const int32_t* __restrict__ nbr, int rank,
                             int32_t* __restrict__ rc, int32_t* __restrict__ sc) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= nloc) return;
  const int32_t* s = sds + (int64_t)glist[j] * 8;
  const int mine = count_rank(s, rank_of_gsd, rank);
  for (int k = 0; k < nnbr; ++k) {
    const int c = count_rank(s, rank_of_gsd, nbr[k]);
    rc[(int64_t)k * nloc + j] = c;
    sc[(int64_t)k * nloc + j] = c > 0 ? mine : 0;
  }
}

__global__ void k_copy_count(int64_t nloc, const int32_t* __restrict__ loc_glob, const uint8_t* __restrict__ nsds,
                             int32_t* __restrict__ cnt) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < nloc) cnt[i] = nsds[loc_glob[i]];
}

__device__ inline int32_t slot_of(const PlanArgs& a, int64_t node, int32_t gsd) {
  const int n = a.n, B = a.B, b1 = a.b1;
  const int k = (int)(node % (n + 1)), j = (int)((node / (n + 1)) % (n + 1)), i = (int)(node / (n + 1) / (n + 1));
  const int64_t bid = a.gblock[gsd];
  const int bi = (int)(bid / a.nb / a.nb), bj = (int)((bid / a.nb) % a.nb), bk = (int)(bid % a.nb);
  return ((i - bi * B) * b1 + (j - bj * B)) * b1 + (k - bk * B);
}

// copy sources (ascending global subdomain) of every local dof, the send
// lists, and the owner slot of interior dofs; thread per local dof in
// ascending-global order j
__global__ void k_fill_plan(int64_t nloc, int nnbr, PlanArgs a, const int32_t* __restrict__ glist,
                            const int32_t* __restrict__ loc_of_dof, const int32_t* __restrict__ sds,
                            const int32_t* __restrict__ nbr_of_rank, const int32_t* __restrict__ rinc,
                            const int32_t* __restrict__ rcnt, const int32_t* __restrict__ sinc,
                            const int32_t* __restrict__ scnt, const int64_t* __restrict__ rbase,
                            const int64_t* __restrict__ sbase, const int32_t* __restrict__ cptr,
                            int32_t* __restrict__ csrc, int32_t* __restrict__ send_src, int32_t* __restrict__ lowner) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= nloc) return;
  const int32_t d = glist[j];
  const int32_t i = loc_of_dof[d];
  const int32_t* s = sds + (int64_t)d * 8;
  const int64_t node = a.node_of_dof[d];
  int pos_q[kMaxRanks];
  for (int q = 0; q < kMaxRanks; ++q) pos_q[q] = 0;
  int m = 0, mloc = 0;
  int32_t p = cptr[i];
  int32_t first_local = -1;
  for (; m < 8 && s[m] >= 0; ++m) {
    const int32_t g = s[m];
    const int q = a.rank_of_gsd[g];
    if (q == a.rank) {
      const int32_t src = a.lsd_of_gsd[g] * a.T + slot_of(a, node, g);
      csrc[p++] = src;
      if (first_local < 0) first_local = src;
      // this copy goes to every neighbour holding a copy, at position mloc
      for (int k = 0; k < nnbr; ++k) {
        const int64_t jj = (int64_t)k * nloc + j;
        if (scnt[jj] > 0) send_src[sbase[k] + (sinc[jj] - scnt[jj]) + mloc] = src;
      }
      ++mloc;
    } else {
      const int k = nbr_of_rank[q];
      const int64_t jj = (int64_t)k * nloc + j;
      csrc[p++] = -1 - (int32_t)(rbase[k] + (rinc[jj] - rcnt[jj]) + pos_q[q]);
      ++pos_q[q];
    }
  }
  lowner[i] = m == 1 ? first_local : -1;
}

__global__ void k_slot_loc(int64_t ns, const int32_t* __restrict__ slot_dof, const int32_t* __restrict__ loc_of_dof,
                           int32_t* __restrict__ slot_loc) {
  const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g >= ns) return;
  const int32_t d = slot_dof[g];
  slot_loc[g] = d >= 0 ? loc_of_dof[d] : -1;
}

// ---------------------------------------------------------------- exchange / sums
__global__ void k_pack(int64_t n, const int32_t* __restrict__ src, const double* __restrict__ w,
                       const double* __restrict__ Y, double* __restrict__ buf, const int* __restrict__ skip) {
  if (skip && *skip) return;
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= n) return;
  const int32_t s = src[k];
  buf[k] = w ? w[s] * Y[s] : Y[s];
}

// out[i] = Σ copies (ascending global sd); with Xs, the sum is also written
// to every local slot copy (the slot vector the operator reads next)
__global__ void k_isum(int64_t nloc, const int32_t* __restrict__ cptr, const int32_t* __restrict__ csrc,
                       const double* __restrict__ w, const double* __restrict__ Y, const double* __restrict__ recv,
                       double* __restrict__ out, double* __restrict__ Xs, const int* __restrict__ skip) {
  if (skip && *skip) return;
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= nloc) return;
  double s = 0.0;
  const int32_t p0 = cptr[i], p1 = cptr[i + 1];
  for (int32_t p = p0; p < p1; ++p) {
    const int32_t c = csrc[p];
    s += c >= 0 ? (w ? w[c] * Y[c] : Y[c]) : recv[-1 - c];
  }
  out[i] = s;
  if (Xs)
    for (int32_t p = p0; p < p1; ++p) {
      const int32_t c = csrc[p];
      if (c >= 0) Xs[c] = s;
    }
}

__global__ void k_to_local(int64_t nloc, const int32_t* __restrict__ loc_glob, const double* __restrict__ xg,
                           double* __restrict__ xl) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < nloc) xl[i] = xg[loc_glob[i]];
}

__global__ void k_to_global(int64_t nown, const int32_t* __restrict__ loc_glob, const double* __restrict__ xl,
                            double* __restrict__ xg) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < nown) xg[loc_glob[i]] = xl[i];
}

// ---------------------------------------------------------------- matrix-free operator
struct SubArgs {
  int n, B, b1, T, nb, nsd;
  const int64_t* block_ids;   // local subdomain -> block id
  const int32_t* eoc;         // per cell: -2 exterior, -1 interior, >= 0 local cut index
  const double* keS;          // cut-cell matrices, packed upper triangle, SoA: keS[36][ncut] (empty cells: 0)
  int64_t ncut;
  const double* kint;         // constant interior element matrix
  const int32_t* slot_loc;
  const uint8_t* mask_int;
  const double* odiag;        // per slot: 1/|neigh| at strong-Dirichlet slots, else 0
};

// cut-cell matrices (8x8 row-major per cell, symmetric) -> packed upper
// triangle SoA keS[36][ncut]
__global__ void k_pack_ke(int64_t ncut, const double* __restrict__ ke, double* __restrict__ keS) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= ncut) return;
  int p = 0;
  for (int i = 0; i < 8; ++i)
    for (int j = i; j < 8; ++j) keS[(int64_t)(p++) * ncut + e] = ke[e * 64 + i * 8 + j];
}

__global__ void k_iota(int64_t n, int32_t* __restrict__ a) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) a[i] = (int32_t)i;
}

// end of the kind 0 / 1 / 2 ranges in a sorted kind array (binary search)
__global__ void k_kind_counts(int64_t n, const uint8_t* __restrict__ kind, int64_t* __restrict__ out) {
  const int k = threadIdx.x;
  if (k >= 3) return;
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (kind[mid] <= k) lo = mid + 1;
    else hi = mid;
  }
  out[k] = lo;
}

// slot vector of a local dof vector (0 at absent slots)
__global__ void k_gather_slots(int64_t ns, const int32_t* __restrict__ slot_loc, const double* __restrict__ x,
                               double* __restrict__ X, const int* __restrict__ skip) {
  if (skip && *skip) return;
  const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g >= ns) return;
  const int32_t l = slot_loc[g];
  X[g] = l >= 0 ? x[l] : 0.0;
}

// Rows of the operator as one list of slots, [interior regular | interior
// irregular | interface] (ascending slots within each): a regular slot has
// all 8 cells inside its block and interior (the bulk), so its row is the
// constant 27-point stencil S27 of the Q1 element; every other row sums its
// cells' element rows. kSubInterior = [0, n_int), kSubInterface =
// [n_int, n_rows), kSubAll = [0, n_rows).
__global__ void k_slot_kind(int64_t ns, int T, int B, int b1, int n, int nb, const int64_t* __restrict__ block_ids,
                            const int32_t* __restrict__ eoc, const int32_t* __restrict__ slot_loc,
                            const uint8_t* __restrict__ mask_int, const double* __restrict__ odiag,
                            uint8_t* __restrict__ kind) {
  const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g >= ns) return;
  if (slot_loc[g] < 0) {
    kind[g] = 3;
    return;
  }
  if (!mask_int[g]) {
    kind[g] = 2;
    return;
  }
  const int sd = (int)(g / T), t = (int)(g - (int64_t)sd * T);
  const int P = b1 * b1, lx = t / P, ly = (t / b1) % b1, lz = t % b1;
  const int64_t bid = block_ids[sd];
  const int bi = (int)(bid / nb / nb), bj = (int)((bid / nb) % nb), bk = (int)(bid % nb);
  bool reg = odiag[g] == 0.0 && lx > 0 && ly > 0 && lz > 0 && lx < B && ly < B && lz < B;
  for (int c = 0; c < 8 && reg; ++c) {
    const int cx = lx - 1 + (c >> 2), cy = ly - 1 + ((c >> 1) & 1), cz = lz - 1 + (c & 1);
    reg = eoc[((int64_t)(bi * B + cx) * n + bj * B + cy) * n + bk * B + cz] == -1;
  }
  kind[g] = reg ? 0 : 1;
}

// S27[q]: the interior element rows summed onto the 27-point stencil (cells
// in (dx,dy,dz) order, nodes in bit order: a fixed order)
__global__ void k_stencil27(const double* __restrict__ kint, double* __restrict__ s27) {
  if (threadIdx.x != 0) return;
  for (int q = 0; q < 27; ++q) s27[q] = 0.0;
  for (int c = 0; c < 8; ++c) {
    const int dx = c >> 2, dy = (c >> 1) & 1, dz = c & 1;
    const int lv = (1 - dx) + 2 * (1 - dy) + 4 * (1 - dz);
    for (int w = 0; w < 8; ++w) s27[(dx + (w & 1)) * 9 + (dy + ((w >> 1) & 1)) * 3 + (dz + ((w >> 2) & 1))] += kint[lv * 8 + w];
  }
}

// partial of cell c (0..7, (dx,dy,dz) order) of the row at slot g: the
// cell's element row times its 8 node values (constant Q1 matrix for
// interior cells, the packed matrix of cut cells, 0 for exterior cells)
__device__ __forceinline__ double cell_part(const SubArgs& a, const double* __restrict__ ks, int64_t g, int c,
                                            const double* __restrict__ X) {
  const int T = a.T, B = a.B, b1 = a.b1, n = a.n, P = b1 * b1;
  const int sd = (int)(g / T), t = (int)(g - (int64_t)sd * T);
  const int lx = t / P, ly = (t / b1) % b1, lz = t % b1;
  const int dx = c >> 2, dy = (c >> 1) & 1, dz = c & 1;
  const int cx = lx - 1 + dx, cy = ly - 1 + dy, cz = lz - 1 + dz;
  double v = 0.0;
  if (cx < 0 || cy < 0 || cz < 0 || cx >= B || cy >= B || cz >= B) return v;
  const int64_t bid = a.block_ids[sd];
  const int bi = (int)(bid / a.nb / a.nb), bj = (int)((bid / a.nb) % a.nb), bk = (int)(bid % a.nb);
  const int32_t e = a.eoc[((int64_t)(bi * B + cx) * n + bj * B + cy) * n + bk * B + cz];
  const int lv = (1 - dx) + 2 * (1 - dy) + 4 * (1 - dz);
  const int64_t n0 = g + (dx - 1) * P + (dy - 1) * b1 + (dz - 1);  // node 0 of the cell
  if (e == -1) {
#pragma unroll
    for (int w = 0; w < 8; ++w) v += ks[lv * 8 + w] * X[n0 + (w & 1) * P + ((w >> 1) & 1) * b1 + ((w >> 2) & 1)];
  } else if (e >= 0) {
#pragma unroll
    for (int w = 0; w < 8; ++w) {
      const int i = lv < w ? lv : w, k = lv < w ? w : lv;  // packed upper-triangle index of (lv, w)
      v += a.keS[(int64_t)(i * 8 - i * (i - 1) / 2 + (k - i)) * a.ncut + e] *
           X[n0 + (w & 1) * P + ((w >> 1) & 1) * b1 + ((w >> 2) & 1)];
    }
  }
  return v;
}

// regular rows, a thread each: S27 on the 27 lattice neighbours (all 8
// cells interior, so every neighbour lies in the lattice)
__global__ void __launch_bounds__(256) k_sub_regular(const int32_t* __restrict__ rows, int64_t nreg, int P, int b1,
                                                     const double* __restrict__ s27, const double* __restrict__ X,
                                                     double* __restrict__ Y, const int* __restrict__ skip) {
  if (skip && *skip) return;
  __shared__ double ss[27];
  if (threadIdx.x < 27) ss[threadIdx.x] = s27[threadIdx.x];
  __syncthreads();
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= nreg) return;
  const int64_t g = rows[j];
  double acc = 0.0;
#pragma unroll
  for (int q = 0; q < 27; ++q) acc += ss[q] * X[g + (q / 9 - 1) * P + ((q / 3) % 3 - 1) * b1 + (q % 3 - 1)];
  Y[g] = acc;
}

// The other rows: the 8 cell partials combined by one fixed tree,
// ((p0+p4)+(p2+p6)) + ((p1+p5)+(p3+p7)). k_sub_cells8 runs 8 lanes per row
// (the xor tree; many-SM parallelism for few rows), k_sub_cells1 a thread
// per row: the same bits either way, so each rank may pick by its row count.
__global__ void __launch_bounds__(256) k_sub_cells8(SubArgs a, const int32_t* __restrict__ rows, int64_t lo, int64_t hi,
                                                    const double* __restrict__ X, double* __restrict__ Y,
                                                    const int* __restrict__ skip) {
  if (skip && *skip) return;
  __shared__ double ks[64];
  if (threadIdx.x < 64) ks[threadIdx.x] = a.kint[threadIdx.x];
  __syncthreads();
  const int64_t j = lo + (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / 8;
  const int c = threadIdx.x & 7;
  const bool live = j < hi;  // whole 8-lane groups are live or not: the shuffles stay convergent
  const int64_t g = live ? rows[j] : 0;
  double v = live ? cell_part(a, ks, g, c, X) : 0.0;
  v += __shfl_xor_sync(0xffffffffu, v, 4);
  v += __shfl_xor_sync(0xffffffffu, v, 2);
  v += __shfl_xor_sync(0xffffffffu, v, 1);
  if (live && c == 0) Y[g] = a.odiag ? v + a.odiag[g] * X[g] : v;
}

__global__ void __launch_bounds__(256) k_sub_cells1(SubArgs a, const int32_t* __restrict__ rows, int64_t lo, int64_t hi,
                                                    const double* __restrict__ X, double* __restrict__ Y,
                                                    const int* __restrict__ skip) {
  if (skip && *skip) return;
  __shared__ double ks[64];
  if (threadIdx.x < 64) ks[threadIdx.x] = a.kint[threadIdx.x];
  __syncthreads();
  const int64_t j = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= hi) return;
  const int64_t g = rows[j];
  double p[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) p[c] = cell_part(a, ks, g, c, X);
  const double v = ((p[0] + p[4]) + (p[2] + p[6])) + ((p[1] + p[5]) + (p[3] + p[7]));
  Y[g] = a.odiag ? v + a.odiag[g] * X[g] : v;
}

// Regular and irregular rows in one launch (the two row classes write disjoint
// entries of Y): blocks [0, nblk_reg) are k_sub_regular's, the rest
// k_sub_cells8's (kEight) or k_sub_cells1's, statement for statement, so the
// bits are those of the separate launches.
template <bool kEight>
__global__ void __launch_bounds__(256) k_sub_fused(SubArgs a, const int32_t* __restrict__ rows, int64_t nreg, int nblk_reg,
                                                   int P, int b1, const double* __restrict__ s27, int64_t lo, int64_t hi,
                                                   const double* __restrict__ X, double* __restrict__ Y,
                                                   const int* __restrict__ skip) {
  if (skip && *skip) return;
  __shared__ double ks[64];
  if ((int)blockIdx.x < nblk_reg) {
    if (threadIdx.x < 27) ks[threadIdx.x] = s27[threadIdx.x];
    __syncthreads();
    const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (j >= nreg) return;
    const int64_t g = rows[j];
    double acc = 0.0;
#pragma unroll
    for (int q = 0; q < 27; ++q) acc += ks[q] * X[g + (q / 9 - 1) * P + ((q / 3) % 3 - 1) * b1 + (q % 3 - 1)];
    Y[g] = acc;
    return;
  }
  if (threadIdx.x < 64) ks[threadIdx.x] = a.kint[threadIdx.x];
  __syncthreads();
  const int64_t t = ((int64_t)blockIdx.x - nblk_reg) * blockDim.x + threadIdx.x;
  if (kEight) {
    const int64_t j = lo + t / 8;
    const int c = threadIdx.x & 7;
    const bool live = j < hi;  // whole 8-lane groups are live or not: the shuffles stay convergent
    const int64_t g = live ? rows[j] : 0;
    double v = live ? cell_part(a, ks, g, c, X) : 0.0;
    v += __shfl_xor_sync(0xffffffffu, v, 4);
    v += __shfl_xor_sync(0xffffffffu, v, 2);
    v += __shfl_xor_sync(0xffffffffu, v, 1);
    if (live && c == 0) Y[g] = a.odiag ? v + a.odiag[g] * X[g] : v;
  } else {
    const int64_t j = lo + t;
    if (j >= hi) return;
    const int64_t g = rows[j];
    double p[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) p[c] = cell_part(a, ks, g, c, X);
    const double v = ((p[0] + p[4]) + (p[2] + p[6])) + ((p[1] + p[5]) + (p[3] + p[7]));
    Y[g] = a.odiag ? v + a.odiag[g] * X[g] : v;
  }
}

}  // namespace

// ---------------------------------------------------------------- distribution
static void dist_common(cutbddc_gpu* h, int block, int nsd_g, const int64_t* bids, const int32_t* rank_of_sd, int rank,
                        int world) {
  if (world < 1 || world > kMaxRanks) throw Failure(CUTBDDC_INVALID_ARGUMENT, "distribution: world size out of range");
  if (rank < 0 || rank >= world) throw Failure(CUTBDDC_INVALID_ARGUMENT, "distribution: rank out of range");
  if (block < 1 || nsd_g < 1 || !bids) throw Failure(CUTBDDC_INVALID_ARGUMENT, "distribution: empty partition");
  h->dist_block = block;
  h->dist_rank = rank;
  h->dist_world = world;
  h->nsd_g = nsd_g;
  h->g_block_ids.assign(bids, bids + nsd_g);
  h->rank_of_gsd.assign((size_t)nsd_g, 0);
  for (int g = 0; g < nsd_g; ++g) {
    if (g && bids[g] <= bids[g - 1]) throw Failure(CUTBDDC_INVALID_ARGUMENT, "partition: block ids must ascend");
    const int r = rank_of_sd ? rank_of_sd[g] : 0;
    if (r < 0 || r >= world) throw Failure(CUTBDDC_INVALID_ARGUMENT, "distribution: rank_of_sd out of range");
    h->rank_of_gsd[(size_t)g] = r;
  }
  std::vector<int> per(world, 0);
  h->lidx_of_gsd.assign((size_t)nsd_g, 0);
  h->global_of_local.clear();
  for (int g = 0; g < nsd_g; ++g) {
    const int r = h->rank_of_gsd[(size_t)g];
    h->lidx_of_gsd[(size_t)g] = per[(size_t)r]++;
    if (r == rank) h->global_of_local.push_back(g);
  }
  if (h->global_of_local.empty())
    throw Failure(CUTBDDC_CONFIG, "distribution: rank " + std::to_string(rank) + " received no subdomain");
  h->maxloc = *std::max_element(per.begin(), per.end());
  std::vector<int32_t> gpos((size_t)nsd_g);
  for (int g = 0; g < nsd_g; ++g) gpos[(size_t)g] = h->rank_of_gsd[(size_t)g] * h->maxloc + h->lidx_of_gsd[(size_t)g];
  h->d_gpos.upload(gpos, h->stream);
  h->dist_set = true;
}

void dist_set(cutbddc_gpu* h, const cutbddc_partition_view* part, const int32_t* rank_of_sd, int rank, int world) {
  if (!part) throw Failure(CUTBDDC_INVALID_ARGUMENT, "distribution: null partition");
  if (h->comm && (rank != h->rank || world != h->world))
    throw Failure(CUTBDDC_INVALID_ARGUMENT, "distribution: rank / world differ from the handle's communicator");
  dist_common(h, part->block, part->n_sd, part->block_ids, rank_of_sd, rank, world);
  h->dist_explicit = true;
}

void dist_default(cutbddc_gpu* h, const cutbddc_partition_view* part) {
  dist_common(h, part->block, part->n_sd, part->block_ids, nullptr, 0, 1);
  h->dist_explicit = false;
}

// ---------------------------------------------------------------- plan
void build_plan_device(cutbddc_gpu* h) {
  cudaStream_t s = h->stream;
  const int64_t nd = h->n_dof;
  const int nsd = h->nsd, nsd_g = h->nsd_g, rank = h->dist_rank;
  const int nb = h->nb, T = h->slots;
  if (nd >= (1ll << 31)) throw Failure(CUTBDDC_INVALID_ARGUMENT, "distribution: more than 2^31 dofs");
  // global subdomain maps on the device
  std::vector<int32_t> gsd_of_block((size_t)nb * nb * nb, -1), lsd_of_gsd((size_t)nsd_g, -1);
  for (int g = 0; g < nsd_g; ++g) {
    gsd_of_block[(size_t)h->g_block_ids[(size_t)g]] = g;
    if (h->rank_of_gsd[(size_t)g] == rank) lsd_of_gsd[(size_t)g] = h->lidx_of_gsd[(size_t)g];
  }
  h->d_gsd_of_block.upload(gsd_of_block, s);
  h->d_rank_of_gsd.upload(h->rank_of_gsd, s);
  h->d_lsd_of_gsd.upload(lsd_of_gsd, s);
  h->d_gblock.upload(h->g_block_ids, s);
  PlanArgs a{h->n, h->block, nb, h->b1, T, rank, h->cls.p, h->node_of_dof.p, h->d_gsd_of_block.p,
             h->d_rank_of_gsd.p, h->d_lsd_of_gsd.p, h->d_gblock.p};
  DevBuf<int32_t>& sds = h->ws_sds;
  DevBuf<uint8_t>& nsds = h->ws_nsds;
  DevBuf<uint8_t>& local = h->ws_local;
  DevBuf<int32_t>& seg = h->ws_seg;
  DevBuf<uint32_t>& rmask = h->ws_rmask;
  sds.alloc((size_t)nd * 8);
  nsds.alloc((size_t)nd);
  local.alloc((size_t)nd);
  seg.alloc((size_t)nd);
  rmask.alloc((size_t)nd);
  k_dof_sds<<<grid_for(nd, 256), 256, 0, s>>>(nd, a, nsd, sds.p, nsds.p, local.p, seg.p, rmask.p);
  CB_LAUNCH();
  // local dofs, ascending global
  DevBuf<int32_t>& glist = h->ws_glist;
  glist.alloc((size_t)nd);
  DevBuf<int64_t>& cnt = h->ws_cnt;
  cnt.alloc(2);
  DevBuf<uint8_t>& tmp = h->ws_tmp;
  size_t tb = 0;
  cub::CountingInputIterator<int32_t> it(0);
  CB_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, it, local.p, glist.p, cnt.p, (int)nd, s));
  tmp.alloc(std::max(tmp.n, tb));
  CB_CUDA(cub::DeviceSelect::Flagged(tmp.p, tb, it, local.p, glist.p, cnt.p, (int)nd, s));
  int64_t nloc = 0;
  CB_CUDA(cudaMemcpyAsync(&nloc, cnt.p, 8, cudaMemcpyDeviceToHost, s));
  CB_CUDA(cudaStreamSynchronize(s));
  h->n_loc = nloc;
  // local numbering: stable sort by segment (ascending global within a segment)
  DevBuf<int32_t>& keys = h->ws_keys;
  keys.alloc((size_t)2 * nloc);
  k_gather_i32<<<grid_for(nloc, 256), 256, 0, s>>>(nloc, glist.p, seg.p, keys.p);
  CB_LAUNCH();
  h->loc_glob.alloc((size_t)nloc);
  int bits = 1;
  while ((1 << bits) <= nsd) ++bits;
  tb = 0;
  CB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, keys.p, keys.p + nloc, glist.p, h->loc_glob.p, (int)nloc, 0,
                                          bits, s));
  tmp.alloc(std::max(tmp.n, tb));
  CB_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tb, keys.p, keys.p + nloc, glist.p, h->loc_glob.p, (int)nloc, 0, bits,
                                          s));
  h->seg_ptr.alloc((size_t)nsd + 1);
  k_seg_ptr<<<grid_for(nsd + 1, 128), 128, 0, s>>>(nsd, nloc, keys.p + nloc, h->seg_ptr.p);
  CB_LAUNCH();
  h->loc_of_dof.alloc((size_t)nd);
  CB_CUDA(cudaMemsetAsync(h->loc_of_dof.p, 0xff, sizeof(int32_t) * nd, s));
  k_scatter_pos<<<grid_for(nloc, 256), 256, 0, s>>>(nloc, h->loc_glob.p, h->loc_of_dof.p);
  CB_LAUNCH();
  std::vector<int32_t> hseg((size_t)nsd + 1);
  CB_CUDA(cudaMemcpyAsync(hseg.data(), h->seg_ptr.p, sizeof(int32_t) * (nsd + 1), cudaMemcpyDeviceToHost, s));
  // neighbour ranks
  DevBuf<unsigned int>& om = h->ws_omask;
  om.alloc(1);
  om.zero(s);
  k_or_mask<<<148, 256, 0, s>>>(nd, rmask.p, om.p);
  CB_LAUNCH();
  unsigned int mask = 0;
  CB_CUDA(cudaMemcpyAsync(&mask, om.p, 4, cudaMemcpyDeviceToHost, s));
  CB_CUDA(cudaStreamSynchronize(s));
  h->n_own = hseg[(size_t)nsd];
  {  // segment-kernel chunks (dist.cuh): per segment, then the ghosts
    std::vector<int4> ch;
    std::vector<int32_t> first((size_t)nsd + 1, 0);
    for (int sd = 0; sd < nsd; ++sd) {
      first[(size_t)sd] = (int32_t)ch.size();
      for (int32_t lo = hseg[(size_t)sd]; lo < hseg[(size_t)sd + 1]; lo += kChunk)
        ch.push_back(make_int4(sd, lo, std::min(lo + kChunk, hseg[(size_t)sd + 1]), 0));
    }
    first[(size_t)nsd] = (int32_t)ch.size();
    for (int64_t lo = hseg[(size_t)nsd]; lo < nloc; lo += kChunk)
      ch.push_back(make_int4(-1, (int)lo, (int)std::min<int64_t>(lo + kChunk, nloc), 0));
    if (ch.empty()) ch.push_back(make_int4(-1, 0, 0, 0));
    h->n_chunks = (int64_t)ch.size();
    h->chunks.upload(ch, s);
    h->seg_chunk.upload(first, s);
    h->cpart.alloc(ch.size());
    h->tickets.alloc((size_t)nsd);
    h->tickets.zero(s);
  }
  h->nbr.clear();
  std::vector<int32_t> nbr_of_rank(kMaxRanks, -1);
  for (int q = 0; q < h->dist_world; ++q)
    if (q != rank && ((mask >> q) & 1u)) {
      nbr_of_rank[(size_t)q] = (int32_t)h->nbr.size();
      h->nbr.push_back(q);
    }
  const int nnbr = (int)h->nbr.size();
  h->d_nbr.upload(h->nbr.empty() ? std::vector<int32_t>{0} : h->nbr, s);
  h->d_nbr_of_rank.upload(nbr_of_rank, s);
  // per-neighbour message layouts (inclusive scans in ascending-global order)
  DevBuf<int32_t>& rc = h->ws_rc;
  DevBuf<int32_t>& sc = h->ws_sc;
  const size_t nn = (size_t)std::max(1, nnbr) * (size_t)nloc;
  rc.alloc(2 * nn);
  sc.alloc(2 * nn);
  std::vector<int64_t> sbase(1, 0), rbase(1, 0);
  if (nnbr > 0) {
    k_nbr_counts<<<grid_for(nloc, 256), 256, 0, s>>>(nloc, nnbr, glist.p, sds.p, h->d_rank_of_gsd.p, h->d_nbr.p, rank,
                                                     rc.p, sc.p);
    CB_LAUNCH();
    tb = 0;
    CB_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tb, rc.p, rc.p + nn, (int)nloc, s));
    tmp.alloc(std::max(tmp.n, tb));
    std::vector<int32_t> tot((size_t)2 * nnbr);
    for (int k = 0; k < nnbr; ++k) {
      const size_t o = (size_t)k * nloc;
      CB_CUDA(cub::DeviceScan::InclusiveSum(tmp.p, tb, rc.p + o, rc.p + nn + o, (int)nloc, s));
      CB_CUDA(cub::DeviceScan::InclusiveSum(tmp.p, tb, sc.p + o, sc.p + nn + o, (int)nloc, s));
      CB_CUDA(cudaMemcpyAsync(&tot[(size_t)2 * k], rc.p + nn + o + nloc - 1, 4, cudaMemcpyDeviceToHost, s));
      CB_CUDA(cudaMemcpyAsync(&tot[(size_t)2 * k + 1], sc.p + nn + o + nloc - 1, 4, cudaMemcpyDeviceToHost, s));
    }
    CB_CUDA(cudaStreamSynchronize(s));
    for (int k = 0; k < nnbr; ++k) {
      rbase.push_back(rbase.back() + tot[(size_t)2 * k]);
      sbase.push_back(sbase.back() + tot[(size_t)2 * k + 1]);
    }
  }
  h->recv_ptr = rbase;
  h->send_ptr = sbase;
  h->d_rbase.upload(rbase, s);
  h->d_sbase.upload(sbase, s);
  h->send_src.alloc((size_t)std::max<int64_t>(1, sbase.back()));
  h->sendbuf.alloc((size_t)std::max<int64_t>(1, sbase.back()));
  h->recvbuf.alloc((size_t)std::max<int64_t>(1, rbase.back()));
  // copy lists (local numbering)
  h->lcopy_ptr.alloc((size_t)nloc + 1);
  DevBuf<int32_t>& cc = h->ws_ccount;
  cc.alloc((size_t)std::max<int64_t>(1, nloc));
  k_copy_count<<<grid_for(nloc, 256), 256, 0, s>>>(nloc, h->loc_glob.p, nsds.p, cc.p);
  CB_LAUNCH();
  CB_CUDA(cudaMemsetAsync(h->lcopy_ptr.p, 0, 4, s));
  tb = 0;
  CB_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tb, cc.p, h->lcopy_ptr.p + 1, (int)nloc, s));
  tmp.alloc(std::max(tmp.n, tb));
  CB_CUDA(cub::DeviceScan::InclusiveSum(tmp.p, tb, cc.p, h->lcopy_ptr.p + 1, (int)nloc, s));
  int32_t ncopy = 0;
  CB_CUDA(cudaMemcpyAsync(&ncopy, h->lcopy_ptr.p + nloc, 4, cudaMemcpyDeviceToHost, s));
  CB_CUDA(cudaStreamSynchronize(s));
  h->n_copies = ncopy;
  h->lcopy_src.alloc((size_t)std::max(1, ncopy));
  h->lowner.alloc((size_t)std::max<int64_t>(1, nloc));
  k_fill_plan<<<grid_for(nloc, 128), 128, 0, s>>>(nloc, nnbr, a, glist.p, h->loc_of_dof.p, sds.p, h->d_nbr_of_rank.p,
                                                  rc.p + nn, rc.p, sc.p + nn, sc.p, h->d_rbase.p, h->d_sbase.p,
                                                  h->lcopy_ptr.p, h->lcopy_src.p, h->send_src.p, h->lowner.p);
  CB_LAUNCH();
  const int64_t ns = (int64_t)nsd * T;
  h->slot_loc.alloc((size_t)ns);
  k_slot_loc<<<grid_for(ns, 256), 256, 0, s>>>(ns, h->slot_dof.p, h->loc_of_dof.p, h->slot_loc.p);
  CB_LAUNCH();
}

// ---------------------------------------------------------------- exchange
void iface_exchange(cutbddc_gpu* h, const double* Y, const double* w, const int* skip) {
  const int nnbr = (int)h->nbr.size();
  if (nnbr == 0) return;
  if (!h->comm) throw Failure(CUTBDDC_CONFIG, "interface exchange: the handle has no communicator (plan-only distribution)");
  cudaStream_t s = h->stream;
  const int64_t nsend = h->send_ptr.back();
  k_pack<<<grid_for(std::max<int64_t>(1, nsend), 256), 256, 0, s>>>(nsend, h->send_src.p, w, Y, h->sendbuf.p, skip);
  CB_LAUNCH();
  nccl_check(ncclGroupStart(), "group start");
  for (int k = 0; k < nnbr; ++k) {
    const size_t ns = (size_t)(h->send_ptr[(size_t)k + 1] - h->send_ptr[(size_t)k]);
    const size_t nr = (size_t)(h->recv_ptr[(size_t)k + 1] - h->recv_ptr[(size_t)k]);
    if (ns) nccl_check(ncclSend(h->sendbuf.p + h->send_ptr[(size_t)k], ns, ncclDouble, h->nbr[(size_t)k], h->comm, s), "send");
    if (nr) nccl_check(ncclRecv(h->recvbuf.p + h->recv_ptr[(size_t)k], nr, ncclDouble, h->nbr[(size_t)k], h->comm, s), "recv");
  }
  nccl_check(ncclGroupEnd(), "group end");
}

void iface_sum(cutbddc_gpu* h, const double* Y, const double* w, double* out, const int* skip, double* Xs) {
  k_isum<<<grid_for(std::max<int64_t>(1, h->n_loc), 256), 256, 0, h->stream>>>(h->n_loc, h->lcopy_ptr.p, h->lcopy_src.p,
                                                                                w, Y, h->recvbuf.p, out, Xs, skip);
  CB_LAUNCH();
}

void gather_partials(cutbddc_gpu* h, double* part) {
  if (h->dist_world == 1) return;
  if (!h->comm) throw Failure(CUTBDDC_CONFIG, "partials: the handle has no communicator (plan-only distribution)");
  nccl_check(ncclAllGather(part + (int64_t)h->dist_rank * h->maxloc, part, (size_t)h->maxloc, ncclDouble, h->comm,
                           h->stream),
             "all-gather");
}

void gather_rows(cutbddc_gpu* h) {
  if (h->dist_world == 1) return;
  if (!h->comm) throw Failure(CUTBDDC_CONFIG, "coarse rows: the handle has no communicator (plan-only distribution)");
  nccl_check(ncclAllGather(h->gl.p + (int64_t)h->dist_rank * h->maxrows, h->gl.p, (size_t)h->maxrows, ncclDouble,
                           h->comm, h->stream),
             "all-gather");
}

void gather_blocks(cutbddc_gpu* h) {
  if (h->dist_world == 1) return;
  if (!h->comm) throw Failure(CUTBDDC_CONFIG, "coarse blocks: the handle has no communicator (plan-only distribution)");
  nccl_check(ncclAllGather(h->ac_loc.p + (int64_t)h->dist_rank * h->maxac, h->ac_loc.p, (size_t)h->maxac, ncclDouble,
                           h->comm, h->stream),
             "all-gather");
}

int agree_status(cutbddc_gpu* h, int code) {
  if (h->dist_world == 1 || !h->comm) return code;
  DevBuf<int>& f = h->ws_flag;
  f.alloc(1);
  CB_CUDA(cudaMemcpyAsync(f.p, &code, sizeof(int), cudaMemcpyHostToDevice, h->stream));
  nccl_check(ncclAllReduce(f.p, f.p, 1, ncclInt32, ncclMax, h->comm, h->stream), "status");
  int out = 0;
  CB_CUDA(cudaMemcpyAsync(&out, f.p, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
  CB_CUDA(cudaStreamSynchronize(h->stream));
  return out;
}

constexpr int64_t kCells8Rows = 65536;  // fewer irregular rows: 8 lanes per row (latency), else a thread per row

void sub_apply(cutbddc_gpu* h, int mode, const double* xloc, const double* Xslot, double* Y, const int* skip) {
  cudaStream_t st = h->stream;
  const int64_t ns = (int64_t)h->nsd * h->slots;
  if (!Xslot) {
    h->sx.alloc((size_t)ns);
    k_gather_slots<<<grid_for(ns, 256), 256, 0, st>>>(ns, h->slot_loc.p, xloc, h->sx.p, skip);
    CB_LAUNCH();
    Xslot = h->sx.p;
  }
  SubArgs a{h->n,    h->block, h->b1, h->slots, h->nb, h->nsd, h->block_ids.p, h->elem_of_cell.p, h->keS.p,
            h->n_cut, h->ws_kint.p, h->slot_loc.p, h->mask_int.p, h->odiag.p};
  const int64_t lo = mode == kSubInterface ? h->rows_nint : 0;
  const int64_t hi = mode == kSubInterior ? h->rows_nint : h->rows_n;
  const int64_t lo2 = std::max(lo, h->rows_nreg);  // irregular rows from here
  const char* env_unfused = std::getenv("CUTBDDC_SUB_UNFUSED");  // A/B and test hook: the separate launches
  const bool unfused = env_unfused && env_unfused[0] == '1';
  if (!unfused && lo < h->rows_nreg && hi > lo2) {
    const int nblk_reg = grid_for(h->rows_nreg, 256);
    if (hi - lo2 < kCells8Rows)
      k_sub_fused<true><<<nblk_reg + grid_for((hi - lo2) * 8, 256), 256, 0, st>>>(
          a, h->op_rows.p, h->rows_nreg, nblk_reg, h->b1 * h->b1, h->b1, h->s27.p, lo2, hi, Xslot, Y, skip);
    else
      k_sub_fused<false><<<nblk_reg + grid_for(hi - lo2, 256), 256, 0, st>>>(
          a, h->op_rows.p, h->rows_nreg, nblk_reg, h->b1 * h->b1, h->b1, h->s27.p, lo2, hi, Xslot, Y, skip);
    CB_LAUNCH();
    return;
  }
  if (lo < h->rows_nreg) {
    k_sub_regular<<<grid_for(h->rows_nreg, 256), 256, 0, st>>>(h->op_rows.p, h->rows_nreg, h->b1 * h->b1, h->b1,
                                                               h->s27.p, Xslot, Y, skip);
    CB_LAUNCH();
  }
  if (hi > lo2) {
    if (hi - lo2 < kCells8Rows)
      k_sub_cells8<<<grid_for((hi - lo2) * 8, 256), 256, 0, st>>>(a, h->op_rows.p, lo2, hi, Xslot, Y, skip);
    else
      k_sub_cells1<<<grid_for(hi - lo2, 256), 256, 0, st>>>(a, h->op_rows.p, lo2, hi, Xslot, Y, skip);
    CB_LAUNCH();
  }
}

// the operator's row list (after the masks, odiag and slot_loc exist)
void build_operator_rows(cutbddc_gpu* h) {
  cudaStream_t st = h->stream;
  const int64_t ns = (int64_t)h->nsd * h->slots;
  DevBuf<uint8_t>& kind = h->ws_local;
  kind.alloc((size_t)ns);
  k_slot_kind<<<grid_for(ns, 256), 256, 0, st>>>(ns, h->slots, h->block, h->b1, h->n, h->nb, h->block_ids.p,
                                                 h->elem_of_cell.p, h->slot_loc.p, h->mask_int.p, h->odiag.p, kind.p);
  CB_LAUNCH();
  h->op_rows.alloc((size_t)ns);
  // stable sort of the slots by kind (radix sort over 2 bits)
  DevBuf<uint8_t>& kind2 = h->ws_nsds;
  kind2.alloc((size_t)ns);
  cub::CountingInputIterator<int32_t> it(0);
  DevBuf<int32_t>& idx = h->ws_glist;
  idx.alloc((size_t)ns);
  k_iota<<<grid_for(ns, 256), 256, 0, st>>>(ns, idx.p);
  CB_LAUNCH();
  size_t tb = 0;
  CB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, kind.p, kind2.p, idx.p, h->op_rows.p, (int)ns, 0, 2, st));
  DevBuf<uint8_t>& tmp = h->ws_tmp;
  tmp.alloc(std::max(tmp.n, tb));
  CB_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tb, kind.p, kind2.p, idx.p, h->op_rows.p, (int)ns, 0, 2, st));
  DevBuf<int64_t>& cnt = h->ws_cnt;
  cnt.alloc(4);
  k_kind_counts<<<1, 32, 0, st>>>(ns, kind2.p, cnt.p);
  CB_LAUNCH();
  int64_t c[4];
  CB_CUDA(cudaMemcpyAsync(c, cnt.p, sizeof(c), cudaMemcpyDeviceToHost, st));
  h->s27.alloc(27);
  k_stencil27<<<1, 32, 0, st>>>(h->ws_kint.p, h->s27.p);
  CB_LAUNCH();
  CB_CUDA(cudaStreamSynchronize(st));
  h->rows_nreg = c[0];
  h->rows_nint = c[1];
  h->rows_n = c[2];
}

void pack_cut_matrices(cutbddc_gpu* h) {
  h->keS.alloc((size_t)36 * std::max<int64_t>(1, h->n_cut));
  if (h->n_cut == 0) return;
  k_pack_ke<<<grid_for(h->n_cut, 256), 256, 0, h->stream>>>(h->n_cut, h->ke.p, h->keS.p);
  CB_LAUNCH();
}

void to_local(cutbddc_gpu* h, const double* xglob, double* xloc) {
  k_to_local<<<grid_for(std::max<int64_t>(1, h->n_loc), 256), 256, 0, h->stream>>>(h->n_loc, h->loc_glob.p, xglob, xloc);
  CB_LAUNCH();
}

void to_global_owned(cutbddc_gpu* h, const double* xloc, double* xglob) {
  k_to_global<<<grid_for(std::max<int64_t>(1, h->n_own), 256), 256, 0, h->stream>>>(h->n_own, h->loc_glob.p, xloc, xglob);
  CB_LAUNCH();
}

}  // namespace cutbddc_b200
