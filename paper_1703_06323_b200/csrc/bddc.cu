// bddc.cu — BDDC setup (K5, K8, K9, K10) and application.
//
//   build_weighting     SPEC.md:370-378  topological 1/|neigh| or stiffness
//                       A^w_xixi / sum_w' A^w'_xixi
//   build_coarse_space  SPEC.md:379-387  C_w rows (corner e_xi, edge/face
//                       (1/|lambda|) sum e_xi); constrained
//                       Neumann solves through the augmented K = A_w + rho_w C^T C
//                       (shell-root factorisation, factor.cu) and the constraint
//                       Schur complement S = C K^{-1} C^T, all in the root space
//                       of K (k_root_h): Phi = K^{-1} C^T S^{-1} is never formed,
//                       A_c,w = Phi^T A_w Phi = S^{-1} - rho_w I, assembled in
//                       subdomain order.
//   apply               SPEC.md:388-396, expanded in SURVEY.md section 3.2, with
//                       r1 := 0 on interior rows.
// Every gather sums in ascending subdomain order; no fp64 atomics.
#include <algorithm>
#include <exception>
#include <thread>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "bddc.cuh"
#include "factor.cuh"
#include "comm.cuh"
#include "dist.cuh"
#include "subst.cuh"

namespace cutbddc_b200 {
namespace {

// slot vector of the A^w diagonals (input of the stiffness-weight denominators)
__global__ void k_diag_slots(int64_t ns, int T, const double* __restrict__ As, double* __restrict__ dg) {
  const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g >= ns) return;
  dg[g] = As[(g / T) * 27 * T + 13ll * T + g % T];
}

// dtot: per local dof, the sum of the A^w diagonals over every copy (all ranks)
__global__ void k_weights(int64_t ns, int T, int mode, const int32_t* __restrict__ slot_dof,
                          const int32_t* __restrict__ slot_loc, const uint8_t* __restrict__ ncount,
                          const double* __restrict__ As, const double* __restrict__ dtot, double* __restrict__ w,
                          int* __restrict__ bad) {
  const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g >= ns) return;
  const int32_t d = slot_dof[g];
  if (d < 0) {
    w[g] = 0.0;
    return;
  }
  const int k = ncount[d];
  if (k == 1) {
    w[g] = 1.0;
    return;
  }
  if (mode == CUTBDDC_WEIGHT_TOPOLOGICAL) {
    w[g] = 1.0 / (double)k;
    return;
  }
  const double tot = dtot[slot_loc[g]];
  if (!(tot != 0.0)) {
    atomicExch(bad, 1);
    w[g] = 0.0;
    return;
  }
  w[g] = As[(g / T) * 27 * T + 13ll * T + g % T] / tot;
}

// rho_w = mean of diag(A_w) over the subdomain's local dofs, summed
// sequentially in ascending local dof (= slot) order: K = A + rho C^T C of a
// small-cut subdomain is so ill-conditioned that a 1-ulp change of rho moves
// the saddle solutions by ~1e-9, so rho is pinned bit-for-bit to the CPU
// restatement's order. One CTA per subdomain stages the diagonal in shared
// memory (coalesced, absent slots as +0.0, which leaves the running sum
// unchanged), then thread 0 adds it in slot order.
__global__ void __launch_bounds__(256) k_rho(int nsd, int T, const int32_t* __restrict__ slot_dof,
                                             const double* __restrict__ As, double* __restrict__ rho) {
  extern __shared__ double dg[];
  __shared__ int cnt;
  const int sd = blockIdx.x;
  if (threadIdx.x == 0) cnt = 0;
  __syncthreads();
  int c = 0;
  for (int t = threadIdx.x; t < T; t += blockDim.x) {
    const bool p = slot_dof[(int64_t)sd * T + t] >= 0;
    dg[t] = p ? As[(int64_t)sd * 27 * T + 13ll * T + t] : 0.0;
    c += p;
  }
  atomicAdd(&cnt, c);
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int t = 0; t < T; ++t) s += dg[t];
    rho[sd] = cnt > 0 ? s / (double)cnt : 1.0;
  }
}

__global__ void k_diag_add(int nsd, int T, const int64_t* __restrict__ m_off, const int64_t* __restrict__ c_ptr,
                           const int32_t* __restrict__ c_slot, const uint8_t* __restrict__ corner,
                           const double* __restrict__ rho, double* __restrict__ dadd) {
  const int sd = blockIdx.x;
  for (int64_t r = m_off[sd] + threadIdx.x; r < m_off[sd + 1]; r += blockDim.x) {
    if (!corner[r]) continue;
    dadd[(int64_t)sd * T + c_slot[c_ptr[r]]] = rho[sd];
  }
}

// In-place SPD inverse of each subdomain's m x m block (symmetrised first),
// Gauss-Jordan without pivoting on the SPD matrix; non-positive pivot -> fail.
__global__ void k_small_spd_inverse(int nblk, const int64_t* __restrict__ m_off, const int64_t* __restrict__ s_off,
                                    double* __restrict__ S, unsigned long long* fail) {
  extern __shared__ double a[];
  const int b = blockIdx.x;
  const int m = (int)(m_off[b + 1] - m_off[b]);
  if (m == 0) return;
  double* g = S + s_off[b];
  for (int q = threadIdx.x; q < m * m; q += blockDim.x) {
    const int r = q / m, c = q % m;
    a[q] = 0.5 * (g[r * m + c] + g[c * m + r]);
  }
  __syncthreads();
  __shared__ double piv;
  for (int k = 0; k < m; ++k) {
    if (threadIdx.x == 0) {
      piv = a[k * m + k];
      if (!(piv > 0.0)) {
        atomicMin(fail, (unsigned long long)b);
        piv = 1.0;
      }
    }
    __syncthreads();
    // row k /= piv ; eliminate column k from other rows (Gauss-Jordan in place)
    const double p = piv;
    double* colk = a + m * m;  // multipliers of column k, staged before the update
    for (int q = threadIdx.x; q < m; q += blockDim.x) {
      colk[q] = a[q * m + k];
      a[k * m + q] = q == k ? 1.0 / p : a[k * m + q] / p;
    }
    __syncthreads();
    for (int q = threadIdx.x; q < m * m; q += blockDim.x) {
      const int r = q / m, c = q % m;
      if (r == k) continue;
      const double f = colk[r];
      if (c == k)
        a[q] = -f * a[k * m + k];
      else
        a[q] -= f * a[k * m + c];
    }
    __syncthreads();
  }
  for (int q = threadIdx.x; q < m * m; q += blockDim.x) g[q] = a[q];
}

// coarse row lambda: sum over its (sd, local row) copies in ascending global
// sd. Rows and the m x m blocks A_c,w are addressed in the gathered staging
// layout (rank-major, dist.cuh): p = staging position of a constraint row,
// srow = {staging position of its subdomain's first row, m, staging offset
// of the subdomain's block}, scoarse = coarse id of every staged row.
__global__ void k_coarse_assemble(int nc, const int64_t* __restrict__ cg_ptr, const int64_t* __restrict__ cg_idx,
                                  const int64_t* __restrict__ srow, const int32_t* __restrict__ scoarse,
                                  const double* __restrict__ Ac, double* __restrict__ A) {
  const int lam = blockIdx.x;
  double* arow = A + (int64_t)lam * nc;
  for (int64_t p = cg_ptr[lam]; p < cg_ptr[lam + 1]; ++p) {
    const int64_t row = cg_idx[p];
    const int64_t first = srow[3 * row];
    const int m = (int)srow[3 * row + 1];
    const int i = (int)(row - first);
    const double* blk = Ac + srow[3 * row + 2] + (int64_t)i * m;
    for (int c = threadIdx.x; c < m; c += blockDim.x) arow[scoarse[first + c]] += blk[c];
    __syncthreads();
  }
}

// ------------------------------------------------------------------ apply
// Vectors are in the rank's local dof space (dist.cuh); slot vectors per
// local subdomain.
__global__ void k_gather_masked(int64_t ns, const int32_t* __restrict__ slot_loc, const uint8_t* __restrict__ mask,
                                const double* __restrict__ r, double* __restrict__ X, const int* __restrict__ skip) {
  if (skip && *skip) return;
  const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g >= ns) return;
  X[g] = mask[g] ? r[slot_loc[g]] : 0.0;
}

// X[slot] = w * r1[dof] with r1 = r - Abar z0 on interface rows and 0 on
// interior rows; (Abar z0)[dof] = Σ over the copies,
// ascending global sd, of (A_w z0_w)[slot] (Y, remote copies from recv)
__global__ void k_scatter_r1(int64_t ns, const int32_t* __restrict__ slot_loc, const uint8_t* __restrict__ mint,
                             const double* __restrict__ w, const double* __restrict__ r,
                             const int32_t* __restrict__ cptr, const int32_t* __restrict__ csrc,
                             const double* __restrict__ Y, const double* __restrict__ recv, double* __restrict__ X,
                             const int* __restrict__ skip) {
  if (skip && *skip) return;
  const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g >= ns) return;
  const int32_t l = slot_loc[g];
  if (l < 0 || mint[g]) {
    X[g] = 0.0;
    return;
  }
  double az = 0.0;
  for (int32_t p = cptr[l]; p < cptr[l + 1]; ++p) {
    const int32_t c = csrc[p];
    az += c >= 0 ? Y[c] : recv[-1 - c];
  }
  X[g] = w[g] * (r[l] - az);
}

// cy[row] = C_row . y
__global__ void k_cy(int64_t mtot, int T, const int32_t* __restrict__ row_sd, const int64_t* __restrict__ c_ptr,
                     const int32_t* __restrict__ c_slot, const double* __restrict__ c_val, const double* __restrict__ Y,
                     double* __restrict__ cy, const int* __restrict__ skip, const uint8_t* __restrict__ skip_sd) {
  if (skip && *skip) return;
  const int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= mtot) return;
  if (skip_sd && skip_sd[row_sd[row]]) return;
  const double* y = Y + (int64_t)row_sd[row] * T;
  double s = 0.0;
  for (int64_t p = c_ptr[row] + lane; p < c_ptr[row + 1]; p += 32) s += c_val[p] * y[c_slot[p]];
  s = warp_sum(s);
  if (lane == 0) cy[row] = s;
}

__global__ void k_coarse_rhs(int nc, const int64_t* __restrict__ cg_ptr, const int64_t* __restrict__ cg_idx,
                             const double* __restrict__ gl, double* __restrict__ g, const int* __restrict__ skip) {
  if (skip && *skip) return;
  const int lam = blockIdx.x * blockDim.x + threadIdx.x;
  if (lam >= nc) return;
  double s = 0.0;
  for (int64_t p = cg_ptr[lam]; p < cg_ptr[lam + 1]; ++p) s += gl[cg_idx[p]];
  g[lam] = s;
}

// Small coarse problems (n_c <= kCoarseInverseMax): A_c^{-1} = X^T X once in
// setup, then one GEMV per apply. 64 x 64 output tiles of the lower
// triangle, mirrored; X's entries above its diagonal tiles are not stored
// and are masked.
constexpr int kCoarseInverseMax = 4096;
__global__ void __launch_bounds__(256) k_xtx(int n, const double* __restrict__ X, double* __restrict__ C) {
  const int ib = blockIdx.x, jb = blockIdx.y;
  if (jb > ib) return;
  const int i0 = ib * 64, j0 = jb * 64;
  __shared__ double xa[32][65], xb[32][65];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  double acc[4][4] = {};
  for (int k0 = i0; k0 < n; k0 += 32) {  // X[k, i] = 0 for k < i, and i >= j
    __syncthreads();
    for (int e = tid; e < 32 * 64; e += 256) {
      const int kk = e & 31, c = e >> 5, k = k0 + kk;
      const int i = i0 + c, j = j0 + c;
      xa[kk][c] = (k < n && i < n && k >= i) ? X[k + (int64_t)i * n] : 0.0;
      xb[kk][c] = (k < n && j < n && k >= j) ? X[k + (int64_t)j * n] : 0.0;
    }
    __syncthreads();
#pragma unroll 8
    for (int kk = 0; kk < 32; ++kk) {
      double a[4], b[4];
#pragma unroll
      for (int x = 0; x < 4; ++x) a[x] = xa[kk][tx + 16 * x];
#pragma unroll
      for (int y = 0; y < 4; ++y) b[y] = xb[kk][ty + 16 * y];
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y) acc[x][y] += a[x] * b[y];
    }
  }
#pragma unroll
  for (int x = 0; x < 4; ++x)
#pragma unroll
    for (int y = 0; y < 4; ++y) {
      const int i = i0 + tx + 16 * x, j = j0 + ty + 16 * y;
      if (i < n && j < n && j <= i) {
        C[(int64_t)i * n + j] = acc[x][y];
        C[(int64_t)j * n + i] = acc[x][y];
      }
    }
}

// zc = A_c^{-1} g: warp per row of the (symmetric) explicit inverse.
__global__ void k_coarse_gemv(int nc, const double* __restrict__ Ainv, const double* __restrict__ g,
                              double* __restrict__ zc, const int* __restrict__ skip) {
  if (skip && *skip) return;
  const int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= nc) return;
  const double* a = Ainv + row * nc;
  double s0 = 0.0, s1 = 0.0;
  int c = lane;
  for (; c + 32 < nc; c += 64) {
    s0 += a[c] * g[c];
    s1 += a[c + 32] * g[c + 32];
  }
  for (; c < nc; c += 32) s0 += a[c] * g[c];
  const double s = warp_sum(s0 + s1);
  if (lane == 0) zc[row] = s;
}

// Large coarse problems: zc = A_c^{-1} g = X^T (X g), X = L^{-1} (lower, column-major n x n):
//  k_xg_part: part[cb][i] = sum_{j in column block cb, j <= i} X[i, j] g[j]
//             (thread per row, coalesced down each column);
//  k_xg_sum:  y[i] = sum over cb <= i / 64 of part[cb][i] (in order);
//  k_xty:     zc[j] = sum_{i >= j} X[i, j] y[i] (warp per column).
__global__ void __launch_bounds__(256) k_xg_part(int n, const double* __restrict__ X, const double* __restrict__ g,
                                                 double* __restrict__ part, const int* __restrict__ skip) {
  if (skip && *skip) return;
  const int i = blockIdx.x * 256 + threadIdx.x, j0 = blockIdx.y * 64;
  if (i >= n || j0 > i) return;
  const int j1 = min(j0 + 64, i + 1);
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  int j = j0;
  for (; j + 4 <= j1; j += 4) {
    s0 += X[i + (int64_t)j * n] * g[j];
    s1 += X[i + (int64_t)(j + 1) * n] * g[j + 1];
    s2 += X[i + (int64_t)(j + 2) * n] * g[j + 2];
    s3 += X[i + (int64_t)(j + 3) * n] * g[j + 3];
  }
  for (; j < j1; ++j) s0 += X[i + (int64_t)j * n] * g[j];
  part[(int64_t)blockIdx.y * n + i] = (s0 + s1) + (s2 + s3);
}

__global__ void k_xg_sum(int n, const double* __restrict__ part, double* __restrict__ y, const int* __restrict__ skip) {
  if (skip && *skip) return;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double s = 0.0;
  for (int cb = 0; cb <= i / 64; ++cb) s += part[(int64_t)cb * n + i];
  y[i] = s;
}

__global__ void k_xty(int n, const double* __restrict__ X, const double* __restrict__ y, double* __restrict__ z,
                      const int* __restrict__ skip) {
  if (skip && *skip) return;
  const int64_t j = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (j >= n) return;
  const double* col = X + j * n;
  double s0 = 0.0, s1 = 0.0;
  int i = (int)j + lane;
  for (; i + 32 < n; i += 64) {
    s0 += col[i] * y[i];
    s1 += col[i + 32] * y[i + 32];
  }
  for (; i < n; i += 32) s0 += col[i] * y[i];
  const double s = warp_sum(s0 + s1);
  if (lane == 0) z[j] = s;
}

// z = z0 + v - X[owner] over the local dofs (z0 = Z0[owner], the first
// interior solve; interior dofs: minus the harmonic correction X), a block
// per segment (dist.cuh); with r, every local
// subdomain's partial of r.z for the PCG (bit-reproducible for any world size)
__global__ void __launch_bounds__(kSegThreads) k_final_z(SegArgs a, const int32_t* __restrict__ owner,
                                                         const double* __restrict__ Z0, const double* __restrict__ v,
                                                         const double* __restrict__ X, double* __restrict__ z,
                                                         const double* __restrict__ r, const int* __restrict__ skip) {
  if (skip && *skip) return;
  int lo, hi;
  const int seg = seg_range(a, lo, hi);
  double acc = 0.0;
  for (int i = lo + threadIdx.x; i < hi; i += kSegThreads) {
    const int32_t o = owner[i];
    const double zi = (o >= 0 ? Z0[o] : 0.0) + v[i] - (o >= 0 ? X[o] : 0.0);
    z[i] = zi;
    if (r) acc += r[i] * zi;
  }
  if (!r || seg < 0) return;
  seg_commit(a, seg, acc);
}

// ---------------------------------------------------------------- root-space coarse basis
// The constraint rows live on the shell, i.e. on the root columns of the
// shell-root factorisation K = L L^T (K = A + rho C^T C), so with G_r the
// explicit root panel (L_r^{-1}) and C_r the rows on root positions:
//   H = G_r C_r^T,  S = C K^{-1} C^T = H^T H,  W_r = (K^{-1} C^T)_root = G_r^T H,
//   A_c,w = Phi^T A Phi = S^{-1} - rho I   (Phi = K^{-1} C^T S^{-1}, K - A = rho C^T C),
//   Phi^T r = S^{-1} C (K^{-1} r),  Phi v = K^{-1} C^T S^{-1} v.
// rinfo[4 sd + {0,1,2,3}] = {c_r, root panel offset, root vector offset, H/W offset}.
__global__ void __launch_bounds__(256) k_root_h(const int64_t* __restrict__ rinfo, const int64_t* __restrict__ m_off,
                                                const int64_t* __restrict__ c_ptr, const int32_t* __restrict__ c_slot,
                                                const double* __restrict__ c_val, const int32_t* __restrict__ root_pos,
                                                const int32_t* __restrict__ pfx_root, int64_t rows_total,
                                                const double* __restrict__ panel, double* __restrict__ H) {
  const int sd = blockIdx.x, a = blockIdx.y;
  const int m = (int)(m_off[sd + 1] - m_off[sd]);
  if (a >= m) return;
  const int cr = (int)rinfo[4 * sd];
  const double* G = panel + rinfo[4 * sd + 1];
  double* h = H + rinfo[4 * sd + 3] + (int64_t)a * cr;
  const int64_t row = m_off[sd] + a;
  const int32_t* pf = pfx_root + (int64_t)sd * rows_total;
  // the row's (root column, coefficient) pairs, staged in shared memory
  __shared__ int cj[512];
  __shared__ double cv[512];
  const int64_t p0 = c_ptr[row], len = c_ptr[row + 1] - p0;
  for (int64_t q0 = 0; q0 < len; q0 += 512) {
    const int nq = len - q0 < 512 ? (int)(len - q0) : 512;
    __syncthreads();
    for (int q = threadIdx.x; q < nq; q += blockDim.x) {
      cj[q] = pf[root_pos[c_slot[p0 + q0 + q]]];
      cv[q] = c_val[p0 + q0 + q];
    }
    __syncthreads();
    for (int i = threadIdx.x; i < cr; i += blockDim.x) {
      double s = q0 == 0 ? 0.0 : h[i];
      for (int q = 0; q < nq; ++q) {
        const int j = cj[q];
        if (j >= 0 && i >= j) s += cv[q] * G[i + (int64_t)j * cr];
      }
      h[i] = s;
    }
  }
}

// S = H^T H per subdomain (both triangles): CTA per (sd, row a), warp per b <= a
__global__ void __launch_bounds__(256) k_root_s(const int64_t* __restrict__ rinfo, const int64_t* __restrict__ m_off,
                                                const int64_t* __restrict__ s_off, const double* __restrict__ H,
                                                double* __restrict__ S, const uint8_t* __restrict__ skip_sd) {
  const int sd = blockIdx.x, a = blockIdx.y;
  if (skip_sd && skip_sd[sd]) return;  // the other formulation's subdomain
  const int m = (int)(m_off[sd + 1] - m_off[sd]);
  if (a >= m) return;
  const int cr = (int)rinfo[4 * sd];
  const double* h = H + rinfo[4 * sd + 3];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int b = wid; b <= a; b += blockDim.x / 32) {
    double s = 0.0;
    for (int i = lane; i < cr; i += 32) s += h[i + (int64_t)a * cr] * h[i + (int64_t)b * cr];
    s = warp_sum(s);
    if (lane == 0) {
      S[s_off[sd] + (int64_t)a * m + b] = s;
      S[s_off[sd] + (int64_t)b * m + a] = s;
    }
  }
}

// sinv = sym(S^{-1}); A_c,w = sinv - rho I (K = A + rho C^T C), or
// sinv - rho I_corner (K_c = A + rho C_corner^T C_corner: corner_row != null)
// A_c,w = S^{-1} - rho I_aug: the augmented rows are the corner rows (K_c)
// or every row (K = A + rho C^T C: no corner_row, or shell_sd[sd] set)
__global__ void k_root_coarse(const int64_t* __restrict__ m_off, const int64_t* __restrict__ s_off,
                              const double* __restrict__ Sinv, const double* __restrict__ rho,
                              const uint8_t* __restrict__ corner_row, double* __restrict__ sinv,
                              double* __restrict__ ac, const uint8_t* __restrict__ shell_sd) {
  const int sd = blockIdx.x;
  const int m = (int)(m_off[sd + 1] - m_off[sd]);
  const int64_t o = s_off[sd];
  for (int q = threadIdx.x; q < m * m; q += blockDim.x) {
    const int a = q / m, b = q % m;
    const double v = 0.5 * (Sinv[o + (int64_t)a * m + b] + Sinv[o + (int64_t)b * m + a]);
    sinv[o + q] = v;
    const bool shift = a == b && (!corner_row || (shell_sd && shell_sd[sd]) || corner_row[m_off[sd] + a]);
    ac[o + q] = v - (shift ? rho[sd] : 0.0);
  }
}

// ---------------------------------------------------------------- corner formulation
// K_c = A + rho sum_corners e e^T = L L^T on the plain ND template. The
// constrained Neumann solve z = K_c^{-1}(r - C^T mu), C z = 0 gives
//   S = C K_c^{-1} C^T = H^T H,  H = L^{-1} C^T (one multi-RHS forward sweep),
//   A_c,w = Phi^T A Phi = S^{-1} - rho I_corner,
//   apply: y' = L^{-1} r_w (forward sweep), cy = C K_c^{-1} r_w = H^T y',
//   u = S^{-1}(z_c - cy), z~ = L^{-T}(y' + H u) (backward sweep).
// H is kept over each subdomain's present slots in front-column order.

// right-hand sides C^T e_a, a = pass * 8 + rr, in slot space (X8 zeroed)
__global__ void k_ct_rhs(int pass, int64_t ns, int T, const int64_t* __restrict__ m_off, const int64_t* __restrict__ c_ptr,
                         const int32_t* __restrict__ c_slot, const double* __restrict__ c_val, double* __restrict__ X8) {
  const int sd = blockIdx.x, rr = blockIdx.y;
  const int64_t a = (int64_t)pass * kSweepMultiRhs + rr;
  if (a >= m_off[sd + 1] - m_off[sd]) return;
  const int64_t row = m_off[sd] + a;
  for (int64_t p = c_ptr[row] + threadIdx.x; p < c_ptr[row + 1]; p += blockDim.x)
    X8[rr * ns + (int64_t)sd * T + c_slot[p]] = c_val[p];
}

// H columns a = pass * 8 + rr from the forward sweep's column values, and
// (pass 0) the slot of every compact position
__global__ void k_h_compact(int pass, int nsn, int64_t ns, const FrontDesc* __restrict__ desc,
                            const int32_t* __restrict__ cslot, const int32_t* __restrict__ coff,
                            const int64_t* __restrict__ m_off, const int64_t* __restrict__ rinfo,
                            const double* __restrict__ Y8, double* __restrict__ H, int32_t* __restrict__ hslot) {
  const int sid = blockIdx.x, sd = blockIdx.y;
  const FrontDesc& d = desc[(int64_t)sd * nsn + sid];
  const int m = (int)(m_off[sd + 1] - m_off[sd]);
  const int np = (int)rinfo[4 * sd];
  if (np == 0) return;  // a shell-formulation subdomain (mixed K): no corner H
  const int k0 = coff[(int64_t)sd * nsn + sid];
  double* hs = H + rinfo[4 * sd + 3];
  for (int j = threadIdx.x; j < d.c; j += blockDim.x) {
    const int sl = cslot[d.vo + j];
    if (pass == 0) hslot[rinfo[4 * sd + 1] + k0 + j] = sl;
#pragma unroll
    for (int rr = 0; rr < kSweepMultiRhs; ++rr) {
      const int a = pass * kSweepMultiRhs + rr;
      if (a < m) hs[(int64_t)a * np + k0 + j] = Y8[rr * ns + sl];
    }
  }
}

// K_c pivots: every column's pivot L_jj^2 = 1 / G_jj^2 against the original
// diagonal of K_c at its slot; a pivot below 1e-12 of it (a fragment whose
// constant mode no corner and no Nitsche boundary controls) sets *bad
__global__ void k_pivot_check(int nsn, int T, const FrontDesc* __restrict__ desc, const double* __restrict__ panel,
                              const int32_t* __restrict__ cslot, const double* __restrict__ As,
                              const double* __restrict__ dadd, int* __restrict__ bad) {
  const int sid = blockIdx.x, sd = blockIdx.y;
  const FrontDesc& d = desc[(int64_t)sd * nsn + sid];
  for (int j = threadIdx.x; j < d.c; j += blockDim.x) {
    const double g = panel[d.po + (int64_t)j * d.r + j];
    const double piv = 1.0 / (g * g);
    const int sl = cslot[d.vo + j];
    const double orig = As[(int64_t)(sl / T) * 27 * T + 13ll * T + sl % T] + dadd[sl];
    if (!(piv > 1e-12 * orig)) bad[sd] = 1;  // per subdomain (benign race: every writer stores 1)
  }
}

// cy[row] = (H^T y')[row] in two steps. k_h_cy: blocks (subdomain, 256
// compact positions k): one gather of y'[k] per thread, then every row's
// H[a][k] y'[k] (coalesced across k), summed over the block in a fixed tree
// into a per-chunk partial. k_h_cy_sum: cy = the chunk partials in chunk order.
constexpr int kHcyMaxM = 128;  // constraint rows per subdomain of this path
__global__ void __launch_bounds__(256) k_h_cy(const int64_t* __restrict__ m_off, const int64_t* __restrict__ rinfo,
                                              const double* __restrict__ H, const int32_t* __restrict__ hslot,
                                              const double* __restrict__ Y, double* __restrict__ hp, int mmax,
                                              const int* __restrict__ skip) {
  if (skip && *skip) return;
  __shared__ double wsum[8][kHcyMaxM];
  const int sd = blockIdx.x, ch = blockIdx.y, lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int m = (int)(m_off[sd + 1] - m_off[sd]), np = (int)rinfo[4 * sd];
  if (m == 0 || ch * 256 >= np) return;
  const int k = ch * 256 + threadIdx.x;
  const double y = k < np ? Y[hslot[rinfo[4 * sd + 1] + k]] : 0.0;
  const double* hc = H + rinfo[4 * sd + 3] + k;
  for (int a = 0; a < m; ++a) {
    const double v = warp_sum(k < np ? hc[(int64_t)a * np] * y : 0.0);
    if (lane == 0) wsum[wid][a] = v;
  }
  __syncthreads();
  for (int a = threadIdx.x; a < m; a += blockDim.x) {
    double v = 0.0;
    for (int w = 0; w < 8; ++w) v += wsum[w][a];
    hp[((int64_t)sd * gridDim.y + ch) * mmax + a] = v;
  }
}

__global__ void k_h_cy_sum(int64_t mtot, int nch, int mmax, const int32_t* __restrict__ row_sd,
                           const int64_t* __restrict__ m_off, const int64_t* __restrict__ rinfo,
                           const double* __restrict__ hp, double* __restrict__ cy, const int* __restrict__ skip,
                           const uint8_t* __restrict__ skip_sd) {
  if (skip && *skip) return;
  const int64_t row = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (row >= mtot) return;
  const int sd = row_sd[row];
  if (skip_sd && skip_sd[sd]) return;
  const int a = (int)(row - m_off[sd]), used = (int)((rinfo[4 * sd] + 255) / 256);
  double v = 0.0;
  for (int c = 0; c < used; ++c) v += hp[((int64_t)sd * nch + c) * mmax + a];
  cy[row] = v;
}

// k_h_cy_sum and k_sinv_apply (gl = S^{-1} cy) in one launch, a block per
// subdomain: the same sums in the same order (chunk partials in chunk order,
// then the row of S^{-1} left to right), so the bits are those of the two.
__global__ void __launch_bounds__(128) k_h_cy_sum_sinv(int nch, int mmax, const int64_t* __restrict__ m_off,
                                                       const int64_t* __restrict__ rinfo, const double* __restrict__ hp,
                                                       const int64_t* __restrict__ s_off, const double* __restrict__ sinv,
                                                       double* __restrict__ cy, double* __restrict__ gl,
                                                       const int* __restrict__ skip) {
  if (skip && *skip) return;
  __shared__ double scy[kHcyMaxM];
  const int sd = blockIdx.x;
  const int64_t b0 = m_off[sd];
  const int m = (int)(m_off[sd + 1] - b0), used = (int)((rinfo[4 * sd] + 255) / 256);
  for (int a = threadIdx.x; a < m; a += blockDim.x) {
    double v = 0.0;
    for (int c = 0; c < used; ++c) v += hp[((int64_t)sd * nch + c) * mmax + a];
    scy[a] = cy[b0 + a] = v;
  }
  __syncthreads();
  for (int a = threadIdx.x; a < m; a += blockDim.x) {
    const double* si = sinv + s_off[sd] + (int64_t)a * m;
    double v = 0.0;
    for (int b = 0; b < m; ++b) v += si[b] * scy[b];
    gl[b0 + a] = v;
  }
}

// y'[slot_k] += (H u)[k]: blocks (subdomain, 256 compact positions)
__global__ void k_h_correct(const int64_t* __restrict__ m_off, const int64_t* __restrict__ rinfo,
                            const double* __restrict__ H, const int32_t* __restrict__ hslot,
                            const double* __restrict__ u, double* __restrict__ Y, const int* __restrict__ skip) {
  if (skip && *skip) return;
  const int sd = blockIdx.x;
  const int np = (int)rinfo[4 * sd];
  const int k = blockIdx.y * blockDim.x + threadIdx.x;
  if (k >= np) return;
  const int64_t b0 = m_off[sd];
  const int m = (int)(m_off[sd + 1] - b0);
  const double* hc = H + rinfo[4 * sd + 3] + k;
  double v = 0.0;
  for (int a = 0; a < m; ++a) v += hc[(int64_t)a * np] * u[b0 + a];
  Y[hslot[rinfo[4 * sd + 1] + k]] += v;
}

// W_r = G_r^T H: 64 root rows j per CTA, all m columns (<= 64 per pass),
// G's lower part only (the panel above the diagonal tiles is not stored).
__global__ void __launch_bounds__(256) k_root_w(const int64_t* __restrict__ rinfo, const int64_t* __restrict__ m_off,
                                                const double* __restrict__ panel, const double* __restrict__ H,
                                                double* __restrict__ W) {
  const int sd = blockIdx.x, j0 = blockIdx.y * 64;
  const int cr = (int)rinfo[4 * sd];
  const int m = (int)(m_off[sd + 1] - m_off[sd]);
  if (j0 >= cr || m == 0) return;
  const double* G = panel + rinfo[4 * sd + 1];
  const double* h = H + rinfo[4 * sd + 3];
  double* w = W + rinfo[4 * sd + 3];
  __shared__ double gs[32][65], hs[32][65];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  for (int l0 = 0; l0 < m; l0 += 64) {
    double acc[4][4] = {};
    for (int i0 = j0; i0 < cr; i0 += 32) {
      __syncthreads();
      for (int e = tid; e < 32 * 64; e += 256) {
        const int ii = e & 31, jj = e >> 5, i = i0 + ii, j = j0 + jj, l = l0 + jj;
        gs[ii][jj] = (i < cr && j < cr && i >= j) ? G[i + (int64_t)j * cr] : 0.0;
        hs[ii][jj] = (i < cr && l < m) ? h[i + (int64_t)l * cr] : 0.0;
      }
      __syncthreads();
#pragma unroll 8
      for (int ii = 0; ii < 32; ++ii) {
        double ga[4], hb[4];
#pragma unroll
        for (int x = 0; x < 4; ++x) ga[x] = gs[ii][tx + 16 * x];
#pragma unroll
        for (int y = 0; y < 4; ++y) hb[y] = hs[ii][ty + 16 * y];
#pragma unroll
        for (int x = 0; x < 4; ++x)
#pragma unroll
          for (int y = 0; y < 4; ++y) acc[x][y] += ga[x] * hb[y];
      }
    }
#pragma unroll
    for (int x = 0; x < 4; ++x)
#pragma unroll
      for (int y = 0; y < 4; ++y) {
        const int j = j0 + tx + 16 * x, l = l0 + ty + 16 * y;
        if (j < cr && l < m) w[j + (int64_t)l * cr] = acc[x][y];
      }
  }
}

// out[row] = sum_b S^{-1}[a][b] (zc[coarse_id] - cy)[b]   (with_zc)
//          = sum_b S^{-1}[a][b] cy[b]                       (otherwise)
__global__ void k_sinv_apply(int64_t mtot, const int32_t* __restrict__ row_sd, const int64_t* __restrict__ m_off,
                             const int64_t* __restrict__ s_off, const double* __restrict__ sinv,
                             const int32_t* __restrict__ coarse_id, const double* __restrict__ zc,
                             const double* __restrict__ cy, double* __restrict__ out, int with_zc,
                             const int* __restrict__ skip) {
  if (skip && *skip) return;
  const int64_t row = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (row >= mtot) return;
  const int sd = row_sd[row];
  const int64_t b0 = m_off[sd];
  const int m = (int)(m_off[sd + 1] - b0), a = (int)(row - b0);
  const double* si = sinv + s_off[sd] + (int64_t)a * m;
  double s = 0.0;
  for (int b = 0; b < m; ++b) s += si[b] * (with_zc ? zc[coarse_id[b0 + b]] - cy[b0 + b] : cy[b0 + b]);
  out[row] = s;
}

// X[root columns] += W_r u (the K^{-1} C^T S^{-1}(zc - cy) correction at the root)
__global__ void k_root_correct(const int64_t* __restrict__ rinfo, const int64_t* __restrict__ m_off,
                               const int32_t* __restrict__ cslot, const double* __restrict__ W,
                               const double* __restrict__ u, double* __restrict__ X, const int* __restrict__ skip) {
  if (skip && *skip) return;
  const int sd = blockIdx.x;
  const int cr = (int)rinfo[4 * sd];
  const int j = blockIdx.y * blockDim.x + threadIdx.x;
  if (j >= cr) return;
  const int64_t b0 = m_off[sd];
  const int m = (int)(m_off[sd + 1] - b0);
  const double* w = W + rinfo[4 * sd + 3] + j;
  double s = 0.0;
  for (int a = 0; a < m; ++a) s += w[(int64_t)a * cr] * u[b0 + a];
  X[cslot[rinfo[4 * sd + 2] + j]] += s;
}

// The apply's coarse problem on one GPU, two launches instead of six (same
// summation orders as k_cy / k_sinv_apply / k_coarse_rhs / k_coarse_gemv /
// k_root_correct). k_coarse_in, one block per subdomain: cy = C y (warp per
// constraint row), gl = S^{-1} cy.
constexpr int kFusedCoarseM = 256;  // constraint rows per subdomain of the fused path
__global__ void __launch_bounds__(256) k_coarse_in(int T, const int64_t* __restrict__ m_off,
                                                   const int64_t* __restrict__ c_ptr, const int32_t* __restrict__ c_slot,
                                                   const double* __restrict__ c_val, const double* __restrict__ Y,
                                                   const int64_t* __restrict__ s_off, const double* __restrict__ sinv,
                                                   double* __restrict__ cy, double* __restrict__ gl,
                                                   const int* __restrict__ skip, const int64_t* __restrict__ rinfo,
                                                   const double* __restrict__ Hc, const int32_t* __restrict__ hslot) {
  if (skip && *skip) return;
  __shared__ double scy[kFusedCoarseM];
  const int sd = blockIdx.x, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int64_t b0 = m_off[sd];
  const int m = (int)(m_off[sd + 1] - b0);
  const double* y = Y + (int64_t)sd * T;
  for (int a = wid; a < m; a += blockDim.x >> 5) {
    const int64_t row = b0 + a;
    double v = 0.0;
    if (Hc) {  // corner formulation: cy = H^T y' (Y: the forward sweep's column values)
      const int np = (int)rinfo[4 * sd];
      const double* hc = Hc + rinfo[4 * sd + 3] + (int64_t)a * np;
      const int32_t* hs = hslot + rinfo[4 * sd + 1];
      for (int k = lane; k < np; k += 32) v += hc[k] * Y[hs[k]];
    } else {
      for (int64_t p = c_ptr[row] + lane; p < c_ptr[row + 1]; p += 32) v += c_val[p] * y[c_slot[p]];
    }
    v = warp_sum(v);
    if (lane == 0) scy[a] = cy[row] = v;
  }
  __syncthreads();
  for (int a = tid; a < m; a += blockDim.x) {
    const double* si = sinv + s_off[sd] + (int64_t)a * m;
    double v = 0.0;
    for (int b = 0; b < m; ++b) v += si[b] * scy[b];
    gl[b0 + a] = v;
  }
}

// k_coarse_out, blocks (subdomain, root column chunk): gc = sum of the gl
// copies (every block, in k_coarse_rhs order), zc at the subdomain's coarse
// dofs (warp per row of A_c^{-1}), u = S^{-1}(zc - cy), then the root
// correction X[root columns] += W_r u of the block's columns.
__global__ void __launch_bounds__(256) k_coarse_out(int nc, const int64_t* __restrict__ cg_ptr,
                                                    const int64_t* __restrict__ cg_idx, const double* __restrict__ gl,
                                                    const double* __restrict__ Ainv, const int32_t* __restrict__ coarse_id,
                                                    const int64_t* __restrict__ m_off, const int64_t* __restrict__ s_off,
                                                    const double* __restrict__ sinv, const double* __restrict__ cy,
                                                    const int64_t* __restrict__ rinfo, const int32_t* __restrict__ cslot,
                                                    const double* __restrict__ W, double* __restrict__ X,
                                                    const int* __restrict__ skip, const double* __restrict__ Hc,
                                                    const int32_t* __restrict__ hslot) {
  if (skip && *skip) return;
  extern __shared__ double gc[];  // nc, then zc and u (kFusedCoarseM each)
  double* zl = gc + nc;
  double* u = zl + kFusedCoarseM;
  const int sd = blockIdx.x, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int64_t b0 = m_off[sd];
  const int m = (int)(m_off[sd + 1] - b0);
#ifndef CUTBDDC_COARSE_OUT_PLAIN
  {  // this block's H (or W_r) columns on their way to L2 while gc, zc and u are formed
    const int cr0 = (int)rinfo[4 * sd], j0 = blockIdx.y * blockDim.x + tid;
    if (j0 < cr0 && (tid & 15) == 0) {  // one request per 128 bytes
      const double* base = (Hc ? Hc : W) + rinfo[4 * sd + 3] + j0;
      for (int a = 0; a < m; ++a) asm volatile("prefetch.global.L2 [%0];" ::"l"(base + (int64_t)a * cr0));
    }
  }
#endif
  for (int lam = tid; lam < nc; lam += blockDim.x) {
    double v = 0.0;
    for (int64_t p = cg_ptr[lam]; p < cg_ptr[lam + 1]; ++p) v += gl[cg_idx[p]];
    gc[lam] = v;
  }
  __syncthreads();
  // zc rows, a warp per row; four rows of a warp in flight at once (each row's
  // sum keeps its order: s0 over c = lane, lane + 64, ..; s1 over lane + 32, ..)
#ifdef CUTBDDC_COARSE_OUT_PLAIN
  constexpr int kRows = 1;
#else
  constexpr int kRows = 4;
#endif
  const int nw = blockDim.x >> 5;
  for (int a0 = wid; a0 < m; a0 += nw * kRows) {
    const double* ar[kRows];
    double s0[kRows], s1[kRows];
#pragma unroll
    for (int r = 0; r < kRows; ++r) {
      const int a = a0 + r * nw;
      ar[r] = Ainv + (int64_t)coarse_id[b0 + (a < m ? a : a0)] * nc;
      s0[r] = s1[r] = 0.0;
    }
    int c = lane;
    for (; c + 32 < nc; c += 64) {
      const double g0 = gc[c], g1 = gc[c + 32];
#pragma unroll
      for (int r = 0; r < kRows; ++r) {
        s0[r] += ar[r][c] * g0;
        s1[r] += ar[r][c + 32] * g1;
      }
    }
    for (; c < nc; c += 32) {
      const double g0 = gc[c];
#pragma unroll
      for (int r = 0; r < kRows; ++r) s0[r] += ar[r][c] * g0;
    }
#pragma unroll
    for (int r = 0; r < kRows; ++r) {
      const double v = warp_sum(s0[r] + s1[r]);
      if (lane == 0 && a0 + r * nw < m) zl[a0 + r * nw] = v;
    }
  }
  __syncthreads();
  for (int a = tid; a < m; a += blockDim.x) {
    const double* si = sinv + s_off[sd] + (int64_t)a * m;
    double v = 0.0;
    for (int b = 0; b < m; ++b) v += si[b] * (zl[b] - cy[b0 + b]);
    u[a] = v;
  }
  __syncthreads();
  const int cr = (int)rinfo[4 * sd];
  const int j = blockIdx.y * blockDim.x + tid;
  if (j >= cr) return;
  if (Hc) {  // corner formulation: y'[slot_j] += (H u)_j (X: the forward sweep's column values)
    const double* hc = Hc + rinfo[4 * sd + 3] + j;
    double v = 0.0;
    for (int a = 0; a < m; ++a) v += hc[(int64_t)a * cr] * u[a];
    X[hslot[rinfo[4 * sd + 1] + j]] += v;
    return;
  }
  const double* w = W + rinfo[4 * sd + 3] + j;
  double v = 0.0;
  for (int a = 0; a < m; ++a) v += w[(int64_t)a * cr] * u[a];
  X[cslot[rinfo[4 * sd + 2] + j]] += v;
}

// Constraint rows expanded on the device, a warp per local row (subdomain sd,
// object o): entry e of the row is the object's e-th dof with coefficient 1
// (corner) or 1 / |object| (edge / face average), stored as
// its slot in the subdomain's (B+1)^3 lattice. The host passes only the row
// pointers and the coarse view's CSR arrays (no per-entry host loop, no
// per-entry upload). bad[1]: 1 + the first subdomain found with an object dof
// outside its block; bad[2]: a dof id outside [0, n_dof).
__global__ void __launch_bounds__(256) k_rows_expand(int64_t mtot, int n, int B, int nb, int b1, int64_t n_dof,
                                                     const int64_t* __restrict__ c_ptr, const int32_t* __restrict__ row_sd,
                                                     const int32_t* __restrict__ coarse_id,
                                                     const uint8_t* __restrict__ corner, const int64_t* __restrict__ dof_ptr,
                                                     const int32_t* __restrict__ dofs, const int64_t* __restrict__ block_ids,
                                                     const int64_t* __restrict__ node_of_dof, int32_t* __restrict__ c_slot,
                                                     double* __restrict__ c_val, int* __restrict__ bad) {
  const int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (row >= mtot) return;
  const int lane = threadIdx.x & 31;
  const int sd = row_sd[row], o = coarse_id[row];
  const int64_t e0 = c_ptr[row], cnt = c_ptr[row + 1] - e0, d0 = dof_ptr[o];
  const double coef = corner[row] ? 1.0 : 1.0 / (double)cnt;
  const int64_t bid = block_ids[sd];
  const int bi = (int)(bid / nb / nb), bj = (int)((bid / nb) % nb), bk = (int)(bid % nb);
  for (int64_t q = lane; q < cnt; q += 32) {
    const int32_t d = dofs[d0 + q];
    int slot = 0;
    if (d < 0 || d >= n_dof) {
      atomicCAS(bad + 2, 0, 1);
    } else {
      const int64_t v = node_of_dof[d];
      const int k = (int)(v % (n + 1)), j = (int)((v / (n + 1)) % (n + 1)), i = (int)(v / (n + 1) / (n + 1));
      const int lx = i - bi * B, ly = j - bj * B, lz = k - bk * B;
      if (lx < 0 || ly < 0 || lz < 0 || lx > B || ly > B || lz > B)
        atomicCAS(bad + 1, 0, 1 + sd);
      else
        slot = (lx * b1 + ly) * b1 + lz;
    }
    c_slot[e0 + q] = slot;
    c_val[e0 + q] = coef;
  }
}

__global__ void k_row_sd(int nsd, const int64_t* __restrict__ m_off, int32_t* __restrict__ row_sd) {
  const int sd = blockIdx.x;
  for (int64_t r = m_off[sd] + threadIdx.x; r < m_off[sd + 1]; r += blockDim.x) row_sd[r] = sd;
}

// Subdomains whose K_c cannot be used: a non-positive pivot in the
// factorisation (flagged by the DAG into bad_dev) or a pivot tiny against
// the original diagonal (k_pivot_check). bad: per subdomain, host.
int corner_bad_subdomains(cutbddc_gpu* h, int* bad_dev, std::vector<uint8_t>& bad) {
  cudaStream_t s = h->stream;
  const int nsn = (int)h->tI.tpl.sn.size();
  k_pivot_check<<<dim3(nsn, h->nsd), 128, 0, s>>>(nsn, h->slots, reinterpret_cast<const FrontDesc*>(h->fK.desc.p),
                                                   h->fK.panel.p, h->fK.cslot.p, h->As.p, h->diag_add.p, bad_dev);
  CB_LAUNCH();
  std::vector<int> hb((size_t)h->nsd);
  CB_CUDA(cudaMemcpyAsync(hb.data(), bad_dev, sizeof(int) * h->nsd, cudaMemcpyDeviceToHost, s));
  CB_CUDA(cudaStreamSynchronize(s));
  bad.assign((size_t)h->nsd, 0);
  // test hook: CUTBDDC_K_MIXED_EVERY=n puts every n-th subdomain on the
  // shell-root K (the mixed path on meshes where K_c is never singular)
  const int every = [] {
    const char* e = std::getenv("CUTBDDC_K_MIXED_EVERY");
    return e ? std::max(0, std::atoi(e)) : 0;
  }();
  int nb = 0;
  for (int sd = 0; sd < h->nsd; ++sd)
    nb += bad[(size_t)sd] = hb[(size_t)sd] != 0 || (every > 0 && sd % every == 0);
  if (nb && std::getenv("CUTBDDC_K_STATS"))
    std::fprintf(stderr, "[cutbddc] K_c unusable in %d of %d subdomains: shell-root K there\n", nb, h->nsd);
  return nb;
}

__global__ void k_mask_sd(int64_t ns, int T, const uint8_t* __restrict__ mask, const uint8_t* __restrict__ sel,
                          uint8_t* __restrict__ out) {
  const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g < ns) out[g] = mask[g] && sel[g / T];
}

// S^{-1} (symmetrised) of every subdomain's m x m block in place; a
// non-positive pivot means dependent constraints
void invert_schur(cutbddc_gpu* h, double* S) {
  cudaStream_t s = h->stream;
  DevBuf<unsigned long long>& fail = h->ws_fail;
  fail.alloc(1);
  CB_CUDA(cudaMemsetAsync(fail.p, 0xff, 8, s));
  const size_t shm = sizeof(double) * ((size_t)h->m_max * h->m_max + h->m_max);
  if (shm > 48 * 1024)
    CB_CUDA(cudaFuncSetAttribute(k_small_spd_inverse, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm));
  k_small_spd_inverse<<<h->nsd, 256, shm, s>>>(h->nsd, h->m_off.p, h->ac_off.p, S, fail.p);
  CB_LAUNCH();
  unsigned long long f = 0;
  CB_CUDA(cudaMemcpyAsync(&f, fail.p, 8, cudaMemcpyDeviceToHost, s));
  CB_CUDA(cudaStreamSynchronize(s));
  if (f != ~0ull)
    throw Failure(CUTBDDC_SINGULAR, "saddle: singular constraint Schur complement (subdomain " + std::to_string(f) +
                                        "); constraints are not independent");
}

// Coarse basis of the corner formulation: H = L^{-1} C^T by multi-RHS
// forward sweeps (kSweepMultiRhs constraint rows of every subdomain per
// pass), S = H^T H, S^{-1}, A_c,w = S^{-1} - rho I_corner.
void coarse_basis_corner(cutbddc_gpu* h, const std::vector<int64_t>& m_off, const std::vector<int64_t>& s_off,
                         const std::vector<uint8_t>& shell_sd, double* S) {
  cudaStream_t s = h->stream;
  const int nsd = h->nsd, T = h->slots, m_max = h->m_max;
  const TplSet& ts = h->tI;
  const FactorSet& f = h->fK;
  const int nsn = (int)ts.tpl.sn.size();
  std::vector<int32_t> coff((size_t)nsd * nsn);
  std::vector<int64_t> rinfo((size_t)4 * nsd);
  int64_t hs = 0, ht = 0;
  int np_max = 0;
  for (int sd = 0; sd < nsd; ++sd) {
    int k = 0;
    for (int sid = 0; sid < nsn; ++sid) {
      coff[(size_t)sd * nsn + sid] = k;
      k += f.h_rc[(size_t)sd * nsn + sid].y;
    }
    if (!shell_sd.empty() && shell_sd[(size_t)sd]) k = 0;  // its K is the shell-root one
    const int64_t m = m_off[(size_t)sd + 1] - m_off[(size_t)sd];
    rinfo[4 * (size_t)sd] = k;
    rinfo[4 * (size_t)sd + 1] = hs;
    rinfo[4 * (size_t)sd + 2] = 0;
    rinfo[4 * (size_t)sd + 3] = ht;
    hs += k;
    ht += (int64_t)k * m;
    np_max = std::max(np_max, k);
  }
  h->np_max = np_max;
  h->root_info.upload(rinfo, s);
  DevBuf<int32_t>& dcoff = h->ws_coff;
  dcoff.upload(coff, s);
  h->hroot.alloc((size_t)std::max<int64_t>(1, ht));
  h->hslot.alloc((size_t)std::max<int64_t>(1, hs));
  const int64_t ns = (int64_t)nsd * T;
  h->ws_x8.alloc((size_t)kSweepMultiRhs * ns);
  h->ws_y8.alloc((size_t)kSweepMultiRhs * ns);
  h->ws_u8.alloc((size_t)kSweepMultiRhs * std::max<int64_t>(1, f.upd_total));
  h->ws_v8.alloc((size_t)kSweepMultiRhs * std::max<size_t>(1, f.vbuf.n));
  ProfScope pc(h->prof, s, "coarse basis H passes");
  for (int pass = 0; pass * kSweepMultiRhs < m_max; ++pass) {
    h->ws_x8.zero(s);
    k_ct_rhs<<<dim3(nsd, kSweepMultiRhs), 128, 0, s>>>(pass, ns, T, h->m_off.p, h->c_ptr.p, h->c_slot.p, h->c_val.p,
                                                        h->ws_x8.p);
    CB_LAUNCH();
    sweep_forward_multi(h, ts, f, h->ws_x8.p, h->ws_y8.p, h->ws_u8.p, h->ws_v8.p);
    k_h_compact<<<dim3(nsn, nsd), 128, 0, s>>>(pass, nsn, ns, reinterpret_cast<const FrontDesc*>(f.desc.p), f.cslot.p,
                                              dcoff.p, h->m_off.p, h->root_info.p, h->ws_y8.p, h->hroot.p, h->hslot.p);
    CB_LAUNCH();
  }
  pc.next("coarse basis S");
  k_root_s<<<dim3(nsd, m_max), 256, 0, s>>>(h->root_info.p, h->m_off.p, h->ac_off.p, h->hroot.p, S,
                                            shell_sd.empty() ? nullptr : h->kform_shell.p);
  CB_LAUNCH();
}

// Coarse basis of the shell-root formulation K = A + rho C^T C on the
// subdomains factorised in fs (all, or the shell part of a mixed K): H =
// G_r C_r^T, S = H^T H, W_r = G_r^T H in the root space (see k_root_h).
void coarse_basis_shell(cutbddc_gpu* h, const std::vector<int64_t>& m_off, const FactorSet& fs, bool mixed,
                        double* S) {
  cudaStream_t s = h->stream;
  const int nsd = h->nsd, m_max = h->m_max;
  const int nsn = (int)h->tK.tpl.sn.size(), root = nsn - 1;
  std::vector<int64_t> rinfo((size_t)4 * nsd);
  int64_t wtot = 0;
  int cr_max = 0;
  for (int sd = 0; sd < nsd; ++sd) {
    const size_t q = (size_t)sd * nsn + root;
    const int cr = fs.h_rc[q].y;  // 0: not a shell subdomain (mixed)
    if (fs.h_rc[q].x != cr) throw Failure(CUTBDDC_INTERNAL, "shell root with update rows");
    const int m = (int)(m_off[(size_t)sd + 1] - m_off[(size_t)sd]);
    rinfo[4 * (size_t)sd] = cr;
    rinfo[4 * (size_t)sd + 1] = fs.h_panel_off[q];
    rinfo[4 * (size_t)sd + 2] = fs.h_vec_off[q];
    rinfo[4 * (size_t)sd + 3] = wtot;
    wtot += (int64_t)cr * m;
    cr_max = std::max(cr_max, cr);
  }
  h->root_info_s.upload(rinfo, s);
  h->hroot_s.alloc((size_t)std::max<int64_t>(1, wtot));
  h->wroot.alloc((size_t)std::max<int64_t>(1, wtot));
  if (cr_max == 0) return;
  const int32_t* pfx_root = fs.pfx.p + h->tK.tpl.sn[(size_t)root].rows_off;
  const int64_t rows_total = (int64_t)h->tK.tpl.rows.size();
  k_root_h<<<dim3(nsd, m_max), 256, 0, s>>>(h->root_info_s.p, h->m_off.p, h->c_ptr.p, h->c_slot.p, h->c_val.p,
                                            h->tK.root_pos.p, pfx_root, rows_total, fs.panel.p, h->hroot_s.p);
  CB_LAUNCH();
  k_root_s<<<dim3(nsd, m_max), 256, 0, s>>>(h->root_info_s.p, h->m_off.p, h->ac_off.p, h->hroot_s.p, S,
                                            mixed ? h->kform_corner.p : nullptr);
  CB_LAUNCH();
  k_root_w<<<dim3(nsd, (cr_max + 63) / 64), 256, 0, s>>>(h->root_info_s.p, h->m_off.p, fs.panel.p, h->hroot_s.p,
                                                        h->wroot.p);
  CB_LAUNCH();
}

}  // namespace

void setup_bddc_device(cutbddc_gpu* h, const cutbddc_coarse_view* cv, int weighting) {
  if (!h->assembled) throw Failure(CUTBDDC_INVALID_ARGUMENT, "setup_bddc: assemble first");
  cudaStream_t s = h->stream;
  const int nsd = h->nsd, T = h->slots, b1 = h->b1;
  const int64_t ns = (int64_t)nsd * T;
  h->weighting = weighting;
  h->bddc_ready = false;
  if (h->graph_exec) {
    cudaGraphExecDestroy(h->graph_exec);
    h->graph_exec = nullptr;
  }
  if (h->graph_exec_ref) {
    cudaGraphExecDestroy(h->graph_exec_ref);
    h->graph_exec_ref = nullptr;
  }
  if (h->plan_only) throw Failure(CUTBDDC_CONFIG, "setup_bddc: plan-only distribution (no communicator)");
  // ---- host: constraint rows per subdomain from the coarse objects. The
  // coarse view names global subdomains (every rank passes the same view).
  // Local rows: this rank's subdomains in order, objects ascending. Staged
  // rows (the rank-major layout the coarse all-gathers fill, dist.cuh): every
  // subdomain's rows at rank(sd) * maxrows + (rows of that rank's earlier
  // subdomains); one rank: staged == local.
  ProfScope ps_host(h->prof, s, "setup 0 host rows+uploads+weights");
  const int nc = cv ? cv->n_objects : 0;
  const int nsd_g = h->nsd_g, world = h->dist_world, rank = h->dist_rank;
  ps_host.next("setup 0a host rows");
  std::vector<std::vector<int>> obj_of_gsd((size_t)nsd_g);  // object ids per global sd (ascending)
  for (int o = 0; o < nc; ++o)
    for (int64_t p = cv->neigh_ptr[o]; p < cv->neigh_ptr[o + 1]; ++p) {
      const int sg = cv->neigh[p];
      if (sg < 0 || sg >= nsd_g) throw Failure(CUTBDDC_INVALID_ARGUMENT, "coarse view: neighbour subdomain out of range");
      if (!obj_of_gsd[(size_t)sg].empty() && obj_of_gsd[(size_t)sg].back() >= o)
        throw Failure(CUTBDDC_INVALID_ARGUMENT, "coarse view: repeated neighbour subdomain");
      obj_of_gsd[(size_t)sg].push_back(o);
    }
  std::vector<int64_t> rows_of_rank((size_t)world, 0), ac_of_rank((size_t)world, 0), roff_g((size_t)nsd_g),
      aoff_g((size_t)nsd_g);
  int64_t m_total_g = 0;
  for (int g = 0; g < nsd_g; ++g) {
    const int q = h->rank_of_gsd[(size_t)g];
    const int64_t m = (int64_t)obj_of_gsd[(size_t)g].size();
    roff_g[(size_t)g] = rows_of_rank[(size_t)q];
    aoff_g[(size_t)g] = ac_of_rank[(size_t)q];
    rows_of_rank[(size_t)q] += m;
    ac_of_rank[(size_t)q] += m * m;
    m_total_g += m;
  }
  h->maxrows = std::max<int64_t>(1, *std::max_element(rows_of_rank.begin(), rows_of_rank.end()));
  h->maxac = std::max<int64_t>(1, *std::max_element(ac_of_rank.begin(), ac_of_rank.end()));
  h->m_total_g = m_total_g;
  const int64_t nstage = (int64_t)world * h->maxrows;
  std::vector<int64_t> srow((size_t)3 * nstage, 0);
  std::vector<int32_t> scoarse((size_t)nstage, 0);
  // cg: per coarse object the staged rows of its copies, ascending global sd (CSR)
  std::vector<int64_t> cg_ptr((size_t)nc + 1, 0);
  for (int o = 0; o < nc; ++o) cg_ptr[(size_t)o + 1] = cg_ptr[(size_t)o] + (cv->neigh_ptr[o + 1] - cv->neigh_ptr[o]);
  std::vector<int64_t> cg_idx((size_t)cg_ptr[(size_t)nc]), cg_cur(cg_ptr.begin(), cg_ptr.end() - 1);
  for (int g = 0; g < nsd_g; ++g) {
    const int q = h->rank_of_gsd[(size_t)g];
    const int64_t first = (int64_t)q * h->maxrows + roff_g[(size_t)g];
    const int64_t m = (int64_t)obj_of_gsd[(size_t)g].size();
    for (int64_t a2 = 0; a2 < m; ++a2) {
      const int64_t p = first + a2;
      srow[(size_t)(3 * p)] = first;
      srow[(size_t)(3 * p + 1)] = m;
      srow[(size_t)(3 * p + 2)] = (int64_t)q * h->maxac + aoff_g[(size_t)g];
      const int o = obj_of_gsd[(size_t)g][(size_t)a2];
      scoarse[(size_t)p] = o;
      cg_idx[(size_t)cg_cur[(size_t)o]++] = p;  // ascending global sd
    }
  }
  // constraint rows: per (subdomain, object) the object's dofs; their slots in
  // the subdomain's lattice are computed on the device (k_rows_expand) from
  // node_of_dof, so the host never needs the mesh maps
  std::vector<int64_t> m_off((size_t)nsd + 1, 0), c_ptr{0};
  std::vector<int32_t> coarse_id;
  std::vector<uint8_t> corner;
  const int n = h->n, B = h->block, nb = h->nb;
  {
    size_t rows = 0;
    for (int sd = 0; sd < nsd; ++sd) rows += obj_of_gsd[(size_t)h->global_of_local[(size_t)sd]].size();
    coarse_id.reserve(rows + 1);
    corner.reserve(rows + 1);
    c_ptr.reserve(rows + 1);
  }
  for (int sd = 0; sd < nsd; ++sd) {
    const int g = h->global_of_local[(size_t)sd];
    for (int o : obj_of_gsd[(size_t)g]) {
      coarse_id.push_back(o);
      corner.push_back(cv->kinds[o] == CUTBDDC_CORNER);
      c_ptr.push_back(c_ptr.back() + (cv->dof_ptr[o + 1] - cv->dof_ptr[o]));  // entries expanded by k_rows_expand
    }
    m_off[(size_t)sd + 1] = (int64_t)coarse_id.size();
  }
  h->n_coarse = nc;
  h->m_total = (int64_t)coarse_id.size();
  h->h_m_off = m_off;
  int m_max = 0;
  std::vector<int64_t> s_off((size_t)nsd + 1, 0);
  for (int sd = 0; sd < nsd; ++sd) {
    const int m = (int)(m_off[(size_t)sd + 1] - m_off[(size_t)sd]);
    s_off[(size_t)sd + 1] = s_off[(size_t)sd] + (int64_t)m * m;
  }
  for (int g = 0; g < nsd_g; ++g) m_max = std::max(m_max, (int)obj_of_gsd[(size_t)g].size());  // uniform over ranks
  h->m_max = m_max;
  const int64_t n_centries = c_ptr.back();
  const int64_t n_rows = (int64_t)coarse_id.size();
  if (coarse_id.empty()) coarse_id.push_back(0), corner.push_back(0);
  if (cg_idx.empty()) cg_idx.push_back(0);
  h->m_off.upload(m_off, s);
  h->c_ptr.upload(c_ptr, s);
  h->coarse_id.upload(coarse_id, s);
  h->corner_row.upload(corner, s);
  const uint8_t* d_corner = h->corner_row.p;
  h->row_sd.alloc((size_t)std::max<int64_t>(1, h->m_total));
  k_row_sd<<<nsd, 128, 0, s>>>(nsd, h->m_off.p, h->row_sd.p);
  CB_LAUNCH();
  {
    DevBuf<int>& flags = h->ws_flag;  // [0] weights, [1] [2] constraint rows: read together after the weights
    flags.alloc(3);
    flags.zero(s);
    h->c_slot.alloc((size_t)std::max<int64_t>(1, n_centries));
    h->c_val.alloc((size_t)std::max<int64_t>(1, n_centries));
    if (n_centries > 0) {
      // the coarse view's object dofs (CSR), expanded per (subdomain, object) row on the device
      h->ws_cdof.upload(cv->dofs, (size_t)cv->dof_ptr[nc], s);
      h->ws_odofptr.upload(cv->dof_ptr, (size_t)nc + 1, s);
      k_rows_expand<<<grid_for(n_rows * 32, 256), 256, 0, s>>>(n_rows, n, B, nb, b1, h->n_dof, h->c_ptr.p, h->row_sd.p,
                                                               h->coarse_id.p, d_corner, h->ws_odofptr.p, h->ws_cdof.p,
                                                               h->block_ids.p, h->node_of_dof.p, h->c_slot.p, h->c_val.p,
                                                               flags.p);
      CB_LAUNCH();
    }
  }
  h->cg_ptr.upload(cg_ptr, s);
  h->cg_idx.upload(cg_idx, s);
  h->srow.upload(srow, s);
  h->scoarse.upload(scoarse, s);
  h->ac_off.upload(s_off, s);
  ps_host.next("setup 0b weights");
  // ---- weights, rho
  DevBuf<int>& bad = h->ws_flag;  // zeroed with the constraint rows above
  h->w.alloc((size_t)ns);
  h->dtot.alloc((size_t)std::max<int64_t>(1, h->n_loc));
  h->sv2.alloc((size_t)ns);
  if (weighting == CUTBDDC_WEIGHT_STIFFNESS) {  // Σ over every copy of the A^w diagonal
    k_diag_slots<<<grid_for(ns, 256), 256, 0, s>>>(ns, T, h->As.p, h->sv2.p);
    CB_LAUNCH();
    iface_exchange(h, h->sv2.p, nullptr, nullptr);
    iface_sum(h, h->sv2.p, nullptr, h->dtot.p, nullptr);
  }
  k_weights<<<grid_for(ns, 256), 256, 0, s>>>(ns, T, weighting, h->slot_dof.p, h->slot_loc.p, h->ncount.p, h->As.p,
                                              h->dtot.p, h->w.p, bad.p);
  CB_LAUNCH();
  // Local failures (non-positive pivots, zero weight denominators, dependent
  // constraints) must not leave other ranks waiting in a collective: each
  // phase runs under `local`, then every rank learns the worst status
  // (agree_status) before the next collective. One rank: no exchange.
  int64_t upd_total = 1;
  cutbddc_status fail_code = CUTBDDC_OK;
  std::string fail_msg;
  auto local = [&](auto&& fn) {
    if (fail_code != CUTBDDC_OK) return;
    try {
      fn();
    } catch (const Failure& e) {
      fail_code = e.code;
      fail_msg = e.what();
    }
  };
  auto agree = [&](int extra) {  // returns the max over ranks of `extra` (0/1); throws on any failure
    const int c = agree_status(h, ((int)fail_code << 1) | extra);
    if (c >> 1) throw Failure((cutbddc_status)(c >> 1), fail_msg.empty() ? "setup_bddc: failed on another rank" : fail_msg);
    return c & 1;
  };
  static const char* kSaddleMsg = "saddle: singular augmented system; constraints do not control the operator kernel";
  h->rho.alloc((size_t)nsd);  // before the FactorInputs take their pointers
  h->diag_add.alloc((size_t)ns);
  FactorInput fi{h->As.p, h->mask_int.p, nullptr, T, b1, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  FactorInput fk{h->As.p, h->mask_all.p, h->diag_add.p, T, b1,
                 h->m_off.p, h->c_ptr.p, h->c_slot.p, h->c_val.p, d_corner, h->rho.p};
  FactorInput fk_c{h->As.p, h->mask_all.p, h->diag_add.p, T, b1, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  // Without an interface (one subdomain) every dof is interior: the weighted
  // residual r_w is identically zero and the constrained Neumann solve drops
  // out of the apply ("preconditioner reduces to exact interior solve").
  h->has_K = h->n_if > 0;
  h->fK.upd_total = 0;
  h->fKs.upd_total = 0;
  // K: corner-augmented K_c = A + rho sum_corners e e^T on the plain ND
  // template (no rho C^T C rows: fk_c has no constraint rows), else the full
  // K = A + rho C^T C on the shell-root template (PEN rows of the root).
  const bool force_shell = [] {
    const char* e = std::getenv("CUTBDDC_K_SHELL");
    return e && e[0] == '1';
  }();
  h->k_corner = !force_shell && m_max > 0;
  int n_bad = 0;                   // subdomains whose K_c is unusable (this rank)
  std::vector<uint8_t> bad_sd;
  DevBuf<int>& bad_dev = h->ws_badsd;
  bad_dev.alloc((size_t)nsd);
  bad_dev.zero(s);
  local([&] {
    const size_t rho_shm = sizeof(double) * (size_t)T;
    if (rho_shm > 48 * 1024) CB_CUDA(cudaFuncSetAttribute(k_rho, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rho_shm));
    k_rho<<<nsd, 256, rho_shm, s>>>(nsd, T, h->slot_dof.p, h->As.p, h->rho.p);
    CB_LAUNCH();
    h->diag_add.zero(s);
    k_diag_add<<<nsd, 128, 0, s>>>(nsd, T, h->m_off.p, h->c_ptr.p, h->c_slot.p, d_corner, h->rho.p, h->diag_add.p);
    CB_LAUNCH();
    int hbad[3] = {0, 0, 0};
    CB_CUDA(cudaMemcpyAsync(hbad, bad.p, 12, cudaMemcpyDeviceToHost, s));
    CB_CUDA(cudaStreamSynchronize(s));
    if (hbad[2]) throw Failure(CUTBDDC_INVALID_ARGUMENT, "coarse view: dof out of range");
    if (hbad[1])
      throw Failure(CUTBDDC_INVALID_ARGUMENT,
                    "coarse view: object dof not in neighbour subdomain " +
                        std::to_string(h->global_of_local[(size_t)(hbad[1] - 1)]));
    if (hbad[0]) throw Failure(CUTBDDC_DEGENERATE, "weighting: zero total diagonal at an interface dof");
    ps_host.next("setup 1 factorisations");
    // ---- factorisations
    if (!h->tI.ready || h->tI.tpl.b1 != b1) upload_template(h, h->tI, false);
    set_split_flags(h->tI, nsd);
    factor_symbolic(h, h->tI, fi, h->fI);
    std::vector<FactorJob> jobs{FactorJob{&h->tI, &fi, &h->fI, "cholesky (interior problem)"}};
    bool k_failed = false;
    if (h->has_K) {
      if (h->k_corner) {
        factor_symbolic(h, h->tI, fk_c, h->fK);
        jobs.push_back(FactorJob{&h->tI, &fk_c, &h->fK, kSaddleMsg, &k_failed, bad_dev.p});
      } else {
        if (!h->tK.ready || h->tK.tpl.b1 != b1) upload_template(h, h->tK, true);
        set_split_flags(h->tK, nsd);
        factor_symbolic(h, h->tK, fk, h->fK);
        jobs.push_back(FactorJob{&h->tK, &fk, &h->fK, kSaddleMsg});
      }
    }
    factor_numeric(h, jobs, [&] {  // the sweep item lists on the host while the GPU factorises
      // two host threads (cfg5: ~50 ms of list building and sorting per factor
      // against 75 ms of factorisation)
      std::exception_ptr kerr;
      std::thread tk;
      if (h->has_K)
        tk = std::thread([&] {
          try {
            CB_CUDA(cudaSetDevice(h->device));
            build_sweep_items(h, h->k_corner ? h->tI : h->tK, h->fK);
          } catch (...) {
            kerr = std::current_exception();
          }
        });
      try {
        build_sweep_items(h, h->tI, h->fI);
      } catch (...) {
        if (tk.joinable()) tk.join();
        throw;
      }
      if (tk.joinable()) tk.join();
      if (kerr) std::rethrow_exception(kerr);
    });
    if (h->has_K && h->k_corner) n_bad = corner_bad_subdomains(h, bad_dev.p, bad_sd);
  });
  // A floating fragment (no corner, no Nitsche boundary) leaves K_c singular
  // on its subdomain: there K = A + rho C^T C on the shell-root template
  // instead (a mixed K: the corner formulation everywhere else). The mode is
  // agreed over the ranks (one apply path: the same numbers for any world size).
  h->k_mixed = false;
  h->n_shell_sd = n_bad;
  if (agree(n_bad > 0 ? 1 : 0) && h->has_K && h->k_corner) {
    h->k_mixed = true;
    local([&] {
      std::vector<uint8_t> corner_sd((size_t)nsd);
      for (int sd = 0; sd < nsd; ++sd) corner_sd[(size_t)sd] = !bad_sd[(size_t)sd];
      h->kform_shell.upload(bad_sd, s);
      h->kform_corner.upload(corner_sd, s);
      exclude_sweep_items(h, h->fK, bad_sd);  // K_c sweeps skip the shell subdomains, fKs's the others
      if (!h->tK.ready || h->tK.tpl.b1 != b1) upload_template(h, h->tK, true);
      set_split_flags(h->tK, nsd);
      DevBuf<uint8_t>& mask_s = h->mask_shell;
      mask_s.alloc((size_t)ns);
      k_mask_sd<<<grid_for(ns, 256), 256, 0, s>>>(ns, T, h->mask_all.p, h->kform_shell.p, mask_s.p);
      CB_LAUNCH();
      FactorInput fk_s = fk;
      fk_s.mask = mask_s.p;
      factor_symbolic(h, h->tK, fk_s, h->fKs);
      factor_numeric(h, {FactorJob{&h->tK, &fk_s, &h->fKs, kSaddleMsg}}, [&] { build_sweep_items(h, h->tK, h->fKs, &corner_sd); }, true);
    });
    agree(0);
  }
  upd_total = std::max<int64_t>(1, std::max(h->fI.upd_total, std::max(h->fK.upd_total, h->k_mixed ? h->fKs.upd_total : 0)));
  local([&] {
    // ---- coarse basis: S = C K^{-1} C^T per subdomain in the formulation's
    // factor space (corner: H = L^{-1} C^T; shell: the root space), then
    // S^{-1} and A_c,w = S^{-1} - rho I_aug; the apply never forms Phi
    h->ac_loc.alloc((size_t)(world * h->maxac));  // staged: this rank's blocks at rank * maxac
    h->ac_loc.zero(s);
    h->sinv.alloc((size_t)std::max<int64_t>(1, s_off[(size_t)nsd]));
    ps_host.next("setup 2 root-space coarse basis");
    if (m_max > 0) {
      if (!h->has_K) throw Failure(CUTBDDC_INTERNAL, "coarse space without an interface");
      DevBuf<double>& S = h->ws_s;
      S.alloc((size_t)std::max<int64_t>(1, s_off[(size_t)nsd]));
      if (h->k_corner) coarse_basis_corner(h, m_off, s_off, h->k_mixed ? bad_sd : std::vector<uint8_t>{}, S.p);
      if (!h->k_corner || h->k_mixed) coarse_basis_shell(h, m_off, h->k_mixed ? h->fKs : h->fK, h->k_mixed, S.p);
      invert_schur(h, S.p);
      k_root_coarse<<<nsd, 256, 0, s>>>(h->m_off.p, h->ac_off.p, S.p, h->rho.p, h->k_corner ? h->corner_row.p : nullptr,
                                        h->sinv.p, h->ac_loc.p + (int64_t)h->dist_rank * h->maxac,
                                        h->k_mixed ? h->kform_shell.p : nullptr);
      CB_LAUNCH();
    }
  });
  agree(0);
  // ---- coarse matrix + factorisation
  ps_host.next("setup 4 coarse assemble+chol+inverse");
  h->acoarse.alloc((size_t)std::max(1, nc * nc));
  // n_c <= kCoarseInverseMax: dense Cholesky + explicit inverse (one GEMV per
  // apply); larger: the nested-dissection factor (coarse_sparse.cu)
  // (CUTBDDC_COARSE=dense / sparse forces one path: A/B runs, tests)
  const char* coarse_env = std::getenv("CUTBDDC_COARSE");
  const std::string coarse_mode = coarse_env ? coarse_env : "";
  h->coarse_sparse = coarse_mode == "sparse" || (nc > kCoarseInverseMax && coarse_mode != "dense");
  if (nc > 0) {
    h->acoarse.zero(s);
    // every subdomain's A_c,w on every rank, then the same assembly in
    // global subdomain order everywhere
    gather_blocks(h);
    k_coarse_assemble<<<nc, 128, 0, s>>>(nc, h->cg_ptr.p, h->cg_idx.p, h->srow.p, h->scoarse.p, h->ac_loc.p,
                                         h->acoarse.p);
    CB_LAUNCH();
    DevBuf<unsigned long long>& fail = h->ws_fail;
    fail.alloc(1);
    CB_CUDA(cudaMemsetAsync(fail.p, 0xff, 8, s));
    if (h->coarse_sparse) {
      coarse_sparse_setup(h, nc, obj_of_gsd);
      coarse_sparse_factor(h, h->acoarse.p, nc, fail.p);
    } else {
      // Cholesky of A_c and X = L^{-1} by the tiled dense DAG (A_c is
      // symmetric, so its row-major buffer is its column-major lower part);
      // the apply solves with X^T (X g): two triangular GEMVs.
      h->acoarse_inv.alloc((size_t)std::max(1, nc * nc));
      DevBuf<double>& Lc = h->ws_lc;
      Lc.alloc((size_t)nc * nc);
      CB_CUDA(cudaMemcpyAsync(Lc.p, h->acoarse.p, sizeof(double) * nc * nc, cudaMemcpyDeviceToDevice, s));
      dense_dag_matrix(h, Lc.p, h->acoarse_inv.p, nc, fail.p);
      if (nc <= kCoarseInverseMax) {
        h->acoarse_full.alloc((size_t)nc * nc);
        const int nb64 = (nc + 63) / 64;
        k_xtx<<<dim3(nb64, nb64), 256, 0, s>>>(nc, h->acoarse_inv.p, h->acoarse_full.p);
        CB_LAUNCH();
      } else {
        h->ws_cpart.alloc((size_t)((nc + 63) / 64) * nc);
      }
    }
    unsigned long long f = 0;
    CB_CUDA(cudaMemcpyAsync(&f, fail.p, 8, cudaMemcpyDeviceToHost, s));
    CB_CUDA(cudaStreamSynchronize(s));
    if (f != ~0ull)
      throw Failure(CUTBDDC_SINGULAR, "coarse matrix: not positive definite (pivot index " + std::to_string(f) + ")");
  }
  // ---- work vectors
  ps_host.next("setup 5 work vectors");
  h->sv0.alloc((size_t)ns);
  h->sv1.alloc((size_t)ns);
  h->sx.alloc((size_t)ns);  // operator input (allocated here: never inside a graph capture)
  h->hcy_part.alloc((size_t)std::max(1, nsd * std::max(1, (h->np_max + 255) / 256) * std::max(1, m_max)));
  h->upd.alloc((size_t)upd_total);
  h->ysave.alloc((size_t)ns);
  h->gv0.alloc((size_t)std::max<int64_t>(1, h->n_loc));
  h->gv2.alloc((size_t)std::max<int64_t>(1, h->n_loc));
  h->gl.alloc((size_t)(world * h->maxrows));
  h->gl.zero(s);
  h->cy.alloc((size_t)std::max<int64_t>(1, h->m_total));
  h->uvec.alloc((size_t)std::max<int64_t>(1, h->m_total));
  h->zc.alloc((size_t)std::max(1, nc));
  h->uvec_c.alloc((size_t)std::max(1, nc));
  h->gc.alloc((size_t)std::max(1, nc));
  CB_CUDA(cudaStreamSynchronize(s));
  h->bddc_ready = true;
}

// cy = H^T y' of every local constraint row (corner formulation)
void h_cy(cutbddc_gpu* h, const double* Yc, const int* skip, double* gl_fused = nullptr) {
  if (h->m_total == 0) return;
  if (h->m_max > kHcyMaxM) throw Failure(CUTBDDC_CONFIG, "coarse basis: more than 128 constraint rows in a subdomain");
  const int nch = std::max(1, (h->np_max + 255) / 256);
  h->hcy_part.alloc((size_t)h->nsd * nch * h->m_max);
  k_h_cy<<<dim3(h->nsd, nch), 256, 0, h->stream>>>(h->m_off.p, h->root_info.p, h->hroot.p, h->hslot.p, Yc,
                                                     h->hcy_part.p, h->m_max, skip);
  CB_LAUNCH();
  if (gl_fused) {  // also gl = S^{-1} cy (not the mixed K: no per-subdomain skip)
    k_h_cy_sum_sinv<<<h->nsd, 128, 0, h->stream>>>(nch, h->m_max, h->m_off.p, h->root_info.p, h->hcy_part.p, h->ac_off.p,
                                                   h->sinv.p, h->cy.p, gl_fused, skip);
    CB_LAUNCH();
    return;
  }
  k_h_cy_sum<<<grid_for(h->m_total, 128), 128, 0, h->stream>>>(h->m_total, nch, h->m_max, h->row_sd.p, h->m_off.p,
                                                              h->root_info.p, h->hcy_part.p, h->cy.p, skip,
                                                              h->k_mixed ? h->kform_shell.p : nullptr);
  CB_LAUNCH();
}

// z = M r (local dof vectors, dist.cuh), enqueued on the handle's stream.
// rz_part: when not null, every local subdomain's partial of r.z (PCG).
void apply_bddc_device(cutbddc_gpu* h, const double* r, double* z, const int* skip, double* rz_part) {
  cudaStream_t s = h->stream;
  const int64_t nl = h->n_loc, ns = (int64_t)h->nsd * h->slots;
  const int T = h->slots;
  ProfScope ps(h->prof, s, "apply vec 1 gather");
  k_gather_masked<<<grid_for(ns, 256), 256, 0, s>>>(ns, h->slot_loc.p, h->mask_int.p, r, h->sv0.p, skip);
  CB_LAUNCH();
  ps.close();
  solve_device(h, h->tI, h->fI, h->sv0.p, h->upd.p, h->ysave.p, skip);  // sv0 keeps z0 (interior slots)
  ps.next("apply vec 2 r1 scatter");
  // (Abar z0) on interface rows = Σ_w A_w,GI z0_w (z0 vanishes on the interface)
  sub_apply(h, kSubInterface, nullptr, h->sv0.p, h->sv2.p, skip);
  iface_exchange(h, h->sv2.p, nullptr, skip);
  k_scatter_r1<<<grid_for(ns, 256), 256, 0, s>>>(ns, h->slot_loc.p, h->mask_int.p, h->w.p, r, h->lcopy_ptr.p,
                                                 h->lcopy_src.p, h->sv2.p, h->recvbuf.p, h->sv1.p, skip);
  CB_LAUNCH();
  ps.close();
  if (h->has_K && h->m_total_g > 0) {  // uniform over ranks (collectives inside)
    // z~ = K^{-1}(r_w + C^T u), u = S^{-1}(zc - C K^{-1} r_w). Corner
    // formulation: the forward sweep (y' = L^{-1} r_w in ysave), cy = H^T y',
    // the coarse problem, y' += H u, the backward sweep. Shell formulation:
    // the forward sweep, the root's backward step, the coarse problem, the
    // root correction W_r u, then the backward sweep below the root (k_root_h).
    // Mixed K: the corner formulation's sweeps skip the shell subdomains and
    // the shell factor fKs holds only those; each subdomain takes one path.
    const bool corner = h->k_corner, mixed = h->k_mixed, shell = !corner || mixed;
    const FactorSet& fs = mixed ? h->fKs : h->fK;  // the shell-root factor
    if (corner) sweep_phase(h, h->tI, h->fK, h->sv1.p, h->ysave.p, h->upd.p, skip, kSweepFwd);
    if (shell) {
      sweep_phase(h, h->tK, fs, h->sv1.p, h->ysave.p, h->upd.p, skip, kSweepFwd);
      sweep_phase(h, h->tK, fs, h->sv1.p, h->ysave.p, h->upd.p, skip, kSweepBwdRoot);
    }
    ps.next("apply vec 3 cy coarse root-correction");
    const int cr_corner = corner ? (h->np_max + 255) / 256 : 0;
    const int cr_shell = shell ? (int)((h->tK.tpl.sn.back().ncols + 255) / 256) : 0;
    const int cr_blocks = std::max(1, std::max(cr_corner, cr_shell));
    double* gl_loc = h->gl.p + (int64_t)h->dist_rank * h->maxrows;  // this rank's rows of the staged gl
    if (!mixed && !h->coarse_sparse && h->n_coarse <= kCoarseInverseMax && h->m_max <= kFusedCoarseM) {
      double* Yc = corner ? h->ysave.p : h->sv1.p;  // where cy is read and the correction lands
      const int64_t* rinfo = corner ? h->root_info.p : h->root_info_s.p;
      if (corner) {  // cy = H^T y' (a warp per constraint row), gl = S^{-1} cy
        const char* env_unfused = std::getenv("CUTBDDC_HCY_UNFUSED");  // A/B and test hook: the separate launches
        if (env_unfused && env_unfused[0] == '1') {
          h_cy(h, Yc, skip);
          k_sinv_apply<<<grid_for(std::max<int64_t>(1, h->m_total), 128), 128, 0, s>>>(
              h->m_total, h->row_sd.p, h->m_off.p, h->ac_off.p, h->sinv.p, h->coarse_id.p, h->zc.p, h->cy.p, gl_loc, 0, skip);
        } else {
          h_cy(h, Yc, skip, gl_loc);
          g_kernel_launches.fetch_sub(1);  // the CB_LAUNCH below counts a launch h_cy has already counted
        }
      } else {
        k_coarse_in<<<h->nsd, 256, 0, s>>>(T, h->m_off.p, h->c_ptr.p, h->c_slot.p, h->c_val.p, Yc, h->ac_off.p,
                                           h->sinv.p, h->cy.p, gl_loc, skip, rinfo, nullptr, nullptr);
      }
      CB_LAUNCH();
      gather_rows(h);
      const size_t shm = sizeof(double) * ((size_t)h->n_coarse + 2 * kFusedCoarseM);
      if (shm > 48 * 1024)  // opt in once per device, to the largest size this kernel can ever need
        device_memo(kMemoCoarseOutShm, [] {
          CB_CUDA(cudaFuncSetAttribute(k_coarse_out, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)(sizeof(double) * (kCoarseInverseMax + 2 * kFusedCoarseM))));
          return 1ll;
        });
      k_coarse_out<<<dim3(h->nsd, cr_blocks), 256, shm, s>>>(
          h->n_coarse, h->cg_ptr.p, h->cg_idx.p, h->gl.p, h->acoarse_full.p, h->coarse_id.p, h->m_off.p, h->ac_off.p,
          h->sinv.p, h->cy.p, rinfo, fs.cslot.p, h->wroot.p, Yc, skip, corner ? h->hroot.p : nullptr, h->hslot.p);
      CB_LAUNCH();
    } else {
      if (corner) h_cy(h, h->ysave.p, skip);
      if (shell)
        k_cy<<<grid_for(std::max<int64_t>(1, h->m_total) * 32, 256), 256, 0, s>>>(
            h->m_total, T, h->row_sd.p, h->c_ptr.p, h->c_slot.p, h->c_val.p, h->sv1.p, h->cy.p, skip,
            mixed ? h->kform_corner.p : nullptr);
      CB_LAUNCH();
      k_sinv_apply<<<grid_for(std::max<int64_t>(1, h->m_total), 128), 128, 0, s>>>(h->m_total, h->row_sd.p, h->m_off.p, h->ac_off.p, h->sinv.p,
                                                             h->coarse_id.p, h->zc.p, h->cy.p, gl_loc, 0, skip);
      CB_LAUNCH();
      gather_rows(h);
      k_coarse_rhs<<<grid_for(h->n_coarse, 128), 128, 0, s>>>(h->n_coarse, h->cg_ptr.p, h->cg_idx.p, h->gl.p, h->gc.p, skip);
      CB_LAUNCH();
      if (h->coarse_sparse) {  // the nested-dissection factor's two level sweeps
        coarse_sparse_solve(h, h->gc.p, h->zc.p, skip);
      } else if (h->n_coarse <= kCoarseInverseMax) {
        k_coarse_gemv<<<grid_for((int64_t)h->n_coarse * 32, 256), 256, 0, s>>>(h->n_coarse, h->acoarse_full.p, h->gc.p,
                                                                             h->zc.p, skip);
        CB_LAUNCH();
      } else {  // zc = X^T (X gc), X = L_c^{-1}
        const int nc = h->n_coarse;
        k_xg_part<<<dim3((nc + 255) / 256, (nc + 63) / 64), 256, 0, s>>>(nc, h->acoarse_inv.p, h->gc.p, h->ws_cpart.p,
                                                                         skip);
        CB_LAUNCH();
        k_xg_sum<<<grid_for(nc, 256), 256, 0, s>>>(nc, h->ws_cpart.p, h->uvec_c.p, skip);
        CB_LAUNCH();
        k_xty<<<grid_for((int64_t)nc * 32, 256), 256, 0, s>>>(nc, h->acoarse_inv.p, h->uvec_c.p, h->zc.p, skip);
        CB_LAUNCH();
      }
      k_sinv_apply<<<grid_for(std::max<int64_t>(1, h->m_total), 128), 128, 0, s>>>(h->m_total, h->row_sd.p, h->m_off.p, h->ac_off.p, h->sinv.p,
                                                             h->coarse_id.p, h->zc.p, h->cy.p, h->uvec.p, 1, skip);
      CB_LAUNCH();
      if (corner) {  // shell subdomains of a mixed K have no H columns (np = 0)
        k_h_correct<<<dim3(h->nsd, std::max(1, cr_corner)), 256, 0, s>>>(h->m_off.p, h->root_info.p, h->hroot.p,
                                                                         h->hslot.p, h->uvec.p, h->ysave.p, skip);
        CB_LAUNCH();
      }
      if (shell) {  // corner subdomains of a mixed K have no root columns in fKs
        k_root_correct<<<dim3(h->nsd, std::max(1, cr_shell)), 256, 0, s>>>(h->root_info_s.p, h->m_off.p, fs.cslot.p,
                                                                          h->wroot.p, h->uvec.p, h->sv1.p, skip);
        CB_LAUNCH();
      }
    }
    ps.close();
    if (corner) sweep_phase(h, h->tI, h->fK, h->sv1.p, h->ysave.p, h->upd.p, skip, kSweepBwd);
    if (shell) sweep_phase(h, h->tK, fs, h->sv1.p, h->ysave.p, h->upd.p, skip, kSweepBwdRest);
    ps.next("apply vec 3b gather Av");
  } else {
    if (h->has_K) solve_k_device(h, h->sv1.p, skip);
    ps.next("apply vec 3b gather Av");
  }
  // v = Σ_copies w z~, every rank forms the same sum, also
  // scattered to the slots (sx) for the operator
  iface_exchange(h, h->sv1.p, h->w.p, skip);
  h->sx.alloc((size_t)ns);
  iface_sum(h, h->sv1.p, h->w.p, h->gv2.p, skip, h->sx.p);
  // harmonic correction: the interior rows of Abar v, one subdomain at a
  // time, and their interior solve (sv2; sv0 still holds z0)
  sub_apply(h, kSubInterior, nullptr, h->sx.p, h->sv2.p, skip);
  ps.close();
  solve_device(h, h->tI, h->fI, h->sv2.p, h->upd.p, h->ysave.p, skip);
  ps.next("apply vec 4 final");
  k_final_z<<<seg_grid(h), kSegThreads, 0, s>>>(seg_args(h, rz_part), h->lowner.p, h->sv0.p, h->gv2.p, h->sv2.p, z,
                                                rz_part ? r : nullptr, skip);
  CB_LAUNCH();
}

}  // namespace cutbddc_b200
