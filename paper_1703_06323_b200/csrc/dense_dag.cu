// dense_dag.cu — the numeric multifrontal factorisation of every subdomain
// as ONE persistent, dataflow-scheduled launch (every front of every level:
// no level barriers, no per-level launches), plus the dense coarse matrix.
//
// Replaces the numeric part of SparseCholesky::compute (linalg.cpp:34-62) for
// A_II and K = A + rho C^T C, batched over subdomains. A front F (r x r,
// column-major, lower part) is cut into tiles of at most 64 x 64 whose
// boundaries are 0, 64, ..., c (the pivot columns) and c, c + 64, ..., r (the
// update rows/columns). Tasks:
//   ASM(i,j)      F_ij assembled in gather form (front_asm.cuh): children's
//                 update blocks + the original stencil entries
//   PEN(row)      F += rho c c^T of one constraint row (root of K)
//   POTRF(k)      F_kk = L_kk L_kk^T and P_kk = L_kk^{-1}          (k < np)
//   TRSM(i,k)     F_ik = F_ik P_kk^T = L_ik                          (i > k)
//   GEMM(i,j,k)   F_ij -= L_ik L_jk^T                     (i >= j > k)
//   ACC(i,j,k)    P_ij (+)= L_ik P_kj                 (j <= k < min(i, np))
//   FIN(i,j)      P_ij = -P_ii P_ij                         (j < i < np)
//   W             a small front whole, by one CTA: assembly, then the tile
//                 tasks above in list order
// "Split" fronts (factor.cu: is_split_front) get the tile tasks, spread over
// many CTAs; the others one W task. P is the explicit panel
// G = [L11^{-1}; L21 L11^{-1}] the solve sweeps use: the first c columns of
// M^{-1}, M = [L11 0; L21 I], with the lower block negated (G21 = +sum L21 X).
// The trailing tiles (j >= np) end as the update matrix the parent gathers.
// A front's ASM / W tasks wait for its children's done counters. The GEMM
// tiles run on the FP64 tensor cores (DMMA). Every tile is updated in a fixed
// order (per-tile counters), so the result is deterministic. The ticket order
// is topological (build_tasks): no deadlock.
#include <algorithm>
#include <chrono>
#include <map>
#include <memory>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include <cub/cub.cuh>

#include "factor.cuh"
#include "front_asm.cuh"

namespace cutbddc_b200 {
namespace {

constexpr int kTile = 64;
constexpr int kDagThreads = 256;
constexpr int kFinal = 1 << 20;  // X tile completed
enum { kPotrf = 0, kTrsm = 1, kGemm = 2, kAcc = 3, kFin = 4, kAsm = 5, kPen = 6, kWhole = 7, kDiag = 8 };

struct DagFront {
  long long fo, po, cnt;  // front (in the chunk's workspace), panel, counter offsets
  int r, c, np, nt;       // rows, pivot columns, pivot / all tile blocks
  int sd, sid;            // subdomain, supernode (-1: a plain dense matrix)
  int ch0, ch1;           // child fronts (list indices, -1: none)
  int ntask, nasm;        // tasks of the front (its done counter's final value); assembly tasks
  int ntile, whole;       // ASM tile tasks (PEN rows wait for them); 1: one W task runs the whole front
  int grp, pad_;          // factorisation (DagArgs::g) the front belongs to
};

// One factorisation of a launch (the interior problems and K share one).
struct DagGroup {
  TplDev t;
  FactorDev f;
  FactorInput in;
  double* panel;
  unsigned long long* fail;
  int* fail_sd;  // optional: per subdomain, set when one of its pivots is non-positive
};

constexpr int kMaxGroups = 2;

struct DagArgs {
  const DagFront* fronts;
  const int4* tasks;
  int n_tasks;
  double* front;  // every group's fronts (DagFront::fo)
  int* counters;
  int* ticket;
  DagGroup g[kMaxGroups];
  unsigned long long* trace;  // CUTBDDC_DAG_TRACE: per task {grab, deps met, done, sm}
};

__device__ __forceinline__ unsigned long long dag_timer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ int tri(int i, int j) { return i * (i + 1) / 2 + j; }

__device__ __forceinline__ int bnd(const DagFront& d, int b) {
  return b < d.np ? b * kTile : (b == d.np ? d.c : min(d.r, d.c + (b - d.np) * kTile));
}

__device__ __forceinline__ int ld_acq(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void wait_eq(const int* p, int v) {
  while (ld_acq(p) < v) __nanosleep(40);
}

// C (m x n, ldc) = (acc ? C : 0) + alpha * A (m x kk, lda) * op(B);
// op(B) = B^T with B n x kk (bt) or B kk x n. 256 threads, 4x4 register
// blocks, k staged in shared memory 32 at a time. A or B may alias C (they are
// read completely before C is written). lower: store only rows >= columns.
// D = A B + C on the FP64 tensor cores (DMMA), m8n8k4: lane l holds
// A[l/4][l%4], B[l%4][l/4] and D[l/4][2(l%4) .. 2(l%4)+1].
__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// 8-byte cp.async (LDGSTS) global -> shared; src-size 0 zero-fills
__device__ __forceinline__ void cp_async8(double* dst, const double* src, bool valid) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d), "l"(src), "r"(valid ? 8 : 0) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// The dense trailing updates on the DMMA tensor cores: 8 warps, each owns a
// 16 x 32 block of the 64 x 64 output (2 x 4 mma tiles). The whole 64-deep A
// and B tiles go to shared memory by cp.async (every load in flight at once,
// no register staging; rows padded to 65 doubles: conflict-free fragment
// loads) while the accumulators are loaded from C (acc: C never aliases A or
// B then); alpha = -1 negates the A fragments, so D = C + alpha A op(B).
__device__ void tile_mm(double* C, int ldc, const double* A, int lda, const double* B, int ldb, int m, int n, int kk,
                        double alpha, bool acc, bool bt, bool lower, double* sm) {
  double(*as)[kTile + 1] = reinterpret_cast<double(*)[kTile + 1]>(sm);
  double(*bs)[kTile + 1] = reinterpret_cast<double(*)[kTile + 1]>(sm + kTile * (kTile + 1));
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int wr = (wid & 3) * 16, wc = (wid >> 2) * 32;  // warp's output block origin
  const int fr = lane >> 2, fk = lane & 3;               // fragment row/col and k index
  const double sa = alpha < 0.0 ? -1.0 : 1.0;           // alpha is +-1 at every call site
  // kk <= kTile: every tile of a front is at most 64 x 64
  __syncthreads();  // previous users of the staging buffers are done
  for (int e = tid; e < kTile * kTile; e += kDagThreads) {
    const int row = e & 63, k = e >> 6;
    const bool v = row < m && k < kk;
    cp_async8(&as[k][row], A + (v ? row + (int64_t)k * lda : 0), v);
  }
  for (int e = tid; e < kTile * kTile; e += kDagThreads) {
    const int lo = e & 63, hi = e >> 6;  // bt: (col, k); else (k, col): coalesced either way
    const int col = bt ? lo : hi, k = bt ? hi : lo;
    const bool v = col < n && k < kk;
    cp_async8(&bs[k][col], B + (v ? (bt ? col + (int64_t)k * ldb : k + (int64_t)col * ldb) : 0), v);
  }
  double d[2][4][2];  // accumulators from C while the tiles are in flight
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int h2 = 0; h2 < 2; ++h2) {
        const int i = wr + 8 * a + fr, j = wc + 8 * b + 2 * fk + h2;
        d[a][b][h2] = (acc && i < m && j < n) ? C[i + (int64_t)j * ldc] : 0.0;
      }
  cp_async_wait_all();
  __syncthreads();
  for (int k = 0; k < kk; k += 4) {
    double fa[2], fb[4];
#pragma unroll
    for (int a = 0; a < 2; ++a) fa[a] = sa * as[k + fk][wr + 8 * a + fr];
#pragma unroll
    for (int b = 0; b < 4; ++b) fb[b] = bs[k + fk][wc + 8 * b + fr];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) dmma_8x8x4(d[a][b][0], d[a][b][1], fa[a], fb[b]);
  }
  __syncthreads();  // A / B (possibly C itself) fully consumed
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int h2 = 0; h2 < 2; ++h2) {
        const int i = wr + 8 * a + fr, j = wc + 8 * b + 2 * fk + h2;
        if (i >= m || j >= n || (lower && i < j)) continue;
        C[i + (int64_t)j * ldc] = d[a][b][h2];
      }
}

// D += sa * A B on one 8 x 8 block (DMMA m8n8k4, K a multiple of 4): lane l
// holds D[l/4][2(l%4) .. 2(l%4)+1]; A[i][k] = pa[i*sia + k*ska], B[k][n] =
// pb[k*skb + n*snb] (shared memory).
__device__ __forceinline__ void mma_block8(double& d0, double& d1, const double* pa, int sia, int ska,
                                           const double* pb, int skb, int snb, int K, double sa) {
  const int lane = threadIdx.x & 31, r = lane >> 2, c = lane & 3;
  const double* a = pa + r * sia + c * ska;
  const double* b = pb + c * skb + r * snb;
  for (int k = 0; k < K; k += 4) dmma_8x8x4(d0, d1, sa * a[k * ska], b[k * skb]);
}

// Cholesky of the n x n diagonal tile and the inverse of its factor,
// blocked by kPb = 16 columns. Per panel p (columns c0 = 16p ..):
//   (a) warp 0: the 16 x 16 diagonal block in shared memory, L_pp (lane =
//       row half) and X_pp = L_pp^{-1} (lane = column half, right-looking),
//       rolled pivot loops with load-first bodies and selects instead of
//       branches; meanwhile warps 1-7 form T = L_p,<p X_<p,<p (block row p
//       of the inverse, before X_pp)
//   (b) L_ip = A_ip X_pp^T for the rows below and X_pj = -X_pp T_pj (j < p)
//   (c) A_iq -= L_ip L_qp^T on the trailing lower triangle
// (b), (c) and T are 8 x 8 DMMA blocks from shared memory. Four barriers per
// panel instead of one per pivot (a dependent DFMA costs ~23 cycles, a shared
// load -> DFMA -> store ~53 on B200: tools/bench_src/lat_probe.cu). In the
// cfg4 task trace (CUTBDDC_DAG_TRACE) a POTRF task takes 37 us against 45 us
// for the unblocked one-barrier-per-pivot form; tools/bench_src/potrf_bench.cu
// shows warp 0's 32 pivot steps still at ~1k cycles each, the open item. Rows / columns >= n are padded with
// the identity and never written back. Non-positive pivots are reported
// (fail) and replaced by 1. Strict upper parts stored as zero.
typedef double SmTile[kTile + 1];
constexpr int kPb = 16;
#ifndef POTRF_STAMP  // phase timestamps for tools/bench_src/potrf_bench.cu
#define POTRF_STAMP(k)
#endif
template <typename Fail>
__device__ void tile_potrf_inv(double* F, int ldf, double* P, int ldp, int n, double* sm, Fail fail) {
  SmTile* ls = reinterpret_cast<SmTile*>(sm);
  SmTile* xs = reinterpret_cast<SmTile*>(sm + kTile * (kTile + 1));
  constexpr int ld = kTile + 1;
  __shared__ double rinv[kPb];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int fr = lane >> 2, fc = lane & 3;  // DMMA fragment row / column pair
  const int npan = (n + kPb - 1) / kPb, N = npan * kPb;  // padded size
  __syncthreads();
  {
    constexpr int kPer = kTile * kTile / kDagThreads;  // loads in flight per thread
    double v[kPer];
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const int e = tid + u * kDagThreads, i = e & 63, j = e >> 6;
      v[u] = (i < n && j < n && i >= j) ? F[i + (int64_t)j * ldf] : (i == j ? 1.0 : 0.0);
    }
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const int e = tid + u * kDagThreads, i = e & 63, j = e >> 6;
      ls[i][j] = v[u];
    }
  }
  POTRF_STAMP(0);
  for (int p = 0; p < npan; ++p) {
    const int c0 = p * kPb;
    __syncthreads();  // the previous panel's trailing update is complete
    POTRF_STAMP(1 + 3 * p);
    if (wid == 0) {
      // (a) L_pp in shared memory: lane (i, h) updates row c0 + i, columns
      // 8h .. 8h + 7. Rolled pivot loop with a short, load-first body: this
      // code runs once per tile, so straight-line unrolled code is bound by
      // cold instruction fetch (~34 cycles per instruction measured).
      const int li = lane & (kPb - 1), h = lane >> 4;
      double* bl = &ls[c0][c0];
      unsigned bad = 0;  // non-positive pivots of the block (the first is reported)
#pragma unroll 1
      for (int j = 0; j < kPb; ++j) {
        double d = bl[j * ld + j];
        const double aij = bl[li * ld + j];
        double lq[8], aq[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          lq[k] = bl[(8 * h + k) * ld + j];
          aq[k] = bl[li * ld + 8 * h + k];
        }
        const bool ok = d > 0.0;
        bad |= ok ? 0u : 1u << j;
        d = ok ? d : 1.0;
        const double r = rsqrt(d);
        const double lij = aij * r;
        __syncwarp();  // column j read by every lane
        // every lane computes every candidate and stores a selected value:
        // per-lane branches around FP64 ops compile to BSSY/BSYNC pairs that
        // cost ~100 cycles each (measured); every entry has one owner lane
        const double dr = d * r;
        const double colj = li > j ? lij : (li == j ? dr : aij);
        rinv[j] = r;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int q = 8 * h + k;
          const double upd = fma(-lij, lq[k] * r, aq[k]);  // computed by every lane: no branches
          double v = aq[k];
          v = (q > j && li >= q) ? upd : v;
          v = q == j ? colj : v;
          bl[li * ld + q] = v;
        }
        __syncwarp();
      }
      if (bad && lane == 0) fail(c0 + __ffs(bad) - 1);
      // X_pp = L_pp^{-1} in place in xs: lane (c, h) owns column c, rows
      // 8h .. 8h + 7; right-looking (x_k final, then every row below updated)
      double* xb = &xs[c0][c0];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int row = 8 * h + k;
        xb[row * ld + li] = row == li ? 1.0 : 0.0;
        bl[row * ld + li] = row < li ? 0.0 : bl[row * ld + li];  // strict upper part of L_pp
      }
      __syncwarp();
#pragma unroll 1
      for (int k = 0; k < kPb; ++k) {
        const double xk = xb[k * ld + li] * rinv[k];
        double lk[8], tk[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          lk[i] = bl[(8 * h + i) * ld + k];
          tk[i] = xb[(8 * h + i) * ld + li];
        }
        __syncwarp();
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int row = 8 * h + i;
          const double upd = fma(-lk[i], xk, tk[i]);
          double v = row > k ? upd : tk[i];
          v = row == k ? xk : v;
          xb[row * ld + li] = v;
        }
        __syncwarp();
      }
    } else if (p > 0) {
      // T_pj = L_p,s X_s,j over s from the 16-block holding column j to c0
      // (X is lower triangular), 8 x 8 blocks into X_pj's place
      const int nt = 2 * (c0 / 8);
      for (int blk = wid - 1; blk < nt; blk += kDagThreads / 32 - 1) {
        const int m0 = 8 * (blk & 1), col0 = 8 * (blk >> 1), s0 = kPb * (col0 / kPb);
        double d0 = 0.0, d1 = 0.0;
        mma_block8(d0, d1, &ls[c0 + m0][s0], ld, 1, &xs[s0][col0], ld, 1, c0 - s0, 1.0);
        xs[c0 + m0 + fr][col0 + 2 * fc] = d0;
        xs[c0 + m0 + fr][col0 + 2 * fc + 1] = d1;
      }
    }
    __syncthreads();
    POTRF_STAMP(2 + 3 * p);
    // (b) L_ip = A_ip X_pp^T (rows below the block) and X_pj = -X_pp T_pj,
    // computed into registers, stored after a barrier (A_ip and T are
    // overwritten in place)
    const int nbr = (N - c0 - kPb) / 8;  // 8-row blocks below the diagonal block
    const int nl = 2 * nbr, nx = 2 * (c0 / 8);
    double o[2][2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int blk = wid + 8 * u;
      o[u][0] = o[u][1] = 0.0;
      if (blk < nl) {
        const int i0 = c0 + kPb + 8 * (blk >> 1), j0 = 8 * (blk & 1);
        mma_block8(o[u][0], o[u][1], &ls[i0][c0], ld, 1, &xs[c0 + j0][c0], 1, ld, kPb, 1.0);
      } else if (blk < nl + nx) {
        const int b2 = blk - nl, m0 = 8 * (b2 & 1), col0 = 8 * (b2 >> 1);
        mma_block8(o[u][0], o[u][1], &xs[c0 + m0][c0], ld, 1, &xs[c0][col0], ld, 1, kPb, -1.0);
      }
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int blk = wid + 8 * u;
      if (blk < nl) {
        const int i0 = c0 + kPb + 8 * (blk >> 1), j0 = c0 + 8 * (blk & 1);
        ls[i0 + fr][j0 + 2 * fc] = o[u][0];
        ls[i0 + fr][j0 + 2 * fc + 1] = o[u][1];
      } else if (blk < nl + nx) {
        const int b2 = blk - nl, m0 = c0 + 8 * (b2 & 1), col0 = 8 * (b2 >> 1);
        xs[m0 + fr][col0 + 2 * fc] = o[u][0];
        xs[m0 + fr][col0 + 2 * fc + 1] = o[u][1];
      }
    }
    if (nbr == 0) continue;
    __syncthreads();
    POTRF_STAMP(3 + 3 * p);
    // (c) trailing lower triangle, 8 x 8 blocks (ib >= qb) of rows / columns >= c0 + 16
    const int ntr = nbr * (nbr + 1) / 2;
    for (int blk = wid; blk < ntr; blk += kDagThreads / 32) {
      int ib = 0;
      while ((ib + 1) * (ib + 2) / 2 <= blk) ++ib;
      const int qb = blk - ib * (ib + 1) / 2;
      const int i0 = c0 + kPb + 8 * ib, q0 = c0 + kPb + 8 * qb;
      double d0 = ls[i0 + fr][q0 + 2 * fc], d1 = ls[i0 + fr][q0 + 2 * fc + 1];
      mma_block8(d0, d1, &ls[i0][c0], ld, 1, &ls[q0][c0], 1, ld, kPb, -1.0);
      if (ib != qb || fr >= 2 * fc) ls[i0 + fr][q0 + 2 * fc] = d0;
      if (ib != qb || fr >= 2 * fc + 1) ls[i0 + fr][q0 + 2 * fc + 1] = d1;
    }
  }
  __syncthreads();
  POTRF_STAMP(15);
  for (int c = wid; c < n; c += kDagThreads / 32)
    for (int r = lane; r < n; r += 32) {
      F[r + (int64_t)c * ldf] = r >= c ? ls[r][c] : 0.0;
      P[r + (int64_t)c * ldp] = r >= c ? xs[r][c] : 0.0;
    }
}

// One tile task of front d (POTRF / TRSM / GEMM / ACC / FIN), no waits.
__device__ void tile_task(const DagArgs& a, const DagFront& d, int kind, int i, int j, int k, double* sm) {
  double* F = a.front + d.fo;
  const DagGroup& G = a.g[d.grp];
  double* P = G.panel + d.po;
  const int r = d.r;
  auto tile = [&](double* base, int ti, int tj) { return base + bnd(d, ti) + (int64_t)bnd(d, tj) * r; };
  auto ext = [&](int b) { return bnd(d, b + 1) - bnd(d, b); };
  if (kind == kPotrf) {
    const int col0 = bnd(d, k);
    tile_potrf_inv(tile(F, k, k), r, tile(P, k, k), r, ext(k), sm, [&](int jj) {
      if (d.sid < 0) {  // plain dense matrix: the pivot index
        atomicMin(G.fail, (unsigned long long)(col0 + jj));
        return;
      }
      // report the template slot of compact column col0 + jj (pivot rule, linalg.cpp:42-54)
      const Supernode s = G.t.sn[d.sid];
      const int q = G.f.tpos[(int64_t)d.sd * G.t.rows_total + s.rows_off + col0 + jj];
      atomicMin(G.fail, (unsigned long long)((int64_t)d.sd * G.t.T + G.t.rows[s.rows_off + q]));
      if (G.fail_sd) G.fail_sd[d.sd] = 1;
    });
    // (the panel above this diagonal tile is never read: the sweeps start
    // every column at the 32-row block holding its diagonal)
  } else if (kind == kTrsm) {
    tile_mm(tile(F, i, k), r, tile(F, i, k), r, tile(P, k, k), r, ext(i), ext(k), ext(k), 1.0, false, true, false, sm);
  } else if (kind == kGemm) {
    tile_mm(tile(F, i, j), r, tile(F, i, k), r, tile(F, j, k), r, ext(i), ext(j), ext(k), -1.0, true, true, i == j, sm);
  } else if (kind == kAcc) {
    tile_mm(tile(P, i, j), r, tile(F, i, k), r, tile(P, k, j), r, ext(i), ext(j), ext(k), 1.0, k != j, false, false, sm);
  } else {  // kFin
    tile_mm(tile(P, i, j), r, tile(P, i, i), r, tile(P, i, j), r, ext(i), ext(j), ext(i), -1.0, false, false, false, sm);
  }
}

__device__ ChildBlocks child_blocks(const DagArgs& a, const DagFront& d) {
  ChildBlocks cb{nullptr, nullptr, 1, 1};
  if (d.ch0 >= 0) {
    const DagFront& c = a.fronts[d.ch0];
    cb.u0 = a.front + c.fo + c.c + (int64_t)c.c * c.r;
    cb.ld0 = c.r;
  }
  if (d.ch1 >= 0) {
    const DagFront& c = a.fronts[d.ch1];
    cb.u1 = a.front + c.fo + c.c + (int64_t)c.c * c.r;
    cb.ld1 = c.r;
  }
  return cb;
}

__device__ __forceinline__ void wait_children(const DagArgs& a, const DagFront& d) {
  if (d.ch0 >= 0) wait_eq(a.counters + a.fronts[d.ch0].cnt, a.fronts[d.ch0].ntask);
  if (d.ch1 >= 0) wait_eq(a.counters + a.fronts[d.ch1].cnt, a.fronts[d.ch1].ntask);
}

// rho c c^T of constraint row `row` on the root front (a corner row is a
// diagonal shift, already in diag_add): entries staged as (compact row,
// value); objects are disjoint, so rows touch distinct entries.
__device__ void penalty_row(const DagArgs& a, const DagFront& d, int64_t row, double* sm) {
  const DagGroup& G = a.g[d.grp];
  const FactorInput& in = G.in;
  if (in.corner[row]) return;
  const int sd = d.sd, r = d.r;
  const Supernode s = G.t.sn[d.sid];
  double* F = a.front + d.fo;
  const double rho = in.rho[sd];
  const int64_t p0 = in.c_ptr[row];
  const int len = (int)(in.c_ptr[row + 1] - p0);
  auto pos = [&](int x) { return G.f.pfx[(int64_t)sd * G.t.rows_total + s.rows_off + G.t.root_pos[in.c_slot[p0 + x]]]; };
  constexpr int kStage = 1024;
  __syncthreads();
  if (len > kStage) {  // very large object: unstaged
    for (int q = threadIdx.x; q < len * len; q += blockDim.x) {
      const int x = q / len, y = q % len;
      const int pa = pos(x), pb = pos(y);
      if (pa < pb || pb < 0) continue;
      F[pa + (int64_t)pb * r] += rho * in.c_val[p0 + x] * in.c_val[p0 + y];
    }
    __syncthreads();
    return;
  }
  double* sv = sm;
  double* sc = sm + kStage;
  int* sp = reinterpret_cast<int*>(sm + 2 * kStage);
  for (int x = threadIdx.x; x < len; x += blockDim.x) {
    sp[x] = pos(x);
    sc[x] = in.c_val[p0 + x];
    sv[x] = rho * sc[x];
  }
  __syncthreads();
  const int n = len * len;
  constexpr int kB = 4;  // entries per thread per pass: loads before stores
  for (int q0 = threadIdx.x; q0 < n; q0 += kB * blockDim.x) {
    double v[kB];
    int64_t at[kB];
#pragma unroll
    for (int u = 0; u < kB; ++u) {
      const int q = q0 + u * blockDim.x, x = q / len, y = q - x * len;
      const int pa = q < n ? sp[x] : -1, pb = q < n ? sp[y] : -1;
      at[u] = (pa >= pb && pb >= 0) ? pa + (int64_t)pb * r : -1;
      v[u] = at[u] >= 0 ? F[at[u]] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < kB; ++u) {
      const int q = q0 + u * blockDim.x, x = q / len, y = q - x * len;
      if (at[u] >= 0) F[at[u]] = v[u] + sv[x] * sc[y];
    }
  }
  __syncthreads();
}

// Assembly of rows [i0, i1) x cols [j0, j1) of front d (gather form).
__device__ void assemble(const DagArgs& a, const DagFront& d, int i0, int i1, int j0, int j1, double* sm) {
  const DagGroup& G = a.g[d.grp];
  const FrontDesc& fd = G.f.desc[(int64_t)d.sd * G.t.nsn + d.sid];
  RowInfo* ri = reinterpret_cast<RowInfo*>(sm);
  RowInfo* rj = ri + (i1 - i0);
  const bool same = i0 == j0 && i1 == j1;
  __syncthreads();
  for (int q = threadIdx.x; q < i1 - i0; q += blockDim.x) ri[q] = row_info(G.f, fd, d.sd, G.in.T, G.in.b1, i0 + q);
  if (!same)
    for (int q = threadIdx.x; q < j1 - j0; q += blockDim.x) rj[q] = row_info(G.f, fd, d.sd, G.in.T, G.in.b1, j0 + q);
  __syncthreads();
  assemble_block(a.front + d.fo, d.r, d.c, i0, i1, j0, j1, ri, same ? ri : rj, child_blocks(a, d), G.in, d.sd);
  __syncthreads();
}

// W task: the whole front by one CTA (assembly, root penalty, then every tile
// task in list order).
__device__ void whole_front(const DagArgs& a, const DagFront& d, double* sm) {
  assemble(a, d, 0, d.r, 0, d.r, sm);
  const DagGroup& G = a.g[d.grp];
  if (d.sid == G.t.root && G.in.c_ptr)
    for (int64_t row = G.in.m_off[d.sd]; row < G.in.m_off[d.sd + 1]; ++row) penalty_row(a, d, row, sm);
  const int np = d.np, nt = d.nt;
  for (int k = 0; k < np; ++k) {
    tile_task(a, d, kPotrf, k, k, k, sm);
    for (int i = k + 1; i < nt; ++i) tile_task(a, d, kTrsm, i, k, k, sm);
    for (int jj = k + 1; jj < nt; ++jj)
      for (int i = jj; i < nt; ++i) tile_task(a, d, kGemm, i, jj, k, sm);
    for (int jj = 0; jj < k; ++jj) tile_task(a, d, kFin, k, jj, k, sm);
    for (int jj = 0; jj <= k; ++jj)
      for (int i = k + 1; i < nt; ++i) tile_task(a, d, kAcc, i, jj, k, sm);
  }
}

__global__ void __launch_bounds__(kDagThreads, 3) k_dense_dag(DagArgs a) {
  extern __shared__ double sm[];
  __shared__ int s_task;
  __shared__ unsigned long long s_t0, s_t1;
  const int tid = threadIdx.x;
  for (;;) {
    __syncthreads();
    if (tid == 0) s_task = atomicAdd(a.ticket, 1);
    __syncthreads();
    const int it = s_task;
    if (a.trace && tid == 0) s_t0 = dag_timer();
    if (it >= a.n_tasks) return;
    const int4 tk = a.tasks[it];
    const int kind = tk.x >> 24, fi = tk.x & 0xffffff, i = tk.y, j = tk.z, k = tk.w;
    const DagFront d = a.fronts[fi];
    int* fdone = a.counters + d.cnt;        // tasks of this front completed
    int* fasm = fdone + 1;                  // assembly tasks completed
    int* A = fdone + 2;                     // factor tiles: updates applied, col + 1 when final
    int* X = A + d.nt * (d.nt + 1) / 2;     // panel tiles: accumulations applied, kFinal when final
    int* done = nullptr;
    int inc = 1;
    if (tid == 0) {  // dependencies
      if (kind == kWhole || kind == kAsm) {
        wait_children(a, d);
      } else if (kind == kPen) {
        wait_eq(fasm, d.ntile);
      } else {
        if (k == 0) wait_eq(fasm, d.nasm);
        if (kind == kPotrf) {
          wait_eq(A + tri(k, k), k);
        } else if (kind == kTrsm) {
          wait_eq(A + tri(k, k), k + 1);
          wait_eq(A + tri(i, k), k);
        } else if (kind == kDiag) {  // i = k + 1
          wait_eq(A + tri(k, k), k + 1);
          wait_eq(A + tri(i, k), k);
          wait_eq(A + tri(i, i), k);
        } else if (kind == kGemm) {
          wait_eq(A + tri(i, k), k + 1);
          wait_eq(A + tri(j, k), k + 1);
          wait_eq(A + tri(i, j), k);
        } else if (kind == kAcc) {
          wait_eq(A + tri(i, k), k + 1);
          if (k == j)
            wait_eq(A + tri(j, j), j + 1);
          else
            wait_eq(X + tri(k, j), kFinal);
          wait_eq(X + tri(i, j), k - j);
        } else {  // kFin
          wait_eq(X + tri(i, j), i - j);
          wait_eq(A + tri(i, i), i + 1);
        }
      }
      if (a.trace) s_t1 = dag_timer();
    }
    __syncthreads();
    __threadfence();
    if (kind == kWhole) {
      whole_front(a, d, sm);
    } else if (kind == kAsm) {
      assemble(a, d, bnd(d, i), bnd(d, i + 1), bnd(d, j), bnd(d, j + 1), sm);
      done = fasm;
    } else if (kind == kPen) {
      penalty_row(a, d, (int64_t)i, sm);
      done = fasm;
    } else if (kind == kDiag) {
      // the critical path of step k in one CTA: L_ik (TRSM, published at
      // once for the other tasks of step k), the diagonal tile's last update
      // F_ii -= L_ik L_ik^T, then POTRF(i)
      tile_task(a, d, kTrsm, i, k, k, sm);
      __syncthreads();
      if (tid == 0) {
        __threadfence();
        atomicAdd(A + tri(i, k), 1);
      }
      tile_task(a, d, kGemm, i, i, k, sm);
      tile_task(a, d, kPotrf, i, i, i, sm);
      done = A + tri(i, i);
      inc = 2;
    } else {
      tile_task(a, d, kind, i, j, k, sm);
      if (kind == kPotrf || kind == kTrsm || kind == kGemm) {
        done = A + tri(i, j);
      } else {
        done = X + tri(i, j);
        if (kind == kFin) inc = kFinal - (i - j);  // P_ij final
      }
    }
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      if (done) atomicAdd(done, inc);
      atomicAdd(fdone, 1);
      if (a.trace) {
        unsigned long long* tr = a.trace + 4ll * it;
        unsigned sm_id;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(sm_id));
        tr[0] = s_t0;
        tr[1] = s_t1;
        tr[2] = dag_timer();
        tr[3] = sm_id;
      }
    }
  }
}

// Host list entry of one front: the device record plus what the task list needs.
struct HostFront {
  DagFront d;
  int parent;          // list index of the parent front, -1: none
  int64_t pen0, pen1;  // constraint rows added by PEN tasks (split root of K)
};

// Task list in decreasing "bottom level" (weighted length of the longest path
// from the task to the end of the whole tree's DAG): the POTRF chains and the
// tasks feeding them first, wide trailing updates later. Every predecessor of
// a task has a strictly larger bottom level (inside a front by construction;
// across fronts every task of a child lies above its parent's first tasks),
// so the order is topological: every wait is on a smaller ticket, held by a
// running CTA, and the persistent launch cannot deadlock.
// A split front's tile tasks and their bottom levels (relative to the front's
// parent entry) depend only on its tile counts (np, nt): computed once per
// shape and reused by every front of that shape.
struct SplitShape {
  std::vector<int4> ft;  // (kind << 24, i, j, k); the front id is or-ed in per front
  std::vector<int> bl;
  int top = 0;           // bottom level of the first POTRF (bl_p[0])
  int maxbl = 0;         // largest entry of bl
  int dev = -1;          // index in the device template table (dense_dag_factor)
};

int g_shape_builds = 0;  // CUTBDDC_DAG_STATS: split shapes built by the last task list
std::chrono::steady_clock::time_point g_bt_sort_t0;  // start of its sort (stats)

// The tile tasks of a split front with np pivot / nt tile blocks and their
// bottom levels relative to the front's parent entry: a pure function of
// (np, nt), kept across calls (per host thread: batched handles run on
// several).
SplitShape& split_shape(int np, int nt) {
  constexpr int kShapeDim = 64;
  thread_local std::vector<std::unique_ptr<SplitShape>> shape_tab((size_t)kShapeDim * kShapeDim);
  thread_local std::map<std::pair<int, int>, SplitShape> shapes;  // (larger fronts)
  SplitShape* shp;
  if (np < kShapeDim && nt < kShapeDim) {
    std::unique_ptr<SplitShape>& u = shape_tab[(size_t)np * kShapeDim + nt];
    if (!u) u = std::make_unique<SplitShape>();
    shp = u.get();
  } else {
    shp = &shapes[std::make_pair(np, nt)];
  }
  SplitShape& sh = *shp;
  if (!sh.ft.empty() || np == 0) return sh;
  ++g_shape_builds;
  std::vector<int4> ft;
  std::vector<int> bl, bl_p, bl_t, bl_g, bl_a, bl_f;
  auto push = [&](int kind, int i, int j, int kk, int b) {
    ft.push_back(make_int4(kind << 24, i, j, kk));
    bl.push_back(b);
  };
      for (int k = 0; k < np; ++k) {  // per front, step by step (successors later)
        push(kPotrf, k, k, k, 0);
        for (int i = k + 1; i < nt; ++i) push(kTrsm, i, k, k, 0);
        for (int jj = k + 1; jj < nt; ++jj)
          for (int i = jj; i < nt; ++i) push(kGemm, i, jj, k, 0);
        for (int jj = 0; jj < k; ++jj) push(kFin, k, jj, k, 0);
        for (int jj = 0; jj <= k; ++jj)
          for (int i = k + 1; i < nt; ++i) push(kAcc, i, jj, k, 0);
      }
      const size_t n2 = (size_t)nt * nt, n3 = n2 * nt;
      bl_p.assign((size_t)nt, 0);
      bl_t.assign(n2, 0);
      bl_f.assign(n2, 0);
      bl_g.assign(n3, 0);
      bl_a.assign(n3, 0);
      auto T = [&](int i, int k) -> int& { return bl_t[(size_t)i * nt + k]; };
      auto Fn = [&](int i, int j) -> int& { return bl_f[(size_t)i * nt + j]; };
      auto G = [&](int i, int j, int k) -> int& { return bl_g[((size_t)i * nt + j) * nt + k]; };
      auto Ac = [&](int i, int j, int k) -> int& { return bl_a[((size_t)i * nt + j) * nt + k]; };
      for (size_t x = ft.size(); x-- > 0;) {
        const int kind = ft[x].x >> 24, i = ft[x].y, j = ft[x].z, k = ft[x].w;
        int s = 0;
        if (kind == kPotrf) {
          for (int y = k + 1; y < nt; ++y) s = std::max({s, T(y, k), Ac(y, k, k)});
          for (int y = 0; y < k; ++y) s = std::max(s, Fn(k, y));
          bl[x] = bl_p[(size_t)k] = 3 + s;  // the diagonal tile weighs ~3 tile updates
        } else if (kind == kTrsm) {
          for (int y = k + 1; y <= i; ++y) s = std::max(s, G(i, y, k));
          for (int y = i; y < nt; ++y) s = std::max(s, G(y, i, k));
          for (int y = 0; y <= k; ++y) s = std::max(s, Ac(i, y, k));
          bl[x] = T(i, k) = 1 + s;
          // DIAG(i) = TRSM(i,k) + GEMM(i,i,k) + POTRF(i) (i = k + 1 < np): the
          // earlier updates of tile (i,i) precede the whole merged task
          if (i == k + 1 && i < np) G(i, i, k) = T(i, k);
        } else if (kind == kGemm) {
          if (k + 1 < j && k + 1 < np)
            s = G(i, j, k + 1);
          else if (j < np)
            s = i == j ? bl_p[(size_t)j] : T(i, j);
          bl[x] = G(i, j, k) = 1 + s;
        } else if (kind == kAcc) {
          if (k + 1 < std::min(i, np))
            s = Ac(i, j, k + 1);
          else if (i < np)
            s = Fn(i, j);
          bl[x] = Ac(i, j, k) = 1 + s;
        } else {  // kFin
          for (int y = i + 1; y < nt; ++y) s = std::max(s, Ac(y, j, i));
          bl[x] = Fn(i, j) = 1 + s;
        }
      }
      // merge the DIAG tasks: TRSM(k+1,k) becomes DIAG(k+1) (its bottom level
      // covers the merged GEMM and POTRF), which are dropped
      {
        size_t w = 0;
        for (size_t x = 0; x < ft.size(); ++x) {
          const int kind = ft[x].x >> 24, i = ft[x].y, j = ft[x].z, k = ft[x].w;
          if (kind == kTrsm && i == k + 1 && i < np) {
            ft[x].x = (kDiag << 24);
          } else if ((kind == kGemm && i == j && i == k + 1 && i < np) || (kind == kPotrf && k > 0)) {
            continue;
          }
          ft[w] = ft[x];
          bl[w] = bl[x];
          ++w;
        }
        ft.resize(w);
        bl.resize(w);
      }
      sh.ft = ft;
      for (int4& t : sh.ft) t.x &= ~0xffffff;  // kind only: the front id is or-ed in per front
      sh.bl = bl;
      sh.top = np > 0 ? bl_p[0] : 0;
  for (int b2 : sh.bl) sh.maxbl = std::max(sh.maxbl, b2);
  return sh;
}

// Per-front task bookkeeping in emission order (fronts from last to first:
// parents before children): bottom-level offsets, task counts and offsets.
struct FrontPlan {
  int q;          // front index
  SplitShape* sh;  // null: one W task
  int off, lvl;   // parent entry offset; W task / ASM bottom level
  int npen;
  int64_t pen0, task_off;
};
int64_t plan_front_tasks(std::vector<HostFront>& fr, std::vector<FrontPlan>& fp, int& maxbl) {
  std::vector<int> entry(fr.size(), 0);  // bottom level of a front's first (children-waiting) tasks
  fp.clear();
  fp.reserve(fr.size());
  maxbl = 0;
  int64_t tot = 0;
  for (size_t q = fr.size(); q-- > 0;) {
    HostFront& hf = fr[q];
    DagFront& d = hf.d;
    const int np = d.np, nt = d.nt;
    const int off = hf.parent >= 0 ? entry[(size_t)hf.parent] : 0;
    FrontPlan f{(int)q, nullptr, off, 0, 0, 0, tot};
    if (d.whole) {
      int w = 1;  // assembly, then the tile tasks in list order (POTRF ~3 tile updates)
      for (int k = 0; k < np; ++k) w += 3 + (nt - k - 1) * (1 + (nt - k) / 2) + k + (k + 1) * (nt - k - 1);
      f.lvl = entry[q] = off + w;
      d.ntask = 1;
      maxbl = std::max(maxbl, f.lvl);
    } else {
      SplitShape& sh = split_shape(np, nt);
      f.sh = &sh;
      const int top = sh.top + off;
      f.npen = (int)(hf.pen1 - hf.pen0);
      f.pen0 = hf.pen0;
      f.lvl = entry[q] = 1 + top + (f.npen > 0 ? 1 : 0);  // ASM tiles, then PEN rows, before every k = 0 task
      d.ntile = nt * (nt + 1) / 2;
      d.nasm = d.ntile + f.npen;
      d.ntask = (int)sh.ft.size() + d.nasm;
      maxbl = std::max(maxbl, std::max(sh.maxbl + off, f.lvl));
    }
    tot += d.ntask;
    fp.push_back(f);
  }
  return tot;
}

// Host task list (the small launches: dense matrices, coarse fronts): every
// front's tasks in emission order, then decreasing bottom level, stable
// (counting sort). The buffers persist per host thread.
std::vector<int4>& build_tasks(std::vector<HostFront>& fr) {
  g_shape_builds = 0;
  thread_local std::vector<int4> all;
  thread_local std::vector<int> all_bl;
  thread_local std::vector<int4> tasks_out;
  thread_local std::vector<FrontPlan> fp;
  int maxbl = 0;
  const int64_t tot = plan_front_tasks(fr, fp, maxbl);
  all.resize((size_t)tot);
  all_bl.resize((size_t)tot);
  for (const FrontPlan& f : fp) {
    const int id = f.q;
    size_t x = (size_t)f.task_off;
    if (!f.sh) {
      all[x] = make_int4((kWhole << 24) | id, 0, 0, 0);
      all_bl[x] = f.lvl;
      continue;
    }
    const SplitShape& sh = *f.sh;
    for (size_t t = 0; t < sh.ft.size(); ++t, ++x) {
      const int4 v = sh.ft[t];
      all[x] = make_int4(v.x | id, v.y, v.z, v.w);
      all_bl[x] = sh.bl[t] + f.off;
    }
    const int nt = fr[(size_t)id].d.nt;
    for (int i = 0; i < nt; ++i)
      for (int j = 0; j <= i; ++j, ++x) {
        all[x] = make_int4((kAsm << 24) | id, i, j, 0);
        all_bl[x] = f.lvl;
      }
    for (int t = 0; t < f.npen; ++t, ++x) {
      all[x] = make_int4((kPen << 24) | id, (int)(f.pen0 + t), 0, 0);
      all_bl[x] = sh.top + f.off + 1;
    }
  }
  g_bt_sort_t0 = std::chrono::steady_clock::now();
  thread_local std::vector<int64_t> start;
  start.assign((size_t)maxbl + 2, 0);
  for (int b2 : all_bl) ++start[(size_t)(maxbl - b2) + 1];
  for (size_t b2 = 1; b2 < start.size(); ++b2) start[b2] += start[b2 - 1];
  tasks_out.resize(all.size());
  for (size_t x = 0; x < all.size(); ++x) tasks_out[(size_t)start[(size_t)(maxbl - all_bl[x])]++] = all[x];
  return tasks_out;
}

// One persistent launch over the plan's task list.
void launch_dag(cutbddc_gpu* h, DagPlan& plan, double* front, const std::vector<DagGroup>& groups,
                const std::vector<int4>* host_tasks) {
  cudaStream_t s = h->stream;
  CB_CUDA(cudaMemsetAsync(plan.counters.p, 0, sizeof(int) * ((size_t)plan.n_counters + 1), s));
  static const char* trace_prefix = [] {
    const char* e = std::getenv("CUTBDDC_DAG_TRACE");
    return e && e[0] ? e : (const char*)nullptr;
  }();
  static DevBuf<unsigned long long> trace;
  if (trace_prefix) trace.alloc(4 * (size_t)plan.n_tasks);
  DagArgs a{};
  a.fronts = reinterpret_cast<const DagFront*>(plan.fronts.p);
  a.tasks = plan.tasks.p;
  a.n_tasks = plan.n_tasks;
  a.front = front;
  a.counters = plan.counters.p;
  a.ticket = plan.counters.p + plan.n_counters;
  if (groups.size() > (size_t)kMaxGroups) throw Failure(CUTBDDC_CONFIG, "dense dag: too many factorisations in one launch");
  for (size_t g = 0; g < groups.size(); ++g) a.g[g] = groups[g];
  a.trace = trace_prefix ? trace.p : nullptr;
  const size_t shm = sizeof(double) * 2 * kTile * (kTile + 1);
  const int grid = (int)device_memo(kMemoDagGrid, [&] {
    CB_CUDA(cudaFuncSetAttribute(k_dense_dag, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm));
    int per_sm = 0, dev = 0, sms = 0;
    CB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_dense_dag, kDagThreads, shm));
    CB_CUDA(cudaGetDevice(&dev));
    CB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    if (const char* e = std::getenv("CUTBDDC_DAG_CTAS_PER_SM")) per_sm = std::min(per_sm, std::atoi(e));  // A/B runs
    return (long long)std::max(1, per_sm) * sms;
  });
  ProfScope ps(h->prof, s, "dense dag kernel");
  cudaEvent_t ev[2] = {nullptr, nullptr};
  if (&plan == &h->dag_factor) {  // device time of the factorisation launches (cutbddc_gpu_time_factor)
    for (cudaEvent_t& e : ev) CB_CUDA(cudaEventCreate(&e));
    CB_CUDA(cudaEventRecord(ev[0], s));
  }
  k_dense_dag<<<std::min<int>(grid, plan.n_tasks), kDagThreads, shm, s>>>(a);
  CB_LAUNCH();
  if (ev[0]) {
    CB_CUDA(cudaEventRecord(ev[1], s));
    h->dag_ev.push_back(ev[0]);
    h->dag_ev.push_back(ev[1]);
  }
  ps.close();
  if (trace_prefix && host_tasks) {  // same layout as the sweep traces (tools/trace_analyze.py)
    static int seq = 0;
    std::vector<unsigned long long> tr(4 * (size_t)plan.n_tasks);
    trace.download(tr.data(), tr.size(), s);
    std::vector<long long> fr(plan.fronts.n);  // front records (DagFront, 10 x int64 each)
    plan.fronts.download(fr.data(), fr.size(), s);
    CB_CUDA(cudaStreamSynchronize(s));
    const std::string path = std::string(trace_prefix) + "_" + std::to_string(seq++) + ".bin";
    if (FILE* fp = std::fopen(path.c_str(), "wb")) {
      const int n = plan.n_tasks;
      std::fwrite(&n, sizeof(int), 1, fp);
      std::fwrite(host_tasks->data(), sizeof(int4), host_tasks->size(), fp);
      std::fwrite(tr.data(), sizeof(unsigned long long), tr.size(), fp);
      const int nf = (int)(fr.size() / 10);
      std::fwrite(&nf, sizeof(int), 1, fp);
      std::fwrite(fr.data(), sizeof(long long), fr.size(), fp);
      std::fclose(fp);
    }
  }
}

// Device copy of a host front list + task list (counters: per front done,
// assembled, then the A and X tile triangles of a split front).
void upload_plan_fronts(cutbddc_gpu* h, DagPlan& plan, std::vector<HostFront>& fr, int64_t n_tasks);
void upload_plan(cutbddc_gpu* h, DagPlan& plan, std::vector<HostFront>& fr, const std::vector<int4>& tasks) {
  upload_plan_fronts(h, plan, fr, (int64_t)tasks.size());
  plan.tasks.upload(tasks, h->stream);
}
void upload_plan_fronts(cutbddc_gpu* h, DagPlan& plan, std::vector<HostFront>& fr, int64_t n_tasks) {
  cudaStream_t s = h->stream;
  if (fr.size() >= (1u << 24)) throw Failure(CUTBDDC_CONFIG, "dense dag: too many fronts");
  thread_local std::vector<DagFront> dv;  // storage kept across calls (every entry rewritten)
  dv.resize(fr.size());
  int64_t cnt = 0;
  for (size_t q = 0; q < fr.size(); ++q) {
    DagFront& d = fr[q].d;
    d.cnt = cnt;
    cnt += 2 + (d.whole ? 0 : (int64_t)d.nt * (d.nt + 1));
    dv[q] = d;
  }
  static_assert(sizeof(DagFront) == 10 * sizeof(long long), "DagFront layout");
  plan.fronts.upload(reinterpret_cast<const long long*>(dv.data()), dv.size() * 10, s);
  if (n_tasks >= (1ll << 31)) throw Failure(CUTBDDC_CONFIG, "dense dag: too many tasks");
  plan.n_tasks = (int)n_tasks;
  plan.n_counters = cnt;
  plan.counters.alloc((size_t)cnt + 1);
}

// Device task list (the subdomain factorisation: up to ~1e6 tasks). The
// host keeps the per-front bookkeeping (plan_front_tasks) and the (np, nt)
// shape templates; one block per front writes its tasks in emission order
// with sort keys maxbl - bottom level, and a stable radix sort gives the
// same list as the host counting sort (build_tasks).
struct DevFrontPlan {
  long long task_off, pen0;
  int q, shape, off, lvl, npen, nt, top, pad_;
};
__global__ void k_expand_tasks(const DevFrontPlan* __restrict__ fp, const int4* __restrict__ tpl,
                               const int* __restrict__ tpl_bl, const int2* __restrict__ tpl_rng, int maxbl,
                               int4* __restrict__ out, unsigned* __restrict__ keys) {
  const DevFrontPlan f = fp[blockIdx.x];
  const long long o = f.task_off;
  if (f.shape < 0) {
    if (threadIdx.x == 0) {
      out[o] = make_int4((kWhole << 24) | f.q, 0, 0, 0);
      keys[o] = (unsigned)(maxbl - f.lvl);
    }
    return;
  }
  const int2 rg = tpl_rng[f.shape];  // (first, count)
  for (int x = threadIdx.x; x < rg.y; x += blockDim.x) {
    const int4 t = tpl[rg.x + x];
    out[o + x] = make_int4(t.x | f.q, t.y, t.z, t.w);
    keys[o + x] = (unsigned)(maxbl - (tpl_bl[rg.x + x] + f.off));
  }
  const int na = f.nt * (f.nt + 1) / 2;
  for (int x = threadIdx.x; x < na; x += blockDim.x) {  // ASM tile (i, j <= i), row-major over the lower triangle
    int i = (int)((sqrt(8.0 * x + 1.0) - 1.0) * 0.5);
    while ((i + 1) * (i + 2) / 2 <= x) ++i;
    while (i * (i + 1) / 2 > x) --i;
    out[o + rg.y + x] = make_int4((kAsm << 24) | f.q, i, x - i * (i + 1) / 2, 0);
    keys[o + rg.y + x] = (unsigned)(maxbl - f.lvl);
  }
  for (int t = threadIdx.x; t < f.npen; t += blockDim.x) {
    out[o + rg.y + na + t] = make_int4((kPen << 24) | f.q, (int)(f.pen0 + t), 0, 0);
    keys[o + rg.y + na + t] = (unsigned)(maxbl - (f.top + f.off + 1));
  }
}

void build_tasks_device(cutbddc_gpu* h, DagPlan& plan, std::vector<HostFront>& fr) {
  cudaStream_t s = h->stream;
  g_shape_builds = 0;
  thread_local std::vector<FrontPlan> fp;
  int maxbl = 0;
  const int64_t tot = plan_front_tasks(fr, fp, maxbl);
  // shape templates used by this list
  std::map<SplitShape*, int> sid;
  std::vector<int4> tpl;
  std::vector<int> tpl_bl;
  std::vector<int2> rng;
  thread_local std::vector<DevFrontPlan> dfp;  // storage kept across calls (every entry rewritten)
  dfp.resize(fp.size());
  for (size_t x = 0; x < fp.size(); ++x) {
    const FrontPlan& f = fp[x];
    int id = -1;
    if (f.sh) {
      auto it = sid.find(f.sh);
      if (it == sid.end()) {
        id = (int)rng.size();
        sid[f.sh] = id;
        rng.push_back(make_int2((int)tpl.size(), (int)f.sh->ft.size()));
        tpl.insert(tpl.end(), f.sh->ft.begin(), f.sh->ft.end());
        tpl_bl.insert(tpl_bl.end(), f.sh->bl.begin(), f.sh->bl.end());
      } else {
        id = it->second;
      }
    }
    dfp[x] = DevFrontPlan{f.task_off, f.pen0, f.q, id, f.off, f.lvl, f.npen, fr[(size_t)f.q].d.nt,
                          f.sh ? f.sh->top : 0, 0};
  }
  upload_plan_fronts(h, plan, fr, tot);
  static_assert(sizeof(DevFrontPlan) == 48, "DevFrontPlan layout");
  plan.d_fplan.upload(reinterpret_cast<const long long*>(dfp.data()), dfp.size() * 6, s);
  plan.d_tpl.upload(tpl.empty() ? std::vector<int4>{make_int4(0, 0, 0, 0)} : tpl, s);
  plan.d_tpl_bl.upload(tpl_bl.empty() ? std::vector<int>{0} : tpl_bl, s);
  plan.d_tpl_rng.upload(rng.empty() ? std::vector<int2>{make_int2(0, 0)} : rng, s);
  plan.keys.alloc((size_t)2 * std::max<int64_t>(1, tot));
  plan.unsorted.alloc((size_t)std::max<int64_t>(1, tot));
  plan.tasks.alloc((size_t)std::max<int64_t>(1, tot));
  k_expand_tasks<<<(unsigned)fp.size(), 128, 0, s>>>(reinterpret_cast<const DevFrontPlan*>(plan.d_fplan.p), plan.d_tpl.p,
                                                     plan.d_tpl_bl.p, plan.d_tpl_rng.p, maxbl, plan.unsorted.p,
                                                     plan.keys.p);
  CB_LAUNCH();
  int bits = 1;
  while (bits < 32 && (maxbl >> bits) != 0) ++bits;
  size_t tmp = 0;
  CB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, plan.keys.p, plan.keys.p + tot, plan.unsorted.p, plan.tasks.p,
                                          (int)tot, 0, bits, s));
  plan.sort_tmp.alloc(std::max<size_t>(1, tmp));
  CB_CUDA(cub::DeviceRadixSort::SortPairs(plan.sort_tmp.p, tmp, plan.keys.p, plan.keys.p + tot, plan.unsorted.p,
                                          plan.tasks.p, (int)tot, 0, bits, s));
}

}  // namespace

// Host: the numeric factorisation of every span (subdomains [sd0, sd1) of
// one factorisation each; fronts at span.front_off + the subdomain's front
// base + the per-front offset in `front`) as ONE dataflow launch: every
// front of every level of every span. The task list is rebuilt only when the
// compact front sizes change.
void dense_dag_factor(cutbddc_gpu* h, const std::vector<FactorSpan>& spans, double* front) {
  cudaStream_t s = h->stream;
  DagPlan& plan = h->dag_factor;
  // The key holds everything the task list is built from: per span the
  // subdomain range, the workspace offset, the template (block lattice and
  // which supernodes are split), the compact front sizes, and -- for the
  // constrained K factorisation -- each subdomain's constraint-row range
  // (PEN tasks store absolute row indices, so new coarse objects on the same
  // geometry must rebuild the list).
  std::vector<int2> key;
  {
    size_t nkey = 0;
    for (const FactorSpan& sp : spans) nkey += 3 + sp.ts->is_split.size() / 2 + 1 + sp.f->h_rc.size() + (size_t)(sp.sd1 - sp.sd0) + 1;
    key.reserve(nkey);
  }
  for (const FactorSpan& sp : spans) {
    key.push_back(make_int2(sp.sd0, sp.sd1));
    key.push_back(make_int2((int)(sp.front_off >> 31), (int)(sp.front_off & 0x7fffffff)));
    key.push_back(make_int2(sp.ts->tpl.b1, (int)sp.ts->tpl.sn.size()));
    for (size_t q = 0; q < sp.ts->is_split.size(); q += 2)
      key.push_back(make_int2(sp.ts->is_split[q], q + 1 < sp.ts->is_split.size() ? sp.ts->is_split[q + 1] : 2));
    key.insert(key.end(), sp.f->h_rc.begin(), sp.f->h_rc.end());
    if (sp.in->c_ptr)
      for (int sd = sp.sd0; sd <= sp.sd1; ++sd) {
        const int64_t m = h->h_m_off[(size_t)sd];
        key.push_back(make_int2((int)(m >> 31), (int)(m & 0x7fffffff)));
      }
  }
  const bool hit = plan.key.size() == key.size() &&
                   std::memcmp(plan.key.data(), key.data(), sizeof(int2) * key.size()) == 0 &&
                   !std::getenv("CUTBDDC_DAG_TRACE") && !std::getenv("CUTBDDC_NO_PLAN_CACHE");
  const std::vector<int4>* tasks = nullptr;
  if (!hit) {
    ProfScope ps(h->prof, s, "dense dag host+upload");
    // the front list and its index scratch keep their storage across calls (per
    // host thread: batched handles run on several): at cfg5 the list is
    // ~120k records, and growing a fresh vector was most of this scope's time
    thread_local std::vector<HostFront> fr;
    thread_local std::vector<int> idx;
    fr.clear();
    {
      size_t nfr = 0;
      for (const FactorSpan& sp : spans) nfr += (size_t)(sp.sd1 - sp.sd0) * sp.ts->tpl.sn.size();
      fr.reserve(nfr);
    }
    for (size_t g = 0; g < spans.size(); ++g) {
      const FactorSpan& sp = spans[g];
      const TplSet& ts = *sp.ts;
      const FactorSet& f = *sp.f;
      const int nsn = (int)ts.tpl.sn.size();
      idx.assign((size_t)(sp.sd1 - sp.sd0) * nsn, -1);
      for (int sd = sp.sd0; sd < sp.sd1; ++sd)
        for (int sid = 0; sid < nsn; ++sid) {  // postorder: children first
          const size_t fs = (size_t)sd * nsn + sid;
          const int2 v = f.h_rc[fs];
          if (v.x == 0) continue;
          const Supernode& sn = ts.tpl.sn[(size_t)sid];
          HostFront hf{};
          DagFront& d = hf.d;
          d.r = v.x;
          d.c = v.y;
          d.np = (v.y + kTile - 1) / kTile;
          d.nt = d.np + (v.x - v.y + kTile - 1) / kTile;
          d.fo = sp.front_off + (f.h_front_base[(size_t)sd] - f.h_front_base[(size_t)sp.sd0]) + f.h_front_off[fs];
          d.po = f.h_panel_off[fs];
          d.sd = sd;
          d.sid = sid;
          d.grp = (int)g;
          d.whole = ts.is_split[(size_t)sid] ? 0 : 1;
          d.ch0 = sn.nchild > 0 ? idx[(size_t)(sd - sp.sd0) * nsn + sn.child[0]] : -1;
          d.ch1 = sn.nchild > 1 ? idx[(size_t)(sd - sp.sd0) * nsn + sn.child[1]] : -1;
          hf.parent = -1;
          hf.pen0 = hf.pen1 = 0;
          if (!d.whole && sid == nsn - 1 && sp.in->c_ptr) {
            hf.pen0 = h->h_m_off[(size_t)sd];
            hf.pen1 = h->h_m_off[(size_t)sd + 1];
          }
          idx[(size_t)(sd - sp.sd0) * nsn + sid] = (int)fr.size();
          fr.push_back(hf);
        }
    }
    for (size_t q = 0; q < fr.size(); ++q) {
      const DagFront& d = fr[q].d;
      if (d.ch0 >= 0) fr[(size_t)d.ch0].parent = (int)q;
      if (d.ch1 >= 0) fr[(size_t)d.ch1].parent = (int)q;
    }
    if (fr.empty()) return;
    const auto t0 = std::chrono::steady_clock::now();
    build_tasks_device(h, plan, fr);
    const auto t1 = std::chrono::steady_clock::now();
    if (std::getenv("CUTBDDC_DAG_CHECK")) {  // test hook: the device list equals the host list
      std::vector<int4> dl = plan.tasks.to_host(s);
      const std::vector<int4>& hl = build_tasks(fr);
      dl.resize((size_t)plan.n_tasks);
      if (dl.size() != hl.size() || std::memcmp(dl.data(), hl.data(), sizeof(int4) * hl.size()) != 0)
        throw Failure(CUTBDDC_INTERNAL, "dense dag: device task list differs from the host list");
    }
    if (std::getenv("CUTBDDC_DAG_TRACE")) {  // the trace dump wants the list on the host
      thread_local std::vector<int4> tl;
      tl = plan.tasks.to_host(s);
      tl.resize((size_t)plan.n_tasks);
      tasks = &tl;
    }
    plan.key = key;
    if (std::getenv("CUTBDDC_DAG_STATS")) {
      const auto t2 = std::chrono::steady_clock::now();
      std::fprintf(stderr, "[dag stats] fronts %zu tasks %d shapes %d build+enqueue %.2f ms, then %.2f ms\n",
                   fr.size(), plan.n_tasks, g_shape_builds,
                   std::chrono::duration<double, std::milli>(t1 - t0).count(),
                   std::chrono::duration<double, std::milli>(t2 - t1).count());
    }
  }
  std::vector<DagGroup> groups;
  for (const FactorSpan& sp : spans)
    groups.push_back(DagGroup{tpl_dev(*sp.ts, h->slots), factor_dev(*sp.f), *sp.in, sp.f->panel.p, sp.fail, sp.fail_sd});
  launch_dag(h, plan, front, groups, hit ? nullptr : tasks);
}

// Cholesky + explicit inverse factor of one dense SPD n x n matrix (A:
// column-major lower part, overwritten by L; X receives L^{-1}, lower part).
// A non-positive pivot is reported as its index in *fail.
void dense_dag_matrix(cutbddc_gpu* h, double* A, double* X, int n, unsigned long long* fail) {
  if (n <= 0) return;
  ProfScope ps(h->prof, h->stream, "dense dag host+upload");
  HostFront hf{};
  DagFront& d = hf.d;
  d.r = d.c = n;
  d.np = d.nt = (n + kTile - 1) / kTile;
  d.sd = d.sid = -1;
  d.ch0 = d.ch1 = -1;
  hf.parent = -1;
  std::vector<HostFront> fr{hf};
  std::vector<int4> tasks = build_tasks(fr);
  fr[0].d.nasm = 0;  // the matrix is assembled: no ASM tasks
  std::vector<int4> kept;
  for (const int4& tk : tasks)
    if ((tk.x >> 24) != kAsm) kept.push_back(tk);
  fr[0].d.ntask = (int)kept.size();
  upload_plan(h, h->dag_dense, fr, kept);
  ps.close();
  launch_dag(h, h->dag_dense, A, {DagGroup{TplDev{}, FactorDev{}, FactorInput{}, X, fail, nullptr}}, &kept);
}

void dense_dag_fronts(cutbddc_gpu* h, DagPlan& plan, double* F, double* X, const std::vector<DenseFront>& fronts,
                      unsigned long long* fail) {
  if (fronts.empty()) return;
  ProfScope ps(h->prof, h->stream, "dense dag host+upload");
  std::vector<HostFront> fr(fronts.size());
  for (size_t q = 0; q < fronts.size(); ++q) {
    HostFront& hf = fr[q];
    hf = HostFront{};
    DagFront& d = hf.d;
    d.fo = fronts[q].fo;
    d.po = fronts[q].po;
    d.r = fronts[q].r;
    d.c = fronts[q].c;
    d.np = (d.c + kTile - 1) / kTile;
    d.nt = d.np + (d.r - d.c + kTile - 1) / kTile;
    d.sd = d.sid = -1;
    d.ch0 = d.ch1 = -1;
    hf.parent = -1;
  }
  std::vector<int4> tasks = build_tasks(fr);
  std::vector<int4> kept;
  std::vector<int> ntask(fr.size(), 0);
  for (const int4& tk : tasks)
    if ((tk.x >> 24) != kAsm) {
      kept.push_back(tk);
      ++ntask[(size_t)(tk.x & 0xffffff)];
    }
  for (size_t q = 0; q < fr.size(); ++q) {  // assembled in place: no ASM tasks
    fr[q].d.nasm = 0;
    fr[q].d.ntask = ntask[q];
  }
  upload_plan(h, plan, fr, kept);
  ps.close();
  launch_dag(h, plan, F, {DagGroup{TplDev{}, FactorDev{}, FactorInput{}, X, fail, nullptr}}, &kept);
}

}  // namespace cutbddc_b200
