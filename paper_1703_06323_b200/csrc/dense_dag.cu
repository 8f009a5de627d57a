// dense_dag.cu — tiled partial Cholesky + explicit inverse panel of the large
// fronts (the dense top of the ND elimination tree), one persistent launch per
// level, dataflow-scheduled.
//
// Replaces, for fronts of >= kSplitRows template rows, the right-looking
// 32-column panel steps (three launches per step, the trailing matrix
// streamed through HBM at every step) and the left-looking k_trinv /
// k_gemm_m. The front F (r x r, column-major, lower part) is cut into tiles
// of at most 64 x 64 whose boundaries are 0, 64, ..., c (the pivot columns)
// and c, c + 64, ..., r (the update rows/columns). Tasks:
//   POTRF(k)      F_kk = L_kk L_kk^T and P_kk = L_kk^{-1}          (k < np)
//   TRSM(i,k)     F_ik = F_ik P_kk^T = L_ik                          (i > k)
//   GEMM(i,j,k)   F_ij -= L_ik L_jk^T                     (i >= j > k)
//   ACC(i,j,k)    P_ij (+)= L_ik P_kj                 (j <= k < min(i, np))
//   FIN(i,j)      P_ij = -P_ii P_ij                         (j < i < np)
// P is the explicit panel G = [L11^{-1}; L21 L11^{-1}] the solve sweeps use:
// the first c columns of M^{-1}, M = [L11 0; L21 I], with the lower block
// negated (G21 = +sum L21 X). The trailing tiles (j >= np) end as the update
// matrix the parent gathers (k_split_extend).
// Every tile is updated in a fixed order (per-tile counters), so the result
// is deterministic. Tasks are listed step by step (k), every task after the
// tasks it waits for, and handed out by an atomic ticket: no deadlock.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "factor.cuh"

namespace cutbddc_b200 {
namespace {

constexpr int kTile = 64;
constexpr int kDagThreads = 256;
constexpr int kFinal = 1 << 20;  // X tile completed
enum { kPotrf = 0, kTrsm = 1, kGemm = 2, kAcc = 3, kFin = 4 };

struct DagFront {
  long long fo, po, cnt;  // front (in the level's workspace), panel, counter offsets
  int r, c, np, nt;       // rows, pivot columns, pivot / all tile blocks
  int sd, sid;
};

struct DagArgs {
  const DagFront* fronts;
  const int4* tasks;
  int n_tasks;
  double* front;
  double* panel;
  int* counters;
  int* ticket;
  unsigned long long* fail;
  TplDev t;
  FactorDev f;
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

// The dense trailing updates on the DMMA tensor cores: 8 warps, each owns a
// 16 x 32 block of the 64 x 64 output (2 x 4 mma tiles); k staged through
// shared memory 32 at a time (rows padded to 65 doubles: conflict-free
// fragment loads).
__device__ void tile_mm(double* C, int ldc, const double* A, int lda, const double* B, int ldb, int m, int n, int kk,
                        double alpha, bool acc, bool bt, bool lower, double* sm) {
  double(*as)[kTile + 1] = reinterpret_cast<double(*)[kTile + 1]>(sm);
  double(*bs)[kTile + 1] = reinterpret_cast<double(*)[kTile + 1]>(sm + 32 * (kTile + 1));
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int wr = (wid & 3) * 16, wc = (wid >> 2) * 32;  // warp's output block origin
  const int fr = lane >> 2, fk = lane & 3;               // fragment row/col and k index
  double d[2][4][2];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) d[a][b][0] = d[a][b][1] = 0.0;
  for (int k0 = 0; k0 < kk; k0 += 32) {
    __syncthreads();
    for (int e = tid; e < 32 * kTile; e += kDagThreads) {
      const int row = e & 63, k = e >> 6;
      as[k][row] = (row < m && k0 + k < kk) ? A[row + (int64_t)(k0 + k) * lda] : 0.0;
    }
    if (bt) {
      for (int e = tid; e < 32 * kTile; e += kDagThreads) {
        const int col = e & 63, k = e >> 6;
        bs[k][col] = (col < n && k0 + k < kk) ? B[col + (int64_t)(k0 + k) * ldb] : 0.0;
      }
    } else {
      for (int e = tid; e < 32 * kTile; e += kDagThreads) {
        const int k = e & 31, col = e >> 5;
        bs[k][col] = (col < n && k0 + k < kk) ? B[(k0 + k) + (int64_t)col * ldb] : 0.0;
      }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 32; k += 4) {
      double fa[2], fb[4];
#pragma unroll
      for (int a = 0; a < 2; ++a) fa[a] = as[k + fk][wr + 8 * a + fr];
#pragma unroll
      for (int b = 0; b < 4; ++b) fb[b] = bs[k + fk][wc + 8 * b + fr];
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) dmma_8x8x4(d[a][b][0], d[a][b][1], fa[a], fb[b]);
    }
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
        double* cp = C + i + (int64_t)j * ldc;
        *cp = (acc ? *cp : 0.0) + alpha * d[a][b][h2];
      }
}

// Cholesky of the n x n diagonal tile and the inverse of its factor; the
// strict upper parts of both stored tiles become zero.
typedef double SmTile[kTile + 1];

// Warp: Cholesky of the m x m block at (o, o) of `ls` (m <= 16); lane i holds
// row o + i in registers, column j values are broadcast by shuffles.
// Non-positive pivots are reported (fail) and replaced by 1.
template <typename Fail>
__device__ void warp_chol16(SmTile* ls, int o, int m, int lane, Fail fail) {
  double a[16];
#pragma unroll
  for (int q = 0; q < 16; ++q) a[q] = (lane < m && q <= lane) ? ls[o + lane][o + q] : 0.0;
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    if (j < m) {
      double djj = __shfl_sync(0xffffffffu, a[j], j);
      if (!(djj > 0.0)) {
        if (lane == 0) fail(o + j);
        djj = 1.0;
      }
      const double rl = rsqrt(djj), l = djj * rl;
      if (lane == j) {
        a[j] = l;
        ls[o + j][kTile] = rl;  // 1 / L_jj in the padding column (used by warp_inv16)
      } else if (lane > j) {
        a[j] *= rl;
      }
#pragma unroll
      for (int q = j + 1; q < 16; ++q) {
        const double lqj = __shfl_sync(0xffffffffu, a[j], q);
        if (lane >= q) a[q] -= a[j] * lqj;
      }
    }
  }
#pragma unroll
  for (int q = 0; q < 16; ++q)
    if (lane < m && q <= lane) ls[o + lane][o + q] = a[q];
}

// Warp: X = L^{-1} of the m x m lower block at (o, o) (m <= 16); lane j
// computes column j in registers (L rows broadcast from shared memory).
__device__ void warp_inv16(SmTile* ls, SmTile* xs, int o, int m, int lane) {
  double x[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    double v = 0.0;
    if (i < m) {
      const double rd = ls[o + i][kTile];  // 1 / L_ii from warp_chol16
      double s = i == lane ? 1.0 : 0.0;
#pragma unroll
      for (int k = 0; k < i; ++k) s -= ls[o + i][o + k] * x[k];
      v = lane <= i ? s * rd : 0.0;
    }
    x[i] = v;
  }
#pragma unroll
  for (int i = 0; i < 16; ++i)
    if (lane < m && i < m) xs[o + i][o + lane] = x[i];
}

// Cholesky of the n x n diagonal tile and the inverse of its factor, blocked
// by 16: per diagonal block a register-resident warp Cholesky + inverse, then
// the panel below (L_ib = A_ib X_bb^T) and the trailing update by the whole
// CTA; the off-diagonal blocks of X = L^{-1} follow by block diagonals,
// X_ij = -X_ii sum_{k=j}^{i-1} L_ik X_kj. Strict upper parts stored as zero.
template <typename Fail>
__device__ void tile_potrf_inv(double* F, int ldf, double* P, int ldp, int n, double* sm, Fail fail) {
  SmTile* ls = reinterpret_cast<SmTile*>(sm);
  SmTile* xs = reinterpret_cast<SmTile*>(sm + kTile * (kTile + 1));
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int nb = (n + 15) / 16;
  __syncthreads();
  for (int e = tid; e < kTile * kTile; e += kDagThreads) {
    const int i = e & 63, j = e >> 6;
    ls[i][j] = (i < n && j < n && i >= j) ? F[i + (int64_t)j * ldf] : 0.0;
    xs[i][j] = 0.0;
  }
  __syncthreads();
  for (int b = 0; b < nb; ++b) {
    const int o = 16 * b, m = min(16, n - o), below = n - o - m;
    if (wid == 0) {
      warp_chol16(ls, o, m, lane, fail);
      __syncwarp();
      warp_inv16(ls, xs, o, m, lane);
    }
    __syncthreads();
    if (below <= 0) break;
    // L_ib = A_ib X_bb^T (rows o+16.., columns o..o+m)
    double l[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = tid + u * kDagThreads, i = o + 16 + (e >> 4), q = e & 15;
      double s = 0.0;
      if (i < n && q < m)
        for (int k = 0; k <= q; ++k) s += ls[i][o + k] * xs[o + q][o + k];
      l[u] = s;
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = tid + u * kDagThreads, i = o + 16 + (e >> 4), q = e & 15;
      if (i < n && q < m) ls[i][o + q] = l[u];
    }
    __syncthreads();
    // trailing update A_ij -= L_ib L_jb^T (o+16 <= j <= i < n)
    for (int e = tid; e < below * below; e += kDagThreads) {
      const int i = o + 16 + e / below, j = o + 16 + e % below;
      if (j > i) continue;
      double s = 0.0;
#pragma unroll
      for (int k = 0; k < 16; ++k) s += ls[i][o + k] * ls[j][o + k];
      ls[i][j] -= s;
    }
    __syncthreads();
  }
  // off-diagonal blocks of X, one block diagonal at a time
  for (int d = 1; d < nb; ++d) {
    const int nblk = nb - d;
    // T_ij = sum_{k=j}^{i-1} L_ik X_kj into xs block (i, j)
    for (int e = tid; e < nblk * 256; e += kDagThreads) {
      const int jb = e >> 8, ib = jb + d, p = (e >> 4) & 15, q = e & 15;
      const int i = 16 * ib + p, j = 16 * jb + q;
      double s = 0.0;
      if (i < n)
        for (int k = 16 * jb; k < 16 * ib; ++k) s += ls[i][k] * xs[k][j];
      xs[i][j] = s;
    }
    __syncthreads();
    double x[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = tid + u * kDagThreads;
      double s = 0.0;
      if (e < nblk * 256) {
        const int jb = e >> 8, ib = jb + d, p = (e >> 4) & 15, q = e & 15;
        const int i = 16 * ib + p, j = 16 * jb + q;
        for (int t = 16 * ib; t <= i; ++t) s += xs[i][t] * xs[t][j];
      }
      x[u] = -s;
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = tid + u * kDagThreads;
      if (e < nblk * 256) {
        const int jb = e >> 8, ib = jb + d, p = (e >> 4) & 15, q = e & 15;
        xs[16 * ib + p][16 * jb + q] = x[u];
      }
    }
    __syncthreads();
  }
  for (int e = tid; e < n * n; e += kDagThreads) {
    const int i = e % n, j = e / n;
    F[i + (int64_t)j * ldf] = i >= j ? ls[i][j] : 0.0;
    P[i + (int64_t)j * ldp] = i >= j ? xs[i][j] : 0.0;
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
    double* F = a.front + d.fo;
    double* P = a.panel + d.po;
    int* A = a.counters + d.cnt;            // factor tiles: updates applied, col + 1 when final
    int* X = A + d.nt * (d.nt + 1) / 2;     // panel tiles: accumulations applied, kFinal when final
    const int r = d.r;
    auto tile = [&](double* base, int ti, int tj) { return base + bnd(d, ti) + (int64_t)bnd(d, tj) * r; };
    auto ext = [&](int b) { return bnd(d, b + 1) - bnd(d, b); };
    int* done = nullptr;
    int inc = 1;
    if (kind == kPotrf) {
      if (tid == 0) wait_eq(A + tri(k, k), k);
      if (a.trace && tid == 0) s_t1 = dag_timer();
      __syncthreads();
      __threadfence();
      const int n = ext(k);
      const int col0 = bnd(d, k);
      tile_potrf_inv(tile(F, k, k), r, tile(P, k, k), r, n, sm, [&](int jj) {
        if (d.sid < 0) {  // plain dense matrix: the pivot index
          atomicMin(a.fail, (unsigned long long)(col0 + jj));
          return;
        }
        // report the template slot of compact column col0 + jj (pivot rule, linalg.cpp:42-54)
        const Supernode s = a.t.sn[d.sid];
        const int q = a.f.tpos[(int64_t)d.sd * a.t.rows_total + s.rows_off + col0 + jj];
        atomicMin(a.fail, (unsigned long long)((int64_t)d.sd * a.t.T + a.t.rows[s.rows_off + q]));
      });
      // (the panel above this diagonal tile is never read: the sweeps start
      // every column at the 32-row block holding its diagonal)
      done = A + tri(k, k);
    } else if (kind == kTrsm) {
      if (tid == 0) {
        wait_eq(A + tri(k, k), k + 1);
        wait_eq(A + tri(i, k), k);
      }
      if (a.trace && tid == 0) s_t1 = dag_timer();
      __syncthreads();
      __threadfence();
      tile_mm(tile(F, i, k), r, tile(F, i, k), r, tile(P, k, k), r, ext(i), ext(k), ext(k), 1.0, false, true, false, sm);
      done = A + tri(i, k);
    } else if (kind == kGemm) {
      if (tid == 0) {
        wait_eq(A + tri(i, k), k + 1);
        wait_eq(A + tri(j, k), k + 1);
        wait_eq(A + tri(i, j), k);
      }
      if (a.trace && tid == 0) s_t1 = dag_timer();
      __syncthreads();
      __threadfence();
      tile_mm(tile(F, i, j), r, tile(F, i, k), r, tile(F, j, k), r, ext(i), ext(j), ext(k), -1.0, true, true, i == j, sm);
      done = A + tri(i, j);
    } else if (kind == kAcc) {
      if (tid == 0) {
        wait_eq(A + tri(i, k), k + 1);
        if (k == j)
          wait_eq(A + tri(j, j), j + 1);
        else
          wait_eq(X + tri(k, j), kFinal);
        wait_eq(X + tri(i, j), k - j);
      }
      if (a.trace && tid == 0) s_t1 = dag_timer();
      __syncthreads();
      __threadfence();
      tile_mm(tile(P, i, j), r, tile(F, i, k), r, tile(P, k, j), r, ext(i), ext(j), ext(k), 1.0, k != j, false, false, sm);
      done = X + tri(i, j);
    } else {  // kFin
      if (tid == 0) {
        wait_eq(X + tri(i, j), i - j);
        wait_eq(A + tri(i, i), i + 1);
      }
      if (a.trace && tid == 0) s_t1 = dag_timer();
      __syncthreads();
      __threadfence();
      tile_mm(tile(P, i, j), r, tile(P, i, i), r, tile(P, i, j), r, ext(i), ext(j), ext(i), -1.0, false, false, false, sm);
      done = X + tri(i, j);
      inc = kFinal - (i - j);
    }
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      atomicAdd(done, inc);
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

// task list (step by step) + one persistent launch over `fr`
void run_dag(cutbddc_gpu* h, std::vector<DagFront>& fr, int64_t cnt, double* front, double* panel,
             unsigned long long* fail, const TplDev& t, const FactorDev& fdv);

}  // namespace

// Host: factorise the split fronts of one level for subdomains [sd0, sd1).
// foff / poff: front-workspace and panel offsets per (sd, supernode); the
// level's front workspace starts at `front` (= subdomain sd0's base).
void dense_dag_level(cutbddc_gpu* h, const TplSet& ts, const FactorSet& f, const std::vector<int>& sids, int sd0,
                     int sd1, const std::vector<int64_t>& foff, const std::vector<int64_t>& poff, double* front,
                     unsigned long long* fail) {
  cudaStream_t s = h->stream;
  const int nsn = (int)ts.tpl.sn.size();
  ProfScope ps(h->prof, s, "dense dag host+upload");
  std::vector<DagFront> fr;
  int64_t cnt = 0;
  for (int sd = sd0; sd < sd1; ++sd)
    for (int sid : sids) {
      const int2 v = f.h_rc[(size_t)sd * nsn + sid];
      if (v.x == 0 || v.y == 0) continue;
      DagFront d{};
      d.r = v.x;
      d.c = v.y;
      d.np = (v.y + kTile - 1) / kTile;
      d.nt = d.np + (v.x - v.y + kTile - 1) / kTile;
      d.fo = (f.h_front_base[(size_t)sd] - f.h_front_base[(size_t)sd0]) + foff[(size_t)sd * nsn + sid];
      d.po = poff[(size_t)sd * nsn + sid];
      d.cnt = cnt;
      d.sd = sd;
      d.sid = sid;
      cnt += (int64_t)d.nt * (d.nt + 1);  // A and X triangles
      fr.push_back(d);
    }
  if (fr.empty()) return;
  ps.close();
  run_dag(h, fr, cnt, front, f.panel.p, fail, tpl_dev(ts, h->slots), factor_dev(f));
}

// Cholesky + explicit inverse factor of one dense SPD n x n matrix (A:
// column-major lower part, overwritten by L; X receives L^{-1}, lower part).
// A non-positive pivot is reported as its index in *fail.
void dense_dag_matrix(cutbddc_gpu* h, double* A, double* X, int n, unsigned long long* fail) {
  if (n <= 0) return;
  DagFront d{};
  d.r = d.c = n;
  d.np = d.nt = (n + kTile - 1) / kTile;
  d.sd = d.sid = -1;
  std::vector<DagFront> fr{d};
  run_dag(h, fr, (int64_t)d.nt * (d.nt + 1), A, X, fail, TplDev{}, FactorDev{});
}

namespace {

void run_dag(cutbddc_gpu* h, std::vector<DagFront>& fr, int64_t cnt, double* front, double* panel,
             unsigned long long* fail, const TplDev& t, const FactorDev& fdv) {
  cudaStream_t s = h->stream;
  ProfScope ps(h->prof, s, "dense dag host+upload");
  // Tasks in decreasing "bottom level" (weighted length of the longest path
  // from the task to the end of its front's DAG): the POTRF chain and the
  // tasks feeding it come first, wide trailing updates later. A predecessor
  // always has a strictly larger bottom level, so this order is topological
  // (every wait is on a smaller ticket: no deadlock).
  std::vector<int> order(fr.size());
  for (size_t q = 0; q < fr.size(); ++q) order[q] = (int)q;
  std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return fr[x].np > fr[y].np; });
  std::vector<std::vector<int4>> bucket;
  std::vector<int4> ft;
  std::vector<int> bl_p, bl_t, bl_g, bl_a, bl_f;
  for (int id : order) {
    const DagFront& d = fr[(size_t)id];
    const int np = d.np, nt = d.nt;
    ft.clear();
    auto push = [&](int kind, int i, int j, int kk) { ft.push_back(make_int4((kind << 24) | id, i, j, kk)); };
    for (int k = 0; k < np; ++k) {  // per front, step by step (successors later)
      push(kPotrf, k, k, k);
      for (int i = k + 1; i < nt; ++i) push(kTrsm, i, k, k);
      for (int jj = k + 1; jj < nt; ++jj)
        for (int i = jj; i < nt; ++i) push(kGemm, i, jj, k);
      for (int jj = 0; jj < k; ++jj) push(kFin, k, jj, k);
      for (int jj = 0; jj <= k; ++jj)
        for (int i = k + 1; i < nt; ++i) push(kAcc, i, jj, k);
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
    std::vector<int> bl(ft.size());
    for (size_t q = ft.size(); q-- > 0;) {
      const int kind = ft[q].x >> 24, i = ft[q].y, j = ft[q].z, k = ft[q].w;
      int s = 0;
      if (kind == kPotrf) {
        for (int x = k + 1; x < nt; ++x) s = std::max({s, T(x, k), Ac(x, k, k)});
        for (int y = 0; y < k; ++y) s = std::max(s, Fn(k, y));
        bl[q] = bl_p[(size_t)k] = 3 + s;  // the diagonal tile weighs ~3 tile updates
      } else if (kind == kTrsm) {
        for (int y = k + 1; y <= i; ++y) s = std::max(s, G(i, y, k));
        for (int x = i; x < nt; ++x) s = std::max(s, G(x, i, k));
        for (int y = 0; y <= k; ++y) s = std::max(s, Ac(i, y, k));
        bl[q] = T(i, k) = 1 + s;
      } else if (kind == kGemm) {
        if (k + 1 < j && k + 1 < np)
          s = G(i, j, k + 1);
        else if (j < np)
          s = i == j ? bl_p[(size_t)j] : T(i, j);
        bl[q] = G(i, j, k) = 1 + s;
      } else if (kind == kAcc) {
        if (k + 1 < std::min(i, np))
          s = Ac(i, j, k + 1);
        else if (i < np)
          s = Fn(i, j);
        bl[q] = Ac(i, j, k) = 1 + s;
      } else {  // kFin
        for (int x = i + 1; x < nt; ++x) s = std::max(s, Ac(x, j, i));
        bl[q] = Fn(i, j) = 1 + s;
      }
    }
    for (size_t q = 0; q < ft.size(); ++q) {
      if ((size_t)bl[q] >= bucket.size()) bucket.resize((size_t)bl[q] + 1);
      bucket[(size_t)bl[q]].push_back(ft[q]);
    }
  }
  std::vector<int4> tasks;
  for (size_t b = bucket.size(); b-- > 0;) tasks.insert(tasks.end(), bucket[b].begin(), bucket[b].end());
  if (fr.size() >= (1u << 24)) throw Failure(CUTBDDC_CONFIG, "dense dag: too many fronts in one level");
  static_assert(sizeof(DagFront) == 6 * sizeof(long long), "DagFront layout");
  DevBuf<long long>& dfr = h->ws_dag_fronts;
  DevBuf<int4>& dtk = h->ws_dag_tasks;
  DevBuf<int>& dcn = h->ws_dag_counters;
  dfr.upload(reinterpret_cast<const long long*>(fr.data()), fr.size() * 6, s);
  dtk.upload(tasks, s);
  dcn.alloc((size_t)cnt + 1);
  CB_CUDA(cudaMemsetAsync(dcn.p, 0, sizeof(int) * ((size_t)cnt + 1), s));
  static const char* trace_prefix = [] {
    const char* e = std::getenv("CUTBDDC_DAG_TRACE");
    return e && e[0] ? e : (const char*)nullptr;
  }();
  static DevBuf<unsigned long long> trace;
  if (trace_prefix) trace.alloc(4 * tasks.size());
  DagArgs a{reinterpret_cast<const DagFront*>(dfr.p), dtk.p, (int)tasks.size(), front, panel, dcn.p, dcn.p + cnt,
            fail, t, fdv, trace_prefix ? trace.p : nullptr};
  const size_t shm = sizeof(double) * 2 * kTile * (kTile + 1);
  static int grid = 0;
  if (!grid) {
    CB_CUDA(cudaFuncSetAttribute(k_dense_dag, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm));
    int per_sm = 0, dev = 0, sms = 0;
    CB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_dense_dag, kDagThreads, shm));
    CB_CUDA(cudaGetDevice(&dev));
    CB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    grid = std::max(1, per_sm) * sms;
  }
  ps.next("dense dag kernel");
  k_dense_dag<<<std::min<int>(grid, (int)tasks.size()), kDagThreads, shm, s>>>(a);
  CB_LAUNCH();
  CB_CUDA(cudaStreamSynchronize(s));  // host task vectors go out of scope
  if (trace_prefix) {  // same layout as the sweep traces (tools/trace_analyze.py)
    static int seq = 0;
    std::vector<unsigned long long> tr(4 * tasks.size());
    trace.download(tr.data(), tr.size(), s);
    CB_CUDA(cudaStreamSynchronize(s));
    const std::string path = std::string(trace_prefix) + "_" + std::to_string(seq++) + ".bin";
    if (FILE* fp = std::fopen(path.c_str(), "wb")) {
      const int n = (int)tasks.size();
      std::fwrite(&n, sizeof(int), 1, fp);
      std::fwrite(tasks.data(), sizeof(int4), tasks.size(), fp);
      std::fwrite(tr.data(), sizeof(unsigned long long), tr.size(), fp);
      std::fclose(fp);
    }
  }
}

}  // namespace

}  // namespace cutbddc_b200
