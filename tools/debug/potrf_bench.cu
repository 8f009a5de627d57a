// Microbenchmark of the dense DAG POTRF tile kernel (phases via clock64).
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <vector>
constexpr int kTile = 64;
constexpr int kDagThreads = 256;
__device__ long long g_stamp[8];
__device__ long long g_ph[64];
#define PH(k) do { __syncthreads(); if (threadIdx.x == 0) g_ph[k] = clock64(); } while (0)
#define STAMP(k) do { __syncthreads(); if (threadIdx.x == 0) g_stamp[k] = clock64(); } while (0)
#define STAMP_W(k) do { if (threadIdx.x == 0) g_stamp[k] = clock64(); } while (0)
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
    PH(b * 4 + 0);
    if (wid == 0) {
      warp_chol16(ls, o, m, lane, fail);
      __syncwarp();
      if (lane == 0) g_ph[b * 4 + 1] = clock64();
      warp_inv16(ls, xs, o, m, lane);
    }
    __syncthreads();
    PH(b * 4 + 2);
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
  PH(20);
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
  PH(21);
  for (int e = tid; e < n * n; e += kDagThreads) {
    const int i = e % n, j = e / n;
    F[i + (int64_t)j * ldf] = i >= j ? ls[i][j] : 0.0;
    P[i + (int64_t)j * ldp] = i >= j ? xs[i][j] : 0.0;
  }
}

__global__ void k_bench(double* F, double* P, int n) {
  extern __shared__ double sm[];
  if (threadIdx.x == 0) g_stamp[0] = clock64();
  tile_potrf_inv(F, n, P, n, n, sm, [](int) {});
  __syncthreads();
  if (threadIdx.x == 0) g_stamp[6] = clock64();
}
int main() {
  const int n = 64;
  std::vector<double> A(n * n);
  for (int i = 0; i < n; ++i) for (int j = 0; j < n; ++j) A[i + j * n] = (i == j ? n + 1.0 : 1.0 / (1 + i + j));
  double *F, *P; cudaMalloc(&F, 8 * n * n); cudaMalloc(&P, 8 * n * n);
  const size_t shm = sizeof(double) * 2 * kTile * (kTile + 1);
  cudaFuncSetAttribute(k_bench, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm);
  for (int rep = 0; rep < 3; ++rep) {
    cudaMemcpy(F, A.data(), 8 * n * n, cudaMemcpyHostToDevice);
    k_bench<<<1, kDagThreads, shm>>>(F, P, n);
    cudaDeviceSynchronize();
  }
  long long st[8]; cudaMemcpyFromSymbol(st, g_stamp, sizeof(st));
  const char* names[] = {"load", "chol11", "inv11", "L21+syrk", "chol22+inv22+X21", "store"};
  int idx[] = {0, 1, 2, 3, 4, 5, 6};
  long long ph[64]; cudaMemcpyFromSymbol(ph, g_ph, sizeof(ph));
  for (int b = 0; b < 4; ++b) printf("block %d: chol %lld inv %lld trsm+syrk %lld\n", b, ph[b*4+1]-ph[b*4], ph[b*4+2]-ph[b*4+1], (b < 3 ? ph[(b+1)*4] : ph[20]) - ph[b*4+2]);
  printf("offdiag inverse %lld store %lld\n", ph[21]-ph[20], st[6]-ph[21]);
  printf("potrf+inv total cycles %lld (err %s)\n", st[6]-st[0], cudaGetErrorString(cudaGetLastError()));
  // check L L^T = A and P L = I
  std::vector<double> L(n*n), X(n*n); cudaMemcpy(L.data(), F, 8*n*n, cudaMemcpyDeviceToHost); cudaMemcpy(X.data(), P, 8*n*n, cudaMemcpyDeviceToHost);
  double e1 = 0, e2 = 0;
  for (int i = 0; i < n; ++i) for (int j = 0; j <= i; ++j) { double s = 0; for (int k = 0; k <= j; ++k) s += L[i + k*n] * L[j + k*n]; e1 = fmax(e1, fabs(s - A[i + j*n])); }
  for (int i = 0; i < n; ++i) for (int j = 0; j < n; ++j) { double s = 0; for (int k = 0; k < n; ++k) s += X[i + k*n] * L[k + j*n]; e2 = fmax(e2, fabs(s - (i==j))); }
  printf("max |LL^T - A| %.3e  max |XL - I| %.3e\n", e1, e2);
}
