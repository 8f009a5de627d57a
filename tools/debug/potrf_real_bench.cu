// Microbenchmark of the dataflow factorisation's POTRF tile task (the exact
// dense_dag.cu code, included): ncta CTAs each factor + invert one 64x64 SPD
// tile; per-CTA time via %globaltimer.
// nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -Ipaper_1703_06323_b200/csrc -Iinclude \
//   -I<nccl include> tools/debug/potrf_real_bench.cu -Lpaper_1703_06323_b200 -lcutbddc
#include "../../paper_1703_06323_b200/csrc/dense_dag.cu"

#include <cstdio>
#include <vector>

namespace cutbddc_b200 {
namespace {
template <typename Fail>
__device__ void potrf_phased(double* F, int ldf, double* P, int ldp, int n, double* sm, Fail fail, unsigned long long* ph) {
  int np_ = 0;
#define STAMP() do { __syncthreads(); if (threadIdx.x == 0) ph[np_] = dag_timer(); ++np_; } while (0)
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
  STAMP();
  for (int b = 0; b < nb; ++b) {
    const int o = 16 * b, m = min(16, n - o), below = n - o - m;
    if (wid == 0) {
      warp_chol16(ls, o, m, lane, fail);
      __syncwarp();
      warp_inv16(ls, xs, o, m, lane);
    }
    STAMP();
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
    STAMP();
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
  STAMP();
  for (int e = tid; e < n * n; e += kDagThreads) {
    const int i = e % n, j = e / n;
    F[i + (int64_t)j * ldf] = i >= j ? ls[i][j] : 0.0;
    P[i + (int64_t)j * ldp] = i >= j ? xs[i][j] : 0.0;
  }
  STAMP();
#undef STAMP
}

__global__ void k_potrf_phases(double* F, double* P, int n, unsigned long long* ph) {
  extern __shared__ double sm[];
  if (threadIdx.x == 0) ph[31] = dag_timer();
  potrf_phased(F, n, P, n, n, sm, [](int) {}, ph);
}

__global__ void __launch_bounds__(kDagThreads, 3) k_potrf_bench(double* F, double* P, int n, unsigned long long* t) {
  extern __shared__ double sm[];
  double* f = F + (size_t)blockIdx.x * n * n;
  double* p = P + (size_t)blockIdx.x * n * n;
  __syncthreads();
  const unsigned long long t0 = dag_timer();
  tile_potrf_inv(f, n, p, n, n, sm, [](int) {});
  __syncthreads();
  if (threadIdx.x == 0) t[blockIdx.x] = dag_timer() - t0;
}
}  // namespace
}  // namespace cutbddc_b200

int main() {
  using namespace cutbddc_b200;
  const int n = 64, maxc = 148 * 3;
  std::vector<double> A((size_t)n * n * maxc);
  for (int c = 0; c < maxc; ++c)
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) A[(size_t)c * n * n + i + j * n] = i == j ? n + 1.0 : 1.0 / (1 + i + j);
  double *F, *P;
  unsigned long long* t;
  cudaMalloc(&F, A.size() * 8);
  cudaMalloc(&P, A.size() * 8);
  cudaMalloc(&t, maxc * 8);
  const size_t shm = sizeof(double) * 2 * kTile * (kTile + 1);
  cudaFuncSetAttribute(k_potrf_bench, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm);
  {
    unsigned long long* ph;
    cudaMalloc(&ph, 32 * 8);
    cudaFuncSetAttribute(k_potrf_phases, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm);
    for (int rep = 0; rep < 3; ++rep) {
      cudaMemcpy(F, A.data(), (size_t)n * n * 8, cudaMemcpyHostToDevice);
      k_potrf_phases<<<1, kDagThreads, shm>>>(F, P, n, ph);
      cudaDeviceSynchronize();
    }
    unsigned long long h[32];
    cudaMemcpy(h, ph, sizeof(h), cudaMemcpyDeviceToHost);
    printf("phases (us from start): load %.2f", (h[0] - h[31]) / 1e3);
    for (int q = 1; q < 14; ++q) printf(" | %.2f", (h[q] - h[31]) / 1e3);
    printf("\n");
  }
  for (int ncta : {1, 148, 296, 444}) {
    std::vector<unsigned long long> ht(ncta);
    for (int rep = 0; rep < 3; ++rep) {
      cudaMemcpy(F, A.data(), A.size() * 8, cudaMemcpyHostToDevice);
      k_potrf_bench<<<ncta, kDagThreads, shm>>>(F, P, n, t);
      cudaDeviceSynchronize();
    }
    cudaMemcpy(ht.data(), t, ncta * 8, cudaMemcpyDeviceToHost);
    double s = 0, mx = 0;
    for (auto v : ht) s += v, mx = std::max(mx, (double)v);
    printf("ctas %4d: potrf+inv 64 mean %.1f us max %.1f us (%s)\n", ncta, s / ncta / 1e3, mx / 1e3,
           cudaGetErrorString(cudaGetLastError()));
  }
}
