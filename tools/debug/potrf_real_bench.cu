// Microbenchmark of the dataflow factorisation's POTRF tile task (the exact
// dense_dag.cu code, included): ncta CTAs each factor + invert one 64x64 SPD
// tile; per-CTA time via %globaltimer.
// nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -Ipaper_1703_06323_b200/csrc -Iinclude \
//   -I<nccl include> tools/debug/potrf_real_bench.cu -Lpaper_1703_06323_b200 -lcutbddc
__device__ unsigned long long g_phase[8];
#define POTRF_PHASE(k)                                                         \
  do {                                                                         \
    if (threadIdx.x == 0 && blockIdx.x == 0) {                                 \
      unsigned long long t_;                                                   \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                  \
      g_phase[k] = t_;                                                         \
    }                                                                          \
  } while (0)
#include "../../paper_1703_06323_b200/csrc/dense_dag.cu"

#include <cmath>
#include <cstdio>
#include <vector>

namespace cutbddc_b200 {
namespace {
__global__ void __launch_bounds__(256, 2) k_potrf_phases(double* F, double* P, int n, unsigned long long* ph) {
  extern __shared__ double sm[];
  if (threadIdx.x == 0) ph[31] = dag_timer();
  tile_potrf_inv(F, n, P, n, n, sm, [](int) {});
  __syncthreads();
  if (threadIdx.x == 0) ph[0] = dag_timer();
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
    printf("single CTA: %.2f us\n", (h[0] - h[31]) / 1e3);
    unsigned long long gp[8];
    cudaMemcpyFromSymbol(gp, g_phase, sizeof(gp));
    printf("phases: load %.2f eliminate %.2f store %.2f us\n", (gp[0] - h[31]) / 1e3, (gp[1] - gp[0]) / 1e3,
           (h[0] - gp[1]) / 1e3);
    std::vector<double> L(n * n), X(n * n);
    cudaMemcpy(L.data(), F, n * n * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(X.data(), P, n * n * 8, cudaMemcpyDeviceToHost);
    double e1 = 0, e2 = 0;
    for (int i = 0; i < n; ++i)
      for (int j = 0; j <= i; ++j) {
        double s = 0, t = 0;
        for (int k = 0; k <= j; ++k) s += L[i + k * n] * L[j + k * n];
        for (int k = j; k <= i; ++k) t += X[i + k * n] * L[k + j * n];
        e1 = std::max(e1, std::fabs(s - A[i + j * n]));
        e2 = std::max(e2, std::fabs(t - (i == j ? 1.0 : 0.0)));
      }
    printf("max |LL^T - A| %.3e  max |XL - I| %.3e\n", e1, e2);
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
