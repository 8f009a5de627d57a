// Microbenchmark of the diagonal-tile POTRF + inverse (dense_dag.cu
// tile_potrf_inv) on one CTA: clock64 stamps at its phase boundaries.
// Build: tools/bench_src/build_potrf_bench.sh; run on the GPU box.
#include <cstdio>
#include <vector>
#include <cmath>
__device__ long long g_stamp[40];
#define POTRF_STAMP(k) do { __syncthreads(); if (threadIdx.x == 0) g_stamp[(k)] = clock64(); } while (0)
#include "../../paper_1703_06323_b200/csrc/dense_dag.cu"

namespace cutbddc_b200 {
namespace {
__global__ void __launch_bounds__(kDagThreads, 3) k_bench(double* F, double* P, const double* A0, int n, int reps,
                                                           long long* out) {
  extern __shared__ double sm[];
  for (int r = 0; r < reps; ++r) {
    for (int e = threadIdx.x; e < 64 * 64; e += blockDim.x) F[e] = A0[e];
    __syncthreads();
    const long long t0 = clock64();
    tile_potrf_inv(F, 64, P, 64, n, sm, [&](int) {});
    __syncthreads();
    if (threadIdx.x == 0) {
      out[r] = clock64() - t0;
      for (int k = 0; k < 40; ++k) out[reps + r * 40 + k] = g_stamp[k] - t0;
    }
  }
}
}  // namespace
}  // namespace cutbddc_b200

int main() {
  using namespace cutbddc_b200;
  const int n = 64, reps = 5;
  std::vector<double> a(64 * 64, 0.0);
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) a[i + 64 * j] = (i == j ? n + 1.0 : 1.0 / (1.0 + std::abs(i - j)));
  double *F, *P, *A0;
  long long* out;
  cudaMalloc(&F, 8 * 4096);
  cudaMalloc(&P, 8 * 4096);
  cudaMalloc(&A0, 8 * 4096);
  cudaMalloc(&out, 8 * (reps + reps * 40));
  cudaMemcpy(A0, a.data(), 8 * 4096, cudaMemcpyHostToDevice);
  const int shm = 2 * 64 * 65 * 8 + 4096;
  cudaFuncSetAttribute(k_bench, cudaFuncAttributeMaxDynamicSharedMemorySize, shm);
  k_bench<<<1, kDagThreads, shm>>>(F, P, A0, n, reps, out);
  std::vector<long long> h(reps + reps * 40);
  cudaMemcpy(h.data(), out, 8 * h.size(), cudaMemcpyDeviceToHost);
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  for (int r = 0; r < reps; ++r) {
    printf("rep %d total %lld cycles | stamps:", r, h[r]);
    for (int k = 0; k < 16; ++k) printf(" %lld", h[reps + r * 40 + k]);
    printf("\n");
  }
  return 0;
}
