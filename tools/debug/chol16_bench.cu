// Microbenchmark: variants of the register-resident 16x16 warp Cholesky
// (dense_dag.cu warp_chol16), one warp, cycles via clock64.
#include <cstdio>
#include <vector>
constexpr int kTile = 64;
typedef double SmTile[kTile + 1];
__device__ long long g_cyc[8];
__device__ unsigned long long g_fail;

template <int V>
__device__ void chol16(SmTile* ls, int o, int m, int lane) {
  double a[16];
#pragma unroll
  for (int q = 0; q < 16; ++q) a[q] = (lane < m && q <= lane) ? ls[o + lane][o + q] : 0.0;
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    if (j < m) {
      double djj = __shfl_sync(0xffffffffu, a[j], j);
      if (V != 2 && !(djj > 0.0)) {
        if (lane == 0) atomicMin(&g_fail, (unsigned long long)(o + j));
        djj = 1.0;
      }
      double rl, l;
      if (V == 1) {
        l = sqrt(djj);
        rl = 1.0 / l;
      } else {
        rl = rsqrt(djj);
        l = djj * rl;
      }
      if (lane == j) {
        a[j] = l;
        if (V != 3) ls[o + j][kTile] = rl;
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

template <int V>
__global__ void k_bench(const double* A, int m) {
  __shared__ SmTile ls[kTile];
  const int lane = threadIdx.x;
  for (int e = lane; e < 16 * 16; e += 32) ls[e & 15][e >> 4] = A[e];
  __syncwarp();
  long long t0 = clock64();
  chol16<V>(ls, 0, m, lane);
  __syncwarp();
  long long t1 = clock64();
  if (lane == 0) g_cyc[V] = t1 - t0;
}

int main() {
  std::vector<double> A(256);
  for (int i = 0; i < 16; ++i)
    for (int j = 0; j < 16; ++j) A[i + 16 * j] = i == j ? 17.0 : 1.0 / (1 + i + j);
  double* d;
  cudaMalloc(&d, 256 * 8);
  cudaMemcpy(d, A.data(), 256 * 8, cudaMemcpyHostToDevice);
  for (int rep = 0; rep < 3; ++rep) {
    k_bench<0><<<1, 32>>>(d, 16);
    k_bench<1><<<1, 32>>>(d, 16);
    k_bench<2><<<1, 32>>>(d, 16);
    k_bench<3><<<1, 32>>>(d, 16);
    cudaDeviceSynchronize();
  }
  long long c[8];
  cudaMemcpyFromSymbol(c, g_cyc, sizeof(c));
  printf("chol16 cycles: current %lld | sqrt+div %lld | no fail check %lld | no rl store %lld (%s)\n", c[0], c[1], c[2],
         c[3], cudaGetErrorString(cudaGetLastError()));
}
