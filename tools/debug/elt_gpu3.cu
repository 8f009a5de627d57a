#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>
__global__ void k_q8(int n, int64_t ncut, const int64_t* __restrict__ cut_cells, const double* __restrict__ phi, double* out) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= ncut) return;
  const int64_t cell = cut_cells[e];
  const int k = (int)(cell % n), j = (int)((cell / n) % n), i = (int)(cell / n / n);
  for (int l = 0; l < 8; ++l)
    out[e * 8 + l] = phi[((int64_t)(i + (l & 1)) * (n + 1) + j + ((l >> 1) & 1)) * (n + 1) + k + ((l >> 2) & 1)];
}
int main() {
  int n; double h; long long ncut;
  scanf("%d %lf %lld", &n, &h, &ncut);
  std::vector<long long> cells(ncut);
  for (auto& c : cells) scanf("%lld", &c);
  size_t nn = (size_t)(n + 1) * (n + 1) * (n + 1);
  std::vector<double> phi(nn);
  for (auto& p : phi) scanf("%lf", &p);
  double *dphi, *dout; int64_t* dc;
  cudaMalloc(&dphi, nn * 8); cudaMalloc(&dout, ncut * 64); cudaMalloc(&dc, ncut * 8);
  cudaMemcpy(dphi, phi.data(), nn * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dc, cells.data(), ncut * 8, cudaMemcpyHostToDevice);
  k_q8<<<(ncut + 63) / 64, 64>>>(n, ncut, dc, dphi, dout);
  std::vector<double> o(ncut * 8);
  cudaMemcpy(o.data(), dout, ncut * 64, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (long long e = 0; e < ncut; ++e) {
    long long c = cells[e];
    int k = c % n, j = (c / n) % n, i = c / n / n;
    for (int l = 0; l < 8; ++l) {
      double q = phi[((size_t)(i + (l & 1)) * (n + 1) + j + ((l >> 1) & 1)) * (n + 1) + k + ((l >> 2) & 1)];
      if (q != o[e * 8 + l]) { if (bad < 5) printf("e %lld l %d host %g dev %g\n", e, l, q, o[e*8+l]); bad++; }
    }
  }
  printf("bad %d\n", bad);
}
