#include "element.cu"
#include <cstdio>
#include <vector>
using namespace cutbddc_b200;
struct Q8 { double v[8]; };
__global__ void __launch_bounds__(64) kv2(int n, double h, int64_t ncut, const int64_t* cut_cells, const double* phi, double* ke, double* fe, double* beta, uint8_t* empty) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= ncut) return;
  const int64_t cell = cut_cells[e];
  const int k = (int)(cell % n), j = (int)((cell / n) % n), i = (int)(cell / n / n);
  double* q8 = fe + e * 8;  // stage q8 in global memory
  for (int l = 0; l < 8; ++l) q8[l] = phi[((int64_t)(i + (l & 1)) * (n + 1) + j + ((l >> 1) & 1)) * (n + 1) + k + ((l >> 2) & 1)];
  double qq[8]; for (int l = 0; l < 8; ++l) qq[l] = q8[l];
  cut_element(qq, h, ke + e * 64, fe + e * 8, beta + e, empty + e);
}
__global__ void kv3(int n, double h, int64_t ncut, const int64_t* cut_cells, const double* phi, double* ke, double* fe, double* beta, uint8_t* empty) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= ncut) return;
  const int64_t cell = cut_cells[e];
  const int k = (int)(cell % n), j = (int)((cell / n) % n), i = (int)(cell / n / n);
  double q8[8];
  for (int l = 0; l < 8; ++l) q8[l] = phi[((int64_t)(i + (l & 1)) * (n + 1) + j + ((l >> 1) & 1)) * (n + 1) + k + ((l >> 2) & 1)];
  cut_element(q8, h, ke + e * 64, fe + e * 8, beta + e, empty + e);
}
int main() {
  int n; double h; long long ncut;
  if (scanf("%d %lf %lld", &n, &h, &ncut) != 3) return 1;
  std::vector<long long> cells(ncut);
  for (auto& c : cells) if (scanf("%lld", &c) != 1) return 1;
  size_t nn = (size_t)(n + 1) * (n + 1) * (n + 1);
  std::vector<double> phi(nn);
  for (auto& p : phi) if (scanf("%lf", &p) != 1) return 1;
  double *dphi, *dK, *dF, *db; int64_t* dc; uint8_t* de; int* dg;
  cudaMalloc(&dphi, nn * 8); cudaMalloc(&dK, ncut * 512); cudaMalloc(&dF, ncut * 64); cudaMalloc(&db, ncut * 8);
  cudaMalloc(&de, ncut); cudaMalloc(&dc, ncut * 8); cudaMalloc(&dg, 4); cudaMemset(dg, 0, 4);
  cudaMemcpy(dphi, phi.data(), nn * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dc, cells.data(), ncut * 8, cudaMemcpyHostToDevice);
  for (int variant = 1; variant <= 5; ++variant) {
    cudaMemset(dK, 0, ncut * 512);
    if (variant == 4) cudaDeviceSetLimit(cudaLimitStackSize, 16384);
    if (variant == 1 || variant == 4) k_cut_elements<<<(ncut + 63) / 64, 64>>>(n, h, ncut, dc, dphi, dK, dF, db, de, dg);
    if (variant == 2) kv2<<<(ncut + 63) / 64, 64>>>(n, h, ncut, dc, dphi, dK, dF, db, de);
    if (variant == 3) kv3<<<(ncut + 63) / 64, 64>>>(n, h, ncut, dc, dphi, dK, dF, db, de);
    if (variant == 5) k_cut_elements<<<(ncut + 31) / 32, 32>>>(n, h, ncut, dc, dphi, dK, dF, db, de, dg);
    cudaError_t err = cudaDeviceSynchronize();
    std::vector<double> K(ncut * 64);
    cudaMemcpy(K.data(), dK, ncut * 512, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (long long e = 0; e < ncut; ++e) {
      long long c = cells[e];
      int k = c % n, j = (c / n) % n, i = c / n / n;
      double q8[8];
      for (int l = 0; l < 8; ++l) q8[l] = phi[((size_t)(i + (l & 1)) * (n + 1) + j + ((l >> 1) & 1)) * (n + 1) + k + ((l >> 2) & 1)];
      double Kh[64], Fh[8], bh; uint8_t eh;
      cut_element(q8, h, Kh, Fh, &bh, &eh);
      double er = 0, mx = 0;
      for (int t = 0; t < 64; ++t) { er = fmax(er, fabs(Kh[t] - K[64 * e + t])); mx = fmax(mx, fabs(Kh[t])); }
      if (er > 1e-12 * mx) bad++;
    }
    printf("variant %d: %s bad %d\n", variant, cudaGetErrorString(err), bad);
  }
}
