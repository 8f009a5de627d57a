#include "element.cu"
#include <cstdio>
#include <vector>
using namespace cutbddc_b200;
int main() {
  int n; double h; long long ncut;
  if (scanf("%d %lf %lld", &n, &h, &ncut) != 3) return 1;
  std::vector<long long> cells(ncut);
  for (auto& c : cells) if (scanf("%lld", &c) != 1) return 1;
  size_t nn = (size_t)(n + 1) * (n + 1) * (n + 1);
  std::vector<double> phi(nn);
  for (auto& p : phi) if (scanf("%lf", &p) != 1) return 1;
  double *dphi, *dK, *dF, *db, *dq; int64_t* dc; uint8_t* de; int* dg;
  cudaMalloc(&dphi, nn * 8); cudaMalloc(&dK, ncut * 512); cudaMalloc(&dF, ncut * 64); cudaMalloc(&db, ncut * 8);
  cudaMalloc(&de, ncut); cudaMalloc(&dc, ncut * 8); cudaMalloc(&dg, 4); cudaMemset(dg, 0, 4); cudaMalloc(&dq, ncut * 64);
  cudaMemcpy(dphi, phi.data(), nn * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dc, cells.data(), ncut * 8, cudaMemcpyHostToDevice);
  k_gather_q8<<<(ncut + 255) / 256, 256>>>(n, ncut, dc, dphi, dq);
  k_cut_elements<<<(ncut + 63) / 64, 64>>>(h, ncut, dq, dK, dF, db, de, dg);
  cudaError_t err = cudaDeviceSynchronize();
  std::vector<double> K(ncut * 64);
  cudaMemcpy(K.data(), dK, ncut * 512, cudaMemcpyDeviceToHost);
  int bad = 0, exact = 0;
  for (long long e = 0; e < ncut; ++e) {
    long long c = cells[e];
    int k = c % n, j = (c / n) % n, i = c / n / n;
    std::vector<double> q8(8);
    for (int l = 0; l < 8; ++l) q8[l] = phi[((size_t)(i + (l & 1)) * (n + 1) + j + ((l >> 1) & 1)) * (n + 1) + k + ((l >> 2) & 1)];
    double Kh[64], Fh[8], bh; uint8_t eh;
    cut_element(q8.data(), h, Kh, Fh, &bh, &eh);
    double er = 0, mx = 0; bool ex = true;
    for (int t = 0; t < 64; ++t) { er = fmax(er, fabs(Kh[t] - K[64 * e + t])); mx = fmax(mx, fabs(Kh[t])); ex = ex && Kh[t] == K[64*e+t]; }
    if (er > 1e-12 * mx) bad++;
    exact += ex;
  }
  printf("%s bad %d exact %d of %lld\n", cudaGetErrorString(err), bad, exact, ncut);
}
