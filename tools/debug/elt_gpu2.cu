// Debug harness 2: launch the library's own k_cut_elements on oracle phi.
#include "element.cu"
#include <cstdio>
#include <vector>
int main() {
  int n; double h; long long ncut;
  scanf("%d %lf %lld", &n, &h, &ncut);
  std::vector<long long> cells(ncut);
  for (auto& c : cells) scanf("%lld", &c);
  size_t nn = (size_t)(n + 1) * (n + 1) * (n + 1);
  std::vector<double> phi(nn);
  for (auto& p : phi) scanf("%lf", &p);
  double *dphi, *dK, *dF, *db; int64_t* dc; uint8_t* de; int* dg;
  cudaMalloc(&dphi, nn * 8); cudaMalloc(&dK, ncut * 512); cudaMalloc(&dF, ncut * 64); cudaMalloc(&db, ncut * 8);
  cudaMalloc(&de, ncut); cudaMalloc(&dc, ncut * 8); cudaMalloc(&dg, 4); cudaMemset(dg, 0, 4);
  cudaMemcpy(dphi, phi.data(), nn * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dc, cells.data(), ncut * 8, cudaMemcpyHostToDevice);
  cutbddc_b200::k_cut_elements<<<(ncut + 63) / 64, 64>>>(n, h, ncut, dc, dphi, dK, dF, db, de, dg);
  printf("launch: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  std::vector<double> K(ncut * 64);
  cudaMemcpy(K.data(), dK, ncut * 512, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (long long e = 0; e < ncut; ++e) {
    long long c = cells[e];
    int k = c % n, j = (c / n) % n, i = c / n / n;
    double q8[8];
    for (int l = 0; l < 8; ++l) q8[l] = phi[((size_t)(i + (l & 1)) * (n + 1) + j + ((l >> 1) & 1)) * (n + 1) + k + ((l >> 2) & 1)];
    double Kh[64], Fh[8], bh; uint8_t eh;
    cutbddc_b200::cut_element(q8, h, Kh, Fh, &bh, &eh);
    double err = 0, mx = 0;
    for (int t = 0; t < 64; ++t) { err = fmax(err, fabs(Kh[t] - K[64 * e + t])); mx = fmax(mx, fabs(Kh[t])); }
    if (err > 1e-12 * mx) bad++;
  }
  printf("ncut %lld bad %d\n", ncut, bad);
}
