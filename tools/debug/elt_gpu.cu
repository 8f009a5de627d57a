// Debug harness: run cut_element on host and device for the same inputs.
#include "element.cu"
#include <cstdio>
#include <vector>
__global__ void k_run(int n, const double* q, double h, double* K, double* F, double* beta, uint8_t* e) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) cutbddc_b200::cut_element(q + 8 * i, h, K + 64 * i, F + 8 * i, beta + i, e + i);
}
int main(int argc, char** argv) {
  if (argc > 1) cudaDeviceSetLimit(cudaLimitStackSize, 16384);
  std::vector<double> q;
  double h, v;
  scanf("%lf", &h);
  while (scanf("%lf", &v) == 1) q.push_back(v);
  int n = (int)q.size() / 8;
  double *dq, *dK, *dF, *db; uint8_t* de;
  cudaMalloc(&dq, q.size() * 8); cudaMalloc(&dK, n * 512); cudaMalloc(&dF, n * 64); cudaMalloc(&db, n * 8); cudaMalloc(&de, n);
  cudaMemcpy(dq, q.data(), q.size() * 8, cudaMemcpyHostToDevice);
  k_run<<<(n + 63) / 64, 64>>>(n, dq, h, dK, dF, db, de);
  printf("launch: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  std::vector<double> K(n * 64), F(n * 8), b(n);
  cudaMemcpy(K.data(), dK, n * 512, cudaMemcpyDeviceToHost);
  cudaMemcpy(b.data(), db, n * 8, cudaMemcpyDeviceToHost);
  int bad = 0, exact = 0;
  for (int i = 0; i < n; ++i) {
    double Kh[64], Fh[8], bh; uint8_t eh;
    cutbddc_b200::cut_element(&q[8 * i], h, Kh, Fh, &bh, &eh);
    double err = 0, mx = 0;
    for (int t = 0; t < 64; ++t) { err = fmax(err, fabs(Kh[t] - K[64 * i + t])); mx = fmax(mx, fabs(Kh[t])); }
    if (err > 1e-12 * mx) { if (bad < 3) printf("cell %d host beta %.17g dev beta %.17g err %g\n", i, bh, b[i], err / mx); bad++; }
    bool ex = bh == b[i]; for (int t = 0; t < 64; ++t) ex = ex && Kh[t] == K[64 * i + t]; exact += ex;
  }
  printf("n %d bad %d exact %d\n", n, bad, exact);
}
