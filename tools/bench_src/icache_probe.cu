// Cold straight-line code: cycles per instruction of a long unrolled block
// of independent FP64 adds run once by one warp, and of a small loop.
#include <cstdio>
__global__ void k_probe(double* out, long long* cyc) {
  double v[8];
  for (int i = 0; i < 8; ++i) v[i] = threadIdx.x + i;
  long long t0 = clock64();
#pragma unroll
  for (int i = 0; i < 2048; ++i) v[i & 7] = v[i & 7] * 1.0000001 + 1e-9;
  long long t1 = clock64();
#pragma unroll 1
  for (int r = 0; r < 256; ++r)
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = v[i] * 1.0000001 + 1e-9;
  long long t2 = clock64();
  double s = 0;
  for (int i = 0; i < 8; ++i) s += v[i];
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; }
}
int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 32 * 8); cudaMalloc(&cyc, 16);
  for (int r = 0; r < 3; ++r) {
    k_probe<<<1, 32>>>(out, cyc);
    long long h[2];
    cudaMemcpy(h, cyc, 16, cudaMemcpyDeviceToHost);
    printf("2048 unrolled dfma: %lld cycles (%.1f/instr) | same work in a loop: %lld cycles (%.1f/instr)\n", h[0],
           h[0] / 2048.0, h[1], h[1] / 2048.0);
  }
  return 0;
}
