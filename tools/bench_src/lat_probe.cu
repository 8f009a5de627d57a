// Latency probes (cycles per step): dependent DFMA chain, shared
// load -> DFMA -> store chain, double shuffle chain, double rsqrt chain.
#include <cstdio>
__global__ void k_probe(double* out, double seed, long long* cyc) {
  __shared__ double sh[1024];
  const int lane = threadIdx.x;
  for (int i = lane; i < 1024; i += 32) sh[i] = seed + i;
  __syncwarp();
  double x = seed + lane;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1000; ++i) x = fma(x, 0.999999, 1e-7);
  long long t1 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1000; ++i) { sh[lane * 17 % 1024] -= x * sh[(i & 511) + 1]; }
  long long t2 = clock64();
  double y = x;
#pragma unroll 1
  for (int i = 0; i < 1000; ++i) y = __shfl_sync(0xffffffffu, y, (lane + 1) & 31);
  long long t3 = clock64();
  double z = 1.0 + x * 1e-9;
#pragma unroll 1
  for (int i = 0; i < 1000; ++i) z = rsqrt(z) + 0.5;
  long long t4 = clock64();
  double w = x;
#pragma unroll 1
  for (int i = 0; i < 1000; ++i) w = w * 1.0000001;
  long long t5 = clock64();
  out[lane] = x + sh[lane] + y + z + w;
  if (lane == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4; }
}
int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 32 * 8); cudaMalloc(&cyc, 8 * 8);
  for (int r = 0; r < 3; ++r) {
    k_probe<<<1, 32>>>(out, 1.0, cyc);
    long long h[5];
    cudaMemcpy(h, cyc, 40, cudaMemcpyDeviceToHost);
    printf("per step cycles: dfma %.1f  lds-dfma-sts %.1f  shfl.f64 %.1f  rsqrt.f64+add %.1f  dmul %.1f\n", h[0] / 1e3,
           h[1] / 1e3, h[2] / 1e3, h[3] / 1e3, h[4] / 1e3);
  }
  return 0;
}
