// Does a warp slow down while the other warps of its CTA wait at a barrier?
// Warp 0 runs a loop of independent shared loads + FMAs; warps 1-7 wait.
#include <cstdio>
__global__ void k_probe(double* out, long long* cyc, int nwarps_wait) {
  __shared__ double sh[64 * 65];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  for (int i = tid; i < 64 * 65; i += blockDim.x) sh[i] = 1.0 + i * 1e-6;
  __syncthreads();
  double acc = 0;
  if (wid == 0) {
    long long t0 = clock64();
#pragma unroll 1
    for (int j = 0; j < 16; ++j) {
      double v[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = sh[(lane & 15) * 65 + j + k * 65 * 2];
      __syncwarp();
#pragma unroll
      for (int k = 0; k < 8; ++k) acc = fma(acc, 0.5, v[k]);
      sh[(lane & 15) * 65 + 40 + j] = acc;
      __syncwarp();
    }
    long long t1 = clock64();
    if (lane == 0) cyc[0] = t1 - t0;
  }
  __syncthreads();
  out[tid] = acc;
}
int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 256 * 8); cudaMalloc(&cyc, 16);
  for (int threads : {32, 256, 32, 256}) {
    k_probe<<<1, threads>>>(out, cyc, 0);
    long long h;
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("threads %d: warp-0 loop %lld cycles (%.0f per iteration)\n", threads, h, h / 16.0);
  }
  return 0;
}
