// peak.cu — FP64 throughput microbenchmarks (the FP64 roofline denominator;
// MEASURED_PEAKS.json carries only HBM and bf16).
//
// k_peak_dmma: every warp issues independent chains of
//   mma.sync.aligned.m8n8k4.row.col.f64 (512 flops per warp instruction; the
//   hardware instruction DMMA.8x8x4 -- m16n8k16.f64 lowers to 8 of them),
// k_peak_dfma: every thread issues independent DFMA chains (2 flops each).
// Both run one persistent grid of (SMs x 4) CTAs of 256 threads for a fixed
// number of iterations; time by CUDA events, best of 5.
#include <cuda_runtime.h>

#include <algorithm>

#include "cutbddc.h"
#include "dev_common.cuh"

namespace cutbddc_b200 {
namespace {

constexpr int kChains = 8;  // independent accumulators per warp (hides the DMMA latency)

__global__ void __launch_bounds__(256) k_peak_dmma(int iters, double seed, double* out) {
  double a = seed + threadIdx.x * 1e-9, b = seed - threadIdx.x * 1e-9;
  double c[kChains][2];
#pragma unroll
  for (int k = 0; k < kChains; ++k) c[k][0] = c[k][1] = 0.0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < kChains; ++k)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[k][0]), "+d"(c[k][1])
                   : "d"(a), "d"(b));
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < kChains; ++k) s += c[k][0] + c[k][1];
  if (s == 1.2345) out[0] = s;  // keep the chains live
}

__global__ void __launch_bounds__(256) k_peak_dfma(int iters, double seed, double* out) {
  double x[kChains];
  const double a = seed + threadIdx.x * 1e-9, b = 1.0 - 1e-12;
#pragma unroll
  for (int k = 0; k < kChains; ++k) x[k] = a + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < kChains; ++k) x[k] = fma(x[k], b, a);
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < kChains; ++k) s += x[k];
  if (s == 1.2345) out[0] = s;
}

template <typename K>
double time_best(K kern, int grid, int iters, double* out) {
  cudaEvent_t e0, e1;
  CB_CUDA(cudaEventCreate(&e0));
  CB_CUDA(cudaEventCreate(&e1));
  kern<<<grid, 256>>>(iters / 8, 1.0, out);  // warm-up
  CB_LAUNCH();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    CB_CUDA(cudaEventRecord(e0));
    kern<<<grid, 256>>>(iters, 1.0, out);
    CB_LAUNCH();
    CB_CUDA(cudaEventRecord(e1));
    CB_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    CB_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    best = std::min(best, ms);
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return best * 1e-3;
}

}  // namespace

void fp64_peaks(int device, double* dmma_tflops, double* dfma_tflops) {
  CB_CUDA(cudaSetDevice(device));
  int sms = 0;
  CB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  const int grid = sms * 4, iters = 4096;
  DevBuf<double> out;
  out.alloc(1);
  const double warps = grid * 8.0;
  const double t_mma = time_best(k_peak_dmma, grid, iters, out.p);
  *dmma_tflops = warps * iters * kChains * 512.0 / t_mma * 1e-12;
  const double t_fma = time_best(k_peak_dfma, grid, iters, out.p);
  *dfma_tflops = grid * 256.0 * iters * kChains * 2.0 / t_fma * 1e-12;
}

}  // namespace cutbddc_b200
