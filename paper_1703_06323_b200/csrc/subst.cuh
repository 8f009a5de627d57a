// subst.cuh — blocked triangular substitution on a dense column-major panel
// [L11; L21] (r x c, lower), executed by one CTA with the right-hand side in
// shared memory. 32-column diagonal blocks are solved by warp 0 from
// registers / a shared tile; the remaining panel rows are applied as
// coalesced GEMV updates by the whole CTA. Used by the multifrontal solves
// (factor.cu) and the coarse solve (bddc.cu).
#pragma once

#include "dev_common.cuh"

namespace cutbddc_b200 {

// v[0:c) <- L11^{-1} v[0:c);  v[c:r) <- v[c:r) - L21 v[0:c)
__device__ inline void panel_forward(const double* __restrict__ P, int r, int c, double* v) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int jb = 0; jb < c; jb += 32) {
    const int nb = min(32, c - jb);
    if (wid == 0) {
      double lr[32];
#pragma unroll
      for (int k = 0; k < 32; ++k) lr[k] = (k < nb && lane < nb) ? P[(jb + lane) + (int64_t)(jb + k) * r] : 0.0;
      double y = lane < nb ? v[jb + lane] : 0.0;
#pragma unroll
      for (int k = 0; k < 32; ++k) {
        if (k < nb) {
          if (lane == k) y = y / lr[k];
          const double yk = __shfl_sync(0xffffffffu, y, k);
          if (lane > k) y -= lr[k] * yk;
        }
      }
      if (lane < nb) v[jb + lane] = y;
    }
    __syncthreads();
    for (int i = jb + nb + threadIdx.x; i < r; i += blockDim.x) {
      double s0 = 0.0, s1 = 0.0;
      int k = 0;
      for (; k + 2 <= nb; k += 2) {
        s0 += P[i + (int64_t)(jb + k) * r] * v[jb + k];
        s1 += P[i + (int64_t)(jb + k + 1) * r] * v[jb + k + 1];
      }
      if (k < nb) s0 += P[i + (int64_t)(jb + k) * r] * v[jb + k];
      v[i] -= s0 + s1;
    }
    __syncthreads();
  }
}

// w[0:c) <- L11^{-T} (w[0:c) - L21^T w[c:r)); w[c:r) holds known values.
// tile: 32 x 33 shared scratch.
__device__ inline void panel_backward(const double* __restrict__ P, int r, int c, double* w, double (*tile)[33]) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int last = ((c - 1) / 32) * 32;
  for (int jb = last; jb >= 0; jb -= 32) {
    const int nb = min(32, c - jb);
    for (int jj = wid; jj < nb; jj += nw) {
      const double* col = P + (int64_t)(jb + jj) * r;
      double s = 0.0;
      for (int i = jb + nb + lane; i < r; i += 32) s += col[i] * w[i];
      s = warp_sum(s);
      if (lane == 0) w[jb + jj] -= s;
    }
    for (int q = threadIdx.x; q < 32 * 32; q += blockDim.x) {
      const int k = q & 31, j = q >> 5;
      tile[k][j] = (k < nb && j < nb) ? P[(jb + k) + (int64_t)(jb + j) * r] : 0.0;
    }
    __syncthreads();
    if (wid == 0) {
      double xv = lane < nb ? w[jb + lane] : 0.0;
#pragma unroll
      for (int k = 31; k >= 0; --k) {
        if (k < nb) {
          if (lane == k) xv = xv / tile[k][k];
          const double xk = __shfl_sync(0xffffffffu, xv, k);
          if (lane < k) xv -= tile[k][lane] * xk;
        }
      }
      if (lane < nb) w[jb + lane] = xv;
    }
    __syncthreads();
  }
}

}  // namespace cutbddc_b200
