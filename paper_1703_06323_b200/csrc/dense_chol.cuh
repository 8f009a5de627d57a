// dense_chol.cuh — single-CTA blocked partial Cholesky of a dense front.
//
// F is r x r, column-major with leading dimension r; only the lower triangle
// is read. The first c columns are factorised (F[:, :c] <- [L11; L21]) and
// the trailing lower triangle F[c:, c:] receives the Schur-complement update
// (the multifrontal update matrix). Right-looking, 32-column panels:
//   (a) the 32x32 diagonal block is factorised by warp 0 in shared memory,
//   (b) the panel rows below are solved against it (TRSM, one row per thread),
//   (c) the trailing lower triangle gets the rank-32 update in 64x64 tiles,
//       each thread accumulating a 4x4 register block from shared-memory
//       staged panel slices (the FP64 FMA-bound part).
// Used by the batched front factorisation (factor.cu) and the coarse matrix
// factorisation (bddc.cu). 256 threads per CTA.
#pragma once

#include "dev_common.cuh"

namespace cutbddc_b200 {

struct CholSmem {
  double d[32][33];       // diagonal block
  double pi[32][64];      // panel slice, rows of the output tile (transposed: [t][row])
  double pj[32][64];      // panel slice, cols of the output tile
  double inv_diag[32];
  int bad;
};

// fail_code(j) -> value recorded (atomicMin) when pivot j is not positive.
template <typename FailFn>
__device__ void front_partial_cholesky(double* __restrict__ F, int r, int c, CholSmem& sm, FailFn&& on_fail) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  for (int k = 0; k < c; k += 32) {
    const int nb = min(32, c - k);
    // (a) diagonal block -> shared, factor by warp 0
    for (int q = tid; q < 32 * 32; q += blockDim.x) {
      const int i = q & 31, j = q >> 5;
      sm.d[i][j] = (i < nb && j < nb && i >= j) ? F[(k + i) + (int64_t)(k + j) * r] : 0.0;
    }
    __syncthreads();
    if (wid == 0) {
      for (int j = 0; j < nb; ++j) {
        double djj = sm.d[j][j];
        if (lane == 0 && !(djj > 0.0)) on_fail(k + j);
        if (!(djj > 0.0)) djj = 1.0;
        const double l = sqrt(djj);
        __syncwarp();
        if (lane == j) sm.d[j][j] = l;
        if (lane > j && lane < nb) sm.d[lane][j] /= l;
        __syncwarp();
        // rank-1 update of the remaining block columns l in (j, lane]
        if (lane > j && lane < nb) {
          const double lij = sm.d[lane][j];
          for (int q = j + 1; q <= lane; ++q) sm.d[lane][q] -= lij * sm.d[q][j];
        }
        __syncwarp();
      }
      if (lane < nb) sm.inv_diag[lane] = 1.0 / sm.d[lane][lane];
    }
    __syncthreads();
    for (int q = tid; q < 32 * 32; q += blockDim.x) {
      const int i = q & 31, j = q >> 5;
      if (i < nb && j < nb && i >= j) F[(k + i) + (int64_t)(k + j) * r] = sm.d[i][j];
    }
    // (b) TRSM: rows below the block, x L^T = a
    for (int i = k + nb + tid; i < r; i += blockDim.x) {
      double x[32];
#pragma unroll
      for (int t = 0; t < 32; ++t) x[t] = t < nb ? F[i + (int64_t)(k + t) * r] : 0.0;
#pragma unroll
      for (int t = 0; t < 32; ++t) {
        if (t < nb) {
          double s = x[t];
#pragma unroll
          for (int u = 0; u < t; ++u) s -= x[u] * sm.d[t][u];
          x[t] = s * sm.inv_diag[t];
        }
      }
#pragma unroll
      for (int t = 0; t < 32; ++t)
        if (t < nb) F[i + (int64_t)(k + t) * r] = x[t];
    }
    __syncthreads();
    // (c) trailing lower-triangle update F[k+nb:, k+nb:] -= P P^T, 64x64 tiles
    const int m0 = k + nb;
    const int mt = (r - m0 + 63) / 64;
    const int tx = tid & 15, ty = tid >> 4;  // 16 x 16 threads, 4x4 each
    for (int tj = 0; tj < mt; ++tj) {
      const int j0 = m0 + tj * 64;
      for (int q = tid; q < 32 * 64; q += blockDim.x) {
        const int jj = q & 63, t = q >> 6;
        const int j = j0 + jj;
        sm.pj[t][jj] = (t < nb && j < r) ? F[j + (int64_t)(k + t) * r] : 0.0;
      }
      for (int ti = tj; ti < mt; ++ti) {
        const int i0 = m0 + ti * 64;
        for (int q = tid; q < 32 * 64; q += blockDim.x) {
          const int ii = q & 63, t = q >> 6;
          const int i = i0 + ii;
          sm.pi[t][ii] = (t < nb && i < r) ? F[i + (int64_t)(k + t) * r] : 0.0;
        }
        __syncthreads();
        double acc[4][4];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
        for (int t = 0; t < nb; ++t) {
          double pa[4], pb[4];
#pragma unroll
          for (int a = 0; a < 4; ++a) pa[a] = sm.pi[t][tx + 16 * a];
#pragma unroll
          for (int b = 0; b < 4; ++b) pb[b] = sm.pj[t][ty + 16 * b];
#pragma unroll
          for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) acc[a][b] += pa[a] * pb[b];
        }
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const int j = j0 + ty + 16 * b;
          if (j >= r) continue;
#pragma unroll
          for (int a = 0; a < 4; ++a) {
            const int i = i0 + tx + 16 * a;
            if (i >= r || i < j) continue;
            F[i + (int64_t)j * r] -= acc[a][b];
          }
        }
        __syncthreads();
      }
    }
  }
}

}  // namespace cutbddc_b200
