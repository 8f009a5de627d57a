// front_asm.cuh — assembly of one front in gather form (device helpers of
// the dataflow factorisation, dense_dag.cu).
//
// Entry (i, j), i >= j, of the compact front of (subdomain sd, supernode s):
//   F_ij = U0[m0(i), m0(j)] + U1[m1(i), m1(j)]            (children's updates)
//        + A(slot_i, slot_j)  if j < c and the slots are stencil neighbours
// m0 / m1: the row of child 0 / 1's update block landing on front row i
// (-1: none; the sweep plan's gmap). Each update block is read in lower
// storage. The original entries follow the assembly rule of the template
// (nd_template.cpp: the lower entries of A in column u belong to the front
// eliminating u, and a stencil neighbour eliminated later is a row of that
// front), evaluated per entry instead of scattered from a map: every entry
// is written once, no zero pass, no read-modify-write.
#pragma once

#include "factor.cuh"

namespace cutbddc_b200 {

// Per compact front row: children's update rows, local slot and packed
// lattice coordinates (x << 20 | y << 10 | z).
struct RowInfo {
  int m0, m1, slot, xyz;
};

struct ChildBlocks {
  const double* u0;  // top-left entry of child 0's update block (nullptr: none)
  const double* u1;
  int ld0, ld1;
};

__device__ __forceinline__ RowInfo row_info(const FactorDev& f, const FrontDesc& d, int sd, int T, int b1, int i) {
  const int2 g = f.gmap[d.vo + i];
  const int u = f.cslot[d.vo + i] - sd * T;
  const int x = u / (b1 * b1), y = (u / b1) % b1, z = u % b1;
  return RowInfo{g.x >= 0 ? (int)(g.x - d.cuo0) : -1, g.y >= 0 ? (int)(g.y - d.cuo1) : -1, u,
                 (x << 20) | (y << 10) | z};
}

// Original entry A(v, u) of the stencil (v = row slot, u = column slot), or 0
// when v is not one of u's 27 neighbours.
__device__ __forceinline__ double stencil_entry(const FactorInput& in, int sd, const RowInfo& v, const RowInfo& u) {
  const int dx = (v.xyz >> 20) - (u.xyz >> 20), dy = ((v.xyz >> 10) & 1023) - ((u.xyz >> 10) & 1023),
            dz = (v.xyz & 1023) - (u.xyz & 1023);
  if (dx < -1 || dx > 1 || dy < -1 || dy > 1 || dz < -1 || dz > 1) return 0.0;
  const int k = (dx + 1) * 9 + (dy + 1) * 3 + (dz + 1);
  double a = in.As[(int64_t)sd * 27 * in.T + (int64_t)k * in.T + u.slot];
  if (k == 13 && in.diag_add) a += in.diag_add[(int64_t)sd * in.T + u.slot];
  return a;
}

// Lower entries of rows [i0, i1) x cols [j0, j1) of the front F (leading
// dimension ld, c pivot columns); ri / rj: row info of those rows / cols
// (ri[i - i0], rj[j - j0]). Four entries per thread per pass, loads before
// stores (independent loads in flight).
__device__ __forceinline__ void assemble_block(double* __restrict__ F, int ld, int c, int i0, int i1, int j0, int j1,
                                               const RowInfo* ri, const RowInfo* rj, const ChildBlocks& cb,
                                               const FactorInput& in, int sd) {
  const int h = i1 - i0, n = h * (j1 - j0);
#ifndef CUTBDDC_ASM_BATCH
#define CUTBDDC_ASM_BATCH 4
#endif
  constexpr int kB = CUTBDDC_ASM_BATCH;
  for (int q0 = threadIdx.x; q0 < n; q0 += kB * blockDim.x) {
    double v[kB];
#pragma unroll
    for (int u = 0; u < kB; ++u) {
      const int q = q0 + u * blockDim.x, jj = q / h, ii = q - jj * h;
      double s = 0.0;
      if (q < n && i0 + ii >= j0 + jj) {
        const RowInfo a = ri[ii], b = rj[jj];
        if (a.m0 >= 0 && b.m0 >= 0) s = cb.u0[max(a.m0, b.m0) + (int64_t)min(a.m0, b.m0) * cb.ld0];
        if (a.m1 >= 0 && b.m1 >= 0) s += cb.u1[max(a.m1, b.m1) + (int64_t)min(a.m1, b.m1) * cb.ld1];
        if (j0 + jj < c) s += stencil_entry(in, sd, a, b);
      }
      v[u] = s;
    }
#pragma unroll
    for (int u = 0; u < kB; ++u) {
      const int q = q0 + u * blockDim.x, jj = q / h, ii = q - jj * h;
      if (q < n && i0 + ii >= j0 + jj) F[(i0 + ii) + (int64_t)(j0 + jj) * ld] = v[u];
    }
  }
}

}  // namespace cutbddc_b200
