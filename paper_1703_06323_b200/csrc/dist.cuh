// dist.cuh — distribution of subdomains over ranks, the local dof space,
// the interface exchange and the matrix-free sub-assembled operator
// (dist.cu).
//
// Local dof space of a rank: every dof of its subdomains, numbered segment by
// segment. Segment s (s < nsd) holds the dofs whose lowest-numbered subdomain
// (global id) is local subdomain s, ascending global dof; the ghost segment
// after them holds the local dofs owned by another rank's subdomain. Every
// dof is owned by exactly one rank, so PCG dot products are sums of
// per-subdomain partials, gathered and added in global subdomain order: the
// result is the same bit for bit on 1, 2, 4 or 8 GPUs.
//
// Interface sums (Σ over the subdomain copies of a dof, ascending global
// subdomain) read local copies from slot vectors and remote
// copies from a receive buffer filled by one grouped NCCL send/recv per
// neighbour rank; every rank holding a copy forms the same sum.
#pragma once

#include "handle.cuh"

namespace cutbddc_b200 {

constexpr int kSegThreads = 256;   // block size of every segment kernel (fixed: reductions are bit-reproducible)

// Distribution set by the caller (cutbddc_gpu_set_distribution), or the
// default one-rank distribution of `part` when none was set.
void dist_set(cutbddc_gpu* h, const cutbddc_partition_view* part, const int32_t* rank_of_sd, int rank, int world);
void dist_default(cutbddc_gpu* h, const cutbddc_partition_view* part);
// Local dof space, copy lists and exchange lists (after assembly has
// slot_dof and the global ncount): device kernels, no host loops over dofs.
void build_plan_device(cutbddc_gpu* h);
// Y (slot values) at remote copies -> h->recvbuf: pack (times w when w is not
// null), then the grouped NCCL send/recv. No-op without neighbours.
void iface_exchange(cutbddc_gpu* h, const double* Y, const double* w, const int* skip);
// out[i] = Σ over the copies of local dof i, ascending global subdomain, of
// (w ? w * Y : Y) (remote copies from h->recvbuf). Call iface_exchange first.
// Xs (optional): the sums also land in every local slot copy.
void iface_sum(cutbddc_gpu* h, const double* Y, const double* w, double* out, const int* skip, double* Xs = nullptr);
// In-place all-gather of the per-subdomain partials (stride h->maxloc).
void gather_partials(cutbddc_gpu* h, double* part);
// Coarse staging (bddc.cu): every rank's constraint-row values h->gl
// (stride maxrows) and coarse blocks h->ac_loc (stride maxac), in place.
void gather_rows(cutbddc_gpu* h);
void gather_blocks(cutbddc_gpu* h);
// max over ranks of a status code (0 = OK), host-synchronous
int agree_status(cutbddc_gpu* h, int code);
// Y = A_w X for every local subdomain, matrix-free: one constant Q1 element
// matrix for interior cells, the stored 8x8 matrix of each cut cell, the
// 1/|neigh| diagonal of strong-Dirichlet dofs. Rows: every present slot
// (kSubAll), interface slots only (kSubInterface) or interior slots only
// (kSubInterior); other slots are not written. The input is the slot vector Xslot, or
// the local dof vector xloc gathered through slot_loc when Xslot is null.
enum { kSubAll = 0, kSubInterface = 1, kSubInterior = 2 };
// the operator's copy of the cut-cell matrices: packed upper triangle, SoA
// (36 doubles per cut cell, coalesced by neighbouring slots)
void pack_cut_matrices(cutbddc_gpu* h);
// the operator's row lists (assembly, after the plan)
void build_operator_rows(cutbddc_gpu* h);
void sub_apply(cutbddc_gpu* h, int mode, const double* xloc, const double* Xslot, double* Y, const int* skip);
// Global <-> local vectors at the boundary: gather every local dof; scatter
// the owned ones (segments, not the ghost segment).
void to_local(cutbddc_gpu* h, const double* xglob, double* xloc);
void to_global_owned(cutbddc_gpu* h, const double* xloc, double* xglob);
// Segment kernels run one block per chunk of kChunk local dofs: the chunks
// of a subdomain's segment (its owned dofs), then the ghost chunks. A chunk
// writes its partial; the last chunk of a segment to finish (ticket) adds
// the segment's chunk partials in chunk order into the subdomain's partial.
// Chunks depend only on the segment's length, so the partials are the same
// bits for every world size.
constexpr int kChunk = 256;
inline int seg_grid(const cutbddc_gpu* h) { return (int)h->n_chunks; }

struct SegArgs {
  const int4* chunks;       // per block: (local subdomain or -1 for ghosts, lo, hi, 0)
  const int32_t* seg_chunk; // nsd + 1: first chunk of each segment
  double* cpart;            // per chunk partial
  int* tickets;             // per segment (0 between kernels)
  double* part;             // this rank's subdomain partials (part_all + rank * maxloc)
};
inline SegArgs seg_args(const cutbddc_gpu* h, double* part_all) {
  return SegArgs{h->chunks.p, h->seg_chunk.p, h->cpart.p, h->tickets.p,
                 part_all ? part_all + (int64_t)h->dist_rank * h->maxloc : nullptr};
}

// Range of the calling block; its subdomain (-1: a ghost chunk, no partial).
__device__ inline int seg_range(const SegArgs& a, int& lo, int& hi) {
  const int4 c = a.chunks[blockIdx.x];
  lo = c.y;
  hi = c.z;
  return c.x;
}

// Every thread of a non-ghost chunk calls this with its accumulator.
__device__ inline void seg_commit(const SegArgs& a, int seg, double acc) {
  __shared__ double sh[32];
  __shared__ int last;
  acc = block_sum<kSegThreads>(acc, sh);
  if (threadIdx.x == 0) {
    a.cpart[blockIdx.x] = acc;
    __threadfence();
    const int n = a.seg_chunk[seg + 1] - a.seg_chunk[seg];
    last = atomicAdd(&a.tickets[seg], 1) == n - 1;
  }
  __syncthreads();
  if (last && threadIdx.x == 0) {
    __threadfence();
    double s = 0.0;
    for (int k = a.seg_chunk[seg]; k < a.seg_chunk[seg + 1]; ++k) s += __ldcg(a.cpart + k);
    a.part[seg] = s;
    a.tickets[seg] = 0;
  }
}

// Σ over global subdomains g (ascending, fixed thread mapping and tree) of
// the gathered partial at gpos[g]; every thread gets the total. Identical on
// every rank and for every world size.
__device__ inline double finish_partials(const double* __restrict__ part, const int32_t* __restrict__ gpos, int nsd_g) {
  __shared__ double sh[32];
  __shared__ double tot;
  double v = 0.0;
  for (int g = threadIdx.x; g < nsd_g; g += kSegThreads) v += part[gpos[g]];
  v = block_sum<kSegThreads>(v, sh);
  if (threadIdx.x == 0) tot = v;
  __syncthreads();
  const double t = tot;
  __syncthreads();
  return t;
}

}  // namespace cutbddc_b200
