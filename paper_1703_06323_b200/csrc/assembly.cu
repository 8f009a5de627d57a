// assembly.cu — sub-assembled subdomain matrices and the global operator (K3).
//
// assemble_subassembled and assemble_global
// as deterministic gathers: every (row, 27-stencil column) entry sums the
// element contributions of the <= 8 active cells around the row node in
// ascending cell id, the same order the CPU restatement's triplet merge
// uses (linalg.cpp:12-32 semantics), so no fp64 atomics are involved.
// Strong-Dirichlet (orphan) dofs: all incident active cells empty ->
// identity row in Abar, 1/|neigh| diagonal in every A^w.
#include <cub/cub.cuh>

#include "handle.cuh"

namespace cutbddc_b200 {

void cut_elements_device(cutbddc_gpu* h);
void interior_element_device(cutbddc_gpu* h, double* kint, double* fint);

namespace {

__global__ void k_cell_flags(int64_t nc, const uint8_t* __restrict__ cls, uint8_t* __restrict__ act,
                             uint8_t* __restrict__ cut) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < nc; c += (int64_t)gridDim.x * blockDim.x) {
    act[c] = cls[c] != CUTBDDC_EXTERIOR;
    cut[c] = cls[c] == CUTBDDC_CUT;
  }
}

__global__ void k_elem_of_cell(int64_t nc, const uint8_t* __restrict__ cls, int32_t* __restrict__ eoc) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < nc; c += (int64_t)gridDim.x * blockDim.x)
    eoc[c] = cls[c] == CUTBDDC_EXTERIOR ? -2 : -1;
}

__global__ void k_scatter_cut(int64_t ncut, const int64_t* __restrict__ cut_cells, int32_t* __restrict__ eoc) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e < ncut) eoc[cut_cells[e]] = (int32_t)e;
}

__global__ void k_sd_of_block(int nsd, const int64_t* __restrict__ bids, int32_t* __restrict__ sob) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s < nsd) sob[bids[s]] = s;
}

struct MeshArgs {
  int n, B, nb, T;
  const int32_t* eoc;
  const int32_t* dof_of_node;
  const int64_t* node_of_dof;
  const double* ke;
  const double* fe;
  const uint8_t* empty;
  const double* kint;
  const double* fint;
  const int32_t* sd_of_block;
};

// Element matrix of an active cell (cut: stored; interior: constant); null if
// the cell contributes nothing (exterior or empty cut cell).
__device__ inline const double* elem_k(const MeshArgs& m, int64_t cell, const double** f) {
  const int32_t e = m.eoc[cell];
  if (e == -2) return nullptr;
  if (e == -1) {
    *f = m.fint;
    return m.kint;
  }
  if (m.empty[e]) return nullptr;
  *f = m.fe + (int64_t)e * 8;
  return m.ke + (int64_t)e * 64;
}

// per dof: |neigh| (distinct blocks among incident active cells), how many of
// them are this handle's subdomains, orphan flag
__global__ void k_dof_info(int64_t ndof, MeshArgs m, uint8_t* __restrict__ ncount, uint8_t* __restrict__ lcount,
                           uint8_t* __restrict__ orphan) {
  const int64_t d = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (d >= ndof) return;
  const int n = m.n;
  const int64_t v = m.node_of_dof[d];
  const int k = (int)(v % (n + 1)), j = (int)((v / (n + 1)) % (n + 1)), i = (int)(v / (n + 1) / (n + 1));
  int64_t blks[8];
  int nbk = 0;
  bool nonvoid = false;
  for (int dx = 0; dx < 2; ++dx)
    for (int dy = 0; dy < 2; ++dy)
      for (int dz = 0; dz < 2; ++dz) {
        const int ci = i - 1 + dx, cj = j - 1 + dy, ck = k - 1 + dz;
        if (ci < 0 || cj < 0 || ck < 0 || ci >= n || cj >= n || ck >= n) continue;
        const int64_t cell = ((int64_t)ci * n + cj) * n + ck;
        const int32_t e = m.eoc[cell];
        if (e == -2) continue;
        if (e == -1 || !m.empty[e]) nonvoid = true;
        const int64_t bid = ((int64_t)(ci / m.B) * m.nb + cj / m.B) * m.nb + ck / m.B;
        bool seen = false;
        for (int q = 0; q < nbk; ++q) seen |= blks[q] == bid;
        if (!seen) blks[nbk++] = bid;
      }
  int nloc = 0;
  for (int q = 0; q < nbk; ++q) nloc += m.sd_of_block[blks[q]] >= 0;
  ncount[d] = (uint8_t)nbk;
  lcount[d] = (uint8_t)nloc;
  orphan[d] = !nonvoid;
}

// Abar as ELL-27 (SoA): row = dof; column k = node + stencil offset.
__global__ void k_abar(int64_t ndof, MeshArgs m, const uint8_t* __restrict__ orphan, double* __restrict__ aval,
                       int32_t* __restrict__ acol, double* __restrict__ b) {
  const int64_t d = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (d >= ndof) return;
  const int n = m.n;
  const int64_t v = m.node_of_dof[d];
  const int k = (int)(v % (n + 1)), j = (int)((v / (n + 1)) % (n + 1)), i = (int)(v / (n + 1) / (n + 1));
  double acc[27];
#pragma unroll
  for (int q = 0; q < 27; ++q) acc[q] = 0.0;
  double bb = 0.0;
  for (int dx = 0; dx < 2; ++dx)
    for (int dy = 0; dy < 2; ++dy)
      for (int dz = 0; dz < 2; ++dz) {
        const int ci = i - 1 + dx, cj = j - 1 + dy, ck = k - 1 + dz;
        if (ci < 0 || cj < 0 || ck < 0 || ci >= n || cj >= n || ck >= n) continue;
        const double* f = nullptr;
        const double* K = elem_k(m, ((int64_t)ci * n + cj) * n + ck, &f);
        if (!K) continue;
        const int lv = (1 - dx) + 2 * (1 - dy) + 4 * (1 - dz);
        bb += f[lv];
#pragma unroll
        for (int w = 0; w < 8; ++w) {
          const int q = stencil_k((w & 1) - (lv & 1), ((w >> 1) & 1) - ((lv >> 1) & 1), ((w >> 2) & 1) - ((lv >> 2) & 1));
          acc[q] += K[lv * 8 + w];
        }
      }
  if (orphan[d]) {
#pragma unroll
    for (int q = 0; q < 27; ++q) acc[q] = 0.0;
    acc[13] = 1.0;
    bb = 0.0;
  }
#pragma unroll
  for (int q = 0; q < 27; ++q) {
    const int ii = i + q / 9 - 1, jj = j + (q / 3) % 3 - 1, kk = k + q % 3 - 1;
    int32_t col = -1;
    if (ii >= 0 && jj >= 0 && kk >= 0 && ii <= n && jj <= n && kk <= n)
      col = m.dof_of_node[((int64_t)ii * (n + 1) + jj) * (n + 1) + kk];
    acol[(int64_t)q * ndof + d] = col < 0 ? (int32_t)d : col;
    aval[(int64_t)q * ndof + d] = col < 0 ? 0.0 : acc[q];
  }
  b[d] = bb;
}

// A^w in slot space: thread per (subdomain, slot).
__global__ void k_subassemble(int nsd, MeshArgs m, const int64_t* __restrict__ bids, const uint8_t* __restrict__ orphan,
                              const uint8_t* __restrict__ ncount, int32_t* __restrict__ slot_dof, double* __restrict__ As) {
  const int T = m.T;
  const int64_t gid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (gid >= (int64_t)nsd * T) return;
  const int s = (int)(gid / T), t = (int)(gid % T);
  const int b1 = m.B + 1, n = m.n;
  const int lx = t / (b1 * b1), ly = (t / b1) % b1, lz = t % b1;
  const int64_t bid = bids[s];
  const int bi = (int)(bid / m.nb / m.nb), bj = (int)((bid / m.nb) % m.nb), bk = (int)(bid % m.nb);
  const int i = bi * m.B + lx, j = bj * m.B + ly, k = bk * m.B + lz;
  double acc[27];
#pragma unroll
  for (int q = 0; q < 27; ++q) acc[q] = 0.0;
  bool local = false;
  for (int dx = 0; dx < 2; ++dx)
    for (int dy = 0; dy < 2; ++dy)
      for (int dz = 0; dz < 2; ++dz) {
        const int cx = lx - 1 + dx, cy = ly - 1 + dy, cz = lz - 1 + dz;
        if (cx < 0 || cy < 0 || cz < 0 || cx >= m.B || cy >= m.B || cz >= m.B) continue;
        const int64_t cell = ((int64_t)(bi * m.B + cx) * n + bj * m.B + cy) * n + bk * m.B + cz;
        if (m.eoc[cell] == -2) continue;
        local = true;
        const double* f = nullptr;
        const double* K = elem_k(m, cell, &f);
        if (!K) continue;
        const int lv = (1 - dx) + 2 * (1 - dy) + 4 * (1 - dz);
#pragma unroll
        for (int w = 0; w < 8; ++w) {
          const int q = stencil_k((w & 1) - (lv & 1), ((w >> 1) & 1) - ((lv >> 1) & 1), ((w >> 2) & 1) - ((lv >> 2) & 1));
          acc[q] += K[lv * 8 + w];
        }
      }
  int32_t dof = -1;
  if (local) {
    dof = m.dof_of_node[((int64_t)i * (n + 1) + j) * (n + 1) + k];
    if (orphan[dof]) {
#pragma unroll
      for (int q = 0; q < 27; ++q) acc[q] = 0.0;
      acc[13] = 1.0 / (double)ncount[dof];
    }
  }
  slot_dof[gid] = dof;
  double* A = As + (int64_t)s * 27 * T + t;
#pragma unroll
  for (int q = 0; q < 27; ++q) A[(int64_t)q * T] = acc[q];
}

// per dof: its (subdomain, slot) copies in this handle's subdomains, ascending
// subdomain order; owner slot for interior dofs of this handle's subdomains.
__global__ void k_copies(int64_t ndof, MeshArgs m, const int64_t* __restrict__ copy_ptr, int64_t* __restrict__ copy_idx,
                         int64_t* __restrict__ owner) {
  const int64_t d = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (d >= ndof) return;
  const int n = m.n, B = m.B, b1 = B + 1;
  const int64_t v = m.node_of_dof[d];
  const int k = (int)(v % (n + 1)), j = (int)((v / (n + 1)) % (n + 1)), i = (int)(v / (n + 1) / (n + 1));
  int64_t blks[8];
  int nbk = 0;
  for (int dx = 0; dx < 2; ++dx)
    for (int dy = 0; dy < 2; ++dy)
      for (int dz = 0; dz < 2; ++dz) {
        const int ci = i - 1 + dx, cj = j - 1 + dy, ck = k - 1 + dz;
        if (ci < 0 || cj < 0 || ck < 0 || ci >= n || cj >= n || ck >= n) continue;
        if (m.eoc[((int64_t)ci * n + cj) * n + ck] == -2) continue;
        const int64_t bid = ((int64_t)(ci / B) * m.nb + cj / B) * m.nb + ck / B;
        bool seen = false;
        for (int q = 0; q < nbk; ++q) seen |= blks[q] == bid;
        if (!seen) blks[nbk++] = bid;
      }
  // ascending block id == ascending subdomain id
  for (int a = 1; a < nbk; ++a)
    for (int c = a; c > 0 && blks[c - 1] > blks[c]; --c) {
      const int64_t tmp = blks[c];
      blks[c] = blks[c - 1];
      blks[c - 1] = tmp;
    }
  const int64_t p = copy_ptr[d];
  int nloc = 0;
  for (int q = 0; q < nbk; ++q) {
    const int64_t bid = blks[q];
    const int32_t sd = m.sd_of_block[bid];
    if (sd < 0) continue;  // another rank's subdomain
    const int bi = (int)(bid / m.nb / m.nb), bj = (int)((bid / m.nb) % m.nb), bk = (int)(bid % m.nb);
    const int slot = ((i - bi * B) * b1 + (j - bj * B)) * b1 + (k - bk * B);
    copy_idx[p + nloc++] = (int64_t)sd * m.T + slot;
  }
  owner[d] = nbk == 1 && nloc == 1 ? copy_idx[p] : -1;
}

__global__ void k_u8_to_i64(int64_t n, const uint8_t* __restrict__ a, int64_t* __restrict__ b) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) b[i] = a[i];
}

struct IsInterface {
  const uint8_t* nc;
  __host__ __device__ bool operator()(const int32_t& d) const { return nc[d] >= 2; }
};

}  // namespace

void assemble_device(cutbddc_gpu* h, int block, int nsd, const int64_t* block_ids) {
  cudaStream_t s = h->stream;
  const int n = h->n;
  if (block < 1 || n % block != 0) throw Failure(CUTBDDC_INVALID_ARGUMENT, "partition: mesh dims not divisible by H/h");
  h->block = block;
  h->b1 = block + 1;
  h->slots = h->b1 * h->b1 * h->b1;
  h->nb = n / block;
  h->nsd = nsd;
  h->nsd_global = 0;  // local numbering until cutbddc_gpu_set_global_ids
  h->global_of_local.clear();
  h->h_block_ids.assign(block_ids, block_ids + nsd);
  for (int i = 1; i < nsd; ++i)
    if (block_ids[i] <= block_ids[i - 1]) throw Failure(CUTBDDC_INVALID_ARGUMENT, "partition: block ids must ascend");
  h->block_ids.upload(h->h_block_ids, s);
  const int64_t nc = h->n_cells;
  const int grid = 148 * 8;
  ProfScope ps(h->prof, s, "assembly 1 cell lists");
  // active / cut cell lists (ascending)
  DevBuf<uint8_t>& act = h->ws_act;
  DevBuf<uint8_t>& cut = h->ws_cut;
  act.alloc((size_t)nc);
  cut.alloc((size_t)nc);
  k_cell_flags<<<grid, 256, 0, s>>>(nc, h->cls.p, act.p, cut.p);
  CB_LAUNCH();
  DevBuf<int64_t>& cnt = h->ws_cnt;
  cnt.alloc(2);
  h->active_cells.alloc((size_t)nc);
  h->cut_cells.alloc((size_t)nc);
  size_t tb = 0, tb2 = 0;
  cub::CountingInputIterator<int64_t> it(0);
  CB_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, it, act.p, h->active_cells.p, cnt.p, nc, s));
  CB_CUDA(cub::DeviceSelect::Flagged(nullptr, tb2, it, cut.p, h->cut_cells.p, cnt.p + 1, nc, s));
  DevBuf<uint8_t>& tmp = h->ws_tmp;
  tmp.alloc(std::max(tb, tb2));
  CB_CUDA(cub::DeviceSelect::Flagged(tmp.p, tb, it, act.p, h->active_cells.p, cnt.p, nc, s));
  CB_CUDA(cub::DeviceSelect::Flagged(tmp.p, tb2, it, cut.p, h->cut_cells.p, cnt.p + 1, nc, s));
  int64_t hc[2];
  CB_CUDA(cudaMemcpyAsync(hc, cnt.p, 16, cudaMemcpyDeviceToHost, s));
  CB_CUDA(cudaStreamSynchronize(s));
  h->n_active = hc[0];
  h->n_cut = hc[1];
  h->elem_of_cell.alloc((size_t)nc);
  k_elem_of_cell<<<grid, 256, 0, s>>>(nc, h->cls.p, h->elem_of_cell.p);
  CB_LAUNCH();
  if (h->n_cut) {
    k_scatter_cut<<<grid_for(h->n_cut, 256), 256, 0, s>>>(h->n_cut, h->cut_cells.p, h->elem_of_cell.p);
    CB_LAUNCH();
  }
  // element matrices
  ps.next("assembly 2 cut elements");
  cut_elements_device(h);
  DevBuf<double>& kint = h->ws_kint;
  kint.alloc(72);
  interior_element_device(h, kint.p, kint.p + 64);
  // subdomain maps
  ps.next("assembly 3 abar+subassembly+copies");
  h->sd_of_block.alloc((size_t)h->nb * h->nb * h->nb);
  CB_CUDA(cudaMemsetAsync(h->sd_of_block.p, 0xff, h->sd_of_block.n * 4, s));
  k_sd_of_block<<<grid_for(nsd, 256), 256, 0, s>>>(nsd, h->block_ids.p, h->sd_of_block.p);
  CB_LAUNCH();
  MeshArgs m{n, block, h->nb, h->slots, h->elem_of_cell.p, h->dof_of_node.p, h->node_of_dof.p,
             h->ke.p, h->fe.p, h->empty.p, kint.p, kint.p + 64, h->sd_of_block.p};
  const int64_t nd = h->n_dof;
  h->ncount.alloc((size_t)nd);
  h->lcount.alloc((size_t)nd);
  h->orphan.alloc((size_t)nd);
  k_dof_info<<<grid_for(nd, 256), 256, 0, s>>>(nd, m, h->ncount.p, h->lcount.p, h->orphan.p);
  CB_LAUNCH();
  h->aval.alloc((size_t)nd * 27);
  h->acol.alloc((size_t)nd * 27);
  h->b.alloc((size_t)nd);
  k_abar<<<grid_for(nd, 128), 128, 0, s>>>(nd, m, h->orphan.p, h->aval.p, h->acol.p, h->b.p);
  CB_LAUNCH();
  const int64_t ns = (int64_t)nsd * h->slots;
  h->slot_dof.alloc((size_t)ns);
  h->As.alloc((size_t)ns * 27);
  k_subassemble<<<grid_for(ns, 128), 128, 0, s>>>(nsd, m, h->block_ids.p, h->orphan.p, h->ncount.p, h->slot_dof.p, h->As.p);
  CB_LAUNCH();
  // copies CSR
  DevBuf<int64_t>& nc64 = h->ws_nc64;
  nc64.alloc((size_t)nd);
  k_u8_to_i64<<<grid_for(nd, 256), 256, 0, s>>>(nd, h->lcount.p, nc64.p);
  CB_LAUNCH();
  h->copy_ptr.alloc((size_t)nd + 1);
  CB_CUDA(cudaMemsetAsync(h->copy_ptr.p, 0, sizeof(int64_t), s));
  tb = 0;
  CB_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tb, nc64.p, h->copy_ptr.p + 1, nd, s));
  tmp.alloc(std::max(tmp.n, tb));
  CB_CUDA(cub::DeviceScan::InclusiveSum(tmp.p, tb, nc64.p, h->copy_ptr.p + 1, nd, s));
  CB_CUDA(cudaMemcpyAsync(&h->n_copies, h->copy_ptr.p + nd, 8, cudaMemcpyDeviceToHost, s));
  CB_CUDA(cudaStreamSynchronize(s));
  h->copy_idx.alloc((size_t)h->n_copies);
  h->owner_slot.alloc((size_t)nd);
  k_copies<<<grid_for(nd, 256), 256, 0, s>>>(nd, m, h->copy_ptr.p, h->copy_idx.p, h->owner_slot.p);
  CB_LAUNCH();
  // interface dof list
  h->if_dofs.alloc((size_t)nd);
  cub::CountingInputIterator<int32_t> it32(0);
  IsInterface pred{h->ncount.p};
  tb = 0;
  CB_CUDA(cub::DeviceSelect::If(nullptr, tb, it32, h->if_dofs.p, cnt.p, (int32_t)nd, pred, s));
  tmp.alloc(std::max(tmp.n, tb));
  CB_CUDA(cub::DeviceSelect::If(tmp.p, tb, it32, h->if_dofs.p, cnt.p, (int32_t)nd, pred, s));
  CB_CUDA(cudaMemcpyAsync(&h->n_if, cnt.p, 8, cudaMemcpyDeviceToHost, s));
  CB_CUDA(cudaStreamSynchronize(s));
  h->assembled = true;
  h->bddc_ready = false;
}

}  // namespace cutbddc_b200
