// assembly.cu — sub-assembled subdomain matrices (K3).
//
// assemble_subassembled as a deterministic gather: every
// (slot, 27-stencil column) entry sums the element contributions of the <= 8
// cells of the subdomain around the slot node in ascending cell id, the same
// order the CPU restatement's triplet merge uses (linalg.cpp:12-32
// semantics), so no fp64 atomics are involved. assemble_global
// is not formed: Abar = Σ_w R_w^T A_w R_w is applied
// matrix-free (dist.cu), and the load vector is the interface sum of the
// sub-assembled ones. Only this rank's subdomains are assembled; cut cells
// of other ranks are never integrated here (their void flags arrive by one
// all-reduce of a byte per cell). Strong-Dirichlet (orphan) dofs: all
// incident active cells empty -> 1/|neigh| diagonal in every A^w, so the sum
// over copies is the identity row of Abar.
#include <cub/cub.cuh>

#include "comm.cuh"
#include "dist.cuh"
#include "handle.cuh"
#include "mms.cuh"

namespace cutbddc_b200 {

void cut_elements_device(cutbddc_gpu* h);
void interior_element_device(cutbddc_gpu* h, double* kint, double* fint);

namespace {

// active cells; cut cells of this rank's subdomains
__global__ void k_cell_flags(int64_t nc, int n, int B, int nb, const uint8_t* __restrict__ cls,
                             const int32_t* __restrict__ sd_of_block, uint8_t* __restrict__ act,
                             uint8_t* __restrict__ cut) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < nc; c += (int64_t)gridDim.x * blockDim.x) {
    act[c] = cls[c] != CUTBDDC_EXTERIOR;
    const int64_t k = c % n, j = (c / n) % n, i = c / n / n;
    cut[c] = cls[c] == CUTBDDC_CUT && sd_of_block[((i / B) * nb + j / B) * nb + k / B] >= 0;
  }
}

// -2 exterior, -1 interior, -3 cut (another rank's, or until k_scatter_cut)
__global__ void k_elem_of_cell(int64_t nc, const uint8_t* __restrict__ cls, int32_t* __restrict__ eoc) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < nc; c += (int64_t)gridDim.x * blockDim.x)
    eoc[c] = cls[c] == CUTBDDC_EXTERIOR ? -2 : (cls[c] == CUTBDDC_CUT ? -3 : -1);
}

__global__ void k_scatter_cut(int64_t ncut, const int64_t* __restrict__ cut_cells, int32_t* __restrict__ eoc) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e < ncut) eoc[cut_cells[e]] = (int32_t)e;
}

// void flag of this rank's cut cells (all-reduced by max over ranks)
__global__ void k_vcell(int64_t ncut, const int64_t* __restrict__ cut_cells, const uint8_t* __restrict__ empty,
                        uint8_t* __restrict__ vcell) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e < ncut) vcell[cut_cells[e]] = empty[e];
}

__global__ void k_sd_of_block(int nsd, const int64_t* __restrict__ bids, int32_t* __restrict__ sob) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s < nsd) sob[bids[s]] = s;
}

struct MeshArgs {
  int n, B, nb, T;
  int problem;          // kProblemManufactured: interior-cell loads from f at the Gauss points
  double ox, oy, oz, h;
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

// per dof: |neigh| (distinct blocks among incident active cells, every
// rank's) and the orphan flag (every incident active cell void)
// load of an interior cell at its local node lv, manufactured problem: the
// 2x2x2 Gauss rule (full_quadrature_ref), h^3 sum_g 1/8 (f(x_g) phi_lv(xi_g))
__device__ double interior_mms_load(const MeshArgs& m, int ci, int cj, int ck, int lv) {
  const double g0 = 0.5 - 0.5 / sqrt(3.0), g1 = 0.5 + 0.5 / sqrt(3.0);
  double s = 0.0;
  for (int l = 0; l < 8; ++l) {
    const double xi[3] = {(l & 1) ? g1 : g0, ((l >> 1) & 1) ? g1 : g0, ((l >> 2) & 1) ? g1 : g0};
    double f[3];
    for (int d = 0; d < 3; ++d) f[d] = ((lv >> d) & 1) ? xi[d] : 1.0 - xi[d];
    const double val = f[0] * f[1] * f[2];
    const double fx = mms_f(m.ox + ((double)ci + xi[0]) * m.h, m.oy + ((double)cj + xi[1]) * m.h,
                            m.oz + ((double)ck + xi[2]) * m.h);
    s += 0.125 * (fx * val);
  }
  return m.h * m.h * m.h * s;
}

__global__ void k_dof_info(int64_t ndof, MeshArgs m, const uint8_t* __restrict__ vcell, uint8_t* __restrict__ ncount,
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
        if (e == -1 || !vcell[cell]) nonvoid = true;
        const int64_t bid = ((int64_t)(ci / m.B) * m.nb + cj / m.B) * m.nb + ck / m.B;
        bool seen = false;
        for (int q = 0; q < nbk; ++q) seen |= blks[q] == bid;
        if (!seen) blks[nbk++] = bid;
      }
  ncount[d] = (uint8_t)nbk;
  orphan[d] = !nonvoid;
}

// A^w in slot space, its load vector and the strong-Dirichlet diagonal:
// thread per (subdomain, slot).
__global__ void k_subassemble(int nsd, MeshArgs m, const int64_t* __restrict__ bids, const uint8_t* __restrict__ orphan,
                              const uint8_t* __restrict__ ncount, int32_t* __restrict__ slot_dof, double* __restrict__ As,
                              double* __restrict__ fs, double* __restrict__ odiag) {
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
  double bb = 0.0, od = 0.0;
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
        bb += (m.problem == kProblemManufactured && m.eoc[cell] == -1)
                  ? interior_mms_load(m, bi * m.B + cx, bj * m.B + cy, bk * m.B + cz, lv)
                  : f[lv];
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
      acc[13] = od = 1.0 / (double)ncount[dof];
      bb = 0.0;
    }
  }
  slot_dof[gid] = dof;
  fs[gid] = bb;
  odiag[gid] = od;
  double* A = As + (int64_t)s * 27 * T + t;
#pragma unroll
  for (int q = 0; q < 27; ++q) A[(int64_t)q * T] = acc[q];
}

__global__ void k_masks(int64_t ns, const int32_t* __restrict__ slot_dof, const uint8_t* __restrict__ ncount,
                        uint8_t* __restrict__ mall, uint8_t* __restrict__ mint) {
  const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g >= ns) return;
  const int32_t d = slot_dof[g];
  mall[g] = d >= 0;
  mint[g] = d >= 0 && ncount[d] == 1;
}

struct IsInterface {
  const uint8_t* nc;
  __host__ __device__ bool operator()(const int32_t& d) const { return nc[d] >= 2; }
};

}  // namespace

void assemble_device(cutbddc_gpu* h, const cutbddc_partition_view* part) {
  cudaStream_t s = h->stream;
  const int n = h->n, block = part->block;
  if (block < 1 || n % block != 0) throw Failure(CUTBDDC_INVALID_ARGUMENT, "partition: mesh dims not divisible by H/h");
  // the distribution: set by the caller (every rank passes the global
  // partition) or every subdomain on this handle
  if (!h->dist_explicit) {
    dist_default(h, part);
  } else if (h->dist_block != block || h->nsd_g != part->n_sd ||
             !std::equal(h->g_block_ids.begin(), h->g_block_ids.end(), part->block_ids)) {
    throw Failure(CUTBDDC_INVALID_ARGUMENT, "assemble: partition differs from the distribution's");
  }
  h->block = block;
  h->b1 = block + 1;
  h->slots = h->b1 * h->b1 * h->b1;
  h->nb = n / block;
  const int nsd = (int)h->global_of_local.size();
  h->nsd = nsd;
  h->h_block_ids.resize((size_t)nsd);
  for (int i = 0; i < nsd; ++i) h->h_block_ids[(size_t)i] = h->g_block_ids[(size_t)h->global_of_local[(size_t)i]];
  h->block_ids.upload(h->h_block_ids, s);
  const int64_t nc = h->n_cells;
  const int grid = 148 * 8;
  ProfScope ps(h->prof, s, "assembly 1 cell lists");
  h->sd_of_block.alloc((size_t)h->nb * h->nb * h->nb);
  CB_CUDA(cudaMemsetAsync(h->sd_of_block.p, 0xff, h->sd_of_block.n * 4, s));
  k_sd_of_block<<<grid_for(nsd, 256), 256, 0, s>>>(nsd, h->block_ids.p, h->sd_of_block.p);
  CB_LAUNCH();
  // active cells (all) / cut cells of this rank's subdomains (ascending)
  DevBuf<uint8_t>& act = h->ws_act;
  DevBuf<uint8_t>& cut = h->ws_cut;
  act.alloc((size_t)nc);
  cut.alloc((size_t)nc);
  k_cell_flags<<<grid, 256, 0, s>>>(nc, n, block, h->nb, h->cls.p, h->sd_of_block.p, act.p, cut.p);
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
  // element matrices of this rank's cut cells
  ps.next("assembly 2 cut elements");
  cut_elements_device(h);
  pack_cut_matrices(h);
  DevBuf<double>& kint = h->ws_kint;
  kint.alloc(72);
  interior_element_device(h, kint.p, kint.p + 64);
  ps.next("assembly 3 subassembly+plan+rhs");
  // void cut cells of every rank: one byte per cell, all-reduced (max)
  h->vcell.alloc((size_t)nc);
  h->vcell.zero(s);
  if (h->n_cut) {
    k_vcell<<<grid_for(h->n_cut, 256), 256, 0, s>>>(h->n_cut, h->cut_cells.p, h->empty.p, h->vcell.p);
    CB_LAUNCH();
  }
  // plan-only distribution (a rank's view without a communicator, for plan
  // inspection): other ranks' void cells and the load vector are unknown
  const bool plan_only = h->dist_world > 1 && !h->comm;
  if (h->dist_world > 1 && !plan_only)
    nccl_check(ncclAllReduce(h->vcell.p, h->vcell.p, (size_t)nc, ncclUint8, ncclMax, h->comm, s), "void cells");
  MeshArgs m{n,          block,         h->nb,         h->slots,      h->problem,      h->origin[0],
             h->origin[1], h->origin[2], h->h,          h->elem_of_cell.p, h->dof_of_node.p, h->node_of_dof.p,
             h->ke.p,      h->fe.p,       h->empty.p,    kint.p,        kint.p + 64,     h->sd_of_block.p};
  const int64_t nd = h->n_dof;
  h->ncount.alloc((size_t)nd);
  h->orphan.alloc((size_t)nd);
  k_dof_info<<<grid_for(nd, 256), 256, 0, s>>>(nd, m, h->vcell.p, h->ncount.p, h->orphan.p);
  CB_LAUNCH();
  const int64_t ns = (int64_t)nsd * h->slots;
  h->slot_dof.alloc((size_t)ns);
  h->As.alloc((size_t)ns * 27);
  h->fs.alloc((size_t)ns);
  h->odiag.alloc((size_t)ns);
  k_subassemble<<<grid_for(ns, 128), 128, 0, s>>>(nsd, m, h->block_ids.p, h->orphan.p, h->ncount.p, h->slot_dof.p, h->As.p,
                                                  h->fs.p, h->odiag.p);
  CB_LAUNCH();
  h->mask_all.alloc((size_t)ns);
  h->mask_int.alloc((size_t)ns);
  k_masks<<<grid_for(ns, 256), 256, 0, s>>>(ns, h->slot_dof.p, h->ncount.p, h->mask_all.p, h->mask_int.p);
  CB_LAUNCH();
  // local dof space, copy and exchange lists; the operator's rows
  build_plan_device(h);
  build_operator_rows(h);
  // load vector: interface sum of the sub-assembled ones
  h->b.alloc((size_t)std::max<int64_t>(1, h->n_loc));
  h->plan_only = plan_only;
  if (!plan_only) {
    iface_exchange(h, h->fs.p, nullptr, nullptr);
    iface_sum(h, h->fs.p, nullptr, h->b.p, nullptr);
  }
  // interface dofs of the global problem
  DevBuf<int32_t>& ifd = h->ws_glist;
  ifd.alloc((size_t)nd);
  cub::CountingInputIterator<int32_t> it32(0);
  IsInterface pred{h->ncount.p};
  tb = 0;
  CB_CUDA(cub::DeviceSelect::If(nullptr, tb, it32, ifd.p, cnt.p, (int32_t)nd, pred, s));
  tmp.alloc(std::max(tmp.n, tb));
  CB_CUDA(cub::DeviceSelect::If(tmp.p, tb, it32, ifd.p, cnt.p, (int32_t)nd, pred, s));
  CB_CUDA(cudaMemcpyAsync(&h->n_if, cnt.p, 8, cudaMemcpyDeviceToHost, s));
  CB_CUDA(cudaStreamSynchronize(s));
  h->assembled = true;
  h->bddc_ready = false;
}

}  // namespace cutbddc_b200
