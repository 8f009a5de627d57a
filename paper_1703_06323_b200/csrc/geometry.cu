// geometry.cu — BackgroundMesh::classify on the device (K1).
// Compiled with -fmad=false: phi = sqrt((dx*dx + dy*dy) + dz*dz) - r with
// IEEE sqrt and no FMA contraction, matching the host op order of
// levelset.cpp:27-31 / mesh.cpp:132-136 bit for bit (checked against the
// reference-generated fixtures in tests/golden/classification.json).
#include <cub/cub.cuh>

#include "handle.cuh"

namespace cutbddc_b200 {

namespace {

// mesh.cpp:132-136: phi at node, snapped to -tol when |phi| <= tol.
__global__ void k_node_phi(int n, double ox, double oy, double oz, double hx, double hy, double hz, double tol,
                           const double* __restrict__ balls, int nballs, double* __restrict__ phi) {
  const int64_t nn = (int64_t)(n + 1) * (n + 1) * (n + 1);
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nn; v += (int64_t)gridDim.x * blockDim.x) {
    const int k = (int)(v % (n + 1));
    const int j = (int)((v / (n + 1)) % (n + 1));
    const int i = (int)(v / (n + 1) / (n + 1));
    const double x = ox + i * hx, y = oy + j * hy, z = oz + k * hz;
    double val = 0;
    for (int b = 0; b < nballs; ++b) {
      const double dx = x - balls[4 * b], dy = y - balls[4 * b + 1], dz = z - balls[4 * b + 2];
      const double s = sqrt(dx * dx + dy * dy + dz * dz) - balls[4 * b + 3];
      val = b == 0 ? s : fmin(val, s);
    }
    if (fabs(val) <= tol) val = -tol;
    phi[v] = val;
  }
}

// mesh.cpp:141-149: negative-vertex count -> Interior / Exterior / Cut.
__global__ void k_cell_class(int n, const double* __restrict__ phi, uint8_t* __restrict__ cls) {
  const int64_t nc = (int64_t)n * n * n;
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < nc; c += (int64_t)gridDim.x * blockDim.x) {
    const int k = (int)(c % n), j = (int)((c / n) % n), i = (int)(c / n / n);
    int neg = 0;
#pragma unroll
    for (int l = 0; l < 8; ++l) {
      const int64_t v = ((int64_t)(i + (l & 1)) * (n + 1) + j + ((l >> 1) & 1)) * (n + 1) + k + ((l >> 2) & 1);
      neg += phi[v] < 0;
    }
    cls[c] = neg == 8 ? CUTBDDC_INTERIOR : (neg == 0 ? CUTBDDC_EXTERIOR : CUTBDDC_CUT);
  }
}

// mesh.cpp:155-158: node carries a dof iff it is a vertex of an active cell.
__global__ void k_node_active(int n, const uint8_t* __restrict__ cls, int32_t* __restrict__ flag) {
  const int64_t nn = (int64_t)(n + 1) * (n + 1) * (n + 1);
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nn; v += (int64_t)gridDim.x * blockDim.x) {
    const int k = (int)(v % (n + 1)), j = (int)((v / (n + 1)) % (n + 1)), i = (int)(v / (n + 1) / (n + 1));
    int act = 0;
    for (int c = 0; c < 8 && !act; ++c) {
      const int ci = i - 1 + (c & 1), cj = j - 1 + ((c >> 1) & 1), ck = k - 1 + ((c >> 2) & 1);
      if (ci < 0 || cj < 0 || ck < 0 || ci >= n || cj >= n || ck >= n) continue;
      act = cls[((int64_t)ci * n + cj) * n + ck] != CUTBDDC_EXTERIOR;
    }
    flag[v] = act;
  }
}

// mesh.cpp:159-166: lexicographic numbering = exclusive scan of the flags.
__global__ void k_number(int64_t nn, const int32_t* __restrict__ flag, int32_t* __restrict__ dof,
                         int64_t* __restrict__ node_of_dof) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nn; v += (int64_t)gridDim.x * blockDim.x) {
    if (flag[v]) {
      node_of_dof[dof[v]] = v;
    } else {
      dof[v] = -1;
    }
  }
}

// node_of_dof from an uploaded dof_of_node map (the caller's BackgroundMesh
// view); bad[0] is set when a dof id is out of range.
__global__ void k_node_of_dof(int64_t nn, int64_t n_dof, const int32_t* __restrict__ dof,
                              int64_t* __restrict__ node_of_dof, int* __restrict__ bad) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nn; v += (int64_t)gridDim.x * blockDim.x) {
    const int32_t d = dof[v];
    if (d < 0) continue;
    if (d >= n_dof)
      atomicExch(bad, 1);
    else
      node_of_dof[d] = v;
  }
}

}  // namespace

void node_of_dof_device(cutbddc_gpu* h) {
  cudaStream_t s = h->stream;
  DevBuf<int>& bad = h->ws_flag;
  bad.alloc(1);
  bad.zero(s);
  h->node_of_dof.alloc((size_t)std::max<int64_t>(1, h->n_dof));
  const int grid = (int)std::min<int64_t>((h->n_nodes + 255) / 256, 148 * 8);
  k_node_of_dof<<<grid, 256, 0, s>>>(h->n_nodes, h->n_dof, h->dof_of_node.p, h->node_of_dof.p, bad.p);
  CB_LAUNCH();
  int hb = 0;
  CB_CUDA(cudaMemcpyAsync(&hb, bad.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  CB_CUDA(cudaStreamSynchronize(s));
  if (hb) throw Failure(CUTBDDC_INVALID_ARGUMENT, "mesh view: dof id out of range");
}

void classify_device(cutbddc_gpu* h, const cutbddc_geometry* g) {
  if (g->cells[0] != g->cells[1] || g->cells[1] != g->cells[2])
    throw Failure(CUTBDDC_INVALID_ARGUMENT, "mesh: only cubic cell counts are supported");
  const int n = g->cells[0];
  if (n < 1) throw Failure(CUTBDDC_INVALID_ARGUMENT, "mesh: needs at least one cell per axis");
  if (g->n_balls < 1) throw Failure(CUTBDDC_INVALID_ARGUMENT, "geometry: needs at least one ball");
  double hh[3];
  for (int d = 0; d < 3; ++d) {
    h->origin[d] = g->box_lo[d] + g->translation[d];   // mesh.cpp:122
    hh[d] = (g->box_hi[d] - g->box_lo[d]) / n;           // mesh.cpp:123
  }
  if (hh[0] != hh[1] || hh[1] != hh[2]) throw Failure(CUTBDDC_INVALID_ARGUMENT, "mesh: cells must be cubes");
  if (!(hh[0] > 0)) throw Failure(CUTBDDC_INVALID_ARGUMENT, "mesh: non-positive cell size");
  h->n = n;
  h->h = hh[0];
  h->tol = 1e-12 * hh[0];                                 // mesh.cpp:128
  h->n_nodes = (int64_t)(n + 1) * (n + 1) * (n + 1);
  h->n_cells = (int64_t)n * n * n;
  cudaStream_t s = h->stream;
  h->balls.upload(g->balls, (size_t)4 * g->n_balls, s);
  h->phi.alloc((size_t)h->n_nodes);
  h->cls.alloc((size_t)h->n_cells);
  h->dof_of_node.alloc((size_t)h->n_nodes);
  const int grid = 148 * 8;
  k_node_phi<<<grid, 256, 0, s>>>(n, h->origin[0], h->origin[1], h->origin[2], hh[0], hh[1], hh[2], h->tol, h->balls.p,
                                  g->n_balls, h->phi.p);
  CB_LAUNCH();
  k_cell_class<<<grid, 256, 0, s>>>(n, h->phi.p, h->cls.p);
  CB_LAUNCH();
  DevBuf<int32_t> flag;
  flag.alloc((size_t)h->n_nodes);
  k_node_active<<<grid, 256, 0, s>>>(n, h->cls.p, flag.p);
  CB_LAUNCH();
  size_t tmp_bytes = 0;
  CB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, flag.p, h->dof_of_node.p, (int64_t)h->n_nodes, s));
  DevBuf<uint8_t> tmp;
  tmp.alloc(tmp_bytes);
  CB_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tmp_bytes, flag.p, h->dof_of_node.p, (int64_t)h->n_nodes, s));
  int32_t last_dof = 0, last_flag = 0;
  CB_CUDA(cudaMemcpyAsync(&last_dof, h->dof_of_node.p + h->n_nodes - 1, 4, cudaMemcpyDeviceToHost, s));
  CB_CUDA(cudaMemcpyAsync(&last_flag, flag.p + h->n_nodes - 1, 4, cudaMemcpyDeviceToHost, s));
  CB_CUDA(cudaStreamSynchronize(s));
  h->n_dof = (int64_t)last_dof + last_flag;
  if (h->n_dof == 0) throw Failure(CUTBDDC_INVALID_ARGUMENT, "mesh: empty active mesh");  // mesh.cpp:153
  h->node_of_dof.alloc((size_t)h->n_dof);
  k_number<<<grid, 256, 0, s>>>(h->n_nodes, flag.p, h->dof_of_node.p, h->node_of_dof.p);
  CB_LAUNCH();
  CB_CUDA(cudaStreamSynchronize(s));
  h->mesh_ready = true;
  h->assembled = false;
  h->bddc_ready = false;
}

}  // namespace cutbddc_b200
