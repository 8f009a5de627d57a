// objects.cu — classify_objects on the device, from the
// resident mesh (device-side object
// classification). Bit-exact with the host restatement
// (host_partition.cpp, cutbddc_classify_objects) for the standard variant:
//
//   neigh(xi)  the nonempty blocks holding node xi as a local dof = the
//              blocks of its non-exterior incident cells (a block is a
//              subdomain iff it holds an active cell);
//              encoded exactly as (lowest block corner, 8-bit offset mask)
//   interface  |neigh| >= 2 and not strong-Dirichlet
//   objects    connected components of equal-neigh interface nodes over
//              active +axis lattice edges (BackgroundMesh::edge_active,
//              mesh.cpp:74-108): lock-free union-find that always hooks the
//              larger root under the smaller, so every component's root is
//              its smallest dof (deterministic labels)
//   kinds      singleton -> Corner, |neigh| = 2 -> Face, else Edge
//   order      by smallest dof, dofs ascending (stable radix sort by label)
//   variants   the paper's improved coarse edges: an edge
//              lattice edge joins two nodes only if neither is a v1 cut node
//              (an incident edge of the object changes the sign of phi,
//              PAPER.md:585-590) / their stiffness weight tuples agree within
//              1e-8 (v2; weights diag_w / Σ_w' diag_w' in
//              ascending subdomain order, the host's summation order)
#include <cub/cub.cuh>

#include "handle.cuh"

namespace cutbddc_b200 {
namespace {

constexpr uint64_t kNoKey = ~0ull;

// node -> (i, j, k), z fastest (mesh.cpp:41-44)
__device__ __forceinline__ void node_ijk(int64_t v, int n, int c[3]) {
  c[2] = (int)(v % (n + 1));
  c[1] = (int)((v / (n + 1)) % (n + 1));
  c[0] = (int)(v / (n + 1) / (n + 1));
}

__global__ void k_block_used(int n, int B, int nb, const uint8_t* __restrict__ cls, int32_t* __restrict__ used) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= (int64_t)n * n * n) return;
  if (cls[c] == CUTBDDC_EXTERIOR) return;
  const int k = (int)(c % n), j = (int)((c / n) % n), i = (int)(c / n / n);
  used[((int64_t)(i / B) * nb + j / B) * nb + k / B] = 1;  // benign: every writer stores 1
}

// neigh-set key per dof, kNoKey for non-interface dofs; parent[d] = d
__global__ void k_obj_keys(int64_t nd, int n, int B, int nb, const uint8_t* __restrict__ cls,
                           const int64_t* __restrict__ node_of_dof, const uint8_t* __restrict__ orphan,
                           uint64_t* __restrict__ key, int32_t* __restrict__ parent, int32_t* __restrict__ size) {
  const int64_t d = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (d >= nd) return;
  parent[d] = (int32_t)d;
  size[d] = 0;
  int c[3];
  node_ijk(node_of_dof[d], n, c);
  int lo[3] = {1 << 30, 1 << 30, 1 << 30};
  int blk[8][3], nbk = 0;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int ci = c[0] - 1 + (q & 1), cj = c[1] - 1 + ((q >> 1) & 1), ck = c[2] - 1 + ((q >> 2) & 1);
    if (ci < 0 || cj < 0 || ck < 0 || ci >= n || cj >= n || ck >= n) continue;
    if (cls[((int64_t)ci * n + cj) * n + ck] == CUTBDDC_EXTERIOR) continue;
    blk[nbk][0] = ci / B;
    blk[nbk][1] = cj / B;
    blk[nbk][2] = ck / B;
    for (int a = 0; a < 3; ++a) lo[a] = min(lo[a], blk[nbk][a]);
    ++nbk;
  }
  unsigned mask = 0;
  for (int q = 0; q < nbk; ++q)
    mask |= 1u << ((blk[q][0] - lo[0]) + 2 * (blk[q][1] - lo[1]) + 4 * (blk[q][2] - lo[2]));
  const bool iface = __popc(mask) >= 2 && !(orphan && orphan[d]);
  key[d] = iface ? ((uint64_t)(((int64_t)lo[0] * nb + lo[1]) * nb + lo[2]) << 8 | mask) : kNoKey;
}

__device__ __forceinline__ int uf_find(int32_t* p, int x) {
  while (true) {
    const int px = ((volatile int32_t*)p)[x];
    if (px == x) return x;
    const int ppx = ((volatile int32_t*)p)[px];
    if (ppx != px) atomicCAS(p + x, px, ppx);  // path halving (pointers only move toward the root)
    x = px;
  }
}

__device__ __forceinline__ void uf_union(int32_t* p, int a, int b) {
  while (true) {
    a = uf_find(p, a);
    b = uf_find(p, b);
    if (a == b) return;
    if (a > b) {
      const int t = a;
      a = b;
      b = t;
    }
    if (atomicCAS(p + b, b, a) == b) return;  // hook the larger root under the smaller
  }
}

__device__ __forceinline__ bool edge_active(const uint8_t* __restrict__ cls, int n, const int c[3], int ax) {
  // edge_active (mesh.cpp:74-108): one of the <= 4 cells around the edge is not exterior
  const int o1 = ax == 0 ? 1 : 0, o2 = ax == 2 ? 1 : 2;
  for (int da = -1; da <= 0; ++da)
    for (int db = -1; db <= 0; ++db) {
      int e[3] = {c[0], c[1], c[2]};
      e[o1] += da;
      e[o2] += db;
      if (e[0] < 0 || e[1] < 0 || e[2] < 0 || e[0] >= n || e[1] >= n || e[2] >= n) continue;
      if (cls[((int64_t)e[0] * n + e[1]) * n + e[2]] != CUTBDDC_EXTERIOR) return true;
    }
  return false;
}

// union along active +axis lattice edges between equal-key interface dofs
// (edge keys: unless a variant splits them, see the header)
__global__ void k_obj_union(int64_t nd, int n, const uint8_t* __restrict__ cls, const int32_t* __restrict__ dof_of_node,
                            const int64_t* __restrict__ node_of_dof, const uint64_t* __restrict__ key,
                            int32_t* parent, int variant, const uint8_t* __restrict__ cut,
                            const double* __restrict__ w8) {
  const int64_t d = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (d >= nd) return;
  const uint64_t kd = key[d];
  if (kd == kNoKey) return;
  const bool edge = __popcll(kd & 0xff) > 2;
  if (edge && variant == CUTBDDC_VARIANT_V1 && cut[d]) return;
  int c[3];
  node_ijk(node_of_dof[d], n, c);
  for (int ax = 0; ax < 3; ++ax) {
    if (c[ax] + 1 > n) continue;
    int cc[3] = {c[0], c[1], c[2]};
    cc[ax] += 1;
    const int32_t d2 = dof_of_node[((int64_t)cc[0] * (n + 1) + cc[1]) * (n + 1) + cc[2]];
    if (d2 < 0 || key[d2] != kd) continue;
    if (edge && variant == CUTBDDC_VARIANT_V1 && cut[d2]) continue;
    if (edge && variant == CUTBDDC_VARIANT_V2) {
      bool same = true;
      for (int q = 0; q < __popcll(kd & 0xff); ++q) {
        const double wa = w8[d * 8 + q], wb = w8[(int64_t)d2 * 8 + q];
        const double scale = fmax(1.0, fmax(fabs(wa), fabs(wb)));
        if (fabs(wa - wb) > 1e-8 * scale) same = false;
      }
      if (!same) continue;
    }
    if (edge_active(cls, n, c, ax)) uf_union(parent, (int)d, (int)d2);
  }
}

// v1: edge-key dofs with an incident active object edge across which phi
// changes sign become corners
__global__ void k_v1_cut(int64_t nd, int n, const uint8_t* __restrict__ cls, const int32_t* __restrict__ dof_of_node,
                         const int64_t* __restrict__ node_of_dof, const uint64_t* __restrict__ key,
                         const double* __restrict__ phi, uint8_t* __restrict__ cut) {
  const int64_t d = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (d >= nd) return;
  cut[d] = 0;
  const uint64_t kd = key[d];
  if (kd == kNoKey || __popcll(kd & 0xff) <= 2) return;
  const int64_t v = node_of_dof[d];
  int c[3];
  node_ijk(v, n, c);
  const bool neg = phi[v] < 0;
  for (int ax = 0; ax < 3; ++ax)
    for (int sgn = -1; sgn <= 1; sgn += 2) {
      int cc[3] = {c[0], c[1], c[2]};
      cc[ax] += sgn;
      if (cc[ax] < 0 || cc[ax] > n) continue;
      const int64_t v2 = ((int64_t)cc[0] * (n + 1) + cc[1]) * (n + 1) + cc[2];
      const int32_t d2 = dof_of_node[v2];
      if (d2 < 0 || key[d2] != kd) continue;
      int lo[3] = {c[0], c[1], c[2]};
      if (sgn < 0) lo[ax] -= 1;
      if (!edge_active(cls, n, lo, ax)) continue;
      if ((phi[v2] < 0) != neg) cut[d] = 1;
    }
}

// v2: stiffness weight tuple of every interface dof (one rank holds every
// copy): w_q = diag_q / Σ diag, copies in ascending subdomain order
__global__ void k_v2_weights(int64_t nloc, int T, const int32_t* __restrict__ loc_glob,
                             const int32_t* __restrict__ cptr, const int32_t* __restrict__ csrc,
                             const double* __restrict__ As, double* __restrict__ w8) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= nloc) return;
  const int32_t p0 = cptr[i], k = cptr[i + 1] - p0;
  if (k < 2) return;
  double dg[8], tot = 0.0;
  for (int q = 0; q < k; ++q) {
    const int32_t c = csrc[p0 + q];
    dg[q] = As[(int64_t)(c / T) * 27 * T + 13ll * T + c % T];
    tot += dg[q];
  }
  const int64_t d = loc_glob[i];
  for (int q = 0; q < k; ++q) w8[d * 8 + q] = dg[q] / tot;
}

__global__ void k_obj_label(int64_t nd, const uint64_t* __restrict__ key, int32_t* parent, int32_t* __restrict__ size) {
  const int64_t d = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (d >= nd || key[d] == kNoKey) return;
  const int r = uf_find(parent, (int)d);
  atomicAdd(size + r, 1);
}

__device__ __forceinline__ int obj_kind(int size, uint64_t key) {
  return size == 1 ? CUTBDDC_CORNER : (__popcll(key & 0xff) == 2 ? CUTBDDC_FACE : CUTBDDC_EDGE);
}
__device__ __forceinline__ bool obj_keep(int kind, int objects) {
  return kind == CUTBDDC_CORNER || (kind == CUTBDDC_EDGE && objects >= CUTBDDC_OBJECTS_CE) ||
         (kind == CUTBDDC_FACE && objects >= CUTBDDC_OBJECTS_CEF);
}

// label = root (no unions run any more, so find is exact); flag the
// selected dofs and the roots of the selected objects
__global__ void k_obj_select(int64_t nd, int objects, const uint64_t* __restrict__ key, int32_t* parent,
                             const int32_t* __restrict__ size, uint8_t* __restrict__ sel, uint8_t* __restrict__ root,
                             int32_t* __restrict__ label) {
  const int64_t d = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (d >= nd) return;
  sel[d] = root[d] = 0;
  const uint64_t kd = key[d];
  if (kd == kNoKey) return;
  const int r = uf_find(parent, (int)d);
  label[d] = r;
  if (!obj_keep(obj_kind(size[r], kd), objects)) return;
  sel[d] = 1;
  root[d] = r == (int)d;
}

// per object (root r, ascending): kind, size, sorted neighbour subdomains
__global__ void k_obj_meta(int n_obj, int nb, const int32_t* __restrict__ roots, const uint64_t* __restrict__ key,
                           const int32_t* __restrict__ size, const int32_t* __restrict__ sd_glob,
                           int32_t* __restrict__ kind, int64_t* __restrict__ dcount, int64_t* __restrict__ ncount,
                           int32_t* __restrict__ neigh8) {
  const int o = blockIdx.x * blockDim.x + threadIdx.x;
  if (o >= n_obj) return;
  const int r = roots[o];
  const uint64_t kd = key[r];
  kind[o] = obj_kind(size[r], kd);
  dcount[o] = size[r];
  const int64_t base = (int64_t)(kd >> 8);
  const int lo2 = (int)(base % nb), lo1 = (int)((base / nb) % nb), lo0 = (int)(base / nb / nb);
  int ids[8], m = 0;
  for (int q = 0; q < 8; ++q)
    if ((kd >> q) & 1) {
      const int id = sd_glob[((int64_t)(lo0 + (q & 1)) * nb + lo1 + ((q >> 1) & 1)) * nb + lo2 + ((q >> 2) & 1)];
      int t = m++;
      while (t > 0 && ids[t - 1] > id) {  // insertion: ascending subdomain ids
        ids[t] = ids[t - 1];
        --t;
      }
      ids[t] = id;
    }
  ncount[o] = m;
  for (int q = 0; q < 8; ++q) neigh8[8 * (int64_t)o + q] = q < m ? ids[q] : -1;
}

__global__ void k_obj_neigh(int n_obj, const int64_t* __restrict__ nptr, const int32_t* __restrict__ neigh8,
                            int32_t* __restrict__ neigh) {
  const int o = blockIdx.x * blockDim.x + threadIdx.x;
  if (o >= n_obj) return;
  for (int64_t q = nptr[o]; q < nptr[o + 1]; ++q) neigh[q] = neigh8[8 * (int64_t)o + (q - nptr[o])];
}

template <typename T>
T* carve(DevBuf<uint8_t>& b, size_t& off, size_t count) {
  off = (off + 255) & ~(size_t)255;
  T* p = reinterpret_cast<T*>(b.p + off);
  off += count * sizeof(T);
  return p;
}

}  // namespace

// Device objects -> host cutbddc_objects (arrays allocated with new[]).
cutbddc_objects* classify_objects_device(cutbddc_gpu* h, int objects, int variant) {
  cudaStream_t s = h->stream;
  const int n = h->n, B = h->block;
  if (B < 1 || n % B != 0) throw Failure(CUTBDDC_INVALID_ARGUMENT, "objects: assemble a partition first");
  const int nb = n / B;
  const int64_t nd = h->n_dof, nblk = (int64_t)nb * nb * nb;
  if (nd >= (1ll << 31)) throw Failure(CUTBDDC_INVALID_ARGUMENT, "objects: more than 2^31 dofs");
  // one grow-only scratch arena
  size_t need = 0;
  auto sz = [&](size_t bytes) { need = ((need + 255) & ~(size_t)255) + bytes; };
  sz(8 * nd); sz(4 * nd); sz(4 * nd); sz(4 * nd); sz(nd); sz(nd);            // key parent size label sel root
  sz(4 * nd); sz(4 * nd); sz(4 * nd); sz(4 * nd);                            // seldofs sellab sortdofs sortlab
  sz(4 * nd); sz(4 * (nblk + 1)); sz(4 * (nblk + 1)); sz(24); sz(8 * nblk);  // roots used sd_glob counts blocks
  sz(4 * nd); sz(8 * (nd + 1)); sz(8 * (nd + 1)); sz(32 * nd); sz(4 * 8 * nd);  // kind dptr nptr neigh8 neigh
  const int nd32 = (int)nd;
  size_t tb = 0, t1 = 0;
  cub::CountingInputIterator<int32_t> it(0);
  CB_CUDA(cub::DeviceSelect::Flagged(nullptr, t1, it, (uint8_t*)nullptr, (int32_t*)nullptr, (int64_t*)nullptr, nd32, s));
  tb = std::max(tb, t1);
  CB_CUDA(cub::DeviceSelect::Flagged(nullptr, t1, cub::CountingInputIterator<int64_t>(0), (int32_t*)nullptr,
                                     (int64_t*)nullptr, (int64_t*)nullptr, (int)nblk, s));
  tb = std::max(tb, t1);
  CB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, t1, (int32_t*)nullptr, (int32_t*)nullptr, (int32_t*)nullptr,
                                          (int32_t*)nullptr, nd32, 0, 32, s));
  tb = std::max(tb, t1);
  CB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, t1, (int32_t*)nullptr, (int32_t*)nullptr, (int)(nblk + 1), s));
  tb = std::max(tb, t1);
  CB_CUDA(cub::DeviceScan::InclusiveSum(nullptr, t1, (int64_t*)nullptr, (int64_t*)nullptr, nd32, s));
  tb = std::max(tb, t1);
  sz(tb);
  DevBuf<uint8_t>& ar = h->ws_obj;
  ar.alloc(need);
  size_t off = 0;
  uint64_t* key = carve<uint64_t>(ar, off, nd);
  int32_t* parent = carve<int32_t>(ar, off, nd);
  int32_t* size = carve<int32_t>(ar, off, nd);
  int32_t* label = carve<int32_t>(ar, off, nd);
  uint8_t* sel = carve<uint8_t>(ar, off, nd);
  uint8_t* rootf = carve<uint8_t>(ar, off, nd);
  int32_t* seldofs = carve<int32_t>(ar, off, nd);
  int32_t* sellab = carve<int32_t>(ar, off, nd);
  int32_t* sortdofs = carve<int32_t>(ar, off, nd);
  int32_t* sortlab = carve<int32_t>(ar, off, nd);
  int32_t* roots = carve<int32_t>(ar, off, nd);
  int32_t* used = carve<int32_t>(ar, off, nblk + 1);
  int32_t* sd_glob = carve<int32_t>(ar, off, nblk + 1);
  int64_t* cnt = carve<int64_t>(ar, off, 3);
  int64_t* blocks = carve<int64_t>(ar, off, nblk);
  int32_t* kind = carve<int32_t>(ar, off, nd);
  int64_t* dptr = carve<int64_t>(ar, off, nd + 1);
  int64_t* nptr = carve<int64_t>(ar, off, nd + 1);
  int32_t* neigh8 = carve<int32_t>(ar, off, 8 * nd);
  int32_t* neigh = carve<int32_t>(ar, off, 8 * nd);
  void* tmp = carve<uint8_t>(ar, off, tb);

  // global subdomain ids: rank of each nonempty block (build_partition order)
  CB_CUDA(cudaMemsetAsync(used, 0, 4 * (nblk + 1), s));
  k_block_used<<<grid_for(h->n_cells, 256), 256, 0, s>>>(n, B, nb, h->cls.p, used);
  CB_LAUNCH();
  t1 = tb;
  CB_CUDA(cub::DeviceScan::ExclusiveSum(tmp, t1, used, sd_glob, (int)(nblk + 1), s));
  cub::CountingInputIterator<int64_t> itb(0);
  t1 = tb;
  CB_CUDA(cub::DeviceSelect::Flagged(tmp, t1, itb, used, blocks, cnt + 2, (int)nblk, s));
  k_obj_keys<<<grid_for(nd, 256), 256, 0, s>>>(nd, n, B, nb, h->cls.p, h->node_of_dof.p, h->orphan.p, key, parent,
                                                size);
  CB_LAUNCH();
  uint8_t* cut = nullptr;
  double* w8 = nullptr;
  if (variant == CUTBDDC_VARIANT_V1) {
    h->ws_cut.alloc((size_t)nd);
    cut = h->ws_cut.p;
    k_v1_cut<<<grid_for(nd, 256), 256, 0, s>>>(nd, n, h->cls.p, h->dof_of_node.p, h->node_of_dof.p, key, h->phi.p, cut);
    CB_LAUNCH();
  } else if (variant == CUTBDDC_VARIANT_V2) {
    if (h->dist_world > 1)
      throw Failure(CUTBDDC_CONFIG, "device objects v2: needs every subdomain's diagonals (one rank only)");
    h->ws_w8.alloc((size_t)nd * 8);
    w8 = h->ws_w8.p;
    k_v2_weights<<<grid_for(h->n_loc, 256), 256, 0, s>>>(h->n_loc, h->slots, h->loc_glob.p, h->lcopy_ptr.p,
                                                         h->lcopy_src.p, h->As.p, w8);
    CB_LAUNCH();
  }
  k_obj_union<<<grid_for(nd, 256), 256, 0, s>>>(nd, n, h->cls.p, h->dof_of_node.p, h->node_of_dof.p, key, parent,
                                                variant, cut, w8);
  CB_LAUNCH();
  k_obj_label<<<grid_for(nd, 256), 256, 0, s>>>(nd, key, parent, size);
  CB_LAUNCH();
  k_obj_select<<<grid_for(nd, 256), 256, 0, s>>>(nd, objects, key, parent, size, sel, rootf, label);
  CB_LAUNCH();
  // selected dofs (ascending), stably sorted by label = smallest dof of the object
  t1 = tb;
  CB_CUDA(cub::DeviceSelect::Flagged(tmp, t1, it, sel, seldofs, cnt, nd32, s));
  t1 = tb;
  CB_CUDA(cub::DeviceSelect::Flagged(tmp, t1, label, sel, sellab, cnt, nd32, s));
  t1 = tb;
  CB_CUDA(cub::DeviceSelect::Flagged(tmp, t1, it, rootf, roots, cnt + 1, nd32, s));
  int64_t hc[3] = {0, 0, 0};
  CB_CUDA(cudaMemcpyAsync(hc, cnt, 24, cudaMemcpyDeviceToHost, s));
  CB_CUDA(cudaStreamSynchronize(s));
  const int n_sel = (int)hc[0], n_obj = (int)hc[1];
  int bits = 1;
  while (bits < 32 && (1ll << bits) <= nd) ++bits;
  if (n_sel > 0) {
    t1 = tb;
    CB_CUDA(cub::DeviceRadixSort::SortPairs(tmp, t1, sellab, sortlab, seldofs, sortdofs, n_sel, 0, bits, s));
  }
  if (n_obj > 0) {
    k_obj_meta<<<grid_for(n_obj, 128), 128, 0, s>>>(n_obj, nb, roots, key, size, sd_glob, kind, dptr + 1, nptr + 1,
                                                    neigh8);
    CB_LAUNCH();
    CB_CUDA(cudaMemsetAsync(dptr, 0, 8, s));
    CB_CUDA(cudaMemsetAsync(nptr, 0, 8, s));
    t1 = tb;
    CB_CUDA(cub::DeviceScan::InclusiveSum(tmp, t1, dptr + 1, dptr + 1, n_obj, s));
    t1 = tb;
    CB_CUDA(cub::DeviceScan::InclusiveSum(tmp, t1, nptr + 1, nptr + 1, n_obj, s));
    k_obj_neigh<<<grid_for(n_obj, 128), 128, 0, s>>>(n_obj, nptr, neigh8, neigh);
    CB_LAUNCH();
  }
  auto* r = new cutbddc_objects{};
  r->n_sd = (int)hc[2];
  r->block_ids = new int64_t[(size_t)hc[2] + 1];
  CB_CUDA(cudaMemcpyAsync(r->block_ids, blocks, 8 * (size_t)hc[2], cudaMemcpyDeviceToHost, s));
  r->n_objects = n_obj;
  r->kinds = new int32_t[(size_t)n_obj + 1];
  r->dof_ptr = new int64_t[(size_t)n_obj + 1];
  r->neigh_ptr = new int64_t[(size_t)n_obj + 1];
  r->dofs = new int32_t[(size_t)n_sel + 1];
  r->dof_ptr[0] = r->neigh_ptr[0] = 0;
  if (n_obj > 0) {
    CB_CUDA(cudaMemcpyAsync(r->kinds, kind, 4 * (size_t)n_obj, cudaMemcpyDeviceToHost, s));
    CB_CUDA(cudaMemcpyAsync(r->dof_ptr, dptr, 8 * ((size_t)n_obj + 1), cudaMemcpyDeviceToHost, s));
    CB_CUDA(cudaMemcpyAsync(r->neigh_ptr, nptr, 8 * ((size_t)n_obj + 1), cudaMemcpyDeviceToHost, s));
    CB_CUDA(cudaMemcpyAsync(r->dofs, sortdofs, 4 * (size_t)n_sel, cudaMemcpyDeviceToHost, s));
  }
  CB_CUDA(cudaStreamSynchronize(s));
  const int64_t nn = r->neigh_ptr[n_obj];
  r->neigh = new int32_t[(size_t)nn + 1];
  if (nn > 0) {
    CB_CUDA(cudaMemcpyAsync(r->neigh, neigh, 4 * (size_t)nn, cudaMemcpyDeviceToHost, s));
    CB_CUDA(cudaStreamSynchronize(s));
  }
  return r;
}

}  // namespace cutbddc_b200
