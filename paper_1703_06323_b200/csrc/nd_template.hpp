// nd_template.hpp — geometric nested-dissection template of one subdomain's
// (B+1)^3 node lattice, shared by every subdomain of a run.
//
// Replaces the per-matrix symbolic analysis of the reference's sparse
// factorisations (SparseCholesky / SimplicialLDLT + AMD, linalg.cpp:34-62;
// SaddleFactorization / SparseLU + COLAMD, linalg.cpp:64-106). Every
// subdomain matrix lives in the same slot space (absent slots are identity
// rows), so one template drives all subdomains and every batched launch has
// uniform front shapes.
//
// Supernodes: recursive bisection of boxes; a box with <= leaf_max nodes is
// a leaf supernode (all its nodes), otherwise its middle plane along the
// longest axis (ties x, y, z) is a separator supernode. rows(s) = cols(s)
// followed by the box halo (nodes within Chebyshev distance 1 outside the
// box) in ascending slot order; that halo is exactly the fill pattern of the
// 27-point stencil eliminated in ND order.
#pragma once

#include <cstdint>
#include <vector>

namespace cutbddc_b200 {

struct Supernode {
  int level = 0;      // depth from the root (root = 0)
  int ncols = 0;      // pivot columns
  int nrows = 0;      // front rows: cols first, then halo (ascending slot)
  int parent = -1;
  int child[2] = {-1, -1};
  int nchild = 0;
  int64_t rows_off = 0;   // into Template::rows
  int64_t panel_off = 0;  // factor panel G (nrows x ncols, column-major) in a subdomain's factor store
  int64_t front_off = 0;  // dense front (nrows x nrows, column-major) in a subdomain's front workspace
  int64_t upd_off = 0;    // forward-solve update vector (nrows - ncols) in a subdomain's solve workspace
  int64_t amap_off = 0;   // assembly entries [amap_off, amap_off + amap_len)
  int amap_len = 0;
  int64_t emap_off = 0;   // extend-add map of THIS node into its parent: nrows-ncols positions
};

struct AmapEntry {
  int32_t pos;   // r + c * nrows inside the front (lower triangle)
  int32_t slot;  // slot u (column node)
  int32_t k;     // stencil index of the row node v relative to u (0..26)
  int32_t pad;
};

struct Template {
  int b1 = 0;            // nodes per side (B + 1)
  int slots = 0;         // b1^3
  int leaf_max = 0;
  bool shell_root = false;              // root supernode = the lattice shell (see build_template)
  std::vector<int32_t> root_pos;        // slot -> position in the root front, -1 if not a root column
  std::vector<Supernode> sn;            // postorder (children before parents)
  std::vector<int32_t> rows;            // slot ids per supernode
  std::vector<AmapEntry> amap;
  std::vector<int32_t> emap;            // positions in the parent front
  std::vector<std::vector<int32_t>> levels;  // supernode ids per level
  int64_t panel_total = 0, front_total = 0, upd_total = 0;
  int max_rows = 0, max_cols = 0;
  double flops = 0;      // dense partial-Cholesky flops per factorisation
  std::vector<int32_t> elim;            // slot -> elimination position
};

// shell_root = false: plain ND of the whole (B+1)^3 lattice (interior
// problems A_II). shell_root = true: the root supernode is the whole lattice
// shell and its single child is the ND of the inner (B-1)^3 box; used for the
// constrained Neumann matrix K = A + rho C^T C, whose edge/face rows couple
// every node of an object (objects live on the shell) densely.
Template build_template(int block, int leaf_max, bool shell_root = false);

}  // namespace cutbddc_b200
