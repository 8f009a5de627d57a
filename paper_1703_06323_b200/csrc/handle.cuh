// handle.cuh — device-resident state of one cutbddc_gpu handle.
//
// HBM layout:
//   mesh:        phi[(n+1)^3] f64, cls[n^3] u8, dof_of_node[(n+1)^3] i32,
//                node_of_dof[n_dof] i64, elem_of_cell[n^3] i32 (cut index, -1 interior, -2 exterior)
//   cut cells:   ke[ncut][64] f64, fe[ncut][8] f64, beta[ncut], empty[ncut]
//   subdomains:  slot space of the (B+1)^3 block lattice, T slots per subdomain:
//                slot_dof[nsd][T] i32, As[nsd][27][T] f64 (stencil of A^w, SoA over slots)
//   Abar:        never assembled (matrix-free Σ_w R_w^T A_w R_w, dist.cu)
//   vectors:     local dof space of the rank (segments per subdomain + ghosts, dist.cuh)
//   bddc:        weights w[nsd][T], interior/present masks, factor panels
//                GI/GK[nsd][panel_total] (column-major per supernode), Phi[sum m][T]
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <memory>
#include <mutex>
#include <vector>

#include "cutbddc.h"
#include "dev_common.cuh"
#include "nd_template.hpp"
#include "prof.cuh"

// One ND template resident on the device.
struct TplSet {
  cutbddc_b200::Template tpl;
  cutbddc_b200::DevBuf<cutbddc_b200::Supernode> sn;
  cutbddc_b200::DevBuf<int32_t> rows, emap, root_pos;
  cutbddc_b200::DevBuf<cutbddc_b200::AmapEntry> amap;
  std::vector<uint8_t> is_split;                // per supernode: tiled DAG front (else one CTA, dense_dag.cu)
  bool ready = false;
};

// Task list of one dataflow factorisation launch (dense_dag.cu).
struct DagPlan {
  cutbddc_b200::DevBuf<long long> fronts;      // per front record (10 x int64)
  cutbddc_b200::DevBuf<int4> tasks;            // (kind << 24 | front, i, j, k) in ticket order
  cutbddc_b200::DevBuf<int> counters;          // per front: done, assembled, tile counters; then the ticket
  std::vector<int2> key;                       // spans + compact front sizes the list was built for
  // device-built task lists (dense_dag.cu build_tasks_device)
  cutbddc_b200::DevBuf<long long> d_fplan;     // per front: DevFrontPlan
  cutbddc_b200::DevBuf<int4> d_tpl, unsorted;  // shape templates; the list before the sort
  cutbddc_b200::DevBuf<int> d_tpl_bl;
  cutbddc_b200::DevBuf<int2> d_tpl_rng;
  cutbddc_b200::DevBuf<unsigned> keys;         // sort keys in / out
  cutbddc_b200::DevBuf<uint8_t> sort_tmp;
  int n_tasks = 0;
  int64_t n_counters = 0;
};

// dense_dag.cu: one dense front of a dense_dag_fronts launch (factor.cuh)
struct DenseFront {
  int64_t fo, po;
  int r, c;
};

// coarse_sparse.cu: the nested-dissection multifrontal factor of A_c
// (n_c > kCoarseInverseMax)
struct CoarseSparse {
  bool ready = false;
  int nlev = 0, rt_max = 0, n_fronts = 0;
  double flops = 0.0;
  std::vector<int> level_ptr;                   // fronts of level l: flist[level_ptr[l] ..)
  std::vector<int> level_rt, level_c;           // per level: largest front / pivot block (solve grids)
  std::vector<std::vector<DenseFront>> dense;  // per level, for dense_dag_fronts
  std::vector<std::unique_ptr<DagPlan>> plans;  // per level
  cutbddc_b200::DevBuf<long long> fronts;      // CsFront records
  cutbddc_b200::DevBuf<int32_t> idx, cmap;     // per front: coarse ids (columns, rows); children's row maps
  cutbddc_b200::DevBuf<int> flist;             // front ids by level
  cutbddc_b200::DevBuf<double> F, P, ybuf, ubuf;
};

// One factorisation over a template, compacted per subdomain (masked-out
// slots dropped from every front).
struct FactorSet {
  cutbddc_b200::DevBuf<double> panel;          // compact [L11; L21] panels
  cutbddc_b200::DevBuf<int32_t> pfx;           // nsd x rows_total
  cutbddc_b200::DevBuf<int32_t> tpos;          // nsd x rows_total (inverse of pfx)
  cutbddc_b200::DevBuf<int2> rc;               // nsd x nsn
  cutbddc_b200::DevBuf<int64_t> panel_off, upd_off;  // nsd x nsn
  std::vector<int2> h_rc;
  std::vector<int64_t> h_front_base;           // nsd + 1 (front workspace prefix)
  int64_t panel_total = 0, upd_total = 0;
  double bytes_per_sweep = 0;                  // algorithmic bytes of fwd + bwd sweeps
  double flops = 0;                            // partial-Cholesky flops
  double flops_inv = 0;                        // explicit inverse panel G = [L11^{-1}; L21 L11^{-1}] flops
  // dataflow sweeps (sweep.cu): one persistent launch per sweep direction
  cutbddc_b200::DevBuf<int4> desc;             // nsd x nsn front descriptors (6 x int4 each, sweep.cu)
  cutbddc_b200::DevBuf<int32_t> cslot;         // vec_total: slot of each compact front row
  cutbddc_b200::DevBuf<int32_t> umap;          // upd_total: parent compact row of each update entry
  cutbddc_b200::DevBuf<int32_t> gmap;          // 2 x vec_total: child 0 / 1 update entry of each front row (-1: none)
  cutbddc_b200::DevBuf<int4> items_f, items_b; // (kind, supernode, subdomain, chunk) in dependency order
  cutbddc_b200::DevBuf<int32_t> counters;      // done_f | ready_f | done_b | ready_b | tickets
  cutbddc_b200::DevBuf<double> vbuf;           // vec_total: assembled vectors of chunked fronts
  cutbddc_b200::DevBuf<unsigned long long> trace;  // CUTBDDC_SWEEP_TRACE only: per-item timestamps
  int64_t vec_total = 0;
  int n_items_f = 0, n_items_b = 0;
  int n_items_b_root = 0;                      // leading backward items of the root level
  bool items_ready = false;                    // item lists built (build_sweep_items)
  std::vector<int4> h_items_f, h_items_b;      // host copies of the full lists (exclude_sweep_items)
  int fwd_cols = 256, bwd_cols = 32;           // sweep item sizes (sweep.cu choose_item_sizes)
  int small_work = 8192;                       // panel entries of the largest one-item forward front
  int sweep_vec = 2048;                        // doubles of the sweeps' shared front vector (largest front, sweep.cu)
  int sweep_slot = 2560, sweep_bwd_rows = 78;  // ring slot doubles / backward chunk rows (sweep.cu build_sweep_plan)
  int l2_policy_f = 2, l2_policy_b = 2;        // panel loads of the forward / backward sweeps: L2 eviction priority
                                               // (0 default, 1 evict_last, 2 evict_first; sweep.cu choose_item_sizes)
  std::vector<int64_t> h_vec_off;              // nsd x nsn compact front vector offsets (host copy)
  std::vector<int64_t> h_panel_off;            // nsd x nsn panel offsets (host copy)
  std::vector<int64_t> h_front_off;            // nsd x nsn front offsets inside the subdomain's workspace
};

struct cutbddc_gpu {
  int device = 0, rank = 0, world = 1;
  cudaStream_t stream = nullptr;
  std::mutex mu;
  cutbddc_b200::Prof prof;                       // CUTBDDC_PROFILE=1 phase timing

  // ---------------------------------------------------------------- multi-GPU (dist.cu)
  // Subdomains are distributed over ranks; each rank holds the vectors of
  // its local dof space (its subdomains' dofs, dist.cuh). comm == nullptr:
  // no collectives (one rank, or a plan-only distribution).
  ncclComm_t comm = nullptr;
  bool dist_set = false, dist_explicit = false;  // distribution known / set by the caller
  bool plan_only = false;                        // world > 1 without a communicator: plan inspection only
  int dist_block = 0, dist_rank = 0, dist_world = 1;
  int nsd_g = 0;                                 // subdomains of the global partition
  std::vector<int64_t> g_block_ids;              // nsd_g, ascending
  std::vector<int32_t> rank_of_gsd;              // nsd_g
  std::vector<int32_t> lidx_of_gsd;              // nsd_g: index among its rank's subdomains
  std::vector<int32_t> global_of_local;          // nsd
  int maxloc = 0;                                // most subdomains on one rank (stride of gathered partials)
  cutbddc_b200::DevBuf<int32_t> d_gpos;          // nsd_g: position of each subdomain's gathered partial
  cutbddc_b200::DevBuf<int32_t> d_gsd_of_block, d_rank_of_gsd, d_lsd_of_gsd, d_nbr, d_nbr_of_rank;
  cutbddc_b200::DevBuf<int64_t> d_gblock, d_rbase, d_sbase;
  // local dof space: segments of owned dofs per local subdomain, then ghosts
  int64_t n_loc = 0, n_own = 0;
  cutbddc_b200::DevBuf<int32_t> loc_glob;        // n_loc: global dof of each local dof
  cutbddc_b200::DevBuf<int32_t> loc_of_dof;      // n_dof: local dof or -1
  cutbddc_b200::DevBuf<int32_t> seg_ptr;         // nsd + 1
  cutbddc_b200::DevBuf<int4> chunks;             // segment-kernel blocks: (segment or -1, lo, hi, 0) (dist.cuh)
  cutbddc_b200::DevBuf<int32_t> seg_chunk;       // nsd + 1: first chunk of each segment
  cutbddc_b200::DevBuf<double> cpart;            // per chunk partial
  cutbddc_b200::DevBuf<int> tickets;             // per segment
  int64_t n_chunks = 0;
  cutbddc_b200::DevBuf<int32_t> slot_loc;        // nsd*T: local dof of each slot or -1
  cutbddc_b200::DevBuf<int32_t> lcopy_ptr;       // n_loc + 1
  cutbddc_b200::DevBuf<int32_t> lcopy_src;       // copies, ascending global sd: >= 0 slot (sd*T+slot), < 0: -1 - receive index
  cutbddc_b200::DevBuf<int32_t> lowner;          // n_loc: slot of an interior dof (one copy), else -1
  // interface exchange: one message per neighbour rank and direction
  std::vector<int32_t> nbr;                      // neighbour ranks, ascending
  std::vector<int64_t> send_ptr, recv_ptr;       // nbr + 1 offsets into sendbuf / recvbuf
  cutbddc_b200::DevBuf<int32_t> send_src;        // slot of every sent value
  cutbddc_b200::DevBuf<double> sendbuf, recvbuf;

  // ---------------------------------------------------------------- mesh
  int n = 0;                   // cells per axis
  int problem = 0;             // load data: 0 f = 1, g = 0; 1 manufactured (mms.cuh)
  double origin[3] = {0, 0, 0}, h = 0, tol = 0;
  int64_t n_nodes = 0, n_cells = 0, n_dof = 0;
  cutbddc_b200::DevBuf<double> phi;
  cutbddc_b200::DevBuf<uint8_t> cls;
  cutbddc_b200::DevBuf<int32_t> dof_of_node;
  cutbddc_b200::DevBuf<int64_t> node_of_dof;
  cutbddc_b200::DevBuf<double> balls;
  bool mesh_ready = false;

  // ---------------------------------------------------------------- cells
  int64_t n_active = 0, n_cut = 0;
  cutbddc_b200::DevBuf<int64_t> active_cells, cut_cells;
  cutbddc_b200::DevBuf<int32_t> elem_of_cell;
  cutbddc_b200::DevBuf<double> ke, fe, beta;
  cutbddc_b200::DevBuf<double> keS;              // ke packed (upper triangle) SoA [36][ncut] for the operator
  cutbddc_b200::DevBuf<uint8_t> empty;

  // ---------------------------------------------------------------- subdomains
  int block = 0, b1 = 0, slots = 0, nsd = 0, nb = 0;
  std::vector<int64_t> h_block_ids;
  cutbddc_b200::DevBuf<int64_t> block_ids;
  cutbddc_b200::DevBuf<int32_t> sd_of_block;     // nb^3, -1 for empty blocks
  cutbddc_b200::DevBuf<int32_t> slot_dof;        // nsd*T
  cutbddc_b200::DevBuf<double> As;               // nsd*27*T
  cutbddc_b200::DevBuf<uint8_t> ncount, orphan;  // per global dof: |neigh| over all ranks, strong-Dirichlet flag
  cutbddc_b200::DevBuf<uint8_t> vcell;           // per cell: void cut cell (empty volume rule), all ranks
  cutbddc_b200::DevBuf<double> dtot;             // per local dof: sum of A^w diagonals over all copies
  cutbddc_b200::DevBuf<double> odiag;            // per slot: 1/|neigh| at strong-Dirichlet slots, else 0
  cutbddc_b200::DevBuf<double> fs;               // per slot: sub-assembled load vector
  int64_t n_copies = 0;
  int64_t n_if = 0;                              // interface dofs of the global problem

  // ---------------------------------------------------------------- operator
  // Abar is never assembled: Abar x = Σ_w R_w^T A_w R_w x, matrix-free (dist.cu sub_apply)
  cutbddc_b200::DevBuf<double> b;                // assembled rhs, local dofs
  bool assembled = false;
  double t_assembly = 0;

  // ---------------------------------------------------------------- template + factors
  TplSet tI;                                     // plain ND template (interior problems A_II)
  TplSet tK;                                     // shell-root template (K = A + rho C^T C)
  FactorSet fI, fK;                              // interior / Neumann factorisations
  bool has_K = false;                            // false without an interface (one subdomain)
  // K formulation: corner-augmented K_c = A + rho
  // sum_corners e e^T on the plain ND template (tI), coarse basis through
  // H = L^{-1} C^T (k_corner); or the full K = A + rho C^T C on the
  // shell-root template (tK), coarse basis in the root space (fallback when a
  // K_c pivot is tiny or non-positive, or CUTBDDC_K_SHELL=1)
  bool k_corner = true;
  const TplSet& tplK() const { return k_corner ? tI : tK; }
  // mixed K: the corner formulation on most subdomains, the shell-root K on
  // the subdomains whose K_c is singular (floating fragments), factorised in fKs
  bool k_mixed = false;
  int n_shell_sd = 0;  // this rank's subdomains on the shell-root K (mixed)
  FactorSet fKs;
  cutbddc_b200::DevBuf<uint8_t> kform_shell, kform_corner;  // per subdomain (mixed K)
  cutbddc_b200::DevBuf<uint8_t> mask_shell;                 // per slot: present slots of the shell subdomains
  cutbddc_b200::DevBuf<int> ws_badsd;                       // per subdomain: K_c unusable
  cutbddc_b200::DevBuf<uint8_t> mask_int, mask_all;  // per (sd, slot)
  cutbddc_b200::DevBuf<double> diag_add;         // per (sd, slot): rho at corner slots
  cutbddc_b200::DevBuf<uint8_t> corner_row;      // per constraint row: 1 if a corner
  cutbddc_b200::DevBuf<int64_t> fail_slot;       // first failing (sd*T+slot) per factorisation

  // ---------------------------------------------------------------- bddc
  int weighting = 0;
  int n_coarse = 0, m_max = 0;
  int64_t m_total = 0;
  std::vector<int64_t> h_m_off;                   // nsd+1
  cutbddc_b200::DevBuf<int64_t> m_off;            // nsd+1 (constraint rows per sd)
  cutbddc_b200::DevBuf<int64_t> c_ptr;            // m_total+1 (entries per row)
  cutbddc_b200::DevBuf<int32_t> c_slot;
  cutbddc_b200::DevBuf<double> c_val;
  cutbddc_b200::DevBuf<int32_t> coarse_id;        // m_total
  cutbddc_b200::DevBuf<int32_t> row_sd;           // m_total: owning subdomain of each constraint row
  cutbddc_b200::DevBuf<int64_t> cg_ptr;           // n_coarse+1
  cutbddc_b200::DevBuf<int64_t> cg_idx;           // staged row position (dist.cuh), ascending global sd
  // staged coarse layout: rows (and m x m blocks) of every subdomain at
  // rank * maxrows (rank * maxac) + the rank's earlier subdomains' share
  int64_t maxrows = 1, maxac = 1, m_total_g = 0;
  cutbddc_b200::DevBuf<int64_t> srow;             // 3 per staged row: first row of its sd, m, block offset
  cutbddc_b200::DevBuf<int32_t> scoarse;          // coarse id of every staged row
  cutbddc_b200::DevBuf<double> w;                 // nsd*T
  cutbddc_b200::DevBuf<double> rho;               // nsd
  cutbddc_b200::DevBuf<double> ac_loc;            // staged m x m blocks A_c,w (this rank's at rank * maxac + ac_off)
  cutbddc_b200::DevBuf<int64_t> ac_off;           // nsd+1
  cutbddc_b200::DevBuf<double> acoarse;
  cutbddc_b200::DevBuf<double> acoarse_inv;       // X = L_c^{-1} (lower, column-major n_c x n_c)
  cutbddc_b200::DevBuf<double> uvec_c;            // n_c: X g of the coarse solve
  cutbddc_b200::DevBuf<double> acoarse_full;      // A_c^{-1} = X^T X (n_c <= 4096: one GEMV per apply)
  // root-space coarse basis (bddc.cu): per sd, with c_r root columns of K
  // and m constraint rows: S^{-1} (m x m, offsets ac_off) and
  // W_r = (K^{-1})_rr C_r^T (c_r x m, column-major); root_info[sd] =
  // {c_r, root panel offset, root vector offset (sweep), W_r offset}
  cutbddc_b200::DevBuf<double> sinv, wroot, hroot;
  cutbddc_b200::DevBuf<int64_t> root_info;       // corner formulation (see below)
  cutbddc_b200::DevBuf<int64_t> root_info_s;     // shell formulation: {c_r, root panel off, root vec off, W_r off}
  cutbddc_b200::DevBuf<double> hroot_s;          // shell formulation: H = G_r C_r^T
  // corner formulation: H = L^{-1} C^T over each subdomain's present slots in
  // front-column order (column-major, np_sd x m_sd at root_info[4 sd + 3]),
  // hslot[root_info[4 sd + 1] + k] = sd * T + slot of compact position k
  cutbddc_b200::DevBuf<int32_t> hslot;
  cutbddc_b200::DevBuf<double> hcy_part;          // H^T y' chunk partials (bddc.cu h_cy)
  int np_max = 0;
  cutbddc_b200::DevBuf<double> uvec;              // m_total: S^{-1}(zc - cy) per constraint row
  bool bddc_ready = false;
  double t_setup = 0;

  // ---------------------------------------------------------------- work vectors
  cutbddc_b200::DevBuf<double> sv0, sv1, sv2;     // slot vectors nsd*T
  cutbddc_b200::DevBuf<double> sx;                // slot-vector input of the matrix-free operator (dist.cu)
  cutbddc_b200::DevBuf<int32_t> op_rows;          // operator rows: [interior regular | interior | interface] slots
  int64_t rows_nreg = 0, rows_nint = 0, rows_n = 0;
  cutbddc_b200::DevBuf<double> s27;               // constant 27-point stencil of interior cells
  cutbddc_b200::DevBuf<double> ysave;             // big-front forward results, nsd*T
  cutbddc_b200::DevBuf<double> upd;               // solve workspace nsd*upd_total (x nrhs for setup)
  cutbddc_b200::DevBuf<double> gv0, gv2;         // local dof vectors (z0, v)
  cutbddc_b200::DevBuf<double> gl, cy, zc, gc;    // m_total, m_total, n_coarse, n_coarse
  cutbddc_b200::DevBuf<double> partials;          // reduction partials
  cutbddc_b200::DevBuf<double> scal;              // device scalars (pcg)
  cutbddc_b200::DevBuf<int32_t> iscal;            // device int scalars (pcg)

  // persistent scratch (grow-only) so repeated solves allocate nothing
  cutbddc_b200::DevBuf<double> ws_front, ws_upd, ws_s, ws_lc, ws_cpart, ws_q8, ws_kint;
  cutbddc_b200::DevBuf<unsigned long long> ws_fail;
  cutbddc_b200::DevBuf<int64_t> ws_cnt, ws_nc64;
  cutbddc_b200::DevBuf<int32_t> ws_sds, ws_seg, ws_glist, ws_keys, ws_rc, ws_sc, ws_ccount;  // plan scratch (dist.cu)
  cutbddc_b200::DevBuf<uint8_t> ws_nsds, ws_local;
  cutbddc_b200::DevBuf<uint32_t> ws_rmask;
  cutbddc_b200::DevBuf<unsigned int> ws_omask;
  cutbddc_b200::DevBuf<uint8_t> ws_act, ws_cut, ws_tmp, ws_obj;
  cutbddc_b200::DevBuf<double> ws_w8;             // device objects v2: weight tuples (8 per dof)
  cutbddc_b200::DevBuf<double> ws_acc;            // cut cells: the 180 quadrature sums per cell (element.cu)
  cutbddc_b200::DevBuf<int> ws_nvs;
  cutbddc_b200::DevBuf<uint8_t> ws_tmp2;
  cutbddc_b200::DevBuf<int64_t> ws_cells;
  cutbddc_b200::DevBuf<int> ws_flag;
  cutbddc_b200::DevBuf<double> ws_global;             // global-numbered staging vector of the host downloads
  cutbddc_b200::DevBuf<int32_t> ws_cdof;            // setup: the coarse view's object dofs (CSR values)
  cutbddc_b200::DevBuf<int64_t> ws_odofptr;         // setup: the coarse view's dof_ptr
  cutbddc_b200::DevBuf<int32_t> ws_coff;                       // corner coarse basis: front column offsets
  cutbddc_b200::DevBuf<double> ws_x8, ws_y8, ws_u8, ws_v8;      // multi-RHS forward sweep vectors
  DagPlan dag_factor;                              // dense_dag.cu: the subdomain factorisations (one launch)
  std::vector<cudaEvent_t> dag_ev;                 // start/stop event pairs of the last numeric factorisation's launches
  DagPlan dag_dense;                               // dense_dag.cu: the coarse matrix factorisation
  CoarseSparse csparse;                            // coarse_sparse.cu: sparse A_c factor (large n_c)
  bool coarse_sparse = false;                      // the apply solves A_c by csparse

  // pcg vectors
  cutbddc_b200::DevBuf<double> px, pr, pz, pp, pq, pb, hist, lal, lbe;
  cutbddc_b200::DevBuf<double> psl;               // p at every local slot copy (the SpMV's input)
  cudaGraphExec_t graph_exec = nullptr;
  cudaGraphExec_t graph_exec_ref = nullptr;      // several ranks: the iteration with the k % 50 refresh
  long long graph_nodes_ref = 0;
  int graph_max_iter = -1;
  long long graph_nodes = 0;                      // kernel nodes per PCG-iteration graph
  bool graph_while = false;                       // graph_exec runs the whole loop (conditional WHILE node)
  double t_pcg = 0;
};
