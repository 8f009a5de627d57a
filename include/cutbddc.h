/* cutbddc.h — C ABI of the B200-native PCG+BDDC solve path.
 *
 * Drop-in boundary for the reference library "cutbddc" (/root/reference):
 * the reference's C boundary exists only as a comment, "the C boundary maps
 * `code` onto cutbddc_status values" (proj/src/core/common.hpp:22-23); its
 * operations are the SPEC.md ops listed beside each entry point below. No
 * torch types cross this boundary: plain pointers, sizes and status codes.
 * Nothing throws across it. Input arrays are borrowed for the duration of the
 * call (copied to the device); outputs go to caller-allocated buffers; a
 * handle owns all device memory until cutbddc_gpu_destroy. A handle is
 * single-caller; separate handles are independent.
 */
#ifndef CUTBDDC_H
#define CUTBDDC_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ErrorCode {InvalidArgument, Config, Io, Singular, Degenerate, NotConverged,
 * Internal} of common.hpp:24-32, plus OK. CUDA and NCCL failures map to
 * CUTBDDC_INTERNAL. */
typedef enum {
  CUTBDDC_OK = 0,
  CUTBDDC_INVALID_ARGUMENT = 1,
  CUTBDDC_CONFIG = 2,
  CUTBDDC_IO = 3,
  CUTBDDC_SINGULAR = 4,
  CUTBDDC_DEGENERATE = 5,
  CUTBDDC_NOT_CONVERGED = 6,
  CUTBDDC_INTERNAL = 7
} cutbddc_status;

/* Thread-local message of the last failing call (pivot index as in
 * linalg.cpp:53-54, subdomain context as in linalg.cpp:86-89 / SPEC.md:383,
 * dimension mismatch as in linalg.cpp:94-95). */
const char* cutbddc_last_error(void);

/* Cell classes, mesh.hpp:17 CellClass {Interior, Exterior, Cut}. */
enum { CUTBDDC_INTERIOR = 0, CUTBDDC_EXTERIOR = 1, CUTBDDC_CUT = 2 };
/* Object kinds, object sets, weighting,
 * variants. */
enum { CUTBDDC_CORNER = 0, CUTBDDC_EDGE = 1, CUTBDDC_FACE = 2 };
enum { CUTBDDC_OBJECTS_C = 0, CUTBDDC_OBJECTS_CE = 1, CUTBDDC_OBJECTS_CEF = 2 };
enum { CUTBDDC_WEIGHT_TOPOLOGICAL = 0, CUTBDDC_WEIGHT_STIFFNESS = 1 };
enum { CUTBDDC_VARIANT_STANDARD = 0, CUTBDDC_VARIANT_V1 = 1, CUTBDDC_VARIANT_V2 = 2 };

typedef struct cutbddc_gpu cutbddc_gpu;

typedef struct {
  int device;      /* CUDA device ordinal */
  int rank;        /* this process' rank (multi-GPU), 0 for one GPU */
  int world_size;  /* number of GPUs (processes), 1 for one GPU */
  const void* nccl_id; /* 128-byte ncclUniqueId (rank 0's, cutbddc_nccl_unique_id); required when
                          world_size > 1; with world_size 1 it creates a one-rank communicator
                          (every exchange runs); NULL: no communicator */
} cutbddc_gpu_opts;

/* Background mesh + level set, MeshParams (mesh.hpp:18-24) and a union of
 * balls (levelset.cpp:22-39 sphere; min-union pattern levelset.cpp:129-133). */
typedef struct {
  int cells[3];
  double box_lo[3], box_hi[3], translation[3];
  int n_balls;
  const double* balls; /* n_balls x {cx, cy, cz, r} */
} cutbddc_geometry;

/* BackgroundMesh view (mesh.hpp:77-80): per-node snapped phi, per-cell
 * class, per-node dof id (-1 = none), as produced by
 * BackgroundMesh::classify (mesh.cpp:114-169). */
typedef struct {
  int cells[3];
  double origin[3], h[3];
  int64_t n_dof;
  const double* phi;        /* (n+1)^3 */
  const uint8_t* cls;       /* n^3 */
  const int32_t* dof_of_node; /* (n+1)^3 */
} cutbddc_mesh_view;

/* SubdomainPartition: block size H/h and the nonempty
 * blocks in ascending block id ((bi*nby+bj)*nbz+bk). */
typedef struct {
  int block;
  int n_sd;
  const int64_t* block_ids;
} cutbddc_partition_view;

/* InterfaceObjects restricted to the selected coarse objects, in coarse-DOF
 * order: kinds[n], dofs (global dof ids) in CSR
 * dof_ptr[n+1], neighbour subdomains in CSR neigh_ptr[n+1]. */
typedef struct {
  int n_objects;
  const int32_t* kinds;
  const int64_t* dof_ptr;
  const int32_t* dofs;
  const int64_t* neigh_ptr;
  const int32_t* neigh;
} cutbddc_coarse_view;

/* SolveReport. residuals must hold max_iter+1 doubles. */
typedef struct {
  int iterations;
  int converged;
  double cond_estimate;
  double lambda_min, lambda_max;
  double* residuals;
  double t_assembly, t_setup, t_pcg; /* device-timed seconds of the last calls */
} cutbddc_solve_report;

cutbddc_status cutbddc_gpu_create(const cutbddc_gpu_opts* opts, cutbddc_gpu** out);
void cutbddc_gpu_destroy(cutbddc_gpu* h);

/* BackgroundMesh::classify (mesh.cpp:114-169) on the device. Outputs
 * (optional, may be NULL) are host buffers of the sizes in cutbddc_mesh_view;
 * n_dof is always written. The mesh stays resident for cutbddc_gpu_assemble. */
cutbddc_status cutbddc_gpu_classify(cutbddc_gpu* h, const cutbddc_geometry* g, double* phi, uint8_t* cls,
                                    int32_t* dof_of_node, int64_t* n_dof);

/* assemble_subassembled + assemble_global:
 * cut quadrature, beta_e, element
 * matrices and the per-subdomain matrices A^w, all on the
 * device. mesh may be NULL to use the mesh left by cutbddc_gpu_classify.
 * dirichlet (optional host buffer, n_dof bytes) receives the strong-Dirichlet
 * (orphan) dof mask. */
cutbddc_status cutbddc_gpu_assemble(cutbddc_gpu* h, const cutbddc_mesh_view* mesh,
                                    const cutbddc_partition_view* part, uint8_t* dirichlet);

/* A^w diagonal entries at every (subdomain, local dof) copy, subdomains in
 * order, local dofs ascending (input of build_weighting / split_edges_v2). */
cutbddc_status cutbddc_gpu_local_diagonals(cutbddc_gpu* h, double* diag, int64_t* n_copies);

/* build_weighting + build_coarse_space:
 * weights, constraint rows, interior / constrained-Neumann factorisations,
 * coarse basis, coarse matrix and its factorisation. */
cutbddc_status cutbddc_gpu_setup_bddc(cutbddc_gpu* h, const cutbddc_coarse_view* coarse, int weighting);

/* krylov::pcg with A = Abar and M = BDDC apply. b may be
 * NULL to use the assembled rhs. x: n_dof output (a distributed handle
 * writes the dofs it owns, see cutbddc_gpu_set_distribution). */
cutbddc_status cutbddc_gpu_pcg(cutbddc_gpu* h, const double* b, double* x, double rtol, int max_iter,
                               cutbddc_solve_report* report);

/* Test hooks: y = Abar x (SparseSymMatrix::apply, linalg.hpp:45; applied
 * matrix-free as Σ_w R_w^T A_w R_w) and z = M r (bddc apply,
 * SPEC.md:388-396), host vectors of n_dof (owned entries written). */
cutbddc_status cutbddc_gpu_spmv(cutbddc_gpu* h, const double* x, double* y);
cutbddc_status cutbddc_gpu_apply_bddc(cutbddc_gpu* h, const double* r, double* z);
/* Assembled rhs b (n_dof) and coarse matrix (n_c x n_c row-major). */
cutbddc_status cutbddc_gpu_rhs(cutbddc_gpu* h, double* b);
cutbddc_status cutbddc_gpu_coarse_matrix(cutbddc_gpu* h, double* ac, int* n_coarse);
/* Per active cell (ascending cell id): beta_e and empty-volume flag. */
cutbddc_status cutbddc_gpu_cells(cutbddc_gpu* h, double* beta, uint8_t* empty, int64_t* n_active);
/* Test hook: cut-cell element data in cut-cell order (ascending cell id):
 * cell ids, 8x8 matrices (row-major) and rhs. Any output may be NULL. */
cutbddc_status cutbddc_gpu_cut_elements(cutbddc_gpu* h, int64_t* cells, double* ke, double* fe, int64_t* n_cut);
/* Test hooks in slot space (nsd x (B+1)^3 slots): the stencil form of A^w
 * (nsd x 27 x T), the factorised matrix masks and diagonal shifts, and an
 * in-place solve with the interior (which=0) or corner-augmented Neumann
 * (which=1) factor. */
cutbddc_status cutbddc_gpu_local_system(cutbddc_gpu* h, double* stencil, uint8_t* mask_interior, uint8_t* mask_present,
                                        double* diag_add, int32_t* slot_dof);
cutbddc_status cutbddc_gpu_local_solve(cutbddc_gpu* h, int which, double* x);
/* Test hook: the tiled dense factorisation the coarse problem uses (one
 * dataflow launch of 64 x 64 tile tasks, POTRF / TRSM / GEMM on DMMA and the
 * explicit inverse) on a plain n x n SPD matrix a (column-major; the lower
 * part is read): l = L (a = L L^T), x = L^{-1}, column-major in their lower
 * parts (the strict upper parts are unspecified); either may be NULL. A non-positive pivot returns
 * CUTBDDC_SINGULAR with its index in *pivot (-1 otherwise). Replaces, for
 * dense matrices, SparseCholesky::compute (linalg.cpp:34-62). */
cutbddc_status cutbddc_gpu_dense_cholesky(cutbddc_gpu* h, int n, const double* a, double* l, double* x,
                                          int64_t* pivot);
/* Statistics (17 slots): [0]=n_dof [1]=n_sd [2]=n_coarse [3]=template slots
 * [4]=factor panel doubles (both factorisations, all subdomains)
 * [5]=supernodes (Neumann template) [6]=levels [7]=max m_w [8]=n_interface
 * [9]=kernel launches so far (process-wide) [10]/[11]=panel doubles of the
 * interior / Neumann factorisation [12]=partial-Cholesky flops of both
 * [13]=world size [14]=1 if the handle owns an NCCL communicator
 * [15]=1 if the constrained Neumann factor is the corner-augmented
 * K_c = A + rho C_corner^T C_corner (else K = A + rho C^T C)
 * [16]=subdomains of this rank on K = A + rho C^T C while the others use K_c
 * (a mixed K: K_c singular there, e.g. a floating fragment); counted in [11]/[12]. */
cutbddc_status cutbddc_gpu_stats(cutbddc_gpu* h, int64_t* stats);
/* Page-lock a caller-owned host buffer (cudaHostRegister) so the uploads of
 * the mesh view in cutbddc_gpu_assemble and the download of the solution in
 * cutbddc_gpu_pcg run as asynchronous DMA instead of staged pageable copies.
 * Optional: the reference's BackgroundMesh arrays (mesh.hpp:77-80) live for
 * many solves, so the caller pins them once. unpin before freeing. */
cutbddc_status cutbddc_host_pin(void* ptr, size_t bytes);
cutbddc_status cutbddc_host_unpin(void* ptr);

/* Measurement hook: average device time of the triangular-solve sweeps of
 * one BDDC apply (interior, Neumann, interior) over `reps` repetitions, and
 * their algorithmic bytes (panel lower parts + front vectors). */
cutbddc_status cutbddc_gpu_time_solves(cutbddc_gpu* h, int reps, double* seconds, double* bytes);

/* Measurement hook: warm average device time (microseconds, `reps`
 * back-to-back calls) of the pieces of one PCG iteration: us[0] the
 * matrix-free operator on every row, [1] on interface rows, [2] on
 * interior rows, [3] one interface sum, [4] one BDDC apply, [5] its three
 * triangular solves, [6] one SpMV (operator + interface sum), [7] unused. */
cutbddc_status cutbddc_gpu_time_parts(cutbddc_gpu* h, int reps, double* us);

/* Measurement hook: device time of the numeric factorisation launch(es)
 * (k_dense_dag) of the last setup, its partial-Cholesky flops
 * (sum over fronts of c^3/3 + (r-c)c^2 + (r-c)^2 c; the reference op is
 * SparseCholesky's factorisation, linalg.cpp:38-56) and the flops of the
 * explicit inverse panels the sweeps use (c^3/3 + (r-c)c^2). */
cutbddc_status cutbddc_gpu_time_factor(cutbddc_gpu* h, double* seconds, double* flops_cholesky, double* flops_inverse);
/* FP64 roofline denominators measured on `device`: mma.sync m8n8k4 f64
 * (DMMA) and DFMA throughput, TFLOP/s. */
cutbddc_status cutbddc_fp64_peak(int device, double* dmma_tflops, double* dfma_tflops);

/* Host-side partition and interface objects (the caller side of the
 * boundary; reference ops build_partition SPEC.md:295-303, classify_objects
 * :304-312, split_edges_v1 :313-321, split_edges_v2 :322-330). The result is
 * owned by the library until cutbddc_objects_free. */
typedef struct {
  int n_sd;
  int64_t* block_ids;
  int n_objects;
  int32_t* kinds;
  int64_t* dof_ptr;
  int32_t* dofs;
  int64_t* neigh_ptr;
  int32_t* neigh;
} cutbddc_objects;

cutbddc_status cutbddc_build_partition(const cutbddc_mesh_view* mesh, int block, int64_t* n_sd, int64_t* block_ids);
/* weights: per (subdomain, local dof) copy (order of cutbddc_gpu_local_diagonals),
 * needed only for CUTBDDC_VARIANT_V2 (else NULL). dirichlet: orphan mask. */
cutbddc_status cutbddc_classify_objects(const cutbddc_mesh_view* mesh, const cutbddc_partition_view* part,
                                        const uint8_t* dirichlet, int objects, int variant, const double* weights,
                                        cutbddc_objects** out);
void cutbddc_objects_free(cutbddc_objects* o);
/* classify_objects and the edge splits split_edges_v1 /
 * split_edges_v2 on the device from the mesh, the
 * strong-Dirichlet mask and (v2) the subdomain matrices left by
 * cutbddc_gpu_assemble: the same objects, bit for bit, as
 * cutbddc_classify_objects. v2 needs every subdomain on this handle
 * (CUTBDDC_CONFIG on a distributed one). Free with cutbddc_objects_free. */
cutbddc_status cutbddc_gpu_classify_objects(cutbddc_gpu* h, int objects, int variant, cutbddc_objects** out);

/* Multi-GPU (one process and one handle per GPU). Subdomains are assigned
 * to ranks in contiguous Morton-curve chunks of equal estimated cost
 * (cost may be NULL: unit cost). rank_of_sd: n_sd outputs. */
cutbddc_status cutbddc_assign_subdomains(const cutbddc_partition_view* part, int cells, int world, const double* cost,
                                         int32_t* rank_of_sd);
/* 128-byte NCCL unique id (rank 0 creates it; the caller broadcasts it). */
cutbddc_status cutbddc_nccl_unique_id(void* id128);
/* Distribution of the subdomains over ranks (one process and one handle per
 * GPU). Every rank passes the same GLOBAL partition and rank_of_sd (e.g.
 * from cutbddc_assign_subdomains); the handle then assembles, factorises and
 * solves the subdomains with rank_of_sd == rank, and cutbddc_gpu_assemble
 * takes that same global partition. Call before cutbddc_gpu_assemble. With a
 * communicator, rank / world must be the handle's own; a handle without one
 * may take any rank's view to inspect its exchange plan
 * (cutbddc_gpu_exchange_plan): assembly then builds the plan only, and the
 * numerical entry points return CUTBDDC_CONFIG.
 *
 * Vectors at the boundary are always in global dof numbering (n_dof
 * doubles). A distributed handle reads its local dofs from inputs and writes
 * the dofs it OWNS into outputs (a dof is owned by the rank of its
 * lowest-numbered subdomain: exactly one rank), leaving other entries
 * untouched. Every scalar (dots, iteration counts, residual histories) and
 * every owned entry is the same, bit for bit, for any world size. */
cutbddc_status cutbddc_gpu_set_distribution(cutbddc_gpu* h, const cutbddc_partition_view* part,
                                            const int32_t* rank_of_sd, int rank, int world);

/* Problem data of the load vector: the BASELINE runs use
 * f = 1 and g^D = 0 (CUTBDDC_PROBLEM_UNIT_LOAD, the default);
 * CUTBDDC_PROBLEM_MANUFACTURED is manufactured(u-case) with u =
 * sin(5 pi |x|) (§5.1): f = -lap u, g^D = u on the embedded
 * boundary through the Nitsche terms. Set before cutbddc_gpu_assemble. */
enum { CUTBDDC_PROBLEM_UNIT_LOAD = 0, CUTBDDC_PROBLEM_MANUFACTURED = 1 };
cutbddc_status cutbddc_gpu_set_problem(cutbddc_gpu* h, int problem);
/* error_norms of the manufactured problem: |u_h - u|_L2
 * and the H1 seminorm |u_h - u|_H1 over the cut-aware volume rules. x:
 * global-numbered nodal values (NULL: the last PCG solution). Collective. */
cutbddc_status cutbddc_gpu_error_norms(cutbddc_gpu* h, const double* x, double* l2, double* h1);

/* Interface exchange plan of one rank (dist.cu builds it on the device;
 * cutbddc_build_exchange_plan builds the same plan on the host):
 *   local dofs: loc_glob[n_loc] global dof ids, segment by segment — the
 *     dofs whose lowest subdomain is local subdomain s are
 *     [seg_ptr[s], seg_ptr[s+1]) (ascending global), the ghost dofs (owned
 *     by another rank) follow from seg_ptr[n_sd_local];
 *   copies of local dof i, ascending global subdomain: copy_src[copy_ptr[i]
 *     .. copy_ptr[i+1]), >= 0: local slot index (local sd * slots + slot of
 *     its (H/h+1)^3 lattice), < 0: receive-buffer index -1 - src;
 *   neighbour ranks nbr[n_nbr] (ascending); message to / from nbr[k]:
 *     send_src[send_ptr[k] .. send_ptr[k+1]) local slot indices, received
 *     into [recv_ptr[k], recv_ptr[k+1]). Messages list the shared dofs in
 *     ascending global dof, each dof's copies in ascending subdomain. */
typedef struct {
  int64_t n_loc, n_own;
  int n_sd_local, n_nbr;
  int32_t* loc_glob;
  int32_t* seg_ptr;
  int32_t* copy_ptr;
  int32_t* copy_src;
  int32_t* nbr;
  int64_t* send_ptr;
  int32_t* send_src;
  int64_t* recv_ptr;
} cutbddc_exchange_plan;
cutbddc_status cutbddc_build_exchange_plan(const cutbddc_mesh_view* mesh, const cutbddc_partition_view* part,
                                           const int32_t* rank_of_sd, int rank, int world,
                                           cutbddc_exchange_plan** out);
cutbddc_status cutbddc_gpu_exchange_plan(cutbddc_gpu* h, cutbddc_exchange_plan** out);
void cutbddc_exchange_plan_free(cutbddc_exchange_plan* p);

#ifdef __cplusplus
}
#endif

#endif /* CUTBDDC_H */
