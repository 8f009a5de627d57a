// factor.cuh — interfaces of the batched multifrontal factorisation/solves.
#pragma once

#include <functional>

#include "front_desc.cuh"
#include "handle.cuh"

namespace cutbddc_b200 {

struct TplDev {
  const Supernode* sn;
  const int32_t* rows;
  const AmapEntry* amap;
  const int32_t* emap;
  const int32_t* root_pos;
  int T;
  int nsn;
  int root;  // id of the root supernode (last in postorder)
  int64_t rows_total;
};

// Per-subdomain compact structure of one factorisation (see factor.cu):
//   pfx[sd][rows_total]  compact row index of every template row position of
//                        every supernode (-1 when the slot is masked out)
//   rc[sd][nsn]          compact (rows, cols) of each front
//   panel_off / upd_off  offsets of the compact panel / forward update vector
struct FactorDev {
  const int32_t* pfx;
  const int32_t* tpos;  // inverse of pfx: compact row -> template row position
  const int2* rc;
  const int64_t* panel_off;
  const int64_t* upd_off;
  int64_t upd_total;  // doubles of the forward-update workspace per right-hand side
  const FrontDesc* desc;  // per (sd, front) descriptors (sweep plan)
  const int2* gmap;       // per compact front row: update entry of child 0 / 1 landing there, or -1
  const int32_t* cslot;   // per compact front row: sd * T + slot
};

// Matrix fed to the factorisation: the A^w stencil restricted to `mask`
// slots, plus diag_add on the diagonal (may be null) and, on the root front,
// rho_w c c^T for every non-corner constraint row c (K = A + rho C^T C; the
// root of the shell template holds every object node).
struct FactorInput {
  const double* As;
  const uint8_t* mask;
  const double* diag_add;
  int T, b1;
  const int64_t* m_off;
  const int64_t* c_ptr;
  const int32_t* c_slot;
  const double* c_val;
  const uint8_t* corner;
  const double* rho;
};

TplDev tpl_dev(const TplSet& t, int slots);
FactorDev factor_dev(const FactorSet& f);
void upload_template(cutbddc_gpu* h, TplSet& t, bool shell_root);
// which fronts the factorisation tiles (depends on the subdomain count)
void set_split_flags(TplSet& ts, int nsd);
// Symbolic phase of one factorisation: compact front sizes, panel / update /
// front-workspace offsets, the sweep plan.
void factor_symbolic(cutbddc_gpu* h, const TplSet& t, const FactorInput& in, FactorSet& f);
// Numeric phase of one or two factorisations (after factor_symbolic), as one
// dataflow launch when their fronts fit the workspace budget together.
struct FactorJob {
  const TplSet* ts;
  const FactorInput* in;
  FactorSet* f;
  const char* what;       // error message prefix (non-positive pivot)
  bool* failed = nullptr;  // set: a non-positive pivot is reported here instead of thrown
  int* fail_sd = nullptr;  // device, optional: per subdomain, 1 where a pivot was non-positive
};
// `overlap`: host work run after the factorisation is enqueued, before the
// pivot check waits for it (the sweep item lists). append_events: keep the
// previous call's timing events (a second factorisation of the same setup)
void factor_numeric(cutbddc_gpu* h, const std::vector<FactorJob>& jobs, const std::function<void()>& overlap = {},
                    bool append_events = false);
// ysave: nsd x T doubles of scratch (forward results of big fronts).
void solve_device(cutbddc_gpu* h, const TplSet& t, const FactorSet& f, double* X, double* upd, double* ysave,
                  const int* skip);
void solve_k_device(cutbddc_gpu* h, double* X, const int* skip);
// algorithmic bytes of one forward + backward sweep (panel lower parts + front vectors)
double sweep_bytes(const FactorSet& f);
// sweep.cu: dataflow sweeps for one right-hand side (plan built per factorisation)
void build_sweep_plan(cutbddc_gpu* h, const TplSet& ts, FactorSet& f, const std::vector<int64_t>& poff,
                      const std::vector<int64_t>& uoff);
// the sweeps' item lists (host; run while the GPU factorises: factor_numeric's overlap hook)
// exclude (optional, per subdomain): subdomains whose fronts get no items
void build_sweep_items(cutbddc_gpu* h, const TplSet& ts, FactorSet& f, const std::vector<uint8_t>* exclude = nullptr);
void exclude_sweep_items(cutbddc_gpu* h, FactorSet& f, const std::vector<uint8_t>& exclude);  // filter the built lists
void sweep_solve(cutbddc_gpu* h, const TplSet& ts, const FactorSet& f, double* X, double* ysave, double* upd,
                 const int* skip);
enum { kSweepFwd = 0, kSweepBwd = 1, kSweepBwdRoot = 2, kSweepBwdRest = 3, kSweepAttrOnly = 4 };
// sweep.cu: forward sweep of kSweepMultiRhs right-hand sides at once
#ifndef CUTBDDC_MULTI_RHS
#define CUTBDDC_MULTI_RHS 13  // tuned on B200 (cfg4, m_max 37: three passes; 8: 731 us, 13: 554 us, 16: 653 us)
#endif
constexpr int kSweepMultiRhs = CUTBDDC_MULTI_RHS;
void sweep_forward_multi(cutbddc_gpu* h, const TplSet& ts, const FactorSet& f, const double* X, double* ysave,
                         double* upd, double* vbuf8);
void sweep_phase(cutbddc_gpu* h, const TplSet& ts, const FactorSet& f, double* X, double* ysave, double* upd,
                 const int* skip, int phase);
// dense_dag.cu: numeric factorisation of every span as one dataflow launch
struct FactorSpan {
  const TplSet* ts;
  const FactorInput* in;
  FactorSet* f;
  int sd0, sd1;                // subdomains of this factorisation in the launch
  int64_t front_off;           // their front workspace offset in the launch's workspace
  unsigned long long* fail;    // pivot failure report
  int* fail_sd = nullptr;      // per-subdomain failure flags (optional)
};
void dense_dag_factor(cutbddc_gpu* h, const std::vector<FactorSpan>& spans, double* front);
// dense_dag.cu: Cholesky (A, column-major lower, overwritten) and X = L^{-1}
// of one dense SPD matrix; a failing pivot index goes to *fail
void dense_dag_matrix(cutbddc_gpu* h, double* A, double* X, int n, unsigned long long* fail);
// dense_dag.cu: partial Cholesky of independent dense fronts in one launch:
// front q is r x r (column-major lower at F + fo), its first c columns are
// eliminated, the panel [L11^{-1}; L21 L11^{-1}] (r x c, ld r) goes to
// X + po and the trailing (r - c) block becomes the update matrix
void dense_dag_fronts(cutbddc_gpu* h, DagPlan& plan, double* F, double* X, const std::vector<DenseFront>& fronts,
                      unsigned long long* fail);
// coarse_sparse.cu: symbolic (nested dissection on the subdomain lattice),
// numeric factorisation of the dense-stored A_c, and z = A_c^{-1} g
void coarse_sparse_setup(cutbddc_gpu* h, int nc, const std::vector<std::vector<int>>& obj_of_gsd);
void coarse_sparse_factor(cutbddc_gpu* h, const double* Ac, int nc, unsigned long long* fail);
void coarse_sparse_solve(cutbddc_gpu* h, const double* g, double* z, const int* skip);
// peak.cu: FP64 tensor (DMMA) and FP64 FMA throughput microbenchmarks, TFLOP/s
void fp64_peaks(int device, double* dmma_tflops, double* dfma_tflops);

}  // namespace cutbddc_b200
