// pcg.cu — preconditioned CG on the device (K4 SpMV, K11 vector ops/dots).
//
// krylov::pcg with the pins of SURVEY.md Appendix B.7:
// x0 = 0, residuals[0] = |b|, r <- b - Abar x after the update at every
// iteration k with k % 50 == 0, stop at the first k with |r|_2 < rtol |b|_2,
// <p,Ap> <= 0 or <r,Mr> <= 0 -> indefiniteness error, max_iter -> a
// non-converged report. Lanczos alpha/beta are recorded for
// condition_estimate (evaluated on the host).
//
// Vectors live in the rank's local dof space (dist.cuh). Abar p is the
// matrix-free sub-assembled product plus the interface sum. Every dot is a
// per-subdomain partial over the subdomain's owned segment, all-gathered
// over ranks and summed in global subdomain order inside each consumer
// kernel: the scalars are the same bits on 1, 2, 4 or 8 GPUs, so every rank
// takes the same branch at the same iteration.
//
// One GPU: the whole loop is one CUDA graph with a conditional WHILE node,
// all scalars on the device. Several GPUs: one captured graph per iteration
// (with or without the k % 50 refresh), launched in batches by the host; a
// device "done" flag turns the kernels of a finished solve into no-ops.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <vector>

#include "bddc.cuh"
#include "comm.cuh"
#include "dist.cuh"

namespace cutbddc_b200 {
namespace {

// rz ping-pongs between S_RZ (even iterations) and S_RZ1 (odd): the fused
// beta/p-update kernel reads the old value in every block while block 0
// stores the new one.
enum { S_RZ = 0, S_PQ, S_ALPHA, S_BETA, S_STOP, S_RN, S_RZ1, S_COUNT };
__device__ __forceinline__ int rz_slot(int k) { return (k & 1) ? S_RZ1 : S_RZ; }
// I_NOREF: 1 unless this iteration replaces r by b - Abar x (k % 50 == 0)
enum { I_DONE = 0, I_ITER, I_ERR, I_ITERS, I_CONV, I_MAXIT, I_NOREF, I_COUNT };

struct Fin {  // where the gathered partials are summed from
  const int32_t* gpos;
  int nsd_g;
};

// q = Σ_copies Y (Abar p), and the p.q partials
__global__ void __launch_bounds__(kSegThreads) k_spmv_dot(SegArgs a, const int32_t* __restrict__ cptr,
                                                          const int32_t* __restrict__ csrc, const double* __restrict__ Y,
                                                          const double* __restrict__ recv, const double* __restrict__ p,
                                                          double* __restrict__ q, const int* __restrict__ skip) {
  if (skip && *skip) return;
  int lo, hi;
  const int seg = seg_range(a, lo, hi);
  double acc = 0.0;
  for (int i = lo + threadIdx.x; i < hi; i += kSegThreads) {
    double v = 0.0;
    for (int32_t c = cptr[i]; c < cptr[i + 1]; ++c) {
      const int32_t src = csrc[c];
      v += src >= 0 ? Y[src] : recv[-1 - src];
    }
    q[i] = v;
    acc += p[i] * v;
  }
  if (seg < 0 || !a.part) return;
  seg_commit(a, seg, acc);
}

// partials of a.b
__global__ void __launch_bounds__(kSegThreads) k_seg_dot(SegArgs a, const double* __restrict__ x,
                                                         const double* __restrict__ y) {
  int lo, hi;
  const int seg = seg_range(a, lo, hi);
  if (seg < 0) return;
  double acc = 0.0;
  for (int i = lo + threadIdx.x; i < hi; i += kSegThreads) acc += x[i] * y[i];
  seg_commit(a, seg, acc);
}

// alpha = rz / pq (pq from the gathered partials, the same in every block),
// x += alpha p, r -= alpha q, and the r.r partials (not at a refresh
// iteration: k_refresh replaces r and writes them)
__global__ void __launch_bounds__(kSegThreads) k_update_xr(SegArgs a, Fin f, const double* __restrict__ pq_part,
                                                           double* __restrict__ sc, const double* __restrict__ p,
                                                           const double* __restrict__ q, double* __restrict__ x,
                                                           double* __restrict__ r, double* __restrict__ lal,
                                                           int* __restrict__ is) {
  if (is[I_DONE]) return;
  const int k = is[I_ITER];
  const double pq = finish_partials(pq_part, f.gpos, f.nsd_g);
  if (!(pq > 0.0)) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      sc[S_PQ] = pq;
      is[I_ERR] = 1;
      is[I_DONE] = 1;
      is[I_NOREF] = 1;
      is[I_ITERS] = k;
    }
    return;
  }
  const double al = sc[rz_slot(k)] / pq;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    sc[S_PQ] = pq;
    sc[S_ALPHA] = al;
    lal[k - 1] = al;
  }
  int lo, hi;
  const int seg = seg_range(a, lo, hi);
  double acc = 0.0;
  for (int i = lo + threadIdx.x; i < hi; i += kSegThreads) {
    x[i] += al * p[i];
    const double ri = r[i] - al * q[i];
    r[i] = ri;
    acc += ri * ri;
  }
  if (seg < 0 || k % 50 == 0) return;
  seg_commit(a, seg, acc);
}

// true residual refresh at k % 50 == 0: r = b - Σ_copies Y (Y = A_w x_w),
// and the r.r partials
__global__ void __launch_bounds__(kSegThreads) k_refresh(SegArgs a, const int32_t* __restrict__ cptr,
                                                         const int32_t* __restrict__ csrc, const double* __restrict__ Y,
                                                         const double* __restrict__ recv, const double* __restrict__ b,
                                                         double* __restrict__ r, const int* __restrict__ is) {
  if (is[I_NOREF]) return;
  int lo, hi;
  const int seg = seg_range(a, lo, hi);
  double acc = 0.0;
  for (int i = lo + threadIdx.x; i < hi; i += kSegThreads) {
    double v = 0.0;
    for (int32_t c = cptr[i]; c < cptr[i + 1]; ++c) {
      const int32_t src = csrc[c];
      v += src >= 0 ? Y[src] : recv[-1 - src];
    }
    const double ri = b[i] - v;
    r[i] = ri;
    acc += ri * ri;
  }
  if (seg < 0) return;
  seg_commit(a, seg, acc);
}

// |r| -> history, convergence / max_iter test
__global__ void __launch_bounds__(kSegThreads) k_check(Fin f, const double* __restrict__ rr_part,
                                                       double* __restrict__ sc, int* __restrict__ is,
                                                       double* __restrict__ hist) {
  if (is[I_DONE]) return;
  const double rr = finish_partials(rr_part, f.gpos, f.nsd_g);
  if (threadIdx.x == 0) {
    const double rn = sqrt(rr);
    const int k = is[I_ITER];
    sc[S_RN] = rn;
    hist[k] = rn;
    if (rn < sc[S_STOP]) {
      is[I_DONE] = 1;
      is[I_CONV] = 1;
      is[I_ITERS] = k;
    } else if (k >= is[I_MAXIT]) {
      is[I_DONE] = 1;
      is[I_CONV] = 0;
      is[I_ITERS] = k;
    }
  }
}

// beta = rz_new / rz (every block from the same gathered partials; rz_new to
// the other ping-pong slot), p = z + beta p
__global__ void __launch_bounds__(kSegThreads) k_update_p(int64_t nloc, Fin f, const double* __restrict__ rz_part,
                                                          double* __restrict__ sc, const double* __restrict__ z,
                                                          double* __restrict__ p, double* __restrict__ lbe,
                                                          const int32_t* __restrict__ cptr,
                                                          const int32_t* __restrict__ csrc, double* __restrict__ Ps,
                                                          int* __restrict__ is) {
  if (is[I_DONE]) return;
  const int k = is[I_ITER];
  const double rz = finish_partials(rz_part, f.gpos, f.nsd_g);
  if (!(rz > 0.0)) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      is[I_ERR] = 2;
      is[I_DONE] = 1;
      is[I_NOREF] = 1;
      is[I_ITERS] = k;
    }
    return;
  }
  const double beta = rz / sc[rz_slot(k)];
  const int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i0 == 0) {
    sc[S_BETA] = beta;
    sc[rz_slot(k + 1)] = rz;
    lbe[k - 1] = beta;
  }
  for (int64_t i = i0; i < nloc; i += (int64_t)gridDim.x * blockDim.x) {
    const double pi = z[i] + beta * p[i];
    p[i] = pi;
    for (int32_t c = cptr[i]; c < cptr[i + 1]; ++c)  // p at its local slot copies (the next SpMV's input)
      if (csrc[c] >= 0) Ps[csrc[c]] = pi;
  }
}

// p = z and its slot copies
__global__ void k_init_p(int64_t nloc, const double* __restrict__ z, double* __restrict__ p,
                         const int32_t* __restrict__ cptr, const int32_t* __restrict__ csrc, double* __restrict__ Ps) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nloc; i += (int64_t)gridDim.x * blockDim.x) {
    p[i] = z[i];
    for (int32_t c = cptr[i]; c < cptr[i + 1]; ++c)
      if (csrc[c] >= 0) Ps[csrc[c]] = z[i];
  }
}

__global__ void k_next(int* __restrict__ is) {
  if (is[I_DONE]) return;
  const int k = is[I_ITER] + 1;
  is[I_ITER] = k;
  is[I_NOREF] = k % 50 != 0;
}

// |b| -> residuals[0] and the stop threshold rtol |b|
__global__ void __launch_bounds__(kSegThreads) k_init_norm(Fin f, const double* __restrict__ bb_part, double rtol,
                                                           double* __restrict__ sc, double* __restrict__ hist) {
  const double bb = finish_partials(bb_part, f.gpos, f.nsd_g);
  if (threadIdx.x == 0) {
    const double bn = sqrt(bb);
    hist[0] = bn;
    sc[S_STOP] = rtol * bn;
  }
}

// initial: rz = r.z (after z = M r), p = z
__global__ void __launch_bounds__(kSegThreads) k_init_rz(Fin f, const double* __restrict__ rz_part,
                                                         double* __restrict__ sc, int* __restrict__ is) {
  const double rz = finish_partials(rz_part, f.gpos, f.nsd_g);
  if (threadIdx.x == 0) {
    sc[rz_slot(1)] = rz;
    if (!(rz > 0.0)) {
      is[I_ERR] = 2;
      is[I_DONE] = 1;
      is[I_NOREF] = 1;
      is[I_ITERS] = 0;
    }
  }
}

__global__ void k_copy(int64_t n, const double* __restrict__ a, double* __restrict__ b) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) b[i] = a[i];
}

// Last node of the whole-solve graph's WHILE body: k_next, then the loop
// condition (another iteration unless done).
__global__ void k_next_cond(cudaGraphConditionalHandle hc, int* __restrict__ is) {
  if (!is[I_DONE]) {
    const int k = is[I_ITER] + 1;
    is[I_ITER] = k;
    is[I_NOREF] = k % 50 != 0;
  }
  cudaGraphSetConditional(hc, is[I_DONE] ? 0u : 1u);
}

constexpr int kFlatBlocks = 592;  // 4 x 148 SMs for the flat vector kernels

Fin fin(const cutbddc_gpu* h) { return Fin{h->d_gpos.p, h->nsd_g}; }
double* part0(cutbddc_gpu* h) { return h->partials.p; }
double* part1(cutbddc_gpu* h) { return h->partials.p + (int64_t)h->dist_world * h->maxloc; }

// One iteration; refresh: include the k % 50 replacement of r (its kernels
// check the device flag; with several ranks it is its own graph, so its
// exchange runs only where it is needed)
void enqueue_iteration(cutbddc_gpu* h, bool refresh, const cudaGraphConditionalHandle* hc = nullptr) {
  cudaStream_t s = h->stream;
  int* is = h->iscal.p;
  double* sc = h->scal.p;
  const int sg = seg_grid(h);
  // q = Abar p (p's slot copies kept by k_update_p / k_init_p)
  sub_apply(h, kSubAll, nullptr, h->psl.p, h->sv2.p, is);
  iface_exchange(h, h->sv2.p, nullptr, is);
  k_spmv_dot<<<sg, kSegThreads, 0, s>>>(seg_args(h, part0(h)), h->lcopy_ptr.p, h->lcopy_src.p, h->sv2.p, h->recvbuf.p,
                                        h->pp.p, h->pq.p, is);
  CB_LAUNCH();
  gather_partials(h, part0(h));
  k_update_xr<<<sg, kSegThreads, 0, s>>>(seg_args(h, part1(h)), fin(h), part0(h), sc, h->pp.p, h->pq.p, h->px.p,
                                         h->pr.p, h->lal.p, is);
  CB_LAUNCH();
  if (refresh) {
    sub_apply(h, kSubAll, h->px.p, nullptr, h->sv2.p, is + I_NOREF);
    iface_exchange(h, h->sv2.p, nullptr, is + I_NOREF);
    k_refresh<<<sg, kSegThreads, 0, s>>>(seg_args(h, part1(h)), h->lcopy_ptr.p, h->lcopy_src.p, h->sv2.p,
                                         h->recvbuf.p, h->pb.p, h->pr.p, is);
    CB_LAUNCH();
  }
  gather_partials(h, part1(h));
  k_check<<<1, kSegThreads, 0, s>>>(fin(h), part1(h), sc, is, h->hist.p);
  CB_LAUNCH();
  apply_bddc_device(h, h->pr.p, h->pz.p, is, part0(h));
  gather_partials(h, part0(h));
  k_update_p<<<kFlatBlocks, kSegThreads, 0, s>>>(h->n_loc, fin(h), part0(h), sc, h->pz.p, h->pp.p, h->lbe.p,
                                                 h->lcopy_ptr.p, h->lcopy_src.p, h->psl.p, is);
  CB_LAUNCH();
  if (hc)  // body of the WHILE node: advance and set the loop condition together
    k_next_cond<<<1, 1, 0, s>>>(*hc, is);
  else
    k_next<<<1, 1, 0, s>>>(is);
  CB_LAUNCH();
}

// One graph for the whole PCG loop on one GPU: a conditional WHILE node whose
// body is the captured iteration ending in k_next_cond. No host polling and no
// no-op iterations after convergence. false (and nothing kept) if the driver
// refuses any step; the caller then uses per-iteration graph launches.
bool build_while_graph(cutbddc_gpu* h) {
  cudaStream_t s = h->stream;
  cudaGraph_t g = nullptr;
  auto fail = [&] {
    cudaGetLastError();
    if (g) cudaGraphDestroy(g);
    return false;
  };
  if (cudaGraphCreate(&g, 0) != cudaSuccess) return fail();
  cudaGraphConditionalHandle hc;
  if (cudaGraphConditionalHandleCreate(&hc, g, 1u, cudaGraphCondAssignDefault) != cudaSuccess) return fail();
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = hc;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t node;
  if (cudaGraphAddNode(&node, g, nullptr, 0, &cp) != cudaSuccess) return fail();
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  const long long c0 = g_kernel_launches.load();
  if (cudaStreamBeginCaptureToGraph(s, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal) != cudaSuccess)
    return fail();
  enqueue_iteration(h, true, &hc);
  const cudaError_t launch_err = cudaGetLastError();
  const cudaError_t cap_err = cudaStreamEndCapture(s, &body);
  g_kernel_launches.store(c0);  // captured, not executed
  if (launch_err != cudaSuccess || cap_err != cudaSuccess) return fail();
  size_t nodes = 0;
  if (cudaGraphGetNodes(body, nullptr, &nodes) != cudaSuccess) return fail();
  if (cudaGraphInstantiate(&h->graph_exec, g, 0) != cudaSuccess) {
    h->graph_exec = nullptr;
    return fail();
  }
  cudaGraphDestroy(g);
  h->graph_nodes = (long long)nodes;
  h->graph_while = true;
  return true;
}

// per-iteration graph (several ranks: NCCL calls inside)
cudaGraphExec_t capture_iteration(cutbddc_gpu* h, bool refresh, long long* nodes) {
  cudaStream_t s = h->stream;
  cudaGraph_t g;
  cudaGraphExec_t ex;
  const long long c0 = g_kernel_launches.load();
  CB_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
  enqueue_iteration(h, refresh);
  CB_CUDA(cudaStreamEndCapture(s, &g));
  CB_CUDA(cudaGraphInstantiate(&ex, g, 0));
  size_t n = 0;
  CB_CUDA(cudaGraphGetNodes(g, nullptr, &n));
  *nodes = (long long)n;
  g_kernel_launches.store(c0);  // captured, not executed
  CB_CUDA(cudaGraphDestroy(g));
  return ex;
}

// SPEC.md:440-448 on the host: extreme eigenvalues of the Lanczos tridiagonal
// by Sturm bisection.
void lanczos_extremes(const std::vector<double>& al, const std::vector<double>& be, double& lmin, double& lmax) {
  const int k = (int)al.size();
  std::vector<double> d((size_t)k), e((size_t)k, 0.0);
  for (int i = 0; i < k; ++i) {
    d[(size_t)i] = 1.0 / al[(size_t)i] + (i > 0 ? be[(size_t)i - 1] / al[(size_t)i - 1] : 0.0);
    if (i + 1 < k) e[(size_t)i] = std::sqrt(be[(size_t)i]) / al[(size_t)i];
  }
  double lo = 1e300, hi = -1e300;
  for (int i = 0; i < k; ++i) {
    const double r = (i > 0 ? std::fabs(e[(size_t)i - 1]) : 0.0) + (i + 1 < k ? std::fabs(e[(size_t)i]) : 0.0);
    lo = std::min(lo, d[(size_t)i] - r);
    hi = std::max(hi, d[(size_t)i] + r);
  }
  auto below = [&](double x) {
    int c = 0;
    double q = d[0] - x;
    if (q < 0) ++c;
    for (int i = 1; i < k; ++i) {
      q = d[(size_t)i] - x - e[(size_t)i - 1] * e[(size_t)i - 1] / (q == 0.0 ? 1e-300 : q);
      if (q < 0) ++c;
    }
    return c;
  };
  auto kth = [&](int idx) {
    double a = lo, b = hi;
    for (int it = 0; it < 200; ++it) {
      const double m = 0.5 * (a + b);
      (below(m) > idx ? b : a) = m;
    }
    return 0.5 * (a + b);
  };
  lmin = kth(0);
  lmax = kth(k - 1);
}

}  // namespace

void spmv_device(cutbddc_gpu* h, const double* x, double* y) {
  if (h->plan_only) throw Failure(CUTBDDC_CONFIG, "spmv: plan-only distribution (no communicator)");
  h->sv2.alloc((size_t)h->nsd * h->slots);
  sub_apply(h, kSubAll, x, nullptr, h->sv2.p, nullptr);
  iface_exchange(h, h->sv2.p, nullptr, nullptr);
  iface_sum(h, h->sv2.p, nullptr, y, nullptr);
}

void pcg_device(cutbddc_gpu* h, const double* b_loc, double rtol, int max_iter, cutbddc_solve_report* rep) {
  if (!h->bddc_ready) throw Failure(CUTBDDC_INVALID_ARGUMENT, "pcg: setup_bddc first");
  if (max_iter < 1) throw Failure(CUTBDDC_INVALID_ARGUMENT, "pcg: max_iter must be >= 1");
  cudaStream_t s = h->stream;
  const int64_t nl = std::max<int64_t>(1, h->n_loc);
  for (auto* v : {&h->px, &h->pr, &h->pz, &h->pp, &h->pq, &h->pb}) v->alloc((size_t)nl);
  h->psl.alloc((size_t)h->nsd * h->slots);
  h->hist.alloc((size_t)max_iter + 1);
  h->lal.alloc((size_t)max_iter + 1);
  h->lbe.alloc((size_t)max_iter + 1);
  h->partials.alloc((size_t)2 * h->dist_world * h->maxloc);  // p.q / r.z, then r.r (gathered layout)
  h->partials.zero(s);
  h->scal.alloc(S_COUNT);
  h->iscal.alloc(I_COUNT);
  cudaEvent_t e0, e1;
  CB_CUDA(cudaEventCreate(&e0));
  CB_CUDA(cudaEventCreate(&e1));
  CB_CUDA(cudaEventRecord(e0, s));
  const int sg = seg_grid(h);
  k_copy<<<kFlatBlocks, kSegThreads, 0, s>>>(h->n_loc, b_loc, h->pb.p);
  CB_LAUNCH();
  k_copy<<<kFlatBlocks, kSegThreads, 0, s>>>(h->n_loc, b_loc, h->pr.p);
  CB_LAUNCH();
  h->px.zero(s);
  h->iscal.zero(s);
  h->scal.zero(s);
  k_seg_dot<<<sg, kSegThreads, 0, s>>>(seg_args(h, part1(h)), h->pb.p, h->pb.p);
  CB_LAUNCH();
  gather_partials(h, part1(h));
  k_init_norm<<<1, kSegThreads, 0, s>>>(fin(h), part1(h), rtol, h->scal.p, h->hist.p);
  CB_LAUNCH();
  double bnorm = 0.0;
  CB_CUDA(cudaMemcpyAsync(&bnorm, h->hist.p, sizeof(double), cudaMemcpyDeviceToHost, s));
  CB_CUDA(cudaStreamSynchronize(s));
  int conv = 0, iters = 0, err = 0;
  if (bnorm == 0.0) {
    h->px.zero(s);
    conv = 1;
  } else {
    const int host_is[I_COUNT] = {0, 1, 0, 0, 0, max_iter, 1};
    CB_CUDA(cudaMemcpyAsync(h->iscal.p, host_is, sizeof(host_is), cudaMemcpyHostToDevice, s));
    apply_bddc_device(h, h->pr.p, h->pz.p, nullptr, part0(h));
    gather_partials(h, part0(h));
    k_init_rz<<<1, kSegThreads, 0, s>>>(fin(h), part0(h), h->scal.p, h->iscal.p);
    CB_LAUNCH();
    k_init_p<<<kFlatBlocks, kSegThreads, 0, s>>>(h->n_loc, h->pz.p, h->pp.p, h->lcopy_ptr.p, h->lcopy_src.p, h->psl.p);
    CB_LAUNCH();
    if (h->graph_exec && h->graph_max_iter != max_iter) {
      cudaGraphExecDestroy(h->graph_exec);
      h->graph_exec = nullptr;
    }
    if (h->graph_exec_ref && h->graph_max_iter != max_iter) {
      cudaGraphExecDestroy(h->graph_exec_ref);
      h->graph_exec_ref = nullptr;
    }
    const bool one_rank = h->dist_world == 1;
    if (!h->graph_exec && one_rank && !std::getenv("CUTBDDC_NO_WHILE_GRAPH")) {
      h->graph_max_iter = max_iter;
      build_while_graph(h);
    }
    if (!h->graph_exec) {
      h->graph_max_iter = max_iter;
      h->graph_while = false;
      // one rank: the refresh kernels check the device flag; several ranks:
      // a second graph carries the refresh (and its exchange)
      h->graph_exec = capture_iteration(h, one_rank, &h->graph_nodes);
      if (!one_rank) h->graph_exec_ref = capture_iteration(h, true, &h->graph_nodes_ref);
    }
    int is_host[I_COUNT] = {0};
    int launched = 0, batch = 4;
    if (h->graph_while) {
      CB_CUDA(cudaGraphLaunch(h->graph_exec, s));
      CB_CUDA(cudaMemcpyAsync(is_host, h->iscal.p, sizeof(is_host), cudaMemcpyDeviceToHost, s));
      CB_CUDA(cudaStreamSynchronize(s));
      g_kernel_launches.fetch_add(h->graph_nodes * (long long)std::max(1, is_host[I_ITER]));  // loop bodies run
    }
    while (!h->graph_while) {
      for (int q = 0; q < batch && launched < max_iter; ++q, ++launched) {
        const bool ref = !one_rank && (launched + 1) % 50 == 0;  // iteration k = launched + 1
        CB_CUDA(cudaGraphLaunch(ref ? h->graph_exec_ref : h->graph_exec, s));
        g_kernel_launches.fetch_add(ref ? h->graph_nodes_ref : h->graph_nodes);
      }
      CB_CUDA(cudaMemcpyAsync(is_host, h->iscal.p, sizeof(is_host), cudaMemcpyDeviceToHost, s));
      CB_CUDA(cudaStreamSynchronize(s));
      if (is_host[I_DONE] || launched >= max_iter) break;
      batch = std::min(8, batch * 2);
    }
    conv = is_host[I_CONV];
    iters = is_host[I_ITERS];
    err = is_host[I_ERR];
  }
  CB_CUDA(cudaEventRecord(e1, s));
  CB_CUDA(cudaEventSynchronize(e1));
  float ms = 0;
  CB_CUDA(cudaEventElapsedTime(&ms, e0, e1));
  h->t_pcg = ms * 1e-3;
  CB_CUDA(cudaEventDestroy(e0));
  CB_CUDA(cudaEventDestroy(e1));
  if (err == 1) throw Failure(CUTBDDC_INTERNAL, "pcg: operator is not positive definite (<p,Ap> <= 0)");
  if (err == 2) throw Failure(CUTBDDC_INTERNAL, "pcg: preconditioner is not positive definite (<r,Mr> <= 0)");
  if (rep) {
    rep->iterations = iters;
    rep->converged = conv;
    rep->cond_estimate = 0;
    rep->lambda_min = rep->lambda_max = 0;
    if (rep->residuals) CB_CUDA(cudaMemcpy(rep->residuals, h->hist.p, sizeof(double) * (size_t)(iters + 1), cudaMemcpyDeviceToHost));
    if (iters >= 2) {
      std::vector<double> al((size_t)iters), be((size_t)iters - 1);
      CB_CUDA(cudaMemcpy(al.data(), h->lal.p, sizeof(double) * al.size(), cudaMemcpyDeviceToHost));
      CB_CUDA(cudaMemcpy(be.data(), h->lbe.p, sizeof(double) * be.size(), cudaMemcpyDeviceToHost));
      lanczos_extremes(al, be, rep->lambda_min, rep->lambda_max);
      rep->cond_estimate = rep->lambda_max / rep->lambda_min;
    }
    rep->t_assembly = h->t_assembly;
    rep->t_setup = h->t_setup;
    rep->t_pcg = h->t_pcg;
  }
}

}  // namespace cutbddc_b200
