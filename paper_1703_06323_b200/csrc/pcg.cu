// pcg.cu — preconditioned CG on the device (K4 SpMV, K11 vector ops/dots).
//
// krylov::pcg with the pins of SURVEY.md Appendix B.7:
// x0 = 0, residuals[0] = |b|, r <- b - Abar x after the update at every
// iteration k with k % 50 == 0, stop at the first k with |r|_2 < rtol |b|_2,
// <p,Ap> <= 0 or <r,Mr> <= 0 -> indefiniteness error, max_iter -> a
// non-converged report. Lanczos alpha/beta are recorded for
// condition_estimate (evaluated on the host).
//
// The whole iteration (SpMV, dots, axpys, BDDC apply) is one CUDA graph with
// all scalars on the device; a device "done" flag turns the remaining
// kernels of a converged solve into no-ops, so the host only polls the flag
// every few graph launches (no per-iteration host round trip). Dots are
// two-stage fixed-order reductions: bit-reproducible run to run.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <vector>

#include "bddc.cuh"
#include "comm.cuh"

namespace cutbddc_b200 {
namespace {

constexpr int kRedBlocks = 592;  // 4 x 148 SMs, fixed for deterministic reductions
constexpr int kRedThreads = 256;

// rz ping-pongs between S_RZ (even iterations) and S_RZ1 (odd): the fused
// beta/p-update kernel reads the old value in every block while block 0
// stores the new one.
enum { S_RZ = 0, S_PQ, S_ALPHA, S_BETA, S_STOP, S_RN, S_RZ1, S_COUNT };
__device__ __forceinline__ int rz_slot(int k) { return (k & 1) ? S_RZ1 : S_RZ; }
enum { I_DONE = 0, I_ITER, I_ERR, I_ITERS, I_CONV, I_MAXIT, I_COUNT };

__global__ void __launch_bounds__(kRedThreads) k_spmv_dot(int64_t nd, const double* __restrict__ aval,
                                                          const int32_t* __restrict__ acol, const double* __restrict__ x,
                                                          double* __restrict__ y, double* __restrict__ partial,
                                                          const int* __restrict__ skip) {
  if (skip && *skip) return;
  __shared__ double sh[32];
  double acc = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nd; i += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < 27; ++k) s += aval[(int64_t)k * nd + i] * x[acol[(int64_t)k * nd + i]];
    y[i] = s;
    acc += x[i] * s;
  }
  acc = block_sum<kRedThreads>(acc, sh);
  if (partial && threadIdx.x == 0) partial[blockIdx.x] = acc;
}

__global__ void __launch_bounds__(kRedThreads) k_dot(int64_t nd, const double* __restrict__ a, const double* __restrict__ b,
                                                     double* __restrict__ partial, const int* __restrict__ skip) {
  if (skip && *skip) return;
  __shared__ double sh[32];
  double acc = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nd; i += (int64_t)gridDim.x * blockDim.x)
    acc += a[i] * b[i];
  acc = block_sum<kRedThreads>(acc, sh);
  if (threadIdx.x == 0) partial[blockIdx.x] = acc;
}

__device__ inline double finish_sum(const double* partial, double* sh) {
  double v = 0.0;
  for (int i = threadIdx.x; i < kRedBlocks; i += blockDim.x) v += partial[i];
  return block_sum<kRedThreads>(v, sh);
}

// finish_sum, the total broadcast to every thread of the block
__device__ inline double finish_sum_all(const double* partial, double* sh) {
  __shared__ double tot;
  const double v = finish_sum(partial, sh);
  if (threadIdx.x == 0) tot = v;
  __syncthreads();
  return tot;
}

// alpha = rz / pq (every block from the same fixed-order sum of `partial`),
// x += alpha p, r -= alpha q, and the partials of r.r for k_check in `rpart`
// (k_dot's mapping; at a refresh iteration k_refresh writes them instead)
__global__ void __launch_bounds__(kRedThreads) k_update_xr(int64_t nd, double* __restrict__ sc,
                                                           const double* __restrict__ p, const double* __restrict__ q,
                                                           double* __restrict__ x, double* __restrict__ r,
                                                           double* __restrict__ lal, const double* __restrict__ partial,
                                                           double* __restrict__ rpart, int* __restrict__ is) {
  if (is[I_DONE]) return;
  __shared__ double sh[32];
  const int k = is[I_ITER];
  const double pq = finish_sum_all(partial, sh);
  if (!(pq > 0.0)) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      sc[S_PQ] = pq;
      is[I_ERR] = 1;
      is[I_DONE] = 1;
      is[I_ITERS] = k;
    }
    return;
  }
  const double a = sc[rz_slot(k)] / pq;
  const int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i0 == 0) {
    sc[S_PQ] = pq;
    sc[S_ALPHA] = a;
    lal[k - 1] = a;
  }
  double acc = 0.0;
  for (int64_t i = i0; i < nd; i += (int64_t)gridDim.x * blockDim.x) {
    x[i] += a * p[i];
    const double ri = r[i] - a * q[i];
    r[i] = ri;
    acc += ri * ri;
  }
  if (k % 50 == 0) return;  // k_refresh replaces r and its partials
  acc = block_sum<kRedThreads>(acc, sh);
  if (threadIdx.x == 0) rpart[blockIdx.x] = acc;
}

// true residual refresh at k % 50 == 0: r = b - Abar x, and the r.r partials
__global__ void __launch_bounds__(kRedThreads) k_refresh(int64_t nd, const double* __restrict__ aval,
                                                         const int32_t* __restrict__ acol, const double* __restrict__ x,
                                                         const double* __restrict__ b, double* __restrict__ r,
                                                         double* __restrict__ rpart, const int* __restrict__ is) {
  if (is[I_DONE] || is[I_ITER] % 50 != 0) return;
  __shared__ double sh[32];
  double acc = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nd; i += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < 27; ++k) s += aval[(int64_t)k * nd + i] * x[acol[(int64_t)k * nd + i]];
    const double ri = b[i] - s;
    r[i] = ri;
    acc += ri * ri;
  }
  acc = block_sum<kRedThreads>(acc, sh);
  if (threadIdx.x == 0) rpart[blockIdx.x] = acc;
}

// |r| -> history, convergence / max_iter test
__global__ void k_check(const double* __restrict__ partial, double* __restrict__ sc, int* __restrict__ is,
                        double* __restrict__ hist) {
  if (is[I_DONE]) return;
  __shared__ double sh[32];
  const double rr = finish_sum(partial, sh);
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

// beta = rz_new / rz (every block from the same fixed-order sum; rz_new to
// the other ping-pong slot), p = z + beta p
__global__ void __launch_bounds__(kRedThreads) k_update_p(int64_t nd, const double* __restrict__ partial,
                                                          double* __restrict__ sc, const double* __restrict__ z,
                                                          double* __restrict__ p, double* __restrict__ lbe,
                                                          int* __restrict__ is) {
  if (is[I_DONE]) return;
  __shared__ double sh[32];
  const int k = is[I_ITER];
  const double rz = finish_sum_all(partial, sh);
  if (!(rz > 0.0)) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      is[I_ERR] = 2;
      is[I_DONE] = 1;
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
  for (int64_t i = i0; i < nd; i += (int64_t)gridDim.x * blockDim.x) p[i] = z[i] + beta * p[i];
}

__global__ void k_next(int* __restrict__ is) {
  if (is[I_DONE]) return;
  is[I_ITER] += 1;
}

// initial: rz = r.z (after z = M r), p = z
__global__ void k_init_rz(const double* __restrict__ partial, double* __restrict__ sc, int* __restrict__ is) {
  __shared__ double sh[32];
  const double rz = finish_sum(partial, sh);
  if (threadIdx.x == 0) {
    sc[rz_slot(1)] = rz;
    if (!(rz > 0.0)) {
      is[I_ERR] = 2;
      is[I_DONE] = 1;
      is[I_ITERS] = 0;
    }
  }
}

__global__ void k_copy(int64_t nd, const double* __restrict__ a, double* __restrict__ b) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nd; i += (int64_t)gridDim.x * blockDim.x) b[i] = a[i];
}

// Loop condition of the whole-solve graph: another iteration unless done.
__global__ void k_loop_cond(cudaGraphConditionalHandle hc, const int* __restrict__ is) {
  cudaGraphSetConditional(hc, is[I_DONE] ? 0u : 1u);
}

void enqueue_iteration(cutbddc_gpu* h);

// One graph for the whole PCG loop on one GPU: a conditional WHILE node whose
// body is the captured iteration plus k_loop_cond. No host polling and no
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
  enqueue_iteration(h);
  k_loop_cond<<<1, 1, 0, s>>>(hc, h->iscal.p);
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

void enqueue_iteration(cutbddc_gpu* h) {
  cudaStream_t s = h->stream;
  const int64_t nd = h->n_dof;
  int* is = h->iscal.p;
  double* sc = h->scal.p;
  k_spmv_dot<<<kRedBlocks, kRedThreads, 0, s>>>(nd, h->aval.p, h->acol.p, h->pp.p, h->pq.p, h->partials.p, is);
  k_update_xr<<<kRedBlocks, kRedThreads, 0, s>>>(nd, sc, h->pp.p, h->pq.p, h->px.p, h->pr.p, h->lal.p, h->partials.p,
                                                 h->partials.p + kRedBlocks, is);
  k_refresh<<<kRedBlocks, kRedThreads, 0, s>>>(nd, h->aval.p, h->acol.p, h->px.p, h->pb.p, h->pr.p,
                                               h->partials.p + kRedBlocks, is);
  k_check<<<1, kRedThreads, 0, s>>>(h->partials.p + kRedBlocks, sc, is, h->hist.p);
  apply_bddc_device(h, h->pr.p, h->pz.p, is);
  k_dot<<<kRedBlocks, kRedThreads, 0, s>>>(nd, h->pr.p, h->pz.p, h->partials.p, is);
  k_update_p<<<kRedBlocks, kRedThreads, 0, s>>>(nd, h->partials.p, sc, h->pz.p, h->pp.p, h->lbe.p, is);
  k_next<<<1, 1, 0, s>>>(is);
  CB_LAUNCH();
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
  k_spmv_dot<<<kRedBlocks, kRedThreads, 0, h->stream>>>(h->n_dof, h->aval.p, h->acol.p, x, y, nullptr, nullptr);
  CB_LAUNCH();
}

void pcg_device(cutbddc_gpu* h, const double* b_dev, double rtol, int max_iter, cutbddc_solve_report* rep) {
  if (!h->bddc_ready) throw Failure(CUTBDDC_INVALID_ARGUMENT, "pcg: setup_bddc first");
  if (max_iter < 1) throw Failure(CUTBDDC_INVALID_ARGUMENT, "pcg: max_iter must be >= 1");
  cudaStream_t s = h->stream;
  const int64_t nd = h->n_dof;
  for (auto* v : {&h->px, &h->pr, &h->pz, &h->pp, &h->pq, &h->pb}) v->alloc((size_t)nd);
  h->hist.alloc((size_t)max_iter + 1);
  h->lal.alloc((size_t)max_iter + 1);
  h->lbe.alloc((size_t)max_iter + 1);
  h->partials.alloc(2 * kRedBlocks);  // p.q / r.z partials, then r.r
  h->scal.alloc(S_COUNT);
  h->iscal.alloc(I_COUNT);
  cudaEvent_t e0, e1;
  CB_CUDA(cudaEventCreate(&e0));
  CB_CUDA(cudaEventCreate(&e1));
  CB_CUDA(cudaEventRecord(e0, s));
  k_copy<<<kRedBlocks, kRedThreads, 0, s>>>(nd, b_dev, h->pb.p);
  CB_LAUNCH();
  k_copy<<<kRedBlocks, kRedThreads, 0, s>>>(nd, b_dev, h->pr.p);
  CB_LAUNCH();
  h->px.zero(s);
  h->iscal.zero(s);
  k_dot<<<kRedBlocks, kRedThreads, 0, s>>>(nd, h->pb.p, h->pb.p, h->partials.p, nullptr);
  CB_LAUNCH();
  std::vector<double> part(kRedBlocks);
  CB_CUDA(cudaMemcpyAsync(part.data(), h->partials.p, sizeof(double) * kRedBlocks, cudaMemcpyDeviceToHost, s));
  CB_CUDA(cudaStreamSynchronize(s));
  // same fixed-order tree as the device finish (block_sum over 256 threads)
  // is not needed for |b|: the host value only seeds the stop threshold.
  double bb = 0.0;
  for (double v : part) bb += v;
  const double bnorm = std::sqrt(bb);
  CB_CUDA(cudaMemcpyAsync(h->hist.p, &bnorm, sizeof(double), cudaMemcpyHostToDevice, s));
  int conv = 0, iters = 0, err = 0;
  if (bnorm == 0.0) {
    h->px.zero(s);
    conv = 1;
  } else {
    const double host_sc[S_COUNT] = {0, 0, 0, 0, rtol * bnorm, 0, 0};
    CB_CUDA(cudaMemcpyAsync(h->scal.p, host_sc, sizeof(host_sc), cudaMemcpyHostToDevice, s));
    const int host_is[I_COUNT] = {0, 1, 0, 0, 0, max_iter};
    CB_CUDA(cudaMemcpyAsync(h->iscal.p, host_is, sizeof(host_is), cudaMemcpyHostToDevice, s));
    apply_bddc_device(h, h->pr.p, h->pz.p, nullptr);
    k_dot<<<kRedBlocks, kRedThreads, 0, s>>>(nd, h->pr.p, h->pz.p, h->partials.p, nullptr);
    CB_LAUNCH();
    k_init_rz<<<1, kRedThreads, 0, s>>>(h->partials.p, h->scal.p, h->iscal.p);
    CB_LAUNCH();
    k_copy<<<kRedBlocks, kRedThreads, 0, s>>>(nd, h->pz.p, h->pp.p);
    CB_LAUNCH();
    if (h->graph_exec && h->graph_max_iter != max_iter) {
      cudaGraphExecDestroy(h->graph_exec);
      h->graph_exec = nullptr;
    }
    if (!h->graph_exec && !distributed(h) && !std::getenv("CUTBDDC_NO_WHILE_GRAPH")) {
      h->graph_max_iter = max_iter;
      build_while_graph(h);
    }
    if (!h->graph_exec) {
      h->graph_max_iter = max_iter;
      h->graph_while = false;
      cudaGraph_t g;
      const long long c0 = g_kernel_launches.load();
      CB_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
      enqueue_iteration(h);
      CB_CUDA(cudaStreamEndCapture(s, &g));
      CB_CUDA(cudaGraphInstantiate(&h->graph_exec, g, 0));
      size_t nodes = 0;
      CB_CUDA(cudaGraphGetNodes(g, nullptr, &nodes));
      h->graph_nodes = (long long)nodes;
      g_kernel_launches.store(c0);  // captured, not executed
      CB_CUDA(cudaGraphDestroy(g));
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
        CB_CUDA(cudaGraphLaunch(h->graph_exec, s));
        g_kernel_launches.fetch_add(h->graph_nodes);
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
