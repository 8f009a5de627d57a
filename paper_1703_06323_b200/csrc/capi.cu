// capi.cu — the extern "C" boundary declared in include/cutbddc.h.
// Every entry point converts Failure / CUDA errors into cutbddc_status
// (common.hpp:22-23: "the C boundary maps `code` onto cutbddc_status values").
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "bddc.cuh"
#include "comm.cuh"
#include "dist.cuh"
#include "factor.cuh"

namespace cutbddc_b200 {
namespace {
thread_local std::string g_last_error;

struct Timer {
  cudaEvent_t a, b;
  cudaStream_t s;
  explicit Timer(cudaStream_t st) : s(st) {
    CB_CUDA(cudaEventCreate(&a));
    CB_CUDA(cudaEventCreate(&b));
    CB_CUDA(cudaEventRecord(a, s));
  }
  double stop() {
    CB_CUDA(cudaEventRecord(b, s));
    CB_CUDA(cudaEventSynchronize(b));
    float ms = 0;
    CB_CUDA(cudaEventElapsedTime(&ms, a, b));
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    return ms * 1e-3;
  }
};

void need(cutbddc_gpu* h) {
  if (!h) throw Failure(CUTBDDC_INVALID_ARGUMENT, "null handle");
  CB_CUDA(cudaSetDevice(h->device));
}
}  // namespace

void set_last_error(const std::string& msg) { g_last_error = msg; }
std::atomic<long long> g_kernel_launches{0};

}  // namespace cutbddc_b200

using namespace cutbddc_b200;

extern "C" {

const char* cutbddc_last_error(void) { return g_last_error.c_str(); }

cutbddc_status cutbddc_gpu_create(const cutbddc_gpu_opts* opts, cutbddc_gpu** out) {
  return guard([&] {
    if (!out) throw Failure(CUTBDDC_INVALID_ARGUMENT, "null output handle");
    auto* h = new cutbddc_gpu();
    try {
      h->device = opts ? opts->device : 0;
      h->rank = opts ? opts->rank : 0;
      h->world = opts ? opts->world_size : 1;
      if (h->world < 1 || h->rank < 0 || h->rank >= h->world)
        throw Failure(CUTBDDC_INVALID_ARGUMENT, "rank / world_size out of range");
      const void* id = opts ? opts->nccl_id : nullptr;
      if (h->world > 1 && !id) throw Failure(CUTBDDC_CONFIG, "world_size > 1 needs the rank-0 NCCL unique id");
      int ndev = 0;
      CB_CUDA(cudaGetDeviceCount(&ndev));
      if (h->device < 0 || h->device >= ndev) throw Failure(CUTBDDC_INVALID_ARGUMENT, "device ordinal out of range");
      CB_CUDA(cudaSetDevice(h->device));
      CB_CUDA(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
      if (id) {
        // one communicator per handle; a world of 1 exercises every exchange
        ncclUniqueId uid;
        std::memcpy(&uid, id, sizeof(uid));
        nccl_check(ncclCommInitRank(&h->comm, h->world, uid, h->rank), "init");
        // first collective outside any stream capture (connection setup)
        DevBuf<double> one;
        one.alloc(1);
        one.zero(h->stream);
        allreduce_sum(h, one.p, 1);
        CB_CUDA(cudaStreamSynchronize(h->stream));
      }
    } catch (...) {
      if (h->stream) cudaStreamDestroy(h->stream);
      delete h;
      throw;
    }
    *out = h;
  });
}

void cutbddc_gpu_destroy(cutbddc_gpu* h) {
  if (!h) return;
  cudaSetDevice(h->device);
  if (h->graph_exec) cudaGraphExecDestroy(h->graph_exec);
  if (h->graph_exec_ref) cudaGraphExecDestroy(h->graph_exec_ref);
  if (h->stream) cudaStreamSynchronize(h->stream);
  h->prof.dump();
  for (cudaEvent_t e : h->dag_ev) cudaEventDestroy(e);
  if (h->comm) ncclCommDestroy(h->comm);
  if (h->stream) cudaStreamDestroy(h->stream);
  delete h;
}

cutbddc_status cutbddc_nccl_unique_id(void* id128) {
  return guard([&] {
    if (!id128) throw Failure(CUTBDDC_INVALID_ARGUMENT, "null id buffer");
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
    ncclUniqueId uid;
    nccl_check(ncclGetUniqueId(&uid), "unique id");
    std::memcpy(id128, &uid, sizeof(uid));
  });
}

// boundary vectors (global numbering) <-> the handle's local dof space
namespace {
void host_to_local(cutbddc_gpu* h, const double* x, DevBuf<double>& loc) {
  DevBuf<double> g;
  g.upload(x, (size_t)h->n_dof, h->stream);
  loc.alloc((size_t)std::max<int64_t>(1, h->n_loc));
  to_local(h, g.p, loc.p);
  CB_CUDA(cudaStreamSynchronize(h->stream));
}
// owned entries into the caller's n_dof buffer (others untouched)
void local_to_host(cutbddc_gpu* h, const double* loc, double* x) {
  DevBuf<double>& g = h->ws_global;  // held by the handle: no cudaMalloc / cudaFree per call
  if (h->n_own == h->n_dof) {
    g.alloc((size_t)h->n_dof);
  } else {
    g.upload(x, (size_t)h->n_dof, h->stream);
  }
  to_global_owned(h, loc, g.p);
  g.download(x, (size_t)h->n_dof, h->stream);
  CB_CUDA(cudaStreamSynchronize(h->stream));
}
void need_numeric(cutbddc_gpu* h) {
  if (h->plan_only) throw Failure(CUTBDDC_CONFIG, "plan-only distribution (no communicator): no numerical calls");
}
}  // namespace

cutbddc_status cutbddc_gpu_set_distribution(cutbddc_gpu* h, const cutbddc_partition_view* part,
                                            const int32_t* rank_of_sd, int rank, int world) {
  return guard([&] {
    need(h);
    if (!rank_of_sd) throw Failure(CUTBDDC_INVALID_ARGUMENT, "distribution: null rank_of_sd");
    std::lock_guard<std::mutex> lk(h->mu);
    dist_set(h, part, rank_of_sd, rank, world);
    h->assembled = false;
    h->bddc_ready = false;
  });
}

cutbddc_status cutbddc_gpu_set_problem(cutbddc_gpu* h, int problem) {
  return guard([&] {
    need(h);
    if (problem != CUTBDDC_PROBLEM_UNIT_LOAD && problem != CUTBDDC_PROBLEM_MANUFACTURED)
      throw Failure(CUTBDDC_CONFIG, "problem must be the unit load or the manufactured solution");
    std::lock_guard<std::mutex> lk(h->mu);
    h->problem = problem;
    h->assembled = false;
    h->bddc_ready = false;
  });
}

cutbddc_status cutbddc_gpu_error_norms(cutbddc_gpu* h, const double* x, double* l2, double* h1) {
  return guard([&] {
    need(h);
    std::lock_guard<std::mutex> lk(h->mu);
    if (!h->assembled) throw Failure(CUTBDDC_INVALID_ARGUMENT, "error norms: assemble first");
    if (h->problem != CUTBDDC_PROBLEM_MANUFACTURED)
      throw Failure(CUTBDDC_CONFIG, "error norms: the problem has no exact solution (set the manufactured problem)");
    need_numeric(h);
    DevBuf<double> xl;
    const double* xp = h->px.p;
    if (x) {
      host_to_local(h, x, xl);
      xp = xl.p;
    } else if (!xp || h->px.n < (size_t)h->n_loc) {
      throw Failure(CUTBDDC_INVALID_ARGUMENT, "error norms: no solution (pass x or solve first)");
    }
    double a = 0.0, b = 0.0;
    error_norms_device(h, xp, &a, &b);
    if (h->comm && h->dist_world > 1) {  // every rank's cells
      DevBuf<double> t;
      const double ab[2] = {a, b};
      t.upload(ab, 2, h->stream);
      nccl_check(ncclAllReduce(t.p, t.p, 2, ncclDouble, ncclSum, h->comm, h->stream), "error norms");
      double r[2];
      t.download(r, 2, h->stream);
      CB_CUDA(cudaStreamSynchronize(h->stream));
      a = r[0];
      b = r[1];
    }
    if (l2) *l2 = std::sqrt(a);
    if (h1) *h1 = std::sqrt(b);
  });
}

cutbddc_status cutbddc_gpu_exchange_plan(cutbddc_gpu* h, cutbddc_exchange_plan** out) {
  return guard([&] {
    need(h);
    if (!out) throw Failure(CUTBDDC_INVALID_ARGUMENT, "exchange plan: null output");
    std::lock_guard<std::mutex> lk(h->mu);
    if (!h->assembled) throw Failure(CUTBDDC_INVALID_ARGUMENT, "exchange plan: assemble first");
    cudaStream_t s = h->stream;
    auto* p = new cutbddc_exchange_plan();
    p->n_loc = h->n_loc;
    p->n_own = h->n_own;
    p->n_sd_local = h->nsd;
    p->n_nbr = (int)h->nbr.size();
    p->loc_glob = new int32_t[(size_t)h->n_loc + 1];
    p->seg_ptr = new int32_t[(size_t)h->nsd + 1];
    p->copy_ptr = new int32_t[(size_t)h->n_loc + 1];
    p->copy_src = new int32_t[(size_t)h->n_copies + 1];
    p->nbr = new int32_t[h->nbr.size() + 1];
    p->send_ptr = new int64_t[h->send_ptr.size()];
    p->recv_ptr = new int64_t[h->recv_ptr.size()];
    p->send_src = new int32_t[(size_t)h->send_ptr.back() + 1];
    h->loc_glob.download(p->loc_glob, (size_t)h->n_loc, s);
    h->seg_ptr.download(p->seg_ptr, (size_t)h->nsd + 1, s);
    h->lcopy_ptr.download(p->copy_ptr, (size_t)h->n_loc + 1, s);
    h->lcopy_src.download(p->copy_src, (size_t)h->n_copies, s);
    h->send_src.download(p->send_src, (size_t)h->send_ptr.back(), s);
    CB_CUDA(cudaStreamSynchronize(s));
    std::copy(h->nbr.begin(), h->nbr.end(), p->nbr);
    std::copy(h->send_ptr.begin(), h->send_ptr.end(), p->send_ptr);
    std::copy(h->recv_ptr.begin(), h->recv_ptr.end(), p->recv_ptr);
    *out = p;
  });
}

void cutbddc_exchange_plan_free(cutbddc_exchange_plan* p) {
  if (!p) return;
  delete[] p->loc_glob;
  delete[] p->seg_ptr;
  delete[] p->copy_ptr;
  delete[] p->copy_src;
  delete[] p->nbr;
  delete[] p->send_ptr;
  delete[] p->send_src;
  delete[] p->recv_ptr;
  delete p;
}

cutbddc_status cutbddc_gpu_classify(cutbddc_gpu* h, const cutbddc_geometry* g, double* phi, uint8_t* cls,
                                    int32_t* dof_of_node, int64_t* n_dof) {
  return guard([&] {
    need(h);
    if (!g) throw Failure(CUTBDDC_INVALID_ARGUMENT, "null geometry");
    std::lock_guard<std::mutex> lk(h->mu);
    classify_device(h, g);
    if (phi) h->phi.download(phi, (size_t)h->n_nodes, h->stream);
    if (cls) h->cls.download(cls, (size_t)h->n_cells, h->stream);
    if (dof_of_node) h->dof_of_node.download(dof_of_node, (size_t)h->n_nodes, h->stream);
    if (n_dof) *n_dof = h->n_dof;
    CB_CUDA(cudaStreamSynchronize(h->stream));
  });
}

cutbddc_status cutbddc_gpu_assemble(cutbddc_gpu* h, const cutbddc_mesh_view* mesh, const cutbddc_partition_view* part,
                                    uint8_t* dirichlet) {
  return guard([&] {
    need(h);
    if (!part || !part->block_ids || part->n_sd < 1) throw Failure(CUTBDDC_INVALID_ARGUMENT, "null or empty partition");
    std::lock_guard<std::mutex> lk(h->mu);
    Timer tm(h->stream);
    if (mesh) {
      // Caller-supplied BackgroundMesh view (host buffers): upload.
      if (mesh->cells[0] != mesh->cells[1] || mesh->cells[1] != mesh->cells[2])
        throw Failure(CUTBDDC_INVALID_ARGUMENT, "mesh view: only cubic cell counts are supported");
      if (mesh->h[0] != mesh->h[1] || mesh->h[1] != mesh->h[2])
        throw Failure(CUTBDDC_INVALID_ARGUMENT, "mesh view: cells must be cubes");
      const int n = mesh->cells[0];
      h->n = n;
      h->h = mesh->h[0];
      for (int d = 0; d < 3; ++d) h->origin[d] = mesh->origin[d];
      h->tol = 1e-12 * h->h;
      h->n_nodes = (int64_t)(n + 1) * (n + 1) * (n + 1);
      h->n_cells = (int64_t)n * n * n;
      h->n_dof = mesh->n_dof;
      h->phi.upload(mesh->phi, (size_t)h->n_nodes, h->stream);
      h->cls.upload(mesh->cls, (size_t)h->n_cells, h->stream);
      h->dof_of_node.upload(mesh->dof_of_node, (size_t)h->n_nodes, h->stream);
      node_of_dof_device(h);  // inverse map on the device (checks the dof ids)
      h->mesh_ready = true;
    }
    if (!h->mesh_ready) throw Failure(CUTBDDC_INVALID_ARGUMENT, "assemble: no mesh (classify first or pass a view)");
    assemble_device(h, part);
    h->t_assembly = tm.stop();
    if (dirichlet) {
      h->orphan.download(dirichlet, (size_t)h->n_dof, h->stream);
      CB_CUDA(cudaStreamSynchronize(h->stream));
    }
  });
}

cutbddc_status cutbddc_gpu_local_diagonals(cutbddc_gpu* h, double* diag, int64_t* n_copies) {
  return guard([&] {
    need(h);
    std::lock_guard<std::mutex> lk(h->mu);
    if (!h->assembled) throw Failure(CUTBDDC_INVALID_ARGUMENT, "assemble first");
    std::vector<int32_t> sdof = h->slot_dof.to_host(h->stream);
    std::vector<double> As((size_t)h->nsd * h->slots);
    for (int s = 0; s < h->nsd; ++s)
      CB_CUDA(cudaMemcpyAsync(As.data() + (size_t)s * h->slots, h->As.p + ((size_t)s * 27 + 13) * h->slots,
                              sizeof(double) * h->slots, cudaMemcpyDeviceToHost, h->stream));
    CB_CUDA(cudaStreamSynchronize(h->stream));
    int64_t c = 0;
    for (size_t g = 0; g < sdof.size(); ++g)
      if (sdof[g] >= 0) {
        if (diag) diag[c] = As[g];
        ++c;
      }
    if (n_copies) *n_copies = c;
  });
}

cutbddc_status cutbddc_gpu_classify_objects(cutbddc_gpu* h, int objects, int variant, cutbddc_objects** out) {
  return guard([&] {
    need(h);
    if (!out) throw Failure(CUTBDDC_INVALID_ARGUMENT, "objects: null output");
    if (objects < CUTBDDC_OBJECTS_C || objects > CUTBDDC_OBJECTS_CEF)
      throw Failure(CUTBDDC_CONFIG, "bddc.objects must be c, ce or cef");
    if (variant < CUTBDDC_VARIANT_STANDARD || variant > CUTBDDC_VARIANT_V2)
      throw Failure(CUTBDDC_CONFIG, "bddc.variant must be standard, v1 or v2");
    std::lock_guard<std::mutex> lk(h->mu);
    if (!h->assembled) throw Failure(CUTBDDC_INVALID_ARGUMENT, "objects: assemble first");
    *out = classify_objects_device(h, objects, variant);
  });
}

cutbddc_status cutbddc_gpu_setup_bddc(cutbddc_gpu* h, const cutbddc_coarse_view* coarse, int weighting) {
  return guard([&] {
    need(h);
    if (weighting != CUTBDDC_WEIGHT_TOPOLOGICAL && weighting != CUTBDDC_WEIGHT_STIFFNESS)
      throw Failure(CUTBDDC_CONFIG, "bddc.weighting must be topological or stiffness");
    std::lock_guard<std::mutex> lk(h->mu);
    Timer tm(h->stream);
    setup_bddc_device(h, coarse, weighting);
    h->t_setup = tm.stop();
  });
}


cutbddc_status cutbddc_gpu_pcg(cutbddc_gpu* h, const double* b, double* x, double rtol, int max_iter,
                               cutbddc_solve_report* report) {
  return guard([&] {
    need(h);
    std::lock_guard<std::mutex> lk(h->mu);
    if (!h->bddc_ready) throw Failure(CUTBDDC_INVALID_ARGUMENT, "pcg: setup_bddc first");
    const double* bd = h->b.p;
    DevBuf<double> bbuf;
    if (b) {
      host_to_local(h, b, bbuf);
      bd = bbuf.p;
    }
    pcg_device(h, bd, rtol, max_iter, report);
    if (x) local_to_host(h, h->px.p, x);
  });
}

cutbddc_status cutbddc_gpu_spmv(cutbddc_gpu* h, const double* x, double* y) {
  return guard([&] {
    need(h);
    std::lock_guard<std::mutex> lk(h->mu);
    if (!h->assembled) throw Failure(CUTBDDC_INVALID_ARGUMENT, "assemble first");
    need_numeric(h);
    DevBuf<double> dx, dy;
    host_to_local(h, x, dx);
    dy.alloc((size_t)std::max<int64_t>(1, h->n_loc));
    spmv_device(h, dx.p, dy.p);
    local_to_host(h, dy.p, y);
  });
}

cutbddc_status cutbddc_gpu_apply_bddc(cutbddc_gpu* h, const double* r, double* z) {
  return guard([&] {
    need(h);
    std::lock_guard<std::mutex> lk(h->mu);
    if (!h->bddc_ready) throw Failure(CUTBDDC_INVALID_ARGUMENT, "apply: setup_bddc first");
    DevBuf<double> dr, dz;
    host_to_local(h, r, dr);
    dz.alloc((size_t)std::max<int64_t>(1, h->n_loc));
    apply_bddc_device(h, dr.p, dz.p, nullptr);
    local_to_host(h, dz.p, z);
  });
}

cutbddc_status cutbddc_gpu_rhs(cutbddc_gpu* h, double* b) {
  return guard([&] {
    need(h);
    std::lock_guard<std::mutex> lk(h->mu);
    if (!h->assembled) throw Failure(CUTBDDC_INVALID_ARGUMENT, "assemble first");
    need_numeric(h);
    local_to_host(h, h->b.p, b);
  });
}

cutbddc_status cutbddc_gpu_coarse_matrix(cutbddc_gpu* h, double* ac, int* n_coarse) {
  return guard([&] {
    need(h);
    std::lock_guard<std::mutex> lk(h->mu);
    if (!h->bddc_ready) throw Failure(CUTBDDC_INVALID_ARGUMENT, "setup_bddc first");
    if (n_coarse) *n_coarse = h->n_coarse;
    if (ac && h->n_coarse) {
      h->acoarse.download(ac, (size_t)h->n_coarse * h->n_coarse, h->stream);
      CB_CUDA(cudaStreamSynchronize(h->stream));
    }
  });
}

cutbddc_status cutbddc_gpu_dense_cholesky(cutbddc_gpu* h, int n, const double* a, double* l, double* x,
                                          int64_t* pivot) {
  return guard([&] {
    need(h);
    std::lock_guard<std::mutex> lk(h->mu);
    if (n < 0 || (n > 0 && !a)) throw Failure(CUTBDDC_INVALID_ARGUMENT, "dense_cholesky: bad matrix");
    if (pivot) *pivot = -1;
    if (n == 0) return;
    const size_t nn = (size_t)n * n;
    DevBuf<double> A, X;
    DevBuf<unsigned long long> fail;
    A.upload(a, nn, h->stream);
    X.alloc(nn);
    fail.alloc(1);
    CB_CUDA(cudaMemsetAsync(fail.p, 0xff, 8, h->stream));
    dense_dag_matrix(h, A.p, X.p, n, fail.p);
    unsigned long long f = 0;
    CB_CUDA(cudaMemcpyAsync(&f, fail.p, 8, cudaMemcpyDeviceToHost, h->stream));
    if (l) A.download(l, nn, h->stream);
    if (x) X.download(x, nn, h->stream);
    CB_CUDA(cudaStreamSynchronize(h->stream));
    if (f != ~0ull) {
      if (pivot) *pivot = (int64_t)f;
      throw Failure(CUTBDDC_SINGULAR, "dense_cholesky: not positive definite (pivot " + std::to_string(f) + ")");
    }
  });
}

cutbddc_status cutbddc_gpu_cells(cutbddc_gpu* h, double* beta, uint8_t* empty, int64_t* n_active) {
  return guard([&] {
    need(h);
    std::lock_guard<std::mutex> lk(h->mu);
    if (!h->assembled) throw Failure(CUTBDDC_INVALID_ARGUMENT, "assemble first");
    if (n_active) *n_active = h->n_active;
    if (!beta && !empty) return;
    std::vector<int64_t> act = h->active_cells.to_host(h->stream);
    std::vector<int32_t> eoc = h->elem_of_cell.to_host(h->stream);
    std::vector<double> hb = h->beta.to_host(h->stream);
    std::vector<uint8_t> he = h->empty.to_host(h->stream);
    for (int64_t a = 0; a < h->n_active; ++a) {
      const int32_t e = eoc[(size_t)act[(size_t)a]];
      if (beta) beta[a] = e >= 0 ? hb[(size_t)e] : 0.0;
      if (empty) empty[a] = e >= 0 ? he[(size_t)e] : 0;
    }
  });
}

cutbddc_status cutbddc_gpu_cut_elements(cutbddc_gpu* h, int64_t* cells, double* ke, double* fe, int64_t* n_cut) {
  return guard([&] {
    need(h);
    std::lock_guard<std::mutex> lk(h->mu);
    if (!h->assembled) throw Failure(CUTBDDC_INVALID_ARGUMENT, "assemble first");
    if (n_cut) *n_cut = h->n_cut;
    if (cells) h->cut_cells.download(cells, (size_t)h->n_cut, h->stream);
    if (ke) h->ke.download(ke, (size_t)h->n_cut * 64, h->stream);
    if (fe) h->fe.download(fe, (size_t)h->n_cut * 8, h->stream);
    CB_CUDA(cudaStreamSynchronize(h->stream));
  });
}

cutbddc_status cutbddc_gpu_local_system(cutbddc_gpu* h, double* stencil, uint8_t* mask_interior, uint8_t* mask_present,
                                        double* diag_add, int32_t* slot_dof) {
  return guard([&] {
    need(h);
    std::lock_guard<std::mutex> lk(h->mu);
    if (!h->bddc_ready) throw Failure(CUTBDDC_INVALID_ARGUMENT, "setup_bddc first");
    const size_t ns = (size_t)h->nsd * h->slots;
    if (stencil) h->As.download(stencil, ns * 27, h->stream);
    if (mask_interior) h->mask_int.download(mask_interior, ns, h->stream);
    if (mask_present) h->mask_all.download(mask_present, ns, h->stream);
    if (diag_add) h->diag_add.download(diag_add, ns, h->stream);
    if (slot_dof) h->slot_dof.download(slot_dof, ns, h->stream);
    CB_CUDA(cudaStreamSynchronize(h->stream));
  });
}

cutbddc_status cutbddc_gpu_local_solve(cutbddc_gpu* h, int which, double* x) {
  return guard([&] {
    need(h);
    std::lock_guard<std::mutex> lk(h->mu);
    if (!h->bddc_ready) throw Failure(CUTBDDC_INVALID_ARGUMENT, "setup_bddc first");
    const size_t ns = (size_t)h->nsd * h->slots;
    if (which != 0 && !h->has_K) throw Failure(CUTBDDC_INVALID_ARGUMENT, "no constrained Neumann factor (no interface)");
    DevBuf<double> X;
    X.upload(x, ns, h->stream);
    if (which == 0)
      solve_device(h, h->tI, h->fI, X.p, h->upd.p, h->ysave.p, nullptr);
    else
      solve_k_device(h, X.p, nullptr);
    X.download(x, ns, h->stream);
    CB_CUDA(cudaStreamSynchronize(h->stream));
  });
}

cutbddc_status cutbddc_gpu_time_solves(cutbddc_gpu* h, int reps, double* seconds, double* bytes) {
  return guard([&] {
    need(h);
    std::lock_guard<std::mutex> lk(h->mu);
    if (!h->bddc_ready) throw Failure(CUTBDDC_INVALID_ARGUMENT, "setup_bddc first");
    if (reps < 1) reps = 1;
    // warm
    solve_device(h, h->tI, h->fI, h->sv0.p, h->upd.p, h->ysave.p, nullptr);
    if (h->has_K) solve_k_device(h, h->sv1.p, nullptr);
    Timer tm(h->stream);
    for (int r = 0; r < reps; ++r) {
      solve_device(h, h->tI, h->fI, h->sv0.p, h->upd.p, h->ysave.p, nullptr);
      if (h->has_K) solve_k_device(h, h->sv1.p, nullptr);
      solve_device(h, h->tI, h->fI, h->sv0.p, h->upd.p, h->ysave.p, nullptr);
    }
    *seconds = tm.stop() / reps;
    *bytes = 2.0 * sweep_bytes(h->fI) + (h->has_K ? sweep_bytes(h->fK) + (h->k_mixed ? sweep_bytes(h->fKs) : 0.0) : 0.0);
  });
}

cutbddc_status cutbddc_gpu_time_parts(cutbddc_gpu* h, int reps, double* us) {
  return guard([&] {
    need(h);
    std::lock_guard<std::mutex> lk(h->mu);
    if (!h->bddc_ready) throw Failure(CUTBDDC_INVALID_ARGUMENT, "setup_bddc first");
    need_numeric(h);
    if (reps < 1) reps = 1;
    cudaStream_t s = h->stream;
    const int64_t nl = std::max<int64_t>(1, h->n_loc);
    DevBuf<double> x, y;
    x.alloc((size_t)nl);
    y.alloc((size_t)nl);
    CB_CUDA(cudaMemcpyAsync(x.p, h->b.p, sizeof(double) * nl, cudaMemcpyDeviceToDevice, s));
    auto timed = [&](auto fn) {
      fn();  // warm
      Timer tm(s);
      for (int r = 0; r < reps; ++r) fn();
      return 1e6 * tm.stop() / reps;
    };
    us[0] = timed([&] { sub_apply(h, kSubAll, x.p, nullptr, h->sv2.p, nullptr); });
    us[1] = timed([&] { sub_apply(h, kSubInterface, nullptr, h->sv0.p, h->sv2.p, nullptr); });
    us[2] = timed([&] { sub_apply(h, kSubInterior, x.p, nullptr, h->sv2.p, nullptr); });
    us[3] = timed([&] { iface_sum(h, h->sv2.p, nullptr, y.p, nullptr); });
    us[4] = timed([&] { apply_bddc_device(h, x.p, y.p, nullptr); });
    us[5] = timed([&] {
      solve_device(h, h->tI, h->fI, h->sv0.p, h->upd.p, h->ysave.p, nullptr);
      if (h->has_K) solve_k_device(h, h->sv1.p, nullptr);
      solve_device(h, h->tI, h->fI, h->sv0.p, h->upd.p, h->ysave.p, nullptr);
    });
    us[6] = timed([&] { spmv_device(h, x.p, y.p); });
    us[7] = 0.0;
  });
}

cutbddc_status cutbddc_gpu_time_factor(cutbddc_gpu* h, double* seconds, double* flops_cholesky, double* flops_inverse) {
  return guard([&] {
    need(h);
    std::lock_guard<std::mutex> lk(h->mu);
    if (!h->bddc_ready) throw Failure(CUTBDDC_INVALID_ARGUMENT, "setup_bddc first");
    double t = 0.0;
    for (size_t k = 0; k + 1 < h->dag_ev.size(); k += 2) {
      CB_CUDA(cudaEventSynchronize(h->dag_ev[k + 1]));
      float ms = 0.f;
      CB_CUDA(cudaEventElapsedTime(&ms, h->dag_ev[k], h->dag_ev[k + 1]));
      t += ms * 1e-3;
    }
    *seconds = t;
    const bool ks = h->has_K && h->k_mixed;
    *flops_cholesky = h->fI.flops + (h->has_K ? h->fK.flops : 0.0) + (ks ? h->fKs.flops : 0.0);
    *flops_inverse = h->fI.flops_inv + (h->has_K ? h->fK.flops_inv : 0.0) + (ks ? h->fKs.flops_inv : 0.0);
  });
}

cutbddc_status cutbddc_fp64_peak(int device, double* dmma_tflops, double* dfma_tflops) {
  return guard([&] { fp64_peaks(device, dmma_tflops, dfma_tflops); });
}

cutbddc_status cutbddc_host_pin(void* ptr, size_t bytes) {
  return guard([&] {
    if (!ptr || bytes == 0) throw Failure(CUTBDDC_INVALID_ARGUMENT, "host_pin: empty buffer");
    CB_CUDA(cudaHostRegister(ptr, bytes, cudaHostRegisterPortable));
  });
}

cutbddc_status cutbddc_host_unpin(void* ptr) {
  return guard([&] {
    if (!ptr) throw Failure(CUTBDDC_INVALID_ARGUMENT, "host_unpin: null buffer");
    CB_CUDA(cudaHostUnregister(ptr));
  });
}

cutbddc_status cutbddc_gpu_stats(cutbddc_gpu* h, int64_t* st) {
  return guard([&] {
    need(h);
    st[0] = h->n_dof;
    st[1] = h->nsd;
    st[2] = h->n_coarse;
    st[3] = h->slots;
    const int64_t pks = h->k_mixed ? h->fKs.panel_total : 0;
    st[4] = h->fI.panel_total + h->fK.panel_total + pks;
    st[5] = (int64_t)h->tplK().tpl.sn.size();
    st[6] = (int64_t)h->tplK().tpl.levels.size();
    st[7] = h->m_max;
    st[8] = h->n_if;
    st[9] = g_kernel_launches.load();
    st[10] = h->fI.panel_total;
    st[11] = h->fK.panel_total + pks;
    st[12] = (int64_t)(h->fI.flops + h->fK.flops + (h->k_mixed ? h->fKs.flops : 0.0));
    st[13] = h->world;
    st[14] = h->comm != nullptr;
    st[15] = h->has_K && h->k_corner;
    st[16] = h->has_K && h->k_mixed ? h->n_shell_sd : 0;
  });
}

}  // extern "C"
