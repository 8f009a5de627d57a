// comm.cuh — the NCCL exchanges of the distributed BDDC.
//
// Subdomains are split over ranks, global dof vectors are replicated. Every
// sum over subdomain copies ("sum the weighted subdomain
// corrections", :386 coarse assembly) is then a local partial sum followed by
// an in-place all-reduce on the handle's stream. NCCL calls are legal inside
// stream capture, so the exchanges sit in the PCG-iteration graph.
#pragma once

#include <nccl.h>

#include <string>

#include "handle.cuh"

namespace cutbddc_b200 {

inline void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw Failure(CUTBDDC_INTERNAL, std::string("nccl ") + what + ": " + ncclGetErrorString(r));
}

// buf[0:n] = sum over ranks of buf[0:n] (no-op without a communicator).
inline void allreduce_sum(cutbddc_gpu* h, double* buf, size_t n) {
  if (!h->comm || n == 0) return;
  nccl_check(ncclAllReduce(buf, buf, n, ncclDouble, ncclSum, h->comm, h->stream), "all-reduce");
}

inline bool distributed(const cutbddc_gpu* h) { return h->comm != nullptr; }

}  // namespace cutbddc_b200
