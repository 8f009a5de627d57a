// dev_common.cuh — device helpers shared by the sm_100a kernels.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <mutex>
#include <cstdint>
#include <string>
#include <vector>

#include "status.hpp"

namespace cutbddc_b200 {

#define CB_CUDA(call)                                                                                    \
  do {                                                                                                   \
    cudaError_t e_ = (call);                                                                             \
    if (e_ != cudaSuccess)                                                                               \
      throw ::cutbddc_b200::Failure(CUTBDDC_INTERNAL, std::string("CUDA error: ") + cudaGetErrorString(e_) + \
                                                          " at " __FILE__ ":" + std::to_string(__LINE__)); \
  } while (0)

// Count of this library's kernel launches (reported by cutbddc_gpu_stats).
extern std::atomic<long long> g_kernel_launches;
#define CB_LAUNCH()                                              \
  do {                                                           \
    ::cutbddc_b200::g_kernel_launches.fetch_add(1);              \
    CB_CUDA(cudaGetLastError());                                 \
  } while (0)

// Owning device buffer; grow-only (a smaller alloc reuses the allocation, so
// repeated solves do no cudaMalloc/cudaFree inside the timed phases).
template <typename T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0, cap = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { release(); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = cap = 0;
  }
  void alloc(size_t count) {
    if (p && count <= cap) {
      n = count;
      return;
    }
    release();
    if (count == 0) return;
    CB_CUDA(cudaMalloc(&p, count * sizeof(T)));
    n = cap = count;
  }
  void zero(cudaStream_t s) {
    if (n) CB_CUDA(cudaMemsetAsync(p, 0, n * sizeof(T), s));
  }
  void upload(const T* h, size_t count, cudaStream_t s) {
    alloc(count);
    if (count) CB_CUDA(cudaMemcpyAsync(p, h, count * sizeof(T), cudaMemcpyHostToDevice, s));
  }
  void upload(const std::vector<T>& v, cudaStream_t s) { upload(v.data(), v.size(), s); }
  void download(T* h, size_t count, cudaStream_t s) const {
    if (count) CB_CUDA(cudaMemcpyAsync(h, p, count * sizeof(T), cudaMemcpyDeviceToHost, s));
  }
  std::vector<T> to_host(cudaStream_t s) const {
    std::vector<T> v(n);
    download(v.data(), n, s);
    CB_CUDA(cudaStreamSynchronize(s));
    return v;
  }
};

// Per-device, thread-safe memo of launch configuration (occupancy-derived
// grid sizes, shared-memory opt-ins): kernel attributes are per device, so a
// value computed (or an attribute set) on one device must not be reused on
// another. `fn` runs once per (slot, device) under a mutex; later calls on the
// same device read the stored value. Slots name the call sites.
enum DeviceMemoSlot { kMemoSweepFwd = 0, kMemoSweepBwd, kMemoSweepAttr, kMemoDagGrid, kMemoCoarseOutShm, kMemoSweepMulti, kMemoCoarseInShm, kMemoHcyShm, kMemoSlots };
template <typename Fn>
long long device_memo(int slot, Fn fn) {
  constexpr int kMaxDev = 64;
  static std::mutex mu;
  static long long val[kMemoSlots][kMaxDev];
  static bool set[kMemoSlots][kMaxDev];
  int dev = 0;
  CB_CUDA(cudaGetDevice(&dev));
  if (dev < 0 || dev >= kMaxDev) dev = kMaxDev - 1;
  std::lock_guard<std::mutex> lk(mu);
  if (!set[slot][dev]) {
    val[slot][dev] = fn();
    set[slot][dev] = true;
  }
  return val[slot][dev];
}

inline int grid_for(int64_t n, int block) { return (int)((n + block - 1) / block); }

// 27-point stencil index k = (dx+1)*9 + (dy+1)*3 + (dz+1); k = 13 is the diagonal.
__host__ __device__ inline int stencil_k(int dx, int dy, int dz) { return (dx + 1) * 9 + (dy + 1) * 3 + (dz + 1); }

__device__ inline double warp_sum(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}

// Deterministic block reduction (fixed tree), result valid in thread 0.
template <int BLOCK>
__device__ inline double block_sum(double v, double* sh) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) sh[w] = v;
  __syncthreads();
  double r = 0;
  if (w == 0) {
    r = lane < BLOCK / 32 ? sh[lane] : 0.0;
    r = warp_sum(r);
  }
  __syncthreads();
  return r;
}

}  // namespace cutbddc_b200
