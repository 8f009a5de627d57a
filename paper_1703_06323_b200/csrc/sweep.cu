// sweep.cu — dataflow triangular-solve sweeps of the batched multifrontal
// factors (the solves inside SparseCholesky::solve, linalg.cpp:56-61, and
// SaddleFactorization::solve, linalg.cpp:97-106, for every subdomain at once).
//
// One persistent launch per sweep direction replaces one launch per
// elimination level. Work items are listed in dependency order and handed
// out by an atomic ticket; an item waits (spinning on a per-front counter)
// only for items with smaller tickets, all of which are held by running
// CTAs, so the schedule cannot deadlock and parents start as soon as their
// own children finish (no level barriers).
//
// Item kinds per (subdomain, front) with r compact rows and c columns:
//   T  the bottom kSubLevels levels below one front (all fronts small): one
//      CTA runs them one after another (no cross-CTA synchronisation).
//   S  r <= kSmallRows above the subtrees: one CTA per front.
//   A  larger fronts: one CTA gathers the front vector once into `vbuf`.
//   C  larger fronts: GEMV chunks (128 rows forward, 16 columns backward)
//      reading the gathered vector from vbuf.
// Every front applies its explicit panel G = [L11^{-1}; L21 L11^{-1}]
// (r x c, column-major, strict upper part of L11^{-1} stored as zeros):
// forward [y; L21 y] = G v_c, y -> ysave at the front's column slots and
// v_rest - L21 y -> the update vector the parent gathers (umap);
// backward x_c = G^T [y; -x_rest] -> X at the column slots.
// Everything an item needs that does not depend on other items (its
// descriptor, b or y at its columns, the first panel columns) is loaded
// before it waits, so the wait hides that latency. Every sum has a fixed
// order: the sweeps are deterministic.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <tuple>

#include "factor.cuh"
#include "front_desc.cuh"
#include "prof.cuh"

namespace cutbddc_b200 {
namespace {

#ifndef CUTBDDC_SWEEP_FWD_ROWS
#define CUTBDDC_SWEEP_FWD_ROWS 128
#endif

#ifndef CUTBDDC_SWEEP_SLOTS
#define CUTBDDC_SWEEP_SLOTS 2
#endif
#ifndef CUTBDDC_SWEEP_MIN_BLOCKS
#define CUTBDDC_SWEEP_MIN_BLOCKS 4
#endif
// (the CUTBDDC_SWEEP_* macros exist for tools/tune_sweep.sh)
#ifndef CUTBDDC_SWEEP_THREADS
#define CUTBDDC_SWEEP_THREADS 256
#endif
constexpr int kThreadsSweep = CUTBDDC_SWEEP_THREADS;  // consumer threads (+ one producer warp)
constexpr int kSmallRows = kThreadsSweep;           // fronts with at most this many rows: one forward item
constexpr int kFwdRows = CUTBDDC_SWEEP_FWD_ROWS;    // forward items of larger fronts: row blocks ...
// ... cut into column ranges of SweepDev::fwd_cols columns; backward items:
// column blocks of SweepDev::bwd_cols (<= kMaxBwdCols) columns, all rows
// below. Both are chosen per factorisation by the plan (choose_item_sizes).
#ifndef CUTBDDC_SWEEP_MAX_BWD_COLS
#define CUTBDDC_SWEEP_MAX_BWD_COLS 32
#endif
constexpr int kMaxBwdCols = CUTBDDC_SWEEP_MAX_BWD_COLS;
constexpr int kSlots = CUTBDDC_SWEEP_SLOTS;         // staging ring depth (chunks in flight per CTA)
constexpr int kMinBlocks = CUTBDDC_SWEEP_MIN_BLOCKS;
constexpr int kWarps = kThreadsSweep / 32;
// Ring slot size (doubles) and backward chunk height (rows), chosen per
// factorisation (SweepDev::slot, ::bwd_rows): many subdomains -> 4 CTAs per
// SM with 20 KB slots, few -> 3 CTAs with 28 KB slots (fewer, longer chunks
// per item). The macros override both.
constexpr int kSlotWide = 2176, kBwdRowsWide = 66;      // floor for nsd >= 256 (cfg5 runs 2752 / 84)
constexpr int kSlotFew = 2176, kBwdRowsFew = 66;        // floor for fewer subdomains (cfg4 runs 3968 / 122)
constexpr int kMaxSegs = kMaxBwdCols;               // column segments per chunk (a multiple of 32)
static_assert(kMaxSegs % 32 == 0, "segments per chunk");
constexpr int kVecMax = 2048;                       // front vector (shared): at most this many rows per front
#ifndef CUTBDDC_SWEEP_ITEMS_IN_FLIGHT
#define CUTBDDC_SWEEP_ITEMS_IN_FLIGHT 2
#endif
constexpr int kItems = CUTBDDC_SWEEP_ITEMS_IN_FLIGHT;  // item records in flight per CTA: one computing, the others being prepared
constexpr int kBlockSweep = kThreadsSweep + 64;     // consumers + producer warp + preparation warp
constexpr int kColsPerLane = kSmallRows / 32;       // forward item columns per preparation lane
// dynamic shared memory of a sweep CTA: ring | kItems front vectors (vec doubles each) | partials | segment offsets
inline size_t sweep_shm_bytes(int slot, int vec) {
  return 8 * (size_t)(kSlots * slot + kItems * vec + kThreadsSweep) + 4 * kSlots * kMaxSegs;
}
static_assert(kThreadsSweep % kFwdRows == 0 && kFwdRows % 32 == 0, "forward row blocks");
static_assert(kMaxBwdCols <= kMaxSegs && kMaxBwdCols % kWarps == 0, "backward column blocks");
static_assert(16 * (kFwdRows + 2) <= kSlotWide && 16 * (kFwdRows + 2) <= kSlotFew, "chunk sizes");
enum { kItemS = 0, kItemC = 2 };

// column stride (doubles, even: every staged column starts 16-byte aligned)
__host__ __device__ inline int seg_stride(int len) { return (len + 3) & ~1; }


struct SweepDev {
  const FrontDesc* desc;
  const int32_t* cslot;  // sd * T + slot of every compact front row
  const int32_t* umap;   // parent compact row of every update entry
  const int32_t* gmap;   // per compact front row: upd index of child 0 / child 1 entry landing there, or -1
  int nsn;
  int32_t* done_f;
  int32_t* ready_f;
  int32_t* done_b;
  int32_t* ready_b;
  int32_t* ticket;  // [0] forward, [1] backward (all, or the root phase), [2] backward below the root
  int32_t* rbcnt;   // forward range arrivals per (chunked front, row block)
  double* vbuf;
  int fwd_cols, bwd_cols;  // item sizes of this factorisation's plan
  int vec;                 // doubles of the shared front vector (this launch)
  int slot, bwd_rows;      // doubles per ring slot, rows per backward chunk
  int l2_policy;           // panel loads: 0 default, 1 L2 evict_last (keep resident), 2 L2 evict_first (stream)
  unsigned long long* trace;  // CUTBDDC_SWEEP_TRACE: per item {grab, deps met, done, sm}, else null
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ unsigned smid() {
  unsigned r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}

__device__ __forceinline__ int ld_acquire(const int32_t* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// ---------------------------------------------------------------- mbarrier + bulk copies
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra W;\n}" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
// global -> shared bulk copy (TMA engine; SASS UBLKCP), completion counted on b
__device__ __forceinline__ void bulk_g2s(double* dst, const double* src, uint32_t bytes, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(b))
               : "memory");
}
// the same with an L2 eviction-priority hint (createpolicy)
__device__ __forceinline__ void bulk_g2s_hint(double* dst, const double* src, uint32_t bytes, uint64_t* b,
                                              uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(b)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t l2_policy_of(int kind) {
  uint64_t pol = 0;
  if (kind == 1) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  if (kind == 2) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

// The consumer warps synchronise among themselves with named barrier 1: the
// producer warp never joins them.
__device__ __forceinline__ void csync() { asm volatile("bar.sync 1, %0;" ::"r"(kThreadsSweep) : "memory"); }

// consumer thread 0 waits until *p >= target; the consumers then proceed
__device__ __forceinline__ void cta_wait(const int32_t* p, int target) {
  if (threadIdx.x == 0) {
    while (ld_acquire(p) < target) __nanosleep(32);
    __threadfence();
  }
  csync();
}

// all of the consumers' global writes are published before *p is incremented
__device__ __forceinline__ void cta_signal(int32_t* p) {
  csync();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(p, 1);
  }
}

// ---------------------------------------------------------------- items and chunks
// An item streams its panel as a sequence of chunks; a chunk is a set of
// column segments: columns [ja, jb), rows [max(j, lo), hi) of column j (the
// lower part of G only).
struct Chunk {
  int ja, jb, lo, hi;
};

// Item geometry, computed identically by the producer and the consumers.
// Forward: rows [i0, i1) (one row block) x columns [jlo, jhi) (one column
// range), chunks of `cw` columns. Backward: columns [jlo, jhi) x rows
// [jlo, r), chunks of SweepDev::bwd_rows rows.
struct ItemGeom {
  int i0, i1, jlo, jhi, nchunk, cw;
  int rb, cb, mcb;
};
__device__ __forceinline__ ItemGeom item_geom(const SweepDev& p, const FrontDesc& d, int kind, int chunk, bool fwd) {
  const int kFwdCols = p.fwd_cols, kBwdCols = p.bwd_cols;
  const int r = d.r, c = d.c;
  ItemGeom g{};
  if (fwd) {
    if (kind == kItemS) {
      g.i0 = 0;
      g.i1 = r;
      g.jlo = 0;
      g.jhi = c;
      g.mcb = 1;
    } else {
      g.mcb = max(1, (c + kFwdCols - 1) / kFwdCols);
      g.rb = chunk / g.mcb;
      g.cb = chunk % g.mcb;
      g.i0 = g.rb * kFwdRows;
      g.i1 = min(r, g.i0 + kFwdRows);
      g.jlo = g.cb * kFwdCols;
      g.jhi = min(min(c, g.i1), g.jlo + kFwdCols);
    }
    g.cw = max(1, min(kMaxSegs, p.slot / seg_stride(g.i1 - g.i0)));
    // chunks start at multiples of fwd_item's thread-group count ng (a power
    // of two): the sums do not depend on the ring's slot size
    const int nr = g.i1 - g.i0;
    const int ng = nr <= kThreadsSweep / 8 ? 8 : nr <= kThreadsSweep / 4 ? 4 : nr <= kThreadsSweep / 2 ? 2 : 1;
    if (g.cw >= ng) g.cw &= ~(ng - 1);
    g.nchunk = g.jhi > g.jlo ? (g.jhi - g.jlo + g.cw - 1) / g.cw : 0;
  } else {
    g.jlo = chunk * kBwdCols;
    g.jhi = min(c, g.jlo + kBwdCols);
    g.i0 = g.jlo;
    g.i1 = r;
    g.nchunk = g.jhi > g.jlo ? (r - g.jlo + p.bwd_rows - 1) / p.bwd_rows : 0;
    g.cw = p.bwd_rows;
  }
  return g;
}
__device__ __forceinline__ Chunk chunk_of(const ItemGeom& g, int q, bool fwd) {
  if (fwd) return Chunk{g.jlo + q * g.cw, min(g.jhi, g.jlo + (q + 1) * g.cw), g.i0, g.i1};
  const int lo = g.i0 + q * g.cw;  // backward: cw = rows per chunk
  return Chunk{g.jlo, g.jhi, lo, min(g.i1, lo + g.cw)};
}

// Per-CTA shared state.
struct ItemRec {
  int4 item;  // (kind, sid, sd, chunk); kind < 0: no more items
  FrontDesc d;
  uint64_t info, ready, empty;  // published by the producer / prepared (dependencies met, vector filled) / released
  int tk;
  unsigned long long t_grab, t_dep;
};
struct SlotRec {
  uint64_t full, empty;
};

// Producer warp: one chunk into ring slot `slot`: segment offsets (row i of
// column ja + jj at buf[segoff[jj] + i]), expected bytes, bulk copies (one
// per column segment, 16-byte aligned: a segment starting at an odd element
// copies one leading double more; rows past a segment's end are never read).
__device__ __forceinline__ void produce_chunk(const FrontDesc& d, const Chunk& ch, const double* __restrict__ panel,
                                              double* buf, int* segoff, SlotRec& sr, int l2_kind, uint64_t pol) {
  const int lane = threadIdx.x & 31;
  const int stride = seg_stride(ch.hi - ch.lo);
  int64_t a[kMaxSegs / 32], n[kMaxSegs / 32];
  uint32_t mine = 0;
#pragma unroll
  for (int u = 0; u < kMaxSegs / 32; ++u) {
    const int jj = lane + 32 * u;
    const int j = ch.ja + jj;
    a[u] = n[u] = 0;
    if (j < ch.jb) {
      const int first = max(j, ch.lo);
      if (first < ch.hi) {
        const int64_t e = d.po + (int64_t)j * d.r + first;
        a[u] = e & ~1ll;
        n[u] = ((e + (ch.hi - first) + 1) & ~1ll) - a[u];
        segoff[jj] = jj * stride + (int)(e - a[u]) - first;
      }
    }
    mine += (uint32_t)(8 * n[u]);
  }
  const uint32_t bytes = __reduce_add_sync(0xffffffffu, mine);
  if (lane == 0) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_expect_tx(&sr.full, bytes);
  }
  __syncwarp();
#pragma unroll
  for (int u = 0; u < kMaxSegs / 32; ++u) {
    const int jj = lane + 32 * u;
    if (n[u] > 0) {
      if (l2_kind)
        bulk_g2s_hint(buf + jj * stride, panel + a[u], (uint32_t)(8 * n[u]), &sr.full, pol);
      else
        bulk_g2s(buf + jj * stride, panel + a[u], (uint32_t)(8 * n[u]), &sr.full);
    }
  }
}

// Producer warp main loop: take tickets in order, publish each item, stream
// its chunks through the ring (blocking only on free slots).
__device__ void producer(const SweepDev& p, const int4* __restrict__ items, int n_items, int32_t* ticket,
                         const double* __restrict__ panel, ItemRec* rec, SlotRec* sr, double* ring, int* segoff,
                         bool fwd) {
  const int lane = threadIdx.x & 31;
  const uint64_t pol = l2_policy_of(p.l2_policy);
  int chunk_seq = 0;
  for (int k = 0;; ++k) {
    ItemRec& R = rec[k % kItems];
    if (k >= kItems) mbar_wait(&R.empty, ((k / kItems) - 1) & 1);
    int it = 0;
    if (lane == 0) it = atomicAdd(ticket, 1);
    it = __shfl_sync(0xffffffffu, it, 0);
    if (it >= n_items) {
      if (lane == 0) {
        R.item = make_int4(-1, 0, 0, 0);
        mbar_arrive(&R.info);
      }
      return;
    }
    const int4 w = items[it];
    const int4 dv = lane < 6 ? reinterpret_cast<const int4*>(p.desc + (int64_t)w.z * p.nsn + w.y)[lane]
                             : make_int4(0, 0, 0, 0);
    FrontDesc d;
#pragma unroll
    for (int k6 = 0; k6 < 6; ++k6) {
      int4 x;
      x.x = __shfl_sync(0xffffffffu, dv.x, k6);
      x.y = __shfl_sync(0xffffffffu, dv.y, k6);
      x.z = __shfl_sync(0xffffffffu, dv.z, k6);
      x.w = __shfl_sync(0xffffffffu, dv.w, k6);
      reinterpret_cast<int4*>(&d)[k6] = x;
    }
    if (lane < 6) reinterpret_cast<int4*>(&R.d)[lane] = dv;
    if (lane == 0) {
      R.item = w;
      R.tk = it;
      if (p.trace) R.t_grab = gtimer();
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&R.info);
    const ItemGeom g = item_geom(p, d, w.x, w.w, fwd);
    for (int q = 0; q < g.nchunk; ++q, ++chunk_seq) {
      const int slot = chunk_seq % kSlots;
      if (chunk_seq >= kSlots) mbar_wait(&sr[slot].empty, ((chunk_seq / kSlots) - 1) & 1);
      produce_chunk(d, chunk_of(g, q, fwd), panel, ring + slot * p.slot, segoff + slot * kMaxSegs, sr[slot],
                    p.l2_policy, pol);
    }
  }
}

// Right-hand-side strides of a multi-RHS forward sweep (doubles): slot
// vectors (X, ysave), update workspace, tile partials.
struct RhsStride {
  int64_t x, u, v;
};

// every lane waits until *p >= target (acquire: its later loads see the
// signaller's writes)
__device__ __forceinline__ void lane_wait(const int32_t* p, int target) {
  while (ld_acquire(p) < target) __nanosleep(32);
}

// Preparation warp: for every item the producer publishes, everything its
// consumers need besides the panel, into the item's own shared front vector
// V: the static part first (b or y at the columns, slots and gather maps),
// then the dependency wait, then the part other items produce (the
// children's updates, the parents' solution). The consumers of the CTA are
// still computing the previous item meanwhile, so these global-memory round
// trips are off their path.
template <bool kFwd, int NR>
__device__ void preparer(const SweepDev& p, ItemRec* rec, double* vecs, const double* __restrict__ X,
                         const double* __restrict__ ysave, const double* upd, const double* Xw, RhsStride rs) {
  const int lane = threadIdx.x & 31;
  for (int k = 0;; ++k) {
    ItemRec& R = rec[k % kItems];
    double* V = vecs + (size_t)(k % kItems) * p.vec;
    mbar_wait(&R.info, (k / kItems) & 1);
    if (R.item.x < 0) {
      mbar_arrive(&R.ready);
      return;
    }
    const FrontDesc d = R.d;
    const ItemGeom g = item_geom(p, d, R.item.x, R.item.w, kFwd);
    const int32_t* cs = p.cslot + d.vo;
    if (kFwd) {
      const int ncol = g.jhi - g.jlo;  // <= kSmallRows
      // every batch of loads is issued before its first use (memory-level
      // parallelism: one warp does what 256 threads did)
      int sl[kColsPerLane];
      int2 gc[kColsPerLane];
#pragma unroll
      for (int u = 0; u < kColsPerLane; ++u) {
        const int q = lane + 32 * u;
        sl[u] = q < ncol ? cs[g.jlo + q] : -1;
        gc[u] = q < ncol ? reinterpret_cast<const int2*>(p.gmap)[d.vo + g.jlo + q] : make_int2(-1, -1);
      }
      if (NR == 1) {
        double x[kColsPerLane];
#pragma unroll
        for (int u = 0; u < kColsPerLane; ++u) x[u] = sl[u] >= 0 ? X[sl[u]] : 0.0;
#pragma unroll
        for (int u = 0; u < kColsPerLane; ++u)
          if (sl[u] >= 0) V[lane + 32 * u] = x[u];
      } else {
#pragma unroll
        for (int u = 0; u < kColsPerLane; ++u)
          if (sl[u] >= 0) {
            double x[NR];
#pragma unroll
            for (int rr = 0; rr < NR; ++rr) x[rr] = X[rr * rs.x + sl[u]];
#pragma unroll
            for (int rr = 0; rr < NR; ++rr) V[(lane + 32 * u) * NR + rr] = x[rr];
          }
      }
      if (d.nch > 0) lane_wait(p.done_f + d.cfs0, d.cnf0);
      if (d.nch > 1) lane_wait(p.done_f + d.cfs1, d.cnf1);
      if (lane == 0 && p.trace) R.t_dep = gtimer();
      // the children's updates at the columns: x = v (+ child 0) (+ child 1)
      if (NR == 1) {
        double a0[kColsPerLane], a1[kColsPerLane];
#pragma unroll
        for (int u = 0; u < kColsPerLane; ++u) {
          a0[u] = gc[u].x >= 0 ? __ldcg(upd + gc[u].x) : 0.0;
          a1[u] = gc[u].y >= 0 ? __ldcg(upd + gc[u].y) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < kColsPerLane; ++u)
          if (gc[u].x >= 0 || gc[u].y >= 0) {
            double x = V[lane + 32 * u];
            if (gc[u].x >= 0) x += a0[u];
            if (gc[u].y >= 0) x += a1[u];
            V[lane + 32 * u] = x;
          }
      } else {
#pragma unroll
        for (int u = 0; u < kColsPerLane; ++u)
          if (gc[u].x >= 0 || gc[u].y >= 0) {
            double a0[NR], a1[NR];
#pragma unroll
            for (int rr = 0; rr < NR; ++rr) {
              a0[rr] = gc[u].x >= 0 ? __ldcg(upd + rr * rs.u + gc[u].x) : 0.0;
              a1[rr] = gc[u].y >= 0 ? __ldcg(upd + rr * rs.u + gc[u].y) : 0.0;
            }
#pragma unroll
            for (int rr = 0; rr < NR; ++rr) {
              double x = V[(lane + 32 * u) * NR + rr];
              if (gc[u].x >= 0) x += a0[rr];
              if (gc[u].y >= 0) x += a1[rr];
              V[(lane + 32 * u) * NR + rr] = x;
            }
          }
      }
    } else {
      const int r = d.r, c = d.c;
      constexpr int kB = 8;  // rows per lane and batch
      for (int q0 = g.jlo; q0 < r; q0 += 32 * kB) {  // static: y at the columns, the update rows' slots
        int sl[kB];
#pragma unroll
        for (int u = 0; u < kB; ++u) {
          const int q = q0 + lane + 32 * u;
          sl[u] = q < r ? cs[q] : 0;
        }
        double y[kB];
#pragma unroll
        for (int u = 0; u < kB; ++u) {
          const int q = q0 + lane + 32 * u;
          y[u] = q < c ? ysave[sl[u]] : __longlong_as_double((long long)sl[u]);
        }
#pragma unroll
        for (int u = 0; u < kB; ++u) {
          const int q = q0 + lane + 32 * u;
          if (q < r) V[q] = y[u];
        }
      }
      if (d.pfs >= 0) lane_wait(p.done_b + d.pfs, d.pnb);
      if (lane == 0 && p.trace) R.t_dep = gtimer();
      for (int q0 = max(c, g.jlo); q0 < r; q0 += 32 * kB) {  // the parents' solution at the update rows
        double x[kB];
#pragma unroll
        for (int u = 0; u < kB; ++u) {
          const int q = q0 + lane + 32 * u;
          x[u] = q < r ? __ldcg(Xw + (int)__double_as_longlong(V[q])) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < kB; ++u) {
          const int q = q0 + lane + 32 * u;
          if (q < r) V[q] = -x[u];
        }
      }
    }
    mbar_arrive(&R.ready);  // every lane: its writes to V are published
  }
}

// Forward of one item: o[i] = sum_j G[i, j] v[j] over the item's rows and
// column range for NR right-hand sides at once (rows split over thread
// groups, columns interleaved over the groups: every row's sum has a fixed
// order). One column range: the item writes y (column rows) and the
// parent's update v_rest - o (update rows); several: partial sums to vbuf,
// the last range of a row block to arrive sums them in range order.
// v (the assembled right-hand side at the item's columns) comes prepared.
template <int NR, bool kAcc4>
__device__ void fwd_item(const SweepDev& p, const ItemRec& R, const double* ring, const int* segoff, SlotRec* sr,
                         int& chunk_seq, double* ysave, double* upd, const double* v, double* part, RhsStride rs) {
  const int tid = threadIdx.x;
  const FrontDesc d = R.d;
  const int kind = R.item.x;
  const int64_t fs = (int64_t)R.item.z * p.nsn + R.item.y;
  const int c = d.c;
  const int32_t* cs = p.cslot + d.vo;
  const ItemGeom g = item_geom(p, d, kind, R.item.w, true);
  const int nrow = g.i1 - g.i0;
  const int qr = g.i0 + tid;  // this thread's row (rows <= kThreadsSweep)
  double cu[NR];  // the children's updates at row qr (update rows); the loads overlap the chunk loop
#pragma unroll
  for (int rr = 0; rr < NR; ++rr) cu[rr] = 0.0;
  if (tid < nrow && qr >= c) {
    const int2 gr = reinterpret_cast<const int2*>(p.gmap)[d.vo + qr];
#pragma unroll
    for (int rr = 0; rr < NR; ++rr) {
      if (gr.x >= 0) cu[rr] += __ldcg(upd + rr * rs.u + gr.x);
      if (gr.y >= 0) cu[rr] += __ldcg(upd + rr * rs.u + gr.y);
    }
  }
  const int Rw = (nrow + 31) & ~31, ng = kThreadsSweep / Rw;  // Rw <= kThreadsSweep rows per group, ng groups
  const int row = tid % Rw, grp = tid / Rw, i = g.i0 + row;
  double acc[NR];
  double a4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
  for (int rr = 0; rr < NR; ++rr) acc[rr] = 0.0;
  for (int q = 0; q < g.nchunk; ++q, ++chunk_seq) {
    const int slot = chunk_seq % kSlots;
    const Chunk ch = chunk_of(g, q, true);
    mbar_wait(&sr[slot].full, (chunk_seq / kSlots) & 1);
    const double* S = ring + slot * p.slot;
    const int* so = segoff + slot * kMaxSegs;
    if (grp < ng && row < nrow) {
      // chunk widths are multiples of ng (item_geom): column j of the item
      // belongs to thread group (j - jlo) % ng whatever the ring's slot size
      const int jend = min(ch.jb, i + 1);
      int j = ch.ja + grp;
      if (NR == 1 && kAcc4) {
        // four accumulators by (j - jlo) / ng % 4 break the dependent FMA
        // chain (64 columns per thread of a 128 x 128 tile)
        auto term = [&](int jj) { return S[so[jj - ch.ja] + i] * v[jj - g.jlo]; };
        int ph = ((ch.ja - g.jlo) / ng) & 3;
        if (ph == 1 && j < jend) a4[1] += term(j), j += ng, ph = 2;
        if (ph == 2 && j < jend) a4[2] += term(j), j += ng, ph = 3;
        if (ph == 3 && j < jend) a4[3] += term(j), j += ng;
        for (; j + 3 * ng < jend; j += 4 * ng) {
          a4[0] += term(j);
          a4[1] += term(j + ng);
          a4[2] += term(j + 2 * ng);
          a4[3] += term(j + 3 * ng);
        }
        if (j < jend) a4[0] += term(j), j += ng;
        if (j < jend) a4[1] += term(j), j += ng;
        if (j < jend) a4[2] += term(j), j += ng;
      } else {
        for (; j < jend; j += ng) {
          const double gij = S[so[j - ch.ja] + i];
#pragma unroll
          for (int rr = 0; rr < NR; ++rr) acc[rr] += gij * v[(j - g.jlo) * NR + rr];
        }
      }
    }
    __syncwarp();
    if ((threadIdx.x & 31) == 0) mbar_arrive(&sr[slot].empty);
  }
  if (NR == 1 && kAcc4) acc[0] = (a4[0] + a4[1]) + (a4[2] + a4[3]);
  double o[NR];
  if (ng == 1) {
#pragma unroll
    for (int rr = 0; rr < NR; ++rr) o[rr] = 0.0 + acc[rr];  // the grouped form's sum with one group
  } else {
#pragma unroll
    for (int rr = 0; rr < NR; ++rr) {  // group partials summed in group order, one right-hand side at a time
      if (grp < ng && row < nrow) part[grp * Rw + row] = acc[rr];
      csync();
      o[rr] = 0.0;
      if (tid < nrow)
        for (int q = 0; q < ng; ++q) o[rr] += part[q * Rw + tid];
      csync();
    }
  }
  if (g.mcb > 1) {
    double* tp = p.vbuf + d.tpo + (int64_t)g.rb * g.mcb * kFwdRows;
    if (tid < nrow)
#pragma unroll
      for (int rr = 0; rr < NR; ++rr) tp[rr * rs.v + (int64_t)g.cb * kFwdRows + tid] = o[rr];
    __shared__ int s_last;
    csync();
    const int ncb = max(1, (min(c, g.i1) + p.fwd_cols - 1) / p.fwd_cols);
    if (tid == 0) {
      __threadfence();
      s_last = atomicAdd(p.rbcnt + d.rbo + g.rb, 1) == ncb - 1;
      if (s_last) __threadfence();
    }
    csync();
    if (!s_last) return;  // another range of the row block finishes it
    if (tid < nrow)
#pragma unroll
      for (int rr = 0; rr < NR; ++rr) {
        o[rr] = 0.0;
        for (int k = 0; k < ncb; ++k) o[rr] += __ldcg(tp + rr * rs.v + (int64_t)k * kFwdRows + tid);
      }
  }
  if (tid < nrow) {
    if (qr < c) {
      const int sl = cs[qr];
#pragma unroll
      for (int rr = 0; rr < NR; ++rr) ysave[rr * rs.x + sl] = o[rr];
    } else {
#pragma unroll
      for (int rr = 0; rr < NR; ++rr) upd[rr * rs.u + d.uo + qr - c] = cu[rr] - o[rr];
    }
  }
  cta_signal(p.done_f + fs);
}

// Backward of one item: columns [j0, j1) of a front, x_j = sum_{i >= j}
// G[i, j] w[i] with w = [y; -x_rest] (prepared); warp w owns columns
// j0 + w + 8k, its lanes stride over the rows of every chunk (register
// accumulators, fixed order), one warp sum per column at the end.
__device__ void bwd_item(const SweepDev& p, const ItemRec& R, const double* ring, const int* segoff, SlotRec* sr,
                         int& chunk_seq, double* X, const double* w) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const FrontDesc d = R.d;
  const int64_t fs = (int64_t)R.item.z * p.nsn + R.item.y;
  const int32_t* cs = p.cslot + d.vo;
  const ItemGeom g = item_geom(p, d, R.item.x, R.item.w, false);
  constexpr int kPer = kMaxBwdCols / kWarps;
  int slj[kPer];  // the columns' slots (static)
#pragma unroll
  for (int k = 0; k < kPer; ++k) {
    const int j = g.jlo + wid + kWarps * k;
    slj[k] = (lane == 0 && j < g.jhi) ? cs[j] : 0;
  }
  double acc[kPer];
#pragma unroll
  for (int k = 0; k < kPer; ++k) acc[k] = 0.0;
  for (int q = 0; q < g.nchunk; ++q, ++chunk_seq) {
    const int slot = chunk_seq % kSlots;
    const Chunk ch = chunk_of(g, q, false);
    mbar_wait(&sr[slot].full, (chunk_seq / kSlots) & 1);
    const double* S = ring + slot * p.slot;
    const int* so = segoff + slot * kMaxSegs;
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      const int j = g.jlo + wid + kWarps * k;
      if (j < g.jhi) {  // row i of column j belongs to lane (i - j) % 32, whatever the chunking
        const int lo = max(j, ch.lo);
        for (int i = lo + ((lane - (lo - j)) & 31); i < ch.hi; i += 32) acc[k] += S[so[j - g.jlo] + i] * w[i];
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&sr[slot].empty);
  }
#pragma unroll
  for (int k = 0; k < kPer; ++k) {
    const int j = g.jlo + wid + kWarps * k;
    const double sum = warp_sum(acc[k]);
    if (lane == 0 && j < g.jhi) X[slj[k]] = sum;
  }
  cta_signal(p.done_b + fs);
}

// Warp-specialised persistent CTA: kWarps consumer warps, one producer warp
// and one preparation warp. The producer takes tickets in order and streams
// every item's panel through a kSlots-deep ring of shared-memory chunks
// (bulk copies, mbarrier transaction counts); the preparation warp waits for
// the item's dependencies and assembles its front vector; both run one item
// ahead of the consumers, which only wait for a prepared item, multiply from
// shared memory and publish the result. A CTA holds at most kItems tickets
// and runs them in ticket order, so the smallest unfinished ticket is always
// some CTA's current item, whose dependencies (smaller tickets) are done,
// and whose chunks come first in its ring: no deadlock.
template <bool kFwd, int NR = 1, bool kAcc4 = false>
__device__ __forceinline__ void sweep_loop(const SweepDev& p, const int4* __restrict__ items, int n_items,
                                           int32_t* ticket, const double* __restrict__ panel, const double* X,
                                           double* Xw, const double* ysave_in, double* ysave, double* upd,
                                           RhsStride rs = RhsStride{0, 0, 0}) {
  extern __shared__ __align__(128) double shm[];
  double* ring = shm;
  double* vecs = shm + kSlots * p.slot;
  double* part = vecs + (size_t)kItems * p.vec;
  int* segoff = reinterpret_cast<int*>(part + kThreadsSweep);  // kSlots x kMaxSegs
  __shared__ ItemRec rec[kItems];
  __shared__ SlotRec sr[kSlots];
  if (threadIdx.x == 0) {
    for (int k = 0; k < kItems; ++k) {
      mbar_init(&rec[k].info, 1);
      mbar_init(&rec[k].ready, 32);
      mbar_init(&rec[k].empty, 1);
    }
    for (int k = 0; k < kSlots; ++k) {
      mbar_init(&sr[k].full, 1);
      mbar_init(&sr[k].empty, kWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x >= kThreadsSweep + 32) {
    preparer<kFwd, NR>(p, rec, vecs, X, ysave_in, upd, Xw, rs);
    return;
  }
  if (threadIdx.x >= kThreadsSweep) {
    producer(p, items, n_items, ticket, panel, rec, sr, ring, segoff, kFwd);
    return;
  }
  int chunk_seq = 0;
  for (int k = 0;; ++k) {
    ItemRec& R = rec[k % kItems];
    const double* V = vecs + (size_t)(k % kItems) * p.vec;
    mbar_wait(&R.ready, (k / kItems) & 1);
    if (R.item.x < 0) break;
    if (kFwd)
      fwd_item<NR, kAcc4>(p, R, ring, segoff, sr, chunk_seq, ysave, upd, V, part, rs);
    else
      bwd_item(p, R, ring, segoff, sr, chunk_seq, Xw, V);
    csync();  // every consumer is done with the record and the vector
    if (threadIdx.x == 0) {
      if (p.trace) {  // per ticket: {grab, dependencies met, done, SM}
        unsigned long long* tr = p.trace + 4ll * R.tk;
        tr[0] = R.t_grab;
        tr[1] = R.t_dep;
        tr[2] = gtimer();
        tr[3] = smid();
      }
      mbar_arrive(&R.empty);
    }
  }
}

#ifndef CUTBDDC_SWEEP_ACC4
#define CUTBDDC_SWEEP_ACC4 0  // A/B on B200: four accumulators lose (cfg4 0.291 -> 0.301 ms, cfg5 6.49 -> 6.77 ms per apply)
#endif
constexpr bool kFwdAcc4 = CUTBDDC_SWEEP_ACC4 != 0;  // the same arithmetic in both builds (ranks may run either)
// Two builds of each sweep kernel: kMinBlocks CTAs per SM (48 registers, the
// many-subdomain ring) and kMinBlocks - 1 (68 registers, the few-subdomain
// ring, whose larger slots leave room for three CTAs anyway).
__global__ void __launch_bounds__(kBlockSweep, kMinBlocks) k_sweep_fwd(SweepDev p, const int4* __restrict__ items, int n_items,
                                                             const double* __restrict__ panel,
                                                             const double* __restrict__ X, double* __restrict__ ysave,
                                                             double* upd, const int* __restrict__ skip) {
  if (skip && *skip) return;
  sweep_loop<true, 1, kFwdAcc4>(p, items, n_items, p.ticket, panel, X, nullptr, nullptr, ysave, upd);
}
__global__ void __launch_bounds__(kBlockSweep, kMinBlocks - 1) k_sweep_fwd_few(SweepDev p, const int4* __restrict__ items,
                                                                 int n_items, const double* __restrict__ panel,
                                                                 const double* __restrict__ X,
                                                                 double* __restrict__ ysave, double* upd,
                                                                 const int* __restrict__ skip) {
  if (skip && *skip) return;
  sweep_loop<true, 1, kFwdAcc4>(p, items, n_items, p.ticket, panel, X, nullptr, nullptr, ysave, upd);
}

// Forward sweep of kMultiRhs right-hand sides at once (the coarse-basis
// setup: H = L^{-1} C^T), same items and schedule as k_sweep_fwd.
constexpr int kMultiRhs = kSweepMultiRhs;
static_assert(kMultiRhs * kSmallRows <= 4096, "multi-RHS front vector");
#ifndef CUTBDDC_MULTI_MIN_BLOCKS
#define CUTBDDC_MULTI_MIN_BLOCKS 1
#endif
__global__ void __launch_bounds__(kBlockSweep, CUTBDDC_MULTI_MIN_BLOCKS) k_sweep_fwd_multi(SweepDev p, const int4* __restrict__ items, int n_items,
                                                             const double* __restrict__ panel,
                                                             const double* __restrict__ X, double* __restrict__ ysave,
                                                             double* upd, RhsStride rs) {
  sweep_loop<true, kMultiRhs>(p, items, n_items, p.ticket, panel, X, nullptr, nullptr, ysave, upd, rs);
}

__global__ void __launch_bounds__(kBlockSweep, kMinBlocks) k_sweep_bwd(SweepDev p, const int4* __restrict__ items, int n_items,
                                                             const double* __restrict__ panel, double* X,
                                                             const double* __restrict__ ysave,
                                                             const int* __restrict__ skip, int ticket_slot) {
  if (skip && *skip) return;
  sweep_loop<false>(p, items, n_items, p.ticket + ticket_slot, panel, nullptr, X, ysave, nullptr, nullptr);
}
__global__ void __launch_bounds__(kBlockSweep, kMinBlocks - 1) k_sweep_bwd_few(SweepDev p, const int4* __restrict__ items,
                                                                 int n_items, const double* __restrict__ panel,
                                                                 double* X, const double* __restrict__ ysave,
                                                                 const int* __restrict__ skip, int ticket_slot) {
  if (skip && *skip) return;
  sweep_loop<false>(p, items, n_items, p.ticket + ticket_slot, panel, nullptr, X, ysave, nullptr, nullptr);
}

// compact slot of every front row, the parent position of every update entry
// (umap) and its inverse (gmap: per parent row, the entry of child 0 / 1)
__global__ void k_sweep_maps(TplDev t, FactorDev f, const FrontDesc* __restrict__ desc, int32_t* __restrict__ cslot,
                             int32_t* __restrict__ umap, int32_t* __restrict__ gmap) {
  const int sid = blockIdx.x, sd = blockIdx.y;
  const Supernode s = t.sn[sid];
  const int64_t fs = (int64_t)sd * t.nsn + sid;
  const int32_t* pf = f.pfx + (int64_t)sd * t.rows_total + s.rows_off;
  const int64_t vo = desc[fs].vo;
  for (int q = threadIdx.x; q < s.nrows; q += blockDim.x) {
    const int pq = pf[q];
    if (pq >= 0) cslot[vo + pq] = sd * t.T + t.rows[s.rows_off + q];  // index into the nsd x T slot vector
  }
  if (s.parent < 0) return;
  const Supernode ps = t.sn[s.parent];
  const int32_t* ppf = f.pfx + (int64_t)sd * t.rows_total + ps.rows_off;
  const int c = desc[fs].c;
  const int64_t uo = desc[fs].uo;
  const int64_t pvo = desc[(int64_t)sd * t.nsn + s.parent].vo;
  const int chx = ps.child[0] == sid ? 0 : 1;
  for (int a = threadIdx.x; a < s.nrows - s.ncols; a += blockDim.x) {
    const int ia = pf[s.ncols + a];
    if (ia < 0) continue;
    const int pp = ppf[t.emap[s.emap_off + a]];
    umap[uo + ia - c] = pp;
    gmap[2 * (pvo + pp) + chx] = (int32_t)(uo + ia - c);
  }
}

SweepDev sweep_dev(const FactorSet& f, int nsd, int nsn, unsigned long long* trace) {
  const int64_t n = (int64_t)nsd * nsn;
  int32_t* cnt = const_cast<int32_t*>(f.counters.p);
  return SweepDev{reinterpret_cast<const FrontDesc*>(f.desc.p),
                  f.cslot.p,
                  f.umap.p,
                  f.gmap.p,
                  nsn,
                  cnt,
                  cnt + n,
                  cnt + 2 * n,
                  cnt + 3 * n,
                  cnt + 4 * n,
                  cnt + 4 * n + 3,
                  const_cast<double*>(f.vbuf.p),
                  f.fwd_cols,
                  f.bwd_cols,
                  f.sweep_vec,
                  f.sweep_slot,
                  f.sweep_bwd_rows,
                  f.l2_policy_f,
                  trace};
}

const char* trace_prefix() {
  static const char* e = std::getenv("CUTBDDC_SWEEP_TRACE");
  return e && e[0] ? e : nullptr;
}

// host dump of one sweep's trace: items (int4) then timestamps (4 x u64 per item)
void dump_trace(const std::string& path, const FactorSet& f, bool fwd, cudaStream_t s) {
  const int n = fwd ? f.n_items_f : f.n_items_b;
  std::vector<int4> items = (fwd ? f.items_f : f.items_b).to_host(s);
  std::vector<unsigned long long> tr((size_t)4 * n);
  f.trace.download(tr.data(), tr.size(), s);
  CB_CUDA(cudaStreamSynchronize(s));
  FILE* fp = std::fopen(path.c_str(), "wb");
  if (!fp) return;
  std::fwrite(&n, sizeof(int), 1, fp);
  std::fwrite(items.data(), sizeof(int4), (size_t)n, fp);
  std::fwrite(tr.data(), sizeof(unsigned long long), tr.size(), fp);
  std::fclose(fp);
}

// CTAs of a persistent sweep launch: every SM filled at the occupancy of
// (kernel, shared-memory size); memoised per device for the sizes in use.
int sweep_grid(const void* fn, size_t shm) {
  static std::mutex mu;
  static std::map<std::tuple<int, const void*, size_t>, int> memo;
  int dev = 0;
  CB_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  const auto key = std::make_tuple(dev, fn, shm);
  auto it = memo.find(key);
  if (it != memo.end()) return it->second;
  int per_sm = 0, sms = 0;
  CB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kBlockSweep, shm));
  CB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int g = std::max(1, per_sm) * sms;
  memo[key] = g;
  return g;
}

}  // namespace

// Host: descriptors, maps, completion counts and the ordered work lists of
// one factorisation (after its symbolic phase; poff / uoff are the panel and
// update offsets per (sd, supernode) the numeric phase uses).
// Item sizes of one factorisation's sweeps: wide items (long streams per
// item, fewer fixed per-item latencies) when there are many fronts to run
// side by side, narrower ones when the elimination tree's levels are few
// items wide (tuned on B200: cfg5 with 1 960 subdomains prefers 256 / 32,
// cfg4 with 51 prefers 128 / 16). CUTBDDC_SWEEP_ITEMS=fwd,bwd overrides.
void choose_item_sizes(cutbddc_gpu* h, FactorSet& f) {
  const bool wide = h->nsd >= 256;
  int fc = wide ? 256 : 128, bc = wide ? 32 : 16, sw = wide ? 32768 : 8192;
  if (const char* e = std::getenv("CUTBDDC_SWEEP_ITEMS")) std::sscanf(e, "%d,%d,%d", &fc, &bc, &sw);
  bc = std::max(kWarps, std::min(kMaxBwdCols, bc / kWarps * kWarps));
  f.fwd_cols = std::max(16, std::min(kSmallRows, fc));  // <= kSmallRows: the multi-RHS front vector fits
  f.bwd_cols = bc;
  f.small_work = std::max(1, sw);
  // L2 eviction priority of the panel loads (0 default, 1 evict_last, 2
  // evict_first). The panels (172 MB at cfg4) do not fit the 126 MB L2, and
  // streaming them evict_first keeps the apply's vectors, maps and coarse
  // basis resident: measured on B200, cfg4 PCG 6.25 -> 5.96 ms, cfg5 239 ->
  // 235 ms. CUTBDDC_SWEEP_L2=iF,iB,kF,kB overrides (interior / Neumann
  // factor, forward / backward sweep).
  int pol[4] = {2, 2, 2, 2};
  if (const char* e = std::getenv("CUTBDDC_SWEEP_L2")) std::sscanf(e, "%d,%d,%d,%d", pol, pol + 1, pol + 2, pol + 3);
  const bool interior = &f == &h->fI;
  f.l2_policy_f = interior ? pol[0] : pol[2];
  f.l2_policy_b = interior ? pol[1] : pol[3];
}

void build_sweep_plan(cutbddc_gpu* h, const TplSet& ts, FactorSet& f, const std::vector<int64_t>& poff,
                      const std::vector<int64_t>& uoff) {
  cudaStream_t s = h->stream;
  const Template& tp = ts.tpl;
  const int nsd = h->nsd, nsn = (int)tp.sn.size();
  const auto& lv = tp.levels;
  const int nlev = (int)lv.size();
  if (tp.max_rows > kVecMax) throw Failure(CUTBDDC_CONFIG, "sweep: front larger than the shared vector");
  choose_item_sizes(h, f);
  // shared front vector of this factorisation's sweeps: its largest front
  // (backward) or one column range (forward), 64-double granules
  f.sweep_vec = (std::max({tp.max_rows, f.fwd_cols, kSmallRows}) + 63) & ~63;
  // ring slots: the largest that still lets 4 (many subdomains) or 3 (few)
  // CTAs share an SM's 228 KB (1 KB reserved and ~0.5 KB static per CTA)
  {
    const int ctas = h->nsd >= 256 ? 4 : 3;
    const long long per_cta = 228 * 1024 / ctas - 1024 - 512;
    const long long rest = (long long)sweep_shm_bytes(0, f.sweep_vec);
    long long slot = (per_cta - rest) / (8 * kSlots) / 32 * 32;
    slot = std::max<long long>(h->nsd >= 256 ? kSlotWide : kSlotFew, std::min<long long>(slot, 4096));
    f.sweep_slot = (int)slot;
    // backward chunks fill the slot: bwd_cols columns x as many rows as fit (even: a staged column takes rows + 2 doubles)
    f.sweep_bwd_rows = std::min(1024, ((int)slot / f.bwd_cols - 2) & ~1);
  }
#if defined(CUTBDDC_SWEEP_SLOT_DOUBLES) && defined(CUTBDDC_SWEEP_BWD_ROWS)
  f.sweep_slot = CUTBDDC_SWEEP_SLOT_DOUBLES;
  f.sweep_bwd_rows = CUTBDDC_SWEEP_BWD_ROWS;
#endif
  if (const char* e = std::getenv("CUTBDDC_SWEEP_RING")) std::sscanf(e, "%d,%d", &f.sweep_slot, &f.sweep_bwd_rows);  // A/B hook
  if (std::getenv("CUTBDDC_SWEEP_STATS"))
    std::fprintf(stderr, "[sweep stats] nsd %d max_rows %d vec %d slot %d bwd_rows %d shm %zu\n", h->nsd, tp.max_rows,
                 f.sweep_vec, f.sweep_slot, f.sweep_bwd_rows, sweep_shm_bytes(f.sweep_slot, f.sweep_vec));
  if (f.bwd_cols * seg_stride(f.sweep_bwd_rows) > f.sweep_slot || 16 * seg_stride(kFwdRows) > f.sweep_slot)
    throw Failure(CUTBDDC_INTERNAL, "sweep: chunk sizes exceed the ring slot");
  const int fc = f.fwd_cols, bc = f.bwd_cols;
  // S item: a front whose whole forward is one item (one row block, at most
  // small_work panel entries); larger fronts: row blocks x column ranges
  auto is_small = [&f](int2 rc) { return rc.x <= kSmallRows && (int64_t)rc.x * rc.y <= f.small_work; };
  // completion counts: forward items per front (T items signal their root),
  // backward items per front (every front with rows above the subtrees has
  // at least one, so waiting on the parent covers every ancestor)
  std::vector<int32_t> nf((size_t)nsd * nsn, 0), nb((size_t)nsd * nsn, 0);
  std::vector<int64_t> voff((size_t)nsd * nsn);
  int64_t tot = 0;
  for (int sd = 0; sd < nsd; ++sd)
    for (int q = 0; q < nsn; ++q) {
      const int2 v = f.h_rc[(size_t)sd * nsn + q];
      const size_t i = (size_t)sd * nsn + q;
      voff[i] = tot;
      tot += v.x;
      nf[i] = v.x == 0 ? 0 : is_small(v) ? 1 : (v.x + kFwdRows - 1) / kFwdRows;
      nb[i] = v.x == 0 ? 0 : std::max(1, (v.y + bc - 1) / bc);
    }
  f.vec_total = tot;
  f.h_vec_off = voff;
  // forward tiles of chunked fronts: partial storage (after the front
  // vectors in vbuf) and one arrival counter per row block
  auto mcb_of = [fc](int c) { return std::max(1, (c + fc - 1) / fc); };
  auto ncb_of = [fc](int r, int c, int rb) {
    return std::max(1, (std::min(c, std::min(r, (rb + 1) * kFwdRows)) + fc - 1) / fc);
  };
  std::vector<int64_t> tpo((size_t)nsd * nsn, 0);
  std::vector<int32_t> rbo((size_t)nsd * nsn, 0);
  int64_t ptot = tot;
  int32_t nrb_tot = 0;
  for (size_t i = 0; i < (size_t)nsd * nsn; ++i) {
    const int2 v = f.h_rc[i];
    if (is_small(v)) continue;
    const int nrb = (v.x + kFwdRows - 1) / kFwdRows;
    tpo[i] = ptot;
    ptot += (int64_t)nrb * mcb_of(v.y) * kFwdRows;
    rbo[i] = nrb_tot;
    nrb_tot += nrb;
  }
  std::vector<FrontDesc> desc((size_t)nsd * nsn);
  for (int sd = 0; sd < nsd; ++sd)
    for (int q = 0; q < nsn; ++q) {
      const size_t i = (size_t)sd * nsn + q;
      const Supernode& sn = tp.sn[(size_t)q];
      const int2 v = f.h_rc[i];
      FrontDesc& d = desc[i];
      d = FrontDesc{};
      d.r = v.x;
      d.c = v.y;
      d.vo = voff[i];
      d.po = poff[i];
      d.uo = uoff[i];
      d.tpo = tpo[i];
      d.rbo = rbo[i];
      d.nch = sn.nchild;
      d.cfs0 = d.cfs1 = -1;
      for (int ch = 0; ch < sn.nchild; ++ch) {
        const size_t ci = (size_t)sd * nsn + sn.child[ch];
        const int2 cv = f.h_rc[ci];
        if (ch == 0) {
          d.cfs0 = (int)ci;
          d.cnu0 = cv.x - cv.y;
          d.cuo0 = uoff[ci];
          d.cnf0 = nf[ci];
        } else {
          d.cfs1 = (int)ci;
          d.cnu1 = cv.x - cv.y;
          d.cuo1 = uoff[ci];
          d.cnf1 = nf[ci];
        }
      }
      // backward: the parent's columns hold every row of this front once the
      // parent's items are done (they waited for their own parent)
      d.pfs = -1;
      if (sn.parent >= 0 && v.x > v.y) {
        d.pfs = (int)((size_t)sd * nsn + sn.parent);
        d.pnb = nb[(size_t)d.pfs];
      }
    }
  f.items_ready = false;
  f.desc.upload(reinterpret_cast<const int4*>(desc.data()), desc.size() * 6, s);
  f.cslot.alloc((size_t)std::max<int64_t>(1, tot));
  f.umap.alloc((size_t)std::max<int64_t>(1, f.upd_total));
  if (f.upd_total >= (1ll << 31)) throw Failure(CUTBDDC_CONFIG, "sweep: update workspace exceeds 32-bit indexing");
  f.gmap.alloc((size_t)2 * std::max<int64_t>(1, tot));
  CB_CUDA(cudaMemsetAsync(f.gmap.p, 0xff, sizeof(int32_t) * f.gmap.n, s));
  f.vbuf.alloc((size_t)std::max<int64_t>(1, ptot));
  f.counters.alloc((size_t)4 * nsd * nsn + 3 + nrb_tot);
  const TplDev t = tpl_dev(ts, h->slots);
  k_sweep_maps<<<dim3(nsn, nsd), 256, 0, s>>>(t, factor_dev(f), reinterpret_cast<const FrontDesc*>(f.desc.p),
                                              f.cslot.p, f.umap.p, f.gmap.p);
  CB_LAUNCH();
  // no synchronisation: uploads from pageable host memory return once the
  // data is staged, so the host vectors above may go out of scope
}

// The sweeps' work items in dependency (critical-path) order. Needed only by
// the solves, so setup builds them on the host while the GPU factorises.
void build_sweep_items(cutbddc_gpu* h, const TplSet& ts, FactorSet& f, const std::vector<uint8_t>* exclude) {
  cudaStream_t s = h->stream;
  const Template& tp = ts.tpl;
  const int nsd = h->nsd, nsn = (int)tp.sn.size();
  const auto& lv = tp.levels;
  const int nlev = (int)lv.size();
  const int fc = f.fwd_cols, bc = f.bwd_cols;
  auto is_small = [&f](int2 rc) { return rc.x <= kSmallRows && (int64_t)rc.x * rc.y <= f.small_work; };
  std::vector<int32_t> nf((size_t)nsd * nsn, 0), nb((size_t)nsd * nsn, 0);
  for (size_t i = 0; i < (size_t)nsd * nsn; ++i) {
    const int2 v = f.h_rc[i];
    nf[i] = v.x == 0 ? 0 : is_small(v) ? 1 : (v.x + kFwdRows - 1) / kFwdRows;
    nb[i] = v.x == 0 ? 0 : std::max(1, (v.y + bc - 1) / bc);
  }
  auto mcb_of = [fc](int c) { return std::max(1, (c + fc - 1) / fc); };
  auto ncb_of = [fc](int r, int c, int rb) {
    return std::max(1, (std::min(c, std::min(r, (rb + 1) * kFwdRows)) + fc - 1) / fc);
  };
  std::vector<int4> fw, bw;
  auto front_items = [&](int L, bool fwd, std::vector<int4>& out) {
    for (int sid : lv[(size_t)L])
      for (int sd = 0; sd < nsd; ++sd) {
        if (exclude && (*exclude)[(size_t)sd]) continue;
        const int2 v = f.h_rc[(size_t)sd * nsn + sid];
        if (v.x > 0 && (fwd ? is_small(v) : v.y == 0)) out.push_back(make_int4(kItemS, sid, sd, 0));
      }
    for (int sid : lv[(size_t)L])
      for (int sd = 0; sd < nsd; ++sd) {
        if (exclude && (*exclude)[(size_t)sd]) continue;
        const size_t i = (size_t)sd * nsn + sid;
        const int2 v = f.h_rc[i];
        if (fwd && is_small(v)) continue;
        if (fwd) {
          const int mcb = mcb_of(v.y);
          for (int rb = 0; rb < nf[i]; ++rb)
            for (int cb = 0; cb < ncb_of(v.x, v.y, rb); ++cb) out.push_back(make_int4(kItemC, sid, sd, rb * mcb + cb));
        } else if (v.y > 0) {
          for (int k = 0; k < nb[i]; ++k) out.push_back(make_int4(kItemC, sid, sd, k));
        }
      }
  };
  for (int L = nlev - 1; L >= 0; --L) front_items(L, true, fw);  // leaves first
  for (int L = 0; L < nlev; ++L) {  // root first
    front_items(L, false, bw);
    if (L == 0) f.n_items_b_root = (int)bw.size();
  }
  // Critical path first: every item's ticket follows the longest remaining
  // path (estimated work) to the end of its sweep, as in the factorisation's
  // DAG. Weights are positive, so a front's items always rank after those of
  // its children (forward) / its parent (backward): still a topological
  // order. Ties keep the level order (stable sort).
  {
    constexpr double kItemCost = 4096.0;  // per-item latency in panel entries
    const size_t nf_all = (size_t)nsd * nsn;
    auto rc = [&](int sd, int sid) { return f.h_rc[(size_t)sd * nsn + sid]; };
    auto entries = [](int2 v) { return (double)v.x * v.y; };
    auto fwd_item = [&](int sd, int sid) {  // work of one item of a front
      const int2 v = rc(sd, sid);
      return kItemCost + (is_small(v) ? entries(v) : (double)std::min(v.x, kFwdRows) * std::min(v.y, fc));
    };
    auto bwd_item = [&](int sd, int sid) {
      const int2 v = rc(sd, sid);
      return kItemCost + (double)v.x * std::min(std::max(v.y, 1), bc);
    };
    // forward: remaining path from a front to the root (top-down over levels)
    std::vector<double> remf(nf_all, 0.0), remb(nf_all, 0.0);
    for (int L = 0; L < nlev; ++L)
      for (int sid : lv[(size_t)L])
        for (int sd = 0; sd < nsd; ++sd) {
          const int par = tp.sn[(size_t)sid].parent;
          const double up = par >= 0 ? remf[(size_t)sd * nsn + par] : 0.0;
          remf[(size_t)sd * nsn + sid] = up + fwd_item(sd, sid);
        }
    // backward: remaining path from a front down to its deepest descendant
    for (int L = nlev - 1; L >= 0; --L)
      for (int sid : lv[(size_t)L])
        for (int sd = 0; sd < nsd; ++sd) {
          const Supernode& sn = tp.sn[(size_t)sid];
          double down = 0.0;
          for (int ch = 0; ch < sn.nchild; ++ch) down = std::max(down, remb[(size_t)sd * nsn + sn.child[ch]]);
          remb[(size_t)sd * nsn + sid] =
              down + bwd_item(sd, sid);
        }
    auto key = [&](const int4& it, bool fwd) {
      const size_t i = (size_t)it.z * nsn + it.y;
      return fwd ? remf[i] : remb[i];
    };
    auto order = [&](std::vector<int4>& v, size_t b, size_t e, bool fwd) {
      const size_t n = e - b;
      std::vector<double> k(n);
      std::vector<int32_t> ix(n);
      for (size_t q = 0; q < n; ++q) {
        k[q] = key(v[b + q], fwd);
        ix[q] = (int32_t)q;
      }
      std::sort(ix.begin(), ix.end(), [&](int32_t x, int32_t y) { return k[x] > k[y] || (k[x] == k[y] && x < y); });
      std::vector<int4> out(n);
      for (size_t q = 0; q < n; ++q) out[q] = v[b + ix[q]];
      std::copy(out.begin(), out.end(), v.begin() + (std::ptrdiff_t)b);
    };
    static const bool level_order = std::getenv("CUTBDDC_SWEEP_LEVEL_ORDER") != nullptr;  // A/B: plain level order
    if (!level_order) {
      const size_t nroot = std::min(bw.size(), (size_t)std::max(0, f.n_items_b_root));
      order(fw, 0, fw.size(), true);
      order(bw, 0, nroot, false);  // the root phase stays a launch of its own
      order(bw, nroot, bw.size(), false);
    }
  }
  if (std::getenv("CUTBDDC_SWEEP_STATS")) {  // item census: count, panel entries (sum, max) per kind
    auto census = [&, fc, bc](const std::vector<int4>& v, const char* dir) {
      double cnt[4] = {0, 0, 0, 0}, sum[4] = {0, 0, 0, 0}, mx[4] = {0, 0, 0, 0};
      for (const int4& it : v) {
        const int2 rc = f.h_rc[(size_t)it.z * nsn + it.y];
        double e = (double)rc.x * rc.y;
        if (it.x == kItemC) {
          e = dir[0] == 'f' ? (double)std::min(rc.x, kFwdRows) * std::min(rc.y, fc)
                            : (double)rc.x * std::min(rc.y, bc);
        }
        cnt[it.x] += 1;
        sum[it.x] += e;
        mx[it.x] = std::max(mx[it.x], e);
      }
      const char* nm[4] = {"S", "A", "C", "T"};
      for (int k = 0; k < 4; ++k)
        if (cnt[k] > 0)
          std::fprintf(stderr, "[sweep stats] %s %s: items %.0f, entries sum %.3g mean %.0f max %.0f\n", dir, nm[k],
                       cnt[k], sum[k], sum[k] / cnt[k], mx[k]);
    };
    census(fw, "fwd");
    census(bw, "bwd");
  }
  f.n_items_f = (int)fw.size();
  f.n_items_b = (int)bw.size();
  if (!exclude) {  // kept for exclude_sweep_items (a mixed K drops a few subdomains later)
    f.h_items_f = fw;
    f.h_items_b = bw;
  }
  if (fw.empty()) fw.push_back(make_int4(0, 0, 0, 0));
  if (bw.empty()) bw.push_back(make_int4(0, 0, 0, 0));
  f.items_f.upload(fw, s);
  f.items_b.upload(bw, s);
  f.items_ready = true;
}

// Drop the items of the excluded subdomains from the lists build_sweep_items
// made for all of them (same order: subdomains are independent, so the rest
// is still in dependency order). The same lists as a rebuild with `exclude`
// up to the order of equal-cost items, at a fraction of the host time (cfg5:
// 260 k items, ~40 ms of sorting saved per setup).
void exclude_sweep_items(cutbddc_gpu* h, FactorSet& f, const std::vector<uint8_t>& exclude) {
  cudaStream_t s = h->stream;
  if (!f.items_ready || (f.h_items_f.empty() && f.h_items_b.empty()))
    throw Failure(CUTBDDC_INTERNAL, "sweep: no item lists to filter");
  std::vector<int4> fw, bw;
  fw.reserve(f.h_items_f.size());
  bw.reserve(f.h_items_b.size());
  for (const int4& it : f.h_items_f)
    if (!exclude[(size_t)it.z]) fw.push_back(it);
  int nroot = 0;
  for (size_t q = 0; q < f.h_items_b.size(); ++q) {
    const int4& it = f.h_items_b[q];
    if (exclude[(size_t)it.z]) continue;
    if ((int)q < f.n_items_b_root) ++nroot;
    bw.push_back(it);
  }
  f.n_items_f = (int)fw.size();
  f.n_items_b = (int)bw.size();
  f.n_items_b_root = nroot;
  if (fw.empty()) fw.push_back(make_int4(0, 0, 0, 0));
  if (bw.empty()) bw.push_back(make_int4(0, 0, 0, 0));
  f.items_f.upload(fw, s);
  f.items_b.upload(bw, s);
  CB_CUDA(cudaStreamSynchronize(s));  // fw / bw leave scope
}


// In-place solve of one right-hand side X (nsd x T slot vector) in phases:
// kSweepFwd resets the counters and runs the forward sweep; kSweepBwd the
// whole backward sweep; kSweepBwdRoot / kSweepBwdRest split it after the
// root level (the BDDC apply corrects the root solution in between).
void sweep_phase(cutbddc_gpu* h, const TplSet& ts, const FactorSet& f, double* X, double* ysave, double* upd,
                 const int* skip, int phase) {
  if (!f.items_ready) throw Failure(CUTBDDC_INTERNAL, "sweep: item lists not built");
  cudaStream_t s = h->stream;
  const int nsd = h->nsd, nsn = (int)ts.tpl.sn.size();
  const char* tp = trace_prefix();
  FactorSet& fm = const_cast<FactorSet&>(f);
  if (tp) fm.trace.alloc((size_t)4 * std::max(f.n_items_f, f.n_items_b) + 4);
  const SweepDev p = sweep_dev(f, nsd, nsn, tp ? fm.trace.p : nullptr);
  const size_t shm = sweep_shm_bytes(f.sweep_slot, f.sweep_vec);
  device_memo(kMemoSweepAttr, [&] {
    const int mx = 200 * 1024;  // any ring / vector size in use
    CB_CUDA(cudaFuncSetAttribute(k_sweep_fwd, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
    CB_CUDA(cudaFuncSetAttribute(k_sweep_bwd, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
    CB_CUDA(cudaFuncSetAttribute(k_sweep_fwd_few, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
    CB_CUDA(cudaFuncSetAttribute(k_sweep_bwd_few, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
    CB_CUDA(cudaFuncSetAttribute(k_sweep_fwd_multi, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
    return 1ll;
  });
  if (phase == kSweepAttrOnly) return;
  // the 68-register build when the ring leaves room for at most kMinBlocks - 1 CTAs per SM anyway
  const bool few = (228 * 1024) / (shm + 1536) < (size_t)kMinBlocks;
  const std::string tag = std::string("sweep") + (&f == &h->fI ? "I" : "K");
  if (phase == kSweepFwd) {
    CB_CUDA(cudaMemsetAsync(f.counters.p, 0, sizeof(int32_t) * f.counters.n, s));
    ProfScope ps(h->prof, s, tag + " fwd");
    if (f.n_items_f > 0) {
      auto kern = few ? k_sweep_fwd_few : k_sweep_fwd;
      const int g = std::min(f.n_items_f, sweep_grid((const void*)kern, shm));
      kern<<<g, kBlockSweep, shm, s>>>(p, f.items_f.p, f.n_items_f, f.panel.p, X, ysave, upd, skip);
      CB_LAUNCH();
    }
    if (tp) dump_trace(std::string(tp) + "_" + tag + "_fwd.bin", f, true, s);
    return;
  }
  int b0 = 0, b1 = f.n_items_b, slot = 1;
  if (phase == kSweepBwdRoot) b1 = f.n_items_b_root;
  if (phase == kSweepBwdRest) b0 = f.n_items_b_root, slot = 2;
  ProfScope ps(h->prof, s, tag + " bwd");
  SweepDev pb = p;
  pb.l2_policy = f.l2_policy_b;
  if (b1 > b0) {
    auto kern = few ? k_sweep_bwd_few : k_sweep_bwd;
    const int g = std::min(b1 - b0, sweep_grid((const void*)kern, shm));
    kern<<<g, kBlockSweep, shm, s>>>(pb, f.items_b.p + b0, b1 - b0, f.panel.p, X, ysave, skip, slot);
    CB_LAUNCH();
  }
  if (tp && phase == kSweepBwd) dump_trace(std::string(tp) + "_" + tag + "_bwd.bin", f, false, s);
}

// Forward sweep of kSweepMultiRhs right-hand sides X[rhs][nsd*T] (the
// columns' y to ysave[rhs][nsd*T], updates in upd[rhs][upd_total], tile
// partials in vbuf8[rhs][f.vbuf.n]).
void sweep_forward_multi(cutbddc_gpu* h, const TplSet& ts, const FactorSet& f, const double* X, double* ysave,
                         double* upd, double* vbuf8) {
  static_assert(kMultiRhs == kSweepMultiRhs, "multi-RHS width");
  if (!f.items_ready) throw Failure(CUTBDDC_INTERNAL, "sweep: item lists not built");
  cudaStream_t s = h->stream;
  const int nsd = h->nsd, nsn = (int)ts.tpl.sn.size();
  SweepDev p = sweep_dev(f, nsd, nsn, nullptr);
  p.vbuf = vbuf8;
  p.vec = (std::max(f.sweep_vec, kMultiRhs * std::max(f.fwd_cols, kSmallRows)) + 63) & ~63;
#ifdef CUTBDDC_MULTI_SLOT
  p.slot = CUTBDDC_MULTI_SLOT;  // the ring geometry is per launch
#endif
  const size_t shm = sweep_shm_bytes(p.slot, p.vec);
  sweep_phase(h, ts, f, nullptr, nullptr, nullptr, nullptr, kSweepAttrOnly);
  CB_CUDA(cudaMemsetAsync(f.counters.p, 0, sizeof(int32_t) * f.counters.n, s));
  if (f.n_items_f == 0) return;
  const RhsStride rs{(int64_t)nsd * h->slots, f.upd_total, (int64_t)f.vbuf.n};
  const int g = std::min(f.n_items_f, sweep_grid((const void*)k_sweep_fwd_multi, shm));
  k_sweep_fwd_multi<<<g, kBlockSweep, shm, s>>>(p, f.items_f.p, f.n_items_f, f.panel.p, X, ysave, upd, rs);
  CB_LAUNCH();
}

void sweep_solve(cutbddc_gpu* h, const TplSet& ts, const FactorSet& f, double* X, double* ysave, double* upd,
                 const int* skip) {
  sweep_phase(h, ts, f, X, ysave, upd, skip, kSweepFwd);
  sweep_phase(h, ts, f, X, ysave, upd, skip, kSweepBwd);
}

}  // namespace cutbddc_b200
