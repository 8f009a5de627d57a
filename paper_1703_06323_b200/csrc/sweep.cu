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

#include "factor.cuh"
#include "front_desc.cuh"
#include "prof.cuh"

namespace cutbddc_b200 {
namespace {

constexpr int kSmallRows = 256;  // S items and subtree fronts
#ifndef CUTBDDC_SWEEP_SMALL_WORK
#define CUTBDDC_SWEEP_SMALL_WORK 4096
#endif
#ifndef CUTBDDC_SWEEP_FWD_ROWS
#define CUTBDDC_SWEEP_FWD_ROWS 128
#endif
#ifndef CUTBDDC_SWEEP_FWD_COLS
#define CUTBDDC_SWEEP_FWD_COLS 64
#endif
#ifndef CUTBDDC_SWEEP_BWD_COLS
#define CUTBDDC_SWEEP_BWD_COLS 16
#endif
#ifndef CUTBDDC_SWEEP_SUB_LEVELS
#define CUTBDDC_SWEEP_SUB_LEVELS 3
#endif
#ifndef CUTBDDC_SWEEP_MIN_BLOCKS
#define CUTBDDC_SWEEP_MIN_BLOCKS 4
#endif
// (the CUTBDDC_SWEEP_* macros exist for tools/tune_sweep.sh; the defaults are the measured best)
constexpr int kSmallWork = CUTBDDC_SWEEP_SMALL_WORK; // S items: at most this many panel entries (r x c), else A + C tiles
constexpr int kFwdRows = CUTBDDC_SWEEP_FWD_ROWS;    // C items forward: 128 x 128 tiles (four rows per lane)
constexpr int kFwdCols = CUTBDDC_SWEEP_FWD_COLS;
constexpr int kBwdCols = CUTBDDC_SWEEP_BWD_COLS;     // C items backward: columns per CTA (two per warp)
constexpr int kSubLevels = CUTBDDC_SWEEP_SUB_LEVELS;    // T items: the bottom levels of the elimination tree
constexpr int kThreadsSweep = 256;
constexpr int kWarps = kThreadsSweep / 32;
constexpr int kMinBlocks = CUTBDDC_SWEEP_MIN_BLOCKS;  // resident CTAs per SM (items in flight): <= 64 registers
constexpr int kVecDoubles = 2048;                   // front vector: >= every template front
constexpr int kPartDoubles = kWarps * kSmallRows;   // per-warp row partials of the forward GEMV
constexpr int kShmDoubles = kVecDoubles + kPartDoubles;
enum { kItemS = 0, kItemA = 1, kItemC = 2, kItemT = 3 };

// one CTA per front (S) or gather + tiles (A/C): wide fronts need the tiles'
// parallelism (one CTA would issue r c / 256 dependent loads per thread)
inline bool is_small(int2 rc) { return rc.x <= kSmallRows && (int64_t)rc.x * rc.y <= kSmallWork; }


struct SweepDev {
  const FrontDesc* desc;
  const int32_t* cslot;  // sd * T + slot of every compact front row
  const int32_t* umap;   // parent compact row of every update entry
  const int32_t* gmap;   // per compact front row: upd index of child 0 / child 1 entry landing there, or -1
  const int32_t* sub_sids;
  const int32_t* sub_meta;
  int nsn;
  int32_t* done_f;
  int32_t* ready_f;
  int32_t* done_b;
  int32_t* ready_b;
  int32_t* ticket;  // [0] forward, [1] backward (all, or the root phase), [2] backward below the root
  int32_t* rbcnt;   // forward tile arrivals per (chunked front, row block)
  double* vbuf;
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

struct TraceState {
  int it;
  unsigned long long t0, t1;
};
__shared__ TraceState s_trace;

__device__ __forceinline__ int ld_acquire(const int32_t* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// thread 0 waits until *p >= target; the whole CTA then proceeds
__device__ __forceinline__ void cta_wait(const SweepDev& sp, const int32_t* p, int target) {
  if (threadIdx.x == 0) {
    while (ld_acquire(p) < target) __nanosleep(32);
    __threadfence();
    if (sp.trace) s_trace.t1 = gtimer();
  }
  __syncthreads();
}

// all of the CTA's global writes are published before *p is incremented
__device__ __forceinline__ void cta_signal(int32_t* p) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(p, 1);
  }
}

__device__ __forceinline__ int next_item(const SweepDev& sp, int32_t* ticket, bool first) {
  __shared__ int s_item;
  __syncthreads();  // previous item finished with shared memory
  if (threadIdx.x == 0) {
    if (sp.trace) {
      const unsigned long long now = gtimer();
      if (!first) {
        unsigned long long* tr = sp.trace + 4ll * s_trace.it;
        tr[0] = s_trace.t0;
        tr[1] = s_trace.t1;
        tr[2] = now;
        tr[3] = smid();
      }
      s_trace.t0 = s_trace.t1 = now;
    }
    s_item = atomicAdd(ticket, 1);
    if (sp.trace) s_trace.it = s_item;
  }
  __syncthreads();
  return s_item;
}

__device__ __forceinline__ FrontDesc load_desc(const FrontDesc* p) {
  FrontDesc d;
  const int4* s = reinterpret_cast<const int4*>(p);
  int4* o = reinterpret_cast<int4*>(&d);
#pragma unroll
  for (int k = 0; k < 6; ++k) o[k] = s[k];
  return d;
}

// acc[k] (k < 16) summed over the warp; lane L returns the total of
// acc[L & 15]. A butterfly over lane bit 4, then recursive halving: 31
// shuffles in a fixed order (deterministic).
__device__ __forceinline__ double reduce_scatter16(double (&acc)[16], int lane) {
#pragma unroll
  for (int k = 0; k < 16; ++k) acc[k] += __shfl_xor_sync(0xffffffffu, acc[k], 16);
#pragma unroll
  for (int off = 8; off >= 1; off >>= 1) {
    const bool up = (lane & off) != 0;
#pragma unroll
    for (int k = 0; k < off; ++k) {
      const double send = up ? acc[k] : acc[k + off];
      const double keep = up ? acc[k + off] : acc[k];
      acc[k] = keep + __shfl_xor_sync(0xffffffffu, send, off);
    }
  }
  return acc[0];
}

// The children's update entries landing on compact row q of a front
// (gmap: child 0, child 1 indices into upd, -1 if none), added in child
// order to b (or 0 at the update rows). `cross`: produced by other CTAs.
__device__ __forceinline__ double child_sum(const SweepDev& p, const FrontDesc& d, const double* upd, int q, double v,
                                            bool cross) {
  const int2 g = reinterpret_cast<const int2*>(p.gmap)[d.vo + q];
  if (g.x >= 0) v += cross ? __ldcg(upd + g.x) : upd[g.x];
  if (g.y >= 0) v += cross ? __ldcg(upd + g.y) : upd[g.y];
  return v;
}

// child_sum with the gmap entry already loaded (static: loaded before the
// dependency wait, so only the update loads remain after it)
__device__ __forceinline__ double child_sum_g(int2 g, const double* upd, double v, bool cross) {
  if (g.x >= 0) v += cross ? __ldcg(upd + g.x) : upd[g.x];
  if (g.y >= 0) v += cross ? __ldcg(upd + g.y) : upd[g.y];
  return v;
}
__device__ __forceinline__ int2 gmap_at(const SweepDev& p, const FrontDesc& d, int q) {
  return reinterpret_cast<const int2*>(p.gmap)[d.vo + q];
}

__device__ __forceinline__ void wait_children(const SweepDev& p, const FrontDesc& d) {
  if (d.nch > 0) cta_wait(p, p.done_f + d.cfs0, d.cnf0);
  if (d.nch > 1) cta_wait(p, p.done_f + d.cfs1, d.cnf1);
}

// HBM -> L2 prefetch of panel data an item is about to stream, issued before
// its dependency wait (no registers or shared memory held): the GEMV after
// the wait then reads L2. Rows [i0, i1) of columns [j0, j1) of a column-major
// panel with leading dimension r, one 128-B line per request, never past a
// column's end.
__device__ __forceinline__ void prefetch_l2(const double* a) { asm volatile("prefetch.global.L2 [%0];" ::"l"(a)); }
__device__ __forceinline__ void prefetch_panel(const double* G, int r, int i0, int i1, int j0, int j1, int tid, int nt) {
  const int seg = i1 - i0;
  if (seg <= 0 || j1 <= j0) return;
  if (seg == r) {  // whole columns: one contiguous range
    const int64_t n = (int64_t)(j1 - j0) * r;
    const double* b = G + (int64_t)j0 * r;
    for (int64_t e = (int64_t)tid * 16; e < n + 15; e += (int64_t)nt * 16) prefetch_l2(b + min(e, n - 1));
    return;
  }
  const int lpc = (seg + 15) / 16 + 1;  // lines per column segment (unaligned start)
  for (int t = tid; t < (j1 - j0) * lpc; t += nt) {
    const int j = j0 + t / lpc, l = t % lpc;
    prefetch_l2(G + (int64_t)j * r + i0 + min(16 * l, seg - 1));
  }
}

// nw consecutive warps w0 .. w0 + nw - 1 of the CTA working on one front;
// named barrier `bar` (the whole CTA: __syncthreads). T items run the
// independent fronts of one subtree level side by side, one group each.
struct Grp {
  int w0, nw, bar;
  __device__ __forceinline__ int lt() const { return (int)threadIdx.x - 32 * w0; }
  __device__ __forceinline__ int nt() const { return 32 * nw; }
  __device__ __forceinline__ void sync() const {
    if (nw == kWarps)
      __syncthreads();
    else if (nw == 1)
      __syncwarp();
    else
      asm volatile("bar.sync %0, %1;" ::"r"(bar), "r"(32 * nw) : "memory");
  }
};
__device__ __forceinline__ Grp whole_cta() { return Grp{0, kWarps, 0}; }

// Forward GEMV o[i] = sum_j G[i + j r] v[j] for rows [i0, i1) (at most 32 R)
// and columns [jlo, jhi): the group's warps split the columns, each lane
// accumulates its R rows in registers (coalesced 256-B column segments, R
// loads in flight per column), the warp partials are summed in warp order
// (deterministic). Row blocks entirely above column j are skipped (zero part
// of L11^{-1}). The first column of every warp is loaded before `between()`
// (which completes v: dependency wait + children's updates).
template <int R, int U, typename Between, typename Out>
__device__ __forceinline__ void grp_gemv_fwd(const Grp& g, const double* __restrict__ G, int r, int jlo, int jhi, int i0,
                                             int i1, double* v, double* part, Between between, Out out) {
  const int lt = g.lt(), lane = threadIdx.x & 31, lw = lt >> 5;
  const int cw = (jhi - jlo + g.nw - 1) / g.nw;
  const int ja = min(jhi, jlo + lw * cw), jb = min(jhi, ja + cw);
  const double* gl = G + i0 + lane;
  double acc[R];
#pragma unroll
  for (int k = 0; k < R; ++k) {
    const bool row = i0 + 32 * k + lane < i1;
    acc[k] = (ja < jb && row && i0 + 32 * k + 31 >= ja) ? gl[(int64_t)ja * r + 32 * k] : 0.0;
  }
  between();
  const double v0 = ja < jb ? v[ja] : 0.0;
#pragma unroll
  for (int k = 0; k < R; ++k) acc[k] *= v0;
#pragma unroll U
  for (int j = ja + 1; j < jb; ++j) {
    const double vj = v[j];
    const double* gj = gl + (int64_t)j * r;
#pragma unroll
    for (int k = 0; k < R; ++k)
      if (i0 + 32 * k + 31 >= j && i0 + 32 * k + lane < i1) acc[k] += gj[32 * k] * vj;
  }
  double* pw = part + (int64_t)g.w0 * 32 * R;
#pragma unroll
  for (int k = 0; k < R; ++k) pw[lw * 32 * R + 32 * k + lane] = acc[k];
  g.sync();
  for (int q = lt; q < i1 - i0; q += g.nt()) {
    double o = 0.0;
    for (int w = 0; w < g.nw; ++w) o += pw[w * 32 * R + q];
    out(i0 + q, o);
  }
  g.sync();
}

// Forward of one front (r <= kSmallRows) by a warp group. `wait` (whole CTA
// only) = the children belong to other items (wait for them, read their
// updates from L2); otherwise they were produced earlier in this CTA.
__device__ void grp_front_fwd(const Grp& g, const SweepDev& p, const FrontDesc& d, const double* __restrict__ panel,
                              const double* __restrict__ X, double* ysave, double* upd, double* v, double* part,
                              bool wait) {
  const int r = d.r, c = d.c;
  if (r == 0) return;
  const int lt = g.lt(), nt = g.nt();
  const int32_t* cs = p.cslot + d.vo;
  for (int q = lt; q < r; q += nt) v[q] = q < c ? X[cs[q]] : 0.0;
  const int2 g0 = lt < r ? gmap_at(p, d, lt) : make_int2(-1, -1);
  double* uo = upd + d.uo;
  grp_gemv_fwd<kSmallRows / 32, 2>(
      g, panel + d.po, r, 0, c, 0, r, v, part,
      [&] {
        if (wait) wait_children(p, d);
        g.sync();
        if (lt < r) v[lt] = child_sum_g(g0, upd, v[lt], wait);
        for (int q = lt + nt; q < r; q += nt) v[q] = child_sum(p, d, upd, q, v[q], wait);
        g.sync();
      },
      [&](int i, double o) {
        if (i < c)
          ysave[cs[i]] = o;
        else
          uo[i - c] = v[i] - o;
      });
}

// Backward of one front (r <= kSmallRows) by a warp group: rows split over
// the warps, 16 columns at a time accumulated in registers, reduce-scattered
// in each warp and the warp partials summed in order. The first row of each
// lane (first column block) and y at the columns are loaded before the wait
// (whole CTA only).
__device__ void grp_front_bwd(const Grp& g, const SweepDev& p, const FrontDesc& d, const double* __restrict__ panel,
                              double* X, const double* __restrict__ ysave, double* w, double (*part)[33], bool wait) {
  const int r = d.r, c = d.c;
  const int lt = g.lt(), nt = g.nt(), lane = threadIdx.x & 31, lw = lt >> 5;
  if (c == 0) {
    if (wait && d.pfs >= 0) cta_wait(p, p.done_b + d.pfs, d.pnb);
    return;
  }
  const int32_t* cs = p.cslot + d.vo;
  for (int q = lt; q < c; q += nt) w[q] = ysave[cs[q]];
  const double* G = panel + d.po;
  const int rw = (r + g.nw - 1) / g.nw;
  const int ra = lw * rw, rb = min(r, ra + rw);
  const int i_first = ra + lane;
  double acc[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) acc[k] = (i_first < rb && k < c) ? G[i_first + (int64_t)k * r] : 0.0;
  const int s0 = c + lt < r ? cs[c + lt] : 0;  // slot of the first update row (static: before the wait)
  if (wait && d.pfs >= 0) cta_wait(p, p.done_b + d.pfs, d.pnb);
  if (c + lt < r) w[c + lt] = -__ldcg(X + s0);
  for (int q = c + lt + nt; q < r; q += nt) w[q] = -__ldcg(X + cs[q]);
  g.sync();
  for (int jb = 0; jb < c; jb += 16) {
    int i = max(ra, jb) + lane;
    if (jb == 0) {
      const double wi = i_first < rb ? w[i_first] : 0.0;
#pragma unroll
      for (int k = 0; k < 16; ++k) acc[k] *= wi;
      i = i_first + 32;
    } else {
#pragma unroll
      for (int k = 0; k < 16; ++k) acc[k] = 0.0;
    }
    for (; i < rb; i += 32) {
      const double wi = w[i];
      const double* gi = G + i + (int64_t)jb * r;
#pragma unroll
      for (int k = 0; k < 16; ++k)
        if (jb + k < c) acc[k] += gi[(int64_t)k * r] * wi;
    }
    part[g.w0 + lw][lane] = reduce_scatter16(acc, lane);
    g.sync();
    if (lw == 0 && lane < 16 && jb + lane < c) {
      double x = 0.0;
      for (int q = 0; q < g.nw; ++q) x += part[g.w0 + q][lane];
      X[cs[jb + lane]] = x;
    }
    g.sync();
  }
}

// One level of a T item: its nf independent fronts (sids[k0 .. k0 + nf))
// side by side, kWarps / 2^ceil(log2 nf) warps each (rounds of kWarps
// fronts), each with its own kSmallRows slice of the vector buffer.
template <typename Fn>
__device__ __forceinline__ void subtree_level(int k0, int k1, Fn fn) {
  const int wid = threadIdx.x >> 5;
  for (int base = k0; base < k1; base += kWarps) {
    const int n = min(kWarps, k1 - base);
    int wpf = kWarps;
    while (wpf > 1 && wpf * n > kWarps) wpf >>= 1;
    const int f = wid / wpf;
    if (f < n) fn(Grp{f * wpf, wpf, 1 + f}, base + f, f);
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kThreadsSweep, kMinBlocks) k_sweep_fwd(SweepDev p, const int4* __restrict__ items, int n_items,
                                                             const double* __restrict__ panel,
                                                             const double* __restrict__ X, double* __restrict__ ysave,
                                                             double* upd, const int* __restrict__ skip) {
  if (skip && *skip) return;
  extern __shared__ double v[];
  const int tid = threadIdx.x;
  for (bool first = true;; first = false) {
    const int it = next_item(p, p.ticket, first);
    if (it >= n_items) return;
    const int4 w = items[it];
    const int kind = w.x, sid = w.y, sd = w.z, chunk = w.w;
    const int64_t fs = (int64_t)sd * p.nsn + sid;
    if (kind == kItemT) {
      // bottom subtree of sid: its fronts deepest level first, one after another
      const int32_t* meta = p.sub_meta + chunk;
      const int ng = meta[0];
      for (int k = meta[1]; k < meta[1 + ng]; ++k) {
        const FrontDesc d = load_desc(p.desc + (int64_t)sd * p.nsn + p.sub_sids[k]);
        prefetch_panel(panel + d.po, d.r, 0, d.r, 0, d.c, tid, kThreadsSweep);
      }
      for (int gi = 0; gi < ng; ++gi)  // deepest level first
        subtree_level(meta[1 + gi], meta[2 + gi], [&](const Grp& g, int k, int f) {
          const FrontDesc d = load_desc(p.desc + (int64_t)sd * p.nsn + p.sub_sids[k]);
          grp_front_fwd(g, p, d, panel, X, ysave, upd, v + f * kSmallRows, v + kVecDoubles, false);
        });
      cta_signal(p.done_f + fs);
      continue;
    }
    const FrontDesc d = load_desc(p.desc + fs);
    if (kind == kItemS) {
      prefetch_panel(panel + d.po, d.r, 0, d.r, 0, d.c, tid, kThreadsSweep);
      grp_front_fwd(whole_cta(), p, d, panel, X, ysave, upd, v, v + kVecDoubles, true);
      cta_signal(p.done_f + fs);
      continue;
    }
    const int r = d.r, c = d.c;
    const int32_t* cs = p.cslot + d.vo;
    // C: tile (row block rb, column block cb) of a chunked front: its own
    // gather of v at the tile's columns, partial row sums to vbuf; the last
    // tile of a row block to arrive sums them in column-block order
    // (deterministic) and writes the rows.
    const int mcb = max(1, (c + kFwdCols - 1) / kFwdCols);
    const int rb = chunk / mcb, cb = chunk % mcb;
    const int i0 = rb * kFwdRows, i1 = min(r, i0 + kFwdRows);
    const int jrow = min(c, i1);
    const int jlo = cb * kFwdCols, jhi = min(jrow, jlo + kFwdCols);
    double* tp = p.vbuf + d.tpo + (int64_t)rb * mcb * kFwdRows;
    prefetch_panel(panel + d.po, r, i0, i1, jlo, jhi, tid, kThreadsSweep);
    static_assert(kFwdCols <= kThreadsSweep && kFwdRows <= kThreadsSweep, "one column / row per thread");
    const int qc = jlo + tid, qr = i0 + tid;  // this thread's column of the tile, row of the row block
    if (qc < jhi) v[qc] = X[cs[qc]];
    const int2 gc = qc < jhi ? gmap_at(p, d, qc) : make_int2(-1, -1);
    const int2 gr = (qr < i1 && qr >= c) ? gmap_at(p, d, qr) : make_int2(-1, -1);
    double cu = 0.0;  // children's updates at update row qr (used by the row block's last tile)
    grp_gemv_fwd<kFwdRows / 32, 4>(
        whole_cta(), panel + d.po, r, jlo, jhi, i0, i1, v, v + kVecDoubles,
        [&] {
          wait_children(p, d);
          __syncthreads();
          if (qc < jhi) v[qc] = child_sum_g(gc, upd, v[qc], true);
          cu = child_sum_g(gr, upd, 0.0, true);
          __syncthreads();
        },
        [&](int i, double o) { tp[(int64_t)cb * kFwdRows + i - i0] = o; });
    __shared__ int s_last;
    if (tid == 0) {
      __threadfence();
      const int ncb = max(1, (jrow + kFwdCols - 1) / kFwdCols);
      s_last = atomicAdd(p.rbcnt + d.rbo + rb, 1) == ncb - 1;
      if (s_last) __threadfence();
    }
    __syncthreads();
    if (!s_last) continue;
    const int ncb = max(1, (jrow + kFwdCols - 1) / kFwdCols);
    double* uo = upd + d.uo;
    if (tid < i1 - i0) {
      const int i = i0 + tid;
      double o = 0.0;
      for (int k = 0; k < ncb; ++k) o += __ldcg(tp + (int64_t)k * kFwdRows + tid);
      if (i < c)
        ysave[cs[i]] = o;
      else
        uo[i - c] = cu - o;
    }
    cta_signal(p.done_f + fs);
  }
}

__global__ void __launch_bounds__(kThreadsSweep, kMinBlocks) k_sweep_bwd(SweepDev p, const int4* __restrict__ items, int n_items,
                                                             const double* __restrict__ panel, double* X,
                                                             const double* __restrict__ ysave,
                                                             const int* __restrict__ skip, int ticket_slot) {
  if (skip && *skip) return;
  extern __shared__ double w[];
  __shared__ double part[kWarps][33];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  for (bool first = true;; first = false) {
    const int it = next_item(p, p.ticket + ticket_slot, first);
    if (it >= n_items) return;
    const int4 iw = items[it];
    const int kind = iw.x, sid = iw.y, sd = iw.z, chunk = iw.w;
    const int64_t fs = (int64_t)sd * p.nsn + sid;
    if (kind == kItemT) {
      // bottom subtree of sid: shallowest level first, one front after another;
      // only its root depends on other items (its parent)
      const int32_t* meta = p.sub_meta + chunk;
      const int ng = meta[0];
      for (int k = meta[1]; k < meta[1 + ng]; ++k) {
        const FrontDesc d = load_desc(p.desc + (int64_t)sd * p.nsn + p.sub_sids[k]);
        prefetch_panel(panel + d.po, d.r, 0, d.r, 0, d.c, tid, kThreadsSweep);
      }
      for (int gi = ng - 1; gi >= 0; --gi)  // shallowest level (the subtree root, one front) first
        subtree_level(meta[1 + gi], meta[2 + gi], [&](const Grp& g, int k, int f) {
          const FrontDesc d = load_desc(p.desc + (int64_t)sd * p.nsn + p.sub_sids[k]);
          grp_front_bwd(g, p, d, panel, X, ysave, w + f * kSmallRows, part, k == meta[1 + ng] - 1);
        });
      continue;  // nothing outside the subtree waits on it
    }
    const FrontDesc d = load_desc(p.desc + fs);
    if (kind == kItemS) {
      prefetch_panel(panel + d.po, d.r, 0, d.r, 0, d.c, tid, kThreadsSweep);
      grp_front_bwd(whole_cta(), p, d, panel, X, ysave, w, part, true);
      cta_signal(p.done_b + fs);
      continue;
    }
    const int r = d.r, c = d.c;
    const int32_t* cs = p.cslot + d.vo;
    // C: columns [j0, j1) of a chunked front, one warp per column; each item
    // gathers [y; -x_rest] itself (rows from j0 on: the columns' G is zero above)
    const double* G = panel + d.po;
    const int j0 = chunk * kBwdCols, j1 = min(c, j0 + kBwdCols);
    prefetch_panel(G, r, j0, r, j0, j1, tid, kThreadsSweep);
    for (int q = j0 + tid; q < c; q += kThreadsSweep) w[q] = ysave[cs[q]];
    int32_t* ci = reinterpret_cast<int32_t*>(w + kVecDoubles);  // update-row slots, staged before the wait
    for (int q = max(c, j0) + tid; q < r; q += kThreadsSweep) ci[q] = cs[q];
    if (d.pfs >= 0) cta_wait(p, p.done_b + d.pfs, d.pnb);  // (its __syncthreads publishes ci)
    if (d.pfs < 0) __syncthreads();
    for (int q = max(c, j0) + tid; q < r; q += kThreadsSweep) w[q] = -__ldcg(X + ci[q]);
    __syncthreads();
    for (int j = j0 + wid; j < j1; j += kWarps) {
      const double* col = G + (int64_t)j * r;
      double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
      int i = j + lane;
      for (; i + 96 < r; i += 128) {
        s0 += col[i] * w[i];
        s1 += col[i + 32] * w[i + 32];
        s2 += col[i + 64] * w[i + 64];
        s3 += col[i + 96] * w[i + 96];
      }
      for (; i < r; i += 32) s0 += col[i] * w[i];
      const double sum = warp_sum((s0 + s1) + (s2 + s3));
      if (lane == 0) X[cs[j]] = sum;
    }
    cta_signal(p.done_b + fs);
  }
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
                  f.sub_sids.p,
                  f.sub_meta.p,
                  nsn,
                  cnt,
                  cnt + n,
                  cnt + 2 * n,
                  cnt + 3 * n,
                  cnt + 4 * n,
                  cnt + 4 * n + 3,
                  const_cast<double*>(f.vbuf.p),
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

int sweep_grid(const void* fn) {
  static int cached[2] = {0, 0};
  const int k = fn == (const void*)k_sweep_fwd ? 0 : 1;
  if (!cached[k]) {
    int per_sm = 0;
    CB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kThreadsSweep, sizeof(double) * kShmDoubles));
    int dev = 0, sms = 0;
    CB_CUDA(cudaGetDevice(&dev));
    CB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    cached[k] = std::max(1, per_sm) * sms;
  }
  return cached[k];
}

}  // namespace

// Host: descriptors, maps, completion counts and the ordered work lists of
// one factorisation (after its symbolic phase; poff / uoff are the panel and
// update offsets per (sd, supernode) the numeric phase uses).
void build_sweep_plan(cutbddc_gpu* h, const TplSet& ts, FactorSet& f, const std::vector<int64_t>& poff,
                      const std::vector<int64_t>& uoff) {
  cudaStream_t s = h->stream;
  const Template& tp = ts.tpl;
  const int nsd = h->nsd, nsn = (int)tp.sn.size();
  const auto& lv = tp.levels;
  const int nlev = (int)lv.size();
  if (tp.max_rows > kVecDoubles) throw Failure(CUTBDDC_CONFIG, "sweep: front larger than the shared vector");
  // subtree level: the shallowest level from which every front is small,
  // and no more than kSubLevels above the deepest level
  int lsub = nlev;
  while (lsub > 0) {
    bool small = true;
    for (int sid : lv[(size_t)lsub - 1]) small &= tp.sn[(size_t)sid].nrows <= kSmallRows;
    if (!small) break;
    --lsub;
  }
  lsub = std::max(lsub, nlev - kSubLevels);
  if (lsub == 0 && nlev > 1) lsub = 1;  // keep the root as its own item
  // template subtrees: descendants of each level-lsub root grouped by level
  std::vector<int32_t> sids, meta;
  std::vector<int> meta_of((size_t)nsn, -1);
  std::vector<uint8_t> in_sub((size_t)nsn, 0);
  if (lsub < nlev) {
    for (int root : lv[(size_t)lsub]) {
      std::vector<std::vector<int>> by((size_t)(nlev - lsub));
      std::vector<int> stack{root};
      while (!stack.empty()) {
        const int x = stack.back();
        stack.pop_back();
        in_sub[(size_t)x] = 1;
        by[(size_t)(tp.sn[(size_t)x].level - lsub)].push_back(x);
        for (int ch = 0; ch < tp.sn[(size_t)x].nchild; ++ch) stack.push_back(tp.sn[(size_t)x].child[ch]);
      }
      meta_of[(size_t)root] = (int)meta.size();
      int ng = 0;
      for (auto& g : by) ng += !g.empty();
      meta.push_back(ng);
      for (int g = (int)by.size() - 1; g >= 0; --g) {  // deepest first
        if (by[(size_t)g].empty()) continue;
        meta.push_back((int)sids.size());
        sids.insert(sids.end(), by[(size_t)g].begin(), by[(size_t)g].end());
      }
      meta.push_back((int)sids.size());
    }
  }
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
      if (in_sub[(size_t)q]) {
        nf[i] = meta_of[(size_t)q] >= 0 ? 1 : 0;
        continue;
      }
      const bool small = is_small(v);
      nf[i] = v.x == 0 ? 0 : small ? 1 : (v.x + kFwdRows - 1) / kFwdRows;
      nb[i] = v.x == 0 ? 0 : (small || v.y == 0) ? 1 : (v.y + kBwdCols - 1) / kBwdCols;
    }
  f.vec_total = tot;
  f.h_vec_off = voff;
  // forward tiles of chunked fronts: partial storage (after the front
  // vectors in vbuf) and one arrival counter per row block
  auto mcb_of = [](int c) { return std::max(1, (c + kFwdCols - 1) / kFwdCols); };
  auto ncb_of = [](int r, int c, int rb) {
    return std::max(1, (std::min(c, std::min(r, (rb + 1) * kFwdRows)) + kFwdCols - 1) / kFwdCols);
  };
  std::vector<int64_t> tpo((size_t)nsd * nsn, 0);
  std::vector<int32_t> rbo((size_t)nsd * nsn, 0);
  int64_t ptot = tot;
  int32_t nrb_tot = 0;
  for (size_t i = 0; i < (size_t)nsd * nsn; ++i) {
    const int2 v = f.h_rc[i];
    if (in_sub[i % (size_t)nsn] || is_small(v)) continue;
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
  std::vector<int4> fw, bw;
  auto front_items = [&](int L, bool fwd, std::vector<int4>& out) {
    for (int sid : lv[(size_t)L])
      for (int sd = 0; sd < nsd; ++sd) {
        const int2 v = f.h_rc[(size_t)sd * nsn + sid];
        if (v.x > 0 && (is_small(v) || (!fwd && v.y == 0))) out.push_back(make_int4(kItemS, sid, sd, 0));
      }
    for (int sid : lv[(size_t)L])
      for (int sd = 0; sd < nsd; ++sd) {
        const size_t i = (size_t)sd * nsn + sid;
        const int2 v = f.h_rc[i];
        if (is_small(v)) continue;
        if (fwd) {
          const int mcb = mcb_of(v.y);
          for (int rb = 0; rb < nf[i]; ++rb)
            for (int cb = 0; cb < ncb_of(v.x, v.y, rb); ++cb) out.push_back(make_int4(kItemC, sid, sd, rb * mcb + cb));
        } else if (v.y > 0) {
          for (int k = 0; k < nb[i]; ++k) out.push_back(make_int4(kItemC, sid, sd, k));
        }
      }
  };
  auto subtree_items = [&](std::vector<int4>& out) {
    if (lsub >= nlev) return;
    for (int root : lv[(size_t)lsub])
      for (int sd = 0; sd < nsd; ++sd) out.push_back(make_int4(kItemT, root, sd, meta_of[(size_t)root]));
  };
  subtree_items(fw);
  for (int L = lsub - 1; L >= 0; --L) front_items(L, true, fw);  // leaves first
  for (int L = 0; L < lsub; ++L) {  // root first
    front_items(L, false, bw);
    if (L == 0) f.n_items_b_root = (int)bw.size();
  }
  subtree_items(bw);
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
    auto t_work = [&](int sd, int root) {  // a T item: every front of the subtree, one CTA
      double w = 0.0;
      const int32_t* m = meta.data() + meta_of[(size_t)root];
      for (int k = m[1]; k < m[1 + m[0]]; ++k) w += kItemCost + entries(rc(sd, sids[(size_t)k]));
      return w;
    };
    auto fwd_item = [&](int sd, int sid) {  // work of one item of a non-subtree front
      const int2 v = rc(sd, sid);
      return kItemCost + (is_small(v) ? entries(v) : (double)std::min(v.x, kFwdRows) * std::min(v.y, kFwdCols));
    };
    auto bwd_item = [&](int sd, int sid) {
      const int2 v = rc(sd, sid);
      return kItemCost + (is_small(v) || v.y == 0 ? entries(v) : (double)v.x * std::min(v.y, kBwdCols));
    };
    // forward: remaining path from a front to the root (top-down over levels)
    std::vector<double> remf(nf_all, 0.0), remb(nf_all, 0.0);
    for (int L = 0; L < nlev; ++L)
      for (int sid : lv[(size_t)L])
        for (int sd = 0; sd < nsd; ++sd) {
          const int par = tp.sn[(size_t)sid].parent;
          const double up = par >= 0 ? remf[(size_t)sd * nsn + par] : 0.0;
          remf[(size_t)sd * nsn + sid] = up + (in_sub[(size_t)sid] ? 0.0 : fwd_item(sd, sid));
        }
    // backward: remaining path from a front down to its deepest descendant
    for (int L = nlev - 1; L >= 0; --L)
      for (int sid : lv[(size_t)L])
        for (int sd = 0; sd < nsd; ++sd) {
          const Supernode& sn = tp.sn[(size_t)sid];
          double down = 0.0;
          for (int ch = 0; ch < sn.nchild; ++ch) down = std::max(down, remb[(size_t)sd * nsn + sn.child[ch]]);
          remb[(size_t)sd * nsn + sid] =
              down + (in_sub[(size_t)sid] ? (meta_of[(size_t)sid] >= 0 ? t_work(sd, sid) : 0.0) : bwd_item(sd, sid));
        }
    auto key = [&](const int4& it, bool fwd) {
      const size_t i = (size_t)it.z * nsn + it.y;
      if (fwd) {
        if (it.x == kItemT) {
          const int par = tp.sn[(size_t)it.y].parent;
          return t_work(it.z, it.y) + (par >= 0 ? remf[(size_t)it.z * nsn + par] : 0.0);
        }
        return remf[i];
      }
      return remb[i];
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
  f.n_items_f = (int)fw.size();
  f.n_items_b = (int)bw.size();
  if (fw.empty()) fw.push_back(make_int4(0, 0, 0, 0));
  if (bw.empty()) bw.push_back(make_int4(0, 0, 0, 0));
  if (sids.empty()) sids.push_back(0);
  if (meta.empty()) meta.push_back(0);
  f.desc.upload(reinterpret_cast<const int4*>(desc.data()), desc.size() * 6, s);
  f.items_f.upload(fw, s);
  f.items_b.upload(bw, s);
  f.sub_sids.upload(sids, s);
  f.sub_meta.upload(meta, s);
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
  CB_CUDA(cudaStreamSynchronize(s));  // the host vectors above are pageable and go out of scope
}

// In-place solve of one right-hand side X (nsd x T slot vector) in phases:
// kSweepFwd resets the counters and runs the forward sweep; kSweepBwd the
// whole backward sweep; kSweepBwdRoot / kSweepBwdRest split it after the
// root level (the BDDC apply corrects the root solution in between).
void sweep_phase(cutbddc_gpu* h, const TplSet& ts, const FactorSet& f, double* X, double* ysave, double* upd,
                 const int* skip, int phase) {
  cudaStream_t s = h->stream;
  const int nsd = h->nsd, nsn = (int)ts.tpl.sn.size();
  const char* tp = trace_prefix();
  FactorSet& fm = const_cast<FactorSet&>(f);
  if (tp) fm.trace.alloc((size_t)4 * std::max(f.n_items_f, f.n_items_b) + 4);
  const SweepDev p = sweep_dev(f, nsd, nsn, tp ? fm.trace.p : nullptr);
  const size_t shm = sizeof(double) * kShmDoubles;
  static bool attr = false;
  if (!attr) {
    CB_CUDA(cudaFuncSetAttribute(k_sweep_fwd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm));
    CB_CUDA(cudaFuncSetAttribute(k_sweep_bwd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm));
    attr = true;
  }
  const std::string tag = std::string("sweep") + (&ts == &h->tI ? "I" : "K");
  if (phase == kSweepFwd) {
    CB_CUDA(cudaMemsetAsync(f.counters.p, 0, sizeof(int32_t) * f.counters.n, s));
    ProfScope ps(h->prof, s, tag + " fwd");
    if (f.n_items_f > 0) {
      const int g = std::min(f.n_items_f, sweep_grid((const void*)k_sweep_fwd));
      k_sweep_fwd<<<g, kThreadsSweep, shm, s>>>(p, f.items_f.p, f.n_items_f, f.panel.p, X, ysave, upd, skip);
      CB_LAUNCH();
    }
    if (tp) dump_trace(std::string(tp) + "_" + tag + "_fwd.bin", f, true, s);
    return;
  }
  int b0 = 0, b1 = f.n_items_b, slot = 1;
  if (phase == kSweepBwdRoot) b1 = f.n_items_b_root;
  if (phase == kSweepBwdRest) b0 = f.n_items_b_root, slot = 2;
  ProfScope ps(h->prof, s, tag + " bwd");
  if (b1 > b0) {
    const int g = std::min(b1 - b0, sweep_grid((const void*)k_sweep_bwd));
    k_sweep_bwd<<<g, kThreadsSweep, shm, s>>>(p, f.items_b.p + b0, b1 - b0, f.panel.p, X, ysave, skip, slot);
    CB_LAUNCH();
  }
  if (tp && phase == kSweepBwd) dump_trace(std::string(tp) + "_" + tag + "_bwd.bin", f, false, s);
}

void sweep_solve(cutbddc_gpu* h, const TplSet& ts, const FactorSet& f, double* X, double* ysave, double* upd,
                 const int* skip) {
  sweep_phase(h, ts, f, X, ysave, upd, skip, kSweepFwd);
  sweep_phase(h, ts, f, X, ysave, upd, skip, kSweepBwd);
}

}  // namespace cutbddc_b200
