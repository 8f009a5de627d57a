// front_desc.cuh — per (subdomain, front) descriptor of one factorisation,
// built with the sweep plan (sweep.cu) and shared by the numeric
// factorisation's extend-add gathers (factor.cu).
#pragma once

namespace cutbddc_b200 {

// Everything one (subdomain, front) needs, in one 96-byte record.
struct __align__(16) FrontDesc {
  int r, c, nch, pfs;      // rows, columns, children, parent front (backward dependency) or -1
  long long vo, po;        // compact front vector / panel offsets
  long long uo, cuo0;      // own update offset, child 0 update offset
  long long cuo1;          // child 1 update offset
  long long tpo;           // forward tile partials of a chunked front (in vbuf)
  int cfs0, cfs1;          // child fronts (sd * nsn + sid)
  int cnu0, cnu1;          // child update lengths
  int cnf0, cnf1;          // child forward completion counts
  int pnb, rbo;            // parent backward completion count; row-block counters of a chunked front
};
static_assert(sizeof(FrontDesc) == 96, "FrontDesc is six int4");

}  // namespace cutbddc_b200
