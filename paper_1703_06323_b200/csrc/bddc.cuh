// bddc.cuh — BDDC setup / apply entry points (bddc.cu) and the pipeline
// stages defined in geometry.cu, assembly.cu and pcg.cu.
#pragma once

#include "handle.cuh"

namespace cutbddc_b200 {

void classify_device(cutbddc_gpu* h, const cutbddc_geometry* g);
void node_of_dof_device(cutbddc_gpu* h);  // geometry.cu: node_of_dof from an uploaded dof_of_node
void assemble_device(cutbddc_gpu* h, const cutbddc_partition_view* part);
cutbddc_objects* classify_objects_device(cutbddc_gpu* h, int objects, int variant);
void setup_bddc_device(cutbddc_gpu* h, const cutbddc_coarse_view* cv, int weighting);
// rz_part: when not null, per-subdomain partials of r.z (gathered layout, dist.cuh)
void apply_bddc_device(cutbddc_gpu* h, const double* r, double* z, const int* skip, double* rz_part = nullptr);
void spmv_device(cutbddc_gpu* h, const double* x, double* y);
// squared error norms of the manufactured solution over this rank's cells (element.cu)
void error_norms_device(cutbddc_gpu* h, const double* xloc, double* l2sq, double* h1sq);
// b_loc, h->px: local dof vectors (dist.cuh)
void pcg_device(cutbddc_gpu* h, const double* b_loc, double rtol, int max_iter, cutbddc_solve_report* rep);

}  // namespace cutbddc_b200
