// factor.cuh — interfaces of the batched multifrontal factorisation/solves.
#pragma once

#include "handle.cuh"

namespace cutbddc_b200 {

struct TplDev {
  const Supernode* sn;
  const int32_t* rows;
  const AmapEntry* amap;
  const int32_t* emap;
  const int32_t* root_pos;
  int T;
  int root;  // id of the root supernode (last in postorder)
  int64_t panel_total, front_total, upd_total;
};

// Matrix fed to the factorisation: A^w stencil restricted to `mask` slots
// (identity rows elsewhere), plus diag_add on the diagonal (may be null) and,
// on the root front, rho_w c c^T for every non-corner constraint row c
// (K = A + rho C^T C; the root of the shell template holds every object node).
struct FactorInput {
  const double* As;
  const uint8_t* mask;
  const double* diag_add;
  int T, b1;
  // dense penalty rows (null for the interior problem)
  const int64_t* m_off;
  const int64_t* c_ptr;
  const int32_t* c_slot;
  const double* c_val;
  const uint8_t* corner;
  const double* rho;
};

TplDev tpl_dev(const TplSet& t, int slots);
void upload_template(cutbddc_gpu* h, TplSet& t, bool shell_root);
void factor_device(cutbddc_gpu* h, const TplSet& t, const FactorInput& in, DevBuf<double>& G, const char* what);
void solve_device(cutbddc_gpu* h, const TplSet& t, const DevBuf<double>& G, double* X, int nrhs, double* upd,
                  const int* skip);

}  // namespace cutbddc_b200
