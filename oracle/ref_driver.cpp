// ref_driver.cpp — C entry point over the REFERENCE's own classification code
// (TEST INFRASTRUCTURE). Links /root/reference/proj/src/core/{common,levelset,
// mesh}.cpp, compiled unmodified against oracle/ref_shim, into oracle/_ref.
// Used only to generate/verify the golden fixtures in tests/golden/.
#include <cstdint>
#include <cstring>
#include <map>
#include <string>

#include "core/levelset.hpp"
#include "core/mesh.hpp"

extern "C" int ref_classify(const int* cells, const double* lo, const double* hi, const double* center, double radius,
                            double* phi, unsigned char* cls, int* dof_of_node, long long* n_dof) {
  using namespace cutbddc;
  try {
    std::map<std::string, double> p{{"radius", radius}, {"center_x", center[0]}, {"center_y", center[1]},
                                    {"center_z", center[2]}};
    LevelSet ls = GeometryCatalog::make("sphere", 3, p);
    MeshParams mp;
    mp.dim = 3;
    mp.box_lo = Vec3(lo[0], lo[1], lo[2]);
    mp.box_hi = Vec3(hi[0], hi[1], hi[2]);
    mp.cells = {cells[0], cells[1], cells[2]};
    BackgroundMesh m = BackgroundMesh::classify(mp, ls);
    const std::int64_t nn = m.n_nodes_total(), nc = m.n_cells_total();
    for (std::int64_t i = 0; i < nn; ++i) {
      phi[i] = m.phi_node(i);
      dof_of_node[i] = m.node_dof(i);
    }
    for (std::int64_t c = 0; c < nc; ++c) cls[c] = (unsigned char)m.cell_class(c);
    *n_dof = m.n_dofs();
    return 0;
  } catch (const std::exception& e) {
    return 1;
  }
}
