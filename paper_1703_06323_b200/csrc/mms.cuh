// mms.cuh — the manufactured problem (§5.1):
// u = sin(5 pi |x|), f = -lap u = 25 pi^2 sin(5 pi r) - 10 pi cos(5 pi r) / r,
// g^D = u on the embedded boundary (Nitsche load terms), grad u = 5 pi
// cos(5 pi r) x / r. The same operation order as the CPU restatement
// (oracle.hpp Manufactured); the device sin/cos may differ from the host's
// by an ulp, so parity with the oracle is to 1e-13, not bitwise.
#pragma once

#include <cmath>

namespace cutbddc_b200 {

enum { kProblemUnitLoad = 0, kProblemManufactured = 1 };

__host__ __device__ inline double mms_r(double x, double y, double z) { return sqrt((x * x + y * y) + z * z); }
__host__ __device__ inline double mms_u(double x, double y, double z) { return sin(5.0 * M_PI * mms_r(x, y, z)); }
__host__ __device__ inline double mms_f(double x, double y, double z) {
  const double r = mms_r(x, y, z);
  return 25.0 * M_PI * M_PI * sin(5.0 * M_PI * r) - 10.0 * M_PI * cos(5.0 * M_PI * r) / r;
}
__host__ __device__ inline void mms_grad(double x, double y, double z, double g[3]) {
  const double r = mms_r(x, y, z), c = 5.0 * M_PI * cos(5.0 * M_PI * r) / r;
  g[0] = c * x;
  g[1] = c * y;
  g[2] = c * z;
}

}  // namespace cutbddc_b200
