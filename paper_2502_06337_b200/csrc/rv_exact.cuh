// Exact (reference-identical) f64 device arithmetic for the voting path.
//
// nvcc contracts a*b+c into DFMA by default; the reference is defined on strict IEEE
// evaluation (oracle parity build: -ffp-contract=off), so every f64 operation whose
// rounding matters is spelled with an explicit round-to-nearest intrinsic here.
#pragma once
#include <cuda_runtime.h>

#include "rv_internal.h"

namespace rvb {

__device__ __forceinline__ double xm(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double xa(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double xs(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double xd(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ double xdot(double a0, double a1, double a2, double b0, double b1, double b2) {
  return xa(xa(xm(a0, b0), xm(a1, b1)), xm(a2, b2));  // Eigen 3-vector dot: (a0b0 + a1b1) + a2b2
}

// orthonormal_basis, geom.cpp:36-43 (Gram-Schmidt from the least-aligned unit axis).
__device__ __forceinline__ void exact_basis(double z0, double z1, double z2, double a1[3], double a2[3]) {
  const double f0 = fabs(z0), f1 = fabs(z1), f2 = fabs(z2);
  int least = 0;
  double m = f0;
  if (f1 < m) {
    least = 1;
    m = f1;
  }
  if (f2 < m) least = 2;
  const double e0 = least == 0 ? 1.0 : 0.0, e1 = least == 1 ? 1.0 : 0.0, e2 = least == 2 ? 1.0 : 0.0;
  const double s = xdot(e0, e1, e2, z0, z1, z2);
  const double v0 = xs(e0, xm(s, z0)), v1 = xs(e1, xm(s, z1)), v2 = xs(e2, xm(s, z2));
  const double n2 = xdot(v0, v1, v2, v0, v1, v2);
  if (n2 > 0.0) {
    const double q = __dsqrt_rn(n2);
    a1[0] = xd(v0, q);
    a1[1] = xd(v1, q);
    a1[2] = xd(v2, q);
  } else {
    a1[0] = v0;
    a1[1] = v1;
    a1[2] = v2;
  }
  a2[0] = xs(xm(z1, a1[2]), xm(z2, a1[1]));  // z x a1
  a2[1] = xs(xm(z2, a1[0]), xm(z0, a1[2]));
  a2[2] = xs(xm(z0, a1[1]), xm(z1, a1[0]));
}

// cell_of, voting.cpp:17-23 (boundary values go to the lower cell; clamp to the grid).
__device__ __forceinline__ int exact_cell_of(double v, double extent, double inv_cell, int grid) {
  const double t = xm(xa(v, extent), inv_cell);
  const double f = floor(t);
  int i = __double2int_rz(f);
  if (f == t && i > 0) --i;
  return min(max(i, 0), grid - 1);
}

// One sample of deposit_one, voting.cpp:33-44: returns the row-major cell index.
__device__ __forceinline__ void exact_sample(const double a1[3], const double a2[3], double co, double si,
                                             const VotePlan& p, int* row, int* col) {
  const double x = xa(xm(a1[0], co), xm(a2[0], si));
  const double y = xa(xm(a1[1], co), xm(a2[1], si));
  const double c = xa(xm(a1[2], co), xm(a2[2], si));
  const double sgn = c > 0.0 ? -1.0 : 1.0;
  const double inv = xd(sgn, xs(1.0, xm(sgn, c)));
  *col = exact_cell_of(xm(x, inv), p.E, p.inv_cell, p.G);
  *row = exact_cell_of(xm(y, inv), p.E, p.inv_cell, p.G);
}

}  // namespace rvb
