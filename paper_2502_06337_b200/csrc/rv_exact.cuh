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

// preprocess of one correspondence (estimator.cpp:264-279): optional normalisation of x and y,
// d = y - x, dropped iff |d| < tau_z (returns false), z = d / |d| -- the reference's op order.
__device__ __forceinline__ bool preprocess_pair(double x0, double x1, double x2, double y0, double y1, double y2,
                                                int normalize, double tau_z, double z[3]) {
  if (normalize) {
    const double nx = __dsqrt_rn(xdot(x0, x1, x2, x0, x1, x2));
    const double ny = __dsqrt_rn(xdot(y0, y1, y2, y0, y1, y2));
    if (nx > 0.0) {
      x0 = xd(x0, nx);
      x1 = xd(x1, nx);
      x2 = xd(x2, nx);
    }
    if (ny > 0.0) {
      y0 = xd(y0, ny);
      y1 = xd(y1, ny);
      y2 = xd(y2, ny);
    }
  }
  const double d0 = xs(y0, x0), d1 = xs(y1, x1), d2 = xs(y2, x2);
  const double len = __dsqrt_rn(xdot(d0, d1, d2, d0, d1, d2));
  z[0] = xd(d0, len);
  z[1] = xd(d1, len);
  z[2] = xd(d2, len);
  return !(len < tau_z);
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

// estimate_from_peak (estimator.cpp:94-101) from an argmax key: the peak cell, interpolate_peak
// (estimator.cpp:32-47: 3x3 vote-weighted centroid, dy outer / dx inner), backproject
// (voting.cpp:172-174: unproject + normalize), canonicalize (geom.cpp:34) -- every operation
// explicitly rounded, in the host's order, so the start axis is bit-identical to the host path's.
__device__ __forceinline__ void exact_peak_axis(unsigned long long key, unsigned long long total,
                                                const uint32_t* grid, int G, double E, uint32_t min_votes,
                                                PeakOut* out) {
  PeakOut r;
  r.total = total;
  r.ok = 0;
  r.ix = r.iy = 0;
  r.votes = 0;
  r.A = r.B = 0.0;
  r.axis[0] = r.axis[1] = 0.0;
  r.axis[2] = -1.0;
  const uint32_t best = (uint32_t)(key >> 32);
  if (key != 0 && best >= min_votes) {
    const uint32_t idx = 0xFFFFFFFFu - (uint32_t)(key & 0xFFFFFFFFu);
    const int iy = (int)idx / G, ix = (int)idx % G;
    const double cw = xd(xm(2.0, E), (double)G);
    double wsum = 0.0, asum = 0.0, bsum = 0.0;
    for (int dy = -1; dy <= 1; ++dy)
      for (int dx = -1; dx <= 1; ++dx) {
        const int x = ix + dx, y = iy + dy;
        if (x < 0 || x >= G || y < 0 || y >= G) continue;
        const double wv = (double)__ldcg(grid + (size_t)y * G + x);
        const double cA = xa(-E, xm(xa((double)x, 0.5), cw)), cB = xa(-E, xm(xa((double)y, 0.5), cw));
        wsum = xa(wsum, wv);
        asum = xa(asum, xm(wv, cA));
        bsum = xa(bsum, xm(wv, cB));
      }
    double A = xa(-E, xm(xa((double)ix, 0.5), cw)), B = xa(-E, xm(xa((double)iy, 0.5), cw));
    if (wsum > 0.0) {
      A = xd(asum, wsum);
      B = xd(bsum, wsum);
    }
    const double AA = xm(A, A), BB = xm(B, B);
    const double s = xa(xa(1.0, AA), BB);
    const double u0 = xd(xm(2.0, A), s), u1 = xd(xm(2.0, B), s), u2 = xd(xs(xa(AA, BB), 1.0), s);
    const double n2 = xa(xa(xm(u0, u0), xm(u1, u1)), xm(u2, u2));
    double b0 = u0, b1 = u1, b2 = u2;
    if (n2 > 0.0) {
      const double q = __dsqrt_rn(n2);
      b0 = xd(u0, q);
      b1 = xd(u1, q);
      b2 = xd(u2, q);
    }
    const bool flip = b2 > 0.0;
    r.axis[0] = flip ? -b0 : b0;
    r.axis[1] = flip ? -b1 : b1;
    r.axis[2] = flip ? -b2 : b2;
    r.A = A;
    r.B = B;
    r.ix = ix;
    r.iy = iy;
    r.votes = best;
    r.ok = 1;
  }
  *out = r;
}

}  // namespace rvb
