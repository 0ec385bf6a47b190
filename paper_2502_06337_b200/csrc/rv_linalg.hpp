// Host 3x3 linear algebra of the estimator (run on the host, as the reference does):
//  * eigen_sym3: the smallest-eigenvector solve of refine_axis (estimator.cpp:303-308).
//    Eigen is not vendored by the reference (version unpinned); this restates Eigen 3.4's
//    SelfAdjointEigenSolver path for a real 3x3 matrix: scale by max |lower coefficient|,
//    closed-form 3x3 Householder tridiagonalization, implicit symmetric QR with Wilkinson
//    shift, ascending selection sort.
//  * svd3: two-sided Jacobi SVD for the Kabsch fallback (estimator.cpp:198-215).
//  * geometry of geom.cpp:10-43 with the reference's evaluation order.
// Compiled without FMA contraction (host: -ffp-contract=off; device: nvcc -fmad=false), the
// host and device instantiations are bit-identical to each other and to the reference.
#pragma once
#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstring>

#if defined(__CUDACC__)
#define RV_HD __host__ __device__ __forceinline__
#else
#define RV_HD inline
#endif

namespace rvb {

// std::hypot of glibc 2.39 (sysdeps/ieee754/dbl-64/e_hypot.c, non-FMA kernel + scaling), which
// Eigen's SelfAdjointEigenSolver calls through numext::hypot; restated so device code matches the
// host bit-for-bit (glibc's hypot is not correctly rounded; verified equal on 3e7 random pairs).
RV_HD double hypot_kernel(double ax, double ay) {
  double t1, t2;
  double h = sqrt(ax * ax + ay * ay);
  if (h <= 2.0 * ay) {
    const double delta = h - ay;
    t1 = ax * (2.0 * delta - ax);
    t2 = (delta - 2.0 * (ax - ay)) * delta;
  } else {
    const double delta = h - ax;
    t1 = 2.0 * delta * (ax - 2.0 * ay);
    t2 = (4.0 * delta - ay) * ay + delta * delta;
  }
  h -= (t1 + t2) / (2.0 * h);
  return h;
}
RV_HD double hypot_glibc(double x, double y) {
  using std::isfinite;
  using std::isinf;
  if (!isfinite(x) || !isfinite(y)) return (isinf(x) || isinf(y)) ? INFINITY : x + y;
  x = fabs(x);
  y = fabs(y);
  const double ax = x < y ? y : x, ay = x < y ? x : y;
  const double SCALE = 0x1p-600, LARGE_VAL = 0x1p+511, TINY_VAL = 0x1p-511, EPS = 0x1p-54;
  if (ax > LARGE_VAL) {
    if (ay <= ax * EPS) return ax + ay;
    return hypot_kernel(ax * SCALE, ay * SCALE) / SCALE;
  }
  if (ay < TINY_VAL) {
    if (ax >= ay / EPS) return ax + ay;
    return hypot_kernel(ax / SCALE, ay / SCALE) * SCALE;
  }
  if (ay <= ax * EPS) return ax + ay;
  return hypot_kernel(ax, ay);
}

constexpr double kPiD = 3.14159265358979323846;

RV_HD double dot3(const double* a, const double* b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }
RV_HD double norm3(const double* a) { return sqrt(dot3(a, a)); }
RV_HD void normalized3(const double* a, double* o) {
  const double n2 = dot3(a, a);
  if (n2 > 0.0) {
    const double s = sqrt(n2);
    o[0] = a[0] / s;
    o[1] = a[1] / s;
    o[2] = a[2] / s;
  } else {
    o[0] = a[0];
    o[1] = a[1];
    o[2] = a[2];
  }
}
RV_HD void cross3(const double* a, const double* b, double* o) {
  const double t0 = a[1] * b[2] - a[2] * b[1];
  const double t1 = a[2] * b[0] - a[0] * b[2];
  const double t2 = a[0] * b[1] - a[1] * b[0];
  o[0] = t0;
  o[1] = t1;
  o[2] = t2;
}
RV_HD void canonicalize3(const double* p, double* o) {  // geom.cpp:34
  if (p[2] > 0.0) {
    o[0] = -p[0];
    o[1] = -p[1];
    o[2] = -p[2];
  } else {
    o[0] = p[0];
    o[1] = p[1];
    o[2] = p[2];
  }
}
RV_HD void unproject2(double A, double B, double* o) {  // geom.cpp:29-32
  const double s = 1.0 + A * A + B * B;
  o[0] = 2.0 * A / s;
  o[1] = 2.0 * B / s;
  o[2] = (A * A + B * B - 1.0) / s;
}
RV_HD bool project3(const double* p, double* A, double* B) {  // geom.cpp:21-27
  if (p[2] >= 1.0 - 1e-9) return false;
  const double inv = 1.0 / (1.0 - p[2]);
  *A = p[0] * inv;
  *B = p[1] * inv;
  return true;
}
RV_HD void backproject(double A, double B, double* o) {  // voting.cpp:172-174
  double u[3];
  unproject2(A, B, u);
  normalized3(u, o);
}
inline void rodrigues3(const double* a, double angle, double* r) {  // geom.cpp:10-14
  const double k[9] = {0, -a[2], a[1], a[2], 0, -a[0], -a[1], a[0], 0};
  const double s = std::sin(angle), c1 = 1.0 - std::cos(angle);
  double sk[9];
  for (int i = 0; i < 9; ++i) sk[i] = c1 * k[i];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      const double p = sk[i * 3 + 0] * k[0 * 3 + j] + sk[i * 3 + 1] * k[1 * 3 + j] + sk[i * 3 + 2] * k[2 * 3 + j];
      const double id = (i == j) ? 1.0 : 0.0;
      r[i * 3 + j] = (id + s * k[i * 3 + j]) + p;
    }
}
inline double rotation_error3(const double* g, const double* o) {  // geom.cpp:16-19
  double tr = 0.0;
  for (int i = 0; i < 3; ++i) {
    const double d = g[0 * 3 + i] * o[0 * 3 + i] + g[1 * 3 + i] * o[1 * 3 + i] + g[2 * 3 + i] * o[2 * 3 + i];
    tr = (i == 0) ? d : tr + d;
  }
  double c = 0.5 * (tr - 1.0);
  c = std::min(1.0, std::max(-1.0, c));
  return std::acos(c);
}
inline void orthonormal_basis3(const double* z, double* a1, double* a2) {  // geom.cpp:36-43
  int least = 0;
  const double az[3] = {fabs(z[0]), fabs(z[1]), fabs(z[2])};
  for (int i = 1; i < 3; ++i)
    if (az[i] < az[least]) least = i;
  double seed[3] = {0, 0, 0};
  seed[least] = 1.0;
  const double s = dot3(seed, z);
  double v[3];
  for (int i = 0; i < 3; ++i) v[i] = seed[i] - s * z[i];
  normalized3(v, a1);
  cross3(z, a1, a2);
}

RV_HD void givens(double p, double q, double* c, double* s) {
  if (q == 0.0) {
    *c = p < 0.0 ? -1.0 : 1.0;
    *s = 0.0;
  } else if (p == 0.0) {
    *c = 0.0;
    *s = q < 0.0 ? 1.0 : -1.0;
  } else if (fabs(p) > fabs(q)) {
    const double t = q / p;
    double u = sqrt(1.0 + t * t);
    if (p < 0.0) u = -u;
    *c = 1.0 / u;
    *s = -t * *c;
  } else {
    const double t = p / q;
    double u = sqrt(1.0 + t * t);
    if (q < 0.0) u = -u;
    *s = -1.0 / u;
    *c = -t * *s;
  }
}

// Symmetric 3x3 eigen-decomposition; sm row-major (lower triangle read). evecs row-major,
// eigenvector k = column k; eigenvalues ascending.
RV_HD void eigen_sym3(const double sm[9], double evals[3], double ev[9]) {
  double m[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
  for (int j = 0; j < 3; ++j)
    for (int i = j; i < 3; ++i) m[i][j] = sm[i * 3 + j];
  double scale = 0.0;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) scale = fabs(m[i][j]) > scale ? fabs(m[i][j]) : scale;
  if (scale == 0.0) scale = 1.0;
  for (int j = 0; j < 3; ++j)
    for (int i = j; i < 3; ++i) m[i][j] /= scale;
  double diag[3], sub[2], q[3][3];
  diag[0] = m[0][0];
  const double v1norm2 = m[2][0] * m[2][0];
  if (v1norm2 <= DBL_MIN) {
    diag[1] = m[1][1];
    diag[2] = m[2][2];
    sub[0] = m[1][0];
    sub[1] = m[2][1];
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) q[i][j] = (i == j) ? 1.0 : 0.0;
  } else {
    const double beta = sqrt(m[1][0] * m[1][0] + v1norm2);
    const double inv_beta = 1.0 / beta;
    const double m01 = m[1][0] * inv_beta;
    const double m02 = m[2][0] * inv_beta;
    const double qq = 2.0 * m01 * m[2][1] + m02 * (m[2][2] - m[1][1]);
    diag[1] = m[1][1] + m02 * qq;
    diag[2] = m[2][2] - m02 * qq;
    sub[0] = beta;
    sub[1] = m[2][1] - m01 * qq;
    q[0][0] = 1;
    q[0][1] = 0;
    q[0][2] = 0;
    q[1][0] = 0;
    q[1][1] = m01;
    q[1][2] = m02;
    q[2][0] = 0;
    q[2][1] = m02;
    q[2][2] = -m01;
  }
  int end = 2, start = 0, iter = 0;
  const double precision_inv = 1.0 / DBL_EPSILON;
  while (end > 0) {
    for (int i = start; i < end; ++i) {
      if (fabs(sub[i]) < DBL_MIN) {
        sub[i] = 0.0;
      } else {
        const double scaled = precision_inv * sub[i];
        if (scaled * scaled <= (fabs(diag[i]) + fabs(diag[i + 1]))) sub[i] = 0.0;
      }
    }
    while (end > 0 && sub[end - 1] == 0.0) end--;
    if (end <= 0) break;
    if (++iter > 30 * 3) break;
    start = end - 1;
    while (start > 0 && sub[start - 1] != 0.0) start--;
    const double td = (diag[end - 1] - diag[end]) * 0.5;
    const double e = sub[end - 1];
    double mu = diag[end];
    if (td == 0.0) {
      mu -= fabs(e);
    } else if (e != 0.0) {
      const double e2 = e * e;
      const double h = hypot_glibc(td, e);
      if (e2 == 0.0)
        mu -= e / ((td + (td > 0.0 ? h : -h)) / e);
      else
        mu -= e2 / (td + (td > 0.0 ? h : -h));
    }
    double x = diag[start] - mu;
    double z = sub[start];
    for (int k = start; k < end && z != 0.0; ++k) {
      double c, s;
      givens(x, z, &c, &s);
      const double sdk = s * diag[k] + c * sub[k];
      const double dkp1 = s * sub[k] + c * diag[k + 1];
      diag[k] = c * (c * diag[k] - s * sub[k]) - s * (c * sub[k] - s * diag[k + 1]);
      diag[k + 1] = s * sdk + c * dkp1;
      sub[k] = c * sdk - s * dkp1;
      if (k > start) sub[k - 1] = c * sub[k - 1] - s * z;
      x = sub[k];
      if (k < end - 1) {
        z = -s * sub[k + 1];
        sub[k + 1] = c * sub[k + 1];
      }
      for (int i = 0; i < 3; ++i) {
        const double qa = q[i][k], qb = q[i][k + 1];
        q[i][k] = c * qa - s * qb;
        q[i][k + 1] = s * qa + c * qb;
      }
    }
  }
  for (int i = 0; i < 2; ++i) {
    int k = i;
    for (int j = i + 1; j < 3; ++j)
      if (diag[j] < diag[k]) k = j;
    if (k != i) {
      const double t = diag[i];
      diag[i] = diag[k];
      diag[k] = t;
      for (int r = 0; r < 3; ++r) {
        const double u = q[r][i];
        q[r][i] = q[r][k];
        q[r][k] = u;
      }
    }
  }
  for (int i = 0; i < 3; ++i) evals[i] = diag[i] * scale;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) ev[i * 3 + j] = q[i][j];
}

// refine_axis from scatter sums (xx xy xz yy yz zz), estimator.cpp:303-308. false = RankDeficient.
RV_HD bool axis_from_scatter(const double s6[6], double axis[3]) {
  const double sm[9] = {s6[0], s6[1], s6[2], s6[1], s6[3], s6[4], s6[2], s6[4], s6[5]};
  double evals[3], ev[9];
  eigen_sym3(sm, evals, ev);
  if (evals[1] <= 1e-10 * (evals[2] > 1e-300 ? evals[2] : 1e-300)) return false;
  const double v0[3] = {ev[0], ev[3], ev[6]};
  double nv[3];
  normalized3(v0, nv);
  canonicalize3(nv, axis);
  return true;
}

// Short-latency variant of axis_from_scatter for the device refine loop (rv_coop.cu), where the
// eigen-solve sits on the critical path of every pass. Same contract (smallest-eigenvalue
// eigenvector, canonicalised; false when evals[1] <= 1e-10 * evals[2]); not bit-identical to
// the Eigen restatement (agreement ~1e-15 / relative eigen-gap, the same order as the
// differences the device's scatter summation order already introduces). Method: smallest root of
// the characteristic cubic by monotone Newton from 0, eigenvector = the largest cross product of
// two rows of M - l3 I (its exact null direction); l1, l2 from the trace and the sum of principal
// minors. No transcendental calls: a short dependency chain for the per-pass device decision.
// l3_hint (optional, in/out): the previous solve's smallest eigenvalue of the normalised scatter.
// Newton then starts just below it when chi is still negative there (the same monotone iteration,
// a few steps instead of a climb from 0 -- consecutive refine passes change the scatter little).
RV_HD bool axis_from_scatter_fast(const double s6[6], double axis[3], double* l3_hint = nullptr) {
  double scale = 0.0;
  for (int k = 0; k < 6; ++k) scale = fabs(s6[k]) > scale ? fabs(s6[k]) : scale;
  if (!(scale > 0.0)) return false;  // all-zero scatter: rank deficient
  const double inv = 1.0 / scale;
  const double a = s6[0] * inv, b = s6[1] * inv, c = s6[2] * inv, d = s6[3] * inv, e = s6[4] * inv,
               f = s6[5] * inv;  // M = [[a b c] [b d e] [c e f]]
  const double c00 = d * f - e * e, c01 = c * e - b * f, c02 = b * e - c * d;
  const double c11 = a * f - c * c, c12 = b * c - a * e, c22 = a * d - b * b;
  const double tr = a + d + f, m2 = c00 + c11 + c22, det = a * c00 + b * c01 + c * c02;
  // smallest eigenvalue: Newton on chi(l) = l^3 - tr l^2 + m2 l - det from l = 0. M is PSD, so
  // 0 <= l3 and chi is increasing and concave on [0, l3]: the iterates increase monotonically to
  // l3 (no overshoot), quadratically once l3 << l2 (one or two steps in the refine loop).
  double l3 = 0.0;
  if (l3_hint && *l3_hint > 0.0) {
    const double l0 = 0.999 * *l3_hint;
    // below the inflection point tr/3 chi is increasing and concave up to l3: chi(l0) < 0 there
    // means l0 < l3, the same monotone start condition as l = 0
    if (l0 < tr / 3.0 && ((l0 - tr) * l0 + m2) * l0 - det < 0.0) l3 = l0;
  }
  for (int it = 0; it < 32; ++it) {
    const double fl = ((l3 - tr) * l3 + m2) * l3 - det;
    const double dl = (3.0 * l3 - 2.0 * tr) * l3 + m2;
    if (!(dl > 0.0)) break;
    const double nl = l3 - fl / dl;
    if (!(nl > l3)) break;  // converged (monotone sequence stopped increasing)
    l3 = nl;
  }
  // l1 + l2 = tr - l3, l1 l2 = m2 - l3 (l1 + l2)
  if (l3_hint) *l3_hint = l3;
  const double s = tr - l3, pm = m2 - l3 * s;
  double disc = s * s - 4.0 * pm;
  disc = disc > 0.0 ? disc : 0.0;
  const double l1 = 0.5 * (s + sqrt(disc));
  const double l2 = l1 > 0.0 ? pm / l1 : 0.0;
  if (l2 <= 1e-10 * (l1 > 1e-300 ? l1 : 1e-300)) return false;  // RankDeficient
  const double r0[3] = {a - l3, b, c}, r1[3] = {b, d - l3, e}, r2[3] = {c, e, f - l3};
  double x01[3], x02[3], x12[3];
  cross3(r0, r1, x01);
  cross3(r0, r2, x02);
  cross3(r1, r2, x12);
  const double q01 = dot3(x01, x01), q02 = dot3(x02, x02), q12 = dot3(x12, x12);
  const double* best = x01;
  double qb = q01;
  if (q02 > qb) {
    best = x02;
    qb = q02;
  }
  if (q12 > qb) best = x12;
  double nv[3];
  normalized3(best, nv);
  canonicalize3(nv, axis);
  return true;
}

// Two-sided Jacobi SVD of a 3x3 (row-major); u, v row-major, singular values descending.
inline void svd3(const double a[9], double u[9], double v[9]) {
  double w[3][3], U[3][3], V[3][3];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      w[i][j] = a[i * 3 + j];
      U[i][j] = V[i][j] = (i == j) ? 1.0 : 0.0;
    }
  const double prec = 2.0 * DBL_EPSILON;
  double max_diag = 0;
  for (int i = 0; i < 3; ++i) max_diag = std::max(max_diag, fabs(w[i][i]));
  bool finished = false;
  for (int sweeps = 0; !finished && sweeps < 100; ++sweeps) {
    finished = true;
    for (int p = 1; p < 3; ++p)
      for (int qi = 0; qi < p; ++qi) {
        const double thr = std::max(4.9e-324, prec * max_diag);
        if (fabs(w[p][qi]) > thr || fabs(w[qi][p]) > thr) {
          finished = false;
          const double m00 = w[qi][qi], m01 = w[qi][p], m10 = w[p][qi], m11 = w[p][p];
          double c1 = 1, s1 = 0;
          const double t = m00 + m11, d = m10 - m01;
          if (fabs(d) >= DBL_MIN) {
            const double uu = t / d;
            const double tmp = sqrt(1.0 + uu * uu);
            s1 = 1.0 / tmp;
            c1 = uu / tmp;
          }
          const double n00 = c1 * m00 + s1 * m10, n01 = c1 * m01 + s1 * m11;
          const double n11 = -s1 * m01 + c1 * m11;
          double jc = 1, js = 0;
          const double deno = 2.0 * fabs(n01);
          if (deno >= DBL_MIN) {
            const double tau = (n00 - n11) / deno;
            const double ww = sqrt(tau * tau + 1.0);
            const double tt = tau > 0.0 ? 1.0 / (tau + ww) : 1.0 / (tau - ww);
            const double sign_t = tt > 0.0 ? 1.0 : -1.0;
            const double nn = 1.0 / sqrt(tt * tt + 1.0);
            js = -sign_t * (n01 / fabs(n01)) * fabs(tt) * nn;
            jc = nn;
          }
          const double lc = c1 * jc - s1 * (-js), ls = c1 * (-js) + s1 * jc;
          for (int k = 0; k < 3; ++k) {
            const double x = w[qi][k], y = w[p][k];
            w[qi][k] = lc * x + ls * y;
            w[p][k] = -ls * x + lc * y;
          }
          for (int k = 0; k < 3; ++k) {
            const double x = U[k][qi], y = U[k][p];
            U[k][qi] = lc * x + ls * y;
            U[k][p] = -ls * x + lc * y;
          }
          for (int k = 0; k < 3; ++k) {
            double x = w[k][qi], y = w[k][p];
            w[k][qi] = jc * x - js * y;
            w[k][p] = js * x + jc * y;
            x = V[k][qi];
            y = V[k][p];
            V[k][qi] = jc * x - js * y;
            V[k][p] = js * x + jc * y;
          }
          max_diag = std::max(max_diag, std::max(fabs(w[p][p]), fabs(w[qi][qi])));
        }
      }
  }
  double sv[3];
  for (int i = 0; i < 3; ++i) {
    sv[i] = fabs(w[i][i]);
    if (w[i][i] < 0.0)
      for (int k = 0; k < 3; ++k) U[k][i] = -U[k][i];
  }
  for (int i = 0; i < 3; ++i) {
    int best = i;
    for (int j = i + 1; j < 3; ++j)
      if (sv[j] > sv[best]) best = j;
    if (best != i) {
      std::swap(sv[i], sv[best]);
      for (int k = 0; k < 3; ++k) {
        std::swap(U[k][i], U[k][best]);
        std::swap(V[k][i], V[k][best]);
      }
    }
  }
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      u[i * 3 + j] = U[i][j];
      v[i * 3 + j] = V[i][j];
    }
}

inline void mat3_mul(const double* a, const double* b, double* o) {
  double t[9];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) t[i * 3 + j] = a[i * 3 + 0] * b[0 * 3 + j] + a[i * 3 + 1] * b[1 * 3 + j] + a[i * 3 + 2] * b[2 * 3 + j];
  std::memcpy(o, t, sizeof t);
}
inline void mat3_t(const double* a, double* o) {
  double t[9];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) t[j * 3 + i] = a[i * 3 + j];
  std::memcpy(o, t, sizeof t);
}
inline double det3(const double* m) {
  return m[0] * (m[4] * m[8] - m[7] * m[5]) - m[3] * (m[1] * m[8] - m[7] * m[2]) + m[6] * (m[1] * m[5] - m[4] * m[2]);
}

// Kabsch from a cross-covariance h (estimator.cpp:211-214).
inline void kabsch(const double h[9], double r[9]) {
  double u[9], v[9], vt[9], uvt[9], d[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
  svd3(h, u, v);
  mat3_t(v, vt);
  mat3_mul(u, vt, uvt);
  d[8] = det3(uvt) < 0.0 ? -1.0 : 1.0;
  double ud[9];
  mat3_mul(u, d, ud);
  mat3_mul(ud, vt, r);
}

// AngleAxisd(r) via Quaternion(r) (Eigen), then the canonical axis/angle of estimator.cpp:242-244.
inline void angle_axis_canonical(const double r[9], double axis[3], double* angle) {
  double qw, qv[3];
  double t = r[0] + r[4] + r[8];
  if (t > 0.0) {
    t = sqrt(t + 1.0);
    qw = 0.5 * t;
    t = 0.5 / t;
    qv[0] = (r[7] - r[5]) * t;
    qv[1] = (r[2] - r[6]) * t;
    qv[2] = (r[3] - r[1]) * t;
  } else {
    int i = 0;
    if (r[4] > r[0]) i = 1;
    if (r[8] > r[i * 4]) i = 2;
    const int j = (i + 1) % 3, k = (j + 1) % 3;
    t = sqrt(r[i * 4] - r[j * 4] - r[k * 4] + 1.0);
    qv[i] = 0.5 * t;
    t = 0.5 / t;
    qw = (r[k * 3 + j] - r[j * 3 + k]) * t;
    qv[j] = (r[j * 3 + i] + r[i * 3 + j]) * t;
    qv[k] = (r[k * 3 + i] + r[i * 3 + k]) * t;
  }
  double n = norm3(qv), aa_angle, aa_axis[3];
  if (n != 0.0) {
    aa_angle = 2.0 * std::atan2(n, fabs(qw));
    if (qw < 0.0) n = -n;
    aa_axis[0] = qv[0] / n;
    aa_axis[1] = qv[1] / n;
    aa_axis[2] = qv[2] / n;
  } else {
    aa_angle = 0.0;
    aa_axis[0] = 1.0;
    aa_axis[1] = 0.0;
    aa_axis[2] = 0.0;
  }
  canonicalize3(aa_axis, axis);
  *angle = dot3(axis, aa_axis) < 0.0 ? -aa_angle : aa_angle;
}

}  // namespace rvb
