/* CPU oracle (TEST INFRASTRUCTURE ONLY) -- plain-C restatement of the reference path.
 * See rv_oracle.h. Citations are relative to /root/reference/proj.
 * Compile with -O2 -ffp-contract=off: every expression below is evaluated in the
 * reference's source order with IEEE double rounding and no FMA contraction.
 */
#include "rv_oracle.h"

#include <float.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

#define RVO_PI 3.14159265358979323846 /* == std::numbers::pi as a double */

static rvo_trace g_trace;
void rvo_last_trace(rvo_trace* out) { *out = g_trace; }
void rvo_free(void* p) { free(p); }

void rvo_config_default(rvo_config* c) { /* estimator.hpp:13-29 */
  c->grid = 512;
  c->extent = 1.05;
  c->theta_samples = 2048;
  c->epsilon = 0.015;
  c->angle_bins = 1024;
  c->max_models = 1;
  c->min_votes_frac = 0.02;
  c->consensus_floor_mult = 1.5;
  c->dedupe_overlap = 0.5;
  c->tau_z = 1e-9;
  c->tau_deg = 1e-6;
  c->suppression_radius = 8;
  c->refine = 1;
  c->normalize_inputs = 1;
  c->threads = 1;
}

/* ---- 3-vector helpers with Eigen's evaluation order for size 3 -------------------- */
static double dot3(const double* a, const double* b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }
static double norm3(const double* a) { return sqrt(dot3(a, a)); }
static void normalized3(const double* a, double* o) { /* Eigen 3.4 normalized() */
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
static void cross3(const double* a, const double* b, double* o) {
  const double t0 = a[1] * b[2] - a[2] * b[1];
  const double t1 = a[2] * b[0] - a[0] * b[2];
  const double t2 = a[0] * b[1] - a[1] * b[0];
  o[0] = t0;
  o[1] = t1;
  o[2] = t2;
}
static void canonicalize3(const double* p, double* o) { /* geom.cpp:34 */
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
static int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

/* ---- geometry: geom.cpp ------------------------------------------------------------ */
void rvo_rodrigues(const double a[3], double angle, double r[9]) { /* geom.cpp:10-14 */
  /* k << 0,-z,y, z,0,-x, -y,x,0 ; R = I + sin*k + ((1-cos)*k)*k  (Eigen parses left to right) */
  const double k[9] = {0, -a[2], a[1], a[2], 0, -a[0], -a[1], a[0], 0};
  const double s = sin(angle), c1 = 1.0 - cos(angle);
  double sk[9];
  for (int i = 0; i < 9; ++i) sk[i] = c1 * k[i];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      const double p = sk[i * 3 + 0] * k[0 * 3 + j] + sk[i * 3 + 1] * k[1 * 3 + j] + sk[i * 3 + 2] * k[2 * 3 + j];
      const double id = (i == j) ? 1.0 : 0.0;
      r[i * 3 + j] = (id + s * k[i * 3 + j]) + p;
    }
}

double rvo_rotation_error(const double g[9], const double o[9]) { /* geom.cpp:16-19 */
  /* trace(g^T o) = sum_i sum_k g(k,i) o(k,i), product entries with inner order k=0..2 */
  double tr = 0.0;
  for (int i = 0; i < 3; ++i) {
    const double d = g[0 * 3 + i] * o[0 * 3 + i] + g[1 * 3 + i] * o[1 * 3 + i] + g[2 * 3 + i] * o[2 * 3 + i];
    tr = (i == 0) ? d : tr + d;
  }
  double c = 0.5 * (tr - 1.0);
  if (c < -1.0) c = -1.0;
  if (c > 1.0) c = 1.0;
  return acos(c);
}

static int project3(const double* p, double* A, double* B) { /* geom.cpp:21-27 */
  if (p[2] >= 1.0 - 1e-9) return RVO_POLE_PROXIMITY;
  const double inv = 1.0 / (1.0 - p[2]);
  *A = p[0] * inv;
  *B = p[1] * inv;
  return RVO_OK;
}

static void unproject2(double A, double B, double* o) { /* geom.cpp:29-32 */
  const double s = 1.0 + A * A + B * B;
  o[0] = 2.0 * A / s;
  o[1] = 2.0 * B / s;
  o[2] = (A * A + B * B - 1.0) / s;
}

void rvo_orthonormal_basis(const double z[3], double a1[3], double a2[3]) { /* geom.cpp:36-43 */
  int least = 0; /* cwiseAbs().minCoeff(&least): first minimum */
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

/* ---- voting: voting.cpp ------------------------------------------------------------ */
static inline int cell_of(double v, double extent, double inv_cell, int grid) { /* voting.cpp:17-23 */
  const double t = (v + extent) * inv_cell;
  const double f = floor(t);
  int i = (int)f;
  if (f == t && i > 0) --i;
  return clampi(i, 0, grid - 1);
}

int32_t rvo_coord_to_cell(double v, int32_t grid, double extent) { /* voting.cpp:55-57 */
  return cell_of(v, extent, grid / (2.0 * extent), grid);
}

static void cell_center(int ix, int iy, int grid, double extent, double* A, double* B) { /* :59-62 */
  const double cs = 2.0 * extent / grid;
  *A = -extent + (ix + 0.5) * cs;
  *B = -extent + (iy + 0.5) * cs;
}

void rvo_circle_table(int32_t samples, double* table) { /* voting.cpp:72-81 */
  const double step = 2.0 * RVO_PI / samples;
  for (int j = 0; j < samples; ++j) {
    const double theta = -RVO_PI + j * step;
    table[2 * j] = cos(theta);
    table[2 * j + 1] = sin(theta);
  }
}

static void deposit_one(const double* z, uint32_t* counts, int grid, double extent, const double* t,
                        int n) { /* voting.cpp:25-45 */
  double a1[3], a2[3];
  rvo_orthonormal_basis(z, a1, a2);
  const double inv_cell = grid / (2.0 * extent);
  for (int j = 0; j < n; ++j) {
    const double co = t[2 * j], si = t[2 * j + 1];
    const double x = a1[0] * co + a2[0] * si;
    const double y = a1[1] * co + a2[1] * si;
    const double c = a1[2] * co + a2[2] * si;
    const double sgn = c > 0.0 ? -1.0 : 1.0;
    const double inv = sgn / (1.0 - sgn * c);
    const int ix = cell_of(x * inv, extent, inv_cell, grid);
    const int iy = cell_of(y * inv, extent, inv_cell, grid);
    counts[(size_t)iy * grid + ix]++;
  }
}

void rvo_deposit_circle(const double z[3], uint32_t* counts, int32_t grid, double extent,
                        int32_t samples) {
  double* table = (double*)malloc(sizeof(double) * 2 * (size_t)samples);
  rvo_circle_table(samples, table);
  deposit_one(z, counts, grid, extent, table, samples);
  free(table);
}

int rvo_accumulate(const double* z, int64_t n, int32_t grid, double extent, int32_t samples,
                   uint32_t* counts) { /* voting.cpp:88-118 */
  if (n <= 0) return RVO_EMPTY_INPUT;
  if (grid < 1 || extent <= 0.0) return RVO_INVALID_CONFIG; /* Accumulator2D ctor, :49-53 */
  memset(counts, 0, sizeof(uint32_t) * (size_t)grid * grid);
  double* table = (double*)malloc(sizeof(double) * 2 * (size_t)samples);
  if (!table) return RVO_OUT_OF_MEMORY;
  rvo_circle_table(samples, table);
  for (int64_t i = 0; i < n; ++i) deposit_one(z + 3 * i, counts, grid, extent, table, samples);
  free(table);
  return RVO_OK;
}

static void mask_disk(uint8_t* masked, int g, int cx, int cy, int r) { /* voting.cpp:126-138 */
  const int r2 = r * r;
  for (int dy = -r; dy <= r; ++dy) {
    const int y = cy + dy;
    if (y < 0 || y >= g) continue;
    for (int dx = -r; dx <= r; ++dx) {
      const int x = cx + dx;
      if (x < 0 || x >= g) continue;
      if (dx * dx + dy * dy <= r2) masked[(size_t)y * g + x] = 1;
    }
  }
}

int rvo_find_peaks(const uint32_t* counts, int32_t g, double extent, int32_t max_peaks, int32_t radius,
                   uint32_t min_votes, rvo_peak* out, int32_t* n_out) { /* voting.cpp:120-170 */
  uint8_t* masked = (uint8_t*)calloc((size_t)g * g, 1);
  if (!masked) return RVO_OUT_OF_MEMORY;
  const double cs = 2.0 * extent / g;
  int np = 0;
  for (int k = 0; k < max_peaks; ++k) {
    uint32_t best = 0;
    size_t best_idx = 0;
    int found = 0;
    for (size_t i = 0; i < (size_t)g * g; ++i) {
      if (!masked[i] && counts[i] > best) {
        best = counts[i];
        best_idx = i;
        found = 1;
      }
    }
    if (!found || best < min_votes || best == 0) break;
    const int iy = (int)best_idx / g;
    const int ix = (int)best_idx % g;
    rvo_peak p;
    p.ix = ix;
    p.iy = iy;
    cell_center(ix, iy, g, extent, &p.A, &p.B);
    p.votes = best;
    out[np++] = p;
    mask_disk(masked, g, ix, iy, radius);
    const double norm = hypot(p.A, p.B);
    if (fabs(norm - 1.0) <= 1.5 * cs && norm > 0.0) {
      const double mx = -p.A / norm;
      const double my = -p.B / norm;
      mask_disk(masked, g, rvo_coord_to_cell(mx, g, extent), rvo_coord_to_cell(my, g, extent), radius);
    }
  }
  free(masked);
  *n_out = np;
  if (np == 0) return RVO_NO_PEAK;
  return RVO_OK;
}

void rvo_backproject_peak(double A, double B, double out[3]) { /* voting.cpp:172-174 */
  double u[3];
  unproject2(A, B, u);
  normalized3(u, out);
}

int rvo_blurred_argmax(const uint32_t* counts, int32_t g, double extent, int32_t radius,
                       rvo_peak* out) { /* voting.cpp:176-216 */
  if (radius < 0) return RVO_INVALID_CONFIG;
  const size_t w = (size_t)g + 1;
  uint64_t* sat = (uint64_t*)calloc(w * w, sizeof(uint64_t));
  if (!sat) return RVO_OUT_OF_MEMORY;
  for (int y = 0; y < g; ++y) {
    uint64_t row = 0;
    for (int x = 0; x < g; ++x) {
      row += counts[(size_t)y * g + x];
      sat[(size_t)(y + 1) * w + (x + 1)] = sat[(size_t)y * w + (x + 1)] + row;
    }
  }
  uint64_t best_sum = 0;
  int found = 0, bx = 0, by = 0;
  for (int cy = 0; cy < g; ++cy) {
    for (int cx = 0; cx < g; ++cx) {
      const int x0 = cx - radius > 0 ? cx - radius : 0, x1 = cx + radius + 1 < g ? cx + radius + 1 : g;
      const int y0 = cy - radius > 0 ? cy - radius : 0, y1 = cy + radius + 1 < g ? cy + radius + 1 : g;
      const uint64_t s = sat[(size_t)y1 * w + x1] - sat[(size_t)y0 * w + x1] - sat[(size_t)y1 * w + x0] +
                         sat[(size_t)y0 * w + x0];
      if (!found || s > best_sum) {
        best_sum = s;
        bx = cx;
        by = cy;
        found = 1;
      }
    }
  }
  free(sat);
  out->ix = bx;
  out->iy = by;
  cell_center(bx, by, g, extent, &out->A, &out->B);
  out->votes = best_sum > 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)best_sum;
  return RVO_OK;
}

/* ---- estimator.cpp: preprocess / classify / refine ---------------------------------- */
int rvo_preprocess(const double* corrs, int64_t n, double tau_z, int normalize, double* z_out,
                   int32_t* kept_out, int32_t* dropped_out, int64_t* n_kept,
                   int64_t* n_dropped) { /* estimator.cpp:259-285 */
  int64_t nk = 0, nd = 0;
  for (int64_t i = 0; i < n; ++i) {
    double x[3] = {corrs[6 * i + 0], corrs[6 * i + 1], corrs[6 * i + 2]};
    double y[3] = {corrs[6 * i + 3], corrs[6 * i + 4], corrs[6 * i + 5]};
    if (normalize) {
      const double nx = norm3(x), ny = norm3(y);
      if (nx > 0.0) {
        x[0] /= nx;
        x[1] /= nx;
        x[2] /= nx;
      }
      if (ny > 0.0) {
        y[0] /= ny;
        y[1] /= ny;
        y[2] /= ny;
      }
    }
    const double d[3] = {y[0] - x[0], y[1] - x[1], y[2] - x[2]};
    const double len = norm3(d);
    if (len < tau_z) {
      dropped_out[nd++] = (int32_t)i;
      continue;
    }
    z_out[3 * nk + 0] = d[0] / len;
    z_out[3 * nk + 1] = d[1] / len;
    z_out[3 * nk + 2] = d[2] / len;
    kept_out[nk++] = (int32_t)i;
  }
  *n_kept = nk;
  *n_dropped = nd;
  if (n > 0 && nk == 0) return RVO_ALL_DEGENERATE;
  return RVO_OK;
}

int64_t rvo_classify_inliers(const double axis[3], const double* z, int64_t n, double eps,
                             int32_t* out) { /* estimator.cpp:287-297 */
  const double ax = axis[0], ay = axis[1], az = axis[2];
  int64_t m = 0;
  for (int64_t i = 0; i < n; ++i) {
    const double d = ax * z[3 * i] + ay * z[3 * i + 1] + az * z[3 * i + 2];
    if (fabs(d) < eps) out[m++] = (int32_t)i;
  }
  return m;
}

/* Eigen 3.4 SelfAdjointEigenSolver<Matrix3d> restated (Eigen is not vendored: version
 * unpinned): scale by max |lower coefficient|, closed-form 3x3 tridiagonalization
 * (tridiagonalization_inplace_selector<...,3,false>), implicit symmetric QR steps with
 * Wilkinson shift (tridiagonal_qr_step), ascending selection sort. s/evecs row-major. */
static void givens(double p, double q, double* c, double* s) { /* JacobiRotation::makeGivens */
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

void rvo_eigen_sym3(const double sm[9], double evals[3], double ev[9]) {
  double m[3][3] = {{0}};
  for (int j = 0; j < 3; ++j)
    for (int i = j; i < 3; ++i) m[i][j] = sm[i * 3 + j]; /* lower triangle */
  double scale = 0.0;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      if (fabs(m[i][j]) > scale) scale = fabs(m[i][j]);
  if (scale == 0.0) scale = 1.0;
  for (int j = 0; j < 3; ++j)
    for (int i = j; i < 3; ++i) m[i][j] /= scale;
  double diag[3], sub[2], q[3][3];
  const double tol = DBL_MIN;
  diag[0] = m[0][0];
  const double v1norm2 = m[2][0] * m[2][0];
  if (v1norm2 <= tol) {
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
    q[0][0] = 1; q[0][1] = 0;   q[0][2] = 0;
    q[1][0] = 0; q[1][1] = m01; q[1][2] = m02;
    q[2][0] = 0; q[2][1] = m02; q[2][2] = -m01;
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
    iter++;
    if (iter > 30 * 3) break;
    start = end - 1;
    while (start > 0 && sub[start - 1] != 0.0) start--;
    /* tridiagonal_qr_step(diag, sub, start, end, Q) */
    const double td = (diag[end - 1] - diag[end]) * 0.5;
    const double e = sub[end - 1];
    double mu = diag[end];
    if (td == 0.0) {
      mu -= fabs(e);
    } else if (e != 0.0) {
      const double e2 = e * e;
      const double h = hypot(td, e);
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

static int refine_from_scatter(const double sc[9], double axis_out[3]) { /* estimator.cpp:303-308 */
  double evals[3], ev[9];
  rvo_eigen_sym3(sc, evals, ev);
  const double hi = evals[2] > 1e-300 ? evals[2] : 1e-300;
  if (evals[1] <= 1e-10 * hi) return RVO_RANK_DEFICIENT;
  const double v0[3] = {ev[0], ev[3], ev[6]};
  double nv[3];
  normalized3(v0, nv);
  canonicalize3(nv, axis_out);
  return RVO_OK;
}

int rvo_refine_axis(const double* z, int64_t n, double axis_out[3]) { /* estimator.cpp:299-309 */
  if (n < 2) return RVO_RANK_DEFICIENT;
  double sc[9] = {0};
  for (int64_t k = 0; k < n; ++k) {
    const double* v = z + 3 * k;
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) sc[i * 3 + j] += v[i] * v[j];
  }
  return refine_from_scatter(sc, axis_out);
}

/* refine_axis over a gathered index subset (estimator.cpp:24-29 gather + :299-309) */
static int refine_axis_idx(const double* z, const int32_t* idx, int64_t n, double axis_out[3]) {
  if (n < 2) return RVO_RANK_DEFICIENT;
  double sc[9] = {0};
  for (int64_t k = 0; k < n; ++k) {
    const double* v = z + 3 * (size_t)idx[k];
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) sc[i * 3 + j] += v[i] * v[j];
  }
  return refine_from_scatter(sc, axis_out);
}

uint32_t rvo_peak_vote_floor(const rvo_config* cfg, int64_t n) { /* estimator.cpp:311-318 */
  const double cell = 2.0 * cfg->extent / cfg->grid;
  const double per_crossing = cfg->theta_samples * cell / (2.0 * RVO_PI);
  const double floor_votes = cfg->min_votes_frac * (double)n * per_crossing;
  return (uint32_t)(floor_votes > 16.0 ? floor_votes : 16.0);
}

/* ---- angles.cpp ---------------------------------------------------------------------- */
static double circular_diff(double a, double b) { /* angles.cpp:14-20 */
  double d = fmod(a - b, 2.0 * RVO_PI);
  if (d <= -RVO_PI) d += 2.0 * RVO_PI;
  if (d > RVO_PI) d -= 2.0 * RVO_PI;
  return d;
}

static int bin_of(double angle, int n) { /* angles.cpp:25-30 */
  const double w = 2.0 * RVO_PI / n;
  const int k = (int)ceil((angle + RVO_PI) / w) - 1;
  return clampi(k, 0, n - 1);
}

int rvo_correspondence_angle(const double axis[3], const double x[3], const double y[3], double tau,
                             double* angle) { /* angles.cpp:36-44 */
  double beta[3], gamma[3], bg[3];
  cross3(axis, x, beta);
  cross3(axis, y, gamma);
  if (norm3(beta) <= tau || norm3(gamma) <= tau) return RVO_DEGENERATE_PROJECTION;
  cross3(beta, gamma, bg);
  *angle = atan2(dot3(bg, axis), dot3(beta, gamma));
  return RVO_OK;
}

int rvo_vote_angles(const double axis[3], const double* corrs, const int32_t* idx, int64_t n_idx,
                    int32_t bin_count, double tau, uint32_t* bins, uint64_t* contributing,
                    uint64_t* degenerate, double* raw_out) { /* angles.cpp:46-68 */
  if (bin_count < 8) return RVO_INVALID_CONFIG;
  memset(bins, 0, sizeof(uint32_t) * (size_t)bin_count);
  uint64_t contrib = 0, degen = 0;
  for (int64_t k = 0; k < n_idx; ++k) {
    const double* c = corrs + 6 * (size_t)idx[k];
    double a;
    if (rvo_correspondence_angle(axis, c, c + 3, tau, &a) != RVO_OK) {
      ++degen;
      continue;
    }
    ++bins[bin_of(a, bin_count)];
    raw_out[contrib++] = a;
  }
  *contributing = contrib;
  *degenerate = degen;
  if (contrib == 0) return RVO_NO_VOTES;
  return RVO_OK;
}

int rvo_peak_angle(const uint32_t* bins, int32_t n, uint64_t contributing, int refine, const double* raw,
                   int64_t n_raw, double* out) { /* angles.cpp:70-90 */
  if (contributing == 0) return RVO_NO_VOTES;
  int k = 0;
  for (int i = 1; i < n; ++i)
    if (bins[i] > bins[k]) k = i; /* max_element: first maximum */
  const double w = 2.0 * RVO_PI / n;
  const double center = -RVO_PI + (k + 0.5) * w;
  if (!refine) {
    *out = center;
    return RVO_OK;
  }
  const double window = 1.5 * w;
  double s = 0.0, c = 0.0;
  for (int64_t i = 0; i < n_raw; ++i) {
    if (fabs(circular_diff(raw[i], center)) <= window) {
      s += sin(raw[i]);
      c += cos(raw[i]);
    }
  }
  if (s == 0.0 && c == 0.0) {
    *out = center;
    return RVO_OK;
  }
  double mean = atan2(s, c);
  if (mean <= -RVO_PI) mean += 2.0 * RVO_PI;
  *out = mean;
  return RVO_OK;
}

/* ---- estimator orchestration ---------------------------------------------------------- */
typedef struct {
  double* z;        /* constraints, n x 3 */
  int32_t* kept;    /* constraint -> input index */
  int32_t* dropped;
  int64_t n, nd;
} pre_t;

typedef struct {
  int32_t* v;
  int64_t n, cap;
} ivec;

static void est_clear(rvo_estimate* e) {
  e->axis[0] = 0;
  e->axis[1] = 0;
  e->axis[2] = -1;
  e->angle = 0;
  for (int i = 0; i < 9; ++i) e->rotation[i] = (i % 4 == 0) ? 1.0 : 0.0;
  e->axis_votes = 0;
  e->n_inliers = 0;
  e->inliers = NULL;
}

/* refine_loop, estimator.cpp:51-69. inl (constraint indices) sized >= n. Returns count. */
static int64_t refine_loop(double axis[3], const pre_t* pre, const rvo_config* cfg, int32_t* inl,
                           int32_t* tmp, int32_t* passes) {
  int64_t m = rvo_classify_inliers(axis, pre->z, pre->n, cfg->epsilon, inl);
  if (passes) *passes = 0;
  if (!cfg->refine) return m;
  for (int pass = 0; pass < 10 && m >= 2; ++pass) {
    double next[3];
    if (refine_axis_idx(pre->z, inl, m, next) != RVO_OK) break; /* RankDeficient: keep axis */
    if (passes) ++*passes;
    const int64_t m2 = rvo_classify_inliers(next, pre->z, pre->n, cfg->epsilon, tmp);
    axis[0] = next[0];
    axis[1] = next[1];
    axis[2] = next[2];
    const int stable = (m2 == m) && memcmp(tmp, inl, sizeof(int32_t) * (size_t)m) == 0;
    memcpy(inl, tmp, sizeof(int32_t) * (size_t)m2);
    m = m2;
    if (stable) break;
  }
  return m;
}

/* build_estimate, estimator.cpp:73-92 */
static int build_estimate(const double axis[3], const int32_t* inl, int64_t m, uint32_t votes,
                          const double* corrs, const pre_t* pre, const rvo_config* cfg,
                          rvo_estimate* est) {
  int32_t* corr_idx = (int32_t*)malloc(sizeof(int32_t) * (size_t)(m > 0 ? m : 1));
  double* raw = (double*)malloc(sizeof(double) * (size_t)(m > 0 ? m : 1));
  uint32_t* bins = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)(cfg->angle_bins > 8 ? cfg->angle_bins : 8));
  if (!corr_idx || !raw || !bins) {
    free(corr_idx);
    free(raw);
    free(bins);
    return RVO_OUT_OF_MEMORY;
  }
  for (int64_t k = 0; k < m; ++k) corr_idx[k] = pre->kept[inl[k]];
  uint64_t contrib = 0, degen = 0;
  int st = rvo_vote_angles(axis, corrs, corr_idx, m, cfg->angle_bins, cfg->tau_deg, bins, &contrib, &degen, raw);
  double angle = 0;
  if (st == RVO_OK) st = rvo_peak_angle(bins, cfg->angle_bins, contrib, cfg->refine, raw, (int64_t)contrib, &angle);
  free(raw);
  free(bins);
  if (st != RVO_OK) {
    free(corr_idx);
    return st;
  }
  est->axis[0] = axis[0];
  est->axis[1] = axis[1];
  est->axis[2] = axis[2];
  est->angle = angle;
  rvo_rodrigues(axis, angle, est->rotation);
  est->inliers = corr_idx;
  est->n_inliers = m;
  est->axis_votes = votes;
  return RVO_OK;
}

static void interpolate_peak(const uint32_t* counts, int g, double extent, const rvo_peak* pk, double* A,
                             double* B) { /* estimator.cpp:32-47 */
  double wsum = 0.0, asum = 0.0, bsum = 0.0;
  for (int dy = -1; dy <= 1; ++dy) {
    for (int dx = -1; dx <= 1; ++dx) {
      const int ix = pk->ix + dx, iy = pk->iy + dy;
      if (ix < 0 || ix >= g || iy < 0 || iy >= g) continue;
      const double w = counts[(size_t)iy * g + ix];
      double cA, cB;
      cell_center(ix, iy, g, extent, &cA, &cB);
      wsum += w;
      asum += w * cA;
      bsum += w * cB;
    }
  }
  if (wsum <= 0.0) {
    *A = pk->A;
    *B = pk->B;
    return;
  }
  *A = asum / wsum;
  *B = bsum / wsum;
}

typedef struct {
  int64_t coherent;
  double* band;
  int64_t nband;
} support_t;

/* model_support, estimator.cpp:117-137 (band collected only if want_band) */
static support_t model_support(const rvo_estimate* est, const double* corrs, const pre_t* pre,
                               const rvo_config* cfg, int want_band) {
  support_t s = {0, NULL, 0};
  if (want_band) s.band = (double*)malloc(sizeof(double) * (size_t)(pre->n > 0 ? pre->n : 1));
  for (int64_t k = 0; k < pre->n; ++k) {
    const double d = fabs(dot3(est->axis, pre->z + 3 * k));
    if (d >= 4.0 * cfg->epsilon) continue;
    const double* c = corrs + 6 * (size_t)pre->kept[k];
    double ang;
    if (rvo_correspondence_angle(est->axis, c, c + 3, cfg->tau_deg, &ang) != RVO_OK) continue;
    if (fabs(remainder(ang - est->angle, 2.0 * RVO_PI)) >= 0.1) continue;
    if (want_band) s.band[s.nband++] = d;
    if (d < cfg->epsilon) ++s.coherent;
  }
  return s;
}

/* anneal_axis, estimator.cpp:145-160 */
static void anneal_axis(double axis[3], double eps0, const pre_t* pre, const rvo_config* cfg, int32_t* buf) {
  double e = eps0 > cfg->epsilon ? eps0 : cfg->epsilon;
  for (;;) {
    const int64_t m = rvo_classify_inliers(axis, pre->z, pre->n, e, buf);
    if (m >= 2) {
      double next[3];
      if (refine_axis_idx(pre->z, buf, m, next) == RVO_OK) {
        axis[0] = next[0];
        axis[1] = next[1];
        axis[2] = next[2];
      }
    }
    if (e <= cfg->epsilon) break;
    const double h = 0.5 * e;
    e = cfg->epsilon > h ? cfg->epsilon : h;
  }
}

/* rescue_axes, estimator.cpp:162-179. axes sized >= 6. Returns count. */
static int rescue_axes(const uint32_t* counts, const pre_t* pre, const rvo_config* cfg, double axes[6][3],
                       int32_t* buf) {
  int na = 0;
  const int ws[5] = {4, 8, 16, 32, 64};
  const double cs = 2.0 * cfg->extent / cfg->grid;
  for (int i = 0; i < 5; ++i) {
    const int w = ws[i];
    if (2 * w + 1 > cfg->grid) break;
    rvo_peak p;
    rvo_blurred_argmax(counts, cfg->grid, cfg->extent, w, &p);
    double b[3], start[3];
    rvo_backproject_peak(p.A, p.B, b);
    canonicalize3(b, start);
    anneal_axis(start, w * cs, pre, cfg, buf);
    axes[na][0] = start[0];
    axes[na][1] = start[1];
    axes[na][2] = start[2];
    ++na;
  }
  double ls[3];
  if (rvo_refine_axis(pre->z, pre->n, ls) == RVO_OK) {
    anneal_axis(ls, 0.25, pre, cfg, buf);
    axes[na][0] = ls[0];
    axes[na][1] = ls[1];
    axes[na][2] = ls[2];
    ++na;
  }
  return na;
}

/* build_candidate, estimator.cpp:183-194 */
static int build_candidate(const double start[3], const uint32_t* counts, const double* corrs, const pre_t* pre,
                           const rvo_config* cfg, int32_t* inl, int32_t* tmp, rvo_estimate* out) {
  double axis[3] = {start[0], start[1], start[2]};
  const int64_t m = refine_loop(axis, pre, cfg, inl, tmp, NULL);
  uint32_t votes = 0;
  double A, B;
  if (project3(axis, &A, &B) == RVO_OK) {
    const int ix = rvo_coord_to_cell(A, cfg->grid, cfg->extent);
    const int iy = rvo_coord_to_cell(B, cfg->grid, cfg->extent);
    votes = counts[(size_t)iy * cfg->grid + ix];
  }
  return build_estimate(axis, inl, m, votes, corrs, pre, cfg, out);
}

static void pre_free(pre_t* p) {
  free(p->z);
  free(p->kept);
  free(p->dropped);
}

static int run_preprocess(const double* corrs, int64_t n, const rvo_config* cfg, pre_t* pre) {
  pre->z = (double*)malloc(sizeof(double) * 3 * (size_t)(n > 0 ? n : 1));
  pre->kept = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
  pre->dropped = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
  if (!pre->z || !pre->kept || !pre->dropped) return RVO_OUT_OF_MEMORY;
  return rvo_preprocess(corrs, n, cfg->tau_z, cfg->normalize_inputs, pre->z, pre->kept, pre->dropped, &pre->n,
                        &pre->nd);
}

static int identity_estimate(const int32_t* idx, int64_t m, rvo_estimate* out) { /* estimator.cpp:251-255 */
  est_clear(out);
  out->inliers = (int32_t*)malloc(sizeof(int32_t) * (size_t)(m > 0 ? m : 1));
  if (!out->inliers) return RVO_OUT_OF_MEMORY;
  memcpy(out->inliers, idx, sizeof(int32_t) * (size_t)m);
  out->n_inliers = m;
  return RVO_OK;
}

int rvo_estimate_single(const double* corrs, int64_t n, const rvo_config* cfg,
                        rvo_estimate* out) { /* estimator.cpp:320-371 */
  memset(&g_trace, 0, sizeof g_trace);
  g_trace.rescue_won = -1;
  est_clear(out);
  if (n <= 0) return RVO_EMPTY_INPUT;
  pre_t pre = {0};
  int st = run_preprocess(corrs, n, cfg, &pre);
  g_trace.n_kept = pre.n;
  g_trace.n_dropped = pre.nd;
  if (st == RVO_ALL_DEGENERATE) {
    int32_t* all = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
    for (int64_t i = 0; i < n; ++i) all[i] = (int32_t)i;
    st = identity_estimate(all, n, out);
    free(all);
    pre_free(&pre);
    return st;
  }
  if (st != RVO_OK) {
    pre_free(&pre);
    return st;
  }
  if (pre.nd * 10 >= n * 9) { /* :336-340 */
    st = identity_estimate(pre.dropped, pre.nd, out);
    pre_free(&pre);
    return st;
  }
  const int g = cfg->grid;
  uint32_t* counts = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)g * g);
  int32_t* inl = (int32_t*)malloc(sizeof(int32_t) * (size_t)pre.n);
  int32_t* tmp = (int32_t*)malloc(sizeof(int32_t) * (size_t)pre.n);
  if (!counts || !inl || !tmp) {
    st = RVO_OUT_OF_MEMORY;
    goto done;
  }
  st = rvo_accumulate(pre.z, pre.n, g, cfg->extent, cfg->theta_samples, counts);
  if (st != RVO_OK) goto done;
  rvo_peak pk;
  int32_t np = 0;
  st = rvo_find_peaks(counts, g, cfg->extent, 1, cfg->suppression_radius, 1, &pk, &np);
  if (st != RVO_OK) goto done;
  g_trace.peak_ix = pk.ix;
  g_trace.peak_iy = pk.iy;
  g_trace.peak_votes = pk.votes;
  { /* estimate_from_peak, estimator.cpp:94-101 */
    double A, B, b[3], axis[3];
    interpolate_peak(counts, g, cfg->extent, &pk, &A, &B);
    rvo_backproject_peak(A, B, b);
    canonicalize3(b, axis);
    memcpy(g_trace.start_axis, axis, sizeof axis);
    const int64_t m = refine_loop(axis, &pre, cfg, inl, tmp, &g_trace.refine_passes);
    st = build_estimate(axis, inl, m, pk.votes, corrs, &pre, cfg, out);
    if (st != RVO_OK) goto done;
  }
  {
    const double chance = cfg->epsilon * (double)pre.n;
    if (cfg->refine && (double)out->n_inliers < 3.0 * chance) { /* :352-368 */
      g_trace.rescued = 1;
      support_t s0 = model_support(out, corrs, &pre, cfg, 0);
      int64_t best = s0.coherent;
      double axes[6][3];
      const int na = rescue_axes(counts, &pre, cfg, axes, inl);
      for (int a = 0; a < na; ++a) {
        rvo_estimate cand;
        est_clear(&cand);
        const int cst = build_candidate(axes[a], counts, corrs, &pre, cfg, inl, tmp, &cand);
        if (cst == RVO_NO_VOTES) continue;
        if (cst != RVO_OK) {
          st = cst;
          goto done;
        }
        support_t s = model_support(&cand, corrs, &pre, cfg, 0);
        if (s.coherent > best) {
          best = s.coherent;
          free(out->inliers);
          *out = cand;
          g_trace.rescue_won = a;
        } else {
          free(cand.inliers);
        }
      }
    }
  }
done:
  free(counts);
  free(inl);
  free(tmp);
  pre_free(&pre);
  return st;
}

/* ---- estimate_multi and its near-identity fallback ------------------------------------ */

/* 3x3 SVD by two-sided Jacobi (restating Eigen's JacobiSVD for real 3x3: per pair a 2x2
 * real SVD from two plane rotations). Only the Kabsch fallback uses it (estimator.cpp:198-215);
 * parity there is to tolerance. a,u,v row-major. */
static void jacobi_svd3(const double a[9], double u[9], double v[9]) {
  double w[3][3], U[3][3], V[3][3];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      w[i][j] = a[i * 3 + j];
      U[i][j] = V[i][j] = (i == j) ? 1.0 : 0.0;
    }
  const double prec = 2.0 * DBL_EPSILON;
  double max_diag = 0;
  for (int i = 0; i < 3; ++i)
    if (fabs(w[i][i]) > max_diag) max_diag = fabs(w[i][i]);
  int finished = 0, sweeps = 0;
  while (!finished && sweeps < 100) {
    finished = 1;
    ++sweeps;
    for (int p = 1; p < 3; ++p)
      for (int q = 0; q < p; ++q) {
        const double thr = prec * max_diag > 4.9e-324 ? prec * max_diag : 4.9e-324;
        if (fabs(w[p][q]) > thr || fabs(w[q][p]) > thr) {
          finished = 0;
          const double m00 = w[q][q], m01 = w[q][p], m10 = w[p][q], m11 = w[p][p];
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
          double jc = 1, js = 0; /* symmetric 2x2 Jacobi of [n00 n01; n01 n11] */
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
          /* jl = rot1 * jr^T */
          const double lc = c1 * jc - s1 * (-js), ls = c1 * (-js) + s1 * jc;
          for (int k = 0; k < 3; ++k) { /* rows q,p of w from the left */
            const double x = w[q][k], y = w[p][k];
            w[q][k] = lc * x + ls * y;
            w[p][k] = -ls * x + lc * y;
          }
          for (int k = 0; k < 3; ++k) { /* U = U * jl^T */
            const double x = U[k][q], y = U[k][p];
            U[k][q] = lc * x + ls * y;
            U[k][p] = -ls * x + lc * y;
          }
          for (int k = 0; k < 3; ++k) { /* w = w * jr, V = V * jr */
            double x = w[k][q], y = w[k][p];
            w[k][q] = jc * x - js * y;
            w[k][p] = js * x + jc * y;
            x = V[k][q];
            y = V[k][p];
            V[k][q] = jc * x - js * y;
            V[k][p] = js * x + jc * y;
          }
          const double mp = fabs(w[p][p]) > fabs(w[q][q]) ? fabs(w[p][p]) : fabs(w[q][q]);
          if (mp > max_diag) max_diag = mp;
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
      const double t = sv[i];
      sv[i] = sv[best];
      sv[best] = t;
      for (int k = 0; k < 3; ++k) {
        double x = U[k][i];
        U[k][i] = U[k][best];
        U[k][best] = x;
        x = V[k][i];
        V[k][i] = V[k][best];
        V[k][best] = x;
      }
    }
  }
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      u[i * 3 + j] = U[i][j];
      v[i * 3 + j] = V[i][j];
    }
}

static void mat3_mul(const double* a, const double* b, double* o) {
  double t[9];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) t[i * 3 + j] = a[i * 3 + 0] * b[0 * 3 + j] + a[i * 3 + 1] * b[1 * 3 + j] + a[i * 3 + 2] * b[2 * 3 + j];
  memcpy(o, t, sizeof t);
}
static void mat3_t(const double* a, double* o) {
  double t[9];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) t[j * 3 + i] = a[i * 3 + j];
  memcpy(o, t, sizeof t);
}
static double det3(const double* m) { /* column expansion, as the shim */
  return m[0] * (m[4] * m[8] - m[7] * m[5]) - m[3] * (m[1] * m[8] - m[7] * m[2]) + m[6] * (m[1] * m[5] - m[4] * m[2]);
}

/* fit_rotation (Kabsch), estimator.cpp:198-215 */
static void fit_rotation(const double* corrs, const int32_t* idx, int64_t m, int normalize, double r[9]) {
  double h[9] = {0};
  for (int64_t k = 0; k < m; ++k) {
    double x[3], y[3];
    memcpy(x, corrs + 6 * (size_t)idx[k], sizeof x);
    memcpy(y, corrs + 6 * (size_t)idx[k] + 3, sizeof y);
    if (normalize) {
      const double nx = norm3(x), ny = norm3(y);
      if (nx > 0.0) { x[0] /= nx; x[1] /= nx; x[2] /= nx; }
      if (ny > 0.0) { y[0] /= ny; y[1] /= ny; y[2] /= ny; }
    }
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) h[i * 3 + j] += y[i] * x[j];
  }
  double u[9], v[9], vt[9], uvt[9], d[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
  jacobi_svd3(h, u, v);
  mat3_t(v, vt);
  mat3_mul(u, vt, uvt);
  d[8] = det3(uvt) < 0.0 ? -1.0 : 1.0;
  double ud[9];
  mat3_mul(u, d, ud);
  mat3_mul(ud, vt, r);
}

/* near_identity_model, estimator.cpp:224-249. sub_kept: input indices of the residual. */
static int near_identity_model(const double* corrs, const int32_t* sub_kept, int64_t nsub, const rvo_config* cfg,
                               int64_t min_cluster, rvo_estimate* out) {
  int32_t* cluster = (int32_t*)malloc(sizeof(int32_t) * (size_t)(nsub > 0 ? nsub : 1));
  int64_t nc = 0;
  for (int64_t k = 0; k < nsub; ++k) {
    const int32_t i = sub_kept[k];
    double x[3], y[3];
    memcpy(x, corrs + 6 * (size_t)i, sizeof x);
    memcpy(y, corrs + 6 * (size_t)i + 3, sizeof y);
    if (cfg->normalize_inputs) {
      const double nx = norm3(x), ny = norm3(y);
      if (nx > 0.0) { x[0] /= nx; x[1] /= nx; x[2] /= nx; }
      if (ny > 0.0) { y[0] /= ny; y[1] /= ny; y[2] /= ny; }
    }
    const double d[3] = {y[0] - x[0], y[1] - x[1], y[2] - x[2]};
    if (norm3(d) < 0.1) cluster[nc++] = i;
  }
  const int64_t need = min_cluster > 3 ? min_cluster : 3;
  if (nc < need) {
    free(cluster);
    return 0;
  }
  double r[9];
  fit_rotation(corrs, cluster, nc, cfg->normalize_inputs, r);
  /* AngleAxisd(r) via Quaternion(r) (Eigen quaternionbase_assign_impl + AngleAxis from quaternion) */
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
    aa_angle = 2.0 * atan2(n, fabs(qw));
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
  est_clear(out);
  canonicalize3(aa_axis, out->axis);
  out->angle = dot3(out->axis, aa_axis) < 0.0 ? -aa_angle : aa_angle;
  memcpy(out->rotation, r, sizeof r);
  out->inliers = cluster;
  out->n_inliers = nc;
  out->axis_votes = (uint32_t)nc;
  return 1;
}

static int cmp_double(const void* a, const void* b) {
  const double x = *(const double*)a, y = *(const double*)b;
  return (x > y) - (x < y);
}

int rvo_estimate_multi(const double* corrs, int64_t n, const rvo_config* cfg, rvo_estimate* out,
                       int32_t* n_models) { /* estimator.cpp:373-493 */
  *n_models = 0;
  if (n <= 0) return RVO_EMPTY_INPUT;
  pre_t pre = {0};
  int st = run_preprocess(corrs, n, cfg, &pre);
  if (st != RVO_OK) {
    pre_free(&pre);
    return st;
  }
  const double chance = cfg->epsilon * (double)pre.n;
  const double cf = cfg->consensus_floor_mult * chance;
  const int64_t consensus_floor = (int64_t)(cf > 2.0 ? cf : 2.0);
  const int g = cfg->grid;
  uint8_t* removed = (uint8_t*)calloc((size_t)(pre.n > 0 ? pre.n : 1), 1);
  pre_t sub = {0};
  sub.z = (double*)malloc(sizeof(double) * 3 * (size_t)(pre.n > 0 ? pre.n : 1));
  sub.kept = (int32_t*)malloc(sizeof(int32_t) * (size_t)(pre.n > 0 ? pre.n : 1));
  uint32_t* counts = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)g * g);
  int32_t* inl = (int32_t*)malloc(sizeof(int32_t) * (size_t)(pre.n > 0 ? pre.n : 1));
  int32_t* tmp = (int32_t*)malloc(sizeof(int32_t) * (size_t)(pre.n > 0 ? pre.n : 1));
  int nm = 0;
  st = RVO_OK;
  while (nm < cfg->max_models) {
    sub.n = 0;
    for (int64_t k = 0; k < pre.n; ++k) {
      if (removed[k]) continue;
      memcpy(sub.z + 3 * sub.n, pre.z + 3 * k, sizeof(double) * 3);
      sub.kept[sub.n++] = pre.kept[k];
    }
    if (sub.n < (consensus_floor > 2 ? consensus_floor : 2)) break;
    st = rvo_accumulate(sub.z, sub.n, g, cfg->extent, cfg->theta_samples, counts);
    if (st != RVO_OK) break;
    rvo_peak pk;
    int32_t np = 0;
    const int have_peak =
        rvo_find_peaks(counts, g, cfg->extent, 1, cfg->suppression_radius, rvo_peak_vote_floor(cfg, sub.n), &pk, &np) ==
        RVO_OK;
    rvo_estimate est;
    est_clear(&est);
    support_t sup = {0, NULL, 0};
    int have = 0;
    if (have_peak) {
      double starts[7][3];
      int ns = 0;
      double A, B, b[3];
      interpolate_peak(counts, g, cfg->extent, &pk, &A, &B);
      rvo_backproject_peak(A, B, b);
      canonicalize3(b, starts[ns++]);
      double axes[6][3];
      const int na = rescue_axes(counts, &sub, cfg, axes, inl);
      for (int a = 0; a < na; ++a) memcpy(starts[ns++], axes[a], sizeof(double) * 3);
      for (int s = 0; s < ns; ++s) {
        rvo_estimate cand;
        est_clear(&cand);
        const int cst = build_candidate(starts[s], counts, corrs, &pre, cfg, inl, tmp, &cand);
        if (cst == RVO_NO_VOTES) continue;
        if (cst != RVO_OK) {
          st = cst;
          goto done;
        }
        if (s == 0) cand.axis_votes = pk.votes;
        support_t cs = model_support(&cand, corrs, &pre, cfg, 1);
        if (!have || cs.coherent > sup.coherent) {
          free(est.inliers);
          free(sup.band);
          est = cand;
          sup = cs;
          have = 1;
        } else {
          free(cand.inliers);
          free(cs.band);
        }
      }
    }
    int identity_model = 0;
    const int64_t need_coh = (est.n_inliers / 5) > 8 ? (est.n_inliers / 5) : 8;
    const int valid = have && est.n_inliers >= consensus_floor && sup.coherent >= need_coh;
    if (!valid) {
      rvo_estimate ident;
      if (!near_identity_model(corrs, sub.kept, sub.n, cfg, consensus_floor, &ident)) {
        free(est.inliers);
        free(sup.band);
        break;
      }
      free(est.inliers);
      est = ident;
      identity_model = 1;
    }
    int duplicate = 0; /* set_intersection of ascending inlier lists */
    for (int mi = 0; mi < nm && !duplicate; ++mi) {
      int64_t a = 0, b = 0, common = 0;
      const rvo_estimate* e = &out[mi];
      while (a < e->n_inliers && b < est.n_inliers) {
        if (e->inliers[a] < est.inliers[b]) ++a;
        else if (est.inliers[b] < e->inliers[a]) ++b;
        else { ++common; ++a; ++b; }
      }
      if ((double)common > cfg->dedupe_overlap * (double)est.n_inliers) duplicate = 1;
    }
    if (duplicate) {
      free(est.inliers);
      free(sup.band);
      break;
    }
    if (identity_model) {
      uint8_t* member = (uint8_t*)calloc((size_t)n, 1);
      for (int64_t k = 0; k < est.n_inliers; ++k) member[est.inliers[k]] = 1;
      for (int64_t k = 0; k < pre.n; ++k)
        if (member[pre.kept[k]]) removed[k] = 1;
      free(member);
    } else {
      double strip = 2.0 * cfg->epsilon;
      if (sup.nband > 0) {
        const int64_t q0 = (sup.nband * 95) / 100;
        const int64_t q = (sup.nband - 1) < q0 ? (sup.nband - 1) : q0;
        qsort(sup.band, (size_t)sup.nband, sizeof(double), cmp_double); /* nth_element value */
        const double v = 1.25 * sup.band[q];
        strip = strip > v ? strip : v;
      }
      for (int64_t k = 0; k < pre.n; ++k)
        if (fabs(dot3(est.axis, pre.z + 3 * k)) < strip) removed[k] = 1;
    }
    free(sup.band);
    out[nm++] = est;
  }
  if (nm == 0 && st == RVO_OK) st = RVO_NO_PEAK;
  if (st == RVO_OK) { /* stable_sort by axis_votes descending (insertion sort is stable) */
    for (int i = 1; i < nm; ++i) {
      rvo_estimate key = out[i];
      int j = i - 1;
      while (j >= 0 && out[j].axis_votes < key.axis_votes) {
        out[j + 1] = out[j];
        --j;
      }
      out[j + 1] = key;
    }
  }
done:
  *n_models = nm;
  free(removed);
  free(sub.z);
  free(sub.kept);
  free(counts);
  free(inl);
  free(tmp);
  pre_free(&pre);
  return st;
}
