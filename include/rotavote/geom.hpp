// Drop-in for proj/include/rotavote/geom.hpp: same types and signatures (geom.hpp:9-43).
// Vec3/Mat3 are Eigen types as in the reference; the arithmetic runs in librotavote_b200
// (host formulas identical to geom.cpp:10-43).
#pragma once

#include <Eigen/Core>
#include <Eigen/Geometry>
#include <utility>

#include "../rotavote_b200.h"
#include "errors.hpp"

namespace rotavote {

using Vec3 = Eigen::Vector3d;
using Mat3 = Eigen::Matrix3d;

struct PlanePoint {
  double A = 0.0;
  double B = 0.0;
};

struct AxisAngle {
  Vec3 axis;
  double angle;
};

namespace detail {
inline void to3(const Vec3& v, double* o) {
  o[0] = v(0);
  o[1] = v(1);
  o[2] = v(2);
}
inline Vec3 from3(const double* o) { return Vec3(o[0], o[1], o[2]); }
inline void to9(const Mat3& m, double* o) {  // row-major
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) o[i * 3 + j] = m(i, j);
}
inline Mat3 from9(const double* o) {
  Mat3 m;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) m(i, j) = o[i * 3 + j];
  return m;
}
}  // namespace detail

inline Mat3 rodrigues(const Vec3& axis, double angle) {
  double a[3], r[9];
  detail::to3(axis, a);
  rv_rodrigues(a, angle, r);
  return detail::from9(r);
}
inline Mat3 rodrigues(const AxisAngle& aa) { return rodrigues(aa.axis, aa.angle); }

inline double rotation_error(const Mat3& r_gt, const Mat3& r_opt) {
  double a[9], b[9];
  detail::to9(r_gt, a);
  detail::to9(r_opt, b);
  return rv_rotation_error(a, b);
}

inline PlanePoint project(const Vec3& p) {
  double a[3];
  detail::to3(p, a);
  PlanePoint q;
  const rv_status st = rv_project(a, &q.A, &q.B);
  if (st != RV_OK) throw PoleProximity("point too close to the projection pole (0,0,1)");
  return q;
}

inline Vec3 unproject(const PlanePoint& q) {
  double o[3];
  rv_unproject(q.A, q.B, o);
  return detail::from3(o);
}

inline Vec3 canonicalize(const Vec3& p) {
  double a[3], o[3];
  detail::to3(p, a);
  rv_canonicalize(a, o);
  return detail::from3(o);
}

inline std::pair<Vec3, Vec3> orthonormal_basis(const Vec3& z) {
  double a[3], a1[3], a2[3];
  detail::to3(z, a);
  rv_orthonormal_basis(a, a1, a2);
  return {detail::from3(a1), detail::from3(a2)};
}

}  // namespace rotavote
