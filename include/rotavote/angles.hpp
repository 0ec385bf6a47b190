// Drop-in for proj/include/rotavote/angles.hpp (angles.hpp:11-51). vote_angles and peak_angle
// run on the device (angles.cpp:46-90); correspondence_angle is the host formula.
#pragma once

#include <cmath>
#include <cstdint>
#include <numbers>
#include <span>
#include <vector>

#include "device.hpp"
#include "geom.hpp"

namespace rotavote {

struct Correspondence {
  Vec3 x;
  Vec3 y;
};

struct AngleHistogram {
  std::vector<std::uint32_t> bins;
  std::uint64_t contributing = 0;
  std::uint64_t degenerate = 0;
  std::vector<double> raw_angles;

  int bin_count() const { return static_cast<int>(bins.size()); }
  double bin_width() const { return 2.0 * std::numbers::pi / bin_count(); }
  int bin_of(double angle) const {  // angles.cpp:25-30
    const int n = bin_count();
    const int k = static_cast<int>(std::ceil((angle + std::numbers::pi) / bin_width())) - 1;
    return k < 0 ? 0 : (k > n - 1 ? n - 1 : k);
  }
  double bin_center(int k) const { return -std::numbers::pi + (k + 0.5) * bin_width(); }
};

namespace detail {
// A span of Correspondence IS the C-ABI's n x 6 f64 row layout (Eigen::Vector3d holds 3 doubles,
// no padding): it is passed straight through, no host copy.
static_assert(sizeof(Vec3) == 3 * sizeof(double) && sizeof(Correspondence) == 6 * sizeof(double),
              "Correspondence must be 6 contiguous doubles");
inline const double* rows(std::span<const Correspondence> c) {
  return c.empty() ? nullptr : reinterpret_cast<const double*>(c.data());
}
}  // namespace detail

inline double correspondence_angle(const Vec3& axis, const Vec3& x, const Vec3& y, double tau = 1e-6) {
  double a[3], xx[3], yy[3], out;
  detail::to3(axis, a);
  detail::to3(x, xx);
  detail::to3(y, yy);
  if (rv_correspondence_angle(a, xx, yy, tau, &out) != RV_OK)
    throw DegenerateProjection("correspondence parallel to the rotation axis");
  return out;
}

inline AngleHistogram vote_angles(const Vec3& axis, std::span<const Correspondence> correspondences,
                                  std::span<const int> indices, int bin_count, double tau = 1e-6) {
  AngleHistogram h;
  if (bin_count < 8) throw InvalidConfig("angle histogram needs bin_count >= 8");
  h.bins.assign(static_cast<std::size_t>(bin_count), 0u);
  h.raw_angles.resize(indices.size());
  double a[3];
  detail::to3(axis, a);
  const double* flat = detail::rows(correspondences);
  std::vector<int32_t> idx(indices.begin(), indices.end());
  uint64_t contrib = 0, degen = 0;
  detail::check(rv_vote_angles(detail::context(), a, flat, static_cast<int64_t>(correspondences.size()),
                               idx.data(), static_cast<int64_t>(idx.size()), bin_count, tau, h.bins.data(), &contrib,
                               &degen, h.raw_angles.data()));
  h.contributing = contrib;
  h.degenerate = degen;
  h.raw_angles.resize(contrib);
  return h;
}

inline double peak_angle(const AngleHistogram& hist, bool refine, std::span<const double> raw_angles) {
  double out = 0;
  detail::check(rv_peak_angle(detail::context(), hist.bins.data(), hist.bin_count(), hist.contributing, refine ? 1 : 0,
                              raw_angles.data(), static_cast<int64_t>(raw_angles.size()), &out));
  return out;
}

inline double peak_angle(const AngleHistogram& hist, bool refine) { return peak_angle(hist, refine, hist.raw_angles); }

}  // namespace rotavote
