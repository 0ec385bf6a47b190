// Drop-in for proj/include/rotavote/voting.hpp (voting.hpp:14-85): Accumulator2D, Peak,
// PeakSet and the voting functions, with accumulate / find_peaks / blurred_argmax /
// deposit_circle_votes executed by the sm_100a kernels of librotavote_b200 (bit-exact with the
// reference's sampled-deposit semantics, voting.cpp:17-216).
#pragma once

#include <charconv>
#include <cmath>
#include <functional>
#include <cstdint>
#include <algorithm>
#include <ostream>
#include <numbers>
#include <numeric>
#include <span>
#include <string>
#include <vector>

#include "device.hpp"
#include "geom.hpp"

namespace rotavote {

class Accumulator2D {
 public:
  Accumulator2D(int grid, double extent)
      : grid_(grid), extent_(extent), counts_(static_cast<std::size_t>(grid > 0 ? grid : 0) * (grid > 0 ? grid : 0), 0u) {
    if (grid < 1 || extent <= 0.0) throw InvalidConfig("accumulator needs grid >= 1, extent > 0");
  }
  int grid() const { return grid_; }
  double extent() const { return extent_; }
  double cell_size() const { return 2.0 * extent_ / grid_; }
  int coord_to_cell(double v) const {  // voting.cpp:17-23
    const double t = (v + extent_) * (grid_ / (2.0 * extent_));
    const double f = std::floor(t);
    int i = static_cast<int>(f);
    if (f == t && i > 0) --i;
    return i < 0 ? 0 : (i > grid_ - 1 ? grid_ - 1 : i);
  }
  PlanePoint cell_center(int ix, int iy) const {  // centre of a cell: -E + (i + 1/2) * cell size
    auto c = [this](int i) { return -extent_ + (i + 0.5) * cell_size(); };
    return {c(ix), c(iy)};
  }
  std::uint32_t& at(int ix, int iy) { return counts_[static_cast<std::size_t>(iy) * grid_ + ix]; }
  std::uint32_t at(int ix, int iy) const { return counts_[static_cast<std::size_t>(iy) * grid_ + ix]; }
  std::span<const std::uint32_t> counts() const { return counts_; }
  std::span<std::uint32_t> counts() { return counts_; }
  std::uint64_t total() const {  // 64-bit sum of all cells
    std::uint64_t t = 0;
    for (std::uint32_t c : counts_) t += c;
    return t;
  }
  void add(const Accumulator2D& other) {  // cell-wise sum (same grid)
    std::transform(counts_.begin(), counts_.end(), other.counts_.begin(), counts_.begin(), std::plus<std::uint32_t>());
  }

 private:
  int grid_;
  double extent_;
  std::vector<std::uint32_t> counts_;
};

struct Peak {
  int ix = 0;
  int iy = 0;
  PlanePoint center;
  std::uint32_t votes = 0;
};

struct PeakSet {
  std::vector<Peak> peaks;
  int suppression_radius = 0;
};

// Interleaved (cos, sin) of the J circle samples theta_j = -pi + j * (2 pi / J) (voting.cpp:72-81).
// The angle expression and host libm cos/sin are what the reference evaluates -- any other
// formula would move sample values by an ulp and change boundary cells.
inline std::vector<double> circle_sample_table(int samples) {
  std::vector<double> cs;
  cs.reserve(2 * static_cast<std::size_t>(samples));
  const double dtheta = 2.0 * std::numbers::pi / samples;
  for (int j = 0; j < samples; ++j) {
    const double a = -std::numbers::pi + j * dtheta;
    cs.push_back(std::cos(a));
    cs.push_back(std::sin(a));
  }
  return cs;
}

inline void deposit_circle_votes(const Vec3& z, Accumulator2D& acc, int samples) {
  double zz[3];
  detail::to3(z, zz);
  detail::check(rv_deposit_circle_votes(detail::context(), zz, acc.counts().data(), acc.grid(), acc.extent(), samples));
}

inline Accumulator2D accumulate(std::span<const Vec3> constraints, int grid, double extent, int samples,
                                int threads = 1) {
  (void)threads;  // the result is independent of host threads, like the reference's; the device
                  // fan-out is ROTAVOTE_DEVICES (detail::multi)
  if (constraints.empty()) throw EmptyInput("no constraints to accumulate");
  Accumulator2D acc(grid, extent);
  std::vector<double> z(3 * constraints.size());
  for (std::size_t i = 0; i < constraints.size(); ++i) detail::to3(constraints[i], z.data() + 3 * i);
  if (rv_multi* m = detail::multi()) {  // ROTAVOTE_DEVICES: chunks over several GPUs (voting.cpp:95-117)
    detail::check_multi(rv_multi_accumulate(m, z.data(), static_cast<int64_t>(constraints.size()), grid, extent,
                                            samples, acc.counts().data()));
    return acc;
  }
  detail::check(rv_accumulate(detail::context(), z.data(), static_cast<int64_t>(constraints.size()), grid, extent,
                              samples, acc.counts().data()));
  return acc;
}

inline PeakSet find_peaks(const Accumulator2D& acc, int max_peaks, int suppression_radius, std::uint32_t min_votes) {
  PeakSet out;
  out.suppression_radius = suppression_radius;
  if (max_peaks < 1) throw NoPeak("no accumulator cell reaches min_votes");
  std::vector<rv_peak> ps(static_cast<std::size_t>(max_peaks));
  int32_t n = 0;
  detail::check(rv_find_peaks(detail::context(), acc.counts().data(), acc.grid(), acc.extent(), max_peaks,
                              suppression_radius, min_votes, ps.data(), &n));
  for (int k = 0; k < n; ++k) out.peaks.push_back(Peak{ps[k].ix, ps[k].iy, {ps[k].A, ps[k].B}, ps[k].votes});
  return out;
}

inline Vec3 backproject_peak(const PlanePoint& center) { return unproject(center).normalized(); }

inline Peak blurred_argmax(const Accumulator2D& acc, int radius) {
  rv_peak p;
  detail::check(rv_blurred_argmax(detail::context(), acc.counts().data(), acc.grid(), acc.extent(), radius, &p));
  return Peak{p.ix, p.iy, {p.A, p.B}, p.votes};
}

// Dump formats (voting.hpp:83-84, plot-ready host formatting; the byte layout of
// voting.cpp:218-239): text = one grid row per line, counts separated by single spaces;
// PGM = binary P5 header, then every count rescaled to 0..255 against the grid maximum
// (integer floor of count*255/max; all zero when the grid is empty).
inline void dump_accumulator_text(const Accumulator2D& acc, std::ostream& out) {
  const auto v = acc.counts();
  const std::size_t g = static_cast<std::size_t>(acc.grid());
  std::string row;
  char num[16];
  for (std::size_t r = 0; r < g; ++r) {
    row.clear();
    for (std::size_t k = 0; k < g; ++k) {
      const auto res = std::to_chars(num, num + sizeof num, v[r * g + k]);
      if (k) row.push_back(' ');
      row.append(num, res.ptr);
    }
    row.push_back('\n');
    out.write(row.data(), static_cast<std::streamsize>(row.size()));
  }
}

inline void dump_accumulator_pgm(const Accumulator2D& acc, std::ostream& out) {
  const auto v = acc.counts();
  const std::uint64_t top = v.empty() ? 0u : *std::max_element(v.begin(), v.end());
  std::vector<unsigned char> px(v.size(), 0u);
  if (top)
    std::transform(v.begin(), v.end(), px.begin(),
                   [top](std::uint32_t c) { return static_cast<unsigned char>(std::uint64_t{c} * 255u / top); });
  const std::string head = "P5\n" + std::to_string(acc.grid()) + " " + std::to_string(acc.grid()) + "\n255\n";
  out.write(head.data(), static_cast<std::streamsize>(head.size()));
  out.write(reinterpret_cast<const char*>(px.data()), static_cast<std::streamsize>(px.size()));
}

}  // namespace rotavote
