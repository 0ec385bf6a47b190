// End-to-end timing of the drop-in C++ API on PAGEABLE host memory -- what a user of the
// reference does: rotavote::estimate_single(std::span<const Correspondence>, cfg)
// (proj/include/rotavote/estimator.hpp:63-64) on a std::vector<Correspondence> they filled.
// Usage: e2e_pageable <rows.f64> <n> <steps> <warmup>   (rows: n x 6 little-endian doubles)
// Every step gets a FRESH vector (allocated and filled outside the timed region); the timed call
// includes the pageable H2D, the solve and the inlier list back in a std::vector. Prints one JSON
// line. With ROTAVOTE_DEVICES set it runs the multi-GPU route.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <vector>

#include "rotavote/estimator.hpp"

int main(int argc, char** argv) {
  if (argc < 5) {
    std::fprintf(stderr, "usage: %s rows.f64 n steps warmup\n", argv[0]);
    return 2;
  }
  const long n = std::atol(argv[2]);
  const int steps = std::atoi(argv[3]), warmup = std::atoi(argv[4]);
  std::vector<double> raw(static_cast<size_t>(n) * 6);
  std::ifstream f(argv[1], std::ios::binary);
  f.read(reinterpret_cast<char*>(raw.data()), static_cast<std::streamsize>(raw.size() * sizeof(double)));
  if (!f) {
    std::fprintf(stderr, "short read\n");
    return 2;
  }
  rotavote::EstimatorConfig cfg;
  std::vector<double> ms;
  size_t inl = 0;
  for (int s = 0; s < warmup + steps; ++s) {
    std::vector<rotavote::Correspondence> v(static_cast<size_t>(n));
    for (long i = 0; i < n; ++i) {
      const double* r = raw.data() + 6 * i;
      v[static_cast<size_t>(i)].x = rotavote::Vec3(r[0], r[1], r[2]);
      v[static_cast<size_t>(i)].y = rotavote::Vec3(r[3], r[4], r[5]);
    }
    const auto t0 = std::chrono::steady_clock::now();
    const rotavote::RotationEstimate e = rotavote::estimate_single(v, cfg);
    const auto t1 = std::chrono::steady_clock::now();
    inl = e.inliers.size();
    if (s >= warmup) ms.push_back(std::chrono::duration<double, std::milli>(t1 - t0).count());
  }
  double tot = 0;
  for (double x : ms) tot += x;
  const double per = tot / ms.size();
  std::printf("{\"ms_per_step\": %.6f, \"value\": %.3f, \"inliers\": %zu, \"steps\": %d}\n", per, n / (per * 1e-3),
              inl, steps);
  return 0;
}
