// Drop-in for proj/include/rotavote/estimator.hpp (estimator.hpp:13-70): same configuration,
// result types and solver signatures; the solve runs in librotavote_b200 (C++ host control flow
// + sm_100a kernels) through the C-ABI.
#pragma once

#include <cstdint>
#include <span>
#include <vector>

#include "angles.hpp"
#include "device.hpp"
#include "geom.hpp"
#include "voting.hpp"

namespace rotavote {

struct EstimatorConfig {
  int grid = 512;
  double extent = 1.05;
  int theta_samples = 2048;
  double epsilon = 0.015;
  int angle_bins = 1024;
  int max_models = 1;
  double min_votes_frac = 0.02;
  double consensus_floor_mult = 1.5;
  double dedupe_overlap = 0.5;
  double tau_z = 1e-9;
  double tau_deg = 1e-6;
  int suppression_radius = 8;
  bool refine = true;
  bool normalize_inputs = true;
  int threads = 1;
};

struct RotationEstimate {
  Vec3 axis = Vec3(0, 0, -1);
  double angle = 0.0;
  Mat3 rotation = Mat3::Identity();
  std::vector<int> inliers;
  std::uint32_t axis_votes = 0;
  double elapsed_s = 0.0;
};

struct PreprocessResult {
  std::vector<Vec3> constraints;
  std::vector<int> kept;
  std::vector<int> dropped;
};

namespace detail {
inline rv_config to_c(const EstimatorConfig& e) {
  rv_config c;
  c.grid = e.grid;
  c.extent = e.extent;
  c.theta_samples = e.theta_samples;
  c.epsilon = e.epsilon;
  c.angle_bins = e.angle_bins;
  c.max_models = e.max_models;
  c.min_votes_frac = e.min_votes_frac;
  c.consensus_floor_mult = e.consensus_floor_mult;
  c.dedupe_overlap = e.dedupe_overlap;
  c.tau_z = e.tau_z;
  c.tau_deg = e.tau_deg;
  c.suppression_radius = e.suppression_radius;
  c.refine = e.refine ? 1 : 0;
  c.normalize_inputs = e.normalize_inputs ? 1 : 0;
  c.threads = e.threads;
  return c;
}
inline RotationEstimate to_est(const rv_estimate& e, int model) {
  RotationEstimate out;
  out.axis = from3(e.axis);
  out.angle = e.angle;
  out.rotation = from9(e.rotation);
  out.axis_votes = e.axis_votes;
  out.elapsed_s = e.elapsed_s;
  out.inliers.resize(static_cast<std::size_t>(e.n_inliers));
  check(rv_result_inliers(context(), model, out.inliers.data(), e.n_inliers));
  return out;
}
}  // namespace detail

inline PreprocessResult preprocess(std::span<const Correspondence> correspondences, double tau_z, bool normalize = true) {
  PreprocessResult out;
  if (correspondences.empty()) return out;
  const double* flat = detail::rows(correspondences);
  const std::size_t n = correspondences.size();
  std::vector<double> z(3 * n);
  std::vector<int32_t> kept(n), dropped(n);
  int64_t nk = 0, nd = 0;
  detail::check(rv_preprocess(detail::context(), flat, static_cast<int64_t>(n), tau_z, normalize ? 1 : 0,
                              z.data(), kept.data(), dropped.data(), &nk, &nd));
  for (int64_t i = 0; i < nk; ++i) out.constraints.push_back(detail::from3(z.data() + 3 * i));
  out.kept.assign(kept.begin(), kept.begin() + nk);
  out.dropped.assign(dropped.begin(), dropped.begin() + nd);
  return out;
}

inline std::vector<int> classify_inliers(const Vec3& axis, std::span<const Vec3> constraints, double epsilon) {
  if (constraints.empty()) return {};
  double a[3];
  detail::to3(axis, a);
  std::vector<double> z(3 * constraints.size());
  for (std::size_t i = 0; i < constraints.size(); ++i) detail::to3(constraints[i], z.data() + 3 * i);
  std::vector<int32_t> out(constraints.size());
  int64_t m = 0;
  detail::check(rv_classify_inliers(detail::context(), a, z.data(), static_cast<int64_t>(constraints.size()), epsilon,
                                    out.data(), &m));
  return std::vector<int>(out.begin(), out.begin() + m);
}

inline Vec3 refine_axis(std::span<const Vec3> constraints) {
  if (constraints.size() < 2) throw RankDeficient("need at least two constraints");
  std::vector<double> z(3 * constraints.size());
  for (std::size_t i = 0; i < constraints.size(); ++i) detail::to3(constraints[i], z.data() + 3 * i);
  double a[3];
  detail::check(rv_refine_axis(detail::context(), z.data(), static_cast<int64_t>(constraints.size()), a));
  return detail::from3(a);
}

inline std::uint32_t peak_vote_floor(const EstimatorConfig& cfg, std::size_t n_constraints) {
  const rv_config c = detail::to_c(cfg);
  return rv_peak_vote_floor(&c, static_cast<int64_t>(n_constraints));
}

inline RotationEstimate estimate_single(std::span<const Correspondence> correspondences, const EstimatorConfig& cfg) {
  if (correspondences.empty()) throw EmptyInput("no correspondences");
  const double* flat = detail::rows(correspondences);
  const rv_config c = detail::to_c(cfg);
  rv_estimate e;
  if (rv_multi* m = detail::multi()) {  // ROTAVOTE_DEVICES: sharded over several GPUs
    detail::check_multi(rv_multi_estimate_single(m, flat, static_cast<int64_t>(correspondences.size()), &c, &e));
    RotationEstimate out;
    out.axis = detail::from3(e.axis);
    out.angle = e.angle;
    out.rotation = detail::from9(e.rotation);
    out.axis_votes = e.axis_votes;
    out.elapsed_s = e.elapsed_s;
    out.inliers.resize(static_cast<std::size_t>(e.n_inliers));
    detail::check_multi(rv_multi_result_inliers(m, out.inliers.data(), e.n_inliers));
    return out;
  }
  detail::check(rv_estimate_single(detail::context(), flat, static_cast<int64_t>(correspondences.size()), &c, &e));
  return detail::to_est(e, 0);
}

inline std::vector<RotationEstimate> estimate_multi(std::span<const Correspondence> correspondences,
                                                    const EstimatorConfig& cfg) {
  if (correspondences.empty()) throw EmptyInput("no correspondences");
  const double* flat = detail::rows(correspondences);
  const rv_config c = detail::to_c(cfg);
  const int cap = cfg.max_models > 0 ? cfg.max_models : 1;
  std::vector<rv_estimate> es(static_cast<std::size_t>(cap));
  int32_t nm = 0;
  detail::check(rv_estimate_multi(detail::context(), flat, static_cast<int64_t>(correspondences.size()), &c,
                                  es.data(), cap, &nm));
  std::vector<RotationEstimate> out;
  for (int k = 0; k < nm && k < cap; ++k) out.push_back(detail::to_est(es[k], k));
  return out;
}

// EXTENSION (not in the reference): one-pass top-K multi-model mode --
// one vote, find_peaks(K = max_models), the single-model finish per peak and estimate_multi's
// acceptance rules, without the sequential strip-and-revote. See rv_estimate_multi_onepass.
inline std::vector<RotationEstimate> estimate_multi_onepass(std::span<const Correspondence> correspondences,
                                                            const EstimatorConfig& cfg) {
  if (correspondences.empty()) throw EmptyInput("no correspondences");
  const double* flat = detail::rows(correspondences);
  const rv_config c = detail::to_c(cfg);
  const int cap = cfg.max_models > 0 ? cfg.max_models : 1;
  std::vector<rv_estimate> es(static_cast<std::size_t>(cap));
  int32_t nm = 0;
  detail::check(rv_estimate_multi_onepass(detail::context(), flat,
                                          static_cast<int64_t>(correspondences.size()), &c, es.data(), cap, &nm));
  std::vector<RotationEstimate> out;
  for (int k = 0; k < nm && k < cap; ++k) out.push_back(detail::to_est(es[k], k));
  return out;
}

}  // namespace rotavote
