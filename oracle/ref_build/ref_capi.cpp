// C entry points over the UNMODIFIED reference library (compiled from /root/reference with
// the Eigen-subset shim) -- TEST INFRASTRUCTURE ONLY. Lets Python (tests/golden generation,
// oracle pinning) and bench.py's "reference" CPU arm call the reference's own public API:
// estimate_single / estimate_multi / accumulate / find_peaks / blurred_argmax /
// preprocess / classify_inliers / refine_axis (estimator.hpp:47-70, voting.hpp:64-80).
// Struct layouts match oracle/rv_oracle.h (rvo_config / rvo_peak / rvo_estimate).
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <span>
#include <vector>

#include "rotavote/errors.hpp"
#include "rotavote/baselines.hpp"
#include "rotavote/estimator.hpp"
#include "rotavote/io.hpp"
#include "rotavote/voting.hpp"

using namespace rotavote;

extern "C" {
struct ref_config {
  int32_t grid;
  double extent;
  int32_t theta_samples;
  double epsilon;
  int32_t angle_bins;
  int32_t max_models;
  double min_votes_frac;
  double consensus_floor_mult;
  double dedupe_overlap;
  double tau_z;
  double tau_deg;
  int32_t suppression_radius;
  int32_t refine;
  int32_t normalize_inputs;
  int32_t threads;
};
struct ref_peak {
  int32_t ix, iy;
  double A, B;
  uint32_t votes;
};
struct ref_estimate {
  double axis[3];
  double angle;
  double rotation[9];
  uint32_t axis_votes;
  int64_t n_inliers;
  int32_t* inliers;
  double elapsed_s;
};
}

namespace {
EstimatorConfig to_cfg(const ref_config* c) {
  EstimatorConfig e;
  e.grid = c->grid;
  e.extent = c->extent;
  e.theta_samples = c->theta_samples;
  e.epsilon = c->epsilon;
  e.angle_bins = c->angle_bins;
  e.max_models = c->max_models;
  e.min_votes_frac = c->min_votes_frac;
  e.consensus_floor_mult = c->consensus_floor_mult;
  e.dedupe_overlap = c->dedupe_overlap;
  e.tau_z = c->tau_z;
  e.tau_deg = c->tau_deg;
  e.suppression_radius = c->suppression_radius;
  e.refine = c->refine != 0;
  e.normalize_inputs = c->normalize_inputs != 0;
  e.threads = c->threads;
  return e;
}
std::vector<Correspondence> to_corrs(const double* p, int64_t n) {
  std::vector<Correspondence> v(static_cast<std::size_t>(n));
  for (int64_t i = 0; i < n; ++i) {
    v[i].x = Vec3(p[6 * i], p[6 * i + 1], p[6 * i + 2]);
    v[i].y = Vec3(p[6 * i + 3], p[6 * i + 4], p[6 * i + 5]);
  }
  return v;
}
std::vector<Vec3> to_vecs(const double* p, int64_t n) {
  std::vector<Vec3> v(static_cast<std::size_t>(n));
  for (int64_t i = 0; i < n; ++i) v[i] = Vec3(p[3 * i], p[3 * i + 1], p[3 * i + 2]);
  return v;
}
void fill(const RotationEstimate& e, ref_estimate* o) {
  for (int i = 0; i < 3; ++i) o->axis[i] = e.axis(i);
  o->angle = e.angle;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) o->rotation[i * 3 + j] = e.rotation(i, j);
  o->axis_votes = e.axis_votes;
  o->n_inliers = static_cast<int64_t>(e.inliers.size());
  o->inliers = static_cast<int32_t*>(std::malloc(sizeof(int32_t) * (e.inliers.size() + 1)));
  std::memcpy(o->inliers, e.inliers.data(), sizeof(int32_t) * e.inliers.size());
  o->elapsed_s = e.elapsed_s;
}
template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const EmptyInput&) {
    return 1;
  } catch (const NoPeak&) {
    return 2;
  } catch (const DegenerateProjection&) {
    return 3;
  } catch (const NoVotes&) {
    return 4;
  } catch (const AllDegenerate&) {
    return 5;
  } catch (const RankDeficient&) {
    return 6;
  } catch (const NoConsensus&) {
    return 7;
  } catch (const InvalidConfig&) {
    return 8;
  } catch (const PoleProximity&) {
    return 9;
  } catch (...) {
    return 99;
  }
}
}  // namespace

extern "C" {
void ref_free(void* p) { std::free(p); }

int ref_estimate_single(const double* corrs, int64_t n, const ref_config* cfg, ref_estimate* out) {
  return guarded([&] {
    const auto c = to_corrs(corrs, n);
    fill(estimate_single(c, to_cfg(cfg)), out);
  });
}

int ref_estimate_multi(const double* corrs, int64_t n, const ref_config* cfg, ref_estimate* out,
                       int32_t* n_models) {
  *n_models = 0;
  return guarded([&] {
    const auto c = to_corrs(corrs, n);
    const auto v = estimate_multi(c, to_cfg(cfg));
    for (std::size_t k = 0; k < v.size() && static_cast<int>(k) < cfg->max_models; ++k) fill(v[k], out + k);
    *n_models = static_cast<int32_t>(v.size());
  });
}

int ref_preprocess(const double* corrs, int64_t n, double tau_z, int normalize, double* z_out,
                   int32_t* kept_out, int32_t* dropped_out, int64_t* n_kept, int64_t* n_dropped) {
  *n_kept = 0;
  *n_dropped = 0;
  return guarded([&] {
    const auto c = to_corrs(corrs, n);
    const auto pre = preprocess(c, tau_z, normalize != 0);
    for (std::size_t i = 0; i < pre.constraints.size(); ++i)
      for (int k = 0; k < 3; ++k) z_out[3 * i + k] = pre.constraints[i](k);
    std::memcpy(kept_out, pre.kept.data(), sizeof(int32_t) * pre.kept.size());
    std::memcpy(dropped_out, pre.dropped.data(), sizeof(int32_t) * pre.dropped.size());
    *n_kept = static_cast<int64_t>(pre.kept.size());
    *n_dropped = static_cast<int64_t>(pre.dropped.size());
  });
}

int ref_accumulate(const double* z, int64_t n, int32_t grid, double extent, int32_t samples, int32_t threads,
                   uint32_t* counts) {
  return guarded([&] {
    const auto acc = accumulate(to_vecs(z, n), grid, extent, samples, threads);
    std::memcpy(counts, acc.counts().data(), sizeof(uint32_t) * acc.counts().size());
  });
}

int ref_find_peaks(const uint32_t* counts, int32_t grid, double extent, int32_t max_peaks, int32_t radius,
                   uint32_t min_votes, ref_peak* out, int32_t* n_out) {
  *n_out = 0;
  return guarded([&] {
    Accumulator2D acc(grid, extent);
    std::memcpy(acc.counts().data(), counts, sizeof(uint32_t) * acc.counts().size());
    const auto ps = find_peaks(acc, max_peaks, radius, min_votes);
    for (std::size_t k = 0; k < ps.peaks.size(); ++k) {
      out[k] = {ps.peaks[k].ix, ps.peaks[k].iy, ps.peaks[k].center.A, ps.peaks[k].center.B, ps.peaks[k].votes};
    }
    *n_out = static_cast<int32_t>(ps.peaks.size());
  });
}

int ref_blurred_argmax(const uint32_t* counts, int32_t grid, double extent, int32_t radius, ref_peak* out) {
  return guarded([&] {
    Accumulator2D acc(grid, extent);
    std::memcpy(acc.counts().data(), counts, sizeof(uint32_t) * acc.counts().size());
    const Peak p = blurred_argmax(acc, radius);
    *out = {p.ix, p.iy, p.center.A, p.center.B, p.votes};
  });
}

int64_t ref_classify_inliers(const double axis[3], const double* z, int64_t n, double eps, int32_t* out) {
  const auto v = classify_inliers(Vec3(axis[0], axis[1], axis[2]), to_vecs(z, n), eps);
  std::memcpy(out, v.data(), sizeof(int32_t) * v.size());
  return static_cast<int64_t>(v.size());
}

int ref_grid_oracle_axis(const double* z, int64_t n, int32_t directions, double eps, double axis_out[3],
                         int32_t* count_out) {
  return guarded([&] {
    OracleConfig oc;
    oc.directions = directions;
    oc.epsilon = eps;
    const auto r = grid_oracle_axis(to_vecs(z, n), oc);
    for (int k = 0; k < 3; ++k) axis_out[k] = r.first(k);
    *count_out = r.second;
  });
}

int ref_ransac_rotation(const double* corrs, int64_t n, int32_t iterations, double eps, uint64_t seed,
                        ref_estimate* out) {
  return guarded([&] { fill(ransac_rotation(to_corrs(corrs, n), iterations, eps, seed), out); });
}

int ref_refine_axis(const double* z, int64_t n, double axis_out[3]) {
  return guarded([&] {
    const Vec3 a = refine_axis(to_vecs(z, n));
    for (int k = 0; k < 3; ++k) axis_out[k] = a(k);
  });
}

// read_correspondences (io.cpp:66-101) -- the parity oracle and CPU baseline of the device CSV
// ingest. Returns 0 (rows in *out, grown with malloc; free with ref_free), 15 ParseError
// (message + line), 16 EmptyFile, 17 IoError (message), 99 other.
int ref_read_correspondences(const char* path, double** out, int64_t* n, int64_t* line, char* msg, int64_t msg_cap) {
  auto put = [&](const std::string& m) {
    if (msg && msg_cap > 0) {
      std::strncpy(msg, m.c_str(), (size_t)msg_cap - 1);
      msg[msg_cap - 1] = 0;
    }
  };
  *out = nullptr;
  *n = 0;
  *line = 0;
  try {
    const auto v = read_correspondences(path);
    double* p = static_cast<double*>(std::malloc(sizeof(double) * 6 * (v.empty() ? 1 : v.size())));
    for (size_t i = 0; i < v.size(); ++i) {
      p[6 * i + 0] = v[i].x.x();
      p[6 * i + 1] = v[i].x.y();
      p[6 * i + 2] = v[i].x.z();
      p[6 * i + 3] = v[i].y.x();
      p[6 * i + 4] = v[i].y.y();
      p[6 * i + 5] = v[i].y.z();
    }
    *out = p;
    *n = static_cast<int64_t>(v.size());
    return 0;
  } catch (const ParseError& e) {
    *line = e.line;
    put(e.what());
    return 15;
  } catch (const EmptyFile& e) {
    put(e.what());
    return 16;
  } catch (const IoError& e) {
    put(e.what());
    return 17;
  } catch (...) {
    return 99;
  }
}
}
