/* CPU oracle for the spatial-voting path of arXiv 2502.06337 -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference ("rotavote", /root/reference/proj) hot path:
 * preprocess, orthonormal basis, sampled circle voting, greedy top-K NMS, blurred argmax,
 * classify / refine (3x3 symmetric eigen-solve), angle voting, estimate_single and
 * estimate_multi. Every function cites the reference file:line it follows.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load this
 * library, and only as the checker. The product (paper_2502_06337_b200) never links it.
 *
 * Pinned against the reference itself: tests/golden/ fixtures are produced by the
 * UNMODIFIED reference sources compiled here (oracle/ref_build, Eigen-subset shim), and
 * tests/test_oracle.py checks this restatement bit-for-bit against them.
 *
 * Build with -O2 -ffp-contract=off (strict IEEE evaluation order, no FMA contraction).
 */
#ifndef RV_ORACLE_H
#define RV_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes: same values as the product C-ABI (include/rotavote_b200.h). */
enum {
  RVO_OK = 0,
  RVO_EMPTY_INPUT = 1,
  RVO_NO_PEAK = 2,
  RVO_DEGENERATE_PROJECTION = 3,
  RVO_NO_VOTES = 4,
  RVO_ALL_DEGENERATE = 5,
  RVO_RANK_DEFICIENT = 6,
  RVO_NO_CONSENSUS = 7,
  RVO_INVALID_CONFIG = 8,
  RVO_POLE_PROXIMITY = 9,
  RVO_OUT_OF_MEMORY = 10
};

/* EstimatorConfig, estimator.hpp:13-29 (same field order as rv_config in the product). */
typedef struct {
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
} rvo_config;

typedef struct { /* Peak, voting.hpp:41-46 */
  int32_t ix, iy;
  double A, B;
  uint32_t votes;
} rvo_peak;

typedef struct { /* RotationEstimate, estimator.hpp:31-38 (rotation row-major) */
  double axis[3];
  double angle;
  double rotation[9];
  uint32_t axis_votes;
  int64_t n_inliers;
  int32_t* inliers; /* malloc'd, ascending input indices; free with rvo_free */
} rvo_estimate;

void rvo_config_default(rvo_config* cfg);
void rvo_free(void* p);

/* estimator.cpp:259-285. corrs: n x 6 doubles (x0 x1 x2 y0 y1 y2). Outputs sized >= n. */
int rvo_preprocess(const double* corrs, int64_t n, double tau_z, int normalize, double* z_out,
                   int32_t* kept_out, int32_t* dropped_out, int64_t* n_kept, int64_t* n_dropped);
/* geom.cpp:36-43 */
void rvo_orthonormal_basis(const double z[3], double a1[3], double a2[3]);
/* voting.cpp:72-81: 2*J doubles (cos, sin) */
void rvo_circle_table(int32_t samples, double* table);
/* voting.cpp:88-118 (sequential order; the reference proves thread-count independence) */
int rvo_accumulate(const double* z, int64_t n, int32_t grid, double extent, int32_t samples,
                   uint32_t* counts);
/* voting.cpp:83-86 deposit_circle_votes: adds one constraint's J votes into counts */
void rvo_deposit_circle(const double z[3], uint32_t* counts, int32_t grid, double extent,
                        int32_t samples);
/* voting.cpp:17-23 / :55-57 */
int32_t rvo_coord_to_cell(double v, int32_t grid, double extent);
/* voting.cpp:120-170 */
int rvo_find_peaks(const uint32_t* counts, int32_t grid, double extent, int32_t max_peaks,
                   int32_t radius, uint32_t min_votes, rvo_peak* out, int32_t* n_out);
/* voting.cpp:176-216 */
int rvo_blurred_argmax(const uint32_t* counts, int32_t grid, double extent, int32_t radius,
                       rvo_peak* out);
/* voting.cpp:172-174 */
void rvo_backproject_peak(double A, double B, double out[3]);
/* estimator.cpp:287-297 */
int64_t rvo_classify_inliers(const double axis[3], const double* z, int64_t n, double eps,
                             int32_t* out);
/* estimator.cpp:299-309 (z: n x 3 contiguous) */
int rvo_refine_axis(const double* z, int64_t n, double axis_out[3]);
/* 3x3 symmetric eigen-solve (Eigen 3.4 SelfAdjointEigenSolver restatement); s row-major */
void rvo_eigen_sym3(const double s[9], double evals[3], double evecs[9]);
/* angles.cpp:36-44 */
int rvo_correspondence_angle(const double axis[3], const double x[3], const double y[3],
                             double tau, double* angle);
/* angles.cpp:46-68; bins: bin_count u32; raw_out sized >= n_idx */
int rvo_vote_angles(const double axis[3], const double* corrs, const int32_t* idx, int64_t n_idx,
                    int32_t bin_count, double tau, uint32_t* bins, uint64_t* contributing,
                    uint64_t* degenerate, double* raw_out);
/* angles.cpp:70-90 */
int rvo_peak_angle(const uint32_t* bins, int32_t bin_count, uint64_t contributing, int refine,
                   const double* raw, int64_t n_raw, double* out);
/* geom.cpp:10-19 */
void rvo_rodrigues(const double axis[3], double angle, double r[9]);
double rvo_rotation_error(const double r_gt[9], const double r_opt[9]);
/* estimator.cpp:311-318 */
uint32_t rvo_peak_vote_floor(const rvo_config* cfg, int64_t n_constraints);
/* estimator.cpp:320-371 */
int rvo_estimate_single(const double* corrs, int64_t n, const rvo_config* cfg, rvo_estimate* out);
/* estimator.cpp:373-493; out sized >= cfg->max_models */
int rvo_estimate_multi(const double* corrs, int64_t n, const rvo_config* cfg, rvo_estimate* out,
                       int32_t* n_models);

/* Stage trace of the last estimate_single call (for stage-by-stage parity checks). */
typedef struct {
  int32_t peak_ix, peak_iy;
  uint32_t peak_votes;
  double start_axis[3];  /* canonicalize(backproject(interpolate_peak)) */
  int32_t refine_passes; /* refine_axis calls in the primary refine_loop */
  int32_t rescued;       /* 1 if the rescue path ran */
  int32_t rescue_won;    /* index of the winning rescue candidate, -1 = primary */
  int64_t n_kept, n_dropped;
} rvo_trace;
void rvo_last_trace(rvo_trace* out);

#ifdef __cplusplus
}
#endif
#endif
