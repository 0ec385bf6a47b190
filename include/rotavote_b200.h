/* rotavote_b200 -- C-ABI of the B200-native spatial-voting path (arXiv 2502.06337).
 *
 * This is the drop-in boundary: plain pointers and sizes, no CUDA/torch types. Each entry
 * point replaces one function of the reference library "rotavote" (C++20, CPU only,
 * /root/reference/proj); the reference signature it replaces is cited next to it
 * (file:line under proj/). Arrays follow the reference's memory layout:
 *   - correspondences: n x 6 doubles, row i = (x0 x1 x2 y0 y1 y2)  == span<const Correspondence>
 *     (Correspondence = {Eigen::Vector3d x, y}, angles.hpp:11-14: 48 B, no padding)
 *   - constraints:     n x 3 doubles                             == span<const Vec3>
 *   - vote grid:       grid*grid uint32, row-major counts[iy*grid + ix]  (voting.hpp:14-39)
 *   - matrices:        3x3 row-major doubles
 * Errors: every call returns rv_status. The reference throws typed exceptions
 * (errors.hpp:8-55); the C++ drop-in headers (include/rotavote/) rethrow the same types.
 *
 * Host-buffer entry points copy inputs to the device (H2D) and results back (D2H) inside
 * the call; *_device variants take device pointers already resident in HBM.
 * A context is not thread-safe: use one context per host thread (the reference estimator is
 * stateless; contexts keep that property per thread).
 */
#ifndef ROTAVOTE_B200_H
#define ROTAVOTE_B200_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RV_ABI_VERSION 5

typedef enum rv_status {
  RV_OK = 0,
  RV_ERR_EMPTY_INPUT = 1,           /* rotavote::EmptyInput */
  RV_ERR_NO_PEAK = 2,               /* rotavote::NoPeak */
  RV_ERR_DEGENERATE_PROJECTION = 3, /* rotavote::DegenerateProjection */
  RV_ERR_NO_VOTES = 4,              /* rotavote::NoVotes */
  RV_ERR_ALL_DEGENERATE = 5,        /* rotavote::AllDegenerate */
  RV_ERR_RANK_DEFICIENT = 6,        /* rotavote::RankDeficient */
  RV_ERR_NO_CONSENSUS = 7,          /* rotavote::NoConsensus */
  RV_ERR_INVALID_CONFIG = 8,        /* rotavote::InvalidConfig */
  RV_ERR_POLE_PROXIMITY = 9,        /* rotavote::PoleProximity */
  RV_ERR_OUT_OF_MEMORY = 10,
  RV_ERR_CUDA = 11,                 /* CUDA runtime failure (message in rv_context_last_error) */
  RV_ERR_NCCL = 12,
  RV_ERR_INVALID_ARGUMENT = 13,
  RV_ERR_NO_DEVICE = 14,
  RV_ERR_PARSE = 15,                /* rotavote::ParseError (line in error_line) */
  RV_ERR_EMPTY_FILE = 16,           /* rotavote::EmptyFile */
  RV_ERR_IO = 17                    /* rotavote::IoError */
} rv_status;

/* EstimatorConfig, estimator.hpp:13-29 -- same fields, same defaults (rv_config_default). */
typedef struct rv_config {
  int32_t grid;                /* accumulator resolution G (512) */
  double extent;               /* accumulator half-width E (1.05) */
  int32_t theta_samples;       /* circle samples J (2048) */
  double epsilon;              /* inlier threshold on |axis . z| (0.015) */
  int32_t angle_bins;          /* 1024 */
  int32_t max_models;          /* 1 */
  double min_votes_frac;       /* 0.02 */
  double consensus_floor_mult; /* 1.5 */
  double dedupe_overlap;       /* 0.5 */
  double tau_z;                /* 1e-9 */
  double tau_deg;              /* 1e-6 */
  int32_t suppression_radius;  /* 8 */
  int32_t refine;              /* 1 */
  int32_t normalize_inputs;    /* 1 */
  int32_t threads;             /* accepted for API parity; the device path ignores it */
} rv_config;

/* Peak, voting.hpp:41-46 (center = cell center (A, B)). */
typedef struct rv_peak {
  int32_t ix, iy;
  double A, B;
  uint32_t votes;
} rv_peak;

/* RotationEstimate, estimator.hpp:31-38. Inliers are fetched with rv_result_inliers. */
typedef struct rv_estimate {
  double axis[3];
  double angle;
  double rotation[9];
  uint32_t axis_votes;
  int64_t n_inliers;
  double elapsed_s;
} rv_estimate;

/* Device time of each stage of the last call (CUDA events on the context stream; only
 * filled when timing is enabled). Used by bench.py for the roofline. */
typedef struct rv_stage_times {
  double preprocess_ms; /* K1: preprocess + basis + band plan */
  double vote_ms;       /* K2: band-tiled vote (+ tile reduction) */
  double peaks_ms;      /* K3: argmax / NMS / blur */
  double refine_ms;     /* K4: classify + scatter + eigen loop */
  double angles_ms;     /* K4: angle histogram + circular mean + model support */
  double total_ms;
  int64_t vote_pairs;       /* sample pairs evaluated by the vote kernel (work incl. padding) */
  int64_t vote_fallback_pairs; /* pairs re-evaluated on the exact f64 path */
  int64_t vote_guard_reruns;   /* votes redone by the generic exact kernel (grid sum != N*J) */
  int64_t vote_samples;     /* algorithmic samples N_kept * J of all vote launches */
  int32_t vote_launches;    /* vote kernel launches in the call */
  int32_t kernel_launches;  /* all kernels launched by the call */
  double vote_kernel_ms;    /* the band-tiled vote kernel alone (CUDA events around its launches) */
  int64_t csv_host_fields;  /* CSV fields outside the device parser's exact fast path, parsed by the
                               host's std::from_chars (rv_*_correspondences_csv) */
} rv_stage_times;

typedef struct rv_context rv_context;

/* ---- context ---------------------------------------------------------------------- */
void rv_config_default(rv_config* cfg);
const char* rv_status_string(rv_status st);
int32_t rv_abi_version(void);
rv_status rv_context_create(int32_t device, rv_context** out);
void rv_context_destroy(rv_context* ctx);
/* Run on an external CUDA stream (cudaStream_t as void*); NULL = the context's own stream. */
rv_status rv_context_set_stream(rv_context* ctx, void* cuda_stream);
const char* rv_context_last_error(const rv_context* ctx);
rv_status rv_context_enable_timing(rv_context* ctx, int32_t enable);
rv_status rv_context_stage_times(const rv_context* ctx, rv_stage_times* out);

/* ---- solver API (the drop-in for estimate_single / estimate_multi) ------------------ */
/* RotationEstimate estimate_single(span<const Correspondence>, const EstimatorConfig&)
 * -- estimator.hpp:63-64, estimator.cpp:320-371 */
rv_status rv_estimate_single(rv_context* ctx, const double* corrs, int64_t n, const rv_config* cfg,
                             rv_estimate* out);
rv_status rv_estimate_single_device(rv_context* ctx, const double* d_corrs, int64_t n,
                                    const rv_config* cfg, rv_estimate* out);
/* vector<RotationEstimate> estimate_multi(span<const Correspondence>, const EstimatorConfig&)
 * -- estimator.hpp:69-70, estimator.cpp:373-493 (sequential extraction, sorted by votes) */
rv_status rv_estimate_multi(rv_context* ctx, const double* corrs, int64_t n, const rv_config* cfg,
                            rv_estimate* out, int32_t capacity, int32_t* n_models);
rv_status rv_estimate_multi_device(rv_context* ctx, const double* d_corrs, int64_t n,
                                   const rv_config* cfg, rv_estimate* out, int32_t capacity,
                                   int32_t* n_models);
/* EXTENSION (no reference counterpart): one-pass top-K multi-model mode.
 * One vote over all correspondences, find_peaks(K = max_models) with the reference NMS
 * (voting.cpp:120-170) at peak_vote_floor (estimator.cpp:311-318), then per peak the
 * single-model finish (estimator.cpp:94-101, :51-92) and estimate_multi's acceptance rules
 * (consensus floor, model_support coherence, dedupe_overlap; estimator.cpp:411-452) -- without
 * the sequential strip-and-revote, so K models cost one vote. Models in descending axis_votes. */
rv_status rv_estimate_multi_onepass(rv_context* ctx, const double* corrs, int64_t n, const rv_config* cfg,
                                    rv_estimate* out, int32_t capacity, int32_t* n_models);
rv_status rv_estimate_multi_onepass_device(rv_context* ctx, const double* d_corrs, int64_t n,
                                           const rv_config* cfg, rv_estimate* out, int32_t capacity,
                                           int32_t* n_models);
/* EXTENSION (the reference's run_benchmark trials, bench.cpp:70-147, call
 * estimate_single once per trial): batched solver for independent problems. Problem k is the
 * correspondences [offsets[k], offsets[k+1]) of corrs (host, n x 6 doubles; offsets has
 * n_problems + 1 entries). Every problem gets estimate_single semantics; problems run
 * concurrently on `workers` device streams (0 = automatic: 8 for problems below ~32k
 * correspondences, else 1), each with its own buffers, so small problems share the GPU instead of
 * running one after another (3-4x measured at n = 1000). status[k] is problem k's code (a failing
 * problem does not stop the batch); on RV_OK, out[k] is its estimate and
 * rv_result_inliers(ctx, k, ...) its inlier indices, relative to offsets[k]. */
rv_status rv_estimate_batch(rv_context* ctx, const double* corrs, const int64_t* offsets, int32_t n_problems,
                            const rv_config* cfg, int32_t workers, rv_estimate* out, int32_t* status);
/* ---- baselines: consensus scoring on the device ---------------- */
/* consensus_count (baselines.cpp:16-24) of m candidate axes (m x 3) over n constraints (n x 3):
 * counts_out[k] = #{i : |axes_k . z_i| < epsilon} (strict; the reference's op order). */
rv_status rv_consensus_counts(rv_context* ctx, const double* axes, int32_t m, const double* z, int64_t n,
                              double epsilon, uint32_t* counts_out);
/* pair<Vec3,int> grid_oracle_axis(span<const Vec3>, const OracleConfig&) -- baselines.hpp:38-39,
 * baselines.cpp:159-174: exhaustive consensus over the Fibonacci layout of oracle_direction
 * (baselines.cpp:150-157); ties keep the lowest direction index. */
rv_status rv_grid_oracle_axis(rv_context* ctx, const double* z, int64_t n, int32_t directions, double epsilon,
                              double axis_out[3], int32_t* count_out);
/* RotationEstimate ransac_rotation(span<const Correspondence>, int iterations, double epsilon,
 * uint64_t seed) -- baselines.hpp:22-23, baselines.cpp:31-109: the same seeded hypothesis stream
 * (std::mt19937_64), all hypotheses scored on the device at once, then the reference's refit. */
rv_status rv_ransac_rotation(rv_context* ctx, const double* corrs, int64_t n, int32_t iterations, double epsilon,
                             uint64_t seed, rv_estimate* out);
/* ---- sharded solve (one process per GPU; the caller runs the collectives) ------------- */
/* Vote of one contiguous shard of the correspondences: preprocess the shard and deposit its
 * constraints' samples into d_grid (grid*grid uint32, device, overwritten). Integer grids of all
 * shards sum (e.g. ncclAllReduce, ncclUint32, ncclSum) to exactly the grid of
 * accumulate(preprocess(all)) -- voting.cpp:88-118 is order-independent. */
rv_status rv_vote_shard(rv_context* ctx, const double* d_corrs_shard, int64_t n_shard, const rv_config* cfg,
                        uint32_t* d_grid, int64_t* n_kept_shard);
/* estimate_single (estimator.cpp:320-371) on all correspondences with the vote grid supplied
 * (the summed shard grids): preprocess, then peak / refine / angle / rescue as usual. */
rv_status rv_estimate_single_prevoted(rv_context* ctx, const double* d_corrs, int64_t n, const rv_config* cfg,
                                      const uint32_t* d_grid, rv_estimate* out);

/* ---- sharded finish steps ------------------------------------------------
 * refine_loop / build_estimate (estimator.cpp:51-92) split so each rank (or device) works on its
 * own shard and only small partials cross the interconnect. After rv_vote_shard on every shard
 * and a sum of the shard grids:
 *   rv_peak_start_axis   find_peaks(K=1) + estimate_from_peak's start axis (estimator.cpp:94-97)
 *                        from the summed grid; *total = grid sum (exactness guard: N_kept * J)
 *   rv_shard_classify    classify_inliers (estimator.cpp:287-297) of this shard into bitmask slot
 *                        0/1, fused with the 6 scatter sums of refine_axis (:299-302) over the same
 *                        inliers and "differs from the other slot" (refine_loop's next_inl == inl)
 *   rv_axis_from_scatter refine_axis's 3x3 eigen-solve of the rank-ordered sum (RV_ERR_RANK_DEFICIENT)
 *   rv_shard_inliers     the slot's inliers as ascending input indices + offset (host dst)
 *   rv_shard_angle_hist  vote_angles (angles.cpp:46-68) of this shard's inliers (bins of this shard)
 *   rv_shard_angle_sums  peak_angle's window sums (angles.cpp:70-90) of this shard's raw angles
 *                        around the peak of the SUMMED histogram: {sum sin, sum cos}
 * Concatenating the shard inlier lists in rank order reproduces the reference's ascending list. */
rv_status rv_peak_start_axis(rv_context* ctx, const uint32_t* d_grid, const rv_config* cfg, double axis[3],
                             uint32_t* votes, uint64_t* total);
rv_status rv_shard_classify(rv_context* ctx, const double axis[3], double epsilon, int32_t slot, int32_t compare_prev,
                            int64_t* count, double scatter[6], int32_t* differs);
rv_status rv_axis_from_scatter(const double scatter[6], double axis[3]);
/* refine_loop (estimator.cpp:51-69) of this shard as ONE device-resident loop, the per-pass
 * partials exchanged between the devices of a multi-GPU solve through peer memory: every device
 * writes its fixed-order partials (8 doubles) to line `rank` of every device's line buffer over
 * NVLink (release at system scope) and sums all devices' lines in rank order (acquire) -- the
 * same decision on every device, no host round trip per pass. peer_lines[q] = device q's buffer
 * (8 x 128 bytes, zeroed before the first use, peer access enabled); epoch increases across
 * solves and is the same on every device of one solve. n_dev = 1 needs no buffers. Leaves the
 * final set in slot 0 (rv_shard_inliers / rv_shard_angle_hist); count = all devices' inliers,
 * local_count = this shard's. Every device of the solve must call it concurrently. */
rv_status rv_shard_refine(rv_context* ctx, const double axis0[3], const rv_config* cfg, int32_t n_dev, int32_t rank,
                          double* const* peer_lines, uint64_t epoch, double axis[3], int64_t* count,
                          int64_t* local_count, double scatter[6], int32_t* refits);
/* Line buffers for rv_shard_refine across PROCESSES (one rank per GPU): rv_shard_lines_export
 * allocates this context's buffer (once, zeroed) and returns it with its CUDA IPC handle (64
 * bytes) for the other ranks; rv_shard_lines_open maps a peer rank's buffer from its handle
 * (closed with the context). Ranks on the same GPU must not use rv_shard_refine together (their
 * cooperative kernels would wait on each other): host-step the passes instead. */
rv_status rv_shard_lines_export(rv_context* ctx, void** lines, uint8_t handle[64]);
rv_status rv_shard_lines_open(rv_context* ctx, const uint8_t handle[64], void** lines);
rv_status rv_shard_inliers(rv_context* ctx, int32_t slot, int64_t offset, int32_t* dst, int64_t capacity,
                           int64_t* count);
rv_status rv_shard_angle_hist(rv_context* ctx, const double axis[3], const rv_config* cfg, uint32_t* bins,
                              uint64_t* contributing);
rv_status rv_shard_angle_sums(rv_context* ctx, const uint32_t* bins_total, const rv_config* cfg, double sums[2]);

/* ---- multi-GPU in one process (reference: accumulate's chunked thread fan-out,
 * voting.cpp:102-117) --------------------------------------------------------------------------
 * rv_multi: one rv_context per listed device plus an NCCL communicator clique (ncclCommInitAll,
 * NVLink/NVSwitch on a B200 box; NCCL is loaded at run time). estimate_single and accumulate on a
 * multi context split the input into contiguous shards (one per device), vote each shard on its
 * device, sum the u32 grids with one in-place ncclAllReduce (bit-identical to the single-device
 * grid), and -- estimate_single -- run the sharded finish above (rank-ordered partial sums, the
 * 3x3 solves on the host). Results equal the single-device path's; the rare rescue / identity /
 * guard branches finish on device 0 from the summed grid. RV_ERR_NCCL if NCCL is unavailable. */
typedef struct rv_multi rv_multi;
rv_status rv_multi_create(const int32_t* devices, int32_t n_devices, rv_multi** out);
void rv_multi_destroy(rv_multi* m);
int32_t rv_multi_size(const rv_multi* m);
const char* rv_multi_last_error(const rv_multi* m);
/* the NCCL version the clique runs (e.g. 22709), 0 before rv_multi_create succeeded */
int32_t rv_multi_nccl_version(const rv_multi* m);
rv_status rv_multi_estimate_single(rv_multi* m, const double* corrs, int64_t n, const rv_config* cfg,
                                   rv_estimate* out);
rv_status rv_multi_result_inliers(rv_multi* m, int32_t* dst, int64_t capacity);
/* accumulate (voting.hpp:64-65) of host constraints (n x 3), grid summed over the devices */
rv_status rv_multi_accumulate(rv_multi* m, const double* z, int64_t n, int32_t grid, double extent, int32_t samples,
                              uint32_t* counts_out);

/* ---- CSV ingest ------------------------------------------
 * read_correspondences (io.hpp:11-13, io.cpp:66-101): CSV rows x0,x1,x2,y0,y1,y2 with an
 * optional header line, parsed ON THE DEVICE (delimiter index + exact decimal->binary
 * conversion; the rare fields outside the exact fast path use the host's std::from_chars). The
 * rows land in context-owned device memory: *d_rows (n_rows x 6 f64, the reference's
 * Correspondence layout) stays valid until the next CSV call on the context and can be passed
 * straight to rv_estimate_single_device. Errors follow the reference: RV_ERR_PARSE with the
 * 1-based line in *error_line and the reference's message in rv_context_last_error
 * ("expected 6 fields, got N", "not a number: 'x'", "empty field"), RV_ERR_EMPTY_FILE, RV_ERR_IO. */
rv_status rv_parse_correspondences_csv(rv_context* ctx, const char* text, int64_t nbytes, const double** d_rows,
                                       int64_t* n_rows, int64_t* error_line);
rv_status rv_read_correspondences_csv(rv_context* ctx, const char* path, const double** d_rows, int64_t* n_rows,
                                      int64_t* error_line);

/* Copy `bytes` from device memory (e.g. the rows of a CSV call) to host memory, ordered after the
 * context's work. */
rv_status rv_device_to_host(rv_context* ctx, void* dst, const void* d_src, int64_t bytes);

/* Inliers (ascending input indices) of model `model` of the last estimate call. */
rv_status rv_result_inliers(rv_context* ctx, int32_t model, int32_t* dst, int64_t capacity);

/* ---- path functions (voting.hpp / estimator.hpp / angles.hpp) ----------------------- */
/* PreprocessResult preprocess(span<const Correspondence>, double tau_z, bool normalize)
 * -- estimator.hpp:47-48, estimator.cpp:259-285. Outputs sized >= n. */
rv_status rv_preprocess(rv_context* ctx, const double* corrs, int64_t n, double tau_z,
                        int32_t normalize, double* constraints_out, int32_t* kept_out,
                        int32_t* dropped_out, int64_t* n_kept, int64_t* n_dropped);
/* Accumulator2D accumulate(span<const Vec3>, int grid, double extent, int samples, int threads)
 * -- voting.hpp:64-65, voting.cpp:88-118. Bit-exact with the reference for every config. */
rv_status rv_accumulate(rv_context* ctx, const double* constraints, int64_t n, int32_t grid,
                        double extent, int32_t samples, uint32_t* counts_out);
rv_status rv_accumulate_device(rv_context* ctx, const double* d_constraints, int64_t n,
                               int32_t grid, double extent, int32_t samples, uint32_t* d_counts);
/* void deposit_circle_votes(const Vec3& z, Accumulator2D& acc, int samples)
 * -- voting.hpp:60, voting.cpp:83-86. counts is read, incremented, written back. */
rv_status rv_deposit_circle_votes(rv_context* ctx, const double z[3], uint32_t* counts,
                                  int32_t grid, double extent, int32_t samples);
/* PeakSet find_peaks(const Accumulator2D&, int max_peaks, int radius, uint32_t min_votes)
 * -- voting.hpp:70-71, voting.cpp:120-170. out sized >= max_peaks. */
rv_status rv_find_peaks(rv_context* ctx, const uint32_t* counts, int32_t grid, double extent,
                        int32_t max_peaks, int32_t radius, uint32_t min_votes, rv_peak* out,
                        int32_t* n_out);
/* Peak blurred_argmax(const Accumulator2D&, int radius) -- voting.hpp:80, voting.cpp:176-216 */
rv_status rv_blurred_argmax(rv_context* ctx, const uint32_t* counts, int32_t grid, double extent,
                            int32_t radius, rv_peak* out);
/* vector<int> classify_inliers(const Vec3&, span<const Vec3>, double) -- estimator.hpp:51-52 */
rv_status rv_classify_inliers(rv_context* ctx, const double axis[3], const double* constraints,
                              int64_t n, double epsilon, int32_t* out, int64_t* n_out);
/* Vec3 refine_axis(span<const Vec3>) -- estimator.hpp:57, estimator.cpp:299-309 */
rv_status rv_refine_axis(rv_context* ctx, const double* constraints, int64_t n, double axis_out[3]);
/* AngleHistogram vote_angles(axis, span<const Correspondence>, span<const int>, bins, tau)
 * -- angles.hpp:37-40, angles.cpp:46-68. raw_angles_out sized >= n_idx (insertion order). */
rv_status rv_vote_angles(rv_context* ctx, const double axis[3], const double* corrs, int64_t n_corrs,
                         const int32_t* indices, int64_t n_idx, int32_t bin_count, double tau,
                         uint32_t* bins_out, uint64_t* contributing, uint64_t* degenerate,
                         double* raw_angles_out);
/* double peak_angle(const AngleHistogram&, bool refine, span<const double>) -- angles.hpp:44-45 */
rv_status rv_peak_angle(rv_context* ctx, const uint32_t* bins, int32_t bin_count,
                        uint64_t contributing, int32_t refine, const double* raw_angles,
                        int64_t n_raw, double* angle_out);
/* uint32_t peak_vote_floor(const EstimatorConfig&, size_t) -- estimator.hpp:61 (host arithmetic) */
uint32_t rv_peak_vote_floor(const rv_config* cfg, int64_t n_constraints);

/* ---- geometry (geom.hpp:25-43; host arithmetic, identical formulas) ----------------- */
void rv_rodrigues(const double axis[3], double angle, double r_out[9]);
double rv_rotation_error(const double r_gt[9], const double r_opt[9]);
rv_status rv_project(const double p[3], double* A, double* B);
void rv_unproject(double A, double B, double out[3]);
void rv_canonicalize(const double p[3], double out[3]);
void rv_orthonormal_basis(const double z[3], double a1[3], double a2[3]);
rv_status rv_correspondence_angle(const double axis[3], const double x[3], const double y[3],
                                  double tau, double* angle_out);

#ifdef __cplusplus
}
#endif
#endif /* ROTAVOTE_B200_H */
