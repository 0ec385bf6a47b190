// Internal interfaces between the host orchestration (rv_api.cpp) and the sm_100a kernels
// (rv_kernels.cu). Not part of the public C-ABI.
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

namespace rvb {

constexpr int kMaxBands = 64;        // row bands of the smem-tiled vote kernel
#ifndef RV_VOTE_THREADS
#define RV_VOTE_THREADS 1024
#endif
constexpr int kVoteThreads = RV_VOTE_THREADS;  // threads per vote CTA (32 warps, <= 64 regs each: latency-bound loop)
constexpr int kPad = 2;              // sample-index padding of each band range (culling slack)
// vote counters: [0] slot counter, [1..kMaxBands] entry grab counters, [kMaxBands+1..2*kMaxBands]
// entries per band, [2*kMaxBands+1] degenerate constraints listed, [2*kMaxBands+2] their grab counter
constexpr int kCounterWords = 2 * kMaxBands + 3;
constexpr int kDegenCount = 2 * kMaxBands + 1;
constexpr int kDegenGrab = 2 * kMaxBands + 2;
constexpr int kEntriesPerConstraint = 3;  // per band: <= 2 sample ranges, one of them split at J
constexpr int kFbqCap = 64;          // per-warp exact-fallback queue entries
constexpr int kReduceThreads = 256;

// Geometry of one accumulate call, computed on the host from (grid, extent, samples).
struct VotePlan {
  int G = 0;         // grid
  int J = 0;         // theta samples
  int halfJ = 0;     // J/2 sample pairs (twins j, j+J/2)
  double E = 0;      // extent
  double inv_cell = 0;  // grid / (2*extent)   (voting.cpp:30)
  double cs = 0;        // 2*extent / grid     (voting.hpp:23)
  float Kf = 0;      // (float) inv_cell
  float CMf = 0;     // G/2 + 1.5*2^(23-S) + 2*2^-S: one FFMA yields t on a 2^-S grid, biased +2 units
  int frac_shift = 0;     // S: fixed-point resolution 2^-S of the cell coordinate t
  uint32_t frac_mask = 0; // ((1<<S)-1) & ~3: bits & mask == 0 <=> round(t*2^S) mod 2^S in [-2, 1]
  int magic_hi = 0;       // bits(1.5*2^(23-S)) >> S
  int clamp = 0;     // 1 if votes can fall outside the unit-disk rows/cols (extent <= 1)
  int r_min = 0, r_max = 0;  // stored rows [r_min, r_max]
  int c_min = 0, c_max = 0;  // stored cols
  int W = 0;                 // c_max - c_min + 1
  float Wf = 0;              // (float)W (RV_FP_CELL vote variant)
  int n_bands = 0;
  int H_max = 0;             // rows of the tallest band
  int band_r0[kMaxBands + 1];   // band b stores rows [band_r0[b], band_r0[b+1])
  float band_ylo[kMaxBands];    // plane-coordinate band limits with culling margin (+-inf at ends)
  float band_yhi[kMaxBands];
  float step_f = 0;             // (float)(2*pi/J)
  int banded = 0;               // 1: smem-tiled kernel; 0: exact generic global-atomic kernel
  int bulk = 0;                 // 1: full-width tiles (c_min = 0, W = G, G % 4 == 0) flushed into the
                                //    grid by TMA bulk reduce-adds (no partial slots, no slot reduction)
  size_t tile_words = 0;        // H_max * W rounded up to a multiple of 4
  size_t smem_bytes = 0;        // dynamic smem of the vote kernel
};

// Device workspace for one accumulate (sizes grow-only, owned by the context).
struct VoteBuffers {
  const double* zx = nullptr;  // constraints SoA (f64)
  const double* zy = nullptr;
  const double* zz = nullptr;
  float4* basis_a = nullptr;   // fl32 of (K a1x, K a1y, -a1z, K a2x), K = G/(2E)
  float2* basis_b = nullptr;   // fl32 of (K a2y, -a2z)
  // [n_bands][entry_cap] work entries of each band: ci | (start | len<<16) << 32, one per
  // non-empty range of CANONICAL samples (c <= 0, exactly as the reference decides it) of a
  // constraint in the band; start is a sample index in [0, J) (order irrelevant: integer sums)
  unsigned long long* entries = nullptr;
  int32_t* degen = nullptr;        // [n] constraints without a clean canonical half circle
                                   // (z = +-e3 exactly): voted sample by sample in f64
  int32_t* entry_count = nullptr;  // [kMaxBands] entries appended per band by K1
  int64_t entry_cap = 0;           // entries stride per band (kEntriesPerConstraint per constraint)
  unsigned long long* band_work = nullptr;  // [kMaxBands] pairs per band (incl. padding)
  float2* table32 = nullptr;   // [J] (cos, sin) of theta_j, rounded to f32
  double2* table64 = nullptr;  // [J] (cos, sin) exactly as the reference (host libm)
  uint32_t* grid = nullptr;    // [G*G] output
  uint32_t* partials = nullptr;        // [max_slots][tile_words]
  int32_t* slot_band = nullptr;        // [max_slots]
  int32_t* counters = nullptr;         // [kCounterWords] (layout above)
  unsigned long long* stats = nullptr; // [0]=pairs evaluated, [1]=fallback pairs
  int max_slots = 0;
  const int32_t* bounds = nullptr;     // device [lo, hi) of constraints for this launch (null: [range_lo, range_lo + n))
  int64_t range_lo = 0;
  // optional, fused into the tile reduction: argmax key + grid sum (find_peaks K=1 and the
  // exactness guard) and the start axis (estimate_from_peak)
  unsigned long long* red_keys = nullptr;  // [2 * reduce blocks] scratch
  unsigned long long* red_out = nullptr;   // [2]: argmax key, grid sum (null: not computed)
  unsigned int* red_done = nullptr;        // last-block counter (zero; reset by the kernel)
  struct PeakOut* peak = nullptr;          // null: no start axis
  uint32_t peak_min_votes = 1;
};

// K1: constraint basis (exact f64 -> f32) and band culling plan per constraint.
void launch_plan(const VotePlan& p, const VoteBuffers& b, int64_t n, cudaStream_t s);
// K2: band-tiled vote into smem tiles, flushed to partial slots; then tile reduction.
void launch_vote_banded(const VotePlan& p, const VoteBuffers& b, int64_t n, int n_ctas, cudaStream_t s);
cudaError_t set_vote_smem(const VotePlan& p);  // opt-in dynamic smem (once per size)
void launch_zero_i32(int32_t* p, int n, cudaStream_t s);
int vote_reduce_blocks_x(const VotePlan& p);  // blocks per band of vote_reduce_kernel
void launch_vote_reduce(const VotePlan& p, const VoteBuffers& b, cudaStream_t s);
// Exact generic vote (any config): one thread per (constraint, sample), global atomics.
void launch_vote_generic(const VotePlan& p, const VoteBuffers& b, int64_t n, cudaStream_t s);
// Single-constraint deposit on top of an existing grid (deposit_circle_votes).
void launch_deposit_one(const VotePlan& p, const double* z3, const double2* table64,
                        uint32_t* grid, cudaStream_t s);

// Preprocess (estimator.cpp:259-285): AoS correspondences -> SoA constraints, order-kept.
struct PrepBuffers {
  const double* corrs = nullptr;  // n x 6
  double* zx = nullptr;
  double* zy = nullptr;
  double* zz = nullptr;
  int32_t* kept = nullptr;
  int32_t* dropped = nullptr;
  unsigned long long* status = nullptr;  // [nblocks] look-back status (zeroed before launch)
  int32_t* block_counter = nullptr;      // dynamic block id (zeroed before launch)
  int32_t* totals = nullptr;             // [0]=n_kept [1]=n_dropped
  int32_t* chunk_hi = nullptr;           // optional: kept count through the end of this launch's range
  // in-order mode (launch_preprocess_inorder): z written at the input index (NaN = dropped), no
  // compaction. Blocks add their kept counts to *kept_acc (zero at rest); the last block of a
  // launch (ticket on *kept_done, reset by it) moves the sum to *kept_total and re-zeroes the
  // accumulator when `kept_publish` is set (the final launch of a solve) -- no memset needed.
  unsigned long long* kept_total = nullptr;
  unsigned long long* kept_acc = nullptr;
  unsigned int* kept_done = nullptr;
  int kept_publish = 1;
  // side job: word ranges to clear (the next vote's grid and counters -- saves separate memsets)
  uint32_t* zero_ptr[4] = {nullptr, nullptr, nullptr, nullptr};
  int64_t zero_n[4] = {0, 0, 0, 0};
};
int prep_blocks(int64_t n);
void launch_preprocess(const PrepBuffers& b, int64_t n, double tau_z, int normalize, cudaStream_t s);
// One chunk [elem_lo, elem_hi) of a pipelined preprocess (elem_lo multiple of 1024; chunks in order).
void launch_preprocess_range(const PrepBuffers& b, int64_t n, int64_t elem_lo, int64_t elem_hi, double tau_z,
                             int normalize, cudaStream_t s);
// In-order preprocess of [elem_lo, elem_hi) (elem_lo multiple of 1024): no look-back, no index maps.
void launch_preprocess_inorder(const PrepBuffers& b, int64_t n, int64_t elem_lo, int64_t elem_hi, double tau_z,
                               int normalize, cudaStream_t s);

// K3: peak search over a device grid (rv_peaks.cu).
struct Disk {
  int cx, cy;
};
int argmax_block_count();
// Argmax over cells not inside any disk (radius r): key = (count << 32) | (~index), count > 0.
void launch_argmax(const uint32_t* grid, int G, const Disk* disks, int n_disks, int r,
                   unsigned long long* block_keys, unsigned long long* out_key, unsigned int* done,
                   cudaStream_t s,
                   const uint32_t* mask = nullptr);
// find_peaks with more disks than the argmax kernel takes directly: a G*G suppression bit image
int max_direct_disks();
void launch_mark_disks(uint32_t* mask, int G, const Disk* disks, int n_disks, int r, cudaStream_t s);
int blur_block_count();
// Box-blurred argmax for up to 8 radii at once (voting.cpp:176-216). sat: (G+1)^2 u64 scratch;
// block_best: [blur_block_count()][8][2]; out_best: [n_radii][2] = (sum, index).
void launch_blur_argmax(const uint32_t* grid, int G, const int* radii, int n_radii, unsigned long long* sat,
                        unsigned long long* block_best, unsigned long long* out_best, unsigned int* done,
                        cudaStream_t s);

// K4: consensus / angle kernels (rv_refine.cu).
struct ClassifyOut {
  uint32_t* flags = nullptr;       // bitmask [ceil(n/32)]
  const uint32_t* prev = nullptr;  // previous bitmask (or null)
  int32_t* block_count = nullptr;  // [nblocks]
  double* block_scatter = nullptr; // [nblocks][6] (xx xy xz yy yz zz) over inliers
  int32_t* block_diff = nullptr;   // [nblocks] any flag word differs from prev
  double* result = nullptr;        // [8]: count, differs, scatter[6]
};
int classify_blocks(int64_t n);
// mode 0: classify + scatter over inliers; 1: scatter over all constraints; 2: classify only.
void launch_classify_mode(const double* zx, const double* zy, const double* zz, int64_t n, const double axis[3],
                          double eps, int mode, const ClassifyOut& o, int32_t* block_offsets, unsigned int* done,
                          cudaStream_t s);
// out_host (optional): mapped pinned memory receiving a copy of the list (zero-copy read-back).
void launch_compact_flags(const uint32_t* flags, int64_t n, const int32_t* map, const int32_t* block_offsets,
                          int32_t* out, cudaStream_t s, int32_t* out_host = nullptr);
// axis_dev / n_dev (optional): axis and index count read on the device (n_idx is then an upper
// bound used for the launch size).
void launch_vote_angles_k(const double axis[3], const double* corrs, const int32_t* idx, int64_t n_idx, int bin_count,
                          double tau, uint32_t* bins, double* raw, unsigned long long* counts, cudaStream_t s,
                          const double* axis_dev = nullptr, const long long* n_dev = nullptr,
                          int32_t* idx_host = nullptr);
void launch_peak_angle_k(const uint32_t* bins, int bin_count, const double* raw, int64_t n_raw, double* block_sums,
                         double* result, unsigned int* done, cudaStream_t s, const long long* n_dev = nullptr);
// model_support of K <= model_support_multi_max() candidates in one pass (block_counts: nblocks *
// 2 * model_support_multi_max() ints; result: [K][2])
// K candidates' angle votes / peak sums in one launch each (blockIdx.y = candidate; candidate k at
// idx + k*idx_stride, bins + k*bin_count, raw + k*raw_stride, and byte offset k*state_stride_b
// from axis_dev / n_dev / counts / result; block_sums: K * 2 * peak_angle_blocks(n); done: K
// counters). Per candidate identical to launch_vote_angles_k / launch_peak_angle_k.
void launch_vote_angles_batch_k(int K, const double* corrs, const int32_t* idx, size_t idx_stride, int64_t n_idx,
                                int bin_count, double tau, uint32_t* bins, double* raw, size_t raw_stride,
                                unsigned long long* counts, const double* axis_dev, const long long* n_dev,
                                size_t state_stride_b, cudaStream_t s);
int peak_angle_blocks(int64_t n_raw);
void launch_peak_angle_batch_k(int K, const uint32_t* bins, int bin_count, const double* raw, size_t raw_stride,
                               int64_t n_raw, double* block_sums, double* result, unsigned int* done,
                               const long long* n_dev, size_t state_stride_b, cudaStream_t s);
// estimate_multi's band strip on the device (no read-back): q-th smallest |axis.z| over the set
// bits of `band` (keys: >= band-size u64 scratch), strip = max(floor_strip, 1.25 * value) into
// strip_dev, then the strip of every constraint with |axis.z| < strip
void launch_band_strip_k(const uint32_t* band, int64_t n, const double* zx, const double* zy, const double* zz,
                         const double axis[3], long long q, double floor_strip, unsigned long long* keys,
                         double* strip_dev, uint8_t* removed, cudaStream_t s);
int model_support_multi_max();
void launch_model_support_multi_k(const double* zx, const double* zy, const double* zz, const int32_t* kept,
                                  const double* corrs, int64_t n, int K, const double (*axes)[3], const double* angles,
                                  double eps, double tau, uint32_t* band_flags, size_t band_stride,
                                  int32_t* block_counts, int32_t* result, unsigned int* done, cudaStream_t s);
void launch_model_support_k(const double* zx, const double* zy, const double* zz, const int32_t* kept,
                            const double* corrs, int64_t n, const double axis[3], double angle, double eps, double tau,
                            uint32_t* band_flags, int32_t* block_counts, int32_t* result, unsigned int* done,
                            cudaStream_t s);
// consensus_count (baselines.cpp:16-24) of m axes (AoS m x 3) over n constraints (AoS n x 3); counts
// must be zeroed. Exact: f32 filter with an f64 re-check near the band edge.
void launch_consensus_counts(const double* axes, int m, const double* z, int64_t n, double eps, uint32_t* counts,
                             int sms, cudaStream_t s);
void launch_strip_k(const double* zx, const double* zy, const double* zz, int64_t n, const double axis[3], double strip,
                    uint8_t* removed, cudaStream_t s);
void launch_strip_identity_k(const double* corrs, const int32_t* kept, int64_t n, int normalize, uint8_t* removed,
                             cudaStream_t s);
void launch_near_identity_k(const double* corrs, const int32_t* sub_kept, int64_t n, int normalize, uint32_t* flags,
                            int32_t* block_count, double* block_h, int32_t* block_offsets, double* result,
                            unsigned int* done, cudaStream_t s);
void launch_gather_residual(const double* zx, const double* zy, const double* zz, const int32_t* kept,
                            const uint8_t* removed, int64_t n, unsigned long long* status,
                            int32_t* block_counter, double* ozx, double* ozy, double* ozz, int32_t* okept,
                            int32_t* total, cudaStream_t s);

// Device-resident refine_loop / anneal_axis (rv_coop.cu): one cooperative launch per call.
struct CoopState {  // published by the kernel after each pass; read by the host at the end
  double axis[3];   // axis of the last classify (refine_loop) / current axis (anneal)
  double next[3];
  double e;
  double scatter[6];
  long long count;  // inliers of the last classify
  int slot;         // flags slot of the last pass (refine_loop copies the final bitmask to flags0)
  int done;
  int refits;
  int rank_deficient;
  long long local_count;  // this device's share of count (cross-device refine)
  int exchange_timeout;   // a peer device never published its line (cross-device refine)
};
// Peak -> start axis on the device (estimate_from_peak, estimator.cpp:94-101): the argmax key,
// interpolate_peak (estimator.cpp:32-47), backproject, canonicalize -- the host's op order.
struct PeakOut {
  double axis[3];
  double A, B;                // interpolated plane coordinates
  unsigned long long total;   // grid sum (exactness guard)
  int ix, iy;
  unsigned int votes;
  int ok;                     // 0: no cell reaches min_votes (NoPeak)
};
void launch_peak_axis(const unsigned long long* okey, const uint32_t* grid, int G, double E, uint32_t min_votes,
                      PeakOut* out, cudaStream_t s);
// Cross-device exchange of a sharded refine (rv_shard_refine): this device's rank among n_dev,
// every device's line buffer (kCoopXLineBytes each, zeroed before the first use), the solve's
// epoch (the same on every device, increasing across solves).
constexpr int kCoopMaxDev = 8;
constexpr size_t kCoopXLineBytes = (size_t)kCoopMaxDev * 16 * sizeof(double);
struct CoopExchange {
  int n_dev = 1, rank = 0;
  double* lines[kCoopMaxDev] = {};
  unsigned long long epoch = 0;
};
// K (<= coop_multi_max()) independent refine_loop / anneal_axis runs from their own start axes
// in ONE cooperative launch (shared per-pass exchange). Per candidate k: CoopState at
// (char*)state + k * state_stride, angle counts [2] zeroed at (char*)counts + k * state_stride,
// mode 0: final bitmask at flags_out + k * flag_stride (optional), inlier indices at
// compact_out + k * compact_stride (optional). block_part: its own buffer, grid * (8 K + 8) doubles,
// zeroed before the first use (not shared with launch_coop_refine's lines).
cudaError_t launch_coop_refine_multi(const double* zx, const double* zy, const double* zz, int64_t n, int mode,
                                     int refine, double eps, int K, const double (*axes)[3], const double* e0s,
                                     void* state, size_t state_stride, unsigned long long* counts, uint32_t* flags_out,
                                     size_t flag_stride, const int32_t* kept, int32_t* compact_out, size_t compact_stride,
                                     uint32_t* zero_bins, int n_bins, double* block_part, unsigned int* barrier,
                                     int grid, cudaStream_t s);
int coop_multi_max();
int coop_refine_grid(int sms);
int coop_tiles(int64_t n);
size_t coop_state_bytes();
// mode 0: refine_loop (estimator.cpp:51-69); mode 1: anneal_axis (estimator.cpp:145-160).
// axis0_dev (optional): start axis read on the device (overrides axis0).
cudaError_t launch_coop_refine(const double* zx, const double* zy, const double* zz, int64_t n, int mode, int refine,
                               double eps, double e0, const double axis0[3], const double* axis0_dev,
                               uint32_t* flags0, uint32_t* flags1,
                               int32_t* tile_count, int32_t* tile_offset, double* block_part, unsigned int* barrier,
                               void* state, int grid, cudaStream_t s, const int32_t* kept = nullptr,
                               int32_t* compact_out = nullptr, uint32_t* zero_bins = nullptr, int n_bins = 0,
                               unsigned long long* zero_counts = nullptr, const CoopExchange* xch = nullptr);

// ---- CSV ingest (rv_io.cu; io.cpp:66-101) ------------------------------------------------
struct CsvFallback {  // a field the device left to the host's from_chars
  int64_t start, end;   // byte range before trimming (line '\r' already removed)
  int64_t row;
  int32_t col, line;    // line: 0-based physical line
};
struct CsvBuffers {
  const uint8_t* text = nullptr;  // ends with '\n'
  int64_t nbytes = 0;
  int2* chunk = nullptr;          // per-8KB-chunk delimiter/newline counts -> exclusive offsets
  int2* totals = nullptr;         // (delimiters, newlines)
  uint32_t* dpos = nullptr;       // byte position of every ',' / '\n'
  int32_t* dline = nullptr;       // 0-based line of every delimiter
  int32_t* nl_delim = nullptr;    // delimiter index of every newline
  int nlines = 0, nfields = 0;
  int skip_first = 0;             // line 1 is a header (decided by the host, io.cpp:76-84)
  int8_t* status = nullptr;       // per line: blank / data / header / bad field count
  int32_t* row = nullptr;         // per line: data flag -> row index (exclusive scan)
  int32_t* block = nullptr;       // scan scratch
  int32_t* nrows = nullptr;       // total rows
  double* out = nullptr;          // rows x 6 f64 (the reference's Correspondence layout)
  int64_t cap_rows = 0;
  unsigned int* err_line = nullptr;  // min 1-based line with an error (~0u: none)
  CsvFallback* fb = nullptr;
  int fb_cap = 0;
  int32_t* fb_count = nullptr;
};
int csv_chunks(int64_t nbytes);
// stage 0: delimiter census + scan (the host then reads `totals`); stage 1: index, lines, rows,
// fields (the host then reads err_line / nrows / fb_count)
cudaError_t launch_csv_parse(const CsvBuffers& b, cudaStream_t s, int stage);
void launch_csv_scatter(const int64_t* idx, const double* vals, int n, double* out, cudaStream_t s);

}  // namespace rvb
