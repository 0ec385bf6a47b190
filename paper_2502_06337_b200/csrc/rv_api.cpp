// Host side of the B200 path: the C-ABI (include/rotavote_b200.h), the device context, and
// the estimator control flow (estimate_single / estimate_multi, refine_loop, rescue,
// sequential multi-model extraction) driving the sm_100a kernels. Every O(N) and O(N*J) step
// runs on the GPU; the host keeps the reference's O(1) decisions and 3x3 solves.
// Compiled with -ffp-contract=off: host arithmetic follows the reference op order.
#include <cuda_runtime.h>

#include <algorithm>
#include <charconv>
#include <string_view>
#include <array>
#include <iterator>
#include <chrono>
#include <deque>
#include <cmath>
#include <cstdio>
#include <atomic>
#include <cstdlib>
#include <random>
#include <thread>
#include <mutex>
#include <condition_variable>
#include <unistd.h>
#include <cstring>
#include <memory>
#include <numbers>
#include <string>
#include <vector>

#include "../../include/rotavote_b200.h"
#include "rv_internal.h"
#include "rv_linalg.hpp"

using namespace rvb;

namespace {

struct RvError {
  rv_status st;
  std::string msg;
};

[[noreturn]] void fail(rv_status st, const std::string& msg) { throw RvError{st, msg}; }

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail(RV_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// Bumped whenever a device or mapped buffer is (re)allocated: captured solve graphs hold raw
// pointers and are only replayed while the generation they were captured at is current.
std::atomic<uint64_t> g_buf_gen{0};

struct DBuf {
  void* p = nullptr;
  size_t cap = 0;
  template <typename T>
  T* get(size_t count) {
    const size_t bytes = std::max<size_t>(count * sizeof(T), 16);
    if (bytes > cap) {
      if (p) cudaFree(p);
      p = nullptr;
      cap = 0;
      const size_t want = bytes + bytes / 4;
      g_buf_gen.fetch_add(1);
      if (cudaMalloc(&p, want) != cudaSuccess) {
        cudaGetLastError();
        fail(RV_ERR_OUT_OF_MEMORY, "cudaMalloc failed");
      }
      cap = want;
    }
    return static_cast<T*>(p);
  }
  ~DBuf() {
    if (p) cudaFree(p);
  }
};

struct StageEvent {
  int stage;
  cudaEvent_t a, b;
};

enum Stage { kPrep = 0, kVote = 1, kPeaks = 2, kRefine = 3, kAngles = 4, kVoteKernel = 5 };

struct Peak {
  int ix, iy;
  double A, B;
  uint32_t votes;
};

struct Estimate {
  double axis[3] = {0, 0, -1};
  double angle = 0;
  double R[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
  uint32_t votes = 0;
  std::vector<int32_t> inliers;
  double elapsed = 0;
  // single solves through the C-ABI: the inlier list stays in the context's mapped buffer (the
  // kernels streamed it there) and rv_result_inliers copies it once, straight from there
  const int32_t* view = nullptr;
  int64_t view_n = 0;
  int64_t dev_count = -1;  // >= 0: inliers not read back yet (left in a device buffer)
  int64_t n_inliers() const { return view ? view_n : dev_count >= 0 ? dev_count : (int64_t)inliers.size(); }
};

// Constraint set on the device (SoA) with its kept map (constraint -> input index).
struct ConstraintSet {
  const double* zx = nullptr;
  const double* zy = nullptr;
  const double* zz = nullptr;
  const int32_t* kept = nullptr;
  int64_t n = 0;
};

// Parallel host memcpy (pageable -> pinned staging of large single-solve inputs): a few worker
// threads, each copying a contiguous slice; the caller copies the first slice itself.
class CopyPool {
 public:
  explicit CopyPool(int threads) {
    for (int t = 1; t < threads; ++t)
      th_.emplace_back([this, t] {
        int seen = 0;
        for (;;) {
          Job j;
          {
            std::unique_lock<std::mutex> lk(mu_);
            cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
            if (stop_) return;
            seen = gen_;
            j = job_;
          }
          slice(j, t);
          std::lock_guard<std::mutex> lk(mu_);
          if (--pending_ == 0) done_.notify_all();
        }
      });
  }
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
  }
  void copy(void* dst, const void* src, size_t bytes) {
    const int parts = (int)th_.size() + 1;
    if (parts == 1 || bytes < ((size_t)1 << 20)) {
      std::memcpy(dst, src, bytes);
      return;
    }
    Job j{static_cast<char*>(dst), static_cast<const char*>(src), bytes, parts};
    {
      std::lock_guard<std::mutex> lk(mu_);
      job_ = j;
      pending_ = parts - 1;
      ++gen_;
    }
    cv_.notify_all();
    slice(j, 0);
    std::unique_lock<std::mutex> lk(mu_);
    done_.wait(lk, [&] { return pending_ == 0; });
  }

 private:
  struct Job {
    char* dst = nullptr;
    const char* src = nullptr;
    size_t bytes = 0;
    int parts = 1;
  };
  static void slice(const Job& j, int t) {
    const size_t lo = (j.bytes * (size_t)t / (size_t)j.parts) & ~(size_t)63;
    const size_t hi = t + 1 == j.parts ? j.bytes : (j.bytes * (size_t)(t + 1) / (size_t)j.parts) & ~(size_t)63;
    if (hi > lo) std::memcpy(j.dst + lo, j.src + lo, hi - lo);
  }
  std::vector<std::thread> th_;
  std::mutex mu_;
  std::condition_variable cv_, done_;
  Job job_;
  int gen_ = 0, pending_ = 0;
  bool stop_ = false;
};

}  // namespace

struct rv_context {
  int device = 0;
  int sms = 148;
  int max_smem = 0;
  cudaStream_t own = nullptr;
  cudaStream_t st = nullptr;
  std::string last_error;
  bool timing = false;
  rv_stage_times times{};
  std::vector<StageEvent> events;
  std::vector<cudaEvent_t> event_pool;
  size_t event_used = 0;
  std::chrono::steady_clock::time_point t0;

  // preprocess
  DBuf corrs, zx, zy, zz, kept, dropped, status, misc32;
  // residual (estimate_multi)
  DBuf rzx, rzy, rzz, rkept, removed;
  // vote
  DBuf basis_a, basis_b, ranges, band_work, table32, table64, grid, partials, slot_band, counters, stats, degen;
  // sharded solve: the constraint set of the last rv_vote_shard and the step state
  ConstraintSet shard_cs{};
  const double* shard_corrs = nullptr;
  int64_t shard_m = 0;               // inliers compacted by rv_shard_inliers
  const int32_t* shard_idx = nullptr;
  struct ShardCls {
    uint32_t* flags = nullptr;
    int32_t* offsets = nullptr;
    int64_t count = -1;
  } shard_cls[2];
  int table_J = -1;
  // peaks
  DBuf arg_keys, arg_out, sat, blur_best, blur_out, done, peak_mask;
  // classify / refine
  DBuf flagsA, flagsB, bcount, bscatter, bdiff, boffA, boffB, cls_result, compact_out;
  DBuf coop_part, coop_state, coop_bar;  // device-resident refine_loop / anneal_axis (rv_coop.cu)
  DBuf peak_out;                         // chained solve: device Summary (peak, state, angles)
  DBuf red_keys;                         // fused argmax scratch of the tile reduction
  DBuf kept_acc;                          // in-order preprocess: kept-count accumulator + ticket
  DBuf cand_sums, cand_idx, cand_sup, cand_band;  // batched rescue candidates (per-candidate slots)
  // CSV ingest (rv_io.cu)
  DBuf csv_text, csv_chunk, csv_misc, csv_dpos, csv_dline, csv_nl, csv_status, csv_row, csv_block, csv_out, csv_fb,
      csv_fix_idx, csv_fix_val;
  char* csv_pinned = nullptr;             // pinned staging of file contents
  size_t csv_pinned_cap = 0;
  double* in_pinned = nullptr;            // pinned staging of small pageable single-solve inputs
  size_t in_pinned_cap = 0;
  double* big_pinned = nullptr;           // pinned staging of large pageable inputs (chunked, parallel copies)
  size_t big_pinned_cap = 0;
  std::unique_ptr<CopyPool> copy_pool;
  bool kept_acc_ready = false;
  DBuf cons_axes, cons_counts, cons_z, cons_idx;  // baseline consensus scoring
  int coop_grid = 0;
  bool coop_bar_ready = false;
  void* xlines_own = nullptr;              // this context's line buffer for a cross-process refine
  std::vector<void*> xlines_peers;          // peer ranks' line buffers mapped by CUDA IPC
  const double* coop_part_zeroed = nullptr;
  DBuf coop_mpart;                          // line buffer of the K-candidate cooperative refine
  const double* coop_mpart_zeroed = nullptr;
  // angles / support
  DBuf bins, raw, angle_counts, angle_sums, angle_result, sup_counts, sup_result, band_flagsA, band_flagsB,
      band_vals, near_h, near_result, strip_val;
  DBuf user_z;  // scratch copy of a constraint span (path functions)
  DBuf chunk_hi;                          // pipelined vote: kept count at each chunk end
  cudaStream_t copy_st = nullptr;         // H2D copies of the pipelined host path
  cudaStream_t cap_st = nullptr;          // capture stream of the solve graphs
  struct SolveGraph {                     // device-resident single solve, captured once, replayed
    const double* corrs = nullptr;        // device input, or the pinned host input (host = true)
    bool host = false;
    const void* aux = nullptr;            // prevoted solves / shard votes: the grid
    int kind = 0;                         // 0 single solve, 1 prevoted finish, 2 shard vote
    int64_t n = 0;
    rv_config cfg{};
    uint64_t gen = 0;
    int seen = 0;                         // eager runs with this key (capture on the second)
    cudaGraphExec_t exec = nullptr;
    rv_stage_times delta{};               // host-side counters the captured enqueue added
  };
  std::vector<SolveGraph> graphs;
  std::vector<cudaEvent_t> chunk_events;
  std::deque<std::pair<VotePlan, int>> plans;  // vote plans by (G, E, J)
  // pinned host scalars
  void* pinned = nullptr;
  std::vector<std::vector<int32_t>> results;
  std::vector<int32_t> spare;       // recycled inlier vector (no page faults on the hot path)
  std::vector<std::vector<int32_t>> spares;  // recycled inlier vectors of the multi-model calls
  bool allow_view = false;          // set by the single-solve entry points (see Estimate::view)
  const int32_t* result0_view = nullptr;  // results[0] lives in the mapped buffer (view)
  int64_t result0_view_n = 0;
  std::vector<rv_context*> pool;    // batch workers (own stream + buffers each), created lazily
  int32_t* inl_host = nullptr;      // mapped pinned buffer: the compaction writes the inlier list here
  size_t inl_cap = 0;
  std::vector<std::vector<uint64_t>> dedupe_bits;  // estimate_multi's inlier bitsets (InlierSets)

  // "last block done" counters of the single-pass reductions: must start at zero; every kernel
  // that uses one resets it before exiting.
  unsigned int* done_ptr() {
    if (!done.p) {
      done.get<unsigned int>(8);
      if (cudaMemset(done.p, 0, done.cap) != cudaSuccess) fail(RV_ERR_CUDA, "memset done counter");
    }
    return static_cast<unsigned int*>(done.p);
  }
};

namespace {

double* pin_d(rv_context* c) { return static_cast<double*>(c->pinned); }
constexpr size_t kPinnedScratch = 4096;  // c->pinned

void sync(rv_context* c) { ck(cudaStreamSynchronize(c->st), "cudaStreamSynchronize"); }

cudaEvent_t take_event(rv_context* c) {
  if (c->event_used == c->event_pool.size()) {
    cudaEvent_t e;
    ck(cudaEventCreate(&e), "cudaEventCreate");
    c->event_pool.push_back(e);
  }
  return c->event_pool[c->event_used++];
}

// Read-back of a few small records (then synchronise): through the pinned scratch when they fit
// -- a pageable D2H stages through the driver, ~10-20 us more per read-back in the multi-model loop
template <class T>
void read_small(rv_context* c, T* dst, const T* src, size_t count, const char* what) {
  const size_t bytes = sizeof(T) * count;
  void* via = bytes <= kPinnedScratch ? c->pinned : static_cast<void*>(dst);
  ck(cudaMemcpyAsync(via, src, bytes, cudaMemcpyDeviceToHost, c->st), what);
  sync(c);
  if (via != dst) std::memcpy(dst, via, bytes);
}

struct StageScope {
  rv_context* c;
  int stage;
  cudaEvent_t a = nullptr;
  StageScope(rv_context* cc, int s) : c(cc), stage(s) {
    if (c->timing) {
      a = take_event(c);
      cudaEventRecord(a, c->st);
    }
  }
  ~StageScope() {
    if (c->timing) {
      cudaEvent_t b = take_event(c);
      cudaEventRecord(b, c->st);
      c->events.push_back({stage, a, b});
    }
  }
};

void begin_call(rv_context* c) {
  c->allow_view = false;  // only the single-solve entry points opt in (after begin_call)
  c->times = rv_stage_times{};
  c->events.clear();
  c->event_used = 0;
  c->t0 = std::chrono::steady_clock::now();
  c->last_error.clear();
}

void end_call(rv_context* c) {
  if (!c->timing) return;
  sync(c);
  for (const auto& e : c->events) {
    float ms = 0;
    cudaEventElapsedTime(&ms, e.a, e.b);
    switch (e.stage) {
      case kPrep: c->times.preprocess_ms += ms; break;
      case kVote: c->times.vote_ms += ms; break;
      case kPeaks: c->times.peaks_ms += ms; break;
      case kRefine: c->times.refine_ms += ms; break;
      case kVoteKernel: c->times.vote_kernel_ms += ms; break;  // nested in kVote: not in total
      default: c->times.angles_ms += ms; break;
    }
  }
  c->times.total_ms = c->times.preprocess_ms + c->times.vote_ms + c->times.peaks_ms + c->times.refine_ms +
                      c->times.angles_ms;
}

void count_launch(rv_context* c, int k = 1) { c->times.kernel_launches += k; }

// ---------------------------------------------------------------------------------------
// Vote plan (geometry of the band-tiled kernel) for (grid, extent, samples).
VotePlan make_plan(rv_context* c, int G, double E, int J) {
  VotePlan p;
  p.G = G;
  p.J = J;
  p.E = E;
  p.inv_cell = G / (2.0 * E);  // voting.cpp:30
  p.cs = 2.0 * E / G;          // voting.hpp:23
  p.halfJ = J / 2;
  p.step_f = (float)(2.0 * std::numbers::pi / J);
  p.banded = 0;
  // twins j, j+J/2 and 64-aligned pair ranges; queue entries hold the pair in 16 bits
  const bool twins_ok = (J % 128 == 0) && p.halfJ <= 32768;
  // Fixed-point shift S of the f32 filter (K2 item 2), the largest S <= 13 with
  //  (range)    t = G/2 + X*K, |X| <= 1, stays inside the magic binade: |t| < 2^(22-S);
  //  (accuracy) the flag window [-2u, 2u), u = 2^-S, covers the f32 error bound:
  //             |t32 - t| <= K*6e-7 (inputs, FMUL/FFMA, FADD, rcp.approx) + u/2  <  2u,
  //             checked with a 10% allowance (6.6e-7). No S -> the exact generic kernel.
  const double Kc = p.inv_cell;
  auto shift_ok = [&](int S) {
    const double half = std::ldexp(1.0, 22 - S);
    const double lo = 0.5 * G - 1.01 * Kc - 4.0, hi = 0.5 * G + 1.01 * Kc + 4.0;
    return lo >= -half && hi < half && Kc * 6.6e-7 < 1.5 * std::ldexp(1.0, -S);
  };
  int S = 13;
  while (S >= 8 && !shift_ok(S)) --S;
  if (!twins_ok || S < 8) return p;
  p.frac_shift = S;
  p.frac_mask = ((1u << S) - 1u) & ~3u;
  const double magic = 1.5 * std::ldexp(1.0, 23 - S);
  const float magic_f = (float)magic;
  uint32_t magic_bits;
  std::memcpy(&magic_bits, &magic_f, 4);
  p.magic_hi = (int)(magic_bits >> S);
  p.Kf = (float)p.inv_cell;
  // E*inv_cell == G/2 exactly in real arithmetic; +2 units of 2^-S bias the frac window to [-2, 1]
  p.CMf = (float)(magic + 0.5 * G + 2.0 * std::ldexp(1.0, -S));
  p.clamp = E <= 1.0 + 1e-6 ? 1 : 0;
  const double lo_t = (E - 1.0) * p.inv_cell, hi_t = (E + 1.0) * p.inv_cell;
  if (p.clamp) {
    p.r_min = 0;
    p.r_max = G - 1;
  } else {
    p.r_min = std::max(0, (int)std::floor(lo_t) - 2);
    p.r_max = std::min(G - 1, (int)std::ceil(hi_t) + 1);
  }
  p.c_min = p.r_min;
  p.c_max = p.r_max;
  p.W = p.c_max - p.c_min + 1;
  // full-width tiles when the grid rows are 16-byte multiples: the vote flushes a band tile into
  // the grid with TMA bulk reduce-adds (no partial slots to reduce); costs the unreachable
  // columns of shared memory per row (24 of 516 at the defaults; the band count is unchanged)
  static const bool bulk_on = [] {
    const char* e = std::getenv("RV_BULK");
    return !(e && e[0] == '0');
  }();
  if (bulk_on && G % 4 == 0) {
    p.bulk = 1;
    p.c_min = 0;
    p.c_max = G - 1;
    p.W = G + 4;  // row stride: 16-byte rows for the bulk copies, rows offset by 4 banks
  }
  p.Wf = (float)p.W;
  const size_t table_bytes = (size_t)(2 * p.halfJ + 64) * sizeof(float2);  // J samples (packed) + 64 slack
  const size_t fbq_bytes = (size_t)(kVoteThreads / 32) * kFbqCap * 4 + 32 * 4;  // + 32 lane sink words
  const size_t reserve = table_bytes + fbq_bytes + 1024;
  if ((size_t)c->max_smem <= reserve) return p;
  const size_t budget_words = ((size_t)c->max_smem - reserve) / 4;
  const int h_allowed = (int)(budget_words / p.W);
  if (h_allowed < 1) return p;
  const int rows = p.r_max - p.r_min + 1;
  const int nb = (rows + h_allowed - 1) / h_allowed;
  if (nb > kMaxBands) return p;
  const int H = (rows + nb - 1) / nb;
  p.n_bands = nb;
  p.H_max = H;
  for (int b = 0; b <= nb; ++b) p.band_r0[b] = std::min(p.r_min + b * H, p.r_max + 1);
  // band boundaries in plane units; the planner solves each boundary once and dilates / erodes
  // the solution for the bands on either side (culling margin)
  for (int b = 0; b < nb; ++b) {
    p.band_ylo[b] = b == 0 ? -INFINITY : (float)(-E + p.band_r0[b] * p.cs);
    p.band_yhi[b] = b == nb - 1 ? INFINITY : (float)(-E + p.band_r0[b + 1] * p.cs);
  }
  p.tile_words = ((size_t)H * p.W + 3) & ~size_t(3);  // multiple of 4: 16-byte aligned partial slots
  p.smem_bytes = (((p.tile_words + 32) * 4 + 15) & ~size_t(15)) + table_bytes + fbq_bytes;  // tile + sinks
  p.banded = p.smem_bytes <= (size_t)c->max_smem ? 1 : 0;
  return p;
}

const VotePlan& cached_plan(rv_context* c, int G, double E, int J) {
  for (const auto& e : c->plans)
    if (e.first.G == G && e.first.E == E && e.first.J == J) return e.first;
  VotePlan p = make_plan(c, G, E, J);
  if (p.banded) {  // opt-in shared memory once per plan
    ck(set_vote_smem(p), "cudaFuncSetAttribute");
  }
  c->plans.emplace_back(p, 0);
  return c->plans.back().first;
}

// Sample table exactly as the reference (voting.cpp:72-81), on the host libm.
void ensure_tables(rv_context* c, int J) {
  if (c->table_J == J) return;
  std::vector<double2> t64(J);
  const double step = 2.0 * std::numbers::pi / J;
  for (int j = 0; j < J; ++j) {
    const double theta = -std::numbers::pi + j * step;
    t64[j] = make_double2(std::cos(theta), std::sin(theta));
  }
  std::vector<float2> t32(std::max(J, 1));  // every sample: the vote reads canonical samples only
  for (int j = 0; j < J; ++j) t32[j] = make_float2((float)t64[j].x, (float)t64[j].y);
  ck(cudaMemcpyAsync(c->table64.get<double2>(J), t64.data(), sizeof(double2) * J, cudaMemcpyHostToDevice, c->st),
     "table64");
  ck(cudaMemcpyAsync(c->table32.get<float2>(std::max(J, 1)), t32.data(), sizeof(float2) * std::max(J, 1),
                     cudaMemcpyHostToDevice, c->st),
     "table32");
  sync(c);
  c->table_J = J;
}

// Device summary of a chained single solve: every scalar the host needs, read back in one copy.
struct Summary {
  PeakOut pk;
  CoopState st;
  unsigned long long counts[2];
  double angle[4];
  unsigned long long n_kept;  // in-order constraint sets: kept pairs, counted by the preprocess
};
Summary* summary_buf(rv_context* c) { return c->peak_out.get<Summary>(1); }

// Optional outputs fused into the vote's tile reduction (banded kernel only).
struct VoteFused {
  unsigned long long* key_out = nullptr;  // [2]: argmax key, grid sum
  PeakOut* peak = nullptr;                // start axis (estimate_from_peak)
  bool done = false;                      // set by vote(): the reduction produced them
};
void set_fused(rv_context* c, VoteBuffers& b, VoteFused* f, const VotePlan& p) {
  if (!f) return;
  b.red_keys = c->red_keys.get<unsigned long long>((size_t)2 * vote_reduce_blocks_x(p) * p.n_bands);
  b.red_out = f->key_out;
  b.red_done = c->done_ptr();
  b.peak = f->peak;
  b.peak_min_votes = 1u;
  f->done = true;
}

// accumulate (voting.cpp:88-118) over device SoA constraints into the context grid.
// prezeroed: the grid and the band counters were already cleared (by the preprocess kernel).
// CTAs of a band-tiled vote launch: one per ~16k planned pairs (a CTA's fixed cost -- clearing and
// flushing its tile -- is a few microseconds, so even small problems spread over many SMs), at
// least one per band, at most one per SM.
#ifndef RV_VOTE_CTA_SHIFT
#define RV_VOTE_CTA_SHIFT 14  // one vote CTA per 2^shift planned pairs (small problems use fewer CTAs)
#endif
int vote_ctas(const rv_context* c, const VotePlan& p, int64_t est_pairs) {
  return (int)std::clamp<int64_t>(est_pairs >> RV_VOTE_CTA_SHIFT, std::min(p.n_bands, c->sms), c->sms);
}

uint32_t* vote(rv_context* c, const double* zx, const double* zy, const double* zz, int64_t n, int G, double E,
               int J, bool force_generic = false, bool prezeroed = false, VoteFused* fused = nullptr) {
  if (n <= 0) fail(RV_ERR_EMPTY_INPUT, "no constraints to accumulate");
  if (G < 1 || !(E > 0.0)) fail(RV_ERR_INVALID_CONFIG, "accumulator needs grid >= 1, extent > 0");
  if (J < 1) fail(RV_ERR_INVALID_CONFIG, "theta_samples must be >= 1");
  ensure_tables(c, J);
  const VotePlan& p = cached_plan(c, G, E, J);
  uint32_t* grid = c->grid.get<uint32_t>((size_t)G * G);
  StageScope sc(c, kVote);
  if (!prezeroed || !p.banded || force_generic)
    ck(cudaMemsetAsync(grid, 0, sizeof(uint32_t) * (size_t)G * G, c->st), "memset grid");
  VoteBuffers b;
  b.zx = zx;
  b.zy = zy;
  b.zz = zz;
  b.grid = grid;
  b.table64 = c->table64.get<double2>(J);
  b.table32 = c->table32.get<float2>(std::max(J, 1));
  c->times.vote_samples += n * (int64_t)J;
  c->times.vote_launches += 1;
  if (!p.banded || force_generic) {
    launch_vote_generic(p, b, n, c->st);
    count_launch(c);
    ck(cudaGetLastError(), "vote_generic");
    return grid;
  }
  b.basis_a = c->basis_a.get<float4>(n);
  b.basis_b = c->basis_b.get<float2>(n);
  b.entry_cap = kEntriesPerConstraint * n;
  b.degen = c->degen.get<int32_t>(n);
  b.entries = c->ranges.get<unsigned long long>((size_t)b.entry_cap * p.n_bands);
  b.band_work = c->band_work.get<unsigned long long>(kMaxBands);
  b.counters = c->counters.get<int32_t>(kCounterWords);
  b.entry_count = b.counters + kMaxBands + 1;
  b.stats = c->stats.get<unsigned long long>(2);
  // enough CTAs to keep every SM busy, but not more than the work can feed (vote_ctas: one CTA per
  // 16k planned pairs, at least one per band, at most one per SM)
  const int64_t est_pairs = n * (int64_t)p.halfJ;
  const int n_ctas = vote_ctas(c, p, est_pairs);
  b.max_slots = p.bulk ? 0 : n_ctas * p.n_bands;  // bulk: tiles are reduced into the grid directly
  if (!p.bulk) {
    b.partials = c->partials.get<uint32_t>((size_t)b.max_slots * p.tile_words);
    b.slot_band = c->slot_band.get<int32_t>(b.max_slots);
  }
  if (!prezeroed) {
    ck(cudaMemsetAsync(b.band_work, 0, sizeof(unsigned long long) * kMaxBands, c->st), "memset band_work");
    ck(cudaMemsetAsync(b.counters, 0, sizeof(int32_t) * kCounterWords, c->st), "memset counters");
    ck(cudaMemsetAsync(b.stats, 0, sizeof(unsigned long long) * 2, c->st), "memset stats");
  }
  set_fused(c, b, fused, p);
  launch_plan(p, b, n, c->st);
  {
    StageScope kv(c, kVoteKernel);
    launch_vote_banded(p, b, n, n_ctas, c->st);
  }
  if (!p.bulk || b.red_out) {  // bulk tiles are already in the grid: reduce only for the fused argmax
    launch_vote_reduce(p, b, c->st);
    count_launch(c);
  }
  count_launch(c, 2);
  ck(cudaGetLastError(), "vote_banded");
  if (c->timing) {
    unsigned long long st[2], work[kMaxBands];
    ck(cudaMemcpyAsync(st, b.stats, sizeof st, cudaMemcpyDeviceToHost, c->st), "stats");
    ck(cudaMemcpyAsync(work, b.band_work, sizeof(unsigned long long) * p.n_bands, cudaMemcpyDeviceToHost, c->st),
       "band work");
    sync(c);
    for (int q = 0; q < p.n_bands; ++q) c->times.vote_pairs += (int64_t)work[q];
    c->times.vote_fallback_pairs += (int64_t)st[1];
  }
  return grid;
}

// ---------------------------------------------------------------------------------------
// Peaks
double cell_center(int i, int G, double E) { return -E + (i + 0.5) * (2.0 * E / G); }
int coord_to_cell(double v, int G, double E) {  // voting.cpp:17-23, :55-57
  const double inv_cell = G / (2.0 * E);
  const double t = (v + E) * inv_cell;
  const double f = std::floor(t);
  int i = (int)f;
  if (f == t && i > 0) --i;
  return std::clamp(i, 0, G - 1);
}

// find_peaks (voting.cpp:120-170): greedy; device argmax per round, host NMS bookkeeping.
std::vector<Peak> find_peaks_dev(rv_context* c, const uint32_t* grid, int G, double E, int max_peaks, int radius,
                                 uint32_t min_votes, unsigned long long* grid_total = nullptr) {
  StageScope sc(c, kPeaks);
  std::vector<Peak> out;
  std::vector<Disk> disks;
  const double cs = 2.0 * E / G;
  unsigned long long* keys = c->arg_keys.get<unsigned long long>(2 * argmax_block_count());
  unsigned long long* okey = c->arg_out.get<unsigned long long>(2);
  // up to max_direct_disks() suppression disks go to the argmax kernel directly; beyond that (any
  // K, like the reference) the disks are painted into a G*G suppression bit image incrementally
  uint32_t* mask = nullptr;
  size_t painted = 0;
  for (int k = 0; k < max_peaks; ++k) {
    if (!mask && (int)disks.size() > max_direct_disks()) {
      const size_t words = ((size_t)G * G + 31) / 32;
      mask = c->peak_mask.get<uint32_t>(words);
      ck(cudaMemsetAsync(mask, 0, sizeof(uint32_t) * words, c->st), "memset peak mask");
    }
    if (mask && painted < disks.size()) {
      launch_mark_disks(mask, G, disks.data() + painted, (int)(disks.size() - painted), radius, c->st);
      count_launch(c);
      painted = disks.size();
    }
    launch_argmax(grid, G, disks.data(), (int)disks.size(), radius, keys, okey, c->done_ptr(), c->st, mask);
    count_launch(c);
    unsigned long long* hk = reinterpret_cast<unsigned long long*>(c->pinned);
    ck(cudaMemcpyAsync(hk, okey, 16, cudaMemcpyDeviceToHost, c->st), "argmax D2H");
    sync(c);
    const unsigned long long key = hk[0];
    if (k == 0 && grid_total) *grid_total = hk[1];
    if (key == 0) break;
    const uint32_t best = (uint32_t)(key >> 32);
    const uint32_t idx = 0xFFFFFFFFu - (uint32_t)(key & 0xFFFFFFFFu);
    if (best < min_votes) break;
    Peak pk;
    pk.iy = (int)idx / G;
    pk.ix = (int)idx % G;
    pk.A = cell_center(pk.ix, G, E);
    pk.B = cell_center(pk.iy, G, E);
    pk.votes = best;
    out.push_back(pk);
    disks.push_back({pk.ix, pk.iy});
    const double norm = std::hypot(pk.A, pk.B);
    if (std::abs(norm - 1.0) <= 1.5 * cs && norm > 0.0) {
      const double mx = -pk.A / norm, my = -pk.B / norm;
      disks.push_back({coord_to_cell(mx, G, E), coord_to_cell(my, G, E)});
    }
  }
  if (out.empty()) fail(RV_ERR_NO_PEAK, "no accumulator cell reaches min_votes");
  return out;
}

// A failed exactness guard (the planner under- or over-covered a sample) is counted and repaired by
// an exact re-vote; RV_STRICT_GUARD=1 (the GPU test-suite) turns it into an error instead, so a
// coverage bug cannot hide behind the repair.
void guard_failed(rv_context* c, unsigned long long total, unsigned long long expect) {
  static const bool strict = [] {
    const char* e = std::getenv("RV_STRICT_GUARD");
    return e && e[0] == '1';
  }();
  c->times.vote_guard_reruns += 1;
  if (strict)
    fail(RV_ERR_CUDA, "exactness guard: vote grid sums to " + std::to_string(total) + ", expected " +
                          std::to_string(expect) + " (RV_STRICT_GUARD)");
}

// accumulate + find_peaks(K=1) with the exactness guard: every constraint deposits exactly J
// votes (voting.cpp:33-44), so the grid must sum to n*J. If the band planner ever under-covered a
// sample the sum would be short: the vote is then redone with the generic exact kernel.
std::pair<const uint32_t*, std::vector<Peak>> vote_and_peak(rv_context* c, const double* zx, const double* zy,
                                                            const double* zz, int64_t n, const rv_config& cfg,
                                                            uint32_t min_votes, bool allow_no_peak,
                                                            const uint32_t* prevoted = nullptr,
                                                            int first_attempt = 0) {
  for (int attempt = first_attempt; attempt < 2; ++attempt) {
    const uint32_t* grid = (attempt == 0 && prevoted)
                               ? prevoted
                               : vote(c, zx, zy, zz, n, cfg.grid, cfg.extent, cfg.theta_samples, attempt == 1);
    unsigned long long total = 0;
    std::vector<Peak> peaks;
    try {
      peaks = find_peaks_dev(c, grid, cfg.grid, cfg.extent, 1, cfg.suppression_radius, min_votes, &total);
    } catch (const RvError& e) {
      if (e.st != RV_ERR_NO_PEAK || !allow_no_peak) throw;
      if (total == 0) {  // NoPeak: re-read the total for the guard
        unsigned long long* keys = c->arg_keys.get<unsigned long long>(2 * argmax_block_count());
        unsigned long long* okey = c->arg_out.get<unsigned long long>(2);
        launch_argmax(grid, cfg.grid, nullptr, 0, cfg.suppression_radius, keys, okey, c->done_ptr(), c->st);
        unsigned long long* hk = reinterpret_cast<unsigned long long*>(c->pinned);
        ck(cudaMemcpyAsync(hk, okey, 16, cudaMemcpyDeviceToHost, c->st), "argmax D2H");
        sync(c);
        total = hk[1];
      }
    }
    if (total == (unsigned long long)n * (unsigned long long)cfg.theta_samples) return {grid, peaks};
    guard_failed(c, total, (unsigned long long)n * (unsigned long long)cfg.theta_samples);
  }
  fail(RV_ERR_CUDA, "vote grid total mismatch after exact rerun");
}

// blurred_argmax for a list of radii (voting.cpp:176-216)
std::vector<Peak> blurred_argmax_dev(rv_context* c, const uint32_t* grid, int G, double E, const std::vector<int>& radii) {
  StageScope sc(c, kPeaks);
  std::vector<Peak> out;
  if (radii.empty()) return out;
  unsigned long long* sat = c->sat.get<unsigned long long>((size_t)(G + 1) * (G + 1));
  unsigned long long* bb = c->blur_best.get<unsigned long long>((size_t)blur_block_count() * 16);
  unsigned long long* ob = c->blur_out.get<unsigned long long>(16);
  for (size_t off = 0; off < radii.size(); off += 8) {
    const int nr = (int)std::min<size_t>(8, radii.size() - off);
    launch_blur_argmax(grid, G, radii.data() + off, nr, sat, bb, ob, c->done_ptr(), c->st);
    count_launch(c, 3);
    unsigned long long* h = reinterpret_cast<unsigned long long*>(c->pinned);
    ck(cudaMemcpyAsync(h, ob, sizeof(unsigned long long) * 2 * nr, cudaMemcpyDeviceToHost, c->st), "blur D2H");
    sync(c);
    for (int k = 0; k < nr; ++k) {
      const unsigned long long sum = h[2 * k], idx = h[2 * k + 1];
      Peak pk;
      pk.iy = (int)(idx / G);
      pk.ix = (int)(idx % G);
      pk.A = cell_center(pk.ix, G, E);
      pk.B = cell_center(pk.iy, G, E);
      pk.votes = (uint32_t)std::min<unsigned long long>(sum, 0xFFFFFFFFull);
      out.push_back(pk);
    }
  }
  return out;
}

// interpolate_peak (estimator.cpp:32-47): 3x3 vote-weighted centroid from the device grid.
void interpolate_peak_dev(rv_context* c, const uint32_t* grid, int G, double E, const Peak& pk, double* A, double* B) {
  const int x0 = std::max(0, pk.ix - 1), x1 = std::min(G - 1, pk.ix + 1);
  const int y0 = std::max(0, pk.iy - 1), y1 = std::min(G - 1, pk.iy + 1);
  uint32_t* h = reinterpret_cast<uint32_t*>(c->pinned);
  const int w = x1 - x0 + 1, hgt = y1 - y0 + 1;
  ck(cudaMemcpy2DAsync(h, sizeof(uint32_t) * 3, grid + (size_t)y0 * G + x0, sizeof(uint32_t) * G,
                       sizeof(uint32_t) * w, hgt, cudaMemcpyDeviceToHost, c->st),
     "interp D2H");
  sync(c);
  double wsum = 0.0, asum = 0.0, bsum = 0.0;
  for (int dy = -1; dy <= 1; ++dy) {
    for (int dx = -1; dx <= 1; ++dx) {
      const int ix = pk.ix + dx, iy = pk.iy + dy;
      if (ix < 0 || ix >= G || iy < 0 || iy >= G) continue;
      const double wv = h[(iy - y0) * 3 + (ix - x0)];
      const double cA = cell_center(ix, G, E), cB = cell_center(iy, G, E);
      wsum += wv;
      asum += wv * cA;
      bsum += wv * cB;
    }
  }
  if (wsum <= 0.0) {
    *A = pk.A;
    *B = pk.B;
    return;
  }
  *A = asum / wsum;
  *B = bsum / wsum;
}

uint32_t grid_cell(rv_context* c, const uint32_t* grid, int G, int ix, int iy) {
  uint32_t* h = reinterpret_cast<uint32_t*>(c->pinned);
  ck(cudaMemcpyAsync(h, grid + (size_t)iy * G + ix, 4, cudaMemcpyDeviceToHost, c->st), "cell D2H");
  sync(c);
  return *h;
}

// ---------------------------------------------------------------------------------------
// Classification state: a bitmask over a constraint set + its block offsets and count.
struct Cls {
  uint32_t* flags;
  int32_t* offsets;
  int64_t count;
  bool differs;
  double scatter[6];
};

// classify (estimator.cpp:287-297) fused with the scatter of the same inliers.
Cls classify_dev(rv_context* c, const ConstraintSet& cs, const double axis[3], double eps, int slot,
                 const uint32_t* prev, int mode = 0) {
  StageScope sc(c, kRefine);
  const int nb = classify_blocks(cs.n);
  const size_t words = (size_t)(cs.n + 31) / 32 + 32;
  Cls r;
  r.flags = slot == 0 ? c->flagsA.get<uint32_t>(words) : c->flagsB.get<uint32_t>(words);
  r.offsets = slot == 0 ? c->boffA.get<int32_t>(nb) : c->boffB.get<int32_t>(nb);
  ClassifyOut o;
  o.flags = r.flags;
  o.prev = prev;
  o.block_count = c->bcount.get<int32_t>(nb);
  o.block_scatter = c->bscatter.get<double>((size_t)nb * 6);
  o.block_diff = c->bdiff.get<int32_t>(nb);
  o.result = c->cls_result.get<double>(8);
  launch_classify_mode(cs.zx, cs.zy, cs.zz, cs.n, axis, eps, mode, o, r.offsets, c->done_ptr(), c->st);
  count_launch(c);
  double* h = pin_d(c);
  ck(cudaMemcpyAsync(h, o.result, sizeof(double) * 8, cudaMemcpyDeviceToHost, c->st), "classify D2H");
  sync(c);
  r.count = (int64_t)h[0];
  r.differs = h[1] != 0.0;
  for (int k = 0; k < 6; ++k) r.scatter[k] = h[2 + k];
  return r;
}

// refine_loop (estimator.cpp:51-69) / anneal_axis (estimator.cpp:145-160) as one cooperative
// launch (rv_coop.cu): every classify pass, scatter reduction and 3x3 eigen-solve stays on the
// device; the host reads the final state once. mode 0 returns the final classification with its
// tile offsets ready for compaction; mode 1 returns the annealed axis in `axis`.
// Mapped pinned inlier buffer (zero-copy target of the compaction), grow-only.
int32_t* inlier_host_buffer(rv_context* c, size_t n) {
  if (c->inl_cap < n) {
    if (c->inl_host) {
      sync(c);
      cudaFreeHost(c->inl_host);
      c->inl_host = nullptr;
      c->inl_cap = 0;
    }
    const size_t cap = std::max<size_t>(n, 1 << 16);
    void* p = nullptr;
    g_buf_gen.fetch_add(1);
    ck(cudaHostAlloc(&p, cap * sizeof(int32_t), cudaHostAllocMapped | cudaHostAllocPortable), "pinned inliers");
    c->inl_host = static_cast<int32_t*>(p);
    c->inl_cap = cap;
  }
  return c->inl_host;
}

// Launches the cooperative loop; the final state stays on the device (CoopState*).
struct CoopFused {  // optional work fused into the last pass of refine_loop
  int32_t* compact_out = nullptr;
  uint32_t* zero_bins = nullptr;
  int n_bins = 0;
  unsigned long long* zero_counts = nullptr;
};
CoopState* coop_refine_launch(rv_context* c, const ConstraintSet& cs, const double* axis, const double* axis_dev,
                              int mode, double e0, const rv_config& cfg, uint32_t** flags, int32_t** offsets,
                              CoopState* state_dst = nullptr, const CoopFused* fz = nullptr,
                              const CoopExchange* xch = nullptr) {
  StageScope sc(c, kRefine);
  if (c->coop_grid == 0) c->coop_grid = coop_refine_grid(c->sms);
  const int nt = std::max(1, coop_tiles(cs.n));
  const size_t words = (size_t)(cs.n + 31) / 32 + 32;
  uint32_t* fa = c->flagsA.get<uint32_t>(words);
  int32_t* toff = c->boffA.get<int32_t>(nt);
  CoopState* dst = state_dst ? state_dst : c->coop_state.get<CoopState>(1);
  uint32_t* fb = c->flagsB.get<uint32_t>(words);
  int32_t* tcount = c->bcount.get<int32_t>(nt);
  double* part = c->coop_part.get<double>((size_t)c->coop_grid * 16);  // one 128-byte line per block
  if (part != c->coop_part_zeroed) {  // sequence numbers start below every launch's epoch
    ck(cudaMemsetAsync(part, 0, sizeof(double) * 16 * (size_t)c->coop_grid, c->st), "coop lines");
    c->coop_part_zeroed = part;
  }
  if (!c->coop_bar_ready) {  // launch epoch + exit counter: zeroed once, maintained by the kernel
    ck(cudaMemsetAsync(c->coop_bar.get<unsigned int>(2), 0, 2 * sizeof(unsigned int), c->st), "coop barrier");
    c->coop_bar_ready = true;
  }
  ck(launch_coop_refine(cs.zx, cs.zy, cs.zz, cs.n, mode, cfg.refine ? 1 : 0, cfg.epsilon, e0, axis, axis_dev, fa, fb,
                        tcount, toff, part, c->coop_bar.get<unsigned int>(2), dst, c->coop_grid, c->st, cs.kept,
                        fz ? fz->compact_out : nullptr, fz ? fz->zero_bins : nullptr, fz ? fz->n_bins : 0,
                        fz ? fz->zero_counts : nullptr, xch),
     "coop refine launch");
  count_launch(c);
  if (flags) *flags = fa;  // refine_loop: final bitmask in flags0
  if (offsets) *offsets = toff;
  return dst;
}

// K start axes at once (launch_coop_refine_multi), in chunks of coop_multi_max(): per candidate k
// its CoopState at (char*)states + k * stride (and the zeroed angle counts at counts + k * stride),
// mode 0: its inlier indices at compact_out + k * compact_stride.
void coop_refine_multi_launch(rv_context* c, const ConstraintSet& cs, const std::vector<std::array<double, 3>>& starts,
                              const std::vector<double>& e0s, int mode, const rv_config& cfg, CoopState* states,
                              size_t stride, unsigned long long* counts, int32_t* compact_out, size_t compact_stride,
                              uint32_t* zero_bins, int n_bins) {
  StageScope sc(c, kRefine);
  if (c->coop_grid == 0) c->coop_grid = coop_refine_grid(c->sms);
  const int km = coop_multi_max();
  const size_t line = (size_t)8 * km + 8;
  double* part = c->coop_mpart.get<double>((size_t)c->coop_grid * line);
  if (part != c->coop_mpart_zeroed) {
    ck(cudaMemsetAsync(part, 0, sizeof(double) * line * (size_t)c->coop_grid, c->st), "coop multi lines");
    c->coop_mpart_zeroed = part;
  }
  if (!c->coop_bar_ready) {
    ck(cudaMemsetAsync(c->coop_bar.get<unsigned int>(2), 0, 2 * sizeof(unsigned int), c->st), "coop barrier");
    c->coop_bar_ready = true;
  }
  for (size_t k0 = 0; k0 < starts.size(); k0 += (size_t)km) {
    const int K = (int)std::min<size_t>((size_t)km, starts.size() - k0);
    auto* st = reinterpret_cast<CoopState*>(reinterpret_cast<char*>(states) + k0 * stride);
    auto* cn = counts ? reinterpret_cast<unsigned long long*>(reinterpret_cast<char*>(counts) + k0 * stride) : nullptr;
    ck(launch_coop_refine_multi(cs.zx, cs.zy, cs.zz, cs.n, mode, cfg.refine ? 1 : 0, cfg.epsilon, K,
                                reinterpret_cast<const double(*)[3]>(starts[k0].data()), e0s.empty() ? nullptr : &e0s[k0],
                                st, stride, cn, nullptr, 0, cs.kept, compact_out ? compact_out + k0 * compact_stride : nullptr,
                                compact_stride, zero_bins, n_bins, part, c->coop_bar.get<unsigned int>(2), c->coop_grid,
                                c->st),
       "coop multi launch");
    count_launch(c);
  }
}

Cls coop_refine_dev(rv_context* c, const ConstraintSet& cs, double axis[3], int mode, double e0, const rv_config& cfg,
                    int* passes = nullptr) {
  Cls r;
  CoopState* dst = coop_refine_launch(c, cs, axis, nullptr, mode, e0, cfg, &r.flags, &r.offsets);
  static_assert(sizeof(CoopState) <= 4096, "pinned scratch");
  CoopState* h = reinterpret_cast<CoopState*>(c->pinned);
  ck(cudaMemcpyAsync(h, dst, sizeof(CoopState), cudaMemcpyDeviceToHost, c->st), "coop state D2H");
  sync(c);
  std::memcpy(axis, h->axis, sizeof(double) * 3);
  r.count = h->count;
  r.differs = false;
  std::memcpy(r.scatter, h->scatter, sizeof r.scatter);
  if (passes) *passes = h->refits;
  return r;
}

Cls refine_loop_dev(rv_context* c, const ConstraintSet& cs, double axis[3], const rv_config& cfg, int* passes = nullptr) {
  return coop_refine_dev(c, cs, axis, 0, 0.0, cfg, passes);
}

// Compact a classification into input indices (through the kept map).
int32_t* compact_dev(rv_context* c, const ConstraintSet& cs, const Cls& cl) {
  int32_t* out = c->compact_out.get<int32_t>((size_t)std::max<int64_t>(cl.count, 1));
  if (cl.count > 0) {
    launch_compact_flags(cl.flags, cs.n, cs.kept, cl.offsets, out, c->st);
    count_launch(c);
  }
  return out;
}

// vote_angles + peak_angle (angles.cpp:46-90) over device input indices. Throws NoVotes.
double angle_dev(rv_context* c, const double axis[3], const double* corrs, const int32_t* idx, int64_t m,
                 const rv_config& cfg) {
  StageScope sc(c, kAngles);
  if (cfg.angle_bins < 8) fail(RV_ERR_INVALID_CONFIG, "angle histogram needs bin_count >= 8");
  uint32_t* bins = c->bins.get<uint32_t>(cfg.angle_bins);
  double* raw = c->raw.get<double>((size_t)std::max<int64_t>(m, 1));
  unsigned long long* cnt = c->angle_counts.get<unsigned long long>(2);
  ck(cudaMemsetAsync(bins, 0, sizeof(uint32_t) * cfg.angle_bins, c->st), "memset bins");
  ck(cudaMemsetAsync(cnt, 0, 16, c->st), "memset counts");
  if (m > 0) {
    launch_vote_angles_k(axis, corrs, idx, m, cfg.angle_bins, cfg.tau_deg, bins, raw, cnt, c->st);
    count_launch(c);
  }
  double* res = c->angle_result.get<double>(4);
  if (m > 0) {
    launch_peak_angle_k(bins, cfg.angle_bins, raw, m, c->angle_sums.get<double>(2 * 296), res, c->done_ptr(), c->st);
    count_launch(c);
  }
  double* h = pin_d(c);
  ck(cudaMemcpyAsync(h, cnt, 16, cudaMemcpyDeviceToHost, c->st), "angle counts D2H");
  if (m > 0) ck(cudaMemcpyAsync(h + 2, res, 32, cudaMemcpyDeviceToHost, c->st), "angle sums D2H");
  sync(c);
  const unsigned long long contributing = reinterpret_cast<unsigned long long*>(h)[0];
  if (contributing == 0) fail(RV_ERR_NO_VOTES, "no correspondence produced an angle vote");
  const double s = h[2], co = h[3], center = h[5];
  if (!cfg.refine) return center;
  if (s == 0.0 && co == 0.0) return center;
  double mean = std::atan2(s, co);
  if (mean <= -kPiD) mean += 2.0 * kPiD;
  return mean;
}

// build_estimate (estimator.cpp:73-92)
Estimate build_estimate_dev(rv_context* c, const ConstraintSet& cs, const double axis[3], const Cls& cl,
                            uint32_t votes, const double* corrs, const rv_config& cfg, bool want_inliers = true) {
  int32_t* idx = compact_dev(c, cs, cl);
  Estimate est;
  est.angle = angle_dev(c, axis, corrs, idx, cl.count, cfg);
  std::memcpy(est.axis, axis, sizeof est.axis);
  rodrigues3(axis, est.angle, est.R);
  est.votes = votes;
  if (want_inliers) {
    est.inliers.resize(cl.count);
    if (cl.count > 0) {
      ck(cudaMemcpyAsync(est.inliers.data(), idx, sizeof(int32_t) * cl.count, cudaMemcpyDeviceToHost, c->st),
         "inliers D2H");
      sync(c);
    }
  } else {
    est.dev_count = cl.count;
  }
  return est;
}

struct Support {
  int64_t coherent = 0;
  int64_t band = 0;
};

// model_support (estimator.cpp:117-137); band flags to `band_flags` if given.
Support model_support_dev(rv_context* c, const ConstraintSet& cs, const double* corrs, const Estimate& est,
                          const rv_config& cfg, uint32_t* band_flags) {
  StageScope sc(c, kAngles);
  const int nb = classify_blocks(cs.n);
  int32_t* bc = c->sup_counts.get<int32_t>((size_t)nb * 2);
  int32_t* res = c->sup_result.get<int32_t>(2);
  launch_model_support_k(cs.zx, cs.zy, cs.zz, cs.kept, corrs, cs.n, est.axis, est.angle, cfg.epsilon, cfg.tau_deg,
                         band_flags, bc, res, c->done_ptr(), c->st);
  count_launch(c);
  int32_t* h = reinterpret_cast<int32_t*>(c->pinned);
  ck(cudaMemcpyAsync(h, res, 8, cudaMemcpyDeviceToHost, c->st), "support D2H");
  sync(c);
  return Support{h[0], h[1]};
}

// anneal_axis (estimator.cpp:145-160)
void anneal_axis_dev(rv_context* c, const ConstraintSet& cs, double axis[3], double eps0, const rv_config& cfg) {
  coop_refine_dev(c, cs, axis, 1, eps0, cfg);
}

// rescue_axes (estimator.cpp:162-179)
std::vector<std::array<double, 3>> rescue_axes_dev(rv_context* c, const uint32_t* grid, const ConstraintSet& cs,
                                                   const rv_config& cfg) {
  std::vector<std::array<double, 3>> out;
  std::vector<int> radii;
  for (int w : {4, 8, 16, 32, 64}) {
    if (2 * w + 1 > cfg.grid) break;
    radii.push_back(w);
  }
  const std::vector<Peak> ps = blurred_argmax_dev(c, grid, cfg.grid, cfg.extent, radii);
  const double cs_ = 2.0 * cfg.extent / cfg.grid;
  std::vector<std::array<double, 3>> starts;
  std::vector<double> e0s;
  for (size_t k = 0; k < ps.size(); ++k) {
    double b[3], start[3];
    backproject(ps[k].A, ps[k].B, b);
    canonicalize3(b, start);
    starts.push_back({start[0], start[1], start[2]});
    e0s.push_back(radii[k] * cs_);
  }
  // least squares over all constraints (refine_axis(constraints))
  if (cs.n >= 2) {
    const Cls all = classify_dev(c, cs, nullptr, 0.0, 0, nullptr, 1);
    double ls[3];
    if (axis_from_scatter(all.scatter, ls)) {
      starts.push_back({ls[0], ls[1], ls[2]});
      e0s.push_back(0.25);
    }
  }
  if (starts.empty()) return out;
  static const bool multi_on = [] {
    const char* e = std::getenv("RV_COOP_MULTI");
    return !(e && e[0] == '0');
  }();
  if (!multi_on) {
    for (size_t k = 0; k < starts.size(); ++k) {
      double a[3] = {starts[k][0], starts[k][1], starts[k][2]};
      anneal_axis_dev(c, cs, a, e0s[k], cfg);
      out.push_back({a[0], a[1], a[2]});
    }
    return out;
  }
  // all anneals (estimator.cpp:145-160) in one cooperative launch, one read-back
  CoopState* st = c->coop_state.get<CoopState>(starts.size());
  coop_refine_multi_launch(c, cs, starts, e0s, 1, cfg, st, sizeof(CoopState), nullptr, nullptr, 0, nullptr, 0);
  std::vector<CoopState> h(starts.size());
  read_small(c, h.data(), st, starts.size(), "anneal D2H");
  for (const CoopState& x : h) out.push_back({x.axis[0], x.axis[1], x.axis[2]});
  return out;
}

// build_candidate (estimator.cpp:183-194). Throws NoVotes.
// ---------------------------------------------------------------------------------------
struct PreResult {
  ConstraintSet cs;
  int64_t n_dropped = 0;
  bool vote_zeroed = false;  // the preprocess kernel cleared the vote grid and counters
  bool inorder = false;      // cs = all n pairs in input order (z = NaN: dropped), kept = null;
                             // the kept count is only on the device (Summary::n_kept)
};

// The side job of the preprocess kernel: clear the state of the banded vote that follows.
void set_vote_zeroing(rv_context* c, int G, PrepBuffers* b) {
  b->zero_ptr[0] = c->grid.get<uint32_t>((size_t)G * G);
  b->zero_n[0] = (int64_t)G * G;
  b->zero_ptr[1] = reinterpret_cast<uint32_t*>(c->band_work.get<unsigned long long>(kMaxBands));
  b->zero_n[1] = 2 * kMaxBands;
  b->zero_ptr[2] = reinterpret_cast<uint32_t*>(c->counters.get<int32_t>(kCounterWords));
  b->zero_n[2] = kCounterWords;
  b->zero_ptr[3] = reinterpret_cast<uint32_t*>(c->stats.get<unsigned long long>(2));
  b->zero_n[3] = 4;
}

// vcfg (optional): also clear the state of the vote that follows (banded plans).
PreResult preprocess_dev(rv_context* c, const double* d_corrs, int64_t n, double tau_z, int normalize,
                         const rv_config* vcfg = nullptr) {
  bool zeroed = false;
  PrepBuffers b;
  if (vcfg && vcfg->grid >= 1 && vcfg->extent > 0.0 && vcfg->theta_samples >= 1) {
    ensure_tables(c, vcfg->theta_samples);
    const VotePlan& p = cached_plan(c, vcfg->grid, vcfg->extent, vcfg->theta_samples);
    if (p.banded) {  // the same grow-only buffers vote() will take
      set_vote_zeroing(c, vcfg->grid, &b);
      zeroed = true;
    }
  }
  StageScope sc(c, kPrep);
  b.corrs = d_corrs;
  b.zx = c->zx.get<double>(n);
  b.zy = c->zy.get<double>(n);
  b.zz = c->zz.get<double>(n);
  b.kept = c->kept.get<int32_t>(n);
  b.dropped = c->dropped.get<int32_t>(n);
  const int nb = prep_blocks(n);
  b.status = c->status.get<unsigned long long>(nb);
  int32_t* misc = c->misc32.get<int32_t>(8);
  b.block_counter = misc;
  b.totals = misc + 2;
  ck(cudaMemsetAsync(b.status, 0, sizeof(unsigned long long) * nb, c->st), "memset status");
  ck(cudaMemsetAsync(misc, 0, sizeof(int32_t) * 8, c->st), "memset misc");
  launch_preprocess(b, n, tau_z, normalize, c->st);
  count_launch(c);
  ck(cudaGetLastError(), "preprocess");
  int32_t* h = reinterpret_cast<int32_t*>(c->pinned);
  ck(cudaMemcpyAsync(h, b.totals, 8, cudaMemcpyDeviceToHost, c->st), "totals D2H");
  sync(c);
  PreResult r;
  r.cs.zx = b.zx;
  r.cs.zy = b.zy;
  r.cs.zz = b.zz;
  r.cs.kept = b.kept;
  r.cs.n = h[0];
  r.n_dropped = h[1];
  r.vote_zeroed = zeroed;
  return r;
}

// In-order preprocess (single solves with a banded plan): z written at the input index with NaN
// for dropped pairs, no compaction, no host sync -- the kept count lands in Summary::n_kept and
// the host reads it with the solve's one summary. The vote's state is cleared as a side job.
bool banded_plan(rv_context* c, const rv_config& cfg) {
  if (cfg.grid < 1 || !(cfg.extent > 0.0) || cfg.theta_samples < 1) return false;
  ensure_tables(c, cfg.theta_samples);
  return cached_plan(c, cfg.grid, cfg.extent, cfg.theta_samples).banded;
}

PrepBuffers inorder_buffers(rv_context* c, const double* d_corrs, int64_t n) {
  PrepBuffers b;
  b.corrs = d_corrs;
  b.zx = c->zx.get<double>(n);
  b.zy = c->zy.get<double>(n);
  b.zz = c->zz.get<double>(n);
  b.kept_total = &summary_buf(c)->n_kept;
  unsigned long long* acc = c->kept_acc.get<unsigned long long>(2);  // [0] accumulator, [1] ticket
  if (!c->kept_acc_ready) {  // zero at rest from here on (the last block of each solve re-zeroes)
    ck(cudaMemsetAsync(acc, 0, 2 * sizeof(unsigned long long), c->st), "memset kept accumulator");
    c->kept_acc_ready = true;
  }
  b.kept_acc = acc;
  b.kept_done = reinterpret_cast<unsigned int*>(acc + 1);
  return b;
}

PreResult inorder_result(const PrepBuffers& b, int64_t n) {
  PreResult r;
  r.cs.zx = b.zx;
  r.cs.zy = b.zy;
  r.cs.zz = b.zz;
  r.cs.kept = nullptr;
  r.cs.n = n;
  r.vote_zeroed = true;
  r.inorder = true;
  return r;
}

PreResult preprocess_inorder_dev(rv_context* c, const double* d_corrs, int64_t n, const rv_config& cfg) {
  PrepBuffers b = inorder_buffers(c, d_corrs, n);
  set_vote_zeroing(c, cfg.grid, &b);
  StageScope sc(c, kPrep);
  launch_preprocess_inorder(b, n, 0, n, cfg.tau_z, cfg.normalize_inputs, c->st);
  count_launch(c);
  ck(cudaGetLastError(), "preprocess");
  return inorder_result(b, n);
}

const double* upload_corrs(rv_context* c, const double* corrs, int64_t n) {
  double* d = c->corrs.get<double>((size_t)n * 6);
  StageScope sc(c, kPrep);
  ck(cudaMemcpyAsync(d, corrs, sizeof(double) * 6 * n, cudaMemcpyHostToDevice, c->st), "H2D corrs");
  return d;
}

std::vector<int32_t> dropped_list(rv_context* c, int64_t nd) {
  std::vector<int32_t> v(nd);
  if (nd > 0) {
    ck(cudaMemcpyAsync(v.data(), c->dropped.get<int32_t>(1), sizeof(int32_t) * nd, cudaMemcpyDeviceToHost, c->st),
       "dropped D2H");
    sync(c);
  }
  return v;
}

Estimate identity_estimate(std::vector<int32_t> idx) {
  Estimate e;
  e.inliers = std::move(idx);
  return e;
}

// Host-buffer input, pipelined: the H2D copy of chunk k+1 (copy stream) overlaps preprocess +
// band plan + vote of chunk k (compute stream). Chunk boundaries are multiples of the preprocess
// block so the single-pass compaction continues across launches; each chunk's kept-constraint
// range [lo, hi) stays on the device (chunk_hi[]) and bounds the plan/vote launches of that
// chunk. Vote tiles flush to partial slots that the final reduction sums once (integer: the grid
// is identical to the one-shot vote). Returns the preprocess result and the voted grid.
struct PipelinedVote {
  PreResult pre;
  const uint32_t* grid = nullptr;
  const double* d_corrs = nullptr;
  bool peak_ready = false;  // argmax + start axis fused into the final tile reduction
};

bool host_pinned(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

PipelinedVote prep_and_vote_host(rv_context* c, const double* h_corrs, int64_t n, const rv_config& cfg) {
  PipelinedVote out;
  double* d = c->corrs.get<double>((size_t)n * 6);
  out.d_corrs = d;
  const int G = cfg.grid, J = cfg.theta_samples;
  if (G < 1 || !(cfg.extent > 0.0)) fail(RV_ERR_INVALID_CONFIG, "accumulator needs grid >= 1, extent > 0");
  if (J < 1) fail(RV_ERR_INVALID_CONFIG, "theta_samples must be >= 1");
  ensure_tables(c, J);
  const VotePlan& p = cached_plan(c, G, cfg.extent, J);
  // chunk k+1's copy overlaps chunk k's compute (~1.4x slower per correspondence than the copy).
  // Default 1, 2, 3, 4, 6 sixteenths (measured best of 14 schedules, tools/_pipe_ab.sh: e2e 1.51
  // ms vs 1.63 for 1, 2, 5, 8): only the first 3 MB copy is exposed, no chunk's compute waits for
  // its copy, and the last chunk -- whose compute trails the last copy -- stays small; each extra
  // chunk costs a vote-launch tail. Bounds are aligned to the preprocess tile (1024).
  // Dev knob: RV_PIPE_CUM="0,1,3,6,10,16" (cumulative sixteenths).
  static const std::vector<int64_t> kCum = [] {
    std::vector<int64_t> v{0, 1, 3, 6, 10, 16};
    if (const char* e = std::getenv("RV_PIPE_CUM")) {
      std::vector<int64_t> w;
      for (const char* q = e; *q;) {
        w.push_back(std::strtoll(q, const_cast<char**>(&q), 10));
        if (*q == ',') ++q;
      }
      if (w.size() >= 2 && w.front() == 0 && w.back() == 16) v = w;
    }
    return v;
  }();
  // pageable input is staged through pinned memory by host threads (below); the host copy is then
  // the slow stage, so it gets 16 equal chunks: each chunk's DMA + compute hides under the next
  // chunk's host copy, and only one sixteenth of the compute trails the last copy
  static const std::vector<int64_t> kCumStaged = [] {
    std::vector<int64_t> v;
    for (int k = 0; k <= 16; ++k) v.push_back(k);
    return v;
  }();
  static const int kPageable = [] {  // dev knob: 0 staging (default), 1 register in place, 2 plain
    const char* e = std::getenv("RV_PAGEABLE");
    return e ? std::atoi(e) : 0;
  }();
  const bool pipelined = p.banded && n >= (int64_t)1 << 18;
  const bool staged = pipelined && kPageable == 0 && !host_pinned(h_corrs);
  const std::vector<int64_t>& cum = staged ? kCumStaged : kCum;
  const int C = pipelined ? (int)cum.size() - 1 : 1;
  if (!c->copy_st) ck(cudaStreamCreateWithFlags(&c->copy_st, cudaStreamNonBlocking), "copy stream");
  while ((int)c->chunk_events.size() < C) {
    cudaEvent_t e;
    ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    c->chunk_events.push_back(e);
  }
  std::vector<int64_t> bounds(C + 1);
  for (int k = 0; k <= C; ++k)
    bounds[k] = k == C ? n : std::min<int64_t>(n, ((C > 1 ? n * cum[k] / 16 : 0) + 1023) / 1024 * 1024);
  StageScope sc(c, kVote);
  // one chunk: the copy goes on the compute stream itself (no cross-stream dependency to resolve);
  // several: on the copy stream, ordered after everything already queued on the compute stream
  cudaStream_t cs = C > 1 ? c->copy_st : c->st;
  if (C > 1) {
    cudaEvent_t start = take_event(c);
    ck(cudaEventRecord(start, c->st), "record");
    ck(cudaStreamWaitEvent(c->copy_st, start, 0), "wait");
  }
  // Large pageable input (what a std::vector<Correspondence> caller passes): each chunk is first
  // copied into a context-owned pinned buffer by a few host threads in parallel, then DMA'd
  // asynchronously -- the host copies chunk k+1 while the device copies and computes chunk k (a
  // pageable cudaMemcpyAsync would stage through the driver's buffers at single-thread speed).
  const double* src = h_corrs;
  bool registered = false;
  if (C > 1 && kPageable == 1 && !host_pinned(h_corrs)) {
    registered = cudaHostRegister(const_cast<double*>(h_corrs), sizeof(double) * 6 * (size_t)n,
                                  cudaHostRegisterReadOnly) == cudaSuccess;
    if (!registered) cudaGetLastError();
  }
  if (staged) {
    const size_t bytes = sizeof(double) * 6 * (size_t)n;
    if (bytes > c->big_pinned_cap) {
      if (c->big_pinned) {
        sync(c);
        cudaFreeHost(c->big_pinned);
        c->big_pinned = nullptr;
        c->big_pinned_cap = 0;
      }
      void* q = nullptr;
      if (cudaHostAlloc(&q, bytes, cudaHostAllocDefault) == cudaSuccess) {
        c->big_pinned = static_cast<double*>(q);
        c->big_pinned_cap = bytes;
      } else {
        cudaGetLastError();
      }
    }
    if (c->big_pinned) {
      if (!c->copy_pool) {
        const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
        unsigned nt = std::min(4u, hw);  // 4: the measured best on a 16-vCPU B200 host (memory-bound)
        if (const char* e = std::getenv("RV_COPY_THREADS")) nt = (unsigned)std::max(1, std::atoi(e));  // dev knob
        c->copy_pool = std::make_unique<CopyPool>((int)nt);
      }
      src = c->big_pinned;
    }
  }
  auto issue_copy = [&](int k) {
    const size_t bytes = sizeof(double) * 6 * (size_t)(bounds[k + 1] - bounds[k]);
    if (src != h_corrs) c->copy_pool->copy(c->big_pinned + 6 * bounds[k], h_corrs + 6 * bounds[k], bytes);
    ck(cudaMemcpyAsync(d + 6 * bounds[k], src + 6 * bounds[k], bytes, cudaMemcpyHostToDevice, cs), "H2D chunk");
    if (C > 1) ck(cudaEventRecord(c->chunk_events[k], cs), "record chunk");
  };
  issue_copy(0);
  uint32_t* grid = c->grid.get<uint32_t>((size_t)G * G);
  VoteBuffers b;
  b.grid = grid;
  b.table64 = c->table64.get<double2>(J);
  b.table32 = c->table32.get<float2>(std::max(J, 1));
  int32_t* h = reinterpret_cast<int32_t*>(c->pinned);
  if (p.banded) {
    // in-order constraint set: chunk k's z land at their input indices, so each chunk's plan and
    // vote cover exactly [bounds[k], bounds[k+1]) -- no device-side chunk bounds, no host sync
    PrepBuffers pb = inorder_buffers(c, d, n);
    set_vote_zeroing(c, G, &pb);  // chunk 0's preprocess clears the vote state
    b.zx = pb.zx;
    b.zy = pb.zy;
    b.zz = pb.zz;
    b.basis_a = c->basis_a.get<float4>(n);
    b.basis_b = c->basis_b.get<float2>(n);
    b.entry_cap = kEntriesPerConstraint * n;
    b.degen = c->degen.get<int32_t>(n);
    b.entries = c->ranges.get<unsigned long long>((size_t)b.entry_cap * p.n_bands);
    b.band_work = c->band_work.get<unsigned long long>(kMaxBands);
    b.counters = c->counters.get<int32_t>(kCounterWords);
    b.entry_count = b.counters + kMaxBands + 1;
    b.stats = c->stats.get<unsigned long long>(2);
    const int64_t est_pairs = (n / C) * (int64_t)p.halfJ;
    const int n_ctas = vote_ctas(c, p, est_pairs);
    b.max_slots = p.bulk ? 0 : C * n_ctas * p.n_bands;
    if (!p.bulk) {
      b.partials = c->partials.get<uint32_t>((size_t)b.max_slots * p.tile_words);
      b.slot_band = c->slot_band.get<int32_t>(b.max_slots);
    }
    for (int k = 0; k < C; ++k) {
      if (C > 1) ck(cudaStreamWaitEvent(c->st, c->chunk_events[k], 0), "wait chunk");
      pb.kept_publish = k == C - 1;  // chunk counts accumulate; the last chunk publishes the total
      launch_preprocess_inorder(pb, n, bounds[k], bounds[k + 1], cfg.tau_z, cfg.normalize_inputs, c->st);
      if (k == 0)
        for (int q = 0; q < 4; ++q) pb.zero_ptr[q] = nullptr;
      // entry lists and their counters are per chunk (reused: the stream orders chunk k's vote
      // before chunk k+1's plan)
      if (k > 0) launch_zero_i32(b.counters + 1, kCounterWords - 1, c->st);
      b.range_lo = bounds[k];
      const int64_t cap = bounds[k + 1] - bounds[k];
      launch_plan(p, b, cap, c->st);
      {
        StageScope kv(c, kVoteKernel);
        launch_vote_banded(p, b, cap, n_ctas, c->st);
      }
      count_launch(c, k > 0 ? 4 : 3);
      // copy k+1 is issued after compute k is queued: with pinned input both run concurrently;
      // with pageable input the host stages copy k+1 while the device computes chunk k
      if (k + 1 < C) issue_copy(k + 1);
    }
    VoteFused vf;
    vf.key_out = c->arg_out.get<unsigned long long>(2);
    vf.peak = &summary_buf(c)->pk;
    set_fused(c, b, &vf, p);
    out.peak_ready = vf.done;
    launch_vote_reduce(p, b, c->st);
    count_launch(c);
    ck(cudaGetLastError(), "pipelined vote");
    out.pre = inorder_result(pb, n);
    out.grid = grid;
  } else {  // generic vote: compacting preprocess, then one vote once all constraints are in
    PrepBuffers pb;
    pb.corrs = d;
    pb.zx = c->zx.get<double>(n);
    pb.zy = c->zy.get<double>(n);
    pb.zz = c->zz.get<double>(n);
    pb.kept = c->kept.get<int32_t>(n);
    pb.dropped = c->dropped.get<int32_t>(n);
    const int nb_prep = prep_blocks(n);
    pb.status = c->status.get<unsigned long long>(nb_prep);
    int32_t* misc = c->misc32.get<int32_t>(8);
    pb.block_counter = misc;
    pb.totals = misc + 2;
    ck(cudaMemsetAsync(pb.status, 0, sizeof(unsigned long long) * nb_prep, c->st), "memset status");
    ck(cudaMemsetAsync(misc, 0, sizeof(int32_t) * 8, c->st), "memset misc");
    for (int k = 0; k < C; ++k) {
      if (C > 1) ck(cudaStreamWaitEvent(c->st, c->chunk_events[k], 0), "wait chunk");
      launch_preprocess_range(pb, n, bounds[k], bounds[k + 1], cfg.tau_z, cfg.normalize_inputs, c->st);
      count_launch(c);
      if (k + 1 < C) issue_copy(k + 1);
    }
    ck(cudaMemcpyAsync(h, pb.totals, 8, cudaMemcpyDeviceToHost, c->st), "totals D2H");
    sync(c);
    out.pre.cs.zx = pb.zx;
    out.pre.cs.zy = pb.zy;
    out.pre.cs.zz = pb.zz;
    out.pre.cs.kept = pb.kept;
    out.pre.cs.n = h[0];
    out.pre.n_dropped = h[1];
    out.grid = out.pre.cs.n > 0 ? vote(c, pb.zx, pb.zy, pb.zz, out.pre.cs.n, G, cfg.extent, J) : grid;
  }
  if (registered) {  // every chunk copy has been issued: wait for the last, then unpin
    ck(cudaEventSynchronize(c->chunk_events[C - 1]), "H2D done");
    cudaHostUnregister(const_cast<double*>(h_corrs));
  }
  return out;
}

// estimate_single from a preprocessed constraint set (identity shortcuts already handled).
Estimate finish_single(rv_context* c, const PreResult& pre, const double* d_corrs, const rv_config& cfg,
                       const uint32_t* prevoted, bool peak_ready = false, bool* identity = nullptr);
Estimate finish_single_stepped(rv_context* c, const PreResult& pre, const double* d_corrs, const rv_config& cfg,
                               const uint32_t* prevoted, int first_attempt);
Estimate rescue_single(rv_context* c, const PreResult& pre, const double* d_corrs, const rv_config& cfg,
                       const uint32_t* grid, Estimate est);

// The identity shortcuts of estimate_single (estimator.cpp:326-340) after an in-order solve saw
// them in the summary: redo the bookkeeping with the compacting preprocess (rare).
Estimate identity_from_inorder(rv_context* c, const double* d_corrs, int64_t n, const rv_config& cfg) {
  const PreResult pc = preprocess_dev(c, d_corrs, n, cfg.tau_z, cfg.normalize_inputs);
  if (pc.cs.n == 0) {
    std::vector<int32_t> all(n);
    for (int64_t i = 0; i < n; ++i) all[i] = (int32_t)i;
    return identity_estimate(std::move(all));
  }
  return identity_estimate(dropped_list(c, pc.n_dropped));
}

const uint32_t* enqueue_single(rv_context* c, const PreResult& pre, const double* d_corrs, const rv_config& cfg,
                               const uint32_t* prevoted, bool peak_ready);
Estimate complete_single(rv_context* c, const PreResult& pre, const double* d_corrs, const rv_config& cfg,
                         const uint32_t* grid, bool prevoted, bool* identity);

bool graphs_enabled() {  // dev A/B knob: RV_GRAPHS=0 always enqueues kernel by kernel
  static const bool on = [] {
    const char* e = std::getenv("RV_GRAPHS");
    return !(e && e[0] == '0');
  }();
  return on;
}

bool same_cfg(const rv_config& a, const rv_config& b) {
  return a.grid == b.grid && a.extent == b.extent && a.theta_samples == b.theta_samples && a.epsilon == b.epsilon &&
         a.angle_bins == b.angle_bins && a.max_models == b.max_models && a.min_votes_frac == b.min_votes_frac &&
         a.consensus_floor_mult == b.consensus_floor_mult && a.dedupe_overlap == b.dedupe_overlap &&
         a.tau_z == b.tau_z && a.tau_deg == b.tau_deg && a.suppression_radius == b.suppression_radius &&
         a.refine == b.refine && a.normalize_inputs == b.normalize_inputs;
}

void add_counts(rv_stage_times& t, const rv_stage_times& d) {
  t.vote_pairs += d.vote_pairs;
  t.vote_fallback_pairs += d.vote_fallback_pairs;
  t.vote_guard_reruns += d.vote_guard_reruns;
  t.vote_samples += d.vote_samples;
  t.vote_launches += d.vote_launches;
  t.kernel_launches += d.kernel_launches;
}

rv_stage_times count_delta(const rv_stage_times& after, const rv_stage_times& before) {
  rv_stage_times d{};
  d.vote_pairs = after.vote_pairs - before.vote_pairs;
  d.vote_fallback_pairs = after.vote_fallback_pairs - before.vote_fallback_pairs;
  d.vote_guard_reruns = after.vote_guard_reruns - before.vote_guard_reruns;
  d.vote_samples = after.vote_samples - before.vote_samples;
  d.vote_launches = after.vote_launches - before.vote_launches;
  d.kernel_launches = after.kernel_launches - before.kernel_launches;
  return d;
}

rv_context::SolveGraph* graph_slot(rv_context* c, const double* d, int64_t n, const rv_config& cfg, bool host,
                                   const void* aux = nullptr, int kind = 0) {
  for (auto& g : c->graphs)
    if (g.corrs == d && g.host == host && g.aux == aux && g.kind == kind && g.n == n && same_cfg(g.cfg, cfg))
      return &g;
  if (c->graphs.size() >= 8) {  // small LRU-less cache: drop the oldest entry
    if (c->graphs.front().exec) cudaGraphExecDestroy(c->graphs.front().exec);
    c->graphs.erase(c->graphs.begin());
  }
  rv_context::SolveGraph g;
  g.corrs = d;
  g.host = host;
  g.aux = aux;
  g.kind = kind;
  g.n = n;
  g.cfg = cfg;
  g.gen = ~0ull;
  c->graphs.push_back(g);
  return &c->graphs.back();
}

// Capture the device part of an in-order single solve (preprocess, plan, vote, reduce, cooperative
// refine, angle kernels, summary D2H; with host input also the chunked H2D copies on the copy
// stream, forked from and joined back into the capture) into g->exec. Returns false (and leaves
// the streams untouched) when the capture fails or a buffer moved while capturing.
template <typename Enqueue>
bool capture_single(rv_context* c, rv_context::SolveGraph* g, Enqueue&& enqueue) {
  if (!c->cap_st) ck(cudaStreamCreateWithFlags(&c->cap_st, cudaStreamNonBlocking), "capture stream");
  const uint64_t gen = g_buf_gen.load();
  const rv_stage_times before = c->times;
  cudaStream_t saved = c->st;
  c->st = c->cap_st;
  if (cudaStreamBeginCapture(c->cap_st, cudaStreamCaptureModeRelaxed) != cudaSuccess) {
    c->st = saved;
    cudaGetLastError();
    return false;
  }
  cudaGraph_t graph = nullptr;
  try {
    enqueue();
  } catch (...) {
    cudaStreamEndCapture(c->cap_st, &graph);
    if (graph) cudaGraphDestroy(graph);
    cudaGetLastError();
    c->st = saved;
    c->times = before;
    return false;
  }
  const cudaError_t e = cudaStreamEndCapture(c->cap_st, &graph);
  c->st = saved;
  c->times = before;
  if (e != cudaSuccess || !graph || g_buf_gen.load() != gen) {
    if (graph) cudaGraphDestroy(graph);
    cudaGetLastError();
    return false;
  }
  cudaGraphExec_t exec = nullptr;
  const cudaError_t ei = cudaGraphInstantiate(&exec, graph, 0);
  cudaGraphDestroy(graph);
  if (ei != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  g->exec = exec;
  g->gen = gen;
  return true;
}

// estimate_single (estimator.cpp:320-371) over device-resident correspondences.
Estimate estimate_single_dev(rv_context* c, const double* d_corrs, int64_t n, const rv_config& cfg) {
  if (n <= 0) fail(RV_ERR_EMPTY_INPUT, "no correspondences");
  static const bool inorder = [] {  // dev A/B knob: RV_INORDER=0 takes the compacting path
    const char* e = std::getenv("RV_INORDER");
    return !(e && e[0] == '0');
  }();
  const bool graphs = graphs_enabled();
  if (inorder && cfg.angle_bins >= 8 && banded_plan(c, cfg)) {  // in-order chain: no host sync until the summary
    // A repeated (input, n, config) replays the captured solve graph: one launch for the whole
    // device chain (no per-kernel host latency between the stages).
    rv_context::SolveGraph* g = graphs && !c->timing ? graph_slot(c, d_corrs, n, cfg, false) : nullptr;
    // capture on the second eager-equivalent call (the first one allocated every buffer); the
    // host counters a replay adds are those the eager run of the same key recorded
    if (g && !g->exec && g->seen > 0 && g->gen == g_buf_gen.load())
      capture_single(c, g, [&] {
        const PreResult pre = preprocess_inorder_dev(c, d_corrs, n, cfg);
        enqueue_single(c, pre, d_corrs, cfg, nullptr, false);
      });
    if (g && g->exec && g->gen == g_buf_gen.load()) {
      ck(cudaGraphLaunch(g->exec, c->st), "solve graph launch");
      add_counts(c->times, g->delta);
      sync(c);
      PreResult pre;
      pre.cs.zx = c->zx.get<double>(n);
      pre.cs.zy = c->zy.get<double>(n);
      pre.cs.zz = c->zz.get<double>(n);
      pre.cs.kept = nullptr;
      pre.cs.n = n;
      pre.vote_zeroed = true;
      pre.inorder = true;
      bool identity = false;
      Estimate est = complete_single(c, pre, d_corrs, cfg, c->grid.get<uint32_t>((size_t)cfg.grid * cfg.grid),
                                     false, &identity);
      return identity ? identity_from_inorder(c, d_corrs, n, cfg) : est;
    }
    const rv_stage_times t0 = c->times;
    const PreResult pre = preprocess_inorder_dev(c, d_corrs, n, cfg);
    const uint32_t* grid = enqueue_single(c, pre, d_corrs, cfg, nullptr, false);
    if (g) {  // remember this enqueue's host counters and the buffer generation it ran with
      g->delta = count_delta(c->times, t0);
      if (g->exec) {  // captured before a buffer moved: stale pointers, never replay it again
        cudaGraphExecDestroy(g->exec);
        g->exec = nullptr;
      }
      g->gen = g_buf_gen.load();
      g->seen += 1;
    }
    sync(c);
    bool identity = false;
    Estimate est = complete_single(c, pre, d_corrs, cfg, grid, false, &identity);
    return identity ? identity_from_inorder(c, d_corrs, n, cfg) : est;
  }
  const PreResult pre = preprocess_dev(c, d_corrs, n, cfg.tau_z, cfg.normalize_inputs, &cfg);
  if (pre.cs.n == 0) {
    std::vector<int32_t> all(n);
    for (int64_t i = 0; i < n; ++i) all[i] = (int32_t)i;
    return identity_estimate(std::move(all));
  }
  if (pre.n_dropped * 10 >= n * 9) return identity_estimate(dropped_list(c, pre.n_dropped));
  return finish_single(c, pre, d_corrs, cfg, nullptr);
}

// estimate_single with host input: pipelined H2D + preprocess + vote, then the same solve.
// Small pageable inputs are staged into a context-owned pinned buffer first (n x 48 B, a few
// microseconds): the H2D then runs at DMA speed and the staged solve is graph-replayable (the
// staging pointer repeats), which is what many small independent solves (estimate_batch) need.
constexpr int64_t kStageMaxRows = (int64_t)1 << 18;
const double* stage_small_input(rv_context* c, const double* h, int64_t n) {
  if (n > kStageMaxRows || host_pinned(h)) return h;
  const size_t bytes = sizeof(double) * 6 * (size_t)n;
  if (bytes > c->in_pinned_cap) {
    if (c->in_pinned) {
      sync(c);
      cudaFreeHost(c->in_pinned);
      c->in_pinned = nullptr;
      c->in_pinned_cap = 0;
    }
    void* p = nullptr;
    const size_t cap = std::max<size_t>(bytes, (size_t)48 << 10);
    g_buf_gen.fetch_add(1);
    if (cudaHostAlloc(&p, cap, cudaHostAllocDefault) != cudaSuccess) {
      cudaGetLastError();
      return h;
    }
    c->in_pinned = static_cast<double*>(p);
    c->in_pinned_cap = cap;
  }
  std::memcpy(c->in_pinned, h, bytes);  // (every call ends synchronised: no copy still reads it)
  return c->in_pinned;
}

Estimate estimate_single_host(rv_context* c, const double* h_corrs, int64_t n, const rv_config& cfg) {
  if (n <= 0) fail(RV_ERR_EMPTY_INPUT, "no correspondences");
  h_corrs = stage_small_input(c, h_corrs, n);
  // Repeated solves from the same pinned host buffer replay a captured graph of the whole
  // pipelined solve (chunked H2D on the copy stream + the in-order device chain): the copy
  // engine and the SMs run without waiting for the host to issue the next copy or launch.
  rv_context::SolveGraph* g = nullptr;
  if (graphs_enabled() && !c->timing && cfg.angle_bins >= 8 && banded_plan(c, cfg) && host_pinned(h_corrs))
    g = graph_slot(c, h_corrs, n, cfg, true);
  if (g && !g->exec && g->seen > 0 && g->gen == g_buf_gen.load())
    capture_single(c, g, [&] {
      const PipelinedVote pv = prep_and_vote_host(c, h_corrs, n, cfg);
      enqueue_single(c, pv.pre, pv.d_corrs, cfg, pv.grid, pv.peak_ready);
    });
  if (g && g->exec && g->gen == g_buf_gen.load()) {
    ck(cudaGraphLaunch(g->exec, c->st), "solve graph launch");
    add_counts(c->times, g->delta);
    sync(c);
    PreResult pre;
    pre.cs.zx = c->zx.get<double>(n);
    pre.cs.zy = c->zy.get<double>(n);
    pre.cs.zz = c->zz.get<double>(n);
    pre.cs.n = n;
    pre.vote_zeroed = true;
    pre.inorder = true;
    const double* d_corrs = c->corrs.get<double>((size_t)n * 6);
    bool identity = false;
    Estimate est = complete_single(c, pre, d_corrs, cfg, c->grid.get<uint32_t>((size_t)cfg.grid * cfg.grid), true,
                                   &identity);
    return identity ? identity_from_inorder(c, d_corrs, n, cfg) : est;
  }
  const rv_stage_times t0 = c->times;
  const PipelinedVote pv = prep_and_vote_host(c, h_corrs, n, cfg);
  if (pv.pre.inorder) {
    const uint32_t* grid = enqueue_single(c, pv.pre, pv.d_corrs, cfg, pv.grid, pv.peak_ready);
    if (g) {
      g->delta = count_delta(c->times, t0);
      if (g->exec) {  // captured before a buffer moved: stale pointers, never replay it again
        cudaGraphExecDestroy(g->exec);
        g->exec = nullptr;
      }
      g->gen = g_buf_gen.load();
      g->seen += 1;
    }
    sync(c);
    bool identity = false;
    Estimate est = complete_single(c, pv.pre, pv.d_corrs, cfg, grid, true, &identity);
    return identity ? identity_from_inorder(c, pv.d_corrs, n, cfg) : est;
  }
  if (pv.pre.cs.n == 0) {
    std::vector<int32_t> all(n);
    for (int64_t i = 0; i < n; ++i) all[i] = (int32_t)i;
    return identity_estimate(std::move(all));
  }
  if (pv.pre.n_dropped * 10 >= n * 9) return identity_estimate(dropped_list(c, pv.pre.n_dropped));
  return finish_single(c, pv.pre, pv.d_corrs, cfg, pv.grid, pv.peak_ready);
}

// estimate_single after preprocess (estimator.cpp:320-371), chained on the device: vote ->
// argmax -> start axis (peak_axis_kernel) -> refine_loop (one cooperative launch) -> compaction
// -> angle histogram + circular mean sums, then ONE summary read-back (and the inlier list). The
// host only validates and finishes (atan2, Rodrigues). Rare cases -- a failed exactness guard
// (grid sum != N*J), or the rescue path -- continue on the host-stepped path below.
// The device part (enqueued on c->st, no host synchronisation: capturable into a graph); returns
// the voted grid. complete_single() reads the summary after the stream is synchronised.
const uint32_t* enqueue_single(rv_context* c, const PreResult& pre, const double* d_corrs, const rv_config& cfg,
                               const uint32_t* prevoted, bool peak_ready) {
  if (cfg.angle_bins < 8) fail(RV_ERR_INVALID_CONFIG, "angle histogram needs bin_count >= 8");
  const ConstraintSet& cs = pre.cs;
  Summary* dsum = summary_buf(c);
  PeakOut* pk = &dsum->pk;
  const uint32_t* grid = prevoted;
  if (!prevoted) {  // vote with find_peaks(K=1) + start axis fused into its tile reduction
    VoteFused vf;
    vf.key_out = c->arg_out.get<unsigned long long>(2);
    vf.peak = pk;
    grid = vote(c, cs.zx, cs.zy, cs.zz, cs.n, cfg.grid, cfg.extent, cfg.theta_samples, false, pre.vote_zeroed, &vf);
    peak_ready = vf.done;
  }
  if (!peak_ready) {
    StageScope sc(c, kPeaks);
    unsigned long long* keys = c->arg_keys.get<unsigned long long>(2 * argmax_block_count());
    unsigned long long* okey = c->arg_out.get<unsigned long long>(2);
    launch_argmax(grid, cfg.grid, nullptr, 0, cfg.suppression_radius, keys, okey, c->done_ptr(), c->st);
    launch_peak_axis(okey, grid, cfg.grid, cfg.extent, 1u, pk, c->st);
    count_launch(c, 2);
  }
  int32_t* idx = c->compact_out.get<int32_t>((size_t)std::max<int64_t>(cs.n, 1));
  unsigned long long* cnt = dsum->counts;
  double* res = dsum->angle;
  uint32_t* bins = c->bins.get<uint32_t>(cfg.angle_bins);
  CoopFused fz;  // compaction + clearing the angle histogram ride on the last refine pass
  fz.compact_out = idx;
  fz.zero_bins = bins;
  fz.n_bins = cfg.angle_bins;
  fz.zero_counts = cnt;
  CoopState* st = coop_refine_launch(c, cs, nullptr, pk->axis, 0, 0.0, cfg, nullptr, nullptr, &dsum->st, &fz);
  {
    StageScope sc(c, kAngles);
    int32_t* hidx = inlier_host_buffer(c, (size_t)std::max<int64_t>(cs.n, 1));
    double* raw = c->raw.get<double>((size_t)std::max<int64_t>(cs.n, 1));
    // the angle vote reads the inlier list coalesced and also streams it to mapped host memory
    launch_vote_angles_k(nullptr, d_corrs, idx, cs.n, cfg.angle_bins, cfg.tau_deg, bins, raw, cnt, c->st, st->axis,
                         &st->count, hidx);
    launch_peak_angle_k(bins, cfg.angle_bins, raw, cs.n, c->angle_sums.get<double>(2 * 296), res, c->done_ptr(),
                        c->st, &st->count);
    count_launch(c, 2);
  }
  // one summary read-back
  static_assert(sizeof(Summary) <= 4096, "pinned scratch");
  Summary* h = reinterpret_cast<Summary*>(c->pinned);
  ck(cudaMemcpyAsync(h, dsum, sizeof(Summary), cudaMemcpyDeviceToHost, c->st), "summary D2H");
  return grid;
}

Estimate complete_single(rv_context* c, const PreResult& pre, const double* d_corrs, const rv_config& cfg,
                         const uint32_t* grid, bool prevoted, bool* identity) {
  const ConstraintSet& cs = pre.cs;
  const Summary sm = *reinterpret_cast<const Summary*>(c->pinned);
  const int64_t n_kept = pre.inorder ? (int64_t)sm.n_kept : cs.n;
  if (pre.inorder) {
    if (prevoted) c->times.vote_launches += 1;
    c->times.vote_samples += (n_kept - (prevoted ? 0 : cs.n)) * (int64_t)cfg.theta_samples;
    if (n_kept == 0 || (cs.n - n_kept) * 10 >= cs.n * 9) {  // estimator.cpp:326-340 shortcuts
      if (!identity) fail(RV_ERR_INVALID_ARGUMENT, "in-order solve without an identity handler");
      *identity = true;
      return Estimate{};
    }
  }
  if (sm.pk.total != (unsigned long long)n_kept * (unsigned long long)cfg.theta_samples) {
    // exactness guard: redo with the generic exact vote
    guard_failed(c, sm.pk.total, (unsigned long long)n_kept * (unsigned long long)cfg.theta_samples);
    if (pre.inorder) {  // ... over the compacted constraint set
      const PreResult pc = preprocess_dev(c, d_corrs, cs.n, cfg.tau_z, cfg.normalize_inputs);
      return finish_single_stepped(c, pc, d_corrs, cfg, nullptr, 1);
    }
    return finish_single_stepped(c, pre, d_corrs, cfg, nullptr, 1);
  }
  if (!sm.pk.ok) fail(RV_ERR_NO_PEAK, "no accumulator cell reaches min_votes");
  Estimate est;
  {  // angle_dev's finish (angles.cpp:46-90)
    if (sm.st.count > 0 && sm.counts[0] == 0) fail(RV_ERR_NO_VOTES, "no correspondence produced an angle vote");
    if (sm.st.count == 0) fail(RV_ERR_NO_VOTES, "no correspondence produced an angle vote");
    const double s = sm.angle[0], co = sm.angle[1], center = sm.angle[3];
    double angle = center;
    if (cfg.refine && !(s == 0.0 && co == 0.0)) {
      angle = std::atan2(s, co);
      if (angle <= -kPiD) angle += 2.0 * kPiD;
    }
    est.angle = angle;
  }
  std::memcpy(est.axis, sm.st.axis, sizeof est.axis);
  rodrigues3(est.axis, est.angle, est.R);
  est.votes = sm.pk.votes;
  const double chance = cfg.epsilon * (double)n_kept;
  const bool rescue = cfg.refine && (double)sm.st.count < 3.0 * chance;
  if (c->allow_view && !rescue) {  // the compaction already wrote the list to mapped memory
    est.view = c->inl_host;
    est.view_n = (int64_t)sm.st.count;
    return est;
  }
  est.inliers = std::move(c->spare);
  est.inliers.assign(c->inl_host, c->inl_host + sm.st.count);
  if (rescue) {
    if (pre.inorder) {  // the rescue path works on the compacted constraint set; the grid is the same
      const PreResult pc = preprocess_dev(c, d_corrs, cs.n, cfg.tau_z, cfg.normalize_inputs);
      est = rescue_single(c, pc, d_corrs, cfg, grid, est);
    } else {
      est = rescue_single(c, pre, d_corrs, cfg, grid, est);
    }
  }
  return est;
}

Estimate finish_single(rv_context* c, const PreResult& pre, const double* d_corrs, const rv_config& cfg,
                       const uint32_t* prevoted, bool peak_ready, bool* identity) {
  const uint32_t* grid = enqueue_single(c, pre, d_corrs, cfg, prevoted, peak_ready);
  sync(c);
  return complete_single(c, pre, d_corrs, cfg, grid, prevoted != nullptr, identity);
}

// The host-stepped solve (same semantics): each stage reads its scalars back before the next.
Estimate finish_single_stepped(rv_context* c, const PreResult& pre, const double* d_corrs, const rv_config& cfg,
                               const uint32_t* prevoted, int first_attempt) {
  const auto [grid, peaks] =
      vote_and_peak(c, pre.cs.zx, pre.cs.zy, pre.cs.zz, pre.cs.n, cfg, 1, false, prevoted, first_attempt);
  Estimate est;
  {  // estimate_from_peak (estimator.cpp:94-101)
    double A, B, b[3], axis[3];
    interpolate_peak_dev(c, grid, cfg.grid, cfg.extent, peaks[0], &A, &B);
    backproject(A, B, b);
    canonicalize3(b, axis);
    const Cls cl = refine_loop_dev(c, pre.cs, axis, cfg);
    est = build_estimate_dev(c, pre.cs, axis, cl, peaks[0].votes, d_corrs, cfg);
  }
  const double chance = cfg.epsilon * (double)pre.cs.n;
  if (cfg.refine && (double)est.inliers.size() < 3.0 * chance) est = rescue_single(c, pre, d_corrs, cfg, grid, est);
  return est;
}

// Rescue (estimator.cpp:352-368): blurred peaks + LS-all annealed candidates, best model support.
// K rescue candidates (build_candidate + model_support each, estimator.cpp:352-368 / 452-466)
// evaluated as ONE device sequence: every candidate's refine (cooperative, compaction fused),
// angle vote and peak are queued back to back with per-candidate summary and inlier slots, read
// back once; the host finishes each angle (libm atan2, as angle_dev) and queues the K model-support
// passes, read back once. Result per candidate: estimate (inliers left in its slot: dev_count),
// coherent/band support, and whether it produced angle votes at all (NoVotes -> skipped).
struct CandResult {
  Estimate est;
  int64_t coherent = 0, band = 0;
  bool ok = false;
  const int32_t* d_idx = nullptr;   // its inlier list on the device
  const uint32_t* d_band = nullptr; // its support band flags (when requested)
};
std::vector<CandResult> evaluate_candidates(rv_context* c, const std::vector<std::array<double, 3>>& starts,
                                            const ConstraintSet& cs, const double* corrs, const rv_config& cfg,
                                            bool want_band) {
  const size_t K = starts.size();
  std::vector<CandResult> out(K);
  if (K == 0) return out;
  if (cfg.angle_bins < 8) fail(RV_ERR_INVALID_CONFIG, "angle histogram needs bin_count >= 8");
  const size_t nn = (size_t)std::max<int64_t>(cs.n, 1);
  const size_t bw = (size_t)(cs.n + 31) / 32 + 32;
  Summary* sums = c->cand_sums.get<Summary>(K);
  int32_t* idx = c->cand_idx.get<int32_t>(K * nn);
  int32_t* sup = c->cand_sup.get<int32_t>(2 * K);
  uint32_t* band = want_band ? c->cand_band.get<uint32_t>(K * bw) : nullptr;
  // every candidate's refine_loop in one cooperative launch (compaction fused), then all K angle
  // votes in one launch and all K peak sums in one launch (per-candidate histograms, angle lists
  // and summary slots): no read-back in between
  static const bool multi_on = [] {
    const char* e = std::getenv("RV_COOP_MULTI");
    return !(e && e[0] == '0');
  }();
  const bool batch = multi_on && K <= 8;  // done counters: c->done_ptr() holds 8
  const size_t KB = batch ? K : 1;
  uint32_t* bins = c->bins.get<uint32_t>(KB * (size_t)cfg.angle_bins);
  double* raw = c->raw.get<double>(KB * nn);
  double* asums = c->angle_sums.get<double>(KB * 2 * 296);
  if (multi_on)
    coop_refine_multi_launch(c, cs, starts, {}, 0, cfg, &sums[0].st, sizeof(Summary), sums[0].counts, idx, nn, bins,
                             cfg.angle_bins);
  if (batch) {
    launch_zero_i32(reinterpret_cast<int32_t*>(bins), (int)(K * (size_t)cfg.angle_bins), c->st);
    launch_vote_angles_batch_k((int)K, corrs, idx, nn, cs.n, cfg.angle_bins, cfg.tau_deg, bins, raw, nn, sums[0].counts,
                               sums[0].st.axis, &sums[0].st.count, sizeof(Summary), c->st);
    launch_peak_angle_batch_k((int)K, bins, cfg.angle_bins, raw, nn, cs.n, asums, sums[0].angle, c->done_ptr(),
                              &sums[0].st.count, sizeof(Summary), c->st);
    count_launch(c, 3);
  }
  for (size_t k = 0; k < K && !batch; ++k) {
    CoopState* st = &sums[k].st;
    if (!multi_on) {
      CoopFused fz;
      fz.compact_out = idx + k * nn;
      fz.zero_bins = bins;
      fz.n_bins = cfg.angle_bins;
      fz.zero_counts = sums[k].counts;
      st = coop_refine_launch(c, cs, starts[k].data(), nullptr, 0, 0.0, cfg, nullptr, nullptr, &sums[k].st, &fz);
    } else if (k > 0) {
      launch_zero_i32(reinterpret_cast<int32_t*>(bins), cfg.angle_bins, c->st);  // histogram of the next vote
      count_launch(c);
    }
    launch_vote_angles_k(nullptr, corrs, idx + k * nn, cs.n, cfg.angle_bins, cfg.tau_deg, bins, raw, sums[k].counts,
                         c->st, st->axis, &st->count, nullptr);
    launch_peak_angle_k(bins, cfg.angle_bins, raw, cs.n, asums, sums[k].angle, c->done_ptr(), c->st, &st->count);
    count_launch(c, 2);
  }
  std::vector<Summary> hs(K);
  read_small(c, hs.data(), sums, K, "candidates D2H");
  const int SM = model_support_multi_max();
  int32_t* bc = c->sup_counts.get<int32_t>((size_t)classify_blocks(cs.n) * 2 * SM);
  std::vector<std::array<double, 3>> ax(K);
  std::vector<double> an(K, 0.0);
  for (size_t k = 0; k < K; ++k) {
    const Summary& sm = hs[k];
    CandResult& r = out[k];
    std::memcpy(ax[k].data(), sm.st.axis, sizeof(double) * 3);
    if (sm.counts[0] == 0) continue;  // angle_dev: NoVotes -> the candidate is skipped
    Estimate& e = r.est;
    std::memcpy(e.axis, sm.st.axis, sizeof e.axis);
    const double sv = sm.angle[0], co = sm.angle[1], center = sm.angle[3];
    double angle = center;
    if (cfg.refine && !(sv == 0.0 && co == 0.0)) {
      angle = std::atan2(sv, co);
      if (angle <= -kPiD) angle += 2.0 * kPiD;
    }
    e.angle = angle;
    an[k] = angle;
    rodrigues3(e.axis, e.angle, e.R);
    e.dev_count = (int64_t)sm.st.count;
    r.d_idx = idx + k * nn;
    r.d_band = band ? band + k * bw : nullptr;
    r.ok = true;
  }
  // every candidate's model_support (estimator.cpp:117-137) in one pass over the constraints per
  // batch of up to SM candidates (skipped candidates are evaluated too and ignored)
  for (size_t k0 = 0; k0 < K; k0 += (size_t)SM) {
    const int kb = (int)std::min<size_t>((size_t)SM, K - k0);
    launch_model_support_multi_k(cs.zx, cs.zy, cs.zz, cs.kept, corrs, cs.n, kb,
                                 reinterpret_cast<const double(*)[3]>(ax[k0].data()), an.data() + k0, cfg.epsilon,
                                 cfg.tau_deg, band ? band + k0 * bw : nullptr, bw, bc, sup + 2 * k0, c->done_ptr(),
                                 c->st);
    count_launch(c);
  }
  std::vector<int32_t> hsup(2 * K);
  read_small(c, hsup.data(), sup, 2 * K, "supports D2H");
  for (size_t k = 0; k < K; ++k) {
    out[k].coherent = hsup[2 * k];
    out[k].band = hsup[2 * k + 1];
  }
  return out;
}

// The winner of a candidate batch: vote lookup at its axis (build_candidate) and its inlier list.
void materialize_candidate(rv_context* c, const uint32_t* grid, const rv_config& cfg, const CandResult& r,
                           Estimate* est, bool look_up_votes) {
  if (look_up_votes) {
    double A, B;
    est->votes = project3(est->axis, &A, &B) ? grid_cell(c, grid, cfg.grid, coord_to_cell(A, cfg.grid, cfg.extent),
                                                          coord_to_cell(B, cfg.grid, cfg.extent))
                                              : 0u;
  }
  est->inliers.clear();
  if (!c->spares.empty()) {  // a previous call's inlier vector: no page faults
    est->inliers = std::move(c->spares.back());
    c->spares.pop_back();
  }
  if (est->dev_count > 0) {  // through the pinned inlier buffer: a pageable D2H stages at a fraction of the rate
    int32_t* h = inlier_host_buffer(c, (size_t)est->dev_count);
    ck(cudaMemcpyAsync(h, r.d_idx, sizeof(int32_t) * (size_t)est->dev_count, cudaMemcpyDeviceToHost, c->st),
       "inliers D2H");
    sync(c);
    est->inliers.assign(h, h + est->dev_count);
  } else {
    est->inliers.clear();
    sync(c);
  }
  est->dev_count = -1;
}

Estimate rescue_single(rv_context* c, const PreResult& pre, const double* d_corrs, const rv_config& cfg,
                       const uint32_t* grid, Estimate est) {
  int64_t best = model_support_dev(c, pre.cs, d_corrs, est, cfg, nullptr).coherent;
  const auto res = evaluate_candidates(c, rescue_axes_dev(c, grid, pre.cs, cfg), pre.cs, d_corrs, cfg, false);
  const CandResult* win = nullptr;
  for (const auto& r : res)  // in order, strictly better than the incumbent (estimator.cpp:360-367)
    if (r.ok && r.coherent > best) {
      best = r.coherent;
      win = &r;
    }
  if (win) {
    est = win->est;
    materialize_candidate(c, grid, cfg, *win, &est, true);
  }
  return est;
}

// near_identity_model (estimator.cpp:224-249) over the residual set.
bool near_identity_dev(rv_context* c, const double* d_corrs, const ConstraintSet& sub, const rv_config& cfg,
                       int64_t min_cluster, Estimate* out) {
  StageScope sc(c, kAngles);
  const int nb = classify_blocks(sub.n);
  uint32_t* flags = c->flagsA.get<uint32_t>((size_t)(sub.n + 31) / 32 + 32);
  int32_t* offs = c->boffA.get<int32_t>(nb);
  double* res = c->near_result.get<double>(10);
  launch_near_identity_k(d_corrs, sub.kept, sub.n, cfg.normalize_inputs, flags, c->bcount.get<int32_t>(nb),
                         c->near_h.get<double>((size_t)nb * 9), offs, res, c->done_ptr(), c->st);
  count_launch(c);
  double* h = pin_d(c);
  ck(cudaMemcpyAsync(h, res, sizeof(double) * 10, cudaMemcpyDeviceToHost, c->st), "near D2H");
  sync(c);
  const int64_t nc = (int64_t)h[0];
  if (nc < std::max<int64_t>(min_cluster, 3)) return false;
  double hm[9];
  std::memcpy(hm, h + 1, sizeof hm);
  int32_t* idx = c->compact_out.get<int32_t>((size_t)nc);
  launch_compact_flags(flags, sub.n, sub.kept, offs, idx, c->st);
  count_launch(c);
  Estimate e;
  e.inliers.resize(nc);
  ck(cudaMemcpyAsync(e.inliers.data(), idx, sizeof(int32_t) * nc, cudaMemcpyDeviceToHost, c->st), "cluster D2H");
  sync(c);
  kabsch(hm, e.R);
  angle_axis_canonical(e.R, e.axis, &e.angle);
  e.votes = (uint32_t)nc;
  *out = std::move(e);
  return true;
}

// One-pass top-K multi-model mode (an extension, not in the reference):
// ONE vote over all constraints, find_peaks with K = max_models (the reference's greedy NMS with
// the equatorial mirror, voting.cpp:120-170) at the reference's peak_vote_floor, then per peak
// the reference's single-model finish (estimate_from_peak + refine_loop + build_estimate) and its
// acceptance rules (consensus floor, model_support coherence, inlier-overlap dedupe). Unlike the
// sequential estimate_multi it does not strip inliers and re-vote, so K models cost one vote.
// Models are returned in peak order (descending axis_votes).
// The dedupe of estimate_multi (estimator.cpp:468-478): |inliers ∩ accepted model's inliers| as the
// popcount of the AND of two input-index bitsets (word-parallel; the per-index lookup loop cost
// ~50 us per accepted model at 1e5 inliers).
// Inlier bitsets of the accepted models for the dedupe test (estimator.cpp:452-458: |common
// inliers| > dedupe_overlap * |inliers| rejects a model), in context-owned storage reused across
// calls -- fresh n-bit vectors per model page-faulted on every call -- and intersected a word at a
// time with the hardware popcount.
#if defined(__x86_64__)
__attribute__((target("popcnt"))) int64_t common_bits_hw(const uint64_t* a, const uint64_t* b, size_t m) {
  int64_t s = 0;
  for (size_t w = 0; w < m; ++w) s += __builtin_popcountll(a[w] & b[w]);
  return s;
}
#endif
int64_t common_bits(const uint64_t* a, const uint64_t* b, size_t m) {
#if defined(__x86_64__)
  static const bool hw = __builtin_cpu_supports("popcnt");
  if (hw) return common_bits_hw(a, b, m);
#endif
  int64_t s = 0;
  for (size_t w = 0; w < m; ++w) s += __builtin_popcountll(a[w] & b[w]);
  return s;
}
class InlierSets {
 public:
  InlierSets(rv_context* c, int64_t n) : pool_(c->dedupe_bits), words_((size_t)(n + 63) / 64) {}
  // true when the model with these inliers repeats an accepted one; otherwise it is accepted
  bool duplicate_else_accept(const std::vector<int32_t>& inl, double overlap) {
    if (pool_.size() <= used_) pool_.resize(used_ + 1);
    std::vector<uint64_t>& bits = pool_[used_];
    bits.assign(words_, 0);  // keeps its capacity: no page faults after the first call
    for (const int32_t i : inl) bits[(size_t)i >> 6] |= 1ull << (i & 63);
    for (size_t k = 0; k < used_; ++k)
      if ((double)common_bits(bits.data(), pool_[k].data(), words_) > overlap * (double)inl.size()) return true;
    ++used_;
    return false;
  }

 private:
  std::vector<std::vector<uint64_t>>& pool_;
  size_t words_;
  size_t used_ = 0;
};

std::vector<Estimate> estimate_multi_onepass_dev(rv_context* c, const double* d_corrs, int64_t n,
                                                 const rv_config& cfg) {
  if (n <= 0) fail(RV_ERR_EMPTY_INPUT, "no correspondences");
  const PreResult pre = preprocess_dev(c, d_corrs, n, cfg.tau_z, cfg.normalize_inputs, &cfg);
  if (pre.cs.n == 0) fail(RV_ERR_ALL_DEGENERATE, "every correspondence pair is degenerate (x ~ y)");
  const double chance = cfg.epsilon * (double)pre.cs.n;
  const int64_t consensus_floor = (int64_t)std::max(2.0, cfg.consensus_floor_mult * chance);
  const uint32_t* grid = vote(c, pre.cs.zx, pre.cs.zy, pre.cs.zz, pre.cs.n, cfg.grid, cfg.extent,
                              cfg.theta_samples, false, pre.vote_zeroed);
  std::vector<Peak> peaks;
  try {
    peaks = find_peaks_dev(c, grid, cfg.grid, cfg.extent, std::max(1, cfg.max_models), cfg.suppression_radius,
                           rv_peak_vote_floor(&cfg, pre.cs.n));
  } catch (const RvError& e) {
    if (e.st != RV_ERR_NO_PEAK) throw;
    return {};
  }
  std::vector<Estimate> out;
  InlierSets accepted(c, n);
  for (const Peak& pk : peaks) {
    double A, B, b[3], axis[3];
    interpolate_peak_dev(c, grid, cfg.grid, cfg.extent, pk, &A, &B);
    backproject(A, B, b);
    canonicalize3(b, axis);
    Estimate est;
    try {
      const Cls cl = refine_loop_dev(c, pre.cs, axis, cfg);
      est = build_estimate_dev(c, pre.cs, axis, cl, pk.votes, d_corrs, cfg);
    } catch (const RvError& e) {
      if (e.st == RV_ERR_NO_VOTES) continue;
      throw;
    }
    const Support sup = model_support_dev(c, pre.cs, d_corrs, est, cfg, nullptr);
    if ((int64_t)est.inliers.size() < consensus_floor ||
        sup.coherent < std::max<int64_t>(8, (int64_t)est.inliers.size() / 5))
      continue;
    if (!accepted.duplicate_else_accept(est.inliers, cfg.dedupe_overlap)) out.push_back(std::move(est));
  }
  return out;
}

// estimate_multi (estimator.cpp:373-493)
std::vector<Estimate> estimate_multi_dev(rv_context* c, const double* d_corrs, int64_t n, const rv_config& cfg) {
  if (n <= 0) fail(RV_ERR_EMPTY_INPUT, "no correspondences");
  const PreResult pre = preprocess_dev(c, d_corrs, n, cfg.tau_z, cfg.normalize_inputs);
  if (pre.cs.n == 0) fail(RV_ERR_ALL_DEGENERATE, "every correspondence pair is degenerate (x ~ y)");
  const double chance = cfg.epsilon * (double)pre.cs.n;
  const int64_t consensus_floor = (int64_t)std::max(2.0, cfg.consensus_floor_mult * chance);
  uint8_t* removed = c->removed.get<uint8_t>(pre.cs.n);
  ck(cudaMemsetAsync(removed, 0, pre.cs.n, c->st), "memset removed");
  std::vector<Estimate> out;
  InlierSets accepted(c, n);
  while ((int)out.size() < cfg.max_models) {
    // residual (estimator.cpp:392-398)
    ConstraintSet sub;
    {
      StageScope sc(c, kPrep);
      const int nb = (int)((pre.cs.n + 255) / 256);
      unsigned long long* stt = c->status.get<unsigned long long>(nb);
      int32_t* misc = c->misc32.get<int32_t>(8);
      ck(cudaMemsetAsync(stt, 0, sizeof(unsigned long long) * nb, c->st), "memset status");
      ck(cudaMemsetAsync(misc, 0, sizeof(int32_t) * 8, c->st), "memset misc");
      double* ozx = c->rzx.get<double>(pre.cs.n);
      double* ozy = c->rzy.get<double>(pre.cs.n);
      double* ozz = c->rzz.get<double>(pre.cs.n);
      int32_t* okept = c->rkept.get<int32_t>(pre.cs.n);
      launch_gather_residual(pre.cs.zx, pre.cs.zy, pre.cs.zz, pre.cs.kept, removed, pre.cs.n, stt, misc, ozx, ozy,
                             ozz, okept, misc + 4, c->st);
      count_launch(c);
      int32_t* h = reinterpret_cast<int32_t*>(c->pinned);
      ck(cudaMemcpyAsync(h, misc + 4, 4, cudaMemcpyDeviceToHost, c->st), "residual D2H");
      sync(c);
      sub.zx = ozx;
      sub.zy = ozy;
      sub.zz = ozz;
      sub.kept = okept;
      sub.n = h[0];
    }
    if (sub.n < std::max<int64_t>(2, consensus_floor)) break;
    const auto [grid, peaks] = vote_and_peak(c, sub.zx, sub.zy, sub.zz, sub.n, cfg, rv_peak_vote_floor(&cfg, sub.n), true);
    const bool have_peak = !peaks.empty();
    Estimate est;
    Support sup;
    bool have = false;
    uint32_t* best_band = c->band_flagsA.get<uint32_t>((size_t)(pre.cs.n + 31) / 32 + 32);
    if (have_peak) {
      std::vector<std::array<double, 3>> starts;
      double A, B, b[3], s0[3];
      interpolate_peak_dev(c, grid, cfg.grid, cfg.extent, peaks[0], &A, &B);
      backproject(A, B, b);
      canonicalize3(b, s0);
      starts.push_back({s0[0], s0[1], s0[2]});
      for (const auto& a : rescue_axes_dev(c, grid, sub, cfg)) starts.push_back(a);
      // all candidates as one device batch (per-candidate slots, two read-backs); the first usable
      // one wins unless a later one has strictly more coherent support (estimator.cpp:415-433)
      const auto res = evaluate_candidates(c, starts, pre.cs, d_corrs, cfg, true);
      const CandResult* win = nullptr;
      size_t win_k = 0;
      for (size_t k = 0; k < res.size(); ++k)
        if (res[k].ok && (!win || res[k].coherent > win->coherent)) {
          win = &res[k];
          win_k = k;
        }
      if (win) {
        est = win->est;
        sup.coherent = win->coherent;
        sup.band = win->band;
        best_band = const_cast<uint32_t*>(win->d_band);
        est.votes = win_k == 0 ? peaks[0].votes : 0u;
        materialize_candidate(c, grid, cfg, *win, &est, win_k != 0);
        have = true;
      }
    }
    bool identity_model = false;
    const bool valid = have && (int64_t)est.inliers.size() >= consensus_floor &&
                       sup.coherent >= std::max<int64_t>(8, (int64_t)est.inliers.size() / 5);
    if (!valid) {
      Estimate ident;
      if (!near_identity_dev(c, d_corrs, sub, cfg, consensus_floor, &ident)) break;
      est = std::move(ident);
      identity_model = true;
    }
    // the strip (estimator.cpp:470-480) is queued before the host's duplicate test, so the GPU runs
    // it while the host intersects the inlier bitsets; a duplicate ends the loop and leaves the
    // strip unused
    if (identity_model) {
      launch_strip_identity_k(d_corrs, pre.cs.kept, pre.cs.n, cfg.normalize_inputs, removed, c->st);
      count_launch(c);
    } else {
      const double strip = 2.0 * cfg.epsilon;
      if (sup.band > 0) {
        // strip = max(2 eps, 1.25 * the 95th-percentile band value) (nth_element's q-th smallest
        // over the winner's support band, whose size the host already has from model_support):
        // selected and applied on the device, no read-back
        const long long acc = (long long)sup.band;
        const long long q = std::min(acc - 1, (acc * 95) / 100);
        unsigned long long* keys = c->band_vals.get<unsigned long long>((size_t)acc + 1);  // count + keys
        double* sdev = c->strip_val.get<double>(1);
        launch_band_strip_k(best_band, pre.cs.n, pre.cs.zx, pre.cs.zy, pre.cs.zz, est.axis, q, strip, keys, sdev,
                            removed, c->st);
        count_launch(c, 3);
      } else {
        launch_strip_k(pre.cs.zx, pre.cs.zy, pre.cs.zz, pre.cs.n, est.axis, strip, removed, c->st);
        count_launch(c);
      }
    }
    if (accepted.duplicate_else_accept(est.inliers, cfg.dedupe_overlap)) break;
    out.push_back(std::move(est));
  }
  if (out.empty()) fail(RV_ERR_NO_PEAK, "no peak produced a usable model");
  std::stable_sort(out.begin(), out.end(), [](const Estimate& a, const Estimate& b) { return a.votes > b.votes; });
  return out;
}

void to_c(const Estimate& e, rv_estimate* o, double elapsed) {
  std::memcpy(o->axis, e.axis, sizeof o->axis);
  o->angle = e.angle;
  std::memcpy(o->rotation, e.R, sizeof o->rotation);
  o->axis_votes = e.votes;
  o->n_inliers = e.n_inliers();
  o->elapsed_s = elapsed;
}

template <typename F>
rv_status guarded(rv_context* c, F&& f) {
  try {
    if (c) begin_call(c);
    f();
    if (c) end_call(c);
    return RV_OK;
  } catch (const RvError& e) {
    if (c) {
      c->last_error = e.msg;
      if (e.st == RV_ERR_CUDA) cudaGetLastError();
    }
    return e.st;
  } catch (const std::bad_alloc&) {
    if (c) c->last_error = "host allocation failed";
    return RV_ERR_OUT_OF_MEMORY;
  } catch (...) {
    if (c) c->last_error = "unexpected exception";
    return RV_ERR_INVALID_ARGUMENT;
  }
}

double seconds_since(const rv_context* c) {
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - c->t0).count();
}

// Constraint span (host, n x 3 AoS) -> device SoA in the context's preprocess buffers.
ConstraintSet upload_constraints(rv_context* c, const double* z, int64_t n) {
  std::vector<double> sx(n), sy(n), szz(n);
  for (int64_t i = 0; i < n; ++i) {
    sx[i] = z[3 * i];
    sy[i] = z[3 * i + 1];
    szz[i] = z[3 * i + 2];
  }
  ConstraintSet cs;
  double* dx = c->zx.get<double>(n);
  double* dy = c->zy.get<double>(n);
  double* dz = c->zz.get<double>(n);
  ck(cudaMemcpyAsync(dx, sx.data(), 8 * n, cudaMemcpyHostToDevice, c->st), "H2D zx");
  ck(cudaMemcpyAsync(dy, sy.data(), 8 * n, cudaMemcpyHostToDevice, c->st), "H2D zy");
  ck(cudaMemcpyAsync(dz, szz.data(), 8 * n, cudaMemcpyHostToDevice, c->st), "H2D zz");
  sync(c);
  cs.zx = dx;
  cs.zy = dy;
  cs.zz = dz;
  cs.kept = nullptr;
  cs.n = n;
  return cs;
}

}  // namespace

// =========================================================================================
extern "C" {

int32_t rv_abi_version(void) { return RV_ABI_VERSION; }

void rv_config_default(rv_config* c) {  // estimator.hpp:13-29
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

const char* rv_status_string(rv_status st) {
  switch (st) {
    case RV_OK: return "ok";
    case RV_ERR_EMPTY_INPUT: return "EmptyInput";
    case RV_ERR_NO_PEAK: return "NoPeak";
    case RV_ERR_DEGENERATE_PROJECTION: return "DegenerateProjection";
    case RV_ERR_NO_VOTES: return "NoVotes";
    case RV_ERR_ALL_DEGENERATE: return "AllDegenerate";
    case RV_ERR_RANK_DEFICIENT: return "RankDeficient";
    case RV_ERR_NO_CONSENSUS: return "NoConsensus";
    case RV_ERR_INVALID_CONFIG: return "InvalidConfig";
    case RV_ERR_POLE_PROXIMITY: return "PoleProximity";
    case RV_ERR_OUT_OF_MEMORY: return "OutOfMemory";
    case RV_ERR_CUDA: return "CudaError";
    case RV_ERR_NCCL: return "NcclError";
    case RV_ERR_INVALID_ARGUMENT: return "InvalidArgument";
    case RV_ERR_NO_DEVICE: return "NoDevice";
    case RV_ERR_PARSE: return "ParseError";
    case RV_ERR_EMPTY_FILE: return "EmptyFile";
    case RV_ERR_IO: return "IoError";
  }
  return "unknown";
}

rv_status rv_context_create(int32_t device, rv_context** out) {
  if (!out) return RV_ERR_INVALID_ARGUMENT;
  *out = nullptr;
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
    cudaGetLastError();
    return RV_ERR_NO_DEVICE;
  }
  if (device < 0 || device >= count) return RV_ERR_INVALID_ARGUMENT;
  auto* c = new (std::nothrow) rv_context();
  if (!c) return RV_ERR_OUT_OF_MEMORY;
  c->device = device;
  if (cudaSetDevice(device) != cudaSuccess || cudaStreamCreateWithFlags(&c->own, cudaStreamNonBlocking) != cudaSuccess ||
      cudaMallocHost(&c->pinned, kPinnedScratch) != cudaSuccess) {
    cudaGetLastError();
    delete c;
    return RV_ERR_CUDA;
  }
  c->st = c->own;
  cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, device);
  cudaDeviceGetAttribute(&c->max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  *out = c;
  return RV_OK;
}

void rv_context_destroy(rv_context* c) {
  if (!c) return;
  for (rv_context* w : c->pool) rv_context_destroy(w);
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->st);
  for (auto e : c->event_pool) cudaEventDestroy(e);
  for (auto e : c->chunk_events) cudaEventDestroy(e);
  if (c->copy_st) cudaStreamDestroy(c->copy_st);
  for (auto& g : c->graphs)
    if (g.exec) cudaGraphExecDestroy(g.exec);
  if (c->cap_st) cudaStreamDestroy(c->cap_st);
  if (c->pinned) cudaFreeHost(c->pinned);
  if (c->inl_host) cudaFreeHost(c->inl_host);
  if (c->csv_pinned) cudaFreeHost(c->csv_pinned);
  if (c->in_pinned) cudaFreeHost(c->in_pinned);
  if (c->big_pinned) cudaFreeHost(c->big_pinned);
  for (void* q : c->xlines_peers) cudaIpcCloseMemHandle(q);
  if (c->xlines_own) cudaFree(c->xlines_own);
  c->copy_pool.reset();
  if (c->own) cudaStreamDestroy(c->own);
  delete c;
}

rv_status rv_context_set_stream(rv_context* c, void* stream) {
  if (!c) return RV_ERR_INVALID_ARGUMENT;
  c->st = stream ? static_cast<cudaStream_t>(stream) : c->own;
  return RV_OK;
}

const char* rv_context_last_error(const rv_context* c) { return c ? c->last_error.c_str() : "null context"; }

rv_status rv_context_enable_timing(rv_context* c, int32_t enable) {
  if (!c) return RV_ERR_INVALID_ARGUMENT;
  c->timing = enable != 0;
  return RV_OK;
}

rv_status rv_context_stage_times(const rv_context* c, rv_stage_times* out) {
  if (!c || !out) return RV_ERR_INVALID_ARGUMENT;
  *out = c->times;
  return RV_OK;
}

static void clear_results(rv_context* c) {
  c->results.clear();
  c->result0_view = nullptr;
  c->result0_view_n = 0;
}

// multi-model calls: every result vector goes back to the spare pool (at most 16 kept)
static void recycle_all_results(rv_context* c) {
  for (auto& v : c->results)
    if (c->spares.size() < 16 && v.capacity() > 0) c->spares.push_back(std::move(v));
  clear_results(c);
}

static void recycle_results(rv_context* c) {
  if (!c->results.empty() && c->results[0].capacity() > c->spare.capacity()) c->spare = std::move(c->results[0]);
  c->results.clear();
  c->result0_view = nullptr;
  c->result0_view_n = 0;
}

// Store a single-solve estimate's inliers as results[0] (a view into the mapped buffer if the
// solve left them there).
static void push_single_result(rv_context* c, Estimate& e) {
  c->results.push_back(std::move(e.inliers));
  c->result0_view = e.view;
  c->result0_view_n = e.view_n;
}

// results[0] of a worker context as an owned vector (a view would be overwritten by the worker's
// next solve).
static std::vector<int32_t> take_result0(rv_context* w) {
  if (w->result0_view) return std::vector<int32_t>(w->result0_view, w->result0_view + w->result0_view_n);
  return std::move(w->results[0]);
}

rv_status rv_estimate_single_device(rv_context* c, const double* d_corrs, int64_t n, const rv_config* cfg,
                                    rv_estimate* out) {
  if (!c || !cfg || !out || (n > 0 && !d_corrs)) return RV_ERR_INVALID_ARGUMENT;
  return guarded(c, [&] {
    cudaSetDevice(c->device);
    recycle_results(c);
    c->allow_view = true;
    Estimate e = estimate_single_dev(c, d_corrs, n, *cfg);
    c->allow_view = false;
    to_c(e, out, seconds_since(c));
    push_single_result(c, e);
  });
}

rv_status rv_estimate_single(rv_context* c, const double* corrs, int64_t n, const rv_config* cfg, rv_estimate* out) {
  if (!c || !cfg || !out || (n > 0 && !corrs)) return RV_ERR_INVALID_ARGUMENT;
  return guarded(c, [&] {
    cudaSetDevice(c->device);
    recycle_results(c);
    if (n <= 0) fail(RV_ERR_EMPTY_INPUT, "no correspondences");
    c->allow_view = true;
    Estimate e = estimate_single_host(c, corrs, n, *cfg);
    c->allow_view = false;
    to_c(e, out, seconds_since(c));
    push_single_result(c, e);
  });
}

static rv_status multi_impl(rv_context* c, const double* d, int64_t n, const rv_config* cfg, rv_estimate* out,
                            int32_t capacity, int32_t* n_models, bool host, bool onepass = false) {
  return guarded(c, [&] {
    cudaSetDevice(c->device);
    recycle_all_results(c);
    *n_models = 0;
    if (n <= 0) fail(RV_ERR_EMPTY_INPUT, "no correspondences");
    const double* dd = host ? upload_corrs(c, d, n) : d;
    std::vector<Estimate> v = onepass ? estimate_multi_onepass_dev(c, dd, n, *cfg) : estimate_multi_dev(c, dd, n, *cfg);
    const double el = seconds_since(c);
    for (size_t k = 0; k < v.size(); ++k) {
      if ((int32_t)k < capacity) to_c(v[k], out + k, el);
      c->results.push_back(std::move(v[k].inliers));
    }
    *n_models = (int32_t)v.size();
  });
}

rv_status rv_estimate_multi(rv_context* c, const double* corrs, int64_t n, const rv_config* cfg, rv_estimate* out,
                            int32_t capacity, int32_t* n_models) {
  if (!c || !cfg || !out || !n_models || (n > 0 && !corrs)) return RV_ERR_INVALID_ARGUMENT;
  return multi_impl(c, corrs, n, cfg, out, capacity, n_models, true);
}

rv_status rv_estimate_multi_device(rv_context* c, const double* d_corrs, int64_t n, const rv_config* cfg,
                                   rv_estimate* out, int32_t capacity, int32_t* n_models) {
  if (!c || !cfg || !out || !n_models || (n > 0 && !d_corrs)) return RV_ERR_INVALID_ARGUMENT;
  return multi_impl(c, d_corrs, n, cfg, out, capacity, n_models, false);
}

rv_status rv_estimate_multi_onepass(rv_context* c, const double* corrs, int64_t n, const rv_config* cfg,
                                    rv_estimate* out, int32_t capacity, int32_t* n_models) {
  if (!c || !cfg || !out || !n_models || (n > 0 && !corrs)) return RV_ERR_INVALID_ARGUMENT;
  return multi_impl(c, corrs, n, cfg, out, capacity, n_models, true, true);
}

rv_status rv_estimate_multi_onepass_device(rv_context* c, const double* d_corrs, int64_t n, const rv_config* cfg,
                                           rv_estimate* out, int32_t capacity, int32_t* n_models) {
  if (!c || !cfg || !out || !n_models || (n > 0 && !d_corrs)) return RV_ERR_INVALID_ARGUMENT;
  return multi_impl(c, d_corrs, n, cfg, out, capacity, n_models, false, true);
}

rv_status rv_estimate_batch(rv_context* c, const double* corrs, const int64_t* offsets, int32_t n_problems,
                            const rv_config* cfg, int32_t workers, rv_estimate* out, int32_t* status) {
  if (!c || !cfg || !offsets || !out || !status || n_problems < 0 || (n_problems > 0 && !corrs))
    return RV_ERR_INVALID_ARGUMENT;
  for (int32_t k = 0; k < n_problems; ++k)
    if (offsets[k + 1] < offsets[k]) return RV_ERR_INVALID_ARGUMENT;
  return guarded(c, [&] {
    cudaSetDevice(c->device);
    clear_results(c);
    c->results.resize((size_t)n_problems);
    // automatic width (measured on B200): small problems are launch/latency bound and overlap
    // well on 8 streams (3-4x); problems >= ~32k correspondences already fill the GPU, where
    // concurrent band-tiled votes only compete for SMs
    int auto_w = 8;
    if (n_problems > 0 && (offsets[n_problems] - offsets[0]) / n_problems >= 32768) auto_w = 1;
    const int W = std::max(1, std::min<int>(n_problems, workers > 0 ? workers : auto_w));
    while ((int)c->pool.size() < W) {  // each worker: own context = own stream and buffers
      rv_context* w = nullptr;
      const rv_status st = rv_context_create(c->device, &w);
      if (st != RV_OK) fail(st, "batch worker context");
      c->pool.push_back(w);
    }
    std::atomic<int32_t> next{0};
    auto work = [&](rv_context* w) {
      cudaSetDevice(c->device);
      for (int32_t k = next.fetch_add(1); k < n_problems; k = next.fetch_add(1)) {
        const int64_t n = offsets[k + 1] - offsets[k];
        status[k] = rv_estimate_single(w, corrs + 6 * offsets[k], n, cfg, &out[k]);
        if (status[k] == RV_OK) c->results[k] = take_result0(w);
      }
    };
    std::vector<std::thread> th;
    for (int i = 1; i < W; ++i) th.emplace_back(work, c->pool[i]);
    work(c->pool[0]);
    for (auto& t : th) t.join();
  });
}

// ---- baselines (reference baselines.cpp) ------------------------------
// Consensus scoring of many axes is the O(M*N) part and runs on the device (consensus_kernel);
// the hypothesis generation of ransac_rotation is the reference's sequential RNG stream on the
// host (std::mt19937_64 + std::uniform_int_distribution, libstdc++ -- the same stream).
std::vector<uint32_t> consensus_counts_dev(rv_context* c, const double* h_axes, int m, const double* d_z_aos,
                                           int64_t n, double eps) {
  std::vector<uint32_t> out((size_t)std::max(m, 0));
  if (m <= 0) return out;
  double* da = c->cons_axes.get<double>((size_t)3 * m);
  uint32_t* dc = c->cons_counts.get<uint32_t>((size_t)m);
  ck(cudaMemcpyAsync(da, h_axes, sizeof(double) * 3 * m, cudaMemcpyHostToDevice, c->st), "H2D axes");
  ck(cudaMemsetAsync(dc, 0, sizeof(uint32_t) * m, c->st), "memset counts");
  launch_consensus_counts(da, m, d_z_aos, n, eps, dc, c->sms, c->st);
  count_launch(c);
  ck(cudaMemcpyAsync(out.data(), dc, sizeof(uint32_t) * m, cudaMemcpyDeviceToHost, c->st), "D2H counts");
  sync(c);
  return out;
}

const double* upload_aos(rv_context* c, DBuf& buf, const double* h, int64_t n_doubles) {
  double* d = buf.get<double>((size_t)std::max<int64_t>(n_doubles, 1));
  if (n_doubles > 0)
    ck(cudaMemcpyAsync(d, h, sizeof(double) * n_doubles, cudaMemcpyHostToDevice, c->st), "H2D");
  return d;
}

// oracle_direction (baselines.cpp:150-157): Fibonacci spiral over the southern hemisphere.
void oracle_direction_host(int k, int directions, double out[3]) {
  constexpr double golden_angle = 2.399963229728653;
  const double cz = -(k + 0.5) / directions;
  const double sz = std::sqrt(std::max(0.0, 1.0 - cz * cz));
  const double phi = golden_angle * k;
  out[0] = sz * std::cos(phi);
  out[1] = sz * std::sin(phi);
  out[2] = cz;
}

// correspondence_angle (angles.cpp:36-44) on the host, the reference's op order; false =
// DegenerateProjection.
bool corr_angle_host(const double a[3], const double* x, const double* y, double tau, double* angle) {
  double b[3], g[3], bg[3];
  cross3(a, x, b);
  cross3(a, y, g);
  if (std::sqrt(dot3(b, b)) <= tau || std::sqrt(dot3(g, g)) <= tau) return false;
  cross3(b, g, bg);
  *angle = std::atan2(dot3(bg, a), dot3(b, g));
  return true;
}

rv_status rv_grid_oracle_axis(rv_context* c, const double* z, int64_t n, int32_t directions, double epsilon,
                              double axis_out[3], int32_t* count_out) {
  if (!c || !axis_out || !count_out || (n > 0 && !z)) return RV_ERR_INVALID_ARGUMENT;
  return guarded(c, [&] {
    cudaSetDevice(c->device);
    if (n <= 0) fail(RV_ERR_EMPTY_INPUT, "no constraints");
    if (directions < 100) fail(RV_ERR_INVALID_CONFIG, "oracle needs at least 100 directions");
    std::vector<double> dirs((size_t)3 * directions);
    for (int k = 0; k < directions; ++k) oracle_direction_host(k, directions, &dirs[3 * (size_t)k]);
    const double* dz = upload_aos(c, c->cons_z, z, 3 * n);
    const std::vector<uint32_t> cnt = consensus_counts_dev(c, dirs.data(), directions, dz, n, epsilon);
    int best = -1, bk = 0;  // strict '>' in direction order: ties keep the lowest index
    for (int k = 0; k < directions; ++k)
      if ((int)cnt[k] > best) {
        best = (int)cnt[k];
        bk = k;
      }
    std::memcpy(axis_out, &dirs[3 * (size_t)bk], sizeof(double) * 3);
    *count_out = best;
  });
}

rv_status rv_consensus_counts(rv_context* c, const double* axes, int32_t m, const double* z, int64_t n,
                              double epsilon, uint32_t* counts_out) {
  if (!c || m < 0 || n < 0 || (m > 0 && (!axes || !counts_out)) || (n > 0 && !z)) return RV_ERR_INVALID_ARGUMENT;
  return guarded(c, [&] {
    cudaSetDevice(c->device);
    if (m == 0) return;
    if (n == 0) {
      std::memset(counts_out, 0, sizeof(uint32_t) * m);
      return;
    }
    const double* dz = upload_aos(c, c->cons_z, z, 3 * n);
    const std::vector<uint32_t> cnt = consensus_counts_dev(c, axes, m, dz, n, epsilon);
    std::memcpy(counts_out, cnt.data(), sizeof(uint32_t) * m);
  });
}

rv_status rv_ransac_rotation(rv_context* c, const double* corrs, int64_t n, int32_t iterations, double epsilon,
                             uint64_t seed, rv_estimate* out) {
  if (!c || !out || (n > 0 && !corrs)) return RV_ERR_INVALID_ARGUMENT;
  return guarded(c, [&] {
    cudaSetDevice(c->device);
    clear_results(c);
    constexpr double kTauZ = 1e-9, kTauDeg = 1e-6;
    if (n < 2) fail(RV_ERR_NO_CONSENSUS, "need at least two correspondences");
    // preprocess(correspondences, kTauZ, true) (baselines.cpp:35, estimator.cpp:259-285) on the
    // device -- the solver's own kernel; the hypothesis stream below draws constraint pairs
    // sequentially from the host RNG, so the compacted z and kept map come back to the host
    const double* dcorr = upload_corrs(c, corrs, n);
    const PreResult pre = preprocess_dev(c, dcorr, n, kTauZ, 1);
    // preprocess throws AllDegenerate when every pair is dropped (estimator.cpp:280-283)
    if (pre.cs.n == 0) fail(RV_ERR_ALL_DEGENERATE, "every correspondence pair is degenerate (x ~ y)");
    const ConstraintSet cs = pre.cs;
    std::vector<double> z((size_t)3 * (size_t)cs.n);
    std::vector<int32_t> kept((size_t)cs.n);
    if (cs.n > 0) {
      std::vector<double> sx((size_t)cs.n), sy((size_t)cs.n), sz((size_t)cs.n);
      ck(cudaMemcpyAsync(sx.data(), cs.zx, 8 * (size_t)cs.n, cudaMemcpyDeviceToHost, c->st), "D2H zx");
      ck(cudaMemcpyAsync(sy.data(), cs.zy, 8 * (size_t)cs.n, cudaMemcpyDeviceToHost, c->st), "D2H zy");
      ck(cudaMemcpyAsync(sz.data(), cs.zz, 8 * (size_t)cs.n, cudaMemcpyDeviceToHost, c->st), "D2H zz");
      ck(cudaMemcpyAsync(kept.data(), cs.kept, 4 * (size_t)cs.n, cudaMemcpyDeviceToHost, c->st), "D2H kept");
      sync(c);
      for (int64_t i = 0; i < cs.n; ++i) {
        z[(size_t)(3 * i)] = sx[(size_t)i];
        z[(size_t)(3 * i + 1)] = sy[(size_t)i];
        z[(size_t)(3 * i + 2)] = sz[(size_t)i];
      }
    }
    const size_t nz = kept.size();
    if (nz < 2) fail(RV_ERR_NO_CONSENSUS, "fewer than two usable constraints");
    // hypotheses: the reference's loop (baselines.cpp:41-77) minus the scoring
    std::mt19937_64 rng(seed);
    std::uniform_int_distribution<std::size_t> pick(0, nz - 1);
    std::vector<double> axes;
    std::vector<double> angles;
    const long attempt_cap = 50L * iterations + 100;
    long attempts = 0;
    for (int it = 0; it < iterations && attempts < attempt_cap; ++it) {
      ++attempts;
      const std::size_t i = pick(rng);
      const std::size_t j = pick(rng);
      if (i == j) {
        --it;
        continue;
      }
      double ax[3];
      cross3(&z[3 * i], &z[3 * j], ax);
      const double nrm = std::sqrt(dot3(ax, ax));
      if (nrm <= 1e-9) {
        --it;
        continue;
      }
      const double u[3] = {ax[0] / nrm, ax[1] / nrm, ax[2] / nrm};
      double a[3];
      canonicalize3(u, a);
      double angle;
      const double* cr = corrs + 6 * (size_t)kept[i];
      if (!corr_angle_host(a, cr, cr + 3, kTauDeg, &angle)) {
        --it;
        continue;
      }
      axes.insert(axes.end(), a, a + 3);
      angles.push_back(angle);
    }
    const int m = (int)angles.size();
    const double* dz = upload_aos(c, c->cons_z, z.data(), (int64_t)z.size());
    const std::vector<uint32_t> score = consensus_counts_dev(c, axes.data(), m, dz, (int64_t)nz, epsilon);
    int best_score = 0, bk = -1;
    for (int k = 0; k < m; ++k)
      if ((int)score[k] > best_score) {
        best_score = (int)score[k];
        bk = k;
      }
    if (best_score < 2) fail(RV_ERR_NO_CONSENSUS, "best hypothesis explains fewer than two constraints");
    double best_axis[3] = {axes[3 * bk], axes[3 * bk + 1], axes[3 * bk + 2]};
    double best_angle = angles[bk];
    // local refit (baselines.cpp:80-94): classify, refine_axis on the consensus set, reclassify
    // (on the device-resident preprocess output)
    auto classify = [&](const double* axis) {
      const Cls cl = classify_dev(c, cs, axis, epsilon, 0, nullptr, 0);
      std::vector<int32_t> v((size_t)cl.count);
      int32_t* idx = compact_dev(c, cs, cl);
      if (cl.count) ck(cudaMemcpyAsync(v.data(), idx, 4 * cl.count, cudaMemcpyDeviceToHost, c->st), "D2H");
      sync(c);
      return std::make_pair(v, cl);
    };
    auto [inl, cl] = classify(best_axis);
    if (inl.size() >= 2) {
      double refit[3];
      if (axis_from_scatter(cl.scatter, refit)) {  // RankDeficient: keep the hypothesis axis
        std::memcpy(best_axis, refit, sizeof refit);
        inl = classify(best_axis).first;
      }
    }
    Estimate est;
    est.inliers.reserve(inl.size());
    for (int32_t i : inl) est.inliers.push_back(kept[(size_t)i]);
    try {  // vote_angles + peak_angle(refine) over the inliers; NoVotes keeps the sample angle
      int32_t* didx = c->cons_idx.get<int32_t>(std::max<size_t>(est.inliers.size(), 1));
      if (!est.inliers.empty())
        ck(cudaMemcpyAsync(didx, est.inliers.data(), 4 * est.inliers.size(), cudaMemcpyHostToDevice, c->st), "H2D");
      rv_config acfg;
      rv_config_default(&acfg);
      acfg.angle_bins = 1024;  // baselines.cpp:99
      acfg.tau_deg = kTauDeg;
      acfg.refine = 1;
      best_angle = angle_dev(c, best_axis, dcorr, didx, (int64_t)est.inliers.size(), acfg);
    } catch (const RvError& e) {
      if (e.st != RV_ERR_NO_VOTES) throw;
    }
    std::memcpy(est.axis, best_axis, sizeof est.axis);
    est.angle = best_angle;
    rodrigues3(est.axis, est.angle, est.R);
    est.votes = (uint32_t)best_score;
    to_c(est, out, seconds_since(c));
    c->results.push_back(std::move(est.inliers));
  });
}

rv_status rv_vote_shard(rv_context* c, const double* d_corrs, int64_t n, const rv_config* cfg, uint32_t* d_grid,
                        int64_t* n_kept) {
  if (!c || !cfg || !d_grid || !n_kept || (n > 0 && !d_corrs)) return RV_ERR_INVALID_ARGUMENT;
  return guarded(c, [&] {
    cudaSetDevice(c->device);
    const size_t cells = (size_t)cfg->grid * cfg->grid;
    *n_kept = 0;
    if (n <= 0) {
      ck(cudaMemsetAsync(d_grid, 0, sizeof(uint32_t) * cells, c->st), "memset");
      sync(c);
      return;
    }
    if (banded_plan(c, *cfg)) {  // in-order preprocess + band-tiled vote, graph-replayed
      unsigned long long* hk = reinterpret_cast<unsigned long long*>(c->pinned);
      auto enqueue = [&] {
        PrepBuffers b = inorder_buffers(c, d_corrs, n);
        set_vote_zeroing(c, cfg->grid, &b);
        launch_preprocess_inorder(b, n, 0, n, cfg->tau_z, cfg->normalize_inputs, c->st);
        count_launch(c);
        const uint32_t* g = vote(c, b.zx, b.zy, b.zz, n, cfg->grid, cfg->extent, cfg->theta_samples, false, true);
        ck(cudaMemcpyAsync(d_grid, g, sizeof(uint32_t) * cells, cudaMemcpyDeviceToDevice, c->st), "D2D grid");
        ck(cudaMemcpyAsync(hk, b.kept_total, sizeof(unsigned long long), cudaMemcpyDeviceToHost, c->st), "kept");
      };
      rv_context::SolveGraph* gr =
          graphs_enabled() && !c->timing ? graph_slot(c, d_corrs, n, *cfg, false, d_grid, 2) : nullptr;
      if (gr && !gr->exec && gr->seen > 0 && gr->gen == g_buf_gen.load()) capture_single(c, gr, enqueue);
      if (gr && gr->exec && gr->gen == g_buf_gen.load()) {
        ck(cudaGraphLaunch(gr->exec, c->st), "shard graph launch");
        add_counts(c->times, gr->delta);
      } else {
        const rv_stage_times t0 = c->times;
        enqueue();
        if (gr) {
          if (gr->exec) {
            cudaGraphExecDestroy(gr->exec);
            gr->exec = nullptr;
          }
          gr->delta = count_delta(c->times, t0);
          gr->gen = g_buf_gen.load();
          gr->seen += 1;
        }
      }
      sync(c);
      *n_kept = (int64_t)*hk;  // (an all-degenerate shard votes nothing: the grid stays zero)
      c->shard_cs = inorder_result(inorder_buffers(c, d_corrs, n), n).cs;
      c->shard_corrs = d_corrs;
      c->shard_cls[0].count = c->shard_cls[1].count = -1;
      return;
    }
    const PreResult pre = preprocess_dev(c, d_corrs, n, cfg->tau_z, cfg->normalize_inputs);
    *n_kept = pre.cs.n;
    c->shard_cs = pre.cs;
    c->shard_corrs = d_corrs;
    c->shard_cls[0].count = c->shard_cls[1].count = -1;
    if (pre.cs.n == 0) {  // an all-degenerate shard votes nothing
      ck(cudaMemsetAsync(d_grid, 0, sizeof(uint32_t) * cells, c->st), "memset");
      sync(c);
      return;
    }
    const auto gp = vote_and_peak(c, pre.cs.zx, pre.cs.zy, pre.cs.zz, pre.cs.n, *cfg, 1, true);
    ck(cudaMemcpyAsync(d_grid, gp.first, sizeof(uint32_t) * cells, cudaMemcpyDeviceToDevice, c->st), "D2D grid");
    sync(c);
  });
}

// The finish of a sharded solve (distributed.py): in-order preprocess of all correspondences,
// the supplied (all-reduced) grid copied in, then the chained single-solve finish -- captured and
// replayed like the other single solves when (input, grid, n, config) repeat.
Estimate estimate_prevoted_dev(rv_context* c, const double* d_corrs, int64_t n, const rv_config& cfg,
                               const uint32_t* d_grid) {
  const size_t cells = (size_t)cfg.grid * cfg.grid;
  auto enqueue = [&]() -> PreResult {
    PrepBuffers b = inorder_buffers(c, d_corrs, n);  // (no clearing side job: the grid is given)
    launch_preprocess_inorder(b, n, 0, n, cfg.tau_z, cfg.normalize_inputs, c->st);
    count_launch(c);
    uint32_t* g = c->grid.get<uint32_t>(cells);
    ck(cudaMemcpyAsync(g, d_grid, sizeof(uint32_t) * cells, cudaMemcpyDeviceToDevice, c->st), "D2D grid");
    PreResult pre = inorder_result(b, n);
    enqueue_single(c, pre, d_corrs, cfg, g, false);
    return pre;
  };
  rv_context::SolveGraph* g =
      graphs_enabled() && !c->timing ? graph_slot(c, d_corrs, n, cfg, false, d_grid, 1) : nullptr;
  if (g && !g->exec && g->seen > 0 && g->gen == g_buf_gen.load()) capture_single(c, g, [&] { enqueue(); });
  PreResult pre;
  if (g && g->exec && g->gen == g_buf_gen.load()) {
    ck(cudaGraphLaunch(g->exec, c->st), "solve graph launch");
    add_counts(c->times, g->delta);
    pre.cs.zx = c->zx.get<double>(n);
    pre.cs.zy = c->zy.get<double>(n);
    pre.cs.zz = c->zz.get<double>(n);
    pre.cs.n = n;
    pre.vote_zeroed = true;
    pre.inorder = true;
  } else {
    const rv_stage_times t0 = c->times;
    pre = enqueue();
    if (g) {
      if (g->exec) {
        cudaGraphExecDestroy(g->exec);
        g->exec = nullptr;
      }
      g->delta = count_delta(c->times, t0);
      g->gen = g_buf_gen.load();
      g->seen += 1;
    }
  }
  sync(c);
  bool identity = false;
  Estimate est = complete_single(c, pre, d_corrs, cfg, c->grid.get<uint32_t>(cells), true, &identity);
  return identity ? identity_from_inorder(c, d_corrs, n, cfg) : est;
}

rv_status rv_estimate_single_prevoted(rv_context* c, const double* d_corrs, int64_t n, const rv_config* cfg,
                                      const uint32_t* d_grid, rv_estimate* out) {
  if (!c || !cfg || !out || !d_grid || (n > 0 && !d_corrs)) return RV_ERR_INVALID_ARGUMENT;
  return guarded(c, [&] {
    cudaSetDevice(c->device);
    clear_results(c);
    if (n <= 0) fail(RV_ERR_EMPTY_INPUT, "no correspondences");
    if (cfg->angle_bins >= 8 && banded_plan(c, *cfg)) {  // in-order chain, graph-replayed
      Estimate e = estimate_prevoted_dev(c, d_corrs, n, *cfg, d_grid);
      to_c(e, out, seconds_since(c));
      c->results.push_back(std::move(e.inliers));
      return;
    }
    const PreResult pre = preprocess_dev(c, d_corrs, n, cfg->tau_z, cfg->normalize_inputs);
    Estimate e;
    if (pre.cs.n == 0) {
      std::vector<int32_t> all(n);
      for (int64_t i = 0; i < n; ++i) all[i] = (int32_t)i;
      e = identity_estimate(std::move(all));
    } else if (pre.n_dropped * 10 >= n * 9) {
      e = identity_estimate(dropped_list(c, pre.n_dropped));
    } else {
      // the supplied grid is copied into the context grid (the guard may re-vote into it)
      uint32_t* g = c->grid.get<uint32_t>((size_t)cfg->grid * cfg->grid);
      ck(cudaMemcpyAsync(g, d_grid, sizeof(uint32_t) * (size_t)cfg->grid * cfg->grid, cudaMemcpyDeviceToDevice,
                         c->st),
         "D2D grid");
      e = finish_single(c, pre, d_corrs, *cfg, g);
    }
    to_c(e, out, seconds_since(c));
    c->results.push_back(std::move(e.inliers));
  });
}


// ---- sharded finish steps: each rank / device runs these on its own shard; the
// caller sums the small partials in rank order (distributed.py over torch.distributed, or
// rv_multi_estimate_single over NCCL in one process) and makes the reference's decisions.
rv_status rv_peak_start_axis(rv_context* c, const uint32_t* d_grid, const rv_config* cfg, double axis[3],
                             uint32_t* votes, uint64_t* total) {
  if (!c || !d_grid || !cfg || !axis || !votes || !total) return RV_ERR_INVALID_ARGUMENT;
  return guarded(c, [&] {
    cudaSetDevice(c->device);
    unsigned long long tot = 0;
    // find_peaks(acc, 1, radius, 1) (estimator.cpp:346) + estimate_from_peak's start axis (:97)
    const std::vector<Peak> pk = find_peaks_dev(c, d_grid, cfg->grid, cfg->extent, 1, cfg->suppression_radius, 1, &tot);
    double A, B, b[3];
    interpolate_peak_dev(c, d_grid, cfg->grid, cfg->extent, pk[0], &A, &B);
    backproject(A, B, b);
    canonicalize3(b, axis);
    *votes = pk[0].votes;
    *total = tot;
  });
}

rv_status rv_shard_classify(rv_context* c, const double axis[3], double epsilon, int32_t slot, int32_t compare_prev,
                            int64_t* count, double scatter[6], int32_t* differs) {
  if (!c || !axis || !count || !scatter || !differs || slot < 0 || slot > 1) return RV_ERR_INVALID_ARGUMENT;
  return guarded(c, [&] {
    cudaSetDevice(c->device);
    if (!c->shard_corrs) fail(RV_ERR_INVALID_ARGUMENT, "no shard voted on this context");
    const auto& other = c->shard_cls[1 - slot];
    const uint32_t* prev = compare_prev && other.count >= 0 ? other.flags : nullptr;
    const Cls r = classify_dev(c, c->shard_cs, axis, epsilon, slot, prev, 0);
    c->shard_cls[slot].flags = r.flags;
    c->shard_cls[slot].offsets = r.offsets;
    c->shard_cls[slot].count = r.count;
    *count = r.count;
    std::memcpy(scatter, r.scatter, sizeof(double) * 6);
    *differs = r.differs ? 1 : 0;
  });
}

rv_status rv_shard_refine(rv_context* c, const double axis0[3], const rv_config* cfg, int32_t n_dev, int32_t rank,
                          double* const* peer_lines, uint64_t epoch, double axis[3], int64_t* count,
                          int64_t* local_count, double scatter[6], int32_t* refits) {
  if (!c || !axis0 || !cfg || !axis || !count || !local_count || !scatter || n_dev < 1 || n_dev > kCoopMaxDev ||
      rank < 0 || rank >= n_dev || (n_dev > 1 && !peer_lines))
    return RV_ERR_INVALID_ARGUMENT;
  return guarded(c, [&] {
    cudaSetDevice(c->device);
    if (!c->shard_corrs) fail(RV_ERR_INVALID_ARGUMENT, "no shard voted on this context");
    CoopExchange x;
    x.n_dev = n_dev;
    x.rank = rank;
    for (int q = 0; q < n_dev && n_dev > 1; ++q) x.lines[q] = peer_lines[q];
    x.epoch = epoch;
    uint32_t* flags = nullptr;
    int32_t* offsets = nullptr;
    CoopState* dst = coop_refine_launch(c, c->shard_cs, axis0, nullptr, 0, 0.0, *cfg, &flags, &offsets, nullptr,
                                        nullptr, &x);
    CoopState* h = reinterpret_cast<CoopState*>(c->pinned);
    ck(cudaMemcpyAsync(h, dst, sizeof(CoopState), cudaMemcpyDeviceToHost, c->st), "coop state D2H");
    sync(c);
    if (h->exchange_timeout) fail(RV_ERR_CUDA, "cross-device refine: a peer device never published its partials");
    std::memcpy(axis, h->axis, sizeof(double) * 3);
    std::memcpy(scatter, h->scatter, sizeof(double) * 6);
    *count = h->count;
    *local_count = h->local_count;
    if (refits) *refits = h->refits;
    // the final set of this shard, for rv_shard_inliers / rv_shard_angle_hist (slot 0)
    c->shard_cls[0].flags = flags;
    c->shard_cls[0].offsets = offsets;
    c->shard_cls[0].count = h->local_count;
    c->shard_cls[1].count = -1;
  });
}

rv_status rv_shard_lines_export(rv_context* c, void** lines, uint8_t handle[64]) {
  if (!c || !lines || !handle) return RV_ERR_INVALID_ARGUMENT;
  return guarded(c, [&] {
    cudaSetDevice(c->device);
    if (!c->xlines_own) {  // allocated once (a fixed address for the peers), zeroed
      ck(cudaMalloc(&c->xlines_own, kCoopXLineBytes), "line buffer");
      ck(cudaMemset(c->xlines_own, 0, kCoopXLineBytes), "line buffer");
    }
    cudaIpcMemHandle_t h;
    ck(cudaIpcGetMemHandle(&h, c->xlines_own), "cudaIpcGetMemHandle");
    static_assert(sizeof(h) == 64, "IPC handle size");
    std::memcpy(handle, &h, 64);
    *lines = c->xlines_own;
  });
}

rv_status rv_shard_lines_open(rv_context* c, const uint8_t handle[64], void** lines) {
  if (!c || !handle || !lines) return RV_ERR_INVALID_ARGUMENT;
  return guarded(c, [&] {
    cudaSetDevice(c->device);
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, 64);
    void* q = nullptr;
    ck(cudaIpcOpenMemHandle(&q, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
    c->xlines_peers.push_back(q);
    *lines = q;
  });
}

rv_status rv_shard_inliers(rv_context* c, int32_t slot, int64_t offset, int32_t* dst, int64_t capacity,
                           int64_t* count) {
  if (!c || !count || slot < 0 || slot > 1 || (capacity > 0 && !dst)) return RV_ERR_INVALID_ARGUMENT;
  return guarded(c, [&] {
    cudaSetDevice(c->device);
    const auto& sc = c->shard_cls[slot];
    if (sc.count < 0) fail(RV_ERR_INVALID_ARGUMENT, "slot not classified");
    Cls cl{};
    cl.flags = sc.flags;
    cl.offsets = sc.offsets;
    cl.count = sc.count;
    c->shard_idx = compact_dev(c, c->shard_cs, cl);  // ascending shard-local input indices
    c->shard_m = sc.count;
    *count = sc.count;
    const int64_t m = std::min(capacity, sc.count);
    if (m > 0) {
      ck(cudaMemcpyAsync(dst, c->shard_idx, sizeof(int32_t) * (size_t)m, cudaMemcpyDeviceToHost, c->st), "inliers");
      sync(c);
      for (int64_t k = 0; k < m; ++k) dst[k] = (int32_t)(dst[k] + offset);
    }
  });
}

rv_status rv_shard_angle_hist(rv_context* c, const double axis[3], const rv_config* cfg, uint32_t* bins,
                              uint64_t* contributing) {
  if (!c || !axis || !cfg || !bins || !contributing) return RV_ERR_INVALID_ARGUMENT;
  return guarded(c, [&] {
    cudaSetDevice(c->device);
    if (cfg->angle_bins < 8) fail(RV_ERR_INVALID_CONFIG, "angle histogram needs bin_count >= 8");
    StageScope sc(c, kAngles);
    uint32_t* db = c->bins.get<uint32_t>(cfg->angle_bins);
    double* raw = c->raw.get<double>((size_t)std::max<int64_t>(c->shard_m, 1));
    unsigned long long* cnt = c->angle_counts.get<unsigned long long>(2);
    ck(cudaMemsetAsync(db, 0, sizeof(uint32_t) * cfg->angle_bins, c->st), "memset bins");
    ck(cudaMemsetAsync(cnt, 0, 16, c->st), "memset counts");
    if (c->shard_m > 0) {  // vote_angles (angles.cpp:46-68) over this shard's inliers
      launch_vote_angles_k(axis, c->shard_corrs, c->shard_idx, c->shard_m, cfg->angle_bins, cfg->tau_deg, db, raw, cnt,
                           c->st);
      count_launch(c);
    }
    ck(cudaMemcpyAsync(bins, db, sizeof(uint32_t) * cfg->angle_bins, cudaMemcpyDeviceToHost, c->st), "bins D2H");
    unsigned long long* h = reinterpret_cast<unsigned long long*>(c->pinned);
    ck(cudaMemcpyAsync(h, cnt, 16, cudaMemcpyDeviceToHost, c->st), "angle counts D2H");
    sync(c);
    *contributing = h[0];
  });
}

rv_status rv_shard_angle_sums(rv_context* c, const uint32_t* bins_total, const rv_config* cfg, double sums[2]) {
  if (!c || !bins_total || !cfg || !sums) return RV_ERR_INVALID_ARGUMENT;
  return guarded(c, [&] {
    cudaSetDevice(c->device);
    sums[0] = sums[1] = 0.0;
    if (c->shard_m <= 0) return;
    StageScope sc(c, kAngles);
    // peak_angle (angles.cpp:70-90): the window around the GLOBAL peak bin, this shard's raw angles
    uint32_t* db = c->bins.get<uint32_t>(cfg->angle_bins);
    ck(cudaMemcpyAsync(db, bins_total, sizeof(uint32_t) * cfg->angle_bins, cudaMemcpyHostToDevice, c->st), "bins H2D");
    double* res = c->angle_result.get<double>(4);
    launch_peak_angle_k(db, cfg->angle_bins, c->raw.get<double>((size_t)c->shard_m), c->shard_m,
                        c->angle_sums.get<double>(2 * 296), res, c->done_ptr(), c->st);
    count_launch(c);
    double* h = pin_d(c);
    ck(cudaMemcpyAsync(h, res, 16, cudaMemcpyDeviceToHost, c->st), "angle sums D2H");
    sync(c);
    sums[0] = h[0];
    sums[1] = h[1];
  });
}

rv_status rv_axis_from_scatter(const double scatter[6], double axis[3]) {  // refine_axis, estimator.cpp:299-309
  if (!scatter || !axis) return RV_ERR_INVALID_ARGUMENT;
  return axis_from_scatter(scatter, axis) ? RV_OK : RV_ERR_RANK_DEFICIENT;
}


// ---------------------------------------------------------------------------------------
// CSV ingest (io.cpp:66-101 read_correspondences) -- device parse, host reference logic for
// the header decision, the rare fallback fields and the exact error messages.

// parse_double (io.cpp:16-29): trim " \t\r", the whole rest must be a from_chars float literal.
bool ref_parse_double(std::string_view f, double* v, std::string* err) {
  const auto b = f.find_first_not_of(" \t\r");
  if (b == std::string_view::npos) {
    if (err) *err = "empty field";
    return false;
  }
  const auto e = f.find_last_not_of(" \t\r");
  f = f.substr(b, e - b + 1);
  double x = 0.0;
  const auto [ptr, ec] = std::from_chars(f.data(), f.data() + f.size(), x);
  if (ec != std::errc{} || ptr != f.data() + f.size()) {
    if (err) *err = "not a number: '" + std::string(f) + "'";
    return false;
  }
  *v = x;
  return true;
}

// The reference's handling of one physical line (io.cpp:71-97): the first error message, or
// "" when the line is blank, a header (line 1) or a valid row.
std::string ref_line_error(std::string_view line, int line_number) {
  if (!line.empty() && line.back() == '\r') line.remove_suffix(1);
  if (line.find_first_not_of(" \t") == std::string_view::npos) return "";
  std::vector<std::string_view> fields;
  for (size_t pos = 0;;) {
    const size_t nx = line.find(',', pos);
    if (nx == std::string_view::npos) {
      fields.push_back(line.substr(pos));
      break;
    }
    fields.push_back(line.substr(pos, nx - pos));
    pos = nx + 1;
  }
  double v;
  if (line_number == 1 && !ref_parse_double(fields[0], &v, nullptr)) return "";  // header
  if (fields.size() != 6) return "expected 6 fields, got " + std::to_string(fields.size());
  // io.cpp:89-92 parses each Vec3's three fields as constructor arguments; GCC evaluates them
  // right to left, so the first reported bad field is the first failing of 2,1,0 then 5,4,3
  std::string err;
  for (const int k : {2, 1, 0, 5, 4, 3})
    if (!ref_parse_double(fields[(size_t)k], &v, &err)) return err;
  return "";
}

std::string_view nth_line(const char* text, int64_t nbytes, int64_t line_number) {
  const char* p = text;
  const char* end = text + nbytes;
  for (int64_t k = 1; k < line_number && p < end; ++k) {
    const void* nl = std::memchr(p, '\n', (size_t)(end - p));
    p = nl ? static_cast<const char*>(nl) + 1 : end;
  }
  const void* nl = std::memchr(p, '\n', (size_t)(end - p));
  return std::string_view(p, (size_t)((nl ? static_cast<const char*>(nl) : end) - p));
}

// uploaded: the text is already in c->csv_text (the file path streams it there while reading).
const double* parse_csv_dev(rv_context* c, const char* text, int64_t nbytes, const std::string& name, int64_t* n_rows,
                            int64_t* err_line, bool uploaded = false) {
  *n_rows = 0;
  *err_line = 0;
  if (nbytes <= 0) fail(RV_ERR_EMPTY_FILE, "no data in " + name);
  const bool add_nl = text[nbytes - 1] != '\n';
  const int64_t total = nbytes + (add_nl ? 1 : 0);
  // int32 delimiter / line / row counts and u32 byte positions: texts below 2 GB
  if (total >= ((int64_t)1 << 31)) fail(RV_ERR_INVALID_ARGUMENT, "CSV text of 2 GB or more");
  CsvBuffers b;
  uint8_t* dtext = c->csv_text.get<uint8_t>((size_t)total + 16);
  b.text = dtext;
  b.nbytes = total;
  if (!uploaded) ck(cudaMemcpyAsync(dtext, text, (size_t)nbytes, cudaMemcpyHostToDevice, c->st), "CSV H2D");
  static const char kNl = '\n';
  if (add_nl) ck(cudaMemcpyAsync(dtext + nbytes, &kNl, 1, cudaMemcpyHostToDevice, c->st), "CSV newline");
  {  // header decision on the host (io.cpp:76-84): line 1, non-blank, first field not a number
    std::string_view l1 = nth_line(text, nbytes, 1);
    if (!l1.empty() && l1.back() == '\r') l1.remove_suffix(1);
    double v;
    b.skip_first = l1.find_first_not_of(" \t") != std::string_view::npos &&
                   !ref_parse_double(l1.substr(0, l1.find(',')), &v, nullptr);
  }
  const int nchunks = csv_chunks(total);
  b.chunk = c->csv_chunk.get<int2>((size_t)nchunks);
  int32_t* misc = c->csv_misc.get<int32_t>(8);  // [0,1] totals, [2] err_line, [3] nrows, [4] fb_count
  b.totals = reinterpret_cast<int2*>(misc);
  StageScope sc(c, kPrep);
  ck(launch_csv_parse(b, c->st, 0), "CSV census");
  count_launch(c, 2);
  int32_t* h = reinterpret_cast<int32_t*>(c->pinned);
  ck(cudaMemcpyAsync(h, misc, 2 * sizeof(int32_t), cudaMemcpyDeviceToHost, c->st), "CSV totals");
  sync(c);
  b.nfields = h[0];
  b.nlines = h[1];
  const int nl = b.nlines;
  b.dpos = c->csv_dpos.get<uint32_t>((size_t)b.nfields);
  b.dline = c->csv_dline.get<int32_t>((size_t)b.nfields);
  b.nl_delim = c->csv_nl.get<int32_t>((size_t)nl);
  b.status = c->csv_status.get<int8_t>((size_t)nl);
  b.row = c->csv_row.get<int32_t>((size_t)nl);
  b.block = c->csv_block.get<int32_t>((size_t)(nl + 1023) / 1024 + 1);
  b.nrows = misc + 3;
  b.out = c->csv_out.get<double>((size_t)nl * 6);
  b.cap_rows = nl;
  b.err_line = reinterpret_cast<unsigned int*>(misc + 2);
  b.fb_cap = 1 << 16;
  b.fb = c->csv_fb.get<CsvFallback>((size_t)b.fb_cap);
  b.fb_count = misc + 4;
  ck(cudaMemsetAsync(misc + 2, 0xFF, sizeof(int32_t), c->st), "CSV err_line");
  ck(cudaMemsetAsync(misc + 4, 0, sizeof(int32_t), c->st), "CSV fb_count");
  ck(launch_csv_parse(b, c->st, 1), "CSV parse");
  count_launch(c, 6);
  ck(cudaMemcpyAsync(h, misc, 5 * sizeof(int32_t), cudaMemcpyDeviceToHost, c->st), "CSV summary");
  sync(c);
  uint32_t errl = (uint32_t)h[2];
  const int64_t nrows = h[3];
  const int64_t nfb = h[4];
  c->times.csv_host_fields += nfb;
  if (nfb > 0) {  // the rare fields outside the device's exact fast path: the host's from_chars
    std::vector<int64_t> idx;
    std::vector<double> val;
    if (nfb <= b.fb_cap) {
      std::vector<CsvFallback> fb((size_t)nfb);
      ck(cudaMemcpyAsync(fb.data(), b.fb, sizeof(CsvFallback) * (size_t)nfb, cudaMemcpyDeviceToHost, c->st),
         "CSV fallback D2H");
      sync(c);
      for (const auto& f : fb) {
        double v;
        if (ref_parse_double(std::string_view(text + f.start, (size_t)(f.end - f.start)), &v, nullptr)) {
          idx.push_back(f.row * 6 + f.col);
          val.push_back(v);
        } else {
          errl = std::min<uint32_t>(errl, (uint32_t)(f.line + 1));
        }
      }
    } else {  // too many to queue: the host parses every row the device marked as data
      std::vector<int8_t> st((size_t)nl);
      std::vector<int32_t> rw((size_t)nl);
      ck(cudaMemcpyAsync(st.data(), b.status, (size_t)nl, cudaMemcpyDeviceToHost, c->st), "CSV status");
      ck(cudaMemcpyAsync(rw.data(), b.row, sizeof(int32_t) * (size_t)nl, cudaMemcpyDeviceToHost, c->st), "CSV rows");
      sync(c);
      const char* p = text;
      for (int64_t l = 0; l < nl; ++l) {
        const void* q = std::memchr(p, '\n', (size_t)(text + nbytes - p));
        const char* e = q ? static_cast<const char*>(q) : text + nbytes;
        if (st[(size_t)l] == 1) {
          std::string_view line(p, (size_t)(e - p));
          if (!line.empty() && line.back() == '\r') line.remove_suffix(1);
          size_t pos = 0;
          for (int col = 0; col < 6; ++col) {
            const size_t nx = col < 5 ? line.find(',', pos) : line.size();
            double v;
            if (ref_parse_double(line.substr(pos, nx - pos), &v, nullptr)) {
              idx.push_back((int64_t)rw[(size_t)l] * 6 + col);
              val.push_back(v);
            } else {
              errl = std::min<uint32_t>(errl, (uint32_t)(l + 1));
            }
            pos = nx + 1;
          }
        }
        p = e + 1;
      }
    }
    if (!idx.empty()) {
      int64_t* di = c->csv_fix_idx.get<int64_t>(idx.size());
      double* dv = c->csv_fix_val.get<double>(val.size());
      ck(cudaMemcpyAsync(di, idx.data(), sizeof(int64_t) * idx.size(), cudaMemcpyHostToDevice, c->st), "CSV fix idx");
      ck(cudaMemcpyAsync(dv, val.data(), sizeof(double) * val.size(), cudaMemcpyHostToDevice, c->st), "CSV fix val");
      launch_csv_scatter(di, dv, (int)idx.size(), b.out, c->st);
      count_launch(c);
      sync(c);  // the host vectors go out of scope
    }
  }
  if (errl != 0xFFFFFFFFu) {
    *err_line = errl;
    std::string msg = ref_line_error(nth_line(text, nbytes, errl), (int)errl);
    if (msg.empty()) msg = "parse error";
    fail(RV_ERR_PARSE, msg);
  }
  if (nrows == 0) fail(RV_ERR_EMPTY_FILE, (b.skip_first ? "no correspondence rows in " : "no data in ") + name);
  *n_rows = nrows;
  return b.out;
}

rv_status rv_device_to_host(rv_context* c, void* dst, const void* d_src, int64_t bytes) {
  if (!c || bytes < 0 || (bytes > 0 && (!dst || !d_src))) return RV_ERR_INVALID_ARGUMENT;
  return guarded(c, [&] {
    cudaSetDevice(c->device);
    if (bytes > 0) ck(cudaMemcpyAsync(dst, d_src, (size_t)bytes, cudaMemcpyDeviceToHost, c->st), "D2H");
    sync(c);
  });
}

rv_status rv_parse_correspondences_csv(rv_context* c, const char* text, int64_t nbytes, const double** d_rows,
                                       int64_t* n_rows, int64_t* error_line) {
  if (!c || !d_rows || !n_rows || !error_line || (nbytes > 0 && !text) || nbytes < 0) return RV_ERR_INVALID_ARGUMENT;
  *d_rows = nullptr;
  return guarded(c, [&] {
    cudaSetDevice(c->device);
    *d_rows = parse_csv_dev(c, text, nbytes, "<memory>", n_rows, error_line);
  });
}

rv_status rv_read_correspondences_csv(rv_context* c, const char* path, const double** d_rows, int64_t* n_rows,
                                      int64_t* error_line) {
  if (!c || !path || !d_rows || !n_rows || !error_line) return RV_ERR_INVALID_ARGUMENT;
  *d_rows = nullptr;
  *n_rows = 0;
  *error_line = 0;
  return guarded(c, [&] {
    cudaSetDevice(c->device);
    FILE* f = std::fopen(path, "rb");
    if (!f) fail(RV_ERR_IO, std::string("cannot open for reading: ") + path);
    std::fseek(f, 0, SEEK_END);
    const long sz = std::ftell(f);
    std::fseek(f, 0, SEEK_SET);
    if (sz < 0) {
      std::fclose(f);
      fail(RV_ERR_IO, std::string("cannot read: ") + path);
    }
    if ((size_t)sz + 1 > c->csv_pinned_cap) {  // pinned staging: the H2D runs at full PCIe rate
      if (c->csv_pinned) {
        sync(c);
        cudaFreeHost(c->csv_pinned);
        c->csv_pinned = nullptr;
        c->csv_pinned_cap = 0;
      }
      void* p = nullptr;
      const size_t cap = (size_t)sz + 1 + (size_t)sz / 4;
      if (cudaHostAlloc(&p, cap, cudaHostAllocDefault) != cudaSuccess) {
        cudaGetLastError();
        std::fclose(f);
        fail(RV_ERR_OUT_OF_MEMORY, "pinned CSV staging");
      }
      c->csv_pinned = static_cast<char*>(p);
      c->csv_pinned_cap = cap;
    }
    // large files: parallel positional reads into the pinned buffer (a single reader is bound by
    // one core's page-cache copy rate, ~10 GB/s)
    const int nthr = sz >= ((long)32 << 20) ? (int)std::min<unsigned>(8u, std::max(1u, std::thread::hardware_concurrency())) : 1;
    bool ok = true;
    if (nthr <= 1) {
      ok = (sz > 0 ? std::fread(c->csv_pinned, 1, (size_t)sz, f) : 0) == (size_t)sz;
    } else {
      // each part is copied to the device as soon as its read finishes (in part order): the H2D
      // of the early parts overlaps the reads of the later ones
      const int fd = fileno(f);
      uint8_t* dtext = c->csv_text.get<uint8_t>((size_t)sz + 1 + 16);
      std::vector<std::thread> th;
      std::vector<char> part_ok((size_t)nthr, 1);
      for (int t = 0; t < nthr; ++t)
        th.emplace_back([&, t] {
          const int64_t lo = (int64_t)sz * t / nthr, hi = (int64_t)sz * (t + 1) / nthr;
          for (int64_t off = lo; off < hi;) {
            const ssize_t r = pread(fd, c->csv_pinned + off, (size_t)(hi - off), (off_t)off);
            if (r <= 0) {
              part_ok[(size_t)t] = 0;
              return;
            }
            off += r;
          }
        });
      for (int t = 0; t < nthr; ++t) {
        th[(size_t)t].join();
        ok = ok && part_ok[(size_t)t];
        const int64_t lo = (int64_t)sz * t / nthr, hi = (int64_t)sz * (t + 1) / nthr;
        if (ok) ck(cudaMemcpyAsync(dtext + lo, c->csv_pinned + lo, (size_t)(hi - lo), cudaMemcpyHostToDevice, c->st),
                   "CSV H2D part");
      }
    }
    std::fclose(f);
    if (!ok) {
      sync(c);
      fail(RV_ERR_IO, std::string("cannot read: ") + path);
    }
    *d_rows = parse_csv_dev(c, c->csv_pinned, (int64_t)sz, path, n_rows, error_line, nthr > 1);
  });
}

rv_status rv_result_inliers(rv_context* c, int32_t model, int32_t* dst, int64_t capacity) {
  if (!c || model < 0 || model >= (int32_t)c->results.size()) return RV_ERR_INVALID_ARGUMENT;
  if (model == 0 && c->result0_view) {
    const int64_t m = c->result0_view_n;
    if (m > capacity || (!dst && m > 0)) return RV_ERR_INVALID_ARGUMENT;
    if (m > 0) std::memcpy(dst, c->result0_view, sizeof(int32_t) * (size_t)m);
    return RV_OK;
  }
  const auto& v = c->results[model];
  if ((int64_t)v.size() > capacity || (!dst && !v.empty())) return RV_ERR_INVALID_ARGUMENT;
  if (!v.empty()) std::memcpy(dst, v.data(), sizeof(int32_t) * v.size());
  return RV_OK;
}

rv_status rv_preprocess(rv_context* c, const double* corrs, int64_t n, double tau_z, int32_t normalize,
                        double* constraints_out, int32_t* kept_out, int32_t* dropped_out, int64_t* n_kept,
                        int64_t* n_dropped) {
  if (!c || !n_kept || !n_dropped || (n > 0 && (!corrs || !constraints_out || !kept_out || !dropped_out)))
    return RV_ERR_INVALID_ARGUMENT;
  return guarded(c, [&] {
    cudaSetDevice(c->device);
    *n_kept = 0;
    *n_dropped = 0;
    if (n == 0) return;
    const double* d = upload_corrs(c, corrs, n);
    const PreResult r = preprocess_dev(c, d, n, tau_z, normalize);
    std::vector<double> sx(r.cs.n), sy(r.cs.n), sz(r.cs.n);
    if (r.cs.n) {
      ck(cudaMemcpyAsync(sx.data(), r.cs.zx, 8 * r.cs.n, cudaMemcpyDeviceToHost, c->st), "D2H");
      ck(cudaMemcpyAsync(sy.data(), r.cs.zy, 8 * r.cs.n, cudaMemcpyDeviceToHost, c->st), "D2H");
      ck(cudaMemcpyAsync(sz.data(), r.cs.zz, 8 * r.cs.n, cudaMemcpyDeviceToHost, c->st), "D2H");
      ck(cudaMemcpyAsync(kept_out, r.cs.kept, 4 * r.cs.n, cudaMemcpyDeviceToHost, c->st), "D2H");
    }
    if (r.n_dropped)
      ck(cudaMemcpyAsync(dropped_out, c->dropped.get<int32_t>(1), 4 * r.n_dropped, cudaMemcpyDeviceToHost, c->st),
         "D2H");
    sync(c);
    for (int64_t i = 0; i < r.cs.n; ++i) {
      constraints_out[3 * i] = sx[i];
      constraints_out[3 * i + 1] = sy[i];
      constraints_out[3 * i + 2] = sz[i];
    }
    *n_kept = r.cs.n;
    *n_dropped = r.n_dropped;
    if (r.cs.n == 0) fail(RV_ERR_ALL_DEGENERATE, "every correspondence pair is degenerate (x ~ y)");
  });
}

rv_status rv_accumulate(rv_context* c, const double* z, int64_t n, int32_t grid, double extent, int32_t samples,
                        uint32_t* counts_out) {
  if (!c || (n > 0 && !z) || !counts_out) return RV_ERR_INVALID_ARGUMENT;
  return guarded(c, [&] {
    cudaSetDevice(c->device);
    if (n <= 0) fail(RV_ERR_EMPTY_INPUT, "no constraints to accumulate");
    if (grid < 1 || !(extent > 0.0)) fail(RV_ERR_INVALID_CONFIG, "accumulator needs grid >= 1, extent > 0");
    const ConstraintSet cs = upload_constraints(c, z, n);
    rv_config cfg;
    rv_config_default(&cfg);
    cfg.grid = grid;
    cfg.extent = extent;
    cfg.theta_samples = samples;
    const auto gp = vote_and_peak(c, cs.zx, cs.zy, cs.zz, n, cfg, 1, true);
    ck(cudaMemcpyAsync(counts_out, gp.first, sizeof(uint32_t) * (size_t)grid * grid, cudaMemcpyDeviceToHost, c->st),
       "D2H grid");
    sync(c);
  });
}

rv_status rv_accumulate_device(rv_context* c, const double* d_z, int64_t n, int32_t grid, double extent,
                               int32_t samples, uint32_t* d_counts) {
  if (!c || (n > 0 && !d_z) || !d_counts) return RV_ERR_INVALID_ARGUMENT;
  return guarded(c, [&] {
    cudaSetDevice(c->device);
    // d_z: n x 3 AoS on the device -> SoA copies (strided device-to-device)
    double* dx = c->zx.get<double>(n);
    double* dy = c->zy.get<double>(n);
    double* dz = c->zz.get<double>(n);
    ck(cudaMemcpy2DAsync(dx, 8, d_z, 24, 8, n, cudaMemcpyDeviceToDevice, c->st), "soa x");
    ck(cudaMemcpy2DAsync(dy, 8, d_z + 1, 24, 8, n, cudaMemcpyDeviceToDevice, c->st), "soa y");
    ck(cudaMemcpy2DAsync(dz, 8, d_z + 2, 24, 8, n, cudaMemcpyDeviceToDevice, c->st), "soa z");
    const uint32_t* g = vote(c, dx, dy, dz, n, grid, extent, samples);
    ck(cudaMemcpyAsync(d_counts, g, sizeof(uint32_t) * (size_t)grid * grid, cudaMemcpyDeviceToDevice, c->st), "D2D");
  });
}

rv_status rv_deposit_circle_votes(rv_context* c, const double z[3], uint32_t* counts, int32_t grid, double extent,
                                  int32_t samples) {
  if (!c || !z || !counts) return RV_ERR_INVALID_ARGUMENT;
  return guarded(c, [&] {
    cudaSetDevice(c->device);
    if (grid < 1 || !(extent > 0.0)) fail(RV_ERR_INVALID_CONFIG, "accumulator needs grid >= 1, extent > 0");
    ensure_tables(c, samples);
    const VotePlan p = make_plan(c, grid, extent, samples);
    uint32_t* g = c->grid.get<uint32_t>((size_t)grid * grid);
    double* dz = c->user_z.get<double>(3);
    ck(cudaMemcpyAsync(g, counts, sizeof(uint32_t) * (size_t)grid * grid, cudaMemcpyHostToDevice, c->st), "H2D");
    ck(cudaMemcpyAsync(dz, z, 24, cudaMemcpyHostToDevice, c->st), "H2D");
    launch_deposit_one(p, dz, c->table64.get<double2>(samples), g, c->st);
    count_launch(c);
    ck(cudaMemcpyAsync(counts, g, sizeof(uint32_t) * (size_t)grid * grid, cudaMemcpyDeviceToHost, c->st), "D2H");
    sync(c);
  });
}

rv_status rv_find_peaks(rv_context* c, const uint32_t* counts, int32_t grid, double extent, int32_t max_peaks,
                        int32_t radius, uint32_t min_votes, rv_peak* out, int32_t* n_out) {
  if (!c || !counts || !n_out || (max_peaks > 0 && !out)) return RV_ERR_INVALID_ARGUMENT;
  return guarded(c, [&] {
    cudaSetDevice(c->device);
    *n_out = 0;
    if (grid < 1 || !(extent > 0.0)) fail(RV_ERR_INVALID_CONFIG, "accumulator needs grid >= 1, extent > 0");
    uint32_t* g = c->grid.get<uint32_t>((size_t)grid * grid);
    ck(cudaMemcpyAsync(g, counts, sizeof(uint32_t) * (size_t)grid * grid, cudaMemcpyHostToDevice, c->st), "H2D");
    const auto ps = find_peaks_dev(c, g, grid, extent, max_peaks, radius, min_votes);
    for (size_t k = 0; k < ps.size(); ++k) out[k] = {ps[k].ix, ps[k].iy, ps[k].A, ps[k].B, ps[k].votes};
    *n_out = (int32_t)ps.size();
  });
}

rv_status rv_blurred_argmax(rv_context* c, const uint32_t* counts, int32_t grid, double extent, int32_t radius,
                            rv_peak* out) {
  if (!c || !counts || !out) return RV_ERR_INVALID_ARGUMENT;
  return guarded(c, [&] {
    cudaSetDevice(c->device);
    if (radius < 0) fail(RV_ERR_INVALID_CONFIG, "blur radius must be non-negative");
    if (grid < 1 || !(extent > 0.0)) fail(RV_ERR_INVALID_CONFIG, "accumulator needs grid >= 1, extent > 0");
    uint32_t* g = c->grid.get<uint32_t>((size_t)grid * grid);
    ck(cudaMemcpyAsync(g, counts, sizeof(uint32_t) * (size_t)grid * grid, cudaMemcpyHostToDevice, c->st), "H2D");
    const auto ps = blurred_argmax_dev(c, g, grid, extent, {radius});
    *out = {ps[0].ix, ps[0].iy, ps[0].A, ps[0].B, ps[0].votes};
  });
}

rv_status rv_classify_inliers(rv_context* c, const double axis[3], const double* z, int64_t n, double eps, int32_t* out,
                              int64_t* n_out) {
  if (!c || !axis || !n_out || (n > 0 && (!z || !out))) return RV_ERR_INVALID_ARGUMENT;
  return guarded(c, [&] {
    cudaSetDevice(c->device);
    *n_out = 0;
    if (n == 0) return;
    const ConstraintSet cs = upload_constraints(c, z, n);
    const Cls cl = classify_dev(c, cs, axis, eps, 0, nullptr, 2);
    int32_t* idx = compact_dev(c, cs, cl);
    if (cl.count) ck(cudaMemcpyAsync(out, idx, 4 * cl.count, cudaMemcpyDeviceToHost, c->st), "D2H");
    sync(c);
    *n_out = cl.count;
  });
}

rv_status rv_refine_axis(rv_context* c, const double* z, int64_t n, double axis_out[3]) {
  if (!c || !axis_out || (n > 0 && !z)) return RV_ERR_INVALID_ARGUMENT;
  return guarded(c, [&] {
    cudaSetDevice(c->device);
    if (n < 2) fail(RV_ERR_RANK_DEFICIENT, "need at least two constraints");
    const ConstraintSet cs = upload_constraints(c, z, n);
    const Cls all = classify_dev(c, cs, nullptr, 0.0, 0, nullptr, 1);
    if (!axis_from_scatter(all.scatter, axis_out)) fail(RV_ERR_RANK_DEFICIENT, "constraints span fewer than two directions");
  });
}

rv_status rv_vote_angles(rv_context* c, const double axis[3], const double* corrs, int64_t n_corrs,
                         const int32_t* indices, int64_t n_idx, int32_t bin_count, double tau, uint32_t* bins_out,
                         uint64_t* contributing, uint64_t* degenerate, double* raw_out) {
  if (!c || !axis || !bins_out || !contributing || !degenerate || (n_idx > 0 && (!indices || !corrs || !raw_out)))
    return RV_ERR_INVALID_ARGUMENT;
  return guarded(c, [&] {
    cudaSetDevice(c->device);
    if (bin_count < 8) fail(RV_ERR_INVALID_CONFIG, "angle histogram needs bin_count >= 8");
    for (int64_t k = 0; k < n_idx; ++k)
      if (indices[k] < 0 || indices[k] >= n_corrs) fail(RV_ERR_INVALID_ARGUMENT, "index out of range");
    const double* d = n_corrs > 0 ? upload_corrs(c, corrs, n_corrs) : c->corrs.get<double>(6);
    int32_t* di = c->compact_out.get<int32_t>((size_t)std::max<int64_t>(n_idx, 1));
    if (n_idx) ck(cudaMemcpyAsync(di, indices, 4 * n_idx, cudaMemcpyHostToDevice, c->st), "H2D idx");
    uint32_t* bins = c->bins.get<uint32_t>(bin_count);
    double* raw = c->raw.get<double>((size_t)std::max<int64_t>(n_idx, 1));
    unsigned long long* cnt = c->angle_counts.get<unsigned long long>(2);
    ck(cudaMemsetAsync(bins, 0, 4 * bin_count, c->st), "memset");
    ck(cudaMemsetAsync(cnt, 0, 16, c->st), "memset");
    if (n_idx) {
      launch_vote_angles_k(axis, d, di, n_idx, bin_count, tau, bins, raw, cnt, c->st);
      count_launch(c);
    }
    std::vector<double> hraw(n_idx);
    unsigned long long hc[2];
    ck(cudaMemcpyAsync(bins_out, bins, 4 * bin_count, cudaMemcpyDeviceToHost, c->st), "D2H");
    ck(cudaMemcpyAsync(hc, cnt, 16, cudaMemcpyDeviceToHost, c->st), "D2H");
    if (n_idx) ck(cudaMemcpyAsync(hraw.data(), raw, 8 * n_idx, cudaMemcpyDeviceToHost, c->st), "D2H");
    sync(c);
    int64_t m = 0;  // raw_angles keeps contributing votes only, in insertion order
    for (int64_t k = 0; k < n_idx; ++k)
      if (hraw[k] == hraw[k]) raw_out[m++] = hraw[k];
    *contributing = hc[0];
    *degenerate = hc[1];
    if (hc[0] == 0) fail(RV_ERR_NO_VOTES, "no correspondence produced an angle vote");
  });
}

rv_status rv_peak_angle(rv_context* c, const uint32_t* bins, int32_t bin_count, uint64_t contributing, int32_t refine,
                        const double* raw, int64_t n_raw, double* angle_out) {
  if (!c || !bins || !angle_out || bin_count < 1 || (n_raw > 0 && !raw)) return RV_ERR_INVALID_ARGUMENT;
  return guarded(c, [&] {
    cudaSetDevice(c->device);
    if (contributing == 0) fail(RV_ERR_NO_VOTES, "empty angle histogram");
    uint32_t* db = c->bins.get<uint32_t>(bin_count);
    double* dr = c->raw.get<double>((size_t)std::max<int64_t>(n_raw, 1));
    ck(cudaMemcpyAsync(db, bins, 4 * bin_count, cudaMemcpyHostToDevice, c->st), "H2D");
    if (n_raw) ck(cudaMemcpyAsync(dr, raw, 8 * n_raw, cudaMemcpyHostToDevice, c->st), "H2D");
    double* res = c->angle_result.get<double>(4);
    launch_peak_angle_k(db, bin_count, dr, n_raw, c->angle_sums.get<double>(2 * 296), res, c->done_ptr(), c->st);
    count_launch(c);
    double* h = pin_d(c);
    ck(cudaMemcpyAsync(h, res, 32, cudaMemcpyDeviceToHost, c->st), "D2H");
    sync(c);
    const double s = h[0], co = h[1], center = h[3];
    if (!refine || (s == 0.0 && co == 0.0)) {
      *angle_out = center;
      return;
    }
    double mean = std::atan2(s, co);
    if (mean <= -kPiD) mean += 2.0 * kPiD;
    *angle_out = mean;
  });
}

uint32_t rv_peak_vote_floor(const rv_config* cfg, int64_t n) {  // estimator.cpp:311-318
  const double cell = 2.0 * cfg->extent / cfg->grid;
  const double per_crossing = cfg->theta_samples * cell / (2.0 * std::numbers::pi);
  const double floor_votes = cfg->min_votes_frac * static_cast<double>(n) * per_crossing;
  return static_cast<uint32_t>(std::max(16.0, floor_votes));
}

void rv_rodrigues(const double axis[3], double angle, double r[9]) { rodrigues3(axis, angle, r); }
double rv_rotation_error(const double g[9], const double o[9]) { return rotation_error3(g, o); }
rv_status rv_project(const double p[3], double* A, double* B) {
  return project3(p, A, B) ? RV_OK : RV_ERR_POLE_PROXIMITY;
}
void rv_unproject(double A, double B, double out[3]) { unproject2(A, B, out); }
void rv_canonicalize(const double p[3], double out[3]) { canonicalize3(p, out); }
void rv_orthonormal_basis(const double z[3], double a1[3], double a2[3]) { orthonormal_basis3(z, a1, a2); }
rv_status rv_correspondence_angle(const double axis[3], const double x[3], const double y[3], double tau,
                                  double* angle_out) {  // angles.cpp:36-44 (host formula; libm atan2)
  double beta[3], gamma[3], bg[3];
  cross3(axis, x, beta);
  cross3(axis, y, gamma);
  if (norm3(beta) <= tau || norm3(gamma) <= tau) return RV_ERR_DEGENERATE_PROJECTION;
  cross3(beta, gamma, bg);
  *angle_out = std::atan2(dot3(bg, axis), dot3(beta, gamma));
  return RV_OK;
}

}  // extern "C"
