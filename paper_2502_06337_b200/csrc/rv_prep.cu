// K1a: preprocess (estimator.cpp:259-285) in one HBM pass.
//
// Reads the reference's AoS correspondence layout (48 B/pair, 3 x 16 B vector loads per
// thread), normalises x and y, forms z = (y-x)/|y-x| with the reference's exact f64 op order,
// and writes kept constraints as SoA f64 in input order (order-preserving compaction by a
// single-pass decoupled look-back scan), the kept index map and the dropped index list.
// Algorithmic bytes: 48 B read + 24 B (z) + 4 B (kept) written per kept pair = 76 B.
#include <cuda_runtime.h>

#include <cstdint>

#include "rv_exact.cuh"
#include "rv_internal.h"
#include "rv_scan.cuh"

namespace rvb {
namespace {

constexpr int kPrepThreads = 512;
constexpr int kPrepPer = 2;                             // elements per thread (r-major in the block)
constexpr int kPrepTile = kPrepThreads * kPrepPer;      // 1024 correspondences per block
constexpr int kPrepWarps = kPrepThreads / 32;
static_assert(kPrepPer * kPrepWarps == 32, "one warp scans the (round, warp) counts");

template <bool kVec, bool kInOrder>
__global__ void __launch_bounds__(kPrepThreads) preprocess_kernel(PrepBuffers b, int64_t n, int64_t elem_lo, int64_t elem_hi,
                                                                  double tau_z, int normalize) {
  __shared__ int s_bid;
  __shared__ int s_cnt[kPrepPer * kPrepWarps];  // kept per (round, warp), then its exclusive scan
  __shared__ int s_total;
  __shared__ long long s_excl;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0 && !kInOrder) s_bid = atomicAdd(b.block_counter, 1);
  {  // side job: clear the next vote's state (grid-stride over the launch's threads)
    const int64_t gstride = (int64_t)gridDim.x * kPrepThreads, g0 = (int64_t)blockIdx.x * kPrepThreads + tid;
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (b.zero_ptr[q])
        for (int64_t w = g0; w < b.zero_n[q]; w += gstride) b.zero_ptr[q][w] = 0u;
  }
  if (!kInOrder) __syncthreads();
  const int bid = kInOrder ? (int)(elem_lo / kPrepTile) + blockIdx.x : s_bid;
  const int64_t base = (int64_t)bid * kPrepTile;
  // in-order launches may carry extra blocks that only clear (small inputs): stay inside the range
  const int64_t lim = kInOrder ? elem_hi : n;
  double c[kPrepPer][6];
#pragma unroll
  for (int r = 0; r < kPrepPer; ++r) {  // all loads first (coalesced per round)
    const int64_t i = base + r * kPrepThreads + tid;
    for (int k = 0; k < 6; ++k) c[r][k] = 0.0;
    if (i < lim) {
      if (kVec) {
        const double2* p = reinterpret_cast<const double2*>(b.corrs + 6 * i);
        const double2 u = p[0], v = p[1], w = p[2];
        c[r][0] = u.x; c[r][1] = u.y; c[r][2] = v.x; c[r][3] = v.y; c[r][4] = w.x; c[r][5] = w.y;
      } else {
        const double* p = b.corrs + 6 * i;
        for (int k = 0; k < 6; ++k) c[r][k] = p[k];
      }
    }
  }
  double zo[kPrepPer][3];
  bool keep[kPrepPer], drop[kPrepPer];
  unsigned km[kPrepPer];
#pragma unroll
  for (int r = 0; r < kPrepPer; ++r) {
    const int64_t i = base + r * kPrepThreads + tid;
    const bool kept = preprocess_pair(c[r][0], c[r][1], c[r][2], c[r][3], c[r][4], c[r][5], normalize, tau_z, zo[r]);
    const bool valid = i < lim;
    drop[r] = valid && !kept;
    keep[r] = valid && kept;
    km[r] = __ballot_sync(0xFFFFFFFFu, keep[r]);
    if (lane == 0) s_cnt[r * kPrepWarps + warp] = __popc(km[r]);
  }
  if constexpr (kInOrder) {  // z at the input index, NaN marks a dropped pair; count the kept ones
#pragma unroll
    for (int r = 0; r < kPrepPer; ++r) {
      const int64_t i = base + r * kPrepThreads + tid;
      if (i < lim) {
        const double q = __longlong_as_double(0x7FF8000000000000ll);
        b.zx[i] = keep[r] ? zo[r][0] : q;
        b.zy[i] = keep[r] ? zo[r][1] : q;
        b.zz[i] = keep[r] ? zo[r][2] : q;
      }
    }
    __syncthreads();
    if (warp == 0) {
      int v = s_cnt[lane];
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
      if (lane == 0) {
        if (v) atomicAdd(b.kept_acc, (unsigned long long)v);
        __threadfence();
        if (atomicAdd(b.kept_done, 1u) == gridDim.x - 1) {  // last block of this launch
          __threadfence();
          if (b.kept_publish) *b.kept_total = atomicExch(b.kept_acc, 0ull);
          *b.kept_done = 0u;
        }
      }
    }
    return;
  }
  __syncthreads();
  if (warp == 0) {  // exclusive scan of the 32 (round, warp) counts in element order
    const int v = s_cnt[lane];
    int incl = v;
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xFFFFFFFFu, incl, o);
      if (lane >= o) incl += t;
    }
    const int total = __shfl_sync(0xFFFFFFFFu, incl, 31);
    s_cnt[lane] = incl - v;
    const long long e = lookback_exclusive(reinterpret_cast<unsigned long long*>(b.status), bid, total);
    if (lane == 0) {
      s_excl = e;
      s_total = total;
    }
  }
  __syncthreads();
  const long long excl = s_excl;
#pragma unroll
  for (int r = 0; r < kPrepPer; ++r) {
    const int64_t i = base + r * kPrepThreads + tid;
    const long long rank = excl + s_cnt[r * kPrepWarps + warp] + __popc(km[r] & ((1u << lane) - 1u));
    if (keep[r]) {
      b.zx[rank] = zo[r][0];
      b.zy[rank] = zo[r][1];
      b.zz[rank] = zo[r][2];
      b.kept[rank] = (int32_t)i;
    } else if (drop[r]) {
      b.dropped[i - rank] = (int32_t)i;
    }
  }
  const int total = s_total;
  const int64_t block_end = base + kPrepTile;
  if (tid == 0 && block_end >= n) {  // the last block publishes the totals
    b.totals[0] = (int32_t)(excl + total);
    b.totals[1] = (int32_t)(n - (excl + total));
  }
  if (tid == 0 && b.chunk_hi && block_end >= elem_hi) *b.chunk_hi = (int32_t)(excl + total);
}

constexpr int kGatherThreads = 256;

__global__ void __launch_bounds__(kGatherThreads)
    gather_residual_kernel(const double* zx, const double* zy, const double* zz, const int32_t* kept,
                           const uint8_t* removed, int64_t n, unsigned long long* status, int32_t* block_counter,
                           double* ozx, double* ozy, double* ozz, int32_t* okept, int32_t* total_out) {
  __shared__ int s_bid;
  __shared__ int s_warp[kGatherThreads / 32];
  __shared__ long long s_excl;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_bid = atomicAdd(block_counter, 1);
  __syncthreads();
  const int bid = s_bid;
  const int64_t i = (int64_t)bid * kGatherThreads + tid;
  const bool keep = i < n && !removed[i];
  const unsigned km = __ballot_sync(0xFFFFFFFFu, keep);
  if (lane == 0) s_warp[warp] = __popc(km);
  __syncthreads();
  int before = 0, total = 0;
  for (int w = 0; w < kGatherThreads / 32; ++w) {
    const int c = s_warp[w];
    if (w < warp) before += c;
    total += c;
  }
  if (warp == 0) {
    const long long e = lookback_exclusive(status, bid, total);
    if (lane == 0) s_excl = e;
  }
  __syncthreads();
  const long long rank = s_excl + before + __popc(km & ((1u << lane) - 1u));
  if (keep) {
    ozx[rank] = zx[i];
    ozy[rank] = zy[i];
    ozz[rank] = zz[i];
    okept[rank] = kept[i];
  }
  if (tid == 0 && (int64_t)(bid + 1) * kGatherThreads >= n) *total_out = (int32_t)(s_excl + total);
}

}  // namespace

int prep_blocks(int64_t n) { return (int)((n + kPrepTile - 1) / kPrepTile); }

void launch_preprocess(const PrepBuffers& b, int64_t n, double tau_z, int normalize, cudaStream_t s) {
  const int blocks = prep_blocks(n);
  const bool vec = (reinterpret_cast<uintptr_t>(b.corrs) & 15u) == 0;
  if (vec)
    preprocess_kernel<true, false><<<blocks, kPrepThreads, 0, s>>>(b, n, 0, n, tau_z, normalize);
  else
    preprocess_kernel<false, false><<<blocks, kPrepThreads, 0, s>>>(b, n, 0, n, tau_z, normalize);
}

void launch_preprocess_range(const PrepBuffers& b, int64_t n, int64_t elem_lo, int64_t elem_hi, double tau_z,
                             int normalize, cudaStream_t s) {
  const int blocks = (int)((elem_hi - elem_lo + kPrepTile - 1) / kPrepTile);
  if (blocks <= 0) return;
  const bool vec = (reinterpret_cast<uintptr_t>(b.corrs) & 15u) == 0;
  if (vec)
    preprocess_kernel<true, false><<<blocks, kPrepThreads, 0, s>>>(b, n, elem_lo, elem_hi, tau_z, normalize);
  else
    preprocess_kernel<false, false><<<blocks, kPrepThreads, 0, s>>>(b, n, elem_lo, elem_hi, tau_z, normalize);
}

void launch_preprocess_inorder(const PrepBuffers& b, int64_t n, int64_t elem_lo, int64_t elem_hi, double tau_z,
                               int normalize, cudaStream_t s) {
  int blocks = (int)((elem_hi - elem_lo + kPrepTile - 1) / kPrepTile);
  if (blocks <= 0) return;
  int64_t zmax = 0;  // the clearing side job: enough blocks for ~16 words per thread
  for (int q = 0; q < 4; ++q)
    if (b.zero_ptr[q]) zmax = zmax > b.zero_n[q] ? zmax : b.zero_n[q];
  const int zblocks = (int)((zmax + 16 * kPrepThreads - 1) / (16 * kPrepThreads));
  if (zblocks > blocks) blocks = zblocks;
  const bool vec = (reinterpret_cast<uintptr_t>(b.corrs) & 15u) == 0;
  if (vec)
    preprocess_kernel<true, true><<<blocks, kPrepThreads, 0, s>>>(b, n, elem_lo, elem_hi, tau_z, normalize);
  else
    preprocess_kernel<false, true><<<blocks, kPrepThreads, 0, s>>>(b, n, elem_lo, elem_hi, tau_z, normalize);
}

void launch_gather_residual(const double* zx, const double* zy, const double* zz, const int32_t* kept,
                            const uint8_t* removed, int64_t n, unsigned long long* status, int32_t* block_counter,
                            double* ozx, double* ozy, double* ozz, int32_t* okept, int32_t* total, cudaStream_t s) {
  const int blocks = (int)((n + kGatherThreads - 1) / kGatherThreads);
  gather_residual_kernel<<<blocks, kGatherThreads, 0, s>>>(zx, zy, zz, kept, removed, n, status, block_counter,
                                                           ozx, ozy, ozz, okept, total);
}

}  // namespace rvb
