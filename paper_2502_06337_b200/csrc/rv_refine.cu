// K4: consensus and angle kernels.
//  * classify (estimator.cpp:287-297): |ax*zx + ay*zy + az*zz| < eps, strict, exact f64
//    op order -> inlier bitmask; fused with the scatter partial sums of refine_axis
//    (estimator.cpp:299-302) over the same inliers and a "set changed" test against the
//    previous bitmask (refine_loop's next_inl == inl, estimator.cpp:64).
//  * compaction of a bitmask into ascending (optionally kept-mapped) indices.
//  * vote_angles / peak_angle sums (angles.cpp:36-90) and model_support (estimator.cpp:117-137).
// Floating-point partial sums are reduced in a fixed tree order (deterministic run to run).
#include <cuda_runtime.h>

#include <cstdint>


#include "rv_exact.cuh"
#include "rv_internal.h"

namespace rvb {
namespace {

constexpr int kClsThreads = 256;
constexpr int kClsPerThread = 4;
constexpr int kClsPerBlock = kClsThreads * kClsPerThread;  // 1024 elements = 32 flag words
constexpr double kPi = 3.14159265358979323846;

template <int K>
__device__ __forceinline__ void block_sum(double (&v)[K], double (*s)[kClsThreads / 32]) {
  // fixed-shape tree: warp xor-shuffle, then warp 0 over warp partials
#pragma unroll
  for (int k = 0; k < K; ++k)
    for (int o = 16; o > 0; o >>= 1) v[k] = __dadd_rn(v[k], __shfl_xor_sync(0xFFFFFFFFu, v[k], o));
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < K; ++k) s[k][warp] = v[k];
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      double t = lane < kClsThreads / 32 ? s[k][lane] : 0.0;
      for (int o = 16; o > 0; o >>= 1) t = __dadd_rn(t, __shfl_xor_sync(0xFFFFFFFFu, t, o));
      v[k] = t;
    }
  }
  __syncthreads();
}

struct ClsArgs {
  const double* zx;
  const double* zy;
  const double* zz;
  int64_t n;
  double ax, ay, az, eps;
  int mode;  // 0 classify, 1 all constraints (refine_axis(constraints)), 2 classify w/o scatter
  uint32_t* flags;
  const uint32_t* prev;
  int32_t* block_count;
  double* block_scatter;
  int32_t* block_diff;
  int32_t* block_offsets;  // exclusive scan of block_count (written by the last block)
  double* result;          // [0]=count [1]=differs [2..7]=scatter
  unsigned int* done;
};

__global__ void __launch_bounds__(kClsThreads) classify_kernel(ClsArgs a) {
  __shared__ double s_red[6][kClsThreads / 32];
  __shared__ int s_cnt[kClsThreads / 32], s_diff[kClsThreads / 32];
  __shared__ bool s_last;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t base = (int64_t)blockIdx.x * kClsPerBlock;
  double sc[6] = {0, 0, 0, 0, 0, 0};
  int cnt = 0, diff = 0;
#pragma unroll
  for (int r = 0; r < kClsPerThread; ++r) {
    const int64_t i = base + r * kClsThreads + tid;
    bool in = false;
    double z0 = 0, z1 = 0, z2 = 0;
    if (i < a.n) {
      z0 = a.zx[i];
      z1 = a.zy[i];
      z2 = a.zz[i];
      if (a.mode == 1) {
        in = true;
      } else {
        const double d = xa(xa(xm(a.ax, z0), xm(a.ay, z1)), xm(a.az, z2));
        in = fabs(d) < a.eps;
      }
    }
    const unsigned word = __ballot_sync(0xFFFFFFFFu, in);
    const int64_t wi = (base + r * kClsThreads + warp * 32) >> 5;
    if (lane == 0 && a.mode != 1 && (base + r * kClsThreads + warp * 32) < a.n) {
      a.flags[wi] = word;
      if (a.prev && a.prev[wi] != word) diff = 1;
    }
    if (in) {
      ++cnt;
      if (a.mode != 2) {
        sc[0] = xa(sc[0], xm(z0, z0));
        sc[1] = xa(sc[1], xm(z0, z1));
        sc[2] = xa(sc[2], xm(z0, z2));
        sc[3] = xa(sc[3], xm(z1, z1));
        sc[4] = xa(sc[4], xm(z1, z2));
        sc[5] = xa(sc[5], xm(z2, z2));
      }
    }
  }
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xFFFFFFFFu, cnt, o);
  diff = __any_sync(0xFFFFFFFFu, diff);
  if (lane == 0) {
    s_cnt[warp] = cnt;
    s_diff[warp] = diff;
  }
  if (a.mode != 2) block_sum<6>(sc, s_red);
  else __syncthreads();
  if (tid == 0) {
    int c = 0, d = 0;
    for (int w = 0; w < kClsThreads / 32; ++w) {
      c += s_cnt[w];
      d |= s_diff[w];
    }
    a.block_count[blockIdx.x] = c;
    a.block_diff[blockIdx.x] = d;
    if (a.mode != 2)
      for (int k = 0; k < 6; ++k) a.block_scatter[(size_t)blockIdx.x * 6 + k] = sc[k];
    __threadfence();
    s_last = atomicAdd(a.done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last) return;
  // last block: fixed-order reduction over blocks + exclusive scan of block counts
  const int nb = gridDim.x;
  volatile int32_t* bc = a.block_count;
  volatile int32_t* bd = a.block_diff;
  volatile double* bs = a.block_scatter;
  double v[6] = {0, 0, 0, 0, 0, 0};
  long long tc = 0;
  int td = 0;
  // each thread owns a contiguous run of blocks (sequential), then a fixed tree across threads
  const int per = (nb + kClsThreads - 1) / kClsThreads;
  const int b0 = tid * per, b1 = min(nb, b0 + per);
  for (int b = b0; b < b1; ++b) {
    tc += bc[b];
    td |= bd[b];
    if (a.mode != 2)
      for (int k = 0; k < 6; ++k) v[k] = xa(v[k], bs[(size_t)b * 6 + k]);
  }
  // exclusive scan of per-thread run totals
  __shared__ long long s_run[kClsThreads];
  s_run[tid] = tc;
  __syncthreads();
  if (tid == 0) {
    long long acc = 0;
    for (int t = 0; t < kClsThreads; ++t) {
      const long long x = s_run[t];
      s_run[t] = acc;
      acc += x;
    }
  }
  __syncthreads();
  long long off = s_run[tid];
  for (int b = b0; b < b1; ++b) {
    a.block_offsets[b] = (int32_t)off;
    off += bc[b];
  }
  for (int o = 16; o > 0; o >>= 1) {
    tc += __shfl_xor_sync(0xFFFFFFFFu, tc, o);
    td |= __shfl_xor_sync(0xFFFFFFFFu, td, o);
  }
  __shared__ long long s_tc[kClsThreads / 32];
  __shared__ int s_td[kClsThreads / 32];
  if (lane == 0) {
    s_tc[warp] = tc;
    s_td[warp] = td;
  }
  if (a.mode != 2) block_sum<6>(v, s_red);
  else __syncthreads();
  if (tid == 0) {
    long long c = 0;
    int d = 0;
    for (int w = 0; w < kClsThreads / 32; ++w) {
      c += s_tc[w];
      d |= s_td[w];
    }
    a.result[0] = (double)c;
    a.result[1] = (double)d;
    for (int k = 0; k < 6; ++k) a.result[2 + k] = a.mode != 2 ? v[k] : 0.0;
    *a.done = 0u;
  }
}

// bitmask -> ascending indices (through map if given). Uses block_offsets from classify.
__global__ void __launch_bounds__(kClsThreads) compact_kernel(const uint32_t* flags, int64_t n, const int32_t* map,
                                                             const int32_t* block_offsets, int32_t* out,
                                                             int32_t* out_host) {
  __shared__ int s_pref[kClsPerBlock / 32 + 1];
  const int tid = threadIdx.x;
  const int64_t wbase = (int64_t)blockIdx.x * (kClsPerBlock / 32);
  const int64_t nwords = (n + 31) / 32;
  if (tid == 0) {
    int acc = 0;
    for (int w = 0; w < kClsPerBlock / 32; ++w) {
      s_pref[w] = acc;
      if (wbase + w < nwords) acc += __popc(flags[wbase + w]);
    }
    s_pref[kClsPerBlock / 32] = acc;
  }
  __syncthreads();
  const int lane = tid & 31, warp = tid >> 5;
  const int off = block_offsets[blockIdx.x];
  for (int w = warp; w < kClsPerBlock / 32; w += kClsThreads / 32) {
    if (wbase + w >= nwords) break;
    const uint32_t word = flags[wbase + w];
    if ((word >> lane) & 1u) {
      const int64_t i = (wbase + w) * 32 + lane;
      const int pos = off + s_pref[w] + __popc(word & ((1u << lane) - 1u));
      const int32_t v = map ? map[i] : (int32_t)i;
      out[pos] = v;
      if (out_host) out_host[pos] = v;
    }
  }
}

// correspondence_angle, angles.cpp:36-44, exact op order (atan2 is CUDA's, <= 2 ulp).
__device__ __forceinline__ bool corr_angle(double a0, double a1, double a2, const double* c, double tau,
                                           double* out) {
  const double x0 = c[0], x1 = c[1], x2 = c[2], y0 = c[3], y1 = c[4], y2 = c[5];
  const double b0 = xs(xm(a1, x2), xm(a2, x1)), b1 = xs(xm(a2, x0), xm(a0, x2)), b2 = xs(xm(a0, x1), xm(a1, x0));
  const double g0 = xs(xm(a1, y2), xm(a2, y1)), g1 = xs(xm(a2, y0), xm(a0, y2)), g2 = xs(xm(a0, y1), xm(a1, y0));
  if (__dsqrt_rn(xdot(b0, b1, b2, b0, b1, b2)) <= tau || __dsqrt_rn(xdot(g0, g1, g2, g0, g1, g2)) <= tau) return false;
  const double c0 = xs(xm(b1, g2), xm(b2, g1)), c1 = xs(xm(b2, g0), xm(b0, g2)), c2 = xs(xm(b0, g1), xm(b1, g0));
  *out = atan2(xdot(c0, c1, c2, a0, a1, a2), xdot(b0, b1, b2, g0, g1, g2));
  return true;
}

__device__ __forceinline__ int bin_of(double angle, int n) {  // angles.cpp:25-30
  const double w = xd(2.0 * kPi, (double)n);
  const int k = __double2int_rz(ceil(xd(xa(angle, kPi), w))) - 1;
  return min(max(k, 0), n - 1);
}

struct AngArgs {
  double a0, a1, a2, tau;
  const double* axis_dev;   // optional: axis on the device
  const long long* n_dev;   // optional: count on the device (n = upper bound)
  int32_t* idx_host;        // optional: mapped pinned copy of idx (coalesced zero-copy read-back)
  const double* corrs;
  const int32_t* idx;
  int64_t n;
  int bins_n;
  uint32_t* bins;
  double* raw;
  unsigned long long* counts;
  // candidate batches (blockIdx.y = candidate): per-candidate offsets; 0 for a single vote
  size_t idx_stride, raw_stride, state_stride_b;  // elements, elements, bytes (axis_dev / n_dev / counts)
};

__global__ void __launch_bounds__(256) vote_angles_kernel(AngArgs a) {
  extern __shared__ uint32_t s_bins[];
  if (blockIdx.y) {  // candidate y of a batch: its own list, histogram, angles, summary slot
    const size_t y = blockIdx.y;
    a.idx += y * a.idx_stride;
    a.raw += y * a.raw_stride;
    a.bins += y * (size_t)a.bins_n;
    if (a.axis_dev) a.axis_dev = reinterpret_cast<const double*>(reinterpret_cast<const char*>(a.axis_dev) + y * a.state_stride_b);
    if (a.n_dev) a.n_dev = reinterpret_cast<const long long*>(reinterpret_cast<const char*>(a.n_dev) + y * a.state_stride_b);
    a.counts = reinterpret_cast<unsigned long long*>(reinterpret_cast<char*>(a.counts) + y * a.state_stride_b);
  }
  const bool use_smem = a.bins_n <= 8192;
  if (use_smem)
    for (int k = threadIdx.x; k < a.bins_n; k += blockDim.x) s_bins[k] = 0;
  __syncthreads();
  unsigned long long contrib = 0, degen = 0;
  const int64_t n = a.n_dev ? min(a.n, (int64_t)*a.n_dev) : a.n;
  const double a0 = a.axis_dev ? a.axis_dev[0] : a.a0, a1 = a.axis_dev ? a.axis_dev[1] : a.a1,
               a2 = a.axis_dev ? a.axis_dev[2] : a.a2;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
    const int32_t ik = a.idx[k];
    if (a.idx_host) a.idx_host[k] = ik;
    const double* c = a.corrs + 6 * (int64_t)ik;
    double ang;
    if (corr_angle(a0, a1, a2, c, a.tau, &ang)) {
      a.raw[k] = ang;
      const int b = bin_of(ang, a.bins_n);
      if (use_smem) atomicAdd(&s_bins[b], 1u);
      else atomicAdd(&a.bins[b], 1u);
      ++contrib;
    } else {
      a.raw[k] = __longlong_as_double(0x7ff8000000000000ll);  // NaN marks a degenerate pair
      ++degen;
    }
  }
  __syncthreads();
  if (use_smem)
    for (int k = threadIdx.x; k < a.bins_n; k += blockDim.x)
      if (s_bins[k]) atomicAdd(&a.bins[k], s_bins[k]);
  for (int o = 16; o > 0; o >>= 1) {
    contrib += __shfl_xor_sync(0xFFFFFFFFu, contrib, o);
    degen += __shfl_xor_sync(0xFFFFFFFFu, degen, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (contrib) atomicAdd(&a.counts[0], contrib);
    if (degen) atomicAdd(&a.counts[1], degen);
  }
}

// peak_angle sums (angles.cpp:70-90): first max bin, then sin/cos sums of raw angles within
// 1.5 bin widths (wrapped difference) of the bin center. result: [0]=s [1]=c [2]=k [3]=center.
__global__ void __launch_bounds__(256) peak_angle_kernel(const uint32_t* bins, int bins_n, const double* raw,
                                                        int64_t n_max, double* block_sums, double* result,
                                                        unsigned int* done, const long long* n_dev,
                                                        size_t raw_stride, size_t state_stride_b) {
  if (blockIdx.y) {  // candidate y of a batch (vote_angles_kernel's layout); its own done counter
    const size_t y = blockIdx.y;
    bins += y * (size_t)bins_n;
    raw += y * raw_stride;
    block_sums += y * 2 * (size_t)gridDim.x;
    result = reinterpret_cast<double*>(reinterpret_cast<char*>(result) + y * state_stride_b);
    done += y;
    if (n_dev) n_dev = reinterpret_cast<const long long*>(reinterpret_cast<const char*>(n_dev) + y * state_stride_b);
  }
  const int64_t n = n_dev ? min(n_max, (int64_t)*n_dev) : n_max;
  __shared__ unsigned long long s_key[8];
  __shared__ double s_red[2][8];
  __shared__ bool s_last;
  // every block finds the peak bin redundantly (bins are tiny)
  unsigned long long key = 0;
  for (int k = threadIdx.x; k < bins_n; k += blockDim.x) {
    const unsigned long long kk = ((unsigned long long)bins[k] << 32) | (0xFFFFFFFFu - (uint32_t)k);
    key = key > kk ? key : kk;
  }
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long t = __shfl_xor_sync(0xFFFFFFFFu, key, o);
    key = key > t ? key : t;
  }
  if ((threadIdx.x & 31) == 0) s_key[threadIdx.x >> 5] = key;
  __syncthreads();
  key = 0;
  for (int w = 0; w < 8; ++w) key = key > s_key[w] ? key : s_key[w];
  const int kpk = (int)(0xFFFFFFFFu - (uint32_t)(key & 0xFFFFFFFFu));
  const double w = xd(2.0 * kPi, (double)bins_n);
  const double center = xa(-kPi, xm(kpk + 0.5, w));
  const double window = xm(1.5, w);
  double v[2] = {0.0, 0.0};
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
    const double a = raw[k];
    if (a != a) continue;  // degenerate
    // fmod(x, 2 pi) is exact and equals x for |x| < 2 pi (a, center in [-pi, pi]): skip the slow call
    const double x = xs(a, center);
    double d = fabs(x) < 2.0 * kPi ? x : fmod(x, 2.0 * kPi);
    if (d <= -kPi) d = xa(d, 2.0 * kPi);
    if (d > kPi) d = xs(d, 2.0 * kPi);
    if (fabs(d) <= window) {
      // sincos shares the argument reduction; its results are bit-identical to sin() and cos()
      // (checked on 16.8M angles over [-pi, pi] on the B200: tools/_bin/sincos_check)
      double sa, ca;
      sincos(a, &sa, &ca);
      v[0] = xa(v[0], sa);
      v[1] = xa(v[1], ca);
    }
  }
  for (int k = 0; k < 2; ++k)
    for (int o = 16; o > 0; o >>= 1) v[k] = xa(v[k], __shfl_xor_sync(0xFFFFFFFFu, v[k], o));
  if ((threadIdx.x & 31) == 0) {
    s_red[0][threadIdx.x >> 5] = v[0];
    s_red[1][threadIdx.x >> 5] = v[1];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0, c = 0;
    for (int ww = 0; ww < 8; ++ww) {
      s = xa(s, s_red[0][ww]);
      c = xa(c, s_red[1][ww]);
    }
    block_sums[2 * blockIdx.x] = s;
    block_sums[2 * blockIdx.x + 1] = c;
    __threadfence();
    s_last = atomicAdd(done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last) return;
  // last block: fixed-order parallel reduction (thread t: blocks t, t+256, ...; then the tree)
  double s2[2] = {0.0, 0.0};
  for (unsigned b = threadIdx.x; b < gridDim.x; b += blockDim.x) {
    s2[0] = xa(s2[0], __ldcg(block_sums + 2 * b));
    s2[1] = xa(s2[1], __ldcg(block_sums + 2 * b + 1));
  }
  for (int k = 0; k < 2; ++k)
    for (int o = 16; o > 0; o >>= 1) s2[k] = xa(s2[k], __shfl_xor_sync(0xFFFFFFFFu, s2[k], o));
  __syncthreads();
  if ((threadIdx.x & 31) == 0) {
    s_red[0][threadIdx.x >> 5] = s2[0];
    s_red[1][threadIdx.x >> 5] = s2[1];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0, c = 0;
    for (int ww = 0; ww < 8; ++ww) {
      s = xa(s, s_red[0][ww]);
      c = xa(c, s_red[1][ww]);
    }
    result[0] = s;
    result[1] = c;
    result[2] = (double)kpk;
    result[3] = center;
    *done = 0u;
  }
}

struct SupArgs {
  const double* zx;
  const double* zy;
  const double* zz;
  const int32_t* kept;
  const double* corrs;
  int64_t n;
  double a0, a1, a2, angle, eps, tau;
  uint32_t* band_flags;  // nullable
  int32_t* block_counts; // [nblocks][2]
  int32_t* result;       // [0]=coherent [1]=band size
  unsigned int* done;
};

__global__ void __launch_bounds__(kClsThreads) model_support_kernel(SupArgs a) {
  __shared__ int s_c[kClsThreads / 32][2];
  __shared__ bool s_last;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t base = (int64_t)blockIdx.x * kClsPerBlock;
  int coh = 0, band = 0;
  for (int r = 0; r < kClsPerThread; ++r) {
    const int64_t i = base + r * kClsThreads + tid;
    bool inb = false;
    if (i < a.n) {
      const double d = fabs(xdot(a.a0, a.a1, a.a2, a.zx[i], a.zy[i], a.zz[i]));
      if (d < 4.0 * a.eps) {
        double ang;
        if (corr_angle(a.a0, a.a1, a.a2, a.corrs + 6 * (int64_t)a.kept[i], a.tau, &ang)) {
          if (fabs(remainder(xs(ang, a.angle), 2.0 * kPi)) < 0.1) {
            inb = true;
            if (d < a.eps) ++coh;
          }
        }
      }
    }
    const unsigned word = __ballot_sync(0xFFFFFFFFu, inb);
    band += inb ? 1 : 0;
    if (a.band_flags && lane == 0 && (base + r * kClsThreads + warp * 32) < a.n)
      a.band_flags[(base + r * kClsThreads + warp * 32) >> 5] = word;
  }
  for (int o = 16; o > 0; o >>= 1) {
    coh += __shfl_xor_sync(0xFFFFFFFFu, coh, o);
    band += __shfl_xor_sync(0xFFFFFFFFu, band, o);
  }
  if (lane == 0) {
    s_c[warp][0] = coh;
    s_c[warp][1] = band;
  }
  __syncthreads();
  if (tid == 0) {
    int c = 0, b = 0;
    for (int w = 0; w < kClsThreads / 32; ++w) {
      c += s_c[w][0];
      b += s_c[w][1];
    }
    a.block_counts[2 * blockIdx.x] = c;
    a.block_counts[2 * blockIdx.x + 1] = b;
    __threadfence();
    s_last = atomicAdd(a.done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last) return;
  // last block: parallel integer reduction (order-free)
  long long c = 0, b = 0;
  for (unsigned k = tid; k < gridDim.x; k += blockDim.x) {
    c += __ldcg(a.block_counts + 2 * k);
    b += __ldcg(a.block_counts + 2 * k + 1);
  }
  for (int o = 16; o > 0; o >>= 1) {
    c += __shfl_xor_sync(0xFFFFFFFFu, c, o);
    b += __shfl_xor_sync(0xFFFFFFFFu, b, o);
  }
  __shared__ long long s_cb[2][kClsThreads / 32];
  if ((tid & 31) == 0) {
    s_cb[0][tid >> 5] = c;
    s_cb[1][tid >> 5] = b;
  }
  __syncthreads();
  if (tid == 0) {
    long long cc = 0, bb = 0;
    for (int w = 0; w < kClsThreads / 32; ++w) {
      cc += s_cb[0][w];
      bb += s_cb[1][w];
    }
    a.result[0] = (int32_t)cc;
    a.result[1] = (int32_t)bb;
    *a.done = 0u;
  }
}

// model_support of up to kSupMax candidates in ONE pass (the rescue / estimate_multi candidate
// batches): each constraint's z is read once and tested against every candidate, with exactly the
// per-candidate predicate of model_support_kernel; per-candidate integer counts (order-free), the
// last block reduces them. Equal to K launches of model_support_kernel, bit for bit.
constexpr int kSupMax = 8;
struct SupMultiArgs {
  const double* zx;
  const double* zy;
  const double* zz;
  const int32_t* kept;
  const double* corrs;
  int64_t n;
  int K;
  double ax[kSupMax][3];
  double angle[kSupMax];
  double eps, tau;
  uint32_t* band_flags;  // nullable: candidate k's words at band_flags + k * band_stride
  size_t band_stride;
  int32_t* block_counts; // [nblocks][kSupMax][2]
  int32_t* result;       // [K][2]: coherent, band size
  unsigned int* done;
};

// Per candidate, the block first compacts its |a.z| < 4 eps constraints (ballot + warp offsets:
// ~6% of them) into a shared list, then all threads run the expensive part -- the
// correspondence angle (f64 cross products + atan2) and the window test -- on that dense list,
// instead of every warp running it for its one or two band lanes. Band bits are set in a shared
// bitmap of the block's 32 words; counts are integers (order-free).
__global__ void __launch_bounds__(kClsThreads) model_support_multi_kernel(SupMultiArgs a) {
  __shared__ int s_list[kClsPerBlock];                 // band candidates: element (r * threads + tid)
  __shared__ double s_d[kClsPerBlock];                 // their |a.z|
  __shared__ uint32_t s_words[kClsPerBlock / 32];      // band bits of the block's elements
  __shared__ int s_wcnt[kClsThreads / 32], s_n;
  __shared__ int s_cnt[kSupMax][2];
  __shared__ bool s_last;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t base = (int64_t)blockIdx.x * kClsPerBlock;
  double z[kClsPerThread][3];
#pragma unroll
  for (int r = 0; r < kClsPerThread; ++r) {
    const int64_t i = base + r * kClsThreads + tid;
    const bool ok = i < a.n;
    z[r][0] = ok ? a.zx[i] : 0.0;
    z[r][1] = ok ? a.zy[i] : 0.0;
    z[r][2] = ok ? a.zz[i] : 0.0;
  }
  if (tid < 2 * kSupMax) s_cnt[tid >> 1][tid & 1] = 0;
  for (int k = 0; k < a.K; ++k) {  // uniform
    const double a0 = a.ax[k][0], a1 = a.ax[k][1], a2 = a.ax[k][2];
    // 1. compaction of the band candidates (in element order within each warp)
    int mine = 0;
    bool cand[kClsPerThread];
    double dv[kClsPerThread];
#pragma unroll
    for (int r = 0; r < kClsPerThread; ++r) {
      const int64_t i = base + r * kClsThreads + tid;
      dv[r] = fabs(xdot(a0, a1, a2, z[r][0], z[r][1], z[r][2]));
      cand[r] = i < a.n && dv[r] < 4.0 * a.eps;
      mine += cand[r] ? 1 : 0;
    }
    int incl = mine;
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) s_wcnt[warp] = incl;
    if (tid < kClsPerBlock / 32) s_words[tid] = 0u;
    __syncthreads();
    int off = 0, tot = 0;
    for (int w = 0; w < kClsThreads / 32; ++w) {
      off += w < warp ? s_wcnt[w] : 0;
      tot += s_wcnt[w];
    }
    int pos = off + incl - mine;
#pragma unroll
    for (int r = 0; r < kClsPerThread; ++r)
      if (cand[r]) {
        s_list[pos] = r * kClsThreads + tid;
        s_d[pos] = dv[r];
        ++pos;
      }
    __syncthreads();
    // 2. the angle test on the dense list
    int coh = 0, band = 0;
    for (int q = tid; q < tot; q += kClsThreads) {
      const int e = s_list[q];
      const int64_t i = base + e;
      double ang;
      if (corr_angle(a0, a1, a2, a.corrs + 6 * (int64_t)a.kept[i], a.tau, &ang) &&
          fabs(remainder(xs(ang, a.angle[k]), 2.0 * kPi)) < 0.1) {
        ++band;
        if (s_d[q] < a.eps) ++coh;
        if (a.band_flags) atomicOr(&s_words[e >> 5], 1u << (e & 31));
      }
    }
    for (int o = 16; o > 0; o >>= 1) {
      coh += __shfl_xor_sync(0xFFFFFFFFu, coh, o);
      band += __shfl_xor_sync(0xFFFFFFFFu, band, o);
    }
    if (lane == 0 && (coh | band)) {
      atomicAdd(&s_cnt[k][0], coh);
      atomicAdd(&s_cnt[k][1], band);
    }
    __syncthreads();
    if (a.band_flags && tid < kClsPerBlock / 32 && base + 32 * tid < a.n)
      a.band_flags[k * a.band_stride + (size_t)(base >> 5) + tid] = s_words[tid];
    __syncthreads();  // s_list / s_words / s_wcnt reused by the next candidate
  }
  if (tid < 2 * a.K) a.block_counts[(size_t)blockIdx.x * (2 * kSupMax) + tid] = s_cnt[tid >> 1][tid & 1];
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    s_last = atomicAdd(a.done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  // last block: one warp per (candidate, count) pair, integer sums (order-free)
  for (int p = warp; p < 2 * a.K; p += kClsThreads / 32) {
    long long v = 0;
    for (unsigned b = lane; b < gridDim.x; b += 32) v += __ldcg(a.block_counts + (size_t)b * (2 * kSupMax) + p);
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
    if (lane == 0) a.result[p] = (int32_t)v;
  }
  __syncthreads();
  if (tid == 0) *a.done = 0u;
}

__global__ void strip_kernel(const double* zx, const double* zy, const double* zz, int64_t n, double a0, double a1,
                             double a2, double strip, uint8_t* removed) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (fabs(xdot(a0, a1, a2, zx[i], zy[i], zz[i])) < strip) removed[i] = 1;
}

// estimate_multi's strip width (estimator.cpp:470-480) on the device, no host read-back: the
// q-th smallest |axis.z| over the winning model's support band (nth_element), then
// strip = max(2 eps, 1.25 * value). One CTA: the band members' values are gathered as u64 keys
// (the bit patterns of non-negative doubles order like the values; output order is irrelevant to a
// selection), then an exact radix select (11-bit digits from the top, six passes) finds the key of
// rank q. Replaces compaction + gather + a full radix sort + two host round trips.
constexpr int kSelThreads = 1024;
constexpr int kSelSmem = 4096;  // keys kept in shared memory once the prefix narrows them down
// gather: one thread per band word (the whole grid), warp-aggregated output reservation; keys[-1]
// (a u64 slot before the keys) counts them
__global__ void band_gather_kernel(const uint32_t* band, int64_t n, const double* zx, const double* zy,
                                   const double* zz, double a0, double a1, double a2, unsigned long long* keys,
                                   unsigned long long* count) {
  const int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  const uint32_t m0 = w < (n + 31) / 32 ? band[w] : 0u;
  uint32_t m = m0;
  if (w * 32 + 32 > n && w < (n + 31) / 32) m &= (n - w * 32) >= 32 ? 0xFFFFFFFFu : ((1u << (n - w * 32)) - 1u);
  const int c = __popc(m);
  int incl = c;
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
    if (lane >= o) incl += y;
  }
  const int tot = __shfl_sync(0xFFFFFFFFu, incl, 31);
  unsigned long long base = 0;
  if (lane == 31 && tot) base = atomicAdd(count, (unsigned long long)tot);
  base = __shfl_sync(0xFFFFFFFFu, base, 31);
  unsigned long long pos = base + (unsigned long long)(incl - c);
  while (m) {
    const int bit = __ffs(m) - 1;
    m &= m - 1u;
    const int64_t i = w * 32 + bit;
    const double d = fabs(xdot(a0, a1, a2, zx[i], zy[i], zz[i]));  // the band value of estimator.cpp:470-480
    keys[pos++] = (unsigned long long)__double_as_longlong(d);
  }
}

// select: the key of rank q by an exact radix select (11-bit digits from the top, six passes); the
// keys still matching the prefix are moved to shared memory as soon as they fit
__global__ void __launch_bounds__(kSelThreads) band_select_kernel(const unsigned long long* keys,
                                                                 const unsigned long long* count, long long q,
                                                                 double floor_strip, double* strip_out) {
  __shared__ unsigned int s_hist[2048];
  __shared__ unsigned long long s_keys[kSelSmem];
  __shared__ unsigned int s_wsum[kSelThreads / 32];
  __shared__ int s_digit, s_m;
  __shared__ long long s_before;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long long acc = (long long)*count;
  if (acc == 0) {  // (the host only launches this with a non-empty band)
    if (tid == 0) *strip_out = floor_strip;
    return;
  }
  unsigned long long prefix = 0ull, pmask = 0ull;
  long long rank = q < acc ? q : acc - 1;  // (q < acc by construction: the host's band size)
  const unsigned long long* src = keys;  // the candidate keys of this pass
  long long m = acc;
  bool in_smem = false;
  const int shifts[6] = {53, 42, 31, 20, 9, 0};
  const int widths[6] = {11, 11, 11, 11, 11, 9};
  for (int p = 0; p < 6; ++p) {
    const int sh = shifts[p];
    const unsigned long long dmask = (1ull << widths[p]) - 1ull;
    for (int b = tid; b < 2048; b += kSelThreads) s_hist[b] = 0u;
    __syncthreads();
    for (long long k = tid; k < m; k += kSelThreads) {
      const unsigned long long key = in_smem ? s_keys[k] : src[k];
      if ((key & pmask) == prefix) atomicAdd(&s_hist[(key >> sh) & dmask], 1u);
    }
    __syncthreads();
    // exclusive scan of the 2048 bins (2 per thread), then the bin holding rank
    const unsigned h0 = s_hist[2 * tid], h1 = s_hist[2 * tid + 1];
    unsigned incl = h0 + h1;
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) s_wsum[warp] = incl;
    __syncthreads();
    unsigned long long before = 0;
    for (int w = 0; w < warp; ++w) before += s_wsum[w];
    before += incl - (h0 + h1);
    if ((long long)before <= rank && rank < (long long)(before + h0)) {
      s_digit = 2 * tid;
      s_before = (long long)before;
      s_m = (int)h0;
    } else if ((long long)(before + h0) <= rank && rank < (long long)(before + h0 + h1)) {
      s_digit = 2 * tid + 1;
      s_before = (long long)(before + h0);
      s_m = (int)h1;
    }
    __syncthreads();
    prefix |= (unsigned long long)s_digit << sh;
    pmask |= dmask << sh;
    rank -= s_before;
    const int left = s_m;  // keys matching the new prefix
    __syncthreads();
    if (!in_smem && left <= kSelSmem && p < 5) {  // compact them into shared memory
      if (tid == 0) s_m = 0;
      __syncthreads();
      for (long long k = tid; k < m; k += kSelThreads) {
        const unsigned long long key = src[k];
        if ((key & pmask) == prefix) s_keys[atomicAdd(&s_m, 1)] = key;
      }
      __syncthreads();
      m = left;
      in_smem = true;
    }
  }
  if (tid == 0) {
    const double v = __longlong_as_double((long long)prefix);
    const double x = 1.25 * v;
    *strip_out = floor_strip < x ? x : floor_strip;  // std::max(strip, 1.25 * v)
  }
}

__global__ void strip_dev_kernel(const double* zx, const double* zy, const double* zz, int64_t n, double a0, double a1,
                                 double a2, const double* strip, uint8_t* removed) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (fabs(xdot(a0, a1, a2, zx[i], zy[i], zz[i])) < *strip) removed[i] = 1;
}


// near_identity_model cluster test + Kabsch cross-covariance (estimator.cpp:198-249).
struct NearArgs {
  const double* corrs;
  const int32_t* sub_kept;
  int64_t n;
  int normalize;
  uint32_t* flags;
  int32_t* block_count;
  double* block_h;  // [nblocks][9]
  int32_t* block_offsets;
  double* result;   // [0]=count [1..9]=H row-major
  unsigned int* done;
};

__device__ __forceinline__ void load_norm(const double* c, int normalize, double* x, double* y) {
  x[0] = c[0]; x[1] = c[1]; x[2] = c[2]; y[0] = c[3]; y[1] = c[4]; y[2] = c[5];
  if (normalize) {
    const double nx = __dsqrt_rn(xdot(x[0], x[1], x[2], x[0], x[1], x[2]));
    const double ny = __dsqrt_rn(xdot(y[0], y[1], y[2], y[0], y[1], y[2]));
    if (nx > 0.0) { x[0] = xd(x[0], nx); x[1] = xd(x[1], nx); x[2] = xd(x[2], nx); }
    if (ny > 0.0) { y[0] = xd(y[0], ny); y[1] = xd(y[1], ny); y[2] = xd(y[2], ny); }
  }
}

__global__ void __launch_bounds__(kClsThreads) near_identity_kernel(NearArgs a) {
  __shared__ double s_red[9][kClsThreads / 32];
  __shared__ int s_cnt[kClsThreads / 32];
  __shared__ bool s_last;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t base = (int64_t)blockIdx.x * kClsPerBlock;
  double h[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  int cnt = 0;
  for (int r = 0; r < kClsPerThread; ++r) {
    const int64_t i = base + r * kClsThreads + tid;
    bool in = false;
    double x[3], y[3];
    if (i < a.n) {
      load_norm(a.corrs + 6 * (int64_t)a.sub_kept[i], a.normalize, x, y);
      const double d0 = xs(y[0], x[0]), d1 = xs(y[1], x[1]), d2 = xs(y[2], x[2]);
      in = __dsqrt_rn(xdot(d0, d1, d2, d0, d1, d2)) < 0.1;
    }
    const unsigned word = __ballot_sync(0xFFFFFFFFu, in);
    if (lane == 0 && (base + r * kClsThreads + warp * 32) < a.n) a.flags[(base + r * kClsThreads + warp * 32) >> 5] = word;
    if (in) {
      ++cnt;
      for (int p = 0; p < 3; ++p)
        for (int q = 0; q < 3; ++q) h[p * 3 + q] = xa(h[p * 3 + q], xm(y[p], x[q]));
    }
  }
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xFFFFFFFFu, cnt, o);
  if (lane == 0) s_cnt[warp] = cnt;
  block_sum<9>(h, s_red);
  if (tid == 0) {
    int c = 0;
    for (int w = 0; w < kClsThreads / 32; ++w) c += s_cnt[w];
    a.block_count[blockIdx.x] = c;
    for (int k = 0; k < 9; ++k) a.block_h[(size_t)blockIdx.x * 9 + k] = h[k];
    __threadfence();
    s_last = atomicAdd(a.done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last) return;
  // last block: each thread owns a contiguous run of blocks (sequential sums), exclusive scan of
  // the run counts, fixed tree for the 9 Kabsch sums
  const int nb = gridDim.x;
  const int per = (nb + kClsThreads - 1) / kClsThreads;
  const int b0 = tid * per, b1 = min(nb, b0 + per);
  long long tc = 0;
  double hh[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  for (int b = b0; b < b1; ++b) {
    tc += __ldcg(a.block_count + b);
    for (int k = 0; k < 9; ++k) hh[k] = xa(hh[k], __ldcg(a.block_h + (size_t)b * 9 + k));
  }
  __shared__ long long s_run[kClsThreads];
  __shared__ double s_h[9][kClsThreads / 32];
  s_run[tid] = tc;
  for (int k = 0; k < 9; ++k)
    for (int o = 16; o > 0; o >>= 1) hh[k] = xa(hh[k], __shfl_xor_sync(0xFFFFFFFFu, hh[k], o));
  if ((tid & 31) == 0)
    for (int k = 0; k < 9; ++k) s_h[k][tid >> 5] = hh[k];
  __syncthreads();
  if (tid == 0) {
    long long acc = 0;
    for (int t = 0; t < kClsThreads; ++t) {
      const long long x = s_run[t];
      s_run[t] = acc;
      acc += x;
    }
    a.result[0] = (double)acc;
    for (int k = 0; k < 9; ++k) {
      double v = 0.0;
      for (int w = 0; w < kClsThreads / 32; ++w) v = xa(v, s_h[k][w]);
      a.result[1 + k] = v;
    }
    *a.done = 0u;
  }
  __syncthreads();
  long long off = s_run[tid];
  for (int b = b0; b < b1; ++b) {
    a.block_offsets[b] = (int32_t)off;
    off += __ldcg(a.block_count + b);
  }
}

// Consensus counts of many candidate axes over one constraint set (baselines.cpp:16-24 consensus_count,
// the scoring of grid_oracle_axis and ransac_rotation): count_k = #{i : |a_k . z_i| < eps}, strict,
// with the reference's op order. Threads own axes (one register counter each); z is staged through
// shared memory in tiles (f32 for the filter, f64 for the exact re-check): a pair whose f32 dot is
// within kConsDelta of eps is re-evaluated exactly (|d32 - d64| <= ~4e-7 for unit vectors).
constexpr int kConsAxes = 256;   // axes per block (threads)
constexpr int kConsTile = 1024;  // constraints per shared-memory tile
constexpr double kConsDelta = 4e-6;
__global__ void __launch_bounds__(kConsAxes) consensus_kernel(const double* axes, int m, const double* z, int64_t n,
                                                             int64_t z_per_block, double eps, uint32_t* counts) {
  __shared__ float s_z32[kConsTile][3];
  __shared__ double s_z64[kConsTile][3];
  const int k = blockIdx.y * kConsAxes + threadIdx.x;
  double a0 = 0, a1 = 0, a2 = 0;
  if (k < m) {
    a0 = axes[3 * k];
    a1 = axes[3 * k + 1];
    a2 = axes[3 * k + 2];
  }
  const float f0 = (float)a0, f1 = (float)a1, f2 = (float)a2;
  const float lo = (float)(eps - kConsDelta), hi = (float)(eps + kConsDelta);
  uint32_t cnt = 0;
  const int64_t z0 = (int64_t)blockIdx.x * z_per_block, z1 = z0 + z_per_block < n ? z0 + z_per_block : n;
  for (int64_t t0 = z0; t0 < z1; t0 += kConsTile) {
    const int len = (int)(z1 - t0 < kConsTile ? z1 - t0 : (int64_t)kConsTile);
    __syncthreads();
    for (int q = threadIdx.x; q < 3 * len; q += blockDim.x) {
      const double v = z[3 * t0 + q];
      s_z64[q / 3][q % 3] = v;
      s_z32[q / 3][q % 3] = (float)v;
    }
    __syncthreads();
    if (k < m) {
#pragma unroll 4
      for (int i = 0; i < len; ++i) {
        const float d = fabsf(fmaf(f2, s_z32[i][2], fmaf(f1, s_z32[i][1], f0 * s_z32[i][0])));
        if (d < lo) {
          ++cnt;
        } else if (d < hi) {  // near the band edge: the reference's exact evaluation
          const double dd = xa(xa(xm(a0, s_z64[i][0]), xm(a1, s_z64[i][1])), xm(a2, s_z64[i][2]));
          if (fabs(dd) < eps) ++cnt;
        }
      }
    }
  }
  if (k < m && cnt) atomicAdd(counts + k, cnt);
}

}  // namespace

int classify_blocks(int64_t n) { return (int)((n + kClsPerBlock - 1) / kClsPerBlock); }

void launch_consensus_counts(const double* axes, int m, const double* z, int64_t n, double eps, uint32_t* counts,
                             int sms, cudaStream_t s) {
  if (m <= 0 || n <= 0) return;
  const int by = (m + kConsAxes - 1) / kConsAxes;
  // enough z-blocks for ~4 blocks per SM overall, each a multiple of the tile
  int64_t bx = (4LL * sms + by - 1) / by;
  const int64_t tiles = (n + kConsTile - 1) / kConsTile;
  if (bx > tiles) bx = tiles;
  if (bx < 1) bx = 1;
  int64_t per = (n + bx - 1) / bx;
  per = (per + kConsTile - 1) / kConsTile * kConsTile;
  bx = (n + per - 1) / per;
  consensus_kernel<<<dim3((unsigned)bx, (unsigned)by), kConsAxes, 0, s>>>(axes, m, z, n, per, eps, counts);
}

void launch_classify_mode(const double* zx, const double* zy, const double* zz, int64_t n, const double axis[3],
                          double eps, int mode, const ClassifyOut& o, int32_t* block_offsets, unsigned int* done,
                          cudaStream_t s) {
  ClsArgs a;
  a.zx = zx;
  a.zy = zy;
  a.zz = zz;
  a.n = n;
  a.ax = axis ? axis[0] : 0;
  a.ay = axis ? axis[1] : 0;
  a.az = axis ? axis[2] : 0;
  a.eps = eps;
  a.mode = mode;
  a.flags = o.flags;
  a.prev = o.prev;
  a.block_count = o.block_count;
  a.block_scatter = o.block_scatter;
  a.block_diff = o.block_diff;
  a.block_offsets = block_offsets;
  a.result = o.result;
  a.done = done;
  classify_kernel<<<classify_blocks(n), kClsThreads, 0, s>>>(a);
}

void launch_compact_flags(const uint32_t* flags, int64_t n, const int32_t* map, const int32_t* block_offsets,
                          int32_t* out, cudaStream_t s, int32_t* out_host) {
  compact_kernel<<<classify_blocks(n), kClsThreads, 0, s>>>(flags, n, map, block_offsets, out, out_host);
}

void launch_vote_angles_k(const double axis[3], const double* corrs, const int32_t* idx, int64_t n_idx, int bin_count,
                          double tau, uint32_t* bins, double* raw, unsigned long long* counts, cudaStream_t s,
                          const double* axis_dev, const long long* n_dev, int32_t* idx_host) {
  AngArgs a;
  a.idx_host = idx_host;
  a.a0 = axis ? axis[0] : 0.0;
  a.a1 = axis ? axis[1] : 0.0;
  a.a2 = axis ? axis[2] : 0.0;
  a.axis_dev = axis_dev;
  a.n_dev = n_dev;
  a.tau = tau;
  a.corrs = corrs;
  a.idx = idx;
  a.n = n_idx;
  a.bins_n = bin_count;
  a.bins = bins;
  a.raw = raw;
  a.counts = counts;
  a.idx_stride = a.raw_stride = a.state_stride_b = 0;
  const int64_t want = (n_idx + 255) / 256;
  const int blocks = (int)(want < 1 ? 1 : (want > 592 ? 592 : want));
  const size_t smem = bin_count <= 8192 ? (size_t)bin_count * 4 : 0;
  vote_angles_kernel<<<blocks, 256, smem, s>>>(a);
}

void launch_vote_angles_batch_k(int K, const double* corrs, const int32_t* idx, size_t idx_stride, int64_t n_idx,
                                int bin_count, double tau, uint32_t* bins, double* raw, size_t raw_stride,
                                unsigned long long* counts, const double* axis_dev, const long long* n_dev,
                                size_t state_stride_b, cudaStream_t s) {
  AngArgs a;
  a.idx_host = nullptr;
  a.a0 = a.a1 = a.a2 = 0.0;
  a.axis_dev = axis_dev;
  a.n_dev = n_dev;
  a.tau = tau;
  a.corrs = corrs;
  a.idx = idx;
  a.n = n_idx;
  a.bins_n = bin_count;
  a.bins = bins;
  a.raw = raw;
  a.counts = counts;
  a.idx_stride = idx_stride;
  a.raw_stride = raw_stride;
  a.state_stride_b = state_stride_b;
  // the same grid per candidate as launch_vote_angles_k (identical thread-to-element mapping)
  const int64_t want = (n_idx + 255) / 256;
  const int blocks = (int)(want < 1 ? 1 : (want > 592 ? 592 : want));
  const size_t smem = bin_count <= 8192 ? (size_t)bin_count * 4 : 0;
  vote_angles_kernel<<<dim3(blocks, K), 256, smem, s>>>(a);
}

void launch_peak_angle_k(const uint32_t* bins, int bin_count, const double* raw, int64_t n_raw, double* block_sums,
                         double* result, unsigned int* done, cudaStream_t s, const long long* n_dev) {
  const int64_t want = (n_raw + 255) / 256;
  const int blocks = (int)(want < 1 ? 1 : (want > 296 ? 296 : want));
  peak_angle_kernel<<<blocks, 256, 0, s>>>(bins, bin_count, raw, n_raw, block_sums, result, done, n_dev, 0, 0);
}

int peak_angle_blocks(int64_t n_raw) {
  const int64_t want = (n_raw + 255) / 256;
  return (int)(want < 1 ? 1 : (want > 296 ? 296 : want));
}

void launch_peak_angle_batch_k(int K, const uint32_t* bins, int bin_count, const double* raw, size_t raw_stride,
                               int64_t n_raw, double* block_sums, double* result, unsigned int* done,
                               const long long* n_dev, size_t state_stride_b, cudaStream_t s) {
  // the same grid (hence the same fixed-order sums) per candidate as launch_peak_angle_k
  peak_angle_kernel<<<dim3(peak_angle_blocks(n_raw), K), 256, 0, s>>>(bins, bin_count, raw, n_raw, block_sums, result,
                                                                     done, n_dev, raw_stride, state_stride_b);
}

void launch_model_support_k(const double* zx, const double* zy, const double* zz, const int32_t* kept,
                            const double* corrs, int64_t n, const double axis[3], double angle, double eps, double tau,
                            uint32_t* band_flags, int32_t* block_counts, int32_t* result, unsigned int* done,
                            cudaStream_t s) {
  SupArgs a;
  a.zx = zx;
  a.zy = zy;
  a.zz = zz;
  a.kept = kept;
  a.corrs = corrs;
  a.n = n;
  a.a0 = axis[0];
  a.a1 = axis[1];
  a.a2 = axis[2];
  a.angle = angle;
  a.eps = eps;
  a.tau = tau;
  a.band_flags = band_flags;
  a.block_counts = block_counts;
  a.result = result;
  a.done = done;
  model_support_kernel<<<classify_blocks(n), kClsThreads, 0, s>>>(a);
}

int model_support_multi_max() { return kSupMax; }

void launch_model_support_multi_k(const double* zx, const double* zy, const double* zz, const int32_t* kept,
                                  const double* corrs, int64_t n, int K, const double (*axes)[3], const double* angles,
                                  double eps, double tau, uint32_t* band_flags, size_t band_stride,
                                  int32_t* block_counts, int32_t* result, unsigned int* done, cudaStream_t s) {
  SupMultiArgs a;
  a.zx = zx;
  a.zy = zy;
  a.zz = zz;
  a.kept = kept;
  a.corrs = corrs;
  a.n = n;
  a.K = K;
  for (int k = 0; k < kSupMax; ++k) {
    for (int q = 0; q < 3; ++q) a.ax[k][q] = k < K ? axes[k][q] : 0.0;
    a.angle[k] = k < K ? angles[k] : 0.0;
  }
  a.eps = eps;
  a.tau = tau;
  a.band_flags = band_flags;
  a.band_stride = band_stride;
  a.block_counts = block_counts;
  a.result = result;
  a.done = done;
  model_support_multi_kernel<<<classify_blocks(n), kClsThreads, 0, s>>>(a);
}

void launch_strip_k(const double* zx, const double* zy, const double* zz, int64_t n, const double axis[3], double strip,
                    uint8_t* removed, cudaStream_t s) {
  strip_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(zx, zy, zz, n, axis[0], axis[1], axis[2], strip, removed);
}

void launch_band_strip_k(const uint32_t* band, int64_t n, const double* zx, const double* zy, const double* zz,
                         const double axis[3], long long q, double floor_strip, unsigned long long* keys,
                         double* strip_dev, uint8_t* removed, cudaStream_t s) {
  // keys[0] counts, keys + 1 holds the keys
  cudaMemsetAsync(keys, 0, sizeof(unsigned long long), s);
  const int64_t nw = (n + 31) / 32;
  band_gather_kernel<<<(unsigned)((nw + 255) / 256), 256, 0, s>>>(band, n, zx, zy, zz, axis[0], axis[1], axis[2],
                                                                 keys + 1, keys);
  band_select_kernel<<<1, kSelThreads, 0, s>>>(keys + 1, keys, q, floor_strip, strip_dev);
  strip_dev_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(zx, zy, zz, n, axis[0], axis[1], axis[2], strip_dev,
                                                              removed);
}


void launch_near_identity_k(const double* corrs, const int32_t* sub_kept, int64_t n, int normalize, uint32_t* flags,
                            int32_t* block_count, double* block_h, int32_t* block_offsets, double* result,
                            unsigned int* done, cudaStream_t s) {
  NearArgs a;
  a.corrs = corrs;
  a.sub_kept = sub_kept;
  a.n = n;
  a.normalize = normalize;
  a.flags = flags;
  a.block_count = block_count;
  a.block_h = block_h;
  a.block_offsets = block_offsets;
  a.result = result;
  a.done = done;
  near_identity_kernel<<<classify_blocks(n), kClsThreads, 0, s>>>(a);
}

}  // namespace rvb

namespace rvb {
namespace {
// Identity-model removal (estimator.cpp:461-467): the residual members with small motion.
__global__ void strip_identity_kernel(const double* corrs, const int32_t* kept, int64_t n, int normalize,
                                      uint8_t* removed) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n || removed[k]) return;
  double x[3], y[3];
  load_norm(corrs + 6 * (int64_t)kept[k], normalize, x, y);
  const double d0 = xs(y[0], x[0]), d1 = xs(y[1], x[1]), d2 = xs(y[2], x[2]);
  if (__dsqrt_rn(xdot(d0, d1, d2, d0, d1, d2)) < 0.1) removed[k] = 1;
}
}  // namespace
void launch_strip_identity_k(const double* corrs, const int32_t* kept, int64_t n, int normalize, uint8_t* removed,
                             cudaStream_t s) {
  if (n <= 0) return;
  strip_identity_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(corrs, kept, n, normalize, removed);
}


}  // namespace rvb

