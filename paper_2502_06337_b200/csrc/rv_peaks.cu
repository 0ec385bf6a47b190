// K3: peak search over the device vote grid.
//  * argmax with non-max-suppression disks (find_peaks inner scan, voting.cpp:145-152):
//    key = (count desc, row-major index asc), cells with count 0 never win. The greedy
//    top-K loop (mask disk + equatorial mirror disk, voting.cpp:142-167) is driven by the
//    host one round at a time, so the mirror test uses the same libm hypot as the reference.
//  * blurred_argmax for several radii (voting.cpp:176-216): u64 summed-area table, window
//    clipped at the grid edge, ties to the lowest row-major index. Integer sums are exact,
//    so the result is identical to the reference for any evaluation order.
#include <cuda_runtime.h>

#include <cstdint>

#include "rv_internal.h"

namespace rvb {
namespace {

constexpr int kArgThreads = 256;
constexpr int kMaxDisks = 16;

struct DiskSet {
  int n, r2, r;
  int cx[kMaxDisks], cy[kMaxDisks];
};

__device__ __forceinline__ unsigned long long umax64(unsigned long long a, unsigned long long b) {
  return a > b ? a : b;
}

__device__ __forceinline__ bool masked(const DiskSet& d, int x, int y) {
  for (int k = 0; k < d.n; ++k) {
    const int dx = x - d.cx[k], dy = y - d.cy[k];
    if (dx >= -d.r && dx <= d.r && dy >= -d.r && dy <= d.r && dx * dx + dy * dy <= d.r2) return true;
  }
  return false;
}

// Also sums every cell (u64) into out_key[1]: the vote's exactness guard (sum == N*J).
// With `mask` (any number of suppression disks: a G*G bit image maintained by mark_disks_kernel),
// masked cells are skipped by one bit test; otherwise the (<= kMaxDisks) disks are tested directly.
__global__ void __launch_bounds__(kArgThreads) argmax_kernel(const uint32_t* grid, int G, DiskSet disks,
                                                             const uint32_t* mask,
                                                             unsigned long long* block_keys,
                                                             unsigned long long* out_key, unsigned int* done) {
  __shared__ unsigned long long s_red[kArgThreads / 32];
  __shared__ unsigned long long s_sum[kArgThreads / 32];
  __shared__ bool s_last;
  const int64_t total = (int64_t)G * G;
  unsigned long long best = 0, sum = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  if ((total & 3) == 0) {
    const uint4* g4 = reinterpret_cast<const uint4*>(grid);
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < total / 4; q += stride) {
      const uint4 v = g4[q];
      const uint32_t c[4] = {v.x, v.y, v.z, v.w};
      sum += (unsigned long long)v.x + v.y + v.z + v.w;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (c[k] == 0) continue;
        const int64_t idx = q * 4 + k;
        if (mask ? ((mask[idx >> 5] >> (idx & 31)) & 1u) : (disks.n && masked(disks, (int)(idx % G), (int)(idx / G))))
          continue;
        best = umax64(best, ((unsigned long long)c[k] << 32) | (0xFFFFFFFFu - (uint32_t)idx));
      }
    }
  } else {
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += stride) {
      const uint32_t c = grid[idx];
      sum += c;
      if (c == 0) continue;
      if (mask ? ((mask[idx >> 5] >> (idx & 31)) & 1u) : (disks.n && masked(disks, (int)(idx % G), (int)(idx / G))))
        continue;
      best = umax64(best, ((unsigned long long)c << 32) | (0xFFFFFFFFu - (uint32_t)idx));
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    best = umax64(best, __shfl_xor_sync(0xFFFFFFFFu, best, o));
    sum += __shfl_xor_sync(0xFFFFFFFFu, sum, o);
  }
  if ((threadIdx.x & 31) == 0) {
    s_red[threadIdx.x >> 5] = best;
    s_sum[threadIdx.x >> 5] = sum;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long b = 0, sm = 0;
    for (int w = 0; w < kArgThreads / 32; ++w) {
      b = umax64(b, s_red[w]);
      sm += s_sum[w];
    }
    block_keys[blockIdx.x] = b;
    block_keys[gridDim.x + blockIdx.x] = sm;
    __threadfence();
    s_last = atomicAdd(done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (s_last) {
    unsigned long long b = 0, sm = 0;
    for (int k = threadIdx.x; k < (int)gridDim.x; k += blockDim.x) {
      b = umax64(b, ((volatile unsigned long long*)block_keys)[k]);
      sm += ((volatile unsigned long long*)block_keys)[gridDim.x + k];
    }
    for (int o = 16; o > 0; o >>= 1) {
      b = umax64(b, __shfl_xor_sync(0xFFFFFFFFu, b, o));
      sm += __shfl_xor_sync(0xFFFFFFFFu, sm, o);
    }
    if ((threadIdx.x & 31) == 0) {
      s_red[threadIdx.x >> 5] = b;
      s_sum[threadIdx.x >> 5] = sm;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned long long bb = 0, ss = 0;
      for (int w = 0; w < kArgThreads / 32; ++w) {
        bb = umax64(bb, s_red[w]);
        ss += s_sum[w];
      }
      out_key[0] = bb;
      out_key[1] = ss;
      *done = 0u;
    }
  }
}

// Sets the bits of every cell within distance r of each disk centre (clipped to the grid) --
// find_peaks' suppression (voting.cpp:145-152, the same dx*dx + dy*dy <= r*r disk).
__global__ void mark_disks_kernel(uint32_t* mask, int G, DiskSet d) {
  const int side = 2 * d.r + 1;
  const int k = blockIdx.y;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < side * side; t += gridDim.x * blockDim.x) {
    const int dx = t % side - d.r, dy = t / side - d.r;
    const int x = d.cx[k] + dx, y = d.cy[k] + dy;
    if (dx * dx + dy * dy > d.r2 || x < 0 || x >= G || y < 0 || y >= G) continue;
    const int64_t idx = (int64_t)y * G + x;
    atomicOr(&mask[idx >> 5], 1u << (idx & 31));
  }
}

// SAT row pass: rowpref[y][x+1] = sum_{x' <= x} counts[y][x'] (u64), rowpref[y][0] = 0.
__global__ void sat_rows_kernel(const uint32_t* grid, int G, unsigned long long* sat) {
  // sat is (G+1) x (G+1); this pass writes rows 1..G with row prefix sums
  __shared__ unsigned long long s[1024];
  const int y = blockIdx.x;
  const int W = G + 1;
  unsigned long long carry = 0;
  for (int x0 = 0; x0 < G; x0 += blockDim.x) {
    const int x = x0 + threadIdx.x;
    unsigned long long v = x < G ? grid[(size_t)y * G + x] : 0ull;
    s[threadIdx.x] = v;
    __syncthreads();
    for (int o = 1; o < (int)blockDim.x; o <<= 1) {  // Hillis-Steele inclusive scan
      const unsigned long long add = threadIdx.x >= (unsigned)o ? s[threadIdx.x - o] : 0ull;
      __syncthreads();
      s[threadIdx.x] += add;
      __syncthreads();
    }
    if (x < G) sat[(size_t)(y + 1) * W + (x + 1)] = carry + s[threadIdx.x];
    carry += s[blockDim.x - 1];
    __syncthreads();
  }
  if (threadIdx.x == 0) sat[(size_t)(y + 1) * W] = 0ull;
}

// SAT column pass: sat[y][x] += sat[y-1][x] down every column; row 0 = 0.
// Column prefix sums of the (G+1)^2 SAT in two levels: the rows are cut into kSatSeg segments;
// thread (x, seg) sums its segment, a per-column scan of the segment totals in shared memory,
// then each thread rescans its segment with the carried prefix (loads issued in batches).
constexpr int kSatSeg = 16;
constexpr int kSatCols = 16;  // columns per block -> blockDim = kSatCols * kSatSeg = 256
__global__ void __launch_bounds__(kSatCols * kSatSeg) sat_cols_kernel(int G, unsigned long long* sat) {
  __shared__ unsigned long long s_seg[kSatSeg][kSatCols];
  const int cx = threadIdx.x % kSatCols, seg = threadIdx.x / kSatCols;
  const int x = blockIdx.x * kSatCols + cx;
  const int W = G + 1;
  const int len = (G + kSatSeg - 1) / kSatSeg;
  const int y0 = 1 + seg * len, y1 = min(G + 1, y0 + len);
  unsigned long long tot = 0;
  if (x < W) {
    if (seg == 0) sat[x] = 0ull;
    for (int y = y0; y < y1; y += 8) {
      unsigned long long v[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = y + k < y1 ? sat[(size_t)(y + k) * W + x] : 0ull;
#pragma unroll
      for (int k = 0; k < 8; ++k) tot += v[k];
    }
  }
  s_seg[seg][cx] = tot;
  __syncthreads();
  unsigned long long carry = 0;
  for (int q = 0; q < seg; ++q) carry += s_seg[q][cx];
  if (x < W) {
    for (int y = y0; y < y1; y += 8) {
      unsigned long long v[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = y + k < y1 ? sat[(size_t)(y + k) * W + x] : 0ull;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        carry += v[k];
        if (y + k < y1) sat[(size_t)(y + k) * W + x] = carry;
      }
    }
  }
}

struct Radii {
  int n;
  int r[8];
};

__device__ __forceinline__ bool better(unsigned long long s, unsigned long long i, unsigned long long bs,
                                       unsigned long long bi) {
  return s > bs || (s == bs && i < bi);
}

// Box sums for every radius; per-block best (sum desc, index asc); the last block reduces.
__global__ void __launch_bounds__(256) blur_box_kernel(const unsigned long long* sat, int G, Radii radii,
                                                       unsigned long long* block_best,
                                                       unsigned long long* out_best, unsigned int* done) {
  __shared__ unsigned long long s_sum[8][256];
  __shared__ unsigned long long s_idx[8][256];
  __shared__ bool s_last;
  const int W = G + 1;
  const int64_t total = (int64_t)G * G;
  unsigned long long bs[8], bi[8];
  for (int k = 0; k < radii.n; ++k) {
    bs[k] = 0;
    bi[k] = ~0ull;
  }
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int cx = (int)(idx % G), cy = (int)(idx / G);
    for (int k = 0; k < radii.n; ++k) {
      const int r = radii.r[k];
      const int x0 = max(0, cx - r), x1 = min(G, cx + r + 1);
      const int y0 = max(0, cy - r), y1 = min(G, cy + r + 1);
      const unsigned long long s = sat[(size_t)y1 * W + x1] - sat[(size_t)y0 * W + x1] -
                                   sat[(size_t)y1 * W + x0] + sat[(size_t)y0 * W + x0];
      if (better(s, (unsigned long long)idx, bs[k], bi[k])) {
        bs[k] = s;
        bi[k] = (unsigned long long)idx;
      }
    }
  }
  for (int k = 0; k < radii.n; ++k) {
    s_sum[k][threadIdx.x] = bs[k];
    s_idx[k][threadIdx.x] = bi[k];
  }
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < (unsigned)o) {
      for (int k = 0; k < radii.n; ++k) {
        if (better(s_sum[k][threadIdx.x + o], s_idx[k][threadIdx.x + o], s_sum[k][threadIdx.x], s_idx[k][threadIdx.x])) {
          s_sum[k][threadIdx.x] = s_sum[k][threadIdx.x + o];
          s_idx[k][threadIdx.x] = s_idx[k][threadIdx.x + o];
        }
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    for (int k = 0; k < radii.n; ++k) {
      block_best[((size_t)blockIdx.x * 8 + k) * 2] = s_sum[k][0];
      block_best[((size_t)blockIdx.x * 8 + k) * 2 + 1] = s_idx[k][0];
    }
    __threadfence();
    s_last = atomicAdd(done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last) return;
  // last block: parallel reduction (better() is a total order: the result is order-independent)
  for (int k = 0; k < radii.n; ++k) {
    unsigned long long s = 0, i = ~0ull;
    for (unsigned b = threadIdx.x; b < gridDim.x; b += blockDim.x) {
      const unsigned long long cs = __ldcg(block_best + ((size_t)b * 8 + k) * 2);
      const unsigned long long ci = __ldcg(block_best + ((size_t)b * 8 + k) * 2 + 1);
      if (better(cs, ci, s, i)) {
        s = cs;
        i = ci;
      }
    }
    __syncthreads();
    s_sum[k][threadIdx.x] = s;
    s_idx[k][threadIdx.x] = i;
  }
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o)
      for (int k = 0; k < radii.n; ++k)
        if (better(s_sum[k][threadIdx.x + o], s_idx[k][threadIdx.x + o], s_sum[k][threadIdx.x], s_idx[k][threadIdx.x])) {
          s_sum[k][threadIdx.x] = s_sum[k][threadIdx.x + o];
          s_idx[k][threadIdx.x] = s_idx[k][threadIdx.x + o];
        }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    for (int k = 0; k < radii.n; ++k) {
      out_best[2 * k] = s_sum[k][0];
      out_best[2 * k + 1] = s_idx[k][0];
    }
    *done = 0u;
  }
}

}  // namespace

int argmax_block_count() { return 296; }

void launch_argmax(const uint32_t* grid, int G, const Disk* disks, int n_disks, int r,
                   unsigned long long* block_keys, unsigned long long* out_key, unsigned int* done,
                   cudaStream_t s, const uint32_t* mask) {
  DiskSet d;
  d.n = mask ? 0 : (n_disks < kMaxDisks ? n_disks : kMaxDisks);
  d.r = r;
  d.r2 = r * r;
  for (int k = 0; k < d.n; ++k) {
    d.cx[k] = disks[k].cx;
    d.cy[k] = disks[k].cy;
  }
  argmax_kernel<<<argmax_block_count(), kArgThreads, 0, s>>>(grid, G, d, mask, block_keys, out_key, done);
}

int max_direct_disks() { return kMaxDisks; }

void launch_mark_disks(uint32_t* mask, int G, const Disk* disks, int n_disks, int r, cudaStream_t s) {
  for (int off = 0; off < n_disks; off += kMaxDisks) {
    DiskSet d;
    d.n = n_disks - off < kMaxDisks ? n_disks - off : kMaxDisks;
    d.r = r;
    d.r2 = r * r;
    for (int k = 0; k < d.n; ++k) {
      d.cx[k] = disks[off + k].cx;
      d.cy[k] = disks[off + k].cy;
    }
    const int cells = (2 * r + 1) * (2 * r + 1);
    mark_disks_kernel<<<dim3((unsigned)((cells + 255) / 256), (unsigned)d.n), 256, 0, s>>>(mask, G, d);
  }
}

int blur_block_count() { return 148; }

void launch_blur_argmax(const uint32_t* grid, int G, const int* radii, int n_radii, unsigned long long* sat,
                        unsigned long long* block_best, unsigned long long* out_best, unsigned int* done,
                        cudaStream_t s) {
  const int t = G >= 1024 ? 1024 : (G >= 256 ? 256 : 32);
  sat_rows_kernel<<<G, t, 0, s>>>(grid, G, sat);
  sat_cols_kernel<<<(G + 1 + kSatCols - 1) / kSatCols, kSatCols * kSatSeg, 0, s>>>(G, sat);
  Radii rr;
  rr.n = n_radii < 8 ? n_radii : 8;
  for (int k = 0; k < rr.n; ++k) rr.r[k] = radii[k];
  blur_box_kernel<<<blur_block_count(), 256, 0, s>>>(sat, G, rr, block_best, out_best, done);
}

}  // namespace rvb
