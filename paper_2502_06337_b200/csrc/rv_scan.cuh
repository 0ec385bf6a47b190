// Single-pass order-preserving compaction support: decoupled look-back over dynamically
// numbered blocks (a block's predecessors were scheduled before it, so the spin terminates).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace rvb {

enum : unsigned long long {
  kLbFlagAgg = 1ull << 62,
  kLbFlagInc = 2ull << 62,
  kLbValMask = (1ull << 62) - 1
};

// Called by ALL threads of warp 0. Publishes `total` for block `bid` and returns the sum of the
// totals of blocks [0, bid). status[] must be zero-initialised before the launch.
__device__ __forceinline__ long long lookback_exclusive(unsigned long long* status, int bid, long long total) {
  const int lane = threadIdx.x & 31;
  volatile unsigned long long* st = status;
  if (bid == 0) {
    if (lane == 0) st[0] = kLbFlagInc | (unsigned long long)total;
    return 0;
  }
  if (lane == 0) st[bid] = kLbFlagAgg | (unsigned long long)total;
  long long excl = 0;
  int j = bid - 1;
  for (;;) {
    const int idx = j - lane;
    const unsigned long long v = idx >= 0 ? st[idx] : kLbFlagInc;
    const unsigned long long flag = v & ~kLbValMask;
    if (__any_sync(0xFFFFFFFFu, flag == 0ull)) continue;
    const unsigned inc = __ballot_sync(0xFFFFFFFFu, flag == kLbFlagInc);
    const int first = inc ? __ffs(inc) - 1 : 32;
    long long val = lane <= first ? (long long)(v & kLbValMask) : 0;
    for (int o = 16; o > 0; o >>= 1) val += __shfl_xor_sync(0xFFFFFFFFu, val, o);
    excl += val;
    if (inc) break;
    j -= 32;
  }
  if (lane == 0) st[bid] = kLbFlagInc | (unsigned long long)(excl + total);
  return excl;
}

}  // namespace rvb
