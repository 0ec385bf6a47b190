// K4': device-resident refine_loop / anneal_axis (estimator.cpp:51-69, :145-160) as ONE
// cooperative kernel per call. Each pass is the strict classify of the constraint set (reference
// op order, bitmask via ballot) fused with the 6 scatter sums of the same inliers. The blocks then
// exchange their 8 partials through per-block 128-byte lines with release/acquire sequence numbers
// (publish_line / load_seq: no arrival counter), EVERY block reduces all lines in the same fixed
// order and runs the same short-latency 3x3 eigen-solve (axis_from_scatter_fast, rv_linalg.hpp,
// warm-started from the previous pass), so all blocks reach the same decision with no second
// exchange; block 0 publishes the state for the host. No host round trip per pass.
//
// Blocks own fixed contiguous tile ranges across passes: their slice of z and the pass's flag
// words stay in shared memory; only the final set is written to flags0.
#include <cuda_runtime.h>

#include <cstdint>
#include <mutex>

#include "rv_exact.cuh"
#include "rv_internal.h"
#include "rv_linalg.hpp"

namespace rvb {
namespace {

constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;
constexpr int kTile = 1024;                  // compaction granularity (compact_kernel): 32 flag words
constexpr int kPerTile = kTile / kThreads;   // elements per thread per tile
constexpr int kChunk = 2;                    // tiles whose loads are issued together
constexpr int kMaxDev = 8;                   // devices of a cross-device exchange

using State = CoopState;

#ifdef RV_COOP_TRACE  // dev instrumentation: block 0's phase timestamps (globaltimer, ns)
__device__ unsigned long long g_trace[8192];
__device__ unsigned int g_trace_n;
__device__ __forceinline__ void trace(int tag) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    const unsigned k = atomicAdd(&g_trace_n, 1u);
    if (k < 8192) g_trace[k] = (t << 4) | (unsigned long long)tag;
  }
}
#else
__device__ __forceinline__ void trace(int) {}
#endif

struct CoopArgs {
  const double* zx;
  const double* zy;
  const double* zz;
  int64_t n;
  int mode;    // 0 refine_loop, 1 anneal_axis
  int refine;  // cfg.refine
  double eps;
  double e0;
  double axis0[3];
  const double* axis0_dev;  // optional: start axis on the device (PeakOut.axis)
  uint32_t* flags0;
  uint32_t* flags1;
  int32_t* tile_count;
  int32_t* tile_offset;
  double* block_part;       // [grid][kLine]: the blocks' partial lines (zeroed once before first use)
  unsigned int* barrier;    // [2] launch epoch / exit counter (zeroed once; the last block out advances the epoch)
  State* state;
  // optional (refine_loop): compaction of the final set fused into the last pass
  const int32_t* kept;      // kept -> input index map (null: identity)
  int32_t* compact_out;     // inlier input indices in order (null: only tile offsets)
  uint32_t* zero_bins;      // angle histogram to clear for the angle vote that follows
  int n_bins;
  unsigned long long* zero_counts;  // [2]
  // > 0: the block's constraint slice stays resident in shared memory after the first pass
  // (SoA, z_cap elements per coordinate); later passes classify from there
  int z_cap;
  int fw_cap;  // flag words per block (shared memory, two slots)
  // cross-device exchange (a shard of a multi-GPU solve; n_dev == 1: none). xlines[q] is device
  // q's buffer of kMaxDev lines; this device's total goes to line dev_rank of every buffer
  int n_dev, dev_rank;
  double* xlines[kMaxDev];
  unsigned long long xepoch;
};

__device__ __forceinline__ double warp_sum_d(double v) {
  for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xFFFFFFFFu, v, o));
  return v;
}

// Grid barrier on a monotonically increasing arrival counter (zeroed before the launch): arrive
// with a release-add, wait until the counter reaches this pass's target with acquire loads. No
// L1 invalidation is needed: the only cross-block data (block partials, tile counts) are read
// with ld.global.cg / atomics.
__device__ __forceinline__ void grid_barrier(unsigned int* bar, unsigned int target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
    unsigned int g;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(g) : "l"(bar) : "memory");
    } while (g < target);
  }
  __syncthreads();
}

// Warp sum of 8 values per lane by transpose-reduction: each round halves the values a lane
// carries (exchange 4, 2, 1, then two plain rounds), 9 double shuffles instead of 40. Lane l ends
// with the warp total of value (l >> 2) & 7 (the 4 lanes of a group agree: commutative adds).
__device__ __forceinline__ double warp_sum8(const double (&v)[8]) {
  const int lane = threadIdx.x & 31;
  const bool h16 = lane & 16, h8 = lane & 8, h4 = lane & 4;
  double a[4], b[2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
    a[i] = xa(h16 ? v[i + 4] : v[i], __shfl_xor_sync(0xFFFFFFFFu, h16 ? v[i] : v[i + 4], 16));
#pragma unroll
  for (int i = 0; i < 2; ++i)
    b[i] = xa(h8 ? a[i + 2] : a[i], __shfl_xor_sync(0xFFFFFFFFu, h8 ? a[i] : a[i + 2], 8));
  double c = xa(h4 ? b[1] : b[0], __shfl_xor_sync(0xFFFFFFFFu, h4 ? b[0] : b[1], 4));
  c = xa(c, __shfl_xor_sync(0xFFFFFFFFu, c, 2));
  return xa(c, __shfl_xor_sync(0xFFFFFFFFu, c, 1));
}
__device__ __forceinline__ void warp_bcast8(double r, double (&v)[8]) {  // lane 4k's r -> v[k]
#pragma unroll
  for (int k = 0; k < 8; ++k) v[k] = __shfl_sync(0xFFFFFFFFu, r, 4 * k);
}

// Fixed-shape block reduction of 8 per-thread values into warp 0 (returned in v there).
__device__ __forceinline__ void block_reduce8(double (&v)[8], double (*s_red)[kWarps]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double r = warp_sum8(v);
  if ((lane & 3) == 0) s_red[lane >> 2][warp] = r;
  __syncthreads();
  if (warp == 0) {
    double x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = lane < kWarps ? s_red[k][lane] : 0.0;
    warp_bcast8(warp_sum8(x), v);
  }
}

// Per-pass exchange without a grid barrier: every block publishes its 8 partials and then a
// sequence number (release) in its own 128-byte line; every block's warp 0 polls the sequence
// numbers of all blocks (acquire) and then all blocks reduce the partials in the same fixed order.
// One L2 round trip after the last block's release, no same-address arrival counter, and the
// release only has to drain this block's 64 bytes (the pass's flag words stay in shared memory).
// Sequence numbers are (launch epoch << 20) | pass; the last block to exit advances the epoch, so
// the lines never need clearing (graph replays included).
constexpr int kLine = 16;  // doubles per block line: 8 partials, the sequence number, padding
__device__ __forceinline__ void publish_line(double* line, const double v[8], unsigned long long seq) {
  for (int k = 0; k < 8; ++k) __stcg(line + k, v[k]);
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(line + 8), "l"(seq) : "memory");
}
__device__ __forceinline__ unsigned long long load_seq(const double* line) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(line + 8) : "memory");
  return v;
}

__global__ void __launch_bounds__(kThreads) coop_refine_kernel(CoopArgs a) {
  extern __shared__ double s_z[];  // [3][z_cap] z (a.z_cap > 0), then [2][fw_cap] flag words
  __shared__ double s_red[8][kWarps];
  __shared__ double s_next[4];  // next axis (3) + next e
  __shared__ int s_done;
  __shared__ unsigned int s_epoch;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t ntiles = (a.n + kTile - 1) / kTile;
  const int64_t t_begin = ntiles * blockIdx.x / gridDim.x, t_end = ntiles * (blockIdx.x + 1) / gridDim.x;
  const int64_t w_begin = t_begin * (kTile / 32);
  const int64_t w_end = min(t_end * (kTile / 32), (a.n + 31) / 32);  // this block's flag words
  uint32_t* s_flags = reinterpret_cast<uint32_t*>(s_z + 3 * (size_t)a.z_cap);  // [2][fw_cap]
  double cls_axis[3] = {a.axis0[0], a.axis0[1], a.axis0[2]};
  if (a.axis0_dev) {
    cls_axis[0] = a.axis0_dev[0];
    cls_axis[1] = a.axis0_dev[1];
    cls_axis[2] = a.axis0_dev[2];
  }
  if (tid == 0) s_epoch = __ldcg(a.barrier);
  __syncthreads();
  const unsigned long long epoch = (unsigned long long)s_epoch << 20;
  double e = a.mode == 1 ? (a.e0 > a.eps ? a.e0 : a.eps) : a.eps;
  int slot = 0, refits = 0, pass = 0;
  double l3 = 0.0;  // Newton warm start of the 3x3 solve across passes (thread 0)
  long long local_count = 0;  // this device's inliers of the last classify (warp 0)
  int xtimeout = 0;           // cross-device exchange timed out (warp 0)
  bool have_prev = false;
  bool first_pass = true;
  const int64_t e_begin = t_begin * kTile;
  const int64_t cap = a.z_cap;
  double tot[8];
  for (;;) {
    // ---- classify pass over this block's tiles ----
    trace(1);
    uint32_t* flags = s_flags + (size_t)slot * a.fw_cap;
    const uint32_t* prev = s_flags + (size_t)(slot ^ 1) * a.fw_cap;
    double v[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // scatter[6], diff, count
    int diff = 0, cnt = 0;
    for (int64_t t0 = t_begin; t0 < t_end; t0 += kChunk) {
      double z[kChunk][kPerTile][3];
#pragma unroll
      for (int c = 0; c < kChunk; ++c)  // all loads of the chunk first
#pragma unroll
        for (int r = 0; r < kPerTile; ++r) {
          const int64_t i = (t0 + c) * kTile + r * kThreads + tid;
          const bool ok = t0 + c < t_end && i < a.n;
          const int64_t li = i - e_begin;  // the same thread owns element i in every pass
          if (cap > 0 && !first_pass) {
            z[c][r][0] = ok ? s_z[li] : 0.0;
            z[c][r][1] = ok ? s_z[cap + li] : 0.0;
            z[c][r][2] = ok ? s_z[2 * cap + li] : 0.0;
          } else {
            z[c][r][0] = ok ? a.zx[i] : 0.0;
            z[c][r][1] = ok ? a.zy[i] : 0.0;
            z[c][r][2] = ok ? a.zz[i] : 0.0;
            if (cap > 0 && ok) {
              s_z[li] = z[c][r][0];
              s_z[cap + li] = z[c][r][1];
              s_z[2 * cap + li] = z[c][r][2];
            }
          }
        }
#pragma unroll
      for (int c = 0; c < kChunk; ++c) {
        if (t0 + c >= t_end) break;  // uniform
#pragma unroll
        for (int r = 0; r < kPerTile; ++r) {
          const int64_t i = (t0 + c) * kTile + r * kThreads + tid;
          const double z0 = z[c][r][0], z1 = z[c][r][1], z2 = z[c][r][2];
          bool in = false;
          if (i < a.n) {
            const double d = xa(xa(xm(cls_axis[0], z0), xm(cls_axis[1], z1)), xm(cls_axis[2], z2));
            in = fabs(d) < e;
          }
          const unsigned word = __ballot_sync(0xFFFFFFFFu, in);
          const int64_t w0 = (t0 + c) * kTile + r * kThreads + warp * 32;
          if (lane == 0 && w0 < a.n) {
            const int64_t lw = (w0 >> 5) - w_begin;
            if (have_prev && prev[lw] != word) diff = 1;
            flags[lw] = word;
          }
          if (in) {
            ++cnt;
            v[0] = xa(v[0], xm(z0, z0));
            v[1] = xa(v[1], xm(z0, z1));
            v[2] = xa(v[2], xm(z0, z2));
            v[3] = xa(v[3], xm(z1, z1));
            v[4] = xa(v[4], xm(z1, z2));
            v[5] = xa(v[5], xm(z2, z2));
          }
        }
      }
    }
    v[6] = (double)__any_sync(0xFFFFFFFFu, diff);  // reduced as a sum: > 0 <=> any block word differs
    v[7] = (double)cnt;
    trace(2);
    block_reduce8(v, s_red);
    const unsigned long long seq = epoch | (unsigned long long)(pass + 1);
    if (tid == 0) publish_line(a.block_part + (size_t)blockIdx.x * kLine, v, seq);
    trace(3);
    // ---- warp 0: wait for every block's line of this pass, reading its partials as it lands;
    // the same fixed order in every block (lane-strided over the lines, then the tree) ----
    if (warp == 0) {
      const unsigned nl = (gridDim.x + 31) / 32;  // lines per lane
      for (;;) {  // every line of this pass seen (all polls of a round issued together)
        bool ok = true;
        for (unsigned j = 0; j < nl; ++j) {
          const unsigned b = lane + 32 * j;
          if (b < gridDim.x) ok &= load_seq(a.block_part + (size_t)b * kLine) >= seq;
        }
        if (__all_sync(0xFFFFFFFFu, ok)) break;
      }
      double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      for (unsigned j0 = 0; j0 < nl; j0 += 4) {  // 4 lines x 8 values in flight per lane
        double x[4][8];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const unsigned b = lane + 32 * (j0 + j);
          const bool in = j0 + j < nl && b < gridDim.x;
#pragma unroll
          for (int k = 0; k < 8; ++k) x[j][k] = in ? __ldcg(a.block_part + (size_t)b * kLine + k) : 0.0;
        }
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
          for (int k = 0; k < 8; ++k) acc[k] = xa(acc[k], x[j][k]);
      }
      warp_bcast8(warp_sum8(acc), tot);
      local_count = (long long)tot[7];
      if (a.n_dev > 1) {
        // ---- cross-device: block 0 writes this device's total (identical in every block) to line
        // dev_rank of every device's buffer over NVLink (data, then the sequence number with
        // release at system scope); every block's warp 0 polls its own buffer for all devices'
        // lines (acquire) and sums them in RANK order -- the same totals on every device
        const unsigned long long xs = (a.xepoch << 20) | (unsigned long long)(pass + 1);
        if (blockIdx.x == 0 && lane == 0)
          for (int q = 0; q < a.n_dev; ++q) {
            double* line = a.xlines[q] + (size_t)a.dev_rank * kLine;
            for (int k = 0; k < 8; ++k) __stcg(line + k, tot[k]);
            asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(line + 8), "l"(xs) : "memory");
          }
        const double* mine = a.xlines[a.dev_rank] + (size_t)lane * kLine;
        double xv[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        unsigned long long t_start;
        asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t_start));
        for (;;) {
          bool ok = true;
          if (lane < a.n_dev) {
            unsigned long long v;
            asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(mine + 8) : "memory");
            ok = v >= xs;
          }
          if (__all_sync(0xFFFFFFFFu, ok)) break;
          unsigned long long t_now;
          asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t_now));
          if (t_now - t_start > 5000000000ull) {  // a peer never arrived: fail instead of hanging
            xtimeout = 1;
            break;
          }
        }
        if (lane < a.n_dev && !xtimeout)
          for (int k = 0; k < 8; ++k) asm volatile("ld.relaxed.sys.global.f64 %0, [%1];" : "=d"(xv[k]) : "l"(mine + k) : "memory");
        for (int k = 0; k < 8; ++k) {
          double g = 0.0;
          for (int r = 0; r < a.n_dev; ++r) g = xa(g, __shfl_sync(0xFFFFFFFFu, xv[k], r));
          tot[k] = g;
        }
      }
    }
    trace(4);
    trace(5);
    if (tid == 0) {
      const long long count = (long long)tot[7];
      const bool differs = tot[6] != 0.0;
      int done = xtimeout, rank_deficient = 0;  // a failed cross-device exchange stops the loop
      double cur[3] = {cls_axis[0], cls_axis[1], cls_axis[2]};  // the set just classified is current
      double nxt[3] = {cls_axis[0], cls_axis[1], cls_axis[2]};
      double e_next = e;
      if (done) {
      } else if (a.mode == 0) {  // refine_loop (estimator.cpp:51-69)
        if (!have_prev && !a.refine) done = 1;
        if (have_prev && !differs) done = 1;  // stable
        if (!done && (refits >= 10 || count < 2)) done = 1;
        if (!done) {
          if (axis_from_scatter_fast(tot, nxt, &l3)) {
            ++refits;
          } else {
            rank_deficient = 1;  // RankDeficient: keep the current axis
            done = 1;
          }
        }
      } else {  // anneal_axis (estimator.cpp:145-160)
        if (count >= 2 && axis_from_scatter_fast(tot, nxt, &l3)) {
          cur[0] = nxt[0];
          cur[1] = nxt[1];
          cur[2] = nxt[2];
        }
        nxt[0] = cur[0];
        nxt[1] = cur[1];
        nxt[2] = cur[2];
        if (e <= a.eps) done = 1;
        const double h = 0.5 * e;
        e_next = a.eps > h ? a.eps : h;
      }
      if (blockIdx.x == 0) {  // publish (host reads it once at the end)
        State* st = a.state;
        for (int k = 0; k < 3; ++k) {
          st->axis[k] = cur[k];
          st->next[k] = nxt[k];
        }
        for (int k = 0; k < 6; ++k) st->scatter[k] = tot[k];
        st->e = e_next;
        st->count = count;
        st->slot = 0;
        st->done = done;
        st->refits = refits;
        st->rank_deficient = rank_deficient;
        st->local_count = local_count;
        st->exchange_timeout = xtimeout;
      }
      for (int k = 0; k < 3; ++k) s_next[k] = nxt[k];
      s_next[3] = e_next;
      s_done = done;
    }
    __syncthreads();
    trace(6);
    const int done = s_done;
    if (done) {
      if (a.mode == 0) {
        // the final set (this pass's words) into flags0; this block's position = the inliers of the
        // blocks before it (their counts, from their lines of this pass)
        for (int64_t w = w_begin + tid; w < w_end; w += kThreads) a.flags0[w] = flags[w - w_begin];
        __shared__ long long s_pre[kWarps];
        long long pre = 0;
        for (unsigned b = tid; b < blockIdx.x; b += kThreads)
          pre += (long long)__ldcg(a.block_part + (size_t)b * kLine + 7);
        for (int o = 16; o > 0; o >>= 1) pre += __shfl_xor_sync(0xFFFFFFFFu, pre, o);
        if (lane == 0) s_pre[warp] = pre;
        __syncthreads();
        long long off = 0;
        for (int w = 0; w < kWarps; ++w) off += s_pre[w];
        trace(7);
        if (a.compact_out) {
          // fused compaction: all own flag words at once, block-wide exclusive popc scan, then
          // each thread writes its own word's set bits
          __shared__ int s_wsum[kWarps];
          for (int64_t c0 = w_begin; c0 < w_end; c0 += kThreads) {  // chunks of kThreads words
            const int64_t wi = c0 + tid;
            const uint32_t word = wi < w_end ? flags[wi - w_begin] : 0u;
            const int cw = __popc(word);
            int incl = cw;
            for (int o = 1; o < 32; o <<= 1) {
              const int y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
              if (lane >= o) incl += y;
            }
            if (lane == 31) s_wsum[warp] = incl;
            __syncthreads();
            int wpre = 0, ctot = 0;
            for (int w = 0; w < kWarps; ++w) {
              wpre += w < warp ? s_wsum[w] : 0;
              ctot += s_wsum[w];
            }
            uint32_t m = word;
            long long pos = off + wpre + (incl - cw);
            while (m) {
              const int bit = __ffs(m) - 1;
              m &= m - 1u;
              const int64_t i = wi * 32 + bit;
              a.compact_out[pos++] = a.kept ? __ldg(a.kept + i) : (int32_t)i;
            }
            off += ctot;
            __syncthreads();
          }
          if (blockIdx.x == 0) {
            for (int k = tid; k < a.n_bins; k += kThreads) a.zero_bins[k] = 0u;
            if (tid < 2 && a.zero_counts) a.zero_counts[tid] = 0ull;
          }
        } else if (warp == 0) {
          // compaction offsets of the final set (tile order): block offset + own tiles' prefix
          long long run = off;
          for (int64_t t0 = t_begin; t0 < t_end; t0 += 32) {
            const int64_t t = t0 + lane;
            int c = 0;
            if (t < t_end)
              for (int w = 0; w < kTile / 32; ++w) {
                const int64_t gw = t * (kTile / 32) + w;
                if (gw < w_end) c += __popc(flags[gw - w_begin]);
              }
            int x = c;
            for (int o = 1; o < 32; o <<= 1) {
              const int y = __shfl_up_sync(0xFFFFFFFFu, x, o);
              if (lane >= o) x += y;
            }
            if (t < t_end) a.tile_offset[t] = (int32_t)(run + x - c);
            run += __shfl_sync(0xFFFFFFFFu, x, 31);
          }
        }
      }
      trace(8);
      // exit: the last block out advances the epoch (the lines' sequence numbers of the next launch)
      __syncthreads();
      if (tid == 0) {
        __threadfence();
        if (atomicAdd(a.barrier + 1, 1u) == gridDim.x - 1) {
          a.barrier[1] = 0u;
          __threadfence();
          atomicAdd(a.barrier, 1u);
        }
      }
      break;
    }
    for (int k = 0; k < 3; ++k) cls_axis[k] = s_next[k];
    e = s_next[3];
    slot ^= 1;
    ++pass;
    have_prev = a.mode == 0;
    first_pass = false;
  }
}

// ---- K candidates at once ------------------------------------------------------------------
// refine_loop / anneal_axis of up to kMaxCand independent start axes (the rescue candidates of
// estimator.cpp:352-368 / 452-466, the anneals of rescue_axes) in ONE cooperative launch: each
// pass classifies the block's (shared-memory resident) constraints once per still-active
// candidate and exchanges ALL candidates' partials in one line per block, so the latency-bound
// per-pass exchange and decision are paid once per pass instead of once per candidate. Each
// candidate follows exactly the single-candidate loop (the same predicate, the same fixed-order
// sums, the same decisions); a candidate that is done is frozen with its final set.
constexpr int kMaxCand = 8;
struct CoopMultiArgs {
  const double* zx;
  const double* zy;
  const double* zz;
  int64_t n;
  int mode, refine, K;
  double eps;
  double axis0[kMaxCand][3];
  double e0[kMaxCand];
  State* state;                // state of candidate k at (char*)state + k * state_stride
  size_t state_stride;
  unsigned long long* counts;  // zeroed [2] at (char*)counts + k * state_stride (angle vote that follows)
  uint32_t* flags_out;         // mode 0: final bitmask of candidate k at flags_out + k * flag_stride
  size_t flag_stride;
  const int32_t* kept;
  int32_t* compact_out;        // mode 0: inlier indices of candidate k at compact_out + k * compact_stride
  size_t compact_stride;
  uint32_t* zero_bins;
  int n_bins;
  double* block_part;          // [grid][line]: line = 8 K partials + the sequence number
  unsigned int* barrier;
  int z_cap, fw_cap;
};

__global__ void __launch_bounds__(kThreads) coop_refine_multi_kernel(CoopMultiArgs a) {
  extern __shared__ double s_z[];  // [3][z_cap] z, then [K][2][fw_cap] flag words
  __shared__ double s_red[8][kWarps];
  __shared__ double s_val[kMaxCand][8];  // this block's partials of the pass
  __shared__ double s_redK[kMaxCand][8][kWarps];  // per-warp partials of every candidate
  __shared__ double s_tot[kMaxCand][8];  // all blocks' totals of the pass
  __shared__ double s_axis[kMaxCand][3], s_e[kMaxCand];
  __shared__ int s_done[kMaxCand], s_fslot[kMaxCand], s_all_done;
  __shared__ unsigned int s_epoch;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int K = a.K;
  const size_t line = (size_t)8 * K + 8;
  const int64_t ntiles = (a.n + kTile - 1) / kTile;
  const int64_t t_begin = ntiles * blockIdx.x / gridDim.x, t_end = ntiles * (blockIdx.x + 1) / gridDim.x;
  const int64_t w_begin = t_begin * (kTile / 32);
  const int64_t w_end = min(t_end * (kTile / 32), (a.n + 31) / 32);
  uint32_t* s_flags = reinterpret_cast<uint32_t*>(s_z + 3 * (size_t)a.z_cap);  // [K][2][fw_cap]
  if (tid == 0) s_epoch = __ldcg(a.barrier);
  if (tid < K) {
    for (int k = 0; k < 3; ++k) s_axis[tid][k] = a.axis0[tid][k];
    s_e[tid] = a.mode == 1 ? (a.e0[tid] > a.eps ? a.e0[tid] : a.eps) : a.eps;
    s_done[tid] = 0;
    s_fslot[tid] = 0;
  }
  __syncthreads();
  const unsigned long long epoch = (unsigned long long)s_epoch << 20;
  int slot = 0, pass = 0;
  bool have_prev = false, first_pass = true;
  int refits = 0;      // thread c < K: candidate c's
  double l3 = 0.0;     // thread c < K: candidate c's Newton warm start
  const int64_t e_begin = t_begin * kTile;
  const int64_t cap = a.z_cap;
  for (;;) {
    for (int c = 0; c < K; ++c) {
      if (s_done[c]) continue;  // uniform
      const double ax0 = s_axis[c][0], ax1 = s_axis[c][1], ax2 = s_axis[c][2], e = s_e[c];
      uint32_t* flags = s_flags + ((size_t)c * 2 + slot) * a.fw_cap;
      const uint32_t* prev = s_flags + ((size_t)c * 2 + (slot ^ 1)) * a.fw_cap;
      double v[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      int diff = 0, cnt = 0;
      const bool from_global = cap == 0 || first_pass;
      for (int64_t t0 = t_begin; t0 < t_end; t0 += kChunk) {
        double z[kChunk][kPerTile][3];
#pragma unroll
        for (int cc = 0; cc < kChunk; ++cc)
#pragma unroll
          for (int r = 0; r < kPerTile; ++r) {
            const int64_t i = (t0 + cc) * kTile + r * kThreads + tid;
            const bool ok = t0 + cc < t_end && i < a.n;
            const int64_t li = i - e_begin;  // the same thread owns element i in every pass
            if (!from_global) {
              z[cc][r][0] = ok ? s_z[li] : 0.0;
              z[cc][r][1] = ok ? s_z[cap + li] : 0.0;
              z[cc][r][2] = ok ? s_z[2 * cap + li] : 0.0;
            } else {
              z[cc][r][0] = ok ? a.zx[i] : 0.0;
              z[cc][r][1] = ok ? a.zy[i] : 0.0;
              z[cc][r][2] = ok ? a.zz[i] : 0.0;
              if (cap > 0 && ok) {
                s_z[li] = z[cc][r][0];
                s_z[cap + li] = z[cc][r][1];
                s_z[2 * cap + li] = z[cc][r][2];
              }
            }
          }
#pragma unroll
        for (int cc = 0; cc < kChunk; ++cc) {
          if (t0 + cc >= t_end) break;  // uniform
#pragma unroll
          for (int r = 0; r < kPerTile; ++r) {
            const int64_t i = (t0 + cc) * kTile + r * kThreads + tid;
            const double z0 = z[cc][r][0], z1 = z[cc][r][1], z2 = z[cc][r][2];
            bool in = false;
            if (i < a.n) {
              const double d = xa(xa(xm(ax0, z0), xm(ax1, z1)), xm(ax2, z2));
              in = fabs(d) < e;
            }
            const unsigned word = __ballot_sync(0xFFFFFFFFu, in);
            const int64_t w0 = (t0 + cc) * kTile + r * kThreads + warp * 32;
            if (lane == 0 && w0 < a.n) {
              const int64_t lw = (w0 >> 5) - w_begin;
              if (have_prev && prev[lw] != word) diff = 1;
              flags[lw] = word;
            }
            if (in) {
              ++cnt;
              v[0] = xa(v[0], xm(z0, z0));
              v[1] = xa(v[1], xm(z0, z1));
              v[2] = xa(v[2], xm(z0, z2));
              v[3] = xa(v[3], xm(z1, z1));
              v[4] = xa(v[4], xm(z1, z2));
              v[5] = xa(v[5], xm(z2, z2));
            }
          }
        }
      }
      first_pass = false;  // z is now in shared memory (each thread reads back its own elements)
      v[6] = (double)__any_sync(0xFFFFFFFFu, diff);
      v[7] = (double)cnt;
      // block_reduce8's first half (warp sums into this candidate's slot); the cross-warp half runs
      // for every candidate after ONE barrier below (the same fixed order)
      const double r8 = warp_sum8(v);
      if ((lane & 3) == 0) s_redK[c][lane >> 2][warp] = r8;
    }
    __syncthreads();
    if (warp == 0)
      for (int c = 0; c < K; ++c) {
        if (s_done[c]) continue;  // uniform
        double x[8], t[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = lane < kWarps ? s_redK[c][k][lane] : 0.0;
        warp_bcast8(warp_sum8(x), t);
        if (lane == 0)
          for (int k = 0; k < 8; ++k) s_val[c][k] = t[k];
      }
    const unsigned long long seq = epoch | (unsigned long long)(pass + 1);
    if (tid == 0) {
      double* ln = a.block_part + (size_t)blockIdx.x * line;
      for (int c = 0; c < K; ++c)
        if (!s_done[c])
          for (int k = 0; k < 8; ++k) __stcg(ln + 8 * c + k, s_val[c][k]);
      asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(ln + 8 * K), "l"(seq) : "memory");
    }
    if (warp == 0) {
      const unsigned nl = (gridDim.x + 31) / 32;
      for (;;) {
        bool ok = true;
        for (unsigned j = 0; j < nl; ++j) {
          const unsigned b = lane + 32 * j;
          if (b < gridDim.x) {
            unsigned long long v;
            asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(a.block_part + (size_t)b * line + 8 * K)
                         : "memory");
            ok &= v >= seq;
          }
        }
        if (__all_sync(0xFFFFFFFFu, ok)) break;
      }
      for (int c = 0; c < K; ++c) {
        if (s_done[c]) continue;  // uniform
        double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        for (unsigned j0 = 0; j0 < nl; j0 += 4) {  // 4 lines x 8 values in flight per lane (same order)
          double x[4][8];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const unsigned b = lane + 32 * (j0 + j);
            const bool in = j0 + j < nl && b < gridDim.x;
#pragma unroll
            for (int k = 0; k < 8; ++k) x[j][k] = in ? __ldcg(a.block_part + (size_t)b * line + 8 * c + k) : 0.0;
          }
#pragma unroll
          for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int k = 0; k < 8; ++k) acc[k] = xa(acc[k], x[j][k]);
        }
        double t[8];
        warp_bcast8(warp_sum8(acc), t);
        if (lane == 0)
          for (int k = 0; k < 8; ++k) s_tot[c][k] = t[k];
      }
      __syncwarp();
      // lane c decides for candidate c (the single-candidate logic)
      if (lane < K && !s_done[lane]) {
        const int c = lane;
        const double* tot = s_tot[c];
        const long long count = (long long)tot[7];
        const bool differs = tot[6] != 0.0;
        int done = 0, rank_deficient = 0;
        const double e = s_e[c];
        double cur[3] = {s_axis[c][0], s_axis[c][1], s_axis[c][2]};
        double nxt[3] = {cur[0], cur[1], cur[2]};
        double e_next = e;
        if (a.mode == 0) {
          if (!have_prev && !a.refine) done = 1;
          if (have_prev && !differs) done = 1;
          if (!done && (refits >= 10 || count < 2)) done = 1;
          if (!done) {
            if (axis_from_scatter_fast(tot, nxt, &l3)) {
              ++refits;
            } else {
              rank_deficient = 1;
              done = 1;
            }
          }
        } else {
          if (count >= 2 && axis_from_scatter_fast(tot, nxt, &l3))
            for (int k = 0; k < 3; ++k) cur[k] = nxt[k];
          for (int k = 0; k < 3; ++k) nxt[k] = cur[k];
          if (e <= a.eps) done = 1;
          const double h = 0.5 * e;
          e_next = a.eps > h ? a.eps : h;
        }
        if (blockIdx.x == 0) {
          State* st = reinterpret_cast<State*>(reinterpret_cast<char*>(a.state) + (size_t)c * a.state_stride);
          for (int k = 0; k < 3; ++k) {
            st->axis[k] = cur[k];
            st->next[k] = nxt[k];
          }
          for (int k = 0; k < 6; ++k) st->scatter[k] = tot[k];
          st->e = e_next;
          st->count = count;
          st->slot = 0;
          st->done = done;
          st->refits = refits;
          st->rank_deficient = rank_deficient;
          st->local_count = count;
          st->exchange_timeout = 0;
        }
        for (int k = 0; k < 3; ++k) s_axis[c][k] = nxt[k];
        s_e[c] = e_next;
        if (done) {
          s_done[c] = 1;
          s_fslot[c] = slot;
        }
      }
      __syncwarp();
      if (lane == 0) {
        int all = 1;
        for (int c = 0; c < K; ++c) all &= s_done[c];
        s_all_done = all;
      }
    }
    __syncthreads();
    if (s_all_done) break;
    slot ^= 1;
    ++pass;
    have_prev = a.mode == 0;
  }
  if (a.mode == 0) {
    // per candidate: final set into its flags_out, fused compaction (this block's offset = the
    // candidate's inliers in the blocks before it, from their lines of the candidate's last pass)
    __shared__ long long s_pre[kWarps];
    __shared__ int s_wsum[kWarps];
    for (int c = 0; c < K; ++c) {
      const uint32_t* flags = s_flags + ((size_t)c * 2 + s_fslot[c]) * a.fw_cap;
      uint32_t* fo = a.flags_out ? a.flags_out + (size_t)c * a.flag_stride : nullptr;
      if (fo)
        for (int64_t w = w_begin + tid; w < w_end; w += kThreads) fo[w] = flags[w - w_begin];
      if (!a.compact_out) continue;
      long long pre = 0;
      for (unsigned b = tid; b < blockIdx.x; b += kThreads) pre += (long long)__ldcg(a.block_part + (size_t)b * line + 8 * c + 7);
      for (int o = 16; o > 0; o >>= 1) pre += __shfl_xor_sync(0xFFFFFFFFu, pre, o);
      if (lane == 0) s_pre[warp] = pre;
      __syncthreads();
      long long off = 0;
      for (int w = 0; w < kWarps; ++w) off += s_pre[w];
      int32_t* out = a.compact_out + (size_t)c * a.compact_stride;
      for (int64_t c0 = w_begin; c0 < w_end; c0 += kThreads) {
        const int64_t wi = c0 + tid;
        const uint32_t word = wi < w_end ? flags[wi - w_begin] : 0u;
        const int cw = __popc(word);
        int incl = cw;
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
          if (lane >= o) incl += y;
        }
        if (lane == 31) s_wsum[warp] = incl;
        __syncthreads();
        int wpre = 0, ctot = 0;
        for (int w = 0; w < kWarps; ++w) {
          wpre += w < warp ? s_wsum[w] : 0;
          ctot += s_wsum[w];
        }
        uint32_t m = word;
        long long pos = off + wpre + (incl - cw);
        while (m) {
          const int bit = __ffs(m) - 1;
          m &= m - 1u;
          const int64_t i = wi * 32 + bit;
          out[pos++] = a.kept ? __ldg(a.kept + i) : (int32_t)i;
        }
        off += ctot;
        __syncthreads();
      }
    }
    if (blockIdx.x == 0) {
      for (int k = tid; k < a.n_bins; k += kThreads) a.zero_bins[k] = 0u;
      if (a.counts)
        for (int c = 0; c < K; ++c)
          if (tid < 2)
            reinterpret_cast<unsigned long long*>(reinterpret_cast<char*>(a.counts) + (size_t)c * a.state_stride)[tid] = 0ull;
    }
  }
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    if (atomicAdd(a.barrier + 1, 1u) == gridDim.x - 1) {
      a.barrier[1] = 0u;
      __threadfence();
      atomicAdd(a.barrier, 1u);
    }
  }
}

// estimate_from_peak on the device (single thread): see exact_peak_axis (rv_exact.cuh).
__global__ void peak_axis_kernel(const unsigned long long* okey, const uint32_t* grid, int G, double E,
                                 uint32_t min_votes, PeakOut* out) {
  exact_peak_axis(okey[0], okey[1], grid, G, E, min_votes, out);
}

}  // namespace

void launch_peak_axis(const unsigned long long* okey, const uint32_t* grid, int G, double E, uint32_t min_votes,
                      PeakOut* out, cudaStream_t s) {
  peak_axis_kernel<<<1, 1, 0, s>>>(okey, grid, G, E, min_votes, out);
}

int coop_refine_grid(int sms) {
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, coop_refine_kernel, kThreads, 0);
  if (per_sm < 1) per_sm = 1;
  return sms * (per_sm < 2 ? per_sm : 2);
}

int coop_tiles(int64_t n) { return (int)((n + kTile - 1) / kTile); }

cudaError_t launch_coop_refine(const double* zx, const double* zy, const double* zz, int64_t n, int mode, int refine,
                               double eps, double e0, const double axis0[3], const double* axis0_dev,
                               uint32_t* flags0, uint32_t* flags1, int32_t* tile_count, int32_t* tile_offset,
                               double* block_part, unsigned int* barrier, void* state, int grid, cudaStream_t s,
                               const int32_t* kept, int32_t* compact_out, uint32_t* zero_bins, int n_bins,
                               unsigned long long* zero_counts, const CoopExchange* xch) {
  CoopArgs a;
  a.n_dev = xch ? xch->n_dev : 1;
  a.dev_rank = xch ? xch->rank : 0;
  for (int q = 0; q < kMaxDev; ++q) a.xlines[q] = xch ? xch->lines[q] : nullptr;
  a.xepoch = xch ? xch->epoch : 0ull;
  static_assert(kMaxDev == kCoopMaxDev, "device count");
  a.zx = zx;
  a.zy = zy;
  a.zz = zz;
  a.n = n;
  a.mode = mode;
  a.refine = refine;
  a.eps = eps;
  a.e0 = e0;
  for (int k = 0; k < 3; ++k) a.axis0[k] = axis0 ? axis0[k] : 0.0;
  a.axis0_dev = axis0_dev;
  a.flags0 = flags0;
  a.flags1 = flags1;
  a.tile_count = tile_count;
  a.tile_offset = tile_offset;
  a.block_part = block_part;
  a.barrier = barrier;
  a.state = static_cast<State*>(state);
  a.kept = kept;
  a.compact_out = compact_out;
  a.zero_bins = zero_bins;
  a.n_bins = n_bins;
  a.zero_counts = zero_counts;
  const int64_t ntiles = (n + kTile - 1) / kTile;
  if (grid > ntiles) grid = (int)(ntiles > 0 ? ntiles : 1);  // every block owns >= 1 tile
  // keep each block's slice of z in shared memory across the passes when it fits (N <= ~1.1M
  // at 148 blocks); the block count (one per SM) is unchanged by the shared memory it takes
  static int smem_max = [] {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    return v;
  }();
  const int64_t per_block = (ntiles + grid - 1) / grid * kTile;
  static const size_t static_bytes = [] {
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, reinterpret_cast<const void*>(coop_refine_kernel));
    return fa.sharedSizeBytes + 1024;  // + the runtime's reserved shared memory per block
  }();
  a.fw_cap = (int)(per_block / 32);
  const size_t flag_bytes = (size_t)2 * a.fw_cap * sizeof(uint32_t);
  size_t dyn = (size_t)(3 * per_block) * sizeof(double) + flag_bytes;
  a.z_cap = (int)per_block;
  if (mode != 0 && mode != 1) a.z_cap = 0;
  if (dyn + static_bytes > (size_t)smem_max) {
    a.z_cap = 0;
    dyn = flag_bytes;
  }
  if (dyn + static_bytes > (size_t)smem_max) return cudaErrorInvalidValue;  // > ~200M constraints
  if (dyn > 0) {
    static std::mutex mu;
    static size_t configured[16] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(mu);
    if (dev < 0 || dev >= 16 || configured[dev] < dyn) {
      const cudaError_t e = cudaFuncSetAttribute(reinterpret_cast<const void*>(coop_refine_kernel),
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
      if (e != cudaSuccess) return e;
      if (dev >= 0 && dev < 16) configured[dev] = dyn;
    }
  }
  void* args[] = {&a};
  // cooperative launch: guarantees co-residency of all blocks (required by the grid barrier)
  return cudaLaunchCooperativeKernel((void*)coop_refine_kernel, dim3(grid), dim3(kThreads), args, dyn, s);
}

cudaError_t launch_coop_refine_multi(const double* zx, const double* zy, const double* zz, int64_t n, int mode,
                                     int refine, double eps, int K, const double (*axes)[3], const double* e0s,
                                     void* state, size_t state_stride, unsigned long long* counts, uint32_t* flags_out,
                                     size_t flag_stride, const int32_t* kept, int32_t* compact_out, size_t compact_stride,
                                     uint32_t* zero_bins, int n_bins, double* block_part, unsigned int* barrier,
                                     int grid, cudaStream_t s) {
  if (K < 1 || K > kMaxCand) return cudaErrorInvalidValue;
  CoopMultiArgs a;
  a.zx = zx;
  a.zy = zy;
  a.zz = zz;
  a.n = n;
  a.mode = mode;
  a.refine = refine;
  a.K = K;
  a.eps = eps;
  for (int c = 0; c < kMaxCand; ++c) {
    for (int k = 0; k < 3; ++k) a.axis0[c][k] = c < K ? axes[c][k] : 0.0;
    a.e0[c] = c < K && e0s ? e0s[c] : 0.0;
  }
  a.state = static_cast<State*>(state);
  a.state_stride = state_stride;
  a.counts = counts;
  a.flags_out = flags_out;
  a.flag_stride = flag_stride;
  a.kept = kept;
  a.compact_out = compact_out;
  a.compact_stride = compact_stride;
  a.zero_bins = zero_bins;
  a.n_bins = n_bins;
  a.block_part = block_part;
  a.barrier = barrier;
  const int64_t ntiles = (n + kTile - 1) / kTile;
  if (grid > ntiles) grid = (int)(ntiles > 0 ? ntiles : 1);
  static int smem_max = [] {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    return v;
  }();
  static const size_t static_bytes = [] {
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, reinterpret_cast<const void*>(coop_refine_multi_kernel));
    return fa.sharedSizeBytes + 1024;
  }();
  const int64_t per_block = (ntiles + grid - 1) / grid * kTile;
  a.fw_cap = (int)(per_block / 32);
  const size_t flag_bytes = (size_t)K * 2 * a.fw_cap * sizeof(uint32_t);
  size_t dyn = (size_t)(3 * per_block) * sizeof(double) + flag_bytes;
  a.z_cap = (int)per_block;
  if (dyn + static_bytes > (size_t)smem_max) {
    a.z_cap = 0;
    dyn = flag_bytes;
  }
  if (dyn + static_bytes > (size_t)smem_max) return cudaErrorInvalidValue;
  {
    static std::mutex mu;
    static size_t configured[16] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(mu);
    if (dev < 0 || dev >= 16 || configured[dev] < dyn) {
      const cudaError_t e = cudaFuncSetAttribute(reinterpret_cast<const void*>(coop_refine_multi_kernel),
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
      if (e != cudaSuccess) return e;
      if (dev >= 0 && dev < 16) configured[dev] = dyn;
    }
  }
  void* args[] = {&a};
  return cudaLaunchCooperativeKernel((void*)coop_refine_multi_kernel, dim3(grid), dim3(kThreads), args, dyn, s);
}

int coop_multi_max() { return kMaxCand; }

size_t coop_state_bytes() { return sizeof(State); }

}  // namespace rvb

#ifdef RV_COOP_TRACE
extern "C" int rv_debug_coop_trace(unsigned long long* out, int max) {
  unsigned int n = 0;
  cudaMemcpyFromSymbol(&n, rvb::g_trace_n, sizeof n);
  if (n > 8192) n = 8192;
  if ((int)n > max) n = (unsigned)max;
  cudaMemcpyFromSymbol(out, rvb::g_trace, sizeof(unsigned long long) * n);
  const unsigned int zero = 0;
  cudaMemcpyToSymbol(rvb::g_trace_n, &zero, sizeof zero);
  return (int)n;
}
#endif

namespace rvb {

}  // namespace rvb
