// K4': device-resident refine_loop / anneal_axis (estimator.cpp:51-69, :145-160) as ONE
// cooperative kernel per call. Each pass is the strict classify of the constraint set (reference
// op order, bitmask via ballot) fused with the 6 scatter sums of the same inliers; after a grid
// barrier block 0 reduces the block partials in a fixed order, runs the 3x3 eigen-solve
// (rv_linalg.hpp, the Eigen 3.4 restatement -- compiled here with -fmad=false so it is
// bit-identical to the host instantiation), decides the next step and publishes it; a second
// barrier hands the new axis to every block. No host round trip per pass.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "rv_exact.cuh"
#include "rv_internal.h"
#include "rv_linalg.hpp"

namespace cg = cooperative_groups;

namespace rvb {
namespace {

constexpr int kThreads = 256;
constexpr int kPerThread = 4;
constexpr int kTile = kThreads * kPerThread;  // 1024 constraints = 32 flag words per tile

using State = CoopState;

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
  uint32_t* flags0;
  uint32_t* flags1;
  int32_t* tile_count;
  int32_t* tile_offset;
  double* block_part;  // [grid][8]
  State* state;
};

__device__ __forceinline__ double warp_sum_d(double v) {
  for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xFFFFFFFFu, v, o));
  return v;
}

__global__ void __launch_bounds__(kThreads) coop_refine_kernel(CoopArgs a) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double s_red[8][kThreads / 32];
  __shared__ long long s_tot[kThreads];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t ntiles = (a.n + kTile - 1) / kTile;
  double cls_axis[3] = {a.axis0[0], a.axis0[1], a.axis0[2]};
  double e = a.mode == 1 ? (a.e0 > a.eps ? a.e0 : a.eps) : a.eps;
  int slot = 0;
  bool have_prev = false;
  for (;;) {
    // ---- classify pass (grid-stride over 1024-constraint tiles) ----
    uint32_t* flags = slot == 0 ? a.flags0 : a.flags1;
    const uint32_t* prev = have_prev ? (slot == 0 ? a.flags1 : a.flags0) : nullptr;
    double sc[6] = {0, 0, 0, 0, 0, 0};
    long long cnt = 0;
    int diff = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
      const int64_t base = t * kTile;
      int tcnt = 0;
#pragma unroll
      for (int r = 0; r < kPerThread; ++r) {
        const int64_t i = base + r * kThreads + tid;
        bool in = false;
        double z0 = 0, z1 = 0, z2 = 0;
        if (i < a.n) {
          z0 = a.zx[i];
          z1 = a.zy[i];
          z2 = a.zz[i];
          const double d = xa(xa(xm(cls_axis[0], z0), xm(cls_axis[1], z1)), xm(cls_axis[2], z2));
          in = fabs(d) < e;
        }
        const unsigned word = __ballot_sync(0xFFFFFFFFu, in);
        const int64_t w0 = base + r * kThreads + warp * 32;
        if (lane == 0 && w0 < a.n) {
          flags[w0 >> 5] = word;
          if (prev && prev[w0 >> 5] != word) diff = 1;
        }
        tcnt += __popc(word);
        if (in) {
          sc[0] = xa(sc[0], xm(z0, z0));
          sc[1] = xa(sc[1], xm(z0, z1));
          sc[2] = xa(sc[2], xm(z0, z2));
          sc[3] = xa(sc[3], xm(z1, z1));
          sc[4] = xa(sc[4], xm(z1, z2));
          sc[5] = xa(sc[5], xm(z2, z2));
        }
      }
      // per-tile count (each warp counted its words; sum the 8 warps of the tile)
      if (lane == 0) s_tot[warp] = tcnt;
      __syncthreads();
      if (tid == 0) {
        int c = 0;
        for (int w = 0; w < kThreads / 32; ++w) c += (int)s_tot[w];
        a.tile_count[t] = c;
        cnt += c;
      }
      __syncthreads();
    }
    // block partials: count (thread 0 holds it), diff, scatter (fixed-shape tree)
    diff = __any_sync(0xFFFFFFFFu, diff);
#pragma unroll
    for (int k = 0; k < 6; ++k) sc[k] = warp_sum_d(sc[k]);
    if (lane == 0) {
      for (int k = 0; k < 6; ++k) s_red[k][warp] = sc[k];
      s_red[6][warp] = (double)diff;
    }
    __syncthreads();
    if (tid == 0) {
      double* bp = a.block_part + (size_t)blockIdx.x * 8;
      for (int k = 0; k < 6; ++k) {
        double v = 0.0;
        for (int w = 0; w < kThreads / 32; ++w) v = xa(v, s_red[k][w]);
        bp[k] = v;
      }
      int d = 0;
      for (int w = 0; w < kThreads / 32; ++w) d |= s_red[6][w] != 0.0;
      bp[6] = (double)d;
      bp[7] = (double)cnt;
    }
    grid.sync();
    // ---- block 0: reduce (fixed order), decide, publish ----
    if (blockIdx.x == 0) {
      __shared__ int s_done;
      double v[6] = {0, 0, 0, 0, 0, 0};
      double vc = 0.0;
      int vd = 0;
      for (unsigned b = tid; b < gridDim.x; b += blockDim.x) {
        const double* bp = a.block_part + (size_t)b * 8;
        for (int k = 0; k < 6; ++k) v[k] = xa(v[k], __ldcg(bp + k));
        vd |= __ldcg(bp + 6) != 0.0;
        vc = xa(vc, __ldcg(bp + 7));
      }
      for (int k = 0; k < 6; ++k) v[k] = warp_sum_d(v[k]);
      vc = warp_sum_d(vc);
      vd = __any_sync(0xFFFFFFFFu, vd);
      if (lane == 0) {
        for (int k = 0; k < 6; ++k) s_red[k][warp] = v[k];
        s_red[6][warp] = (double)vd;
        s_red[7][warp] = vc;
      }
      __syncthreads();
      if (tid == 0) {
        double tot[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        for (int w = 0; w < kThreads / 32; ++w) {
          for (int k = 0; k < 6; ++k) tot[k] = xa(tot[k], s_red[k][w]);
          if (s_red[6][w] != 0.0) tot[6] = 1.0;
          tot[7] = xa(tot[7], s_red[7][w]);
        }
        State* st = a.state;
        const long long count = (long long)tot[7];
        const bool differs = tot[6] != 0.0;
        int done = 0;
        int refits = have_prev ? st->refits : 0;
        if (!have_prev) st->rank_deficient = 0;
        // the set just classified becomes the current one (estimator.cpp:63-65)
        for (int k = 0; k < 3; ++k) st->axis[k] = cls_axis[k];
        for (int k = 0; k < 6; ++k) st->scatter[k] = tot[k];
        st->count = count;
        st->slot = slot;
        double nxt[3] = {cls_axis[0], cls_axis[1], cls_axis[2]};
        if (a.mode == 0) {
          if (!have_prev && !a.refine) done = 1;
          if (have_prev && !differs) done = 1;  // stable
          if (!done && (refits >= 10 || count < 2)) done = 1;
          if (!done) {
            if (axis_from_scatter(tot, nxt)) {
              ++refits;
            } else {
              st->rank_deficient = 1;  // RankDeficient: keep the current axis
              done = 1;
            }
          }
        } else {  // anneal_axis
          double ax[3] = {cls_axis[0], cls_axis[1], cls_axis[2]};
          if (count >= 2 && axis_from_scatter(tot, nxt)) {
            ax[0] = nxt[0];
            ax[1] = nxt[1];
            ax[2] = nxt[2];
          }
          for (int k = 0; k < 3; ++k) {
            st->axis[k] = ax[k];
            nxt[k] = ax[k];
          }
          if (e <= a.eps) done = 1;
          const double h = 0.5 * e;
          st->e = a.eps > h ? a.eps : h;
        }
        for (int k = 0; k < 3; ++k) st->next[k] = nxt[k];
        st->refits = refits;
        st->done = done;
        s_done = done;
      }
      __syncthreads();
      if (s_done && a.mode == 0) {  // compaction offsets of the final set (tile order), block-parallel
        const int64_t per = (ntiles + kThreads - 1) / kThreads;
        const int64_t t0 = tid * per, t1 = t0 + per < ntiles ? t0 + per : ntiles;
        long long acc = 0;
        for (int64_t t = t0; t < t1; ++t) acc += __ldcg(a.tile_count + t);
        s_tot[tid] = acc;
        __syncthreads();
        if (tid == 0) {
          long long run = 0;
          for (int k = 0; k < kThreads; ++k) {
            const long long x = s_tot[k];
            s_tot[k] = run;
            run += x;
          }
        }
        __syncthreads();
        long long off = s_tot[tid];
        for (int64_t t = t0; t < t1; ++t) {
          a.tile_offset[t] = (int32_t)off;
          off += __ldcg(a.tile_count + t);
        }
      }
      __threadfence();
    }
    grid.sync();
    const State* st = a.state;
    if (__ldcg(&st->done)) break;
    for (int k = 0; k < 3; ++k) cls_axis[k] = __ldcg(&st->next[k]);
    if (a.mode == 1) e = __ldcg(&st->e);
    slot ^= 1;
    have_prev = a.mode == 0;
  }
}

}  // namespace

int coop_refine_grid(int sms) {
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, coop_refine_kernel, kThreads, 0);
  if (per_sm < 1) per_sm = 1;
  return sms * (per_sm < 4 ? per_sm : 4);
}

int coop_tiles(int64_t n) { return (int)((n + kTile - 1) / kTile); }

cudaError_t launch_coop_refine(const double* zx, const double* zy, const double* zz, int64_t n, int mode, int refine,
                               double eps, double e0, const double axis0[3], uint32_t* flags0, uint32_t* flags1,
                               int32_t* tile_count, int32_t* tile_offset, double* block_part, void* state, int grid,
                               cudaStream_t s) {
  CoopArgs a;
  a.zx = zx;
  a.zy = zy;
  a.zz = zz;
  a.n = n;
  a.mode = mode;
  a.refine = refine;
  a.eps = eps;
  a.e0 = e0;
  for (int k = 0; k < 3; ++k) a.axis0[k] = axis0[k];
  a.flags0 = flags0;
  a.flags1 = flags1;
  a.tile_count = tile_count;
  a.tile_offset = tile_offset;
  a.block_part = block_part;
  a.state = static_cast<State*>(state);
  void* args[] = {&a};
  return cudaLaunchCooperativeKernel((void*)coop_refine_kernel, dim3(grid), dim3(kThreads), args, 0, s);
}

size_t coop_state_bytes() { return sizeof(State); }

}  // namespace rvb
