// K1 (band plan) and K2 (band-tiled vote) of the spatial-voting path.
//
// Reference semantics (voting.cpp:25-45, :88-118): every constraint z deposits exactly J
// votes, one per sample theta_j = -pi + j*2pi/J of the great circle {v : z.v = 0}; each
// sample is flipped to the southern hemisphere, stereographically projected and counted in
// its cell of a G x G uint32 grid. The device result is BIT-EXACT with that definition:
//
//  * Twins. Samples j and j+J/2 are antipodal, so after the hemisphere flip they land on
//    the same plane point (up to ~1e-15). K2 evaluates one "pair" per twin and deposits 2.
//  * f32 filter + exact f64 fallback. The pair is evaluated in f32 from an f64 basis; the
//    cell coordinate t is produced on a 2^-S grid (S <= 13, chosen per geometry by make_plan) by
//    one FFMA against a magic constant. |t32 - t64| <= K*6e-7 + 2^-(S+1) cells, so
//    whenever t32 is at least 2*2^-S from an integer (and |c| >= 2e-6, no hemisphere ambiguity)
//    the f32 cell IS the reference cell. Otherwise the pair is queued and both twins are
//    recomputed exactly in f64 (same op order, no FMA) -- ~0.2% of pairs.
//  * Band tiling. The grid's reachable rows are split into bands that fit one CTA's shared
//    memory (u32 counters, 1 CTA/SM). K1 computes per (constraint, band) the pair-index
//    ranges whose projected points can fall in the band (analytic circle/line intersection,
//    padded), so K2 only evaluates pairs near its band; an exact ownership test on the row
//    decides the deposit, so a sample is counted by exactly one band.
//  * Tiles are flushed once per (CTA, band) to partial slots; a reduction kernel sums the
//    slots of each band (integer sums: order-free, deterministic).
#include <cuda_runtime.h>

#include <cstdint>
#include <mutex>
#include <type_traits>

#include "rv_exact.cuh"
#include "rv_internal.h"

namespace rvb {

namespace {

constexpr float kPiF = 3.14159265358979323846f;
constexpr float kTwoPiF = 6.28318530717958647692f;
constexpr float kRcMin = 1e-3f;     // |c| amplitude below which a circle is treated as all-band
constexpr float kDc = 2e-6f;        // |c| below this: hemisphere flip ambiguous -> exact path
#ifndef RV_RED_GROUPS
#define RV_RED_GROUPS 2
#endif
#ifndef RV_NP
#define RV_NP 2  // pairs per lane per full step of the vote loop (2 or 4)
#endif
#ifndef RV_PRED
#define RV_PRED 0  // 1: predicated deposit instead of the per-lane sink word
#endif
#ifndef RV_STEP_UNROLL
#define RV_STEP_UNROLL 1  // unroll of the 64-pair step loop
#endif
constexpr int kStepUnroll = RV_STEP_UNROLL;
#ifndef RV_FB_INLINE
#define RV_FB_INLINE __forceinline__  // exact path inlined: as a call, the ABI forced per-step remats (dev knob)
#endif
#ifndef RV_PACK
#define RV_PACK 1  // 1: a lane's two pairs of a 64-pair step are adjacent and evaluated with f32x2 math
#endif
static_assert(!(RV_PACK && RV_NP != 2), "packed steps walk 2 adjacent pairs per lane");

// sm_100 packed f32 pairs (FMUL2/FFMA2: one issue slot for two IEEE round-to-nearest ops, each
// lane of the pair bit-identical to the scalar FMUL/FFMA)
typedef unsigned long long f32x2;
__device__ __forceinline__ f32x2 pk2(float a, float b) {
  f32x2 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void upk2(f32x2 v, uint32_t& a, uint32_t& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=r"(a), "=r"(b) : "l"(v));
}
__device__ __forceinline__ f32x2 mul2(f32x2 a, f32x2 b) {
  f32x2 r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f32x2 fma2(f32x2 a, f32x2 b, f32x2 c) {
  f32x2 r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}

__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// per-warp fallback queue in shared memory (32-bit shared-window addresses)
__device__ __forceinline__ void sts_u32(uint32_t saddr, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(saddr), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t lds_u32(uint32_t saddr) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(saddr) : "memory");
  return v;
}

// ---- K1b: band plan --------------------------------------------------------------------
// Cheap trig for the planner: errors (~1e-5 rad) are far below the 2-pair padding (6e-3 rad at
// J=2048); coverage only has to be a superset, ownership is decided exactly per sample.
__device__ __forceinline__ float atan2_fast(float y, float x) {
  const float ax = fabsf(x), ay = fabsf(y);
  const float mx = fmaxf(ax, ay), mn = fminf(ax, ay);
  const float a = mx > 0.f ? __fdividef(mn, mx) : 0.f;
  const float s = a * a;
  float r = fmaf(fmaf(fmaf(-0.0464964749f, s, 0.15931422f), s, -0.327622764f), s * a, a);
  if (ay > ax) r = 1.57079637f - r;
  if (x < 0.f) r = 3.14159274f - r;
  return y < 0.f ? -r : r;
}
__device__ __forceinline__ float acos_fast(float x) {  // Abramowitz-Stegun 4.4.46, |err| <= 2e-8 (+f32)
  const float ax = fminf(fabsf(x), 1.f);
  float p = -0.0012624911f;
  p = fmaf(p, ax, 0.0066700901f);
  p = fmaf(p, ax, -0.0170881256f);
  p = fmaf(p, ax, 0.0308918810f);
  p = fmaf(p, ax, -0.0501743046f);
  p = fmaf(p, ax, 0.0889789874f);
  p = fmaf(p, ax, -0.2145988016f);
  p = fmaf(p, ax, 1.5707963050f);
  const float r = sqrtf(1.f - ax) * p;
  return x < 0.f ? kPiF - r : r;
}

// Up to two disjoint, sorted intervals of s in [0, pi] (register-resident, no dynamic indexing).
struct Arc2 {
  float a0, b0, a1, b1;
  int n;
};

// { s in [0, pi] : A cos(theta_a + s) + B sin(theta_a + s) >= y0 } -- on the canonical arc this is
// { Y(s) >= y0 } because 1 - c > 0 there. `dil` widens (>0) or narrows (<0) the interval by ~10x the
// trig approximation error (atan2_fast <= 2.1e-4 rad), so a nearly-empty interval is never lost.
constexpr float kArcDilate = 2e-3f;
__device__ __forceinline__ Arc2 arc_ge(float A, float B, float y0, float theta_a, float dil) {
  Arc2 r{0.f, 0.f, 0.f, 0.f, 0};
  const float R = sqrtf(fmaf(A, A, B * B));
  if (!(R > 0.f)) {
    if (y0 <= 0.f) r = Arc2{0.f, kPiF, 0.f, 0.f, 1};
    return r;
  }
  const float ratio = __fdividef(y0, R);
  if (ratio <= -1.f) return Arc2{0.f, kPiF, 0.f, 0.f, 1};
  if (!(ratio < 1.f)) return r;
  const float alpha = acos_fast(ratio);
  float sig = atan2_fast(B, A) - theta_a;
  sig -= kTwoPiF * floorf((sig + kPiF) * (1.f / kTwoPiF));
  const float half = alpha + dil;
  const float lo0 = fmaxf(sig - half, 0.f), hi0 = fminf(sig + half, kPiF);
  const float lo1 = fmaxf(sig - half + kTwoPiF, 0.f), hi1 = fminf(sig + half + kTwoPiF, kPiF);
  if (lo0 <= hi0) {
    r.a0 = lo0;
    r.b0 = hi0;
    r.n = 1;
    if (lo1 <= hi1) {
      r.a1 = lo1;
      r.b1 = hi1;
      r.n = 2;
    }
  } else if (lo1 <= hi1) {
    r.a0 = lo1;
    r.b0 = hi1;
    r.n = 1;
  }
  return r;
}

// Appends an integer pair interval [lo, hi] (u coordinates, increasing starts) to a running
// merge of at most 3 output intervals held in registers.
struct Runs {
  int l0, h0, l1, h1, l2, h2, n;
};
__device__ __forceinline__ void runs_push(Runs& r, int lo, int hi) {
  if (r.n == 0) {
    r.l0 = lo;
    r.h0 = hi;
    r.n = 1;
  } else if (r.n == 1) {
    if (lo <= r.h0 + 1) r.h0 = max(r.h0, hi);
    else {
      r.l1 = lo;
      r.h1 = hi;
      r.n = 2;
    }
  } else if (r.n == 2) {
    if (lo <= r.h1 + 1) r.h1 = max(r.h1, hi);
    else {
      r.l2 = lo;
      r.h2 = hi;
      r.n = 3;
    }
  } else {
    if (lo <= r.h2 + 1) r.h2 = max(r.h2, hi);
    else r.n = 4;  // overflow: caller goes conservative
  }
}

// x mod M in [0, M) (M = J/2 pairs; a power of two for every J the reference ships, else the
// generic integer modulo)
__device__ __forceinline__ int wrap_pair(int x, int M) {
  if ((M & (M - 1)) == 0) return x & (M - 1);
  x %= M;
  return x < 0 ? x + M : x;
}

// Ranges of one band from its lower/upper arc sets: S = U_lo \ U_hi, padded, merged, wrapped.
__device__ __forceinline__ uint2 plan_from_sets(const Arc2& ulo, const Arc2& uhi, float pa, float inv_step, int M,
                                                unsigned long long* work) {
  // gaps of uhi inside [0, pi] (sorted): [0, a0], [b0, a1], [b_last, pi]
  float g[6];
  int ng;
  if (uhi.n == 0) {
    g[0] = 0.f;
    g[1] = kPiF;
    ng = 1;
  } else if (uhi.n == 1) {
    g[0] = 0.f;
    g[1] = uhi.a0;
    g[2] = uhi.b0;
    g[3] = kPiF;
    ng = 2;
  } else {
    g[0] = 0.f;
    g[1] = uhi.a0;
    g[2] = uhi.b0;
    g[3] = uhi.a1;
    g[4] = uhi.b1;
    g[5] = kPiF;
    ng = 3;
  }
  const float lo_a[2] = {ulo.a0, ulo.a1}, lo_b[2] = {ulo.b0, ulo.b1};
  Runs runs{0, 0, 0, 0, 0, 0, 0};
#pragma unroll
  for (int i = 0; i < 2; ++i) {
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      if (i < ulo.n && j < ng) {
        // strict: a zero-length gap/piece only arises where U_hi (eroded) robustly covers an arc
        // end, so it holds no sample of this band
        const float s1 = fmaxf(lo_a[i], g[2 * j]), s2 = fminf(lo_b[i], g[2 * j + 1]);
        if (s1 < s2)
          runs_push(runs, __float2int_rd(fmaf(s1, inv_step, pa)) - kPad, __float2int_ru(fmaf(s2, inv_step, pa)) + kPad);
      }
    }
  }
  const uint2 full = make_uint2((uint32_t)M << 16, 0u);
  if (runs.n == 0) return make_uint2(0u, 0u);
  if (runs.n > 3) {
    *work += (unsigned long long)M;
    return full;
  }
  // u spans [pa - pad, pa + M + pad]: the last run may wrap onto the first
  int nl = runs.n;
  int L0 = runs.l0, H0 = runs.h0, L1 = runs.l1, H1 = runs.h1;
  if (nl == 3) {
    if (runs.h2 - M >= runs.l0 - 1) {  // join last with first across the wrap
      L0 = runs.l2;
      H0 = runs.h0 + M;
      nl = 2;  // (L0,H0) and (l1,h1)
    } else {
      *work += (unsigned long long)M;
      return full;
    }
  } else if (nl == 2) {
    if (H1 - M >= L0 - 1) {
      L0 = L1;
      H0 = runs.h0 + M;
      nl = 1;
    }
  }
  // even starts (M is a multiple of 64): K2's packed steps give each lane two adjacent pairs
  L0 &= ~1;
  L1 &= ~1;
  int s0 = wrap_pair(L0, M), l0 = H0 - L0 + 1;
  int s1 = wrap_pair(L1, M), l1 = nl == 2 ? H1 - L1 + 1 : 0;
  if (l0 >= M || l1 >= M) {
    *work += (unsigned long long)M;
    return full;
  }
  // 32-pair alignment (K2 walks 32 consecutive pairs per lane-step) and a final overlap merge
  l0 = (l0 + 31) & ~31;
  if (nl == 2) {
    l1 = (l1 + 31) & ~31;
    const int d01 = wrap_pair(s1 - s0, M), d10 = wrap_pair(s0 - s1, M);
    if (d01 < l0) {
      l0 = (max(l0, d01 + l1) + 31) & ~31;
      nl = 1;
    } else if (d10 < l1) {
      s0 = s1;
      l0 = (max(l1, d10 + l0) + 31) & ~31;
      nl = 1;
    }
  }
  if (l0 >= M || (nl == 2 && l0 + l1 >= M)) {
    *work += (unsigned long long)M;
    return full;
  }
  *work += (unsigned long long)(l0 + (nl == 2 ? l1 : 0));
  return make_uint2((uint32_t)s0 | ((uint32_t)l0 << 16), nl == 2 ? ((uint32_t)s1 | ((uint32_t)l1 << 16)) : 0u);
}

// kNB > 0: n_bands <= kNB, ranges kept in registers and entries reserved once per (block, band)
// (same-address global atomics were the planner's bottleneck); kNB == 0: any band count, one
// reservation per (warp, band).
template <int kNB>
__global__ void __launch_bounds__(256) plan_kernel(VotePlan p, VoteBuffers b, int64_t n) {
  __shared__ unsigned long long s_work[kMaxBands];
  __shared__ int s_cnt[kMaxBands], s_base[kMaxBands];
  for (int t = threadIdx.x; t < p.n_bands; t += blockDim.x) {
    s_work[t] = 0;
    s_cnt[t] = 0;
  }
  __syncthreads();
  const int64_t lo = b.bounds ? b.bounds[0] : b.range_lo, hi = b.bounds ? b.bounds[1] : b.range_lo + n;
  const int64_t i = lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double z0 = 0.0, z1 = 0.0, z2 = 0.0;
  if (i < hi) {
    z0 = b.zx[i];
    z1 = b.zy[i];
    z2 = b.zz[i];
  }
  const bool valid = i < hi && !isnan(z0);  // in-order constraint sets mark dropped pairs with NaN
  const int M = p.halfJ;
  float f1[3] = {0.f, 0.f, 0.f}, f2[3] = {0.f, 0.f, 0.f};
  if (valid) {
    double a1[3], a2[3];
    exact_basis(z0, z1, z2, a1, a2);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      f1[k] = __double2float_rn(a1[k]);
      f2[k] = __double2float_rn(a2[k]);
    }
    // the vote reads fl32(K * a_xy) (one rounding, like fl32(a_xy)): saves a multiply per pair
    const double K = p.inv_cell;
    b.basis_a[i] = make_float4(__double2float_rn(a1[0] * K), __double2float_rn(a1[1] * K), f1[2],
                               __double2float_rn(a2[0] * K));
    b.basis_b[i] = make_float2(__double2float_rn(a2[1] * K), f2[2]);
  }
  // near-polar constraint: c ~ 0 everywhere, every band sees all pairs
  const bool polar = !(sqrtf(fmaf(f1[2], f1[2], f2[2] * f2[2])) >= kRcMin);
  const float theta_a = atan2_fast(f2[2], f1[2]) + 0.5f * kPiF;  // c(theta_a + s) = -rc sin(s)
  const float inv_step = 1.f / p.step_f;
  const float pa = (theta_a + kPiF) * inv_step;
  const int lane = threadIdx.x & 31;
  const unsigned lt_mask = (1u << lane) - 1u;
  const unsigned long long ci = (unsigned long long)(uint32_t)i;
  Arc2 ulo{0.f, kPiF, 0.f, 0.f, 1};  // band 0: Y >= -inf
  // ranges of this constraint in band `band` (+ planned pairs into *w)
  auto plan_band = [&](int band, unsigned long long* w) -> uint2 {
    if (!valid) return make_uint2(0u, 0u);
    if (polar) {
      *w = (unsigned long long)M;
      return make_uint2((uint32_t)M << 16, 0u);
    }
    if (band > 0) {
      const float y0 = p.band_ylo[band];
      ulo = arc_ge(fmaf(y0, f1[2], f1[1]), fmaf(y0, f2[2], f2[1]), y0, theta_a, kArcDilate);
    }
    Arc2 uhi{0.f, 0.f, 0.f, 0.f, 0};  // last band: Y >= +inf is empty
    if (band < p.n_bands - 1) {
      const float y1 = p.band_yhi[band];
      uhi = arc_ge(fmaf(y1, f1[2], f1[1]), fmaf(y1, f2[2], f2[1]), y1, theta_a, -kArcDilate);
    }
    return plan_from_sets(ulo, uhi, pa, inv_step, M, w);
  };
  // warp-level bookkeeping of one band: entry offset of this lane inside the warp's block of
  // entries, reserved in s_cnt (kNB > 0) or directly in the global list (kNB == 0)
  auto book = [&](int band, uint2 r, unsigned long long w, bool global) -> int {
    const unsigned m0 = __ballot_sync(0xFFFFFFFFu, r.x >= 0x10000u);  // r.y != 0 => r.x != 0
    const unsigned m1 = __ballot_sync(0xFFFFFFFFu, r.y >= 0x10000u);
    const int total = __popc(m0) + __popc(m1);
    int wbase = 0;
    if (lane == 0 && total) wbase = global ? atomicAdd(&b.entry_count[band], total) : atomicAdd(&s_cnt[band], total);
    wbase = __shfl_sync(0xFFFFFFFFu, wbase, 0);
    const unsigned ws = __reduce_add_sync(0xFFFFFFFFu, (unsigned)w);  // w <= J/2 pairs per lane
    if (lane == 0 && ws) atomicAdd(&s_work[band], (unsigned long long)ws);
    return wbase + __popc(m0 & lt_mask) + __popc(m1 & lt_mask);
  };
  auto emit = [&](int band, uint2 r, int64_t off) {
    if (r.x >= 0x10000u) {
      unsigned long long* ep = b.entries + (int64_t)band * b.entry_cap + off;
      ep[0] = ci | ((unsigned long long)r.x << 32);
      if (r.y >= 0x10000u) ep[1] = ci | ((unsigned long long)r.y << 32);
    }
  };
  if constexpr (kNB > 0) {
    // per-thread ranges/offsets parked in shared memory (a rolled band loop keeps the code small)
    __shared__ uint2 s_r[kNB][256];
    __shared__ int s_off[kNB][256];
#pragma unroll 1
    for (int band = 0; band < p.n_bands; ++band) {  // uniform
      unsigned long long w = 0;
      const uint2 r = plan_band(band, &w);
      s_r[band][threadIdx.x] = r;
      s_off[band][threadIdx.x] = book(band, r, w, false);
    }
    __syncthreads();
    for (int t = threadIdx.x; t < p.n_bands; t += blockDim.x)
      s_base[t] = s_cnt[t] ? atomicAdd(&b.entry_count[t], s_cnt[t]) : 0;
    __syncthreads();
#pragma unroll 1
    for (int band = 0; band < p.n_bands; ++band)
      emit(band, s_r[band][threadIdx.x], (int64_t)s_base[band] + s_off[band][threadIdx.x]);
  } else {
    for (int band = 0; band < p.n_bands; ++band) {  // uniform trip count: warp collectives inside
      unsigned long long w = 0;
      const uint2 r = plan_band(band, &w);
      emit(band, r, book(band, r, w, true));
    }
    __syncthreads();
  }
  for (int t = threadIdx.x; t < p.n_bands; t += blockDim.x)
    if (s_work[t]) atomicAdd(&b.band_work[t], s_work[t]);
}

// ---- K2 ------------------------------------------------------------------------------

// f32 evaluation of one pair: tile-relative linear cell index `rel` (>= tile_cells: not this
// band's tile) and whether the f32 cell is not provably the reference cell. Shared by the hot
// loop and the exact path (which undoes the hot loop's deposit), so both see identical values.
struct F32Geom {
  float CMf;
  int S;
  uint32_t fmask;
  uint32_t W;
  uint32_t lin_off;  // non-clamp: (magic_hi + r0) * W + magic_hi + c_min
  int magic_hi, G, r0, c_min;
};
template <bool kClamp, int kS>
__device__ __forceinline__ uint32_t cell_of_bits(const F32Geom& g, float c, uint32_t bx, uint32_t by, bool* flag);
template <bool kClamp, int kS>  // kS: compile-time fixed-point shift (0: g.S at run time)
__device__ __forceinline__ uint32_t f32_cell(const F32Geom& g, float4 ba, float2 bb, float2 t, bool* flag) {
  // x, y carry the cell scale K = G/(2E) (folded into the f32 basis by the planner)
  const float xk = fmaf(ba.w, t.y, ba.x * t.x);
  const float yk = fmaf(bb.x, t.y, ba.y * t.x);
  const float c = fmaf(bb.y, t.y, ba.z * t.x);
  const float r = rcp_approx(1.f + fabsf(c));
  const float rs = __int_as_float(__float_as_int(r) | (~__float_as_int(c) & 0x80000000));
  const uint32_t bx = (uint32_t)__float_as_int(fmaf(xk, rs, g.CMf));
  const uint32_t by = (uint32_t)__float_as_int(fmaf(yk, rs, g.CMf));
  return cell_of_bits<kClamp, kS>(g, c, bx, by, flag);
}

// Two pairs of f32_cell at once, t = {cos_a, cos_b, sin_a, sin_b}: the same IEEE operations in
// the same order, lane-parallel in f32x2, so each cell and flag is bit-identical to f32_cell's
// (the exact path recomputes a queued pair with the scalar f32_cell to undo its deposit).
template <bool kClamp, int kS>
__device__ __forceinline__ void f32_cell2(const F32Geom& g, float4 ba, float2 bb, float4 t, uint32_t* rel,
                                          bool* flag) {
  const f32x2 C = pk2(t.x, t.y), Sn = pk2(t.z, t.w);
  const f32x2 X = fma2(pk2(ba.w, ba.w), Sn, mul2(pk2(ba.x, ba.x), C));
  const f32x2 Y = fma2(pk2(bb.x, bb.x), Sn, mul2(pk2(ba.y, ba.y), C));
  const f32x2 Cc = fma2(pk2(bb.y, bb.y), Sn, mul2(pk2(ba.z, ba.z), C));
  uint32_t cb[2];
  upk2(Cc, cb[0], cb[1]);
  float rs[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const float r = rcp_approx(1.f + fabsf(__uint_as_float(cb[h])));
    rs[h] = __int_as_float(__float_as_int(r) | (int)(~cb[h] & 0x80000000u));
  }
  const f32x2 RS = pk2(rs[0], rs[1]), CM = pk2(g.CMf, g.CMf);
  uint32_t bx[2], by[2];
  upk2(fma2(X, RS, CM), bx[0], bx[1]);
  upk2(fma2(Y, RS, CM), by[0], by[1]);
#pragma unroll
  for (int h = 0; h < 2; ++h) rel[h] = cell_of_bits<kClamp, kS>(g, __uint_as_float(cb[h]), bx[h], by[h], &flag[h]);
}

template <bool kClamp, int kS>
__device__ __forceinline__ uint32_t cell_of_bits(const F32Geom& g, float c, uint32_t bx, uint32_t by, bool* flag) {
  const int S = kS ? kS : g.S;
  *flag = (fabsf(c) < kDc) | ((bx & g.fmask) == 0u) | ((by & g.fmask) == 0u);
  // the column is always inside [c_min, c_min+W) (|X| <= 1 < extent, or clamped), so one
  // unsigned range test on the linear index is the band-ownership test
  if (kClamp) {
    const int row = min(max((int)(by >> S) - g.magic_hi, 0), g.G - 1) - g.r0;
    const int col = min(max((int)(bx >> S) - g.magic_hi, 0), g.G - 1) - g.c_min;
    return (uint32_t)(row * (int)g.W + col);
  }
  return (by >> S) * g.W + (bx >> S) - g.lin_off;
}


// Exact f64 evaluation of both twins of a queued pair; deposits the ones this band owns.
// Cold path (~0.6% of pairs), kept out of line so the hot loop keeps its registers.
struct FbCtx {  // the few scalars the exact path needs (keeps the kernel-param struct in cbank)
  const double* zx;
  const double* zy;
  const double* zz;
  const double2* table64;
  uint32_t* grid;
  double E, inv_cell;
  int G, halfJ, c_min, W, own_lo, own_hi;
};

// (cos, sin) of pair p in the shared table. RV_PACK layout: float4 q = {cos_2q, cos_2q+1,
// sin_2q, sin_2q+1}, so one LDS.128 feeds a lane's two adjacent pairs as f32x2 operands.
__device__ __forceinline__ float2 tab_pair(const float2* tab, int p) {
#if RV_PACK
  const float* t = reinterpret_cast<const float*>(tab) + 4 * (p >> 1) + (p & 1);
  return make_float2(t[0], t[2]);
#else
  return tab[p];
#endif
}

// Exact path of queued pairs: the hot loop deposited +2 at the pair's f32 cell (if in this tile)
// unconditionally; undo that, then deposit both twins at their exact f64 cells (row-owned).
template <bool kClamp, int kS>
__device__ RV_FB_INLINE void fallback_pairs(FbCtx f, F32Geom g, uint32_t q_s, int count, uint32_t my_ci,
                                            float4 my_a, float2 my_b, const float2* tab, uint32_t* tile,
                                            uint32_t tile_cells, int hb) {
  const int lane = threadIdx.x & 31;
  const uint32_t e = lane < count ? lds_u32(q_s + 4u * lane) : 0u;
  const int k = (int)(e >> 16) & 31;  // entry index within the warp's grab
  const uint32_t ci = __shfl_sync(0xFFFFFFFFu, my_ci, k);
  float4 ba;
  float2 bb;
  ba.x = __shfl_sync(0xFFFFFFFFu, my_a.x, k);
  ba.y = __shfl_sync(0xFFFFFFFFu, my_a.y, k);
  ba.z = __shfl_sync(0xFFFFFFFFu, my_a.z, k);
  ba.w = __shfl_sync(0xFFFFFFFFu, my_a.w, k);
  bb.x = __shfl_sync(0xFFFFFFFFu, my_b.x, k);
  bb.y = __shfl_sync(0xFFFFFFFFu, my_b.y, k);
  if (lane < count) {
    const int pair = (int)(e & 0xFFFFu);
    bool fl;
    const uint32_t rel = f32_cell<kClamp, kS>(g, ba, bb, tab_pair(tab, pair), &fl);
    if (rel < tile_cells) atomicSub(&tile[rel], 2u);
    double a1[3], a2[3];
    exact_basis(f.zx[ci], f.zy[ci], f.zz[ci], a1, a2);
    VotePlan p1;
    p1.E = f.E;
    p1.inv_cell = f.inv_cell;
    p1.G = f.G;
#pragma unroll
    for (int tw = 0; tw < 2; ++tw) {
      const double2 cs = f.table64[pair + tw * f.halfJ];
      int row, col;
      exact_sample(a1, a2, cs.x, cs.y, p1, &row, &col);
      if (row < f.own_lo || row >= f.own_hi) continue;
      const int lr = row - g.r0, lc = col - f.c_min;
      if ((unsigned)lr < (unsigned)hb && (unsigned)lc < (unsigned)f.W)
        atomicAdd(&tile[lr * f.W + lc], 1u);
      else
        atomicAdd(&f.grid[(size_t)row * f.G + col], 1u);
    }
  }
  __syncwarp();
}

// table read (read-only after the prologue's barrier, so no memory clobber)
__device__ __forceinline__ float2 lds_f2(uint32_t saddr) {
  float2 t;
  asm("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(t.x), "=f"(t.y) : "r"(saddr));
  return t;
}

__device__ __forceinline__ float lds_f1(uint32_t saddr) {
  float t;
  asm("ld.shared.f32 %0, [%1];" : "=f"(t) : "r"(saddr));
  return t;
}

__device__ __forceinline__ uint32_t umin(uint32_t a, uint32_t b) { return a < b ? a : b; }

__device__ __forceinline__ void red_shared(uint32_t saddr, uint32_t v) {
  asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(saddr), "r"(v));
}

__device__ __forceinline__ void red_shared_if(uint32_t saddr, uint32_t v, bool pred) {
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q red.shared.add.u32 [%0], %1;\n\t}" ::"r"(saddr), "r"(v),
      "r"((uint32_t)pred));
}

// The work-entry loop of one band tile (shared by the band-tiled vote and the fused front kernel):
// per-warp dynamic grabs of 32 entries from `counter` (lane k holds entry k: range + f32 basis),
// 64-pair steps, deposit-always into the tile, exact path for flagged pairs. fetch(j) returns
// entry j of the band's list (j < n_ent).
struct VoteCtx {
  const float2* tab;
  uint32_t tab_s;
  uint32_t* tile;
  uint32_t tile_s, sink_rel, vote2, fbq_s;
  unsigned lt_mask;
  int M;
  uint32_t tile_cells;
  int hb;
  const float4* basis_a;
  const float2* basis_b;
  int grab;  // entries per warp grab (<= 32)
};
template <bool kClamp, int kS, class Fetch>
__device__ __forceinline__ void vote_entries(const VoteCtx& v, const F32Geom& geo, const FbCtx& fc, Fetch fetch,
                                             int n_ent, int* counter, unsigned int& my_fb) {
  const int lane = threadIdx.x & 31;
  const float2* tab = v.tab;
  const uint32_t tab_s = v.tab_s, tile_s = v.tile_s, sink_rel = v.sink_rel, vote2 = v.vote2, fbq_s = v.fbq_s;
  const unsigned lt_mask = v.lt_mask;
  const int M = v.M, hb = v.hb;
  const uint32_t tile_cells = v.tile_cells;
  uint32_t* tile = v.tile;
  const int grab = v.grab;
  for (;;) {  // per-warp dynamic grabs of up to 32 entries (lane k holds entry k: range + f32 basis)
    int g0 = 0;
    if (lane == 0) g0 = atomicAdd(counter, grab);
    g0 = __shfl_sync(0xFFFFFFFFu, g0, 0);
    if (g0 >= n_ent) break;
    const int ne = min(grab, n_ent - g0);
    uint32_t my_ci = 0, my_enc = 0;
    float4 my_a = make_float4(0.f, 0.f, 0.f, 0.f);
    float2 my_b = make_float2(0.f, 0.f);
    if (lane < ne) {
      const unsigned long long e = fetch(g0 + lane);
      my_ci = (uint32_t)e;
      my_enc = (uint32_t)(e >> 32);
      my_a = v.basis_a[my_ci];
      my_b = v.basis_b[my_ci];
    }
    int qn = 0;
    for (int k = 0; k < ne; ++k) {
      const uint32_t enc = __shfl_sync(0xFFFFFFFFu, my_enc, k);
      float4 ba;
      float2 bb;
      ba.x = __shfl_sync(0xFFFFFFFFu, my_a.x, k);
      ba.y = __shfl_sync(0xFFFFFFFFu, my_a.y, k);
      ba.z = __shfl_sync(0xFFFFFFFFu, my_a.z, k);
      ba.w = __shfl_sync(0xFFFFFFFFu, my_a.w, k);
      bb.x = __shfl_sync(0xFFFFFFFFu, my_b.x, k);
      bb.y = __shfl_sync(0xFFFFFFFFu, my_b.y, k);
      const uint32_t local_k = (uint32_t)k << 16;
      const int start = (int)(enc & 0xFFFFu), len = (int)(enc >> 16);
      const uint32_t tp_s = tab_s + 8u * (uint32_t)start;
#if RV_PACK  // tab_s = table + 16*lane (packed steps); the scalar tail reads pair start + lane
      const uint32_t tp1_s = tp_s - 8u * (uint32_t)lane - 4u * (uint32_t)(lane & 1);
#endif
      // NP pairs per lane per step (32*NP consecutive pairs per warp); ranges are 32-aligned:
      // 64-pair steps while they fit, then one 32-pair tail step
      auto step = [&](int k0, auto np_tag) {
        constexpr int NP = decltype(np_tag)::value;
        bool flag[NP];
        uint32_t addr[NP];
        uint32_t relp[NP];
        // pair of (lane, h): packed steps walk adjacent pairs k0 + 2*lane + h, the others k0 + 32*h + lane
        constexpr bool kPacked = RV_PACK && NP == 2;
        if constexpr (kPacked) {
          float4 t4;
          asm("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
              : "=f"(t4.x), "=f"(t4.y), "=f"(t4.z), "=f"(t4.w)
              : "r"(tp_s + 8u * (uint32_t)k0));
          f32_cell2<kClamp, kS>(geo, ba, bb, t4, relp, flag);
        }
#pragma unroll
        for (int h = 0; h < NP; ++h) {
          float2 t;
          if constexpr (!kPacked) {
#if RV_PACK  // scalar (tail) step over the packed layout: lane's pair k0 + lane
            const uint32_t a1 = tp1_s + 8u * (uint32_t)(k0 + 32 * h);
            t = make_float2(lds_f1(a1), lds_f1(a1 + 8u));
#else
            t = lds_f2(tp_s + 8u * (uint32_t)(k0 + 32 * h));
#endif
            relp[h] = f32_cell<kClamp, kS>(geo, ba, bb, t, &flag[h]);
          }
          const uint32_t rel = relp[h];
          // deposit even if flagged: the exact path undoes it (no select on the flag here)
#if RV_PRED
          addr[h] = rel;
#else
          addr[h] = tile_s + 4u * umin(rel, sink_rel);
#endif
        }
#pragma unroll
        for (int h = 0; h < NP; ++h) {
#if RV_PRED
          asm volatile("{\n\t.reg .pred q;\n\tsetp.lt.u32 q, %1, %2;\n\t@q red.shared.add.u32 [%0], %3;\n\t}" ::"r"(
                           tile_s + 4u * addr[h]),
                       "r"(addr[h]), "r"(tile_cells), "r"(vote2));
#else
          red_shared(addr[h], vote2);
#endif
        }
        bool any = false;
#pragma unroll
        for (int h = 0; h < NP; ++h) any |= flag[h];
        if (__any_sync(0xFFFFFFFFu, any)) {  // cold: queue for the exact f64 path
#pragma unroll
          for (int h = 0; h < NP; ++h) {
            const unsigned fm = __ballot_sync(0xFFFFFFFFu, flag[h]);
            if (flag[h]) {
              int pair = kPacked ? start + k0 + 2 * lane + h : start + k0 + 32 * h + lane;
              if (pair >= M) pair -= M;
              sts_u32(fbq_s + 4u * (uint32_t)(qn + __popc(fm & lt_mask)), local_k | (uint32_t)pair);
            }
            qn += __popc(fm);
            my_fb += __popc(fm);
            __syncwarp();
            if (qn >= 32) {
              fallback_pairs<kClamp, kS>(fc, geo, fbq_s, 32, my_ci, my_a, my_b, tab, tile, tile_cells, hb);
              qn -= 32;
              if (lane < qn) sts_u32(fbq_s + 4u * lane, lds_u32(fbq_s + 4u * (32 + lane)));
              __syncwarp();
            }
          }
        }
      };
      int k0 = 0;
      if constexpr (RV_NP == 4) {
#pragma unroll 1
        for (; k0 + 128 <= len; k0 += 128) step(k0, std::integral_constant<int, 4>{});
        if (k0 + 64 <= len) {
          step(k0, std::integral_constant<int, 2>{});
          k0 += 64;
        }
      } else {
#pragma unroll kStepUnroll
        for (; k0 + 64 <= len; k0 += 64) step(k0, std::integral_constant<int, 2>{});
      }
      if (k0 < len) step(k0, std::integral_constant<int, 1>{});
    }
    if (qn > 0) fallback_pairs<kClamp, kS>(fc, geo, fbq_s, qn, my_ci, my_a, my_b, tab, tile, tile_cells, hb);
  }
}

// K2: persistent, one CTA per SM, 16 warps. A CTA owns one row band's u32 tile in shared
// memory at a time. Warps grab 32 work entries at a time from the band's entry list (K1 appends
// one entry per non-empty (constraint, band) pair range; lane k loads entry k and its f32 basis,
// the warp then walks the entries, broadcasting each by shuffles); no CTA barrier per grab. When
// the band is exhausted the CTA flushes its tile to a partial slot and steals the band with the
// most remaining entries. Lanes walk 64 consecutive sample pairs per step of a range (32-aligned
// lengths, table doubled so ranges never wrap). Pairs whose f32 cell is not provably the
// reference cell are queued per warp and recomputed exactly in f64.

#ifdef RV_VOTE_TRACE  // dev instrumentation: per-CTA phase timestamps (globaltimer, ns)
__device__ unsigned long long g_vtrace[2 * 65536];
__device__ unsigned int g_vtrace_n;
__device__ __forceinline__ void vtrace(int tag, int band) {
  if (threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    const unsigned k = atomicAdd(&g_vtrace_n, 1u);
    if (k < 65536) {
      g_vtrace[2 * k] = t;
      g_vtrace[2 * k + 1] = ((unsigned long long)blockIdx.x << 16) | ((unsigned)tag << 8) | (unsigned)(band & 255);
    }
  }
}
#else
__device__ __forceinline__ void vtrace(int, int) {}
#endif

template <bool kClamp, int kS>
__global__ void __launch_bounds__(kVoteThreads, 1) vote_banded_kernel(VotePlan p, VoteBuffers b, int64_t n) {
  extern __shared__ uint4 smem_raw[];
  uint32_t* tile = reinterpret_cast<uint32_t*>(smem_raw);
  // [tile_words] tile, [32] per-lane sink words, table, fallback queues
  float2* tab = reinterpret_cast<float2*>(tile + ((p.tile_words + 32 + 3) & ~size_t(3)));
  const int M = p.halfJ;
  uint32_t* fbq_all = reinterpret_cast<uint32_t*>(tab + 2 * M + 64);
  __shared__ int s_band, s_slot;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint32_t fbq_s = (uint32_t)__cvta_generic_to_shared(fbq_all + warp * kFbqCap);  // this warp's queue
#if RV_PACK  // pair p of the doubled table lives in float4 p/2 = {cos_2q, cos_2q+1, sin_2q, sin_2q+1}
  for (int q = tid; q < M + 32; q += blockDim.x) {
    const float2 e = b.table32[(2 * q) % M], o = b.table32[(2 * q + 1) % M];
    reinterpret_cast<float4*>(tab)[q] = make_float4(e.x, o.x, e.y, o.y);
  }
#else
  for (int k = tid; k < 2 * M + 64; k += blockDim.x) tab[k] = b.table32[k % M];
#endif

  if (tid == 0) {  // initial band: CTAs split across bands in proportion to planned work
    unsigned long long total = 0;
    for (int q = 0; q < p.n_bands; ++q) total += b.band_work[q];
    int band = p.n_bands - 1;
    if (total > 0) {
      const double pos = ((double)blockIdx.x + 0.5) / gridDim.x * (double)total;
      double acc = 0;
      for (int q = 0; q < p.n_bands; ++q) {
        acc += (double)b.band_work[q];
        if (pos < acc) {
          band = q;
          break;
        }
      }
    }
    s_band = band;
  }
  vtrace(0, 0);
  for (size_t k = tid; k < p.tile_words; k += blockDim.x) tile[k] = 0u;
  __syncthreads();
  vtrace(1, s_band);
  unsigned int my_fb = 0;
  unsigned lt_mask = (1u << lane) - 1u;
  // per-lane table address (shared window): loaded by ld.shared below
  uint32_t tab_s = (uint32_t)__cvta_generic_to_shared(tab) + (RV_PACK ? 16u : 8u) * (uint32_t)lane;
  asm volatile("" : "+r"(lt_mask), "+r"(tab_s), "+r"(fbq_s));
  // opaque to the optimizer: otherwise the shared-window base is rematerialised every step
  uint32_t tile_s = (uint32_t)__cvta_generic_to_shared(tile);
  // deposits outside this band's rows go to tile rows >= hb (never flushed) or, beyond the tile,
  // to this lane's sink word: addr = tile + 4 * min(rel, tile_words + lane)
  uint32_t sink_rel = (uint32_t)p.tile_words + (uint32_t)lane;
  uint32_t vote2 = 2u;
  asm volatile("" : "+r"(tile_s), "+r"(sink_rel), "+r"(vote2));
  const float CMf = p.CMf;
  const int W = p.W, G = p.G;
  const int S = p.frac_shift;
  const uint32_t fmask = p.frac_mask;
  FbCtx fc;
  fc.zx = b.zx;
  fc.zy = b.zy;
  fc.zz = b.zz;
  fc.table64 = b.table64;
  fc.grid = b.grid;
  fc.E = p.E;
  fc.inv_cell = p.inv_cell;
  fc.G = G;
  fc.halfJ = M;
  fc.c_min = p.c_min;
  fc.W = W;

  for (;;) {
    const int band = s_band;
    if (band < 0) break;
    const int r0 = p.band_r0[band], hb = p.band_r0[band + 1] - r0;
    fc.own_lo = band == 0 ? 0 : r0;
    fc.own_hi = band == p.n_bands - 1 ? G : r0 + hb;
    const int row_off = p.magic_hi + r0;      // row_local = (bits_y >> S) - row_off
    const int col_off = p.magic_hi + p.c_min; // col_local = (bits_x >> S) - col_off
    const uint32_t lin_off = (uint32_t)row_off * (uint32_t)W + (uint32_t)col_off;
    const uint32_t tile_cells = (uint32_t)hb * (uint32_t)W;
    F32Geom geo;
    geo.CMf = CMf;
    geo.S = S;  // (run-time copy; kS != 0 overrides)
    geo.fmask = fmask;
    geo.W = (uint32_t)W;
    geo.lin_off = lin_off;
    geo.magic_hi = p.magic_hi;
    geo.G = G;
    geo.r0 = r0;
    geo.c_min = p.c_min;
    const unsigned long long* ebase = b.entries + (int64_t)band * b.entry_cap;
    const int n_ent = b.entry_count[band];
    int* counter = &b.counters[1 + band];
    // grab size: 32 entries when every warp of the launch still gets several grabs, smaller for
    // small problems (otherwise a handful of warps would walk all entries while the rest idle)
    const int per = (int)(((long long)gridDim.x * (kVoteThreads / 32) * 4) / p.n_bands);
    const int grab = max(1, min(32, n_ent / max(per, 1)));
    VoteCtx v{tab, tab_s, tile, tile_s, sink_rel, vote2, fbq_s, lt_mask, M, tile_cells, hb, b.basis_a, b.basis_b, grab};
    vote_entries<kClamp, kS>(v, geo, fc, [&](int j) { return __ldcs(ebase + j); }, n_ent, counter, my_fb);
    // band exhausted for this CTA: flush the tile to a partial slot, steal the next band
    __syncthreads();
    vtrace(2, band);
    if (p.bulk && warp == 0) {
      // the TMA engine adds each tile row (G words; tile row stride W = G + 4 keeps the ATOMS
      // bank spread) into its grid row (L2 reduce-adds, integer: order-free); the lanes wait only
      // until the tile has been read, then it can be cleared
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      const unsigned long long dst = reinterpret_cast<unsigned long long>(b.grid + (size_t)r0 * G);
      for (int r = lane; r < hb; r += 32)
        asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.u32 [%0], [%1], %2;" ::"l"(
                         dst + (unsigned long long)r * (unsigned)G * 4u),
                     "r"(tile_s + (uint32_t)r * (uint32_t)W * 4u), "r"((uint32_t)G * 4u)
                     : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    }
    if (tid == 0) {
      if (p.bulk) {
        s_slot = b.max_slots;  // no partial slot
      } else {
        const int slot = atomicAdd(&b.counters[0], 1);
        s_slot = slot;
        if (slot < b.max_slots) b.slot_band[slot] = band;
      }
      int best = -1;
      long long best_rem = 0;
      for (int q = 0; q < p.n_bands; ++q) {
        const long long rem = (long long)b.entry_count[q] - *((volatile int*)&b.counters[1 + q]);
        if (rem > best_rem) {
          best_rem = rem;
          best = q;
        }
      }
      s_band = best;
    }
    __syncthreads();
    const int slot = s_slot;
    const size_t words = (size_t)hb * W;
    if (p.bulk) {
      // flushed by the bulk reduce above
    } else if (slot < b.max_slots) {
      uint4* dst = reinterpret_cast<uint4*>(b.partials + (size_t)slot * p.tile_words);
      const uint4* src = reinterpret_cast<const uint4*>(tile);
      for (size_t k = tid; k < (words + 3) / 4; k += blockDim.x) __stcg(dst + k, src[k]);
    } else {  // cannot happen (a CTA visits each band at most once); stay exact anyway
      for (size_t k = tid; k < words; k += blockDim.x)
        if (tile[k]) atomicAdd(&b.grid[(size_t)(r0 + k / W) * G + p.c_min + k % W], tile[k]);
    }
    __syncthreads();
    vtrace(3, band);
    if (s_band >= 0)
      for (size_t k = tid; k < p.tile_words; k += blockDim.x) tile[k] = 0u;
    __syncthreads();
  }
  vtrace(4, 0);
  if (p.bulk && warp == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // flushes landed
  if (lane == 0 && my_fb) atomicAdd(&b.stats[1], (unsigned long long)my_fb);
}

// Sum the partial tiles of every band into the output grid.
constexpr int kRedGroups = RV_RED_GROUPS;  // slot groups per block
constexpr int kRedVecs = kReduceThreads / kRedGroups;
__global__ void __launch_bounds__(kReduceThreads) vote_reduce_kernel(VotePlan p, VoteBuffers b) {
  __shared__ int s_slots[1024];
  __shared__ int s_n;
  const int band = blockIdx.y;
  const int r0 = p.band_r0[band], hb = p.band_r0[band + 1] - r0;
  const int words = hb * p.W;
  int used = min(b.counters[0], b.max_slots);
  if (threadIdx.x == 0) s_n = 0;
  __syncthreads();
  // slot list of this band (order irrelevant: integer sums)
  for (int s = threadIdx.x; s < used; s += blockDim.x) {
    if (b.slot_band[s] == band) {
      const int k = atomicAdd(&s_n, 1);
      if (k < 1024) s_slots[k] = s;
    }
  }
  __syncthreads();
  const int ns = s_n;
  const bool fused = b.red_out != nullptr;
  unsigned long long best = 0, gsum = 0;
  // 4 words per thread (tile_words is a multiple of 4: slots are 16-byte aligned); the block's
  // threads form kRedGroups slot groups over kRedVecs vectors (more loads in flight per vector),
  // combined through shared memory
  const int nv = (words + 3) / 4;
  const int vl = threadIdx.x % kRedVecs, g = threadIdx.x / kRedVecs;
  __shared__ uint4 s_acc[kRedGroups - 1][kRedVecs];
  for (int v0 = blockIdx.x * kRedVecs; v0 < nv; v0 += gridDim.x * kRedVecs) {
    const int v = v0 + vl;
    uint4 acc = make_uint4(0u, 0u, 0u, 0u);
    if (v < nv) {
      auto add = [&](int slot) {
        const uint4 x = __ldcs(reinterpret_cast<const uint4*>(b.partials + (size_t)slot * p.tile_words) + v);
        acc.x += x.x;
        acc.y += x.y;
        acc.z += x.z;
        acc.w += x.w;
      };
      if (ns <= 1024) {
#pragma unroll 4
        for (int k = g; k < ns; k += kRedGroups) add(s_slots[k]);
      } else {
        for (int s = g; s < used; s += kRedGroups)
          if (b.slot_band[s] == band) add(s);
      }
    }
    if (g > 0) s_acc[g - 1][vl] = acc;
    __syncthreads();
    if (g == 0 && v < nv) {
#pragma unroll
      for (int q = 0; q < kRedGroups - 1; ++q) {
        const uint4 x = s_acc[q][vl];
        acc.x += x.x;
        acc.y += x.y;
        acc.z += x.z;
        acc.w += x.w;
      }
      const uint32_t a4[4] = {acc.x, acc.y, acc.z, acc.w};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int w = 4 * v + i;
        if (w < words && w % p.W <= p.c_max - p.c_min) {  // (bulk tiles: padded row stride)
          const int row = r0 + w / p.W, col = p.c_min + w % p.W;
          const size_t gi = (size_t)row * p.G + col;
          if (fused) {  // final cell value (the exact path may have added to the global grid)
            const uint32_t val = b.grid[gi] + a4[i];
            if (a4[i]) b.grid[gi] = val;
            gsum += val;
            if (val) best = max(best, ((unsigned long long)val << 32) | (0xFFFFFFFFu - (uint32_t)gi));
          } else if (a4[i]) {
            b.grid[gi] += a4[i];
          }
        }
      }
    }
    __syncthreads();
  }
  if (!fused) return;
  // fused find_peaks(K=1) argmax + exactness-guard sum (argmax_kernel's key: count, then lowest
  // index), and on the last block estimate_from_peak (exact_peak_axis)
  __shared__ unsigned long long s_best[kReduceThreads / 32], s_sum[kReduceThreads / 32];
  __shared__ bool s_last;
  for (int o = 16; o > 0; o >>= 1) {
    best = max(best, __shfl_xor_sync(0xFFFFFFFFu, best, o));
    gsum += __shfl_xor_sync(0xFFFFFFFFu, gsum, o);
  }
  if ((threadIdx.x & 31) == 0) {
    s_best[threadIdx.x >> 5] = best;
    s_sum[threadIdx.x >> 5] = gsum;
  }
  __syncthreads();
  const unsigned nblk = gridDim.x * gridDim.y, bid = blockIdx.y * gridDim.x + blockIdx.x;
  if (threadIdx.x == 0) {
    unsigned long long bb = 0, ss = 0;
    for (int w = 0; w < kReduceThreads / 32; ++w) {
      bb = max(bb, s_best[w]);
      ss += s_sum[w];
    }
    __stcg(b.red_keys + 2 * bid, bb);
    __stcg(b.red_keys + 2 * bid + 1, ss);
    __threadfence();
    s_last = atomicAdd(b.red_done, 1u) == nblk - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  best = 0;
  gsum = 0;
  for (unsigned k = threadIdx.x; k < nblk; k += blockDim.x) {
    best = max(best, __ldcg(b.red_keys + 2 * k));
    gsum += __ldcg(b.red_keys + 2 * k + 1);
  }
  for (int o = 16; o > 0; o >>= 1) {
    best = max(best, __shfl_xor_sync(0xFFFFFFFFu, best, o));
    gsum += __shfl_xor_sync(0xFFFFFFFFu, gsum, o);
  }
  __syncthreads();
  if ((threadIdx.x & 31) == 0) {
    s_best[threadIdx.x >> 5] = best;
    s_sum[threadIdx.x >> 5] = gsum;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long bb = 0, ss = 0;
    for (int w = 0; w < kReduceThreads / 32; ++w) {
      bb = max(bb, s_best[w]);
      ss += s_sum[w];
    }
    b.red_out[0] = bb;
    b.red_out[1] = ss;
    *b.red_done = 0u;
    if (b.peak) exact_peak_axis(bb, ss, b.grid, p.G, p.E, b.peak_min_votes, b.peak);
  }
}

// Exact generic vote: one warp per constraint, lanes over samples, global atomics.
__global__ void __launch_bounds__(256) vote_generic_kernel(VotePlan p, const double* zx, const double* zy,
                                                           const double* zz, const double2* table64,
                                                           uint32_t* grid, int64_t n) {
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= n) return;
  double a1[3], a2[3];
  exact_basis(zx[w], zy[w], zz[w], a1, a2);
  for (int j = lane; j < p.J; j += 32) {
    const double2 cs = table64[j];
    int row, col;
    exact_sample(a1, a2, cs.x, cs.y, p, &row, &col);
    atomicAdd(&grid[(size_t)row * p.G + col], 1u);
  }
}

__global__ void deposit_one_kernel(VotePlan p, const double* z3, const double2* table64, uint32_t* grid) {
  double a1[3], a2[3];
  exact_basis(z3[0], z3[1], z3[2], a1, a2);
  for (int j = threadIdx.x; j < p.J; j += blockDim.x) {
    const double2 cs = table64[j];
    int row, col;
    exact_sample(a1, a2, cs.x, cs.y, p, &row, &col);
    atomicAdd(&grid[(size_t)row * p.G + col], 1u);
  }
}

}  // namespace

void launch_plan(const VotePlan& p, const VoteBuffers& b, int64_t n, cudaStream_t s) {
  const int threads = 256;
  const int64_t blocks = (n + threads - 1) / threads;
  if (p.n_bands <= 8)
    plan_kernel<8><<<(unsigned)blocks, threads, 0, s>>>(p, b, n);
  else
    plan_kernel<0><<<(unsigned)blocks, threads, 0, s>>>(p, b, n);
}

using VoteKernel = void (*)(VotePlan, VoteBuffers, int64_t);
static VoteKernel vote_kernel_for(const VotePlan& p, int* slot) {
  // S = 13 / 12 (every grid <= 1000 at the reference extents) get a compile-time shift; other S
  // use the run-time variant
  const int ks = p.frac_shift == 13 ? 2 : (p.frac_shift == 12 ? 1 : 0);
  const int k = (p.clamp ? 3 : 0) + ks;
  *slot = k;
  switch (k) {
    case 0: return vote_banded_kernel<false, 0>;
    case 1: return vote_banded_kernel<false, 12>;
    case 2: return vote_banded_kernel<false, 13>;
    case 3: return vote_banded_kernel<true, 0>;
    case 4: return vote_banded_kernel<true, 12>;
    default: return vote_banded_kernel<true, 13>;
  }
}

cudaError_t set_vote_smem(const VotePlan& p) {
  // largest dynamic smem opted in, per (device, instantiation): the attribute is per device, and
  // worker threads of one process (batch API) may race here
  constexpr int kDevs = 16;
  static int configured[kDevs][6] = {};
  static std::mutex mu;
  int dev = 0;
  cudaGetDevice(&dev);
  int k;
  VoteKernel f = vote_kernel_for(p, &k);
  std::lock_guard<std::mutex> lock(mu);
  int* slot = dev >= 0 && dev < kDevs ? &configured[dev][k] : nullptr;
  if (slot && (int)p.smem_bytes <= *slot) return cudaSuccess;
  const cudaError_t e =
      cudaFuncSetAttribute(reinterpret_cast<const void*>(f), cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)p.smem_bytes);
  if (e == cudaSuccess && slot) *slot = (int)p.smem_bytes;
  return e;
}

void launch_vote_banded(const VotePlan& p, const VoteBuffers& b, int64_t n, int n_ctas, cudaStream_t s) {
  int k;
  VoteKernel f = vote_kernel_for(p, &k);
  f<<<n_ctas, kVoteThreads, p.smem_bytes, s>>>(p, b, n);
}

int vote_reduce_blocks_x(const VotePlan& p) {
  const int vecs = (p.H_max * p.W + 3) / 4;
  return min((vecs + kRedVecs - 1) / kRedVecs, 1024);
}

void launch_vote_reduce(const VotePlan& p, const VoteBuffers& b, cudaStream_t s) {
  dim3 grid((unsigned)vote_reduce_blocks_x(p), (unsigned)p.n_bands);
  vote_reduce_kernel<<<grid, kReduceThreads, 0, s>>>(p, b);
}

void launch_vote_generic(const VotePlan& p, const VoteBuffers& b, int64_t n, cudaStream_t s) {
  const int threads = 256;
  const int64_t blocks = (n * 32 + threads - 1) / threads;
  vote_generic_kernel<<<(unsigned)blocks, threads, 0, s>>>(p, b.zx, b.zy, b.zz, b.table64, b.grid, n);
}

// Small counter reset as a kernel: a cudaMemsetAsync can queue behind a concurrent H2D on the
// copy engine (pipelined host-input path).
__global__ void zero_i32_kernel(int32_t* p, int n) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) p[i] = 0;
}
void launch_zero_i32(int32_t* p, int n, cudaStream_t s) { zero_i32_kernel<<<1, 256, 0, s>>>(p, n); }

void launch_deposit_one(const VotePlan& p, const double* z3, const double2* table64, uint32_t* grid,
                        cudaStream_t s) {
  deposit_one_kernel<<<1, 256, 0, s>>>(p, z3, table64, grid);
}

}  // namespace rvb

#ifdef RV_VOTE_TRACE
extern "C" int rv_debug_vote_trace(unsigned long long* out, int max_events) {
  unsigned int n = 0;
  cudaMemcpyFromSymbol(&n, rvb::g_vtrace_n, sizeof n);
  if (n > 65536) n = 65536;
  if ((int)n > max_events) n = (unsigned)max_events;
  cudaMemcpyFromSymbol(out, rvb::g_vtrace, sizeof(unsigned long long) * 2 * n);
  const unsigned int zero = 0;
  cudaMemcpyToSymbol(rvb::g_vtrace_n, &zero, sizeof zero);
  return (int)n;
}
#endif
