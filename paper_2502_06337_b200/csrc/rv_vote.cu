// K1 (band plan) and K2 (band-tiled vote) of the spatial-voting path.
//
// Reference semantics (voting.cpp:25-45, :88-118): every constraint z deposits exactly J
// votes, one per sample theta_j = -pi + j*2pi/J of the great circle {v : z.v = 0}; each
// sample is flipped to the southern hemisphere (iff c > 0), stereographically projected and
// counted in its cell of a G x G uint32 grid. The device result is BIT-EXACT with that definition:
//
//  * Canonical half circle. Samples j and j+J/2 are antipodal; after the flip they land on the
//    same plane point (up to ~1e-15). Exactly one of each pair has c <= 0 (is "canonical"), and
//    the canonical samples form J/2 consecutive sample indices j0 .. j0+J/2-1 (mod J). K1 finds j0
//    with the reference's own f64 test (so K2 never decides a hemisphere), deposits the rare pairs
//    with both / neither twin canonical (|c| at the rounding level) exactly, and K2 evaluates
//    only canonical samples, depositing 2 each.
//  * f32 filter + exact f64 fallback. A sample is evaluated in f32 from an f64 basis; the cell
//    coordinate t is produced on a 2^-S grid (S <= 13, chosen per geometry by make_plan) by one
//    FFMA against a magic constant. |t32 - t64| <= K*6e-7 + 2^-(S+1) cells, so
//    whenever t32 is at least 2*2^-S from an integer the f32 cell IS the reference cell.
//    Otherwise the sample is queued and both twins are recomputed exactly in f64 (same op order,
//    no FMA) -- ~0.15% of samples.
//  * Band tiling. The grid's reachable rows are split into bands that fit one CTA's shared
//    memory (u32 counters, 1 CTA/SM). K1 computes per (constraint, band) the canonical sample
//    ranges whose projected points can fall in the band (analytic circle/line intersection,
//    padded), so K2 only evaluates samples near its band; an exact ownership test on the row
//    decides the deposit, so a sample is counted by exactly one band.
//  * Tiles are flushed once per (CTA, band) into the grid by TMA bulk reduce-adds (or partial
//    slots summed by a reduction kernel): integer sums, order-free, deterministic.
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
#ifndef RV_BCAST_REDUX
#define RV_BCAST_REDUX 1  // 0: broadcast each entry with shuffles (A/B knob; REDUX measured ~1.5% faster)
#endif
#ifndef RV_UNIFORM_STEP
#define RV_UNIFORM_STEP 1
#endif
#ifndef RV_GRAB_PER
#define RV_GRAB_PER 4  // target grabs per warp and band below which grabs shrink from 32 entries
#endif
#ifndef RV_BAND_ENTRY_W
#define RV_BAND_ENTRY_W 110  // per-entry cost (in samples) in the initial CTA-to-band split (A/B: 0 -> 110 is -1.8% vote time at C3, -0.8% at C4)
#endif
#ifndef RV_RED_GROUPS
#define RV_RED_GROUPS 2
#endif

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
__device__ __forceinline__ f32x2 fma2_rz(f32x2 a, f32x2 b, f32x2 c) {
  f32x2 r;
  asm("fma.rz.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ f32x2 add2(f32x2 a, f32x2 b) {
  f32x2 r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f32x2 add2_rm(f32x2 a, f32x2 b) {
  f32x2 r;
  asm("add.rm.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f32x2 add2_rz(f32x2 a, f32x2 b) {
  f32x2 r;
  asm("add.rz.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
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
__device__ __forceinline__ void sts_u2(uint32_t saddr, uint32_t a, uint32_t b) {
  asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(saddr), "r"(a), "r"(b) : "memory");
}
__device__ __forceinline__ uint2 lds_u2(uint32_t saddr) {
  uint2 v;
  asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(saddr) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t lds_u32(uint32_t saddr) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(saddr) : "memory");
  return v;
}

// f32 evaluation of one canonical sample: tile-relative linear cell index `rel` (>= tile_cells: not
// this band's tile) and whether the f32 cell is not provably the reference cell. The sample is
// canonical (c <= 0 in the reference's own arithmetic, decided by the planner), so there is no
// hemisphere logic: c' = 1 - c from two FFMAs off the constant 1, r = rcp.approx(c'). Shared by the
// hot loop (packed, f32_cell2) and the exact path (which undoes the hot loop's deposit), so both
// see identical values.
struct F32Geom {
  float CMf;
  int S;
  uint32_t fmask;
  uint32_t W;
  uint32_t lin_off;  // non-clamp: (magic_hi + r0) * W + magic_hi + c_min
  int magic_hi, G, r0, c_min;
  float Wf;         // RV_FP_CELL: (float)W
  uint32_t fp_off;  // RV_FP_CELL: bits(2^23) + magic + r0 * W + c_min
};
// RV_FP_CELL (A/B knob, off: measured slower): the fixed-S no-clamp variants compute the
// tile-relative cell in f32 instead of shifting and multiplying the fixed-point bits (8 instead of
// 10 issue slots per sample pair, but 4 more FMA-pipe ops and a longer dependent chain):
//   F = (ty + (1.5*2^23 - magic)) rounded down - 1.5*2^23 = floor(t_y), exact
//   L = F*W + tx rounded toward zero (all terms >= 0, L < 2^23): floor(L) = row*W + floor(t_x) + magic
//   bits(L + 2^23, toward zero) = bits(2^23) + floor(L)
#ifndef RV_FP_CELL
#define RV_FP_CELL 0
#endif
template <bool kClamp, int kS>
struct FpCellSel : std::integral_constant<bool, RV_FP_CELL && !kClamp && kS != 0> {};
constexpr float kBig23 = 8388608.f;   // 2^23
constexpr float kBig15 = 12582912.f;  // 1.5 * 2^23
template <int kS>
__device__ __forceinline__ constexpr float fp_ky() { return kBig15 - 1.5f * (float)(1 << (23 - kS)); }
template <bool kClamp, int kS>
__device__ __forceinline__ uint32_t cell_of_bits(const F32Geom& g, uint32_t bx, uint32_t by, bool* flag) {
  const int S = kS ? kS : g.S;
  *flag = ((bx & g.fmask) == 0u) | ((by & g.fmask) == 0u);
  if (FpCellSel<kClamp, kS>::value) {
    const float F = __fadd_rn(__fadd_rd(__uint_as_float(by), fp_ky<kS>()), -kBig15);
    const float L = __fmaf_rz(F, g.Wf, __uint_as_float(bx));
    return __float_as_uint(__fadd_rz(L, kBig23)) - g.fp_off;
  }
  // the column is always inside [c_min, c_min+W) (|X| <= 1 < extent, or clamped), so one
  // unsigned range test on the linear index is the band-ownership test
  if (kClamp) {
    const int row = min(max((int)(by >> S) - g.magic_hi, 0), g.G - 1) - g.r0;
    const int col = min(max((int)(bx >> S) - g.magic_hi, 0), g.G - 1) - g.c_min;
    return (uint32_t)(row * (int)g.W + col);
  }
  return (by >> S) * g.W + (bx >> S) - g.lin_off;
}
// ba = (K a1x, K a1y, -a1z, K a2x), bb = (K a2y, -a2z), t = (cos, sin) of the sample
template <bool kClamp, int kS>
__device__ __forceinline__ uint32_t f32_cell(const F32Geom& g, float4 ba, float2 bb, float2 t, bool* flag) {
  const float xk = fmaf(ba.w, t.y, ba.x * t.x);
  const float yk = fmaf(bb.x, t.y, ba.y * t.x);
  const float cp = fmaf(bb.y, t.y, fmaf(ba.z, t.x, 1.f));
  const float r = rcp_approx(cp);
  const uint32_t bx = (uint32_t)__float_as_int(fmaf(xk, r, g.CMf));
  const uint32_t by = (uint32_t)__float_as_int(fmaf(yk, r, g.CMf));
  return cell_of_bits<kClamp, kS>(g, bx, by, flag);
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
__device__ __forceinline__ float sqrt_approx(float x) {  // MUFU.SQRT, ~1 ulp: fine for culling
  float r;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
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
  const float r = sqrt_approx(1.f - ax) * p;
  return x < 0.f ? kPiF - r : r;
}

// One band boundary (level y0) in SAMPLE space on the whole circle (sample u <-> theta = -pi +
// u * step). For every sample, Y >= y0 on the canonical arc (where 1 - c > 0) is equivalent to
// A cos(theta) + B sin(theta) >= y0 with A = a1y + y0 a1z, B = a2y + y0 a2z -- on the whole circle
// this is the stereographic image of the UNflipped point, so the level sets of all boundaries are
// single arcs centred at atan2(B, A), NESTED in y0. A, B and y0 carry f32 errors (~4e-7 absolute),
// so the two uses solve shifted levels: the OUTER arc (a superset: the band above) solves
// y0 - kArcSlack and is dilated, the INNER arc (a subset: the band below subtracts it) solves
// y0 + kArcSlack and is eroded -- by kArcDilate (>> the fast-trig error, incl. near tangency) plus
// kPad samples. This keeps both sides right where the level is ill-conditioned: near-tangent
// visits, and a near-constant A cos + B sin (R ~ 0: z = +-e2 has Y == 0 on a band boundary).
// State: 0 empty, 1 the whole circle, 2 the arc [lo, hi] (integers, unwrapped around c).
struct Bnd {
  int olo, ohi, ilo, ihi;
  int ost, ist;
  float c;
};
constexpr float kArcDilate = 2e-3f;  // rad, >> acos/atan2_fast error near tangency (~8e-4 rad)
constexpr float kArcSlack = 2e-6f;   // plane units, >> the f32 error of A cos + B sin - y0
__device__ __forceinline__ Bnd band_boundary(float A, float B, float y0, float inv_step, float pad_s, int J) {
  Bnd r;
  const float R = sqrt_approx(fmaf(A, A, B * B));
  const float lo = y0 - kArcSlack, hi = y0 + kArcSlack;
  float r_sup, r_sub;
  if (R > 0.f) {
    const float inv = __fdividef(1.f, R);
    r_sup = lo * inv;
    r_sub = hi * inv;
  } else {  // constant 0 >= level: decided by the level's sign
    r_sup = lo <= 0.f ? -2.f : 2.f;
    r_sub = hi <= 0.f ? -2.f : 2.f;
  }
  r.ost = r_sup <= -1.f ? 1 : (r_sup < 1.f ? 2 : 0);
  r.ist = r_sub <= -1.f ? 1 : (r_sub < 1.f ? 2 : 0);
  r.c = (atan2_fast(B, A) + kPiF) * inv_step;
  const float wo = acos_fast(fmaxf(r_sup, -1.f)) * inv_step + pad_s;
  const float wi = acos_fast(fminf(r_sub, 1.f)) * inv_step - pad_s;
  r.olo = __float2int_rd(r.c - wo);
  r.ohi = __float2int_ru(r.c + wo);
  if (r.ost == 2 && r.ohi - r.olo + 1 >= J) r.ost = 1;  // the dilated arc covers the circle
  r.ilo = __float2int_ru(r.c - wi);
  r.ihi = __float2int_rd(r.c + wi);
  if (r.ist == 2 && r.ilo > r.ihi) r.ist = 0;  // eroded to nothing
  return r;
}

// Up to two inclusive sample runs (increasing) inside the canonical arc [A0, A1] (n = 0, 1, 2).
struct Runs2 {
  int l0, h0, l1, h1, n;
};
// Entries (start | len << 16, start in [0, J)) of one band: e0 / e1 from the first / second run,
// e2 the part of a run past the wrap at J (at most one run crosses J); zero = none.
struct Ent3 {
  uint32_t e0, e1, e2;
};

// The part of the circle run [x, y] (y - x < J) inside the canonical arc [A0, A1] (unwrapped,
// A1 - A0 < J): a main piece [m_lo, m_hi] and, when the run wraps past A0 + J, the piece
// [A0, w_hi] at the arc start (empty pieces: m_lo > m_hi, w_hi < A0).
__device__ __forceinline__ void canon_pieces(int x, int y, int A0, int A1, int J, int* m_lo, int* m_hi,
                                             int* w_hi) {
  int t = x - A0;  // in (-2J, 2J): reduce mod J without a division
  t += t < 0 ? J : 0;
  t += t < 0 ? J : 0;
  t -= t >= J ? J : 0;
  const int xs = A0 + t, ys = xs + (y - x);
  *m_lo = xs;
  *m_hi = min(ys, A1);
  *w_hi = min(A1, ys - J);
}

// Sample runs of band b inside the canonical arc: the outer arc of its lower boundary minus the
// inner arc of its upper boundary (nested on the circle: at most two circle runs), intersected
// with [A0, A1]. The pieces are disjoint; touching ones are merged, and three are merged to two
// across the smaller gap (a superset: the vote's row test decides every deposit). Straight-line
// code (selects): the warp's lanes stay converged.
__device__ __forceinline__ Runs2 band_runs(const Bnd& lo_b, const Bnd& hi_b, int A0, int A1, int J) {
  const bool none = lo_b.ost == 0 || hi_b.ist == 1 || A0 > A1;
  const bool in_empty = hi_b.ist == 0, out_full = lo_b.ost == 1;
  const float d = hi_b.c - lo_b.c;  // the inner arc next to the outer one (same turn)
  const int sh = d > 0.5f * (float)J ? -J : (d < -0.5f * (float)J ? J : 0);
  // circle run 0: the outer arc, the whole circle from A0, the circle minus the inner arc, or the
  // part of the outer arc before the inner one; circle run 1: the part after it
  const int x0 = out_full ? (in_empty ? A0 : hi_b.ihi + 1) : lo_b.olo;
  const int y0 = out_full ? (in_empty ? A0 + J - 1 : hi_b.ilo - 1 + J) : (in_empty ? lo_b.ohi : hi_b.ilo + sh - 1);
  const int x1 = hi_b.ihi + sh + 1, y1 = lo_b.ohi;
  const bool v0 = !none && x0 <= y0, v1 = !none && !out_full && !in_empty && x1 <= y1;
  int m0lo, m0hi, w0, m1lo, m1hi, w1;
  canon_pieces(x0, y0, A0, A1, J, &m0lo, &m0hi, &w0);
  canon_pieces(x1, y1, A0, A1, J, &m1lo, &m1hi, &w1);
  // pieces in increasing order: the wrapped one at A0 (at most one run wraps), then the mains
  const int wh = max(v0 ? w0 : A0 - 1, v1 ? w1 : A0 - 1);
  const bool pw = wh >= A0;
  const bool p0 = v0 && m0lo <= m0hi, p1 = v1 && m1lo <= m1hi;
  const bool sw = p1 && (!p0 || m1lo < m0lo);
  const int alo = sw ? m1lo : m0lo, ahi = sw ? m1hi : m0hi, blo = sw ? m0lo : m1lo, bhi = sw ? m0hi : m1hi;
  const bool pa = p0 || p1, pb = p0 && p1;
  // compact the valid pieces into c0 <= c1 (<= the third, blo..bhi)
  const int c0lo = pw ? A0 : alo, c0hi = pw ? wh : ahi;
  const int c1lo = pw ? alo : blo, c1hi = pw ? ahi : bhi;
  const int k = (int)pw + (int)pa + (int)pb;
  Runs2 r{c0lo, c0hi, c1lo, c1hi, min(k, 2)};
  if (k == 3) {  // merge across the smaller gap
    if (c1lo - c0hi <= blo - c1hi) {
      r.h0 = c1hi;
      r.l1 = blo;
      r.h1 = bhi;
    } else {
      r.h1 = bhi;
    }
  }
  if (r.n == 2 && r.l1 <= r.h0 + 1) {  // touching
    r.h0 = max(r.h0, r.h1);
    r.n = 1;
  }
  return r;
}

// Final entries of one band from its (<= 2) runs inside the canonical arc [A0, A1] (A0 even, A1
// odd): each run is widened to an even start and a whole number of 64-sample steps where the arc
// and the neighbouring run leave room (extra samples are canonical and land outside the band, in
// the vote's sink -- they never overlap another entry of this constraint and band, so nothing is
// counted twice), then split where the sample index wraps at J, at a step boundary (the last step
// before the wrap reads the table's 64-sample slack), so the vote's step grid never shifts.
// Straight-line over two run slots.
__device__ __forceinline__ void finalize_run(int lo, int hi, int prev_hi, int ub, int J, uint32_t* ea, uint32_t* eb,
                                             int* hi_out, uint32_t* work) {
  lo = max(lo & ~1, prev_hi + 1);
  hi |= 1;
  int need = ((hi - lo + 64) & ~63) - (hi - lo + 1);
  const int up = min(need, ub - hi);
  hi += up;
  need -= up;
  lo -= min(need, lo - (prev_hi + 1));
  *hi_out = hi;
  *work += (uint32_t)((hi - lo + 64) & ~63);
  const int cut = lo + (((J - lo) + 63) & ~63);  // first step boundary at or after J
  const bool below = hi < J, above = lo >= J, split = !below && !above && cut <= hi;
  const int s0 = above ? lo - J : lo, h0 = above ? hi - J : (split ? cut - 1 : hi);
  *ea = (uint32_t)s0 | ((uint32_t)(h0 - s0 + 1) << 16);
  *eb = split ? ((uint32_t)(cut - J) | ((uint32_t)(hi - cut + 1) << 16)) : 0u;
}
__device__ __forceinline__ Ent3 finalize_runs(const Runs2& runs, int A0, int A1, int J, uint32_t* work) {
  Ent3 o{0u, 0u, 0u};
  uint32_t a0, b0, a1, b1;
  int h0, h1;
  uint32_t w0 = 0, w1 = 0;
  finalize_run(runs.l0, runs.h0, A0 - 1, runs.n == 2 ? (runs.l1 & ~1) - 1 : A1, J, &a0, &b0, &h0, &w0);
  finalize_run(runs.l1, runs.h1, h0, A1, J, &a1, &b1, &h1, &w1);
  const bool one = runs.n >= 1, two = runs.n == 2;
  *work += (one ? w0 : 0u) + (two ? w1 : 0u);
  o.e0 = one ? a0 : 0u;
  o.e1 = two ? a1 : 0u;
  o.e2 = (one ? b0 : 0u) | (two ? b1 : 0u);
  return o;
}

// Reference hemisphere decision (voting.cpp:36-38: flip iff c > 0) of sample j in [0, 2J).
__device__ __forceinline__ bool canonical(const double a1[3], const double a2[3], const double2* t64, int j, int J) {
  const double2 cs = t64[j >= J ? j - J : j];
  return !(xa(xm(a1[2], cs.x), xm(a2[2], cs.y)) > 0.0);
}

// One sample exactly (f64, reference op order) into the global grid.
__device__ __forceinline__ void exact_global(const double a1[3], const double a2[3], const double2* t64, int j,
                                             const VotePlan& p, uint32_t* grid) {
  const double2 cs = t64[j >= p.J ? j - p.J : j];
  int row, col;
  exact_sample(a1, a2, cs.x, cs.y, p, &row, &col);
  atomicAdd(&grid[(size_t)row * p.G + col], 1u);
}

// K1b: per constraint, the exact f64 basis (orthonormal_basis, geom.cpp:36-43) and its f32 copy for
// the vote; the CANONICAL half circle in sample space -- the J/2 consecutive samples j0 .. j0+J/2-1
// whose hemisphere test c <= 0 holds in the reference's own f64 arithmetic (voting.cpp:36-38), so
// the vote never decides a hemisphere; and per row band the sample ranges whose projected points
// can fall in the band (band_boundary / band_runs: nested level arcs, padded, superset). The few
// pairs whose two twins are BOTH (or NEITHER) canonical -- |c| at the rounding level -- are
// deposited here exactly; constraints without a clean canonical half circle (z = +-e3 exactly:
// c == 0) are listed for the vote kernel's exact sample-by-sample path.
// kNB > 0: n_bands <= kNB, entries kept in shared memory and reserved once per (block, band)
// (same-address global atomics were the planner's bottleneck); kExact: n_bands == kNB (the band
// loop unrolled); kNB == 0: any band count, one reservation per (warp, band).
#ifndef RV_PLAN_THREADS
#define RV_PLAN_THREADS 256
#endif
constexpr int kPlanThreads = RV_PLAN_THREADS;
template <int kNB, bool kExact>
#ifndef RV_PLAN_MINB
#define RV_PLAN_MINB 5  // minimum resident plan blocks per SM: 48 registers (A/B: 1 -> 5 saves ~6 us at C3)
#endif
__global__ void __launch_bounds__(kPlanThreads, RV_PLAN_MINB) plan_kernel(VotePlan p, VoteBuffers b, int64_t n) {
  constexpr int kWarps = kPlanThreads / 32;
  __shared__ uint32_t s_wcnt[kMaxBands][kWarps], s_wwork[kMaxBands][kWarps];
  __shared__ int s_base[kMaxBands];
  const int64_t lo = b.bounds ? b.bounds[0] : b.range_lo, hi = b.bounds ? b.bounds[1] : b.range_lo + n;
  const int64_t i = lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double z0 = 0.0, z1 = 0.0, z2 = 0.0;
  if (i < hi) {
    z0 = b.zx[i];
    z1 = b.zy[i];
    z2 = b.zz[i];
  }
  bool valid = i < hi && !isnan(z0);  // in-order constraint sets mark dropped pairs with NaN
  const int M = p.halfJ, J = p.J;
  float f1y = 0.f, f2y = 0.f, f1z = 0.f, f2z = 0.f;  // fl32 of a1y, a2y, a1z, a2z (boundary solves)
  int A0 = 0, A1 = -1;  // canonical samples of the fast path: [A0, A1] (unwrapped, in [0, 2J))
  const float inv_step = 1.f / p.step_f;
  if (valid) {
    double a1[3], a2[3];
    exact_basis(z0, z1, z2, a1, a2);
    const double K = p.inv_cell;
    // the vote reads fl32(K * a_xy) (one rounding, like fl32(a_xy)) and fl32(-a_z): c' = 1 - c is
    // then two FFMAs from the constant 1
    const float4 fa = make_float4(__double2float_rn(a1[0] * K), __double2float_rn(a1[1] * K),
                                  __double2float_rn(-a1[2]), __double2float_rn(a2[0] * K));
    const float2 fb = make_float2(__double2float_rn(a2[1] * K), __double2float_rn(-a2[2]));
    b.basis_a[i] = fa;
    b.basis_b[i] = fb;
    f1y = __double2float_rn(a1[1]);
    f2y = __double2float_rn(a2[1]);
    f1z = __double2float_rn(a1[2]);
    f2z = __double2float_rn(a2[2]);
    // c(theta) = rc cos(theta - phi): the canonical arc (c <= 0) starts at theta_a = phi + pi/2,
    // sample coordinate pa in [J/4, 5J/4]; the exact start is the false -> true transition of
    // canonical(j), normally at ceil(pa), and the exact end normally M samples later
    const float theta_a = atan2_fast(f2z, f1z) + 0.5f * kPiF;
    const int jc = __float2int_ru((theta_a + kPiF) * inv_step);
    int j0 = -1, e = -1;
    if (!canonical(a1, a2, b.table64, jc - 1, J) && canonical(a1, a2, b.table64, jc, J) &&
        canonical(a1, a2, b.table64, jc + M - 1, J) && !canonical(a1, a2, b.table64, jc + M, J)) {
      j0 = jc;
      e = jc + M;
    } else {  // rare: |c| at the rounding level next to an end, or pa next to an integer
      unsigned sm = 0;
#pragma unroll
      for (int q = 0; q < 6; ++q) sm |= (unsigned)canonical(a1, a2, b.table64, jc - 3 + q, J) << q;
#pragma unroll
      for (int q = 1; q < 6; ++q)
        if (j0 < 0 && !((sm >> (q - 1)) & 1u) && ((sm >> q) & 1u)) j0 = jc - 3 + q;
      if (j0 >= 0) {  // exact end: first non-canonical sample after the arc (normally j0 + M)
        unsigned em = 0;
#pragma unroll
        for (int q = 0; q < 4; ++q) em |= (unsigned)canonical(a1, a2, b.table64, j0 + M - 2 + q, J) << q;
#pragma unroll
        for (int q = 1; q < 4; ++q)
          if (e < 0 && ((em >> (q - 1)) & 1u) && !((em >> q) & 1u)) e = j0 + M - 2 + q;
      }
    }
    if (j0 < 0 || e < 0 || f1z == 0.f && f2z == 0.f) {
      // no clean canonical half circle: every sample of this constraint goes the exact way
      const int k = atomicAdd(&b.counters[kDegenCount], 1);
      b.degen[k] = (int)i;
      valid = false;
    } else {
      A0 = j0;
      A1 = e - 1;
      if (e == j0 + M + 1) {  // pair j0: both twins canonical -> both deposited exactly, separately
        exact_global(a1, a2, b.table64, j0, p, b.grid);
        exact_global(a1, a2, b.table64, j0 + M, p, b.grid);
        A0 = j0 + 1;
        A1 = j0 + M - 1;
      } else if (e == j0 + M - 1) {  // pair j0 - 1: neither twin canonical
        exact_global(a1, a2, b.table64, j0 - 1, p, b.grid);
        exact_global(a1, a2, b.table64, j0 + M - 1, p, b.grid);
      }
      // the vote walks adjacent sample pairs from even indices: an odd first / even last sample of
      // the arc is deposited here exactly (both twins), so every entry can start even and end odd
      // (the f32 filter first, exactly as the vote evaluates it: an unflagged cell is the
      // reference cell of both twins; a flagged pair goes the exact way)
      F32Geom gg;
      gg.CMf = p.CMf;
      gg.S = p.frac_shift;
      gg.fmask = p.frac_mask;
      gg.W = (uint32_t)p.G;
      gg.lin_off = (uint32_t)p.magic_hi * (uint32_t)p.G + (uint32_t)p.magic_hi;
      gg.magic_hi = p.magic_hi;
      gg.G = p.G;
      gg.r0 = 0;
      gg.c_min = 0;
      auto exact_pair = [&](int j) {
        const int jj = j >= J ? j - J : j;
        bool fl;
        const uint32_t cell = p.clamp ? f32_cell<true, 0>(gg, fa, fb, b.table32[jj], &fl)
                                      : f32_cell<false, 0>(gg, fa, fb, b.table32[jj], &fl);
        if (!fl) {
          atomicAdd(&b.grid[cell], 2u);
          return;
        }
        const int q = jj % M;
        exact_global(a1, a2, b.table64, q, p, b.grid);
        exact_global(a1, a2, b.table64, q + M, p, b.grid);
      };
      if (A0 & 1) exact_pair(A0++);
      if (!(A1 & 1)) exact_pair(A1--);
    }
  }
  if (!valid) {
    A0 = 0;
    A1 = -1;  // no ranges
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned lt_mask = (1u << lane) - 1u;
  const unsigned long long ci = (unsigned long long)(uint32_t)i;
  const float pad_s = kArcDilate * inv_step + (float)kPad;
  Bnd b_lo;  // band 0's lower boundary: Y >= -inf, the whole circle
  b_lo.ost = 1;
  b_lo.ist = 1;
  b_lo.olo = b_lo.ohi = b_lo.ilo = b_lo.ihi = 0;
  b_lo.c = 0.f;
  // entries of this constraint in band `band` (+ planned samples into *w)
  auto plan_band = [&](int band, uint32_t* w) -> Ent3 {
    Bnd b_hi;  // the last band's upper boundary: Y >= +inf, empty
    b_hi.ost = 0;
    b_hi.ist = 0;
    b_hi.olo = b_hi.ohi = b_hi.ilo = b_hi.ihi = 0;
    b_hi.c = 0.f;
    if (band < (kExact ? kNB : p.n_bands) - 1) {
      const float y1 = p.band_ylo[band + 1];
      b_hi = band_boundary(fmaf(y1, f1z, f1y), fmaf(y1, f2z, f2y), y1, inv_step, pad_s, J);
    }
    const Runs2 runs = band_runs(b_lo, b_hi, A0, A1, J);
    b_lo = b_hi;  // the upper boundary of this band is the lower boundary of the next
    return finalize_runs(runs, A0, A1, J, w);
  };
  // warp-level bookkeeping of one band: this lane's entry offset inside the warp's block of
  // entries; the warp's count and planned samples are parked per (band, warp) for the block scan
  // (kNB > 0) or reserved in the global list directly (kNB == 0)
  auto book = [&](int band, const Ent3& r, uint32_t w, bool global) -> int {
    const unsigned m0 = __ballot_sync(0xFFFFFFFFu, r.e0 != 0u);
    const unsigned m1 = __ballot_sync(0xFFFFFFFFu, r.e1 != 0u);
    const unsigned m2 = __ballot_sync(0xFFFFFFFFu, r.e2 != 0u);
    const int total = __popc(m0) + __popc(m1) + __popc(m2);
    const unsigned ws = __reduce_add_sync(0xFFFFFFFFu, (unsigned)w);  // w <= J + 128 per lane
    int wbase = 0;
    if (global) {
      if (lane == 0 && total) wbase = atomicAdd(&b.entry_count[band], total);
      wbase = __shfl_sync(0xFFFFFFFFu, wbase, 0);
      if (lane == 0 && ws) atomicAdd(&b.band_work[band], (unsigned long long)ws);
    } else if (lane == 0) {
      s_wcnt[band][warp] = (uint32_t)total;
      s_wwork[band][warp] = ws;
    }
    return wbase + __popc(m0 & lt_mask) + __popc(m1 & lt_mask) + __popc(m2 & lt_mask);
  };
  auto emit = [&](int band, const Ent3& r, int64_t off) {
    unsigned long long* ep = b.entries + (int64_t)band * b.entry_cap + off;
    const int o1 = r.e0 != 0u, o2 = o1 + (r.e1 != 0u);  // the slots may have gaps: packed here
    if (r.e0) ep[0] = ci | ((unsigned long long)r.e0 << 32);
    if (r.e1) ep[o1] = ci | ((unsigned long long)r.e1 << 32);
    if (r.e2) ep[o2] = ci | ((unsigned long long)r.e2 << 32);
  };
  if constexpr (kNB > 0) {
    // per-thread entries/offsets parked in shared memory (a rolled band loop keeps the code small)
    __shared__ uint32_t s_r[kNB][3][kPlanThreads];
    __shared__ int s_off[kNB][kPlanThreads];
    const int nb = kExact ? kNB : p.n_bands;
#pragma unroll(kExact ? kNB : 1)
    for (int band = 0; band < nb; ++band) {  // uniform
      uint32_t w = 0;
      const Ent3 r = plan_band(band, &w);
      s_r[band][0][threadIdx.x] = r.e0;
      s_r[band][1][threadIdx.x] = r.e1;
      s_r[band][2][threadIdx.x] = r.e2;
      s_off[band][threadIdx.x] = book(band, r, w, false);
    }
    __syncthreads();
    // per band: the block's entries (one global reservation) and the warps' offsets inside it
    if (threadIdx.x < p.n_bands) {
      const int band = threadIdx.x;
      uint32_t tot = 0, work = 0;
#pragma unroll
      for (int q = 0; q < kWarps; ++q) {
        const uint32_t c = s_wcnt[band][q];
        s_wcnt[band][q] = tot;  // exclusive prefix
        tot += c;
        work += s_wwork[band][q];
      }
      s_base[band] = tot ? atomicAdd(&b.entry_count[band], (int)tot) : 0;
      if (work) atomicAdd(&b.band_work[band], (unsigned long long)work);
    }
    __syncthreads();
#pragma unroll(kExact ? kNB : 1)
    for (int band = 0; band < nb; ++band)
      emit(band, Ent3{s_r[band][0][threadIdx.x], s_r[band][1][threadIdx.x], s_r[band][2][threadIdx.x]},
           (int64_t)s_base[band] + s_wcnt[band][warp] + s_off[band][threadIdx.x]);
  } else {
    for (int band = 0; band < p.n_bands; ++band) {  // uniform trip count: warp collectives inside
      uint32_t w = 0;
      const Ent3 r = plan_band(band, &w);
      emit(band, r, book(band, r, w, true));
    }
  }
}

// ---- K2 ------------------------------------------------------------------------------

// Two adjacent samples of f32_cell at once, t = {cos_a, cos_b, sin_a, sin_b}: the same IEEE
// operations in the same order, lane-parallel in f32x2 (sm_100 FMUL2/FFMA2), so each cell and
// flag is bit-identical to f32_cell's.
template <bool kClamp, int kS>
__device__ __forceinline__ void f32_cell2(const F32Geom& g, float4 ba, float2 bb, float4 t, f32x2 one2,
                                          uint32_t* rel, bool* flag) {
  const f32x2 C = pk2(t.x, t.y), Sn = pk2(t.z, t.w);
  const f32x2 X = fma2(pk2(ba.w, ba.w), Sn, mul2(pk2(ba.x, ba.x), C));
  const f32x2 Y = fma2(pk2(bb.x, bb.x), Sn, mul2(pk2(ba.y, ba.y), C));
  const f32x2 CP = fma2(pk2(bb.y, bb.y), Sn, fma2(pk2(ba.z, ba.z), C, one2));
  uint32_t cb[2];
  upk2(CP, cb[0], cb[1]);
  const f32x2 R = pk2(rcp_approx(__uint_as_float(cb[0])), rcp_approx(__uint_as_float(cb[1])));
  const f32x2 CM = pk2(g.CMf, g.CMf);
  uint32_t bx[2], by[2];
  const f32x2 TX = fma2(X, R, CM), TY = fma2(Y, R, CM);
  upk2(TX, bx[0], bx[1]);
  upk2(TY, by[0], by[1]);
  if (FpCellSel<kClamp, kS>::value) {  // cell_of_bits' f32 cell, lane-parallel
    const f32x2 F = add2(add2_rm(TY, pk2(fp_ky<kS>(), fp_ky<kS>())), pk2(-kBig15, -kBig15));
    const f32x2 L = fma2_rz(F, pk2(g.Wf, g.Wf), TX);
    uint32_t lb[2];
    upk2(add2_rz(L, pk2(kBig23, kBig23)), lb[0], lb[1]);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      flag[h] = ((bx[h] & g.fmask) == 0u) | ((by[h] & g.fmask) == 0u);
      rel[h] = lb[h] - g.fp_off;
    }
    return;
  }
#pragma unroll
  for (int h = 0; h < 2; ++h) rel[h] = cell_of_bits<kClamp, kS>(g, bx[h], by[h], &flag[h]);
}

// (cos, sin) of sample j in the shared table: float4 q = {cos_2q, cos_2q+1, sin_2q, sin_2q+1}, so
// one LDS.128 feeds a lane's two adjacent samples as f32x2 operands.
__device__ __forceinline__ float2 tab_sample(const float4* tab, int j) {
  const float* t = reinterpret_cast<const float*>(tab) + 4 * (j >> 1) + (j & 1);
  return make_float2(t[0], t[2]);
}

// Everything the exact path needs, parked in shared memory at kernel start (and per band): the
// cold path reads it there (its loads cannot be hoisted past the queue stores), so none of it is
// kept in registers or re-loaded from the constant bank around the hot step loop.
struct ColdCtx {
  const double* zx;
  const double* zy;
  const double* zz;
  const double2* table64;
  const float4* basis_a;
  const float2* basis_b;
  uint32_t* grid;
  double E, inv_cell;
  int G, W, c_min, J, M;
  int r0, hb, own_lo, own_hi;  // current band
};

__device__ __forceinline__ void set_cold_band(ColdCtx& c, const VotePlan& p, int band) {
  c.r0 = p.band_r0[band];
  c.hb = p.band_r0[band + 1] - c.r0;
  c.own_lo = band == 0 ? 0 : c.r0;
  c.own_hi = band == p.n_bands - 1 ? p.G : c.r0 + c.hb;
}

// Exact path of queued samples: the hot loop deposited +2 at the sample's f32 cell (if in this
// tile) unconditionally; undo that, then deposit BOTH twins of its pair (samples p and p + J/2,
// each with the reference's own hemisphere decision) at their exact f64 cells (row-owned).
#ifndef RV_FB_NOINLINE
#define RV_FB_NOINLINE 1  // exact path as a real call: its registers stay out of the hot loop
#endif
#if RV_FB_NOINLINE
#define RV_FB_ATTR __noinline__
#else
#define RV_FB_ATTR __forceinline__
#endif
template <bool kClamp, int kS>
__device__ RV_FB_ATTR void fallback_samples(const ColdCtx* cc_s, const F32Geom& g, uint32_t q_s, int count,
                                            const float4* tab, uint32_t* tile) {
  const volatile ColdCtx& f = *cc_s;
  const int lane = threadIdx.x & 31;
  const uint2 e = lane < count ? lds_u2(q_s + 8u * lane) : make_uint2(0u, 0u);  // (constraint, sample)
  const uint32_t ci = e.x;
  if (lane < count) {
    const float4 ba = __ldg(f.basis_a + ci);
    const float2 bb = __ldg(f.basis_b + ci);
    const int j = (int)e.y;
    bool fl;
    const int r0 = f.r0, hb = f.hb, own_lo = f.own_lo, own_hi = f.own_hi, W = f.W, G = f.G, c_min = f.c_min;
    const uint32_t rel = f32_cell<kClamp, kS>(g, ba, bb, tab_sample(tab, j), &fl);
    if (rel < (uint32_t)hb * (uint32_t)W) atomicSub(&tile[rel], 2u);
    double a1[3], a2[3];
    exact_basis(f.zx[ci], f.zy[ci], f.zz[ci], a1, a2);
    const int M = f.M, J = f.J, jj = j >= J ? j - J : j;  // (the last step of a range may cross J)
    const int pr = jj >= M ? jj - M : jj;
    VotePlan p1;
    p1.E = f.E;
    p1.inv_cell = f.inv_cell;
    p1.G = G;
    const double2* t64 = f.table64;
    uint32_t* grid = f.grid;
#pragma unroll
    for (int tw = 0; tw < 2; ++tw) {
      const double2 cs = t64[pr + tw * M];
      int row, col;
      exact_sample(a1, a2, cs.x, cs.y, p1, &row, &col);
      if (row < own_lo || row >= own_hi) continue;
      const int lr = row - r0, lc = col - c_min;
      if ((unsigned)lr < (unsigned)hb && (unsigned)lc < (unsigned)W)
        atomicAdd(&tile[lr * W + lc], 1u);
      else
        atomicAdd(&grid[(size_t)row * G + col], 1u);
    }
  }
  __syncwarp();
}

__device__ __forceinline__ uint32_t umin(uint32_t a, uint32_t b) { return a < b ? a : b; }

__device__ __forceinline__ void red_shared(uint32_t saddr, uint32_t v) {
  asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(saddr), "r"(v));
}

// K2: persistent, one CTA per SM, 32 warps. A CTA owns one row band's u32 tile in shared memory
// at a time. Warps grab up to 32 work entries at a time from the band's entry list (K1b appends
// one entry per range of canonical samples of a constraint in the band; lane k loads entry k and
// its f32 basis, the warp then walks the entries, broadcasting each by shuffles); no CTA barrier
// per grab. A range is walked 64 samples per step, lane l taking the adjacent samples a+2l and
// a+2l+1 (one LDS.128 of the packed table, f32x2 math); the first and last steps of a range are
// masked where it starts odd or ends mid-step. Every sample deposits +2 (its twin lands in the same
// cell unless flagged) -- out-of-band and masked samples into never-flushed tile rows or the lane's
// sink word. Samples whose f32 cell is not provably the reference cell are queued per warp and
// recomputed exactly in f64 with both twins. When the band is exhausted the CTA flushes its tile
// (TMA bulk reduce-adds, or a partial slot) and steals the band with the most remaining entries.
// Degenerate constraints (no clean canonical half circle) are voted sample by sample at the end.

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
  // [tile_words] tile, [32] per-lane sink words, packed table (J/2 + 32 float4), fallback queues
  float4* tab = reinterpret_cast<float4*>(tile + ((p.tile_words + 32 + 3) & ~size_t(3)));
  const int M = p.halfJ, J = p.J;
  uint32_t* fbq_all = reinterpret_cast<uint32_t*>(tab + M + 32);
  __shared__ int s_band, s_slot;
  __shared__ ColdCtx s_cold;
  __shared__ unsigned int s_fb;  // flagged samples of this CTA (stats)

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // this warp's exact-path queue (shared window); recomputed in the cold path from the warp index
  // so that it holds no register across the hot loop
  const uint32_t fbq_s0 = (uint32_t)__cvta_generic_to_shared(fbq_all);
  auto fbq_addr = [&]() -> uint32_t {
    return fbq_s0 + (uint32_t)(threadIdx.x >> 5) * (uint32_t)(kFbqCap * 4);
  };
  for (int q = tid; q < M + 32; q += blockDim.x) {
    int j0 = 2 * q, j1 = 2 * q + 1;
    j0 = j0 >= J ? j0 - J : j0;
    j1 = j1 >= J ? j1 - J : j1;
    const float2 e = b.table32[j0], o = b.table32[j1];
    tab[q] = make_float4(e.x, o.x, e.y, o.y);
  }

  if (tid == 0) {  // initial band: CTAs split across bands in proportion to planned work
    unsigned long long total = 0;
    // band cost = planned samples + a per-entry overhead in sample equivalents (RV_BAND_ENTRY_W)
    auto band_cost = [&](int q) -> unsigned long long {
      return b.band_work[q] + (unsigned long long)RV_BAND_ENTRY_W * (unsigned long long)b.entry_count[q];
    };
    for (int q = 0; q < p.n_bands; ++q) total += band_cost(q);
    int band = p.n_bands - 1;
    if (total > 0) {
      const double pos = ((double)blockIdx.x + 0.5) / gridDim.x * (double)total;
      double acc = 0;
      for (int q = 0; q < p.n_bands; ++q) {
        acc += (double)band_cost(q);
        if (pos < acc) {
          band = q;
          break;
        }
      }
    }
    s_band = band;
    s_fb = 0;
    set_cold_band(s_cold, p, band);
    s_cold.zx = b.zx;
    s_cold.zy = b.zy;
    s_cold.zz = b.zz;
    s_cold.table64 = b.table64;
    s_cold.basis_a = b.basis_a;
    s_cold.basis_b = b.basis_b;
    s_cold.grid = b.grid;
    s_cold.E = p.E;
    s_cold.inv_cell = p.inv_cell;
    s_cold.G = p.G;
    s_cold.W = p.W;
    s_cold.c_min = p.c_min;
    s_cold.J = p.J;
    s_cold.M = p.halfJ;
  }
  vtrace(0, 0);
  for (size_t k = tid; k < p.tile_words; k += blockDim.x) tile[k] = 0u;
  __syncthreads();
  vtrace(1, s_band);
  // per-lane table address (shared window): lane l's float4 of a step at even sample a is
  // tab_s + 8 a (tab_s = table + 16 l)
  uint32_t tab_s = (uint32_t)__cvta_generic_to_shared(tab) + 16u * (uint32_t)lane;
  asm volatile("" : "+r"(tab_s));
  // opaque to the optimizer: otherwise the shared-window base is rematerialised every step
  uint32_t tile_s = (uint32_t)__cvta_generic_to_shared(tile);
  // deposits outside this band's rows go to tile rows >= hb (never flushed) or, beyond the tile,
  // to this lane's sink word: addr = tile + 4 * min(rel, tile_words + lane)
  uint32_t sink_rel = (uint32_t)p.tile_words + (uint32_t)lane;
  uint32_t vote2 = 2u;
  asm volatile("" : "+r"(tile_s), "+r"(sink_rel), "+r"(vote2));
  const f32x2 one2 = pk2(1.f, 1.f);
  const float CMf = p.CMf;
  const int W = p.W, G = p.G;
  const int S = p.frac_shift;
  const uint32_t fmask = p.frac_mask;

  for (;;) {
    // REDUX broadcasts (uniform-register results): the band, its entry count and each grab offset
    // are provably warp-uniform, so the vote loops carry no divergence checks
    const int band = __reduce_max_sync(0xFFFFFFFFu, s_band);
    if (band < 0) break;
    const int r0 = p.band_r0[band], hb = p.band_r0[band + 1] - r0;
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
    geo.Wf = p.Wf;
    geo.fp_off = 0x4B000000u + (3u << (22 - (kS ? kS : 13))) + (uint32_t)r0 * (uint32_t)W + (uint32_t)p.c_min;
    const unsigned long long* ebase = b.entries + (int64_t)band * b.entry_cap;
    const int n_ent = __reduce_max_sync(0xFFFFFFFFu, b.entry_count[band]);
    int* counter = &b.counters[1 + band];
    // grab size: 32 entries when every warp of the launch still gets several grabs, smaller for
    // small problems (otherwise a handful of warps would walk all entries while the rest idle)
    const int per = (int)(((long long)gridDim.x * (kVoteThreads / 32) * RV_GRAB_PER) / p.n_bands);
    const int grab = max(1, min(32, n_ent / max(per, 1)));
    // Entries are fetched in per-warp grabs of up to 32 (lane k holds entry k); flagged samples
    // are queued per warp as (constraint, sample) and drained in batches of up to 32.
    uint32_t my_ci = 0, my_enc = 0;
    int ne = 0, qn = 0, g0 = 0;
    float4 ba = make_float4(0.f, 0.f, 0.f, 0.f);
    float2 bb = make_float2(0.f, 0.f);
    // one step: samples a + 2 lane + {0, 1} (a = the step's even first sample, recovered from the
    // table address tp); masked steps drop samples outside [mstart, mstart + mlen)
    // The exact path is a real call; reloading the grab and the entry's basis after it (rare)
    // keeps them out of the call's save set, so the hot loop holds them in registers (no
    // per-entry spill reloads through L1).
    auto after_drain = [&](uint32_t cik) {
      my_ci = 0;
      my_enc = 0;
      if (lane < ne) {
        const unsigned long long e = __ldg(ebase + g0 + lane);
        my_ci = (uint32_t)e;
        my_enc = (uint32_t)(e >> 32);
      }
      ba = __ldg(b.basis_a + cik);
      bb = __ldg(b.basis_b + cik);
    };
    auto step = [&](uint32_t tpa, bool masked, uint32_t cik, int mstart, int mlen) {
      float4 t4;
      asm("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(t4.x), "=f"(t4.y), "=f"(t4.z), "=f"(t4.w) : "r"(tpa));
      uint32_t rel[2];
      bool flag[2];
      f32_cell2<kClamp, kS>(geo, ba, bb, t4, one2, rel, flag);
      if (masked) {
        const int a = (int)((tpa - tab_s) >> 3);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const bool ok = (uint32_t)(a + 2 * lane + h - mstart) < (uint32_t)mlen;
          rel[h] = ok ? rel[h] : 0xFFFFFFFFu;
          flag[h] = flag[h] && ok;
        }
      }
      // deposit even if flagged: the exact path undoes it (no select on the flag here)
      red_shared(tile_s + 4u * umin(rel[0], sink_rel), vote2);
      red_shared(tile_s + 4u * umin(rel[1], sink_rel), vote2);
      if (__any_sync(0xFFFFFFFFu, flag[0] | flag[1])) {  // cold: queue for the exact f64 path
        // queue entries are (constraint, sample), so the queue outlives the grab; it is drained
        // before it would pass 32 entries (one exact-path batch = one sample per lane). Both
        // samples of the step are compacted at once (one capacity check).
        const uint32_t j = (uint32_t)((tpa - tab_s) >> 3) + 2u * lane;
        unsigned lt_mask;
        asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lt_mask));
        const uint32_t fbq_s = fbq_addr();
        const unsigned fm0 = __ballot_sync(0xFFFFFFFFu, flag[0]), fm1 = __ballot_sync(0xFFFFFFFFu, flag[1]);
        const int c0 = __popc(fm0), c = c0 + __popc(fm1);
        if (qn + c > 32) {
          fallback_samples<kClamp, kS>(&s_cold, geo, fbq_s, qn, tab, tile);
          after_drain(cik);
          qn = 0;
        }
        if (c <= 32) {
          if (flag[0]) sts_u2(fbq_s + 8u * (uint32_t)(qn + __popc(fm0 & lt_mask)), cik, j);
          if (flag[1]) sts_u2(fbq_s + 8u * (uint32_t)(qn + c0 + __popc(fm1 & lt_mask)), cik, j + 1u);
          qn += c;
        } else {  // more than 32 flagged samples in one step (never seen): two batches
          if (flag[0]) sts_u2(fbq_s + 8u * (uint32_t)__popc(fm0 & lt_mask), cik, j);
          __syncwarp();
          fallback_samples<kClamp, kS>(&s_cold, geo, fbq_s, c0, tab, tile);
          after_drain(cik);
          if (flag[1]) sts_u2(fbq_s + 8u * (uint32_t)__popc(fm1 & lt_mask), cik, j + 1u);
          qn = c - c0;
        }
        if (lane == 0) red_shared((uint32_t)__cvta_generic_to_shared(&s_fb), (uint32_t)c);
        __syncwarp();
      }
    };
    // grab loop / entry loop / step loop
    const int gsz = grab;
    for (;;) {
      g0 = 0;
      if (lane == 0) g0 = atomicAdd(counter, gsz);
      // REDUX broadcasts (uniform-register results): everything derived from them is provably
      // warp-uniform, so the loops carry no divergence checks around their votes
      g0 = __reduce_max_sync(0xFFFFFFFFu, g0);
      if (g0 >= n_ent) break;
      ne = min(gsz, n_ent - g0);
      my_ci = 0;
      my_enc = 0;
      if (lane < ne) {
        const unsigned long long e = __ldcs(ebase + g0 + lane);
        my_ci = (uint32_t)e;
        my_enc = (uint32_t)(e >> 32);
        // warm L1 with this entry's basis: the warp reads it back as one broadcast load
        asm volatile("prefetch.global.L1 [%0];" ::"l"(b.basis_a + my_ci));
        asm volatile("prefetch.global.L1 [%0];" ::"l"(b.basis_b + my_ci));
      }
      for (int kk = 0; kk < ne; ++kk) {
#if RV_BCAST_REDUX
        const uint32_t enc = __reduce_max_sync(0xFFFFFFFFu, lane == kk ? my_enc : 0u);
        const uint32_t cik = __reduce_max_sync(0xFFFFFFFFu, lane == kk ? my_ci : 0u);
#else
        // shuffles for the entry; the loop trip count below goes through REDUX, so the step
        // loop stays provably warp-uniform
        const uint32_t enc = __shfl_sync(0xFFFFFFFFu, my_enc, kk);
        const uint32_t cik = __shfl_sync(0xFFFFFFFFu, my_ci, kk);
#endif
        ba = __ldg(b.basis_a + cik);
        bb = __ldg(b.basis_b + cik);
        const int start = (int)(enc & 0xFFFFu), len = (int)(enc >> 16);
        if ((start & 1) | (len & 63)) {  // rare: a range the planner could not align (enc is uniform)
          const int a0 = start & ~1;
          const int nst = (start + len - a0 + 63) >> 6;
          uint32_t tpm = tab_s + 8u * (uint32_t)a0;
#pragma unroll 1
          for (int q = 0; q < nst; ++q, tpm += 512u) step(tpm, true, cik, start, len);
          continue;
        }
#if RV_UNIFORM_STEP
        // uniform step offset (UR): the loop is one UIADD3 + UISETP + BRA.U, the lane's table
        // address is its fixed base + the offset
        const uint32_t u0 = 8u * (uint32_t)start;
        const uint32_t uend = u0 + 8u * (uint32_t)len;  // len is a multiple of 64 here
#pragma unroll 1
        for (uint32_t u = u0; u != uend; u += 512u) step(tab_s + u, false, cik, 0, 0);
#else
        uint32_t tpf = tab_s + 8u * (uint32_t)start;
#pragma unroll 1
        for (int r = __reduce_max_sync(0xFFFFFFFFu, (unsigned)len >> 6); r > 0; --r, tpf += 512u)
          step(tpf, false, cik, 0, 0);
#endif
      }
    }
    if (qn > 0) fallback_samples<kClamp, kS>(&s_cold, geo, fbq_addr(), qn, tab, tile);  // before the flush
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
      if (best >= 0) set_cold_band(s_cold, p, best);
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
  // degenerate constraints (planner list): one warp per constraint, lanes over all J samples,
  // exact f64 with the reference's per-sample hemisphere decision, global atomics
  const int nd = b.counters[kDegenCount];
  if (nd > 0) {
    VotePlan p1;
    p1.E = p.E;
    p1.inv_cell = p.inv_cell;
    p1.G = G;
    for (;;) {
      int d = 0;
      if (lane == 0) d = atomicAdd(&b.counters[kDegenGrab], 1);
      d = __shfl_sync(0xFFFFFFFFu, d, 0);
      if (d >= nd) break;
      const int ci = b.degen[d];
      double a1[3], a2[3];
      exact_basis(b.zx[ci], b.zy[ci], b.zz[ci], a1, a2);
      for (int j = lane; j < J; j += 32) {
        const double2 cs = b.table64[j];
        int row, col;
        exact_sample(a1, a2, cs.x, cs.y, p1, &row, &col);
        atomicAdd(&b.grid[(size_t)row * G + col], 1u);
      }
    }
  }
  if (p.bulk && warp == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // flushes landed
  __syncthreads();
  if (tid == 0 && s_fb) atomicAdd(&b.stats[1], (unsigned long long)s_fb);
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
  const int threads = kPlanThreads;
  const int64_t blocks = (n + threads - 1) / threads;
  if (p.n_bands == 5)  // the default geometry
    plan_kernel<5, true><<<(unsigned)blocks, threads, 0, s>>>(p, b, n);
  else if (p.n_bands <= 8)
    plan_kernel<8, false><<<(unsigned)blocks, threads, 0, s>>>(p, b, n);
  else
    plan_kernel<0, false><<<(unsigned)blocks, threads, 0, s>>>(p, b, n);
}

using VoteKernel = void (*)(VotePlan, VoteBuffers, int64_t);
static VoteKernel vote_kernel_for(const VotePlan& p, int* slot) {
  // S = 13 / 12 (every grid <= 1000 at the reference extents) get a compile-time shift; other S
  // use the run-time variant
  // RV_FP_CELL: the fixed-S variants need every f32 cell intermediate below 2^23
  const bool fp_ok = !RV_FP_CELL || (double)(p.G + 1) * p.W + 3.0 * std::ldexp(1.0, 23 - p.frac_shift) < 8388608.0;
  const int ks = !fp_ok ? 0 : p.frac_shift == 13 ? 2 : (p.frac_shift == 12 ? 1 : 0);
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
