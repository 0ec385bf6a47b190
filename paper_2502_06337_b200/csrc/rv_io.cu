// CSV ingest of correspondences on the device (io.cpp:66-101
// read_correspondences, io.hpp:11-13): the text is indexed and parsed where the solve runs.
//
//   K_io1 delimiter census   per 8 KB chunk: count ',' and '\n' (uint4 loads)
//   K_io2 chunk scan         exclusive scan of the per-chunk counts (one block)
//   K_io3 delimiter index    byte position and line of every delimiter, delimiter index of every
//                            newline (block scan + chunk offset)
//   K_io4 lines              per line: field count, blank test (spaces/tabs after one trailing
//                            '\r'), status (blank / data / header / bad field count)
//   K_io5 rows               row index of every data line (scan of the data flags)
//   K_io6 fields             one thread per field: trim " \t\r", strict float syntax of
//                            std::from_chars (general format: no '+', no hex), exact conversion by
//                            the Eisel-Lemire algorithm (Lemire 2021) for <= 19 significant digits
//                            and normal results; anything else (more digits, inf/nan, subnormal,
//                            overflow, a halfway ambiguity) is queued for the host's from_chars.
//
// Errors: every bad line reports its 1-based physical line number with atomicMin; the host
// re-runs the reference's line logic on the first one for the exact message. Layout: the text
// must end with '\n' (the host appends one); counts are int32 and positions u32 (text < 2 GB).
#include <cuda_runtime.h>

#include <cstdint>

#include "rv_internal.h"

namespace rvb {
namespace {

#include "rv_pow5.inc"

constexpr int kIoThreads = 256;
constexpr int kIoBytesPerThread = 32;  // two uint4 loads
constexpr int kIoChunk = kIoThreads * kIoBytesPerThread;

__device__ __forceinline__ void count_bytes(uint4 v, int& nd, int& nn) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int k = 0; k < 4; ++k) {
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const uint32_t ch = (w[k] >> (8 * b)) & 0xFFu;
      nd += (ch == ',') | (ch == '\n');
      nn += ch == '\n';
    }
  }
}

__device__ __forceinline__ uint4 load16(const uint8_t* t, int64_t nbytes, int64_t off) {
  if (off + 16 <= nbytes) return *reinterpret_cast<const uint4*>(t + off);
  uint32_t w[4] = {0, 0, 0, 0};  // tail: bytes past the end read as 0 (no delimiter)
  for (int i = 0; i < 16 && off + i < nbytes; ++i) w[i >> 2] |= (uint32_t)t[off + i] << (8 * (i & 3));
  return make_uint4(w[0], w[1], w[2], w[3]);
}

__global__ void __launch_bounds__(kIoThreads) io_count_kernel(const uint8_t* t, int64_t nbytes, int2* chunk) {
  const int64_t off = (int64_t)blockIdx.x * kIoChunk + (int64_t)threadIdx.x * kIoBytesPerThread;
  int nd = 0, nn = 0;
  if (off < nbytes) {
    count_bytes(load16(t, nbytes, off), nd, nn);
    count_bytes(load16(t, nbytes, off + 16), nd, nn);
  }
  __shared__ int s_d[kIoThreads / 32], s_n[kIoThreads / 32];
  nd = __reduce_add_sync(0xFFFFFFFFu, (unsigned)nd);
  nn = __reduce_add_sync(0xFFFFFFFFu, (unsigned)nn);
  if ((threadIdx.x & 31) == 0) {
    s_d[threadIdx.x >> 5] = nd;
    s_n[threadIdx.x >> 5] = nn;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int a = 0, b = 0;
    for (int w = 0; w < kIoThreads / 32; ++w) {
      a += s_d[w];
      b += s_n[w];
    }
    chunk[blockIdx.x] = make_int2(a, b);
  }
}

// Exclusive scan of n int2 values in place (one block of 1024 threads); totals to *total.
__global__ void __launch_bounds__(1024) io_scan2_kernel(int2* v, int n, int2* total) {
  __shared__ int2 s[1024];
  const int per = (n + 1023) / 1024;
  const int lo = threadIdx.x * per, hi = min(lo + per, n);
  int2 acc = make_int2(0, 0);
  for (int i = lo; i < hi; ++i) {
    acc.x += v[i].x;
    acc.y += v[i].y;
  }
  s[threadIdx.x] = acc;
  __syncthreads();
  for (int o = 1; o < 1024; o <<= 1) {
    int2 x = make_int2(0, 0);
    if (threadIdx.x >= o) x = s[threadIdx.x - o];
    __syncthreads();
    s[threadIdx.x].x += x.x;
    s[threadIdx.x].y += x.y;
    __syncthreads();
  }
  int2 run = threadIdx.x ? s[threadIdx.x - 1] : make_int2(0, 0);
  for (int i = lo; i < hi; ++i) {
    const int2 x = v[i];
    v[i] = run;
    run.x += x.x;
    run.y += x.y;
  }
  if (threadIdx.x == 1023) *total = s[1023];
}

// Block-wide exclusive scan of two counters (kIoThreads threads).
__device__ __forceinline__ int2 block_excl2(int a, int b, int2* s_w) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int ia = a, ib = b;
  for (int o = 1; o < 32; o <<= 1) {
    const int xa = __shfl_up_sync(0xFFFFFFFFu, ia, o), xb = __shfl_up_sync(0xFFFFFFFFu, ib, o);
    if (lane >= o) {
      ia += xa;
      ib += xb;
    }
  }
  if (lane == 31) s_w[warp] = make_int2(ia, ib);
  __syncthreads();
  int pa = 0, pb = 0;
  for (int w = 0; w < warp; ++w) {
    pa += s_w[w].x;
    pb += s_w[w].y;
  }
  return make_int2(pa + ia - a, pb + ib - b);
}

__global__ void __launch_bounds__(kIoThreads) io_index_kernel(const uint8_t* t, int64_t nbytes, const int2* chunk,
                                                              uint32_t* dpos, int32_t* dline, int32_t* nl_delim) {
  const int64_t off = (int64_t)blockIdx.x * kIoChunk + (int64_t)threadIdx.x * kIoBytesPerThread;
  uint4 v0 = make_uint4(0, 0, 0, 0), v1 = v0;
  int nd = 0, nn = 0;
  if (off < nbytes) {
    v0 = load16(t, nbytes, off);
    v1 = load16(t, nbytes, off + 16);
    count_bytes(v0, nd, nn);
    count_bytes(v1, nd, nn);
  }
  __shared__ int2 s_w[kIoThreads / 32];
  const int2 ex = block_excl2(nd, nn, s_w);
  int d = chunk[blockIdx.x].x + ex.x, l = chunk[blockIdx.x].y + ex.y;
  const uint32_t w[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
#pragma unroll
  for (int k = 0; k < 8; ++k) {
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const uint32_t ch = (w[k] >> (8 * b)) & 0xFFu;
      if (ch == ',' || ch == '\n') {
        dpos[d] = (uint32_t)(off + 4 * k + b);
        dline[d] = l;
        if (ch == '\n') {
          nl_delim[l] = d;
          ++l;
        }
        ++d;
      }
    }
  }
}

enum : int8_t { kLineBlank = 0, kLineData = 1, kLineHeader = 2, kLineBad = 3 };

// Line l: delimiters [first, last], last = its newline. Bytes [start, end) without the newline
// and without one trailing '\r' (io.cpp:72).
__device__ __forceinline__ void line_span(const uint32_t* dpos, const int32_t* nl_delim, int l, int& first, int& last,
                                          int64_t& start, int64_t& end) {
  first = l == 0 ? 0 : nl_delim[l - 1] + 1;
  last = nl_delim[l];
  start = l == 0 ? 0 : (int64_t)dpos[nl_delim[l - 1]] + 1;
  end = dpos[last];
}

__global__ void io_lines_kernel(const uint8_t* t, const uint32_t* dpos, const int32_t* nl_delim, int nlines,
                                int skip_first, int8_t* status, int32_t* is_data, unsigned int* err_line) {
  const int l = blockIdx.x * blockDim.x + threadIdx.x;
  if (l >= nlines) return;
  int first, last;
  int64_t start, end;
  line_span(dpos, nl_delim, l, first, last, start, end);
  if (end > start && t[end - 1] == '\r') --end;
  const int nf = last - first + 1;
  int8_t st = kLineData;
  if (nf == 1) {  // blank: only spaces and tabs (io.cpp:73)
    bool blank = true;
    for (int64_t i = start; i < end && blank; ++i) blank = t[i] == ' ' || t[i] == '\t';
    if (blank) st = kLineBlank;
  }
  if (st == kLineData && l == 0 && skip_first) st = kLineHeader;
  if (st == kLineData && nf != 6) {
    st = kLineBad;
    atomicMin(err_line, (unsigned)(l + 1));
  }
  status[l] = st;
  is_data[l] = st == kLineData;
}

// Exclusive scan of n ints in place: per-block totals -> scan -> add (three launches).
__global__ void __launch_bounds__(1024) io_block_sums_kernel(const int32_t* v, int n, int32_t* sums) {
  const int i = blockIdx.x * 1024 + threadIdx.x;
  const int x = i < n ? v[i] : 0;
  __shared__ int s[32];
  const int r = __reduce_add_sync(0xFFFFFFFFu, (unsigned)x);
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = r;
  __syncthreads();
  if (threadIdx.x == 0) {
    int a = 0;
    for (int w = 0; w < 32; ++w) a += s[w];
    sums[blockIdx.x] = a;
  }
}

__global__ void __launch_bounds__(1024) io_scan1_kernel(int32_t* v, int n, int32_t* total) {
  __shared__ int s[1024];
  const int per = (n + 1023) / 1024;
  const int lo = threadIdx.x * per, hi = min(lo + per, n);
  int acc = 0;
  for (int i = lo; i < hi; ++i) acc += v[i];
  s[threadIdx.x] = acc;
  __syncthreads();
  for (int o = 1; o < 1024; o <<= 1) {
    const int x = threadIdx.x >= o ? s[threadIdx.x - o] : 0;
    __syncthreads();
    s[threadIdx.x] += x;
    __syncthreads();
  }
  int run = threadIdx.x ? s[threadIdx.x - 1] : 0;
  for (int i = lo; i < hi; ++i) {
    const int x = v[i];
    v[i] = run;
    run += x;
  }
  if (threadIdx.x == 1023) *total = s[1023];
}

__global__ void __launch_bounds__(1024) io_block_scan_kernel(int32_t* v, int n, const int32_t* offsets) {
  const int i = blockIdx.x * 1024 + threadIdx.x;
  const int x = i < n ? v[i] : 0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int incl = x;
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
    if (lane >= o) incl += y;
  }
  __shared__ int s[32];
  if (lane == 31) s[warp] = incl;
  __syncthreads();
  int pre = 0;
  for (int w = 0; w < warp; ++w) pre += s[w];
  if (i < n) v[i] = offsets[blockIdx.x] + pre + incl - x;
}

// ---- exact decimal -> binary64 (Eisel-Lemire) -------------------------------------------

__device__ __forceinline__ bool is_digit(uint32_t c) { return c - '0' < 10u; }

// Result: 0 = ok (*bits), 1 = syntax error (not a from_chars float literal), 2 = host fallback.
__device__ int parse_field(const uint8_t* t, int64_t s, int64_t e, unsigned long long* bits) {
  while (s < e && (t[s] == ' ' || t[s] == '\t' || t[s] == '\r')) ++s;  // io.cpp:20-23
  while (e > s && (t[e - 1] == ' ' || t[e - 1] == '\t' || t[e - 1] == '\r')) --e;
  if (s >= e) return 1;  // "empty field"
  bool neg = false;
  if (t[s] == '-') {
    neg = true;
    ++s;
    if (s >= e) return 1;
  }
  const uint32_t c0 = t[s] | 0x20u;
  if (c0 == 'i' || c0 == 'n') return 2;  // inf / infinity / nan: from_chars decides
  unsigned long long w = 0;
  int nd = 0;             // significant digits taken into w
  int drop = 0;           // significant digits beyond 19 (-> fallback)
  int dexp = 0;           // decimal exponent adjustment of w
  bool any = false, seen_nz = false;
  while (s < e && is_digit(t[s])) {
    const uint32_t dgt = t[s] - '0';
    any = true;
    if (dgt || seen_nz) {
      seen_nz = true;
      if (nd < 19) {
        w = w * 10 + dgt;
        ++nd;
      } else {
        ++drop;
      }
    }
    ++s;
  }
  if (drop) return 2;
  if (s < e && t[s] == '.') {
    ++s;
    while (s < e && is_digit(t[s])) {
      const uint32_t dgt = t[s] - '0';
      any = true;
      if (dgt || seen_nz) {
        seen_nz = true;
        if (nd < 19) {
          w = w * 10 + dgt;
          ++nd;
          --dexp;
        } else {
          return 2;
        }
      } else {
        --dexp;  // leading zeros after the point
      }
      ++s;
    }
  }
  if (!any) return 1;
  if (s < e && (t[s] == 'e' || t[s] == 'E')) {
    int64_t p = s + 1;
    bool eneg = false;
    if (p < e && (t[p] == '+' || t[p] == '-')) {
      eneg = t[p] == '-';
      ++p;
    }
    if (p >= e || !is_digit(t[p])) return 1;  // "1e" / "1e+": from_chars stops before 'e'
    int ev = 0;
    while (p < e && is_digit(t[p])) {
      if (ev < 100000) ev = ev * 10 + (int)(t[p] - '0');
      ++p;
    }
    if (ev >= 100000) return 2;
    dexp += eneg ? -ev : ev;
    s = p;
  }
  if (s != e) return 1;  // trailing garbage
  if (w == 0) {
    *bits = neg ? 0x8000000000000000ull : 0ull;
    return 0;
  }
  const int q = dexp;
  if (q < kPow5Min || q > kPow5Max) return 2;
  const int lz = __clzll((long long)w);
  const unsigned long long wn = w << lz;
  const int idx = 2 * (q - kPow5Min);
  const unsigned long long t_hi = kPow5Table[idx], t_lo = kPow5Table[idx + 1];
  unsigned long long hi = __umul64hi(wn, t_hi), lo = wn * t_hi;
  constexpr unsigned long long kMask = 0x1FFull;  // 64 - 52 - 3 low bits of the upper word
  if ((hi & kMask) == kMask) {                    // refine with the lower half of the power
    const unsigned long long s_hi = __umul64hi(wn, t_lo);
    const unsigned long long nlo = lo + s_hi;
    if (nlo < lo) ++hi;
    lo = nlo;
    if ((hi & kMask) == kMask && lo == ~0ull) return 2;  // still inconclusive
  }
  const int upper = (int)(hi >> 63);
  unsigned long long mant = hi >> (upper + 9);
  // binary exponent: floor(log2(10^q)) + 63 (Lemire's 217706 * q >> 16 form)
  int p2 = (int)(((152170 + 65536) * (long long)q) >> 16) + 63 + upper - lz + 1023;
  if (lo <= 1 && (hi & kMask) == 0 && (mant & 3) == 1) return 2;  // possible halfway case
  mant += mant & 1;
  mant >>= 1;
  if (mant >= (2ull << 52)) {
    mant = 1ull << 52;
    ++p2;
  }
  mant &= ~(1ull << 52);
  if (p2 <= 0 || p2 >= 0x7FF) return 2;  // subnormal / overflow: from_chars decides
  *bits = mant | ((unsigned long long)p2 << 52) | (neg ? 0x8000000000000000ull : 0ull);
  return 0;
}

__global__ void io_fields_kernel(const uint8_t* t, const uint32_t* dpos, const int32_t* dline,
                                 const int32_t* nl_delim, int nfields, const int8_t* status, const int32_t* row,
                                 double* out, int64_t cap_rows, unsigned int* err_line, CsvFallback* fb,
                                 int fb_cap, int32_t* fb_count) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nfields) return;
  const int l = dline[k];
  if (status[l] != kLineData) return;
  const int first = l == 0 ? 0 : nl_delim[l - 1] + 1;
  const int col = k - first;
  const int64_t s = k == 0 ? 0 : (int64_t)dpos[k - 1] + 1;
  int64_t e = dpos[k];
  if (k == nl_delim[l] && e > s && t[e - 1] == '\r') --e;  // the line's trailing '\r' (io.cpp:72)
  unsigned long long bits = 0;
  const int r = parse_field(t, s, e, &bits);
  const int64_t rw = row[l];
  if (r == 0) {
    if (rw < cap_rows) reinterpret_cast<unsigned long long*>(out)[rw * 6 + col] = bits;
  } else if (r == 1) {
    atomicMin(err_line, (unsigned)(l + 1));
  } else {
    const int slot = atomicAdd(fb_count, 1);
    if (slot < fb_cap) fb[slot] = CsvFallback{s, e, rw, col, l};
  }
}

__global__ void io_scatter_kernel(const int64_t* idx, const double* vals, int n, double* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[idx[i]] = vals[i];
}

}  // namespace

cudaError_t launch_csv_parse(const CsvBuffers& b, cudaStream_t s, int stage) {
  const int nchunks = (int)((b.nbytes + kIoChunk - 1) / kIoChunk);
  if (stage == 0) {  // census: delimiters and newlines per chunk, scanned
    io_count_kernel<<<nchunks, kIoThreads, 0, s>>>(b.text, b.nbytes, b.chunk);
    io_scan2_kernel<<<1, 1024, 0, s>>>(b.chunk, nchunks, b.totals);
    return cudaGetLastError();
  }
  // stage 1 (the host read the totals and sized the index): index, lines, rows, fields
  const int nl = b.nlines, nf = b.nfields;
  io_index_kernel<<<nchunks, kIoThreads, 0, s>>>(b.text, b.nbytes, b.chunk, b.dpos, b.dline, b.nl_delim);
  io_lines_kernel<<<(nl + 255) / 256, 256, 0, s>>>(b.text, b.dpos, b.nl_delim, nl, b.skip_first, b.status, b.row,
                                                   b.err_line);
  const int nb = (nl + 1023) / 1024;
  io_block_sums_kernel<<<nb, 1024, 0, s>>>(b.row, nl, b.block);
  io_scan1_kernel<<<1, 1024, 0, s>>>(b.block, nb, b.nrows);
  io_block_scan_kernel<<<nb, 1024, 0, s>>>(b.row, nl, b.block);
  io_fields_kernel<<<(nf + 255) / 256, 256, 0, s>>>(b.text, b.dpos, b.dline, b.nl_delim, nf, b.status, b.row, b.out,
                                                    b.cap_rows, b.err_line, b.fb, b.fb_cap, b.fb_count);
  return cudaGetLastError();
}

int csv_chunks(int64_t nbytes) { return (int)((nbytes + kIoChunk - 1) / kIoChunk); }

void launch_csv_scatter(const int64_t* idx, const double* vals, int n, double* out, cudaStream_t s) {
  if (n > 0) io_scatter_kernel<<<(n + 255) / 256, 256, 0, s>>>(idx, vals, n, out);
}

}  // namespace rvb
