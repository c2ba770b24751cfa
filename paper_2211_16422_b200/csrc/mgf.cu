// MGF text -> CSR spectra on the device: parse_mgf, src/mgf.cpp:93-181, with
// finalize_block (:66-89), re-designed as data-parallel passes over the file image in HBM.
//
// The reference is a sequential line state machine.  Its outcome is reproduced exactly -- same
// spectra, same doubles bit for bit, same first ParseError (line and message) -- by these passes:
//
//   M1 lines      newline positions -> line table (block scan), std::getline semantics (:100)
//   M2 classify   per line: strip (:18-26), kind = blank | '#' | BEGIN | END | alpha-first with or
//                 without '=' | other
//   (scan)        BEGIN / END prefix counts -> "inside a block" for every line; a line's state is
//                 the sequential parser's state as long as no earlier line was an error, and only
//                 the FIRST error (smallest detection line) is reported, so later garbage is moot
//   M3 structure  per line: structural errors (:106-119, :131-139), block begin / end tables,
//                 peak-line flags
//   (scan)        peak-line prefix -> position of every raw peak
//   M4 peaks      per peak line: two from_chars doubles (:28-33, :163-177) -> raw (m/z, intensity)
//   M5 headers    per block: KEY=VALUE lines in order, last one wins (:134-161)
//   M6 hard       the rare numbers the one-rounding fast path cannot decide (more than 19 digits,
//                 decimal exponent beyond +-22) -> exact big-integer conversion
//   M7 finalize   per block: stable sort by m/z + duplicate merge when not already strictly
//                 ascending (:78-88), compaction only if some block shrank
//
// Decimal -> double: a token with <= 19 significant digits w <= 2^53 and |e10| <= 22 is w * 10^e10
// or w / 10^-e10 with both operands exact, i.e. ONE IEEE rounding == the correctly rounded result
// std::from_chars produces.  Everything else goes to M6, which computes floor(A / B) of the exact
// rational value with 54 quotient bits by shift-and-subtract on multi-word integers in shared
// memory and rounds to nearest even; overflow and underflow-to-zero are from_chars' out-of-range
// errors.  No value is ever approximated.

#include <algorithm>
#include <string>
#include <vector>

#include "common.cuh"
#include "radix.cuh"

namespace hb {

enum MgfKind : uint8_t { kBlank = 0, kHash = 1, kBegin = 2, kEnd = 3, kKeyVal = 4, kAlphaNoEq = 5, kOther = 6 };
// error codes, ordered as the messages below
enum MgfErr : uint32_t {
  kErrNone = 0, kErrOutside, kErrMissingPepmass, kErrBeginInside, kErrExpectedKv, kErrPepmass, kErrCharge,
  kErrPeakNumbers, kErrPeakMz, kErrPeakIntensity, kErrUnterminated
};
static const char* const kMgfMessages[] = {
    "", "unexpected content outside BEGIN IONS/END IONS", "spectrum block is missing PEPMASS",
    "BEGIN IONS inside an open spectrum block", "expected KEY=VALUE header or peak line",
    "PEPMASS must be a positive number", "CHARGE must be a positive integer like 2+",
    "peak line must be two numbers: m/z intensity", "peak m/z must be positive",
    "peak intensity must be non-negative", "spectrum block not closed by END IONS"};

__device__ __forceinline__ bool mg_space(uint8_t c) {
  return c == ' ' || (c >= 9 && c <= 13);  // \t \n \v \f \r
}
__device__ __forceinline__ bool mg_alpha(uint8_t c) { return (uint8_t)((c | 32) - 'a') < 26; }
__device__ __forceinline__ bool mg_digit(uint8_t c) { return (uint8_t)(c - '0') < 10; }

__device__ __forceinline__ void mg_error(unsigned long long* err, uint64_t detect_line, uint32_t code) {
  atomicMin(err, (static_cast<unsigned long long>(detect_line) << 8) | code);
}

// ---- M1: line table ---------------------------------------------------------------------------

constexpr int kM1Threads = 256, kM1Bytes = 16;  // bytes per thread

__global__ void mgf_count_newlines_kernel(const uint8_t* __restrict__ text, uint64_t n, uint32_t* __restrict__ tile_count) {
  const uint64_t base = (uint64_t(blockIdx.x) * kM1Threads + threadIdx.x) * kM1Bytes;
  uint32_t c = 0;
  if (base + kM1Bytes <= n) {
    const uint4 v = *reinterpret_cast<const uint4*>(text + base);
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) c += ((w[i] >> (8 * j)) & 0xFFu) == '\n';
  } else {
    for (uint64_t i = base; i < n; ++i) c += text[i] == '\n';
  }
  const uint32_t total = block_sum_u32<kM1Threads>(c);
  if (threadIdx.x == 0) tile_count[blockIdx.x] = total;
}

__global__ void mgf_line_starts_kernel(const uint8_t* __restrict__ text, uint64_t n,
                                       const uint32_t* __restrict__ tile_base, uint32_t* __restrict__ line_start) {
  const uint64_t base = (uint64_t(blockIdx.x) * kM1Threads + threadIdx.x) * kM1Bytes;
  uint32_t mask = 0;
  for (int i = 0; i < kM1Bytes; ++i)
    if (base + i < n && text[base + i] == '\n') mask |= 1u << i;
  const uint32_t before = block_exclusive_sum_u32<kM1Threads>(__popc(mask));
  uint32_t k = tile_base[blockIdx.x] + before;  // newlines before this thread's bytes
  while (mask) {
    const int i = __ffs(mask) - 1;
    mask &= mask - 1;
    line_start[++k] = static_cast<uint32_t>(base + i + 1);  // the line after newline k-1 starts here
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) line_start[0] = 0;
}

// ---- M2: classify -------------------------------------------------------------------------------

__global__ void mgf_classify_kernel(const uint8_t* __restrict__ text, uint64_t n, uint32_t n_lines,
                                    const uint32_t* __restrict__ line_start, uint8_t* __restrict__ kind,
                                    uint32_t* __restrict__ ls, uint32_t* __restrict__ ll,
                                    uint32_t* __restrict__ is_begin, uint32_t* __restrict__ is_end) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_lines) return;
  uint32_t s = line_start[i];
  // the line ends before its '\n'; line_start has n_lines + 1 valid entries only when the text ends in '\n'
  uint32_t e = (i + 1 < n_lines) ? line_start[i + 1] - 1 : static_cast<uint32_t>(n);
  if (i + 1 == n_lines && e > s && text[e - 1] == '\n') --e;
  while (s < e && mg_space(text[s])) ++s;
  while (e > s && mg_space(text[e - 1])) --e;
  const uint32_t len = e - s;
  const uint8_t* p = text + s;
  uint8_t k;
  if (len == 0) k = kBlank;
  else if (len == 10 && p[0] == 'B' && p[1] == 'E' && p[2] == 'G' && p[3] == 'I' && p[4] == 'N' && p[5] == ' ' &&
           p[6] == 'I' && p[7] == 'O' && p[8] == 'N' && p[9] == 'S')
    k = kBegin;
  else if (len == 8 && p[0] == 'E' && p[1] == 'N' && p[2] == 'D' && p[3] == ' ' && p[4] == 'I' && p[5] == 'O' &&
           p[6] == 'N' && p[7] == 'S')
    k = kEnd;
  else if (p[0] == '#') k = kHash;
  else if (mg_alpha(p[0])) {
    bool eq = false;
    for (uint32_t j = 1; j < len && !eq; ++j) eq = p[j] == '=';
    k = eq ? kKeyVal : kAlphaNoEq;
  } else k = kOther;
  kind[i] = k;
  ls[i] = s;
  ll[i] = len;
  is_begin[i] = k == kBegin;
  is_end[i] = k == kEnd;
}

// ---- M3: structure ------------------------------------------------------------------------------

__global__ void mgf_structure_kernel(uint32_t n_lines, const uint8_t* __restrict__ kind,
                                     const uint32_t* __restrict__ begin_before, const uint32_t* __restrict__ end_before,
                                     uint32_t* __restrict__ block_begin, uint32_t* __restrict__ block_end,
                                     uint32_t* __restrict__ is_peak, unsigned long long* err) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_lines) return;
  const uint8_t k = kind[i];
  const uint32_t b = begin_before[i], e = end_before[i];
  uint32_t peak = 0;
  if (k == kBegin) {
    if (b != e) mg_error(err, i, kErrBeginInside);  // mgf.cpp:131-133
    else block_begin[b] = i;
  } else if (k == kEnd) {
    if (b != e + 1) mg_error(err, i, kErrOutside);  // "END IONS" outside: no '=' (mgf.cpp:114-119)
    else block_end[e] = i;
  } else if (b > e) {  // inside a block (exact while the prefix is well-formed)
    if (k == kAlphaNoEq) mg_error(err, i, kErrExpectedKv);  // mgf.cpp:136-139
    else if (k == kHash || k == kOther) peak = 1;           // '#' is no comment inside a block
  } else {
    if (k == kAlphaNoEq || k == kOther) mg_error(err, i, kErrOutside);
  }
  is_peak[i] = peak;
}

// ---- number parsing -------------------------------------------------------------------------------

__constant__ double kPow10[23] = {1e0,  1e1,  1e2,  1e3,  1e4,  1e5,  1e6,  1e7,  1e8,  1e9,  1e10, 1e11,
                                  1e12, 1e13, 1e14, 1e15, 1e16, 1e17, 1e18, 1e19, 1e20, 1e21, 1e22};

__device__ __forceinline__ bool mg_ieq(const uint8_t* p, uint32_t n, const char* lit, uint32_t m) {
  if (n != m) return false;
  for (uint32_t i = 0; i < n; ++i)
    if ((p[i] | 32) != static_cast<uint8_t>(lit[i])) return false;
  return true;
}

// decimal token split the way from_chars(general) reads it; returns false on a grammar violation
struct MgDecimal {
  bool neg, special;   // special: inf / nan, value in `spec`
  double spec;
  uint64_t w;          // first <= 19 significant digits
  int32_t e10;         // value = w * 10^e10 (+ dropped digits when `truncated`)
  bool truncated;      // nonzero digits beyond the 19 kept
  bool nonzero;        // any nonzero mantissa digit
};

__device__ bool mg_scan_decimal(const uint8_t* p, uint32_t n, MgDecimal* d) {
  uint32_t i = 0;
  d->neg = false;
  d->special = false;
  if (i < n && p[i] == '-') d->neg = true, ++i;
  if (i < n && mg_alpha(p[i])) {
    if (mg_ieq(p + i, n - i, "inf", 3) || mg_ieq(p + i, n - i, "infinity", 8)) {
      d->special = true;
      d->spec = d->neg ? -__longlong_as_double(0x7FF0000000000000ll) : __longlong_as_double(0x7FF0000000000000ll);
      return true;
    }
    if (n - i >= 3 && mg_ieq(p + i, 3, "nan", 3)) {
      const uint32_t j = i + 3;
      if (j < n) {
        if (p[j] != '(' || p[n - 1] != ')') return false;
        for (uint32_t k = j + 1; k + 1 < n; ++k)
          if (!(mg_alpha(p[k]) || mg_digit(p[k]) || p[k] == '_')) return false;
      }
      d->special = true;
      d->spec = __longlong_as_double(0x7FF8000000000000ll);
      return true;
    }
    return false;
  }
  uint64_t w = 0;
  int32_t e10 = 0;
  uint32_t digits = 0, kept = 0;
  bool truncated = false, nonzero = false;
  for (; i < n && mg_digit(p[i]); ++i, ++digits) {
    const uint32_t c = p[i] - '0';
    nonzero |= c != 0;
    if (kept < 19) {
      if (w != 0 || c != 0) w = w * 10 + c, ++kept;
    } else {
      ++e10;
      truncated |= c != 0;
    }
  }
  if (i < n && p[i] == '.') {
    ++i;
    for (; i < n && mg_digit(p[i]); ++i, ++digits) {
      const uint32_t c = p[i] - '0';
      nonzero |= c != 0;
      if (kept < 19) {
        if (w != 0 || c != 0) w = w * 10 + c, ++kept;
        --e10;
      } else {
        truncated |= c != 0;
      }
    }
  }
  if (digits == 0) return false;
  if (i < n && (p[i] | 32) == 'e') {
    uint32_t j = i + 1;
    bool eneg = false;
    if (j < n && (p[j] == '+' || p[j] == '-')) eneg = p[j] == '-', ++j;
    if (j < n && mg_digit(p[j])) {
      int32_t ex = 0;
      for (; j < n && mg_digit(p[j]); ++j) ex = ex < 100000 ? ex * 10 + (p[j] - '0') : ex;
      e10 += eneg ? -ex : ex;
      i = j;
    }
  }
  if (i != n) return false;
  d->w = w;
  d->e10 = e10;
  d->truncated = truncated;
  d->nonzero = nonzero;
  return true;
}

// 0 = not a number, 1 = *out is the correctly rounded value, 2 = needs the exact path (M6)
__device__ int mg_parse_fast(const uint8_t* p, uint32_t n, double* out) {
  MgDecimal d;
  if (!mg_scan_decimal(p, n, &d)) return 0;
  if (d.special) {
    *out = d.spec;
    return 1;
  }
  if (!d.nonzero) {
    *out = d.neg ? -0.0 : 0.0;
    return 1;
  }
  if (d.truncated || d.w > (1ull << 53) || d.e10 < -22 || d.e10 > 22) return 2;
  double v = static_cast<double>(d.w);  // exact
  v = d.e10 < 0 ? v / kPow10[-d.e10] : v * kPow10[d.e10];  // one rounding
  *out = d.neg ? -v : v;
  return 1;
}

__device__ __forceinline__ uint32_t mg_token(const uint8_t* p, uint32_t n) {  // first_token, mgf.cpp:50-54
  uint32_t i = 0;
  while (i < n && !mg_space(p[i])) ++i;
  return i;
}

// ---- M4: peak lines -------------------------------------------------------------------------------

struct MgHard {
  uint32_t line;   // line index
  uint32_t block;  // kNone: a peak line; else the PEPMASS line of this block
};

__global__ void mgf_peaks_kernel(const uint8_t* __restrict__ text, uint32_t n_lines, const uint32_t* __restrict__ is_peak,
                                 const uint32_t* __restrict__ peak_rank, const uint32_t* __restrict__ ls,
                                 const uint32_t* __restrict__ ll, double* __restrict__ raw_mz,
                                 double* __restrict__ raw_int, MgHard* __restrict__ hard, uint32_t* hard_count,
                                 unsigned long long* err) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_lines || !is_peak[i]) return;
  const uint8_t* p = text + ls[i];
  const uint32_t len = ll[i];
  const uint32_t mz_n = mg_token(p, len);
  uint32_t r = mz_n;
  while (r < len && mg_space(p[r])) ++r;
  const uint32_t in_n = mg_token(p + r, len - r);
  double m = 0.0, v = 0.0;
  const int a = mg_parse_fast(p, mz_n, &m);
  const int b = mg_parse_fast(p + r, in_n, &v);
  const uint32_t slot = peak_rank[i];
  raw_mz[slot] = m;
  raw_int[slot] = v;
  if (a == 0 || b == 0) {
    mg_error(err, i, kErrPeakNumbers);
  } else if (a == 2 || b == 2) {
    hard[atomicAdd(hard_count, 1u)] = MgHard{i, kNone};
  } else if (!(m > 0.0)) {
    mg_error(err, i, kErrPeakMz);
  } else if (!(v >= 0.0)) {
    mg_error(err, i, kErrPeakIntensity);
  }
}

// ---- M5: block headers ------------------------------------------------------------------------------

__global__ void mgf_headers_kernel(const uint8_t* __restrict__ text, uint32_t n_blocks, uint32_t n_closed,
                                   const uint32_t* __restrict__ block_begin, const uint32_t* __restrict__ block_end,
                                   const uint8_t* __restrict__ kind, const uint32_t* __restrict__ ls,
                                   const uint32_t* __restrict__ ll, double* __restrict__ pepmass,
                                   uint32_t* __restrict__ pepmass_line, uint8_t* __restrict__ charge,
                                   uint32_t* __restrict__ title_off, uint32_t* __restrict__ title_len,
                                   uint32_t* __restrict__ seq_off, uint32_t* __restrict__ seq_len,
                                   MgHard* __restrict__ hard, uint32_t* hard_count, unsigned long long* err) {
  const uint32_t b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= n_blocks) return;
  const uint32_t l0 = block_begin[b], l1 = block_end[b];
  double mass = 0.0;
  uint32_t mass_line = kNone;
  uint8_t ch = 0;
  uint32_t t_off = 0, t_len = 0, s_off = 0, s_len = 0;
  for (uint32_t i = l0 + 1; i < l1; ++i) {
    if (kind[i] != kKeyVal) continue;
    const uint8_t* p = text + ls[i];
    const uint32_t len = ll[i];
    uint32_t eq = 0;
    while (p[eq] != '=') ++eq;  // kKeyVal: there is one
    uint32_t vs = eq + 1, ve = len;  // value = strip(after '=')
    while (vs < ve && mg_space(p[vs])) ++vs;
    while (ve > vs && mg_space(p[ve - 1])) --ve;
    const uint8_t* v = p + vs;
    const uint32_t vn = ve - vs;
    if (eq == 7 && p[0] == 'P' && p[1] == 'E' && p[2] == 'P' && p[3] == 'M' && p[4] == 'A' && p[5] == 'S' && p[6] == 'S') {
      double x = 0.0;
      const int r = mg_parse_fast(v, mg_token(v, vn), &x);
      if (r == 0 || (r == 1 && !(x > 0.0))) {
        mg_error(err, i, kErrPepmass);  // mgf.cpp:145-147
      } else if (r == 2) {
        hard[atomicAdd(hard_count, 1u)] = MgHard{i, b};
      }
      mass = x;
      mass_line = i;  // last PEPMASS line wins; a hard one is filled in by M6
    } else if (eq == 6 && p[0] == 'C' && p[1] == 'H' && p[2] == 'A' && p[3] == 'R' && p[4] == 'G' && p[5] == 'E') {
      // parse_charge, mgf.cpp:35-48: "2", "2+", "+2"; from_chars<unsigned> must consume everything
      const uint8_t* c = v;
      uint32_t cn = vn;
      bool ok = cn > 0;
      if (ok) {
        if (c[0] == '+') ++c, --cn;
        else if (c[cn - 1] == '+') --cn;
        ok = cn > 0;
      }
      uint64_t val = 0;
      for (uint32_t j = 0; ok && j < cn; ++j) {
        if (!mg_digit(c[j])) ok = false;
        else {
          val = val * 10 + (c[j] - '0');
          if (val > 0xFFFFFFFFull) ok = false;  // result_out_of_range
        }
      }
      if (!ok || val < 1 || val > 99) mg_error(err, i, kErrCharge);
      else ch = static_cast<uint8_t>(val);
    } else if (eq == 5 && p[0] == 'T' && p[1] == 'I' && p[2] == 'T' && p[3] == 'L' && p[4] == 'E') {
      t_off = ls[i] + vs;
      t_len = vn;
    } else if (eq == 3 && p[0] == 'S' && p[1] == 'E' && p[2] == 'Q') {
      s_off = ls[i] + vs;
      s_len = vn;
    }
  }
  // thrown at END IONS (mgf.cpp:123-125); a block still open where parsing stops never gets there
  if (mass_line == kNone && b < n_closed) mg_error(err, l1, kErrMissingPepmass);
  pepmass[b] = mass;
  pepmass_line[b] = mass_line;
  charge[b] = ch;
  title_off[b] = t_off;
  title_len[b] = t_len;
  seq_off[b] = s_off;
  seq_len[b] = s_len;
}

// ---- M6: exact decimal -> double for the hard tokens ------------------------------------------------

constexpr int kBigLimbs = 152;       // 4864 bits: 801 digits (2661 bits) + 2^1074 + headroom
constexpr int kHardThreads = 32;     // one token per thread, three big integers each in shared memory
constexpr uint32_t kMaxDigits = 800;

struct Big {
  uint32_t* v;
  int n;  // limbs in use (v[n-1] != 0, or n == 0 for zero)
};
__device__ void big_set(Big& a, uint32_t x) {
  a.n = x ? 1 : 0;
  a.v[0] = x;
}
__device__ void big_mul_add(Big& a, uint32_t m, uint32_t add) {
  uint64_t carry = add;
  for (int i = 0; i < a.n; ++i) {
    const uint64_t t = uint64_t(a.v[i]) * m + carry;
    a.v[i] = static_cast<uint32_t>(t);
    carry = t >> 32;
  }
  if (carry && a.n < kBigLimbs) a.v[a.n++] = static_cast<uint32_t>(carry);
}
__device__ void big_mul_pow10(Big& a, uint32_t k) {
  for (; k >= 9; k -= 9) big_mul_add(a, 1000000000u, 0);
  uint32_t m = 1;
  for (; k > 0; --k) m *= 10;
  if (m > 1) big_mul_add(a, m, 0);
}
__device__ int big_bits(const Big& a) { return a.n == 0 ? 0 : 32 * (a.n - 1) + (32 - __clz(a.v[a.n - 1])); }
__device__ void big_shl(Big& a, uint32_t s) {
  if (a.n == 0 || s == 0) return;
  const int ws = s >> 5, bs = s & 31;
  int nn = a.n + ws + 1;
  if (nn > kBigLimbs) nn = kBigLimbs;
  for (int i = nn - 1; i >= 0; --i) {
    const int src = i - ws;
    uint32_t lo = (src >= 0 && src < a.n) ? a.v[src] : 0;
    uint32_t below = (src - 1 >= 0 && src - 1 < a.n) ? a.v[src - 1] : 0;
    a.v[i] = bs ? (lo << bs) | (below >> (32 - bs)) : lo;
  }
  a.n = nn;
  while (a.n > 0 && a.v[a.n - 1] == 0) --a.n;
}
__device__ void big_shr1(Big& a) {
  for (int i = 0; i < a.n; ++i) a.v[i] = (a.v[i] >> 1) | (i + 1 < a.n ? a.v[i + 1] << 31 : 0);
  while (a.n > 0 && a.v[a.n - 1] == 0) --a.n;
}
__device__ int big_cmp(const Big& a, const Big& b) {
  if (a.n != b.n) return a.n < b.n ? -1 : 1;
  for (int i = a.n - 1; i >= 0; --i)
    if (a.v[i] != b.v[i]) return a.v[i] < b.v[i] ? -1 : 1;
  return 0;
}
__device__ void big_sub(Big& a, const Big& b) {  // a -= b, a >= b
  uint64_t borrow = 0;
  for (int i = 0; i < a.n; ++i) {
    const uint64_t t = uint64_t(a.v[i]) - (i < b.n ? b.v[i] : 0) - borrow;
    a.v[i] = static_cast<uint32_t>(t);
    borrow = (t >> 32) & 1;
  }
  while (a.n > 0 && a.v[a.n - 1] == 0) --a.n;
}
__device__ void big_copy(Big& d, const Big& s) {
  d.n = s.n;
  for (int i = 0; i < s.n; ++i) d.v[i] = s.v[i];
}

// exact value of the token (grammar already accepted) -> correctly rounded double; false = out of range
__device__ bool mg_parse_exact(const uint8_t* p, uint32_t n, uint32_t* mem, double* out) {
  Big A{mem, 0}, B{mem + kBigLimbs, 0}, T{mem + 2 * kBigLimbs, 0};
  uint32_t i = 0;
  const bool neg = p[0] == '-';
  if (neg) ++i;
  // all significant digits -> A (at most kMaxDigits, the rest folded into one sticky digit)
  int64_t e10 = 0;
  uint32_t nd = 0;
  bool sticky = false, frac = false;
  uint32_t chunk = 0, chunk_n = 0;
  big_set(A, 0);
  auto flush = [&]() {
    if (chunk_n == 0) return;
    uint32_t m = 1;
    for (uint32_t k = 0; k < chunk_n; ++k) m *= 10;
    if (A.n == 0) big_set(A, chunk);
    else big_mul_add(A, m, chunk);
    chunk = 0;
    chunk_n = 0;
  };
  for (; i < n; ++i) {
    const uint8_t c = p[i];
    if (c == '.') {
      frac = true;
      continue;
    }
    if (!mg_digit(c)) break;
    const uint32_t dgt = c - '0';
    if (nd == 0 && dgt == 0) {  // leading zero
      if (frac) --e10;
      continue;
    }
    if (nd < kMaxDigits) {
      chunk = chunk * 10 + dgt;
      ++nd;
      if (++chunk_n == 9) flush();
      if (frac) --e10;
    } else {
      sticky |= dgt != 0;
      if (!frac) ++e10;
    }
  }
  flush();
  if (sticky) {  // a nonzero tail only matters as "strictly above": append a 1
    big_mul_add(A, 10, 1);
    --e10;
    ++nd;
  }
  if (i < n && (p[i] | 32) == 'e') {
    ++i;
    bool eneg = false;
    if (p[i] == '+' || p[i] == '-') eneg = p[i] == '-', ++i;
    int64_t ex = 0;
    for (; i < n && mg_digit(p[i]); ++i) ex = ex < 1000000 ? ex * 10 + (p[i] - '0') : ex;
    e10 += eneg ? -ex : ex;
  }
  // value in [10^(dexp-1), 10^dexp)
  const int64_t dexp = int64_t(nd) + e10;
  if (dexp > 310) return false;   // >= 1e310: overflow
  if (dexp < -326) return false;  // < 1e-326 < 2^-1075: rounds to zero
  big_set(B, 1);
  if (e10 >= 0) big_mul_pow10(A, static_cast<uint32_t>(e10));
  else big_mul_pow10(B, static_cast<uint32_t>(-e10));
  // v = A / B in (2^(L-1), 2^(L+1)); pick e2 so that floor(v / 2^e2) has 53 or 54 bits, then fix up
  const int L = big_bits(A) - big_bits(B);
  int e2 = L - 53;
  if (e2 < -1074) e2 = -1074;
  if (e2 > 0) big_shl(B, e2);
  else big_shl(A, -e2);
  big_copy(T, B);
  big_shl(T, 54);
  uint64_t q = 0;
  for (int bit = 54; bit >= 0; --bit) {  // q = floor(A / B) < 2^54, A becomes the remainder
    if (big_cmp(A, T) >= 0) {
      big_sub(A, T);
      q |= 1ull << bit;
    }
    big_shr1(T);  // exact: T = B << bit had `bit` zero low bits
  }
  if (q >= (1ull << 53)) {
    // 54 bits: halve the scale once.  v / 2^(e2+1) = (q >> 1) + ((q & 1) * B + A) / (2 B): fold the
    // dropped quotient bit into the remainder instead of dividing again
    if (q & 1) {  // A += B
      uint64_t carry = 0;
      const int m = A.n > B.n ? A.n : B.n;
      for (int k = 0; k < m; ++k) {
        const uint64_t t = uint64_t(k < A.n ? A.v[k] : 0) + (k < B.n ? B.v[k] : 0) + carry;
        A.v[k] = static_cast<uint32_t>(t);
        carry = t >> 32;
      }
      A.n = m;
      if (carry) A.v[A.n++] = static_cast<uint32_t>(carry);
    }
    q >>= 1;
    big_shl(B, 1);
    ++e2;
  }
  // round to nearest even on remainder A against B: compare 2A with B
  big_shl(A, 1);
  const int c = big_cmp(A, B);
  if (c > 0 || (c == 0 && (q & 1))) ++q;
  uint64_t bits;
  if (q >= (1ull << 53)) {  // rounding carried out of 53 bits
    q >>= 1;
    ++e2;
  }
  if (q >= (1ull << 52)) {
    const int64_t ef = int64_t(e2) + 52 + 1023;
    if (ef >= 2047) return false;  // overflow
    bits = (static_cast<uint64_t>(ef) << 52) | (q & ((1ull << 52) - 1));
  } else {
    bits = q;  // subnormal (e2 == -1074)
    if (q == 0) return false;  // underflow to zero
  }
  if (neg) bits |= 1ull << 63;
  *out = __longlong_as_double(static_cast<long long>(bits));
  return true;
}

__device__ bool mg_parse_any(const uint8_t* p, uint32_t n, uint32_t* mem, double* out) {
  const int r = mg_parse_fast(p, n, out);
  if (r != 2) return r == 1;
  return mg_parse_exact(p, n, mem, out);
}

__global__ void __launch_bounds__(kHardThreads)
mgf_hard_kernel(const uint8_t* __restrict__ text, uint32_t n_hard, const MgHard* __restrict__ hard,
                const uint32_t* __restrict__ peak_rank, const uint32_t* __restrict__ ls,
                const uint32_t* __restrict__ ll, double* __restrict__ raw_mz, double* __restrict__ raw_int,
                double* __restrict__ pepmass, const uint32_t* __restrict__ pepmass_line, unsigned long long* err) {
  extern __shared__ uint32_t big_mem[];
  const uint32_t h = blockIdx.x * kHardThreads + threadIdx.x;
  if (h >= n_hard) return;
  uint32_t* mem = big_mem + size_t(threadIdx.x) * 3 * kBigLimbs;
  const MgHard item = hard[h];
  const uint8_t* p = text + ls[item.line];
  const uint32_t len = ll[item.line];
  if (item.block == kNone) {  // peak line: redo it with the complete parser (mgf.cpp:163-177)
    const uint32_t mz_n = mg_token(p, len);
    uint32_t r = mz_n;
    while (r < len && mg_space(p[r])) ++r;
    const uint32_t in_n = mg_token(p + r, len - r);
    double m = 0.0, v = 0.0;
    const bool a = mg_parse_any(p, mz_n, mem, &m);
    const bool b = a && mg_parse_any(p + r, in_n, mem, &v);
    if (!a || !b) mg_error(err, item.line, kErrPeakNumbers);
    else if (!(m > 0.0)) mg_error(err, item.line, kErrPeakMz);
    else if (!(v >= 0.0)) mg_error(err, item.line, kErrPeakIntensity);
    raw_mz[peak_rank[item.line]] = m;
    raw_int[peak_rank[item.line]] = v;
  } else {  // PEPMASS value
    uint32_t eq = 0;
    while (p[eq] != '=') ++eq;
    uint32_t vs = eq + 1;
    while (vs < len && mg_space(p[vs])) ++vs;
    const uint32_t tn = mg_token(p + vs, len - vs);
    double x = 0.0;
    if (!mg_parse_any(p + vs, tn, mem, &x) || !(x > 0.0)) mg_error(err, item.line, kErrPepmass);
    if (pepmass_line[item.block] == item.line) pepmass[item.block] = x;
  }
}

// ---- M7: finalize_block (mgf.cpp:78-88) ---------------------------------------------------------------

// warp per block.  Already strictly ascending: nothing to do.  Otherwise rank-sort by (m/z, position)
// == std::stable_sort by m/z into tmp, then merge runs of equal m/z (sequential sums, in order)
// back into the raw arrays at the block's start.
__global__ void mgf_finalize_kernel(uint32_t n_blocks, const uint32_t* __restrict__ block_begin,
                                    const uint32_t* __restrict__ block_end, const uint32_t* __restrict__ peak_rank,
                                    double* __restrict__ raw_mz, double* __restrict__ raw_int,
                                    double* __restrict__ tmp_mz, double* __restrict__ tmp_int,
                                    uint64_t* __restrict__ out_count, uint32_t* any_shrunk) {
  const uint32_t b = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t lane = threadIdx.x & 31;
  if (b >= n_blocks) return;
  const uint32_t p0 = peak_rank[block_begin[b]], p1 = peak_rank[block_end[b]];
  const uint32_t cnt = p1 - p0;
  double* mz = raw_mz + p0;
  double* in = raw_int + p0;
  bool asc = true;
  for (uint32_t e = lane + 1; e < cnt; e += 32) asc &= mz[e - 1] < mz[e];
  if (__all_sync(0xffffffffu, asc)) {
    if (lane == 0) out_count[b] = cnt;
    return;
  }
  double* tm = tmp_mz + p0;
  double* ti = tmp_int + p0;
  for (uint32_t e = lane; e < cnt; e += 32) {
    const double m = mz[e];
    uint32_t rank = 0;
    for (uint32_t j = 0; j < cnt; ++j) {
      const double mj = mz[j];
      rank += (mj < m) || (mj == m && j < e);
    }
    tm[rank] = m;
    ti[rank] = in[e];
  }
  __syncwarp();
  uint32_t kept = 0;
  for (uint32_t c0 = 0; c0 < cnt; c0 += 32) {
    const uint32_t e = c0 + lane;
    const bool head = e < cnt && (e == 0 || tm[e - 1] != tm[e]);
    const uint32_t mask = __ballot_sync(0xffffffffu, head);
    if (head) {
      double sum = ti[e];
      for (uint32_t t = e + 1; t < cnt && tm[t] == tm[e]; ++t) sum += ti[t];  // s.peaks.back().intensity += ...
      const uint32_t slot = kept + __popc(mask & ((1u << lane) - 1u));
      mz[slot] = tm[e];
      in[slot] = sum;
    }
    kept += __popc(mask);
  }
  if (lane == 0) {
    out_count[b] = kept;
    if (kept != cnt) atomicOr(any_shrunk, 1u);
  }
}

__global__ void mgf_raw_counts_kernel(uint32_t n_blocks, const uint32_t* __restrict__ block_begin,
                                      const uint32_t* __restrict__ block_end, const uint32_t* __restrict__ peak_rank,
                                      uint64_t* __restrict__ raw_off) {
  const uint32_t b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b > n_blocks) return;
  raw_off[b] = b < n_blocks ? peak_rank[block_begin[b]] : (n_blocks ? peak_rank[block_end[n_blocks - 1]] : 0);
}

__global__ void mgf_compact_kernel(uint32_t n_blocks, const uint64_t* __restrict__ raw_off,
                                   const uint64_t* __restrict__ out_off, const double* __restrict__ raw_mz,
                                   const double* __restrict__ raw_int, double* __restrict__ out_mz,
                                   double* __restrict__ out_int) {
  const uint32_t b = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t lane = threadIdx.x & 31;
  if (b >= n_blocks) return;
  const uint64_t s = raw_off[b], d = out_off[b], cnt = out_off[b + 1] - d;
  for (uint64_t e = lane; e < cnt; e += 32) {
    out_mz[d + e] = raw_mz[s + e];
    out_int[d + e] = raw_int[s + e];
  }
}

// ---- host orchestration -------------------------------------------------------------------------------

template <typename T>
static int scan_u32(homs_b200_ctx* ctx, const T* d_in, T* d_out, uint64_t n) {
  HB_TRY(ensure(ctx, ctx->scratch[kScrCub], exclusive_sum_temp_bytes(n)));
  return exclusive_sum<T>(ctx, d_in, d_out, n, ctx->scratch[kScrCub].p);
}

}  // namespace hb

using namespace hb;

extern "C" {

}  // extern "C"

static int mgf_parse_locked(homs_b200_ctx* ctx, const void* image, bool on_device, uint64_t n_bytes,
                            homs_b200_mgf_info* info) {
  MgfState& st = ctx->mgf;
  st = MgfState{};
  *info = homs_b200_mgf_info{};
  HB_REQUIRE(ctx, n_bytes == 0 || image, HOMS_B200_ERR_ARGUMENT, "mgf_parse: null image");
  HB_REQUIRE(ctx, n_bytes < 0xFFFFFF00ull, HOMS_B200_ERR_ARGUMENT,
             "mgf_parse: images of 4 GiB and more must be split at END IONS by the caller");
  cudaStream_t s = ctx->stream;
  const uint64_t n = n_bytes;
  // scratch map (all grow-only): text | line tables | per-block tables | peaks
  DevBuf& b_text = ctx->scratch[kScrMgfText];
  HB_TRY(ensure(ctx, b_text, n + 64));
  auto* d_text = b_text.as<uint8_t>();
  if (n)
    HB_CUDA(ctx, cudaMemcpyAsync(d_text, image, n, on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, s));
  HB_CUDA(ctx, cudaMemsetAsync(d_text + n, 0, 64, s));
  uint8_t last = '\n';
  if (n && on_device) HB_CUDA(ctx, cudaMemcpyAsync(&last, d_text + n - 1, 1, cudaMemcpyDeviceToHost, s));
  else if (n) last = static_cast<const uint8_t*>(image)[n - 1];

  // M1
  const uint32_t tiles = static_cast<uint32_t>((n + kM1Threads * kM1Bytes - 1) / (kM1Threads * kM1Bytes));
  HB_TRY(ensure(ctx, ctx->scratch[kScrMgfTiles], (size_t(tiles) + 1) * 8));
  auto* d_tile_cnt = ctx->scratch[kScrMgfTiles].as<uint32_t>();
  auto* d_tile_base = d_tile_cnt + tiles + 1;
  HB_TRY(ensure(ctx, ctx->scratch[kScrMisc], 64));
  auto* d_small = ctx->scratch[kScrMisc].as<unsigned long long>();  // [0] error key, [1] hard count, [2] any_shrunk
  const unsigned long long init[3] = {~0ull, 0, 0};
  HB_CUDA(ctx, cudaMemcpyAsync(d_small, init, sizeof init, cudaMemcpyHostToDevice, s));
  uint32_t n_newlines = 0;
  if (tiles) {
    mgf_count_newlines_kernel<<<tiles, kM1Threads, 0, s>>>(d_text, n, d_tile_cnt);
    HB_LAUNCHED(ctx);
    HB_CUDA(ctx, cudaMemsetAsync(d_tile_cnt + tiles, 0, 4, s));
    HB_TRY(scan_u32(ctx, d_tile_cnt, d_tile_base, tiles + 1));
    HB_CUDA(ctx, cudaMemcpyAsync(&n_newlines, d_tile_base + tiles, 4, cudaMemcpyDeviceToHost, s));
    HB_CUDA(ctx, cudaStreamSynchronize(s));
  }
  if (!tiles) HB_CUDA(ctx, cudaStreamSynchronize(s));
  const uint64_t n_lines64 = uint64_t(n_newlines) + (n > 0 && last != '\n' ? 1 : 0);  // std::getline
  HB_REQUIRE(ctx, n_lines64 < 0x7FFFFFF0ull, HOMS_B200_ERR_ARGUMENT, "mgf_parse: too many lines");
  const uint32_t n_lines = static_cast<uint32_t>(n_lines64);
  info->n_lines = n_lines;
  if (n_lines == 0) {
    st.ready = true;
    return HOMS_B200_OK;
  }
  const unsigned lb = (n_lines + 255) / 256;
  // line tables: start[n_newlines + 1], ls, ll, begin_flag, end_flag, begin_before, end_before, is_peak, peak_rank
  // (+1 entries for the scans' totals), kind
  const size_t L1 = size_t(n_lines) + 2;
  HB_TRY(ensure(ctx, ctx->scratch[kScrMgfLines], L1 * 4 * 10 + L1));
  auto* d_start = ctx->scratch[kScrMgfLines].as<uint32_t>();
  auto* d_ls = d_start + L1;
  auto* d_ll = d_ls + L1;
  auto* d_isb = d_ll + L1;
  auto* d_ise = d_isb + L1;
  auto* d_bb = d_ise + L1;
  auto* d_eb = d_bb + L1;
  auto* d_isp = d_eb + L1;
  auto* d_pr = d_isp + L1;
  auto* d_spare = d_pr + L1;
  auto* d_kind = reinterpret_cast<uint8_t*>(d_spare + L1);
  mgf_line_starts_kernel<<<tiles, kM1Threads, 0, s>>>(d_text, n, d_tile_base, d_start);
  HB_LAUNCHED(ctx);
  // M2
  mgf_classify_kernel<<<lb, 256, 0, s>>>(d_text, n, n_lines, d_start, d_kind, d_ls, d_ll, d_isb, d_ise);
  HB_LAUNCHED(ctx);
  HB_CUDA(ctx, cudaMemsetAsync(d_isb + n_lines, 0, 4, s));
  HB_CUDA(ctx, cudaMemsetAsync(d_ise + n_lines, 0, 4, s));
  HB_TRY(scan_u32(ctx, d_isb, d_bb, uint64_t(n_lines) + 1));
  HB_TRY(scan_u32(ctx, d_ise, d_eb, uint64_t(n_lines) + 1));
  uint32_t totals[2] = {0, 0};
  HB_CUDA(ctx, cudaMemcpyAsync(&totals[0], d_bb + n_lines, 4, cudaMemcpyDeviceToHost, s));
  HB_CUDA(ctx, cudaMemcpyAsync(&totals[1], d_eb + n_lines, 4, cudaMemcpyDeviceToHost, s));
  HB_CUDA(ctx, cudaStreamSynchronize(s));
  const uint32_t n_begin = totals[0], n_end = totals[1];
  // M3 (tables sized by the BEGIN count: a well-formed prefix never has more blocks than that)
  const size_t NB = size_t(std::max(n_begin, n_end)) + 2;
  HB_TRY(ensure(ctx, ctx->scratch[kScrMgfBlocks], NB * (4 * 7 + 8 * 4) + NB));
  auto* d_pepmass = ctx->scratch[kScrMgfBlocks].as<double>();
  auto* d_outcnt = reinterpret_cast<uint64_t*>(d_pepmass + NB);
  auto* d_outoff = d_outcnt + NB;
  auto* d_rawoff = d_outoff + NB;
  auto* d_bbeg = reinterpret_cast<uint32_t*>(d_rawoff + NB);
  auto* d_bend = d_bbeg + NB;
  auto* d_pline = d_bend + NB;
  auto* d_toff = d_pline + NB;
  auto* d_tlen = d_toff + NB;
  auto* d_soff = d_tlen + NB;
  auto* d_slen = d_soff + NB;
  auto* d_charge = reinterpret_cast<uint8_t*>(d_slen + NB);
  HB_CUDA(ctx, cudaMemsetAsync(d_bbeg, 0xFF, NB * 8, s));  // block_begin / block_end = kNone
  mgf_structure_kernel<<<lb, 256, 0, s>>>(n_lines, d_kind, d_bb, d_eb, d_bbeg, d_bend, d_isp,
                                          d_small);
  HB_LAUNCHED(ctx);
  HB_CUDA(ctx, cudaMemsetAsync(d_isp + n_lines, 0, 4, s));
  HB_TRY(scan_u32(ctx, d_isp, d_pr, uint64_t(n_lines) + 1));
  uint32_t n_raw = 0;
  unsigned long long err_key = ~0ull;
  HB_CUDA(ctx, cudaMemcpyAsync(&n_raw, d_pr + n_lines, 4, cudaMemcpyDeviceToHost, s));
  HB_CUDA(ctx, cudaMemcpyAsync(&err_key, d_small, 8, cudaMemcpyDeviceToHost, s));
  HB_CUDA(ctx, cudaStreamSynchronize(s));

  // a structural error earlier than line X makes everything at and after X meaningless; blocks that
  // end before the first structural error are well-formed and are still checked (their errors come first)
  const uint64_t first_struct = err_key == ~0ull ? ~0ull : (err_key >> 8);
  uint32_t n_blocks = n_end;  // closed blocks
  bool open_block = n_begin > n_end;  // a block still open where parsing stops: its headers are checked too
  uint32_t open_end = n_lines;
  if (first_struct != ~0ull) {
    uint32_t be[2] = {0, 0};  // BEGIN / END lines before the structural error
    HB_CUDA(ctx, cudaMemcpy(&be[0], d_bb + first_struct, 4, cudaMemcpyDeviceToHost));
    HB_CUDA(ctx, cudaMemcpy(&be[1], d_eb + first_struct, 4, cudaMemcpyDeviceToHost));
    n_blocks = be[1];
    open_block = be[0] > be[1];
    open_end = static_cast<uint32_t>(first_struct);
  }
  if (open_block) HB_CUDA(ctx, cudaMemcpyAsync(d_bend + n_blocks, &open_end, 4, cudaMemcpyHostToDevice, s));
  HB_TRY(ensure(ctx, ctx->scratch[kScrMgfPeaks], (size_t(n_raw) + 2) * 8 * 6));
  auto* d_raw_mz = ctx->scratch[kScrMgfPeaks].as<double>();
  auto* d_raw_int = d_raw_mz + n_raw + 2;
  auto* d_tmp_mz = d_raw_int + n_raw + 2;
  auto* d_tmp_int = d_tmp_mz + n_raw + 2;
  auto* d_out_mz = d_tmp_int + n_raw + 2;
  auto* d_out_int = d_out_mz + n_raw + 2;
  HB_TRY(ensure(ctx, ctx->scratch[kScrMgfHard], (size_t(n_lines) + 2) * sizeof(MgHard)));
  auto* d_hard = ctx->scratch[kScrMgfHard].as<MgHard>();
  auto* d_hard_cnt = reinterpret_cast<uint32_t*>(d_small + 1);
  auto* d_shrunk = reinterpret_cast<uint32_t*>(d_small + 2);
  // M4 + M5
  mgf_peaks_kernel<<<lb, 256, 0, s>>>(d_text, n_lines, d_isp, d_pr, d_ls, d_ll, d_raw_mz, d_raw_int, d_hard,
                                      d_hard_cnt, d_small);
  HB_LAUNCHED(ctx);
  const uint32_t n_header_blocks = n_blocks + (open_block ? 1 : 0);
  if (n_header_blocks) {
    mgf_headers_kernel<<<(n_header_blocks + 127) / 128, 128, 0, s>>>(
        d_text, n_header_blocks, n_blocks, d_bbeg, d_bend, d_kind, d_ls, d_ll, d_pepmass, d_pline, d_charge, d_toff,
        d_tlen, d_soff, d_slen, d_hard, d_hard_cnt, d_small);
    HB_LAUNCHED(ctx);
  }
  // M6
  unsigned long long small[3];
  HB_CUDA(ctx, cudaMemcpyAsync(small, d_small, sizeof small, cudaMemcpyDeviceToHost, s));
  HB_CUDA(ctx, cudaStreamSynchronize(s));
  const uint32_t n_hard = static_cast<uint32_t>(small[1]);
  info->n_hard_numbers = n_hard;
  if (n_hard) {
    const size_t smem = size_t(kHardThreads) * 3 * kBigLimbs * 4;
    HB_CUDA(ctx, cudaFuncSetAttribute(mgf_hard_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(smem)));
    mgf_hard_kernel<<<(n_hard + kHardThreads - 1) / kHardThreads, kHardThreads, smem, s>>>(
        d_text, n_hard, d_hard, d_pr, d_ls, d_ll, d_raw_mz, d_raw_int, d_pepmass, d_pline, d_small);
    HB_LAUNCHED(ctx);
    HB_CUDA(ctx, cudaMemcpyAsync(small, d_small, 8, cudaMemcpyDeviceToHost, s));
    HB_CUDA(ctx, cudaStreamSynchronize(s));
  }
  err_key = small[0];
  // unterminated last block: detected at end of input, after every line (mgf.cpp:178-180)
  if (err_key == ~0ull && n_begin > n_end) err_key = (static_cast<unsigned long long>(n_lines) << 8) | kErrUnterminated;
  if (err_key != ~0ull) {
    const uint32_t code = static_cast<uint32_t>(err_key & 0xFF);
    const uint64_t detect = err_key >> 8;
    uint64_t line = detect + 1;  // 1-based
    if (code == kErrMissingPepmass || code == kErrUnterminated) {  // these name the block's BEGIN line
      uint32_t blk = 0, bl = 0;
      if (code == kErrMissingPepmass) HB_CUDA(ctx, cudaMemcpy(&blk, d_eb + detect, 4, cudaMemcpyDeviceToHost));
      else blk = n_end;
      HB_CUDA(ctx, cudaMemcpy(&bl, d_bbeg + blk, 4, cudaMemcpyDeviceToHost));
      line = uint64_t(bl) + 1;
    }
    info->error_line = line;
    info->error_code = code;
    return set_error(ctx, HOMS_B200_ERR_PARSE, "line " + std::to_string(line) + ": " + kMgfMessages[code]);
  }
  // M7
  info->n_spectra = n_blocks;
  const uint64_t* d_offsets = d_rawoff;
  const double* f_mz = d_raw_mz;
  const double* f_int = d_raw_int;
  uint64_t n_peaks = n_raw;
  if (n_blocks) {
    mgf_raw_counts_kernel<<<(n_blocks + 1 + 255) / 256, 256, 0, s>>>(n_blocks, d_bbeg, d_bend, d_pr, d_rawoff);
    HB_LAUNCHED(ctx);
    const uint64_t threads = uint64_t(n_blocks) * 32;
    mgf_finalize_kernel<<<static_cast<unsigned>((threads + 255) / 256), 256, 0, s>>>(
        n_blocks, d_bbeg, d_bend, d_pr, d_raw_mz, d_raw_int, d_tmp_mz, d_tmp_int, d_outcnt, d_shrunk);
    HB_LAUNCHED(ctx);
    uint32_t shrunk = 0;
    HB_CUDA(ctx, cudaMemcpyAsync(&shrunk, d_shrunk, 4, cudaMemcpyDeviceToHost, s));
    HB_CUDA(ctx, cudaStreamSynchronize(s));
    if (shrunk) {  // some block merged duplicates: compact
      HB_CUDA(ctx, cudaMemsetAsync(d_outcnt + n_blocks, 0, 8, s));
      HB_TRY(scan_u32(ctx, d_outcnt, d_outoff, uint64_t(n_blocks) + 1));
      mgf_compact_kernel<<<static_cast<unsigned>((threads + 255) / 256), 256, 0, s>>>(
          n_blocks, d_rawoff, d_outoff, d_raw_mz, d_raw_int, d_out_mz, d_out_int);
      HB_LAUNCHED(ctx);
      HB_CUDA(ctx, cudaMemcpyAsync(&n_peaks, d_outoff + n_blocks, 8, cudaMemcpyDeviceToHost, s));
      HB_CUDA(ctx, cudaStreamSynchronize(s));
      d_offsets = d_outoff;
      f_mz = d_out_mz;
      f_int = d_out_int;
    }
  }
  info->n_peaks = n_peaks;
  st.ready = true;
  st.n_spectra = n_blocks;
  st.n_peaks = n_peaks;
  st.d_offsets = d_offsets;
  st.d_mz = f_mz;
  st.d_int = f_int;
  st.d_pepmass = d_pepmass;
  st.d_charge = d_charge;
  st.d_title_off = d_toff;
  st.d_title_len = d_tlen;
  st.d_seq_off = d_soff;
  st.d_seq_len = d_slen;
  return HOMS_B200_OK;
}

extern "C" {

int homs_b200_mgf_parse(homs_b200_ctx* ctx, const void* image, uint64_t n_bytes, homs_b200_mgf_info* info) {
  if (!ctx || !info) return HOMS_B200_ERR_ARGUMENT;
  Lock lock(ctx);
  return mgf_parse_locked(ctx, image, false, n_bytes, info);
}

int homs_b200_mgf_parse_dev(homs_b200_ctx* ctx, const void* d_image, uint64_t n_bytes, homs_b200_mgf_info* info) {
  if (!ctx || !info) return HOMS_B200_ERR_ARGUMENT;
  Lock lock(ctx);
  return mgf_parse_locked(ctx, d_image, true, n_bytes, info);
}

int homs_b200_mgf_fetch(homs_b200_ctx* ctx, uint64_t* offsets, double* mz, double* intensity,
                        double* precursor_mz, uint8_t* charge, uint32_t* title_off, uint32_t* title_len,
                        uint32_t* seq_off, uint32_t* seq_len) {
  if (!ctx) return HOMS_B200_ERR_ARGUMENT;
  Lock lock(ctx);
  const MgfState& st = ctx->mgf;
  HB_REQUIRE(ctx, st.ready, HOMS_B200_ERR_STATE, "mgf_fetch: no parsed MGF image in this context");
  const uint64_t n = st.n_spectra;
  cudaStream_t s = ctx->stream;
  if (offsets) {
    if (n) HB_CUDA(ctx, cudaMemcpyAsync(offsets, st.d_offsets, (n + 1) * 8, cudaMemcpyDeviceToHost, s));
    else offsets[0] = 0;
  }
  if (n) {
    if (mz && st.n_peaks) HB_CUDA(ctx, cudaMemcpyAsync(mz, st.d_mz, st.n_peaks * 8, cudaMemcpyDeviceToHost, s));
    if (intensity && st.n_peaks)
      HB_CUDA(ctx, cudaMemcpyAsync(intensity, st.d_int, st.n_peaks * 8, cudaMemcpyDeviceToHost, s));
    if (precursor_mz) HB_CUDA(ctx, cudaMemcpyAsync(precursor_mz, st.d_pepmass, n * 8, cudaMemcpyDeviceToHost, s));
    if (charge) HB_CUDA(ctx, cudaMemcpyAsync(charge, st.d_charge, n, cudaMemcpyDeviceToHost, s));
    if (title_off) HB_CUDA(ctx, cudaMemcpyAsync(title_off, st.d_title_off, n * 4, cudaMemcpyDeviceToHost, s));
    if (title_len) HB_CUDA(ctx, cudaMemcpyAsync(title_len, st.d_title_len, n * 4, cudaMemcpyDeviceToHost, s));
    if (seq_off) HB_CUDA(ctx, cudaMemcpyAsync(seq_off, st.d_seq_off, n * 4, cudaMemcpyDeviceToHost, s));
    if (seq_len) HB_CUDA(ctx, cudaMemcpyAsync(seq_len, st.d_seq_len, n * 4, cudaMemcpyDeviceToHost, s));
  }
  HB_CUDA(ctx, cudaStreamSynchronize(s));
  return HOMS_B200_OK;
}

int homs_b200_mgf_device_csr(homs_b200_ctx* ctx, uint64_t* out_n_spectra, uint64_t* out_n_peaks,
                             const uint64_t** d_offsets, const double** d_mz, const double** d_intensity,
                             const double** d_precursor_mz, const uint8_t** d_charge) {
  if (!ctx) return HOMS_B200_ERR_ARGUMENT;
  Lock lock(ctx);
  const MgfState& st = ctx->mgf;
  HB_REQUIRE(ctx, st.ready, HOMS_B200_ERR_STATE, "mgf_device_csr: no parsed MGF image in this context");
  if (out_n_spectra) *out_n_spectra = st.n_spectra;
  if (out_n_peaks) *out_n_peaks = st.n_peaks;
  if (d_offsets) *d_offsets = st.d_offsets;
  if (d_mz) *d_mz = st.d_mz;
  if (d_intensity) *d_intensity = st.d_int;
  if (d_precursor_mz) *d_precursor_mz = st.d_pepmass;
  if (d_charge) *d_charge = st.d_charge;
  return HOMS_B200_OK;
}

}  // extern "C"
