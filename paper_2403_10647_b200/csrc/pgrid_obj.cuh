// Device OBJ ingestion: the v/f subset of Wavefront OBJ parsed on the
// GPU with the reference loader's semantics (geometry.py:65-112, load_obj):
//   * lines split on universal newlines ("\n", "\r\n", lone "\r"), numbered from 1;
//   * everything from '#' on is dropped; tokens split on Python's ASCII whitespace
//     (space, \t, \n, \r, \v, \f, \x1c-\x1f);
//   * "v x y z ...": three coordinates parsed as Python float() does -- correctly rounded
//     decimal -> double, "inf"/"infinity"/"nan" any case with a sign, '_' between digits;
//   * "f a b c ...": the part of each token before the first '/' parsed as Python int();
//     1-based, negative = relative to the vertices read so far, 0 invalid; polygons are
//     fan-triangulated (i0, ik, ik+1);
//   * the first offending line (in file order) is the error the host reports.
// Lines that hold bytes >= 0x80 before '#' are handled only where ASCII tokenisation is
// provably what Python does: a non-ASCII line whose first token is "v"/"f", or that holds
// a non-ASCII Unicode whitespace character, is reported as unsupported (flag 1 << 30).
//
// Exactness of the float conversion: up to 19 significant digits with |decimal exponent|
// <= 27 are converted with exact 128-bit integer arithmetic (a product with 5^q, or a
// quotient by 5^-q with the remainder as sticky bit); everything else goes through an exact
// big-integer path (768 significant digits kept, the rest folded into the sticky bit,
// which cannot change a correctly rounded double). Rounding is round-half-even, with
// subnormals and overflow handled as IEEE 754 requires.
#pragma once

#include <cstdint>

namespace pgrid {

constexpr int OBJ_CHUNK = 8192;  // bytes per CTA of the line-break kernels
__constant__ double kObjPow10[23] = {1e0,  1e1,  1e2,  1e3,  1e4,  1e5,  1e6,  1e7,  1e8,  1e9,  1e10, 1e11,
                                     1e12, 1e13, 1e14, 1e15, 1e16, 1e17, 1e18, 1e19, 1e20, 1e21, 1e22};
constexpr unsigned OBJ_ERR_UNSUPPORTED = 1u << 30;

__device__ __forceinline__ bool obj_ws(unsigned char c) {
  return c == ' ' || (c >= 9 && c <= 13) || (c >= 0x1c && c <= 0x1f);
}
__device__ __forceinline__ bool obj_break_at(const unsigned char* __restrict__ s, unsigned long long n,
                                             unsigned long long i) {
  const unsigned char c = s[i];
  return c == '\n' || (c == '\r' && (i + 1 >= n || s[i + 1] != '\n'));
}

// ---- line splitting ---------------------------------------------------------------------
__global__ void __launch_bounds__(256)
k_obj_count_breaks(const unsigned char* __restrict__ s, unsigned long long n, unsigned* __restrict__ cnt) {
  __shared__ unsigned w[8];
  const unsigned long long base = (unsigned long long)blockIdx.x * OBJ_CHUNK;
  unsigned c = 0;
  for (int k = threadIdx.x; k < OBJ_CHUNK; k += 256) {
    const unsigned long long i = base + k;
    if (i < n) c += obj_break_at(s, n, i);
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) c += __shfl_xor_sync(0xffffffffu, c, d);
  if ((threadIdx.x & 31) == 0) w[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned t = 0;
    for (int q = 0; q < 8; ++q) t += w[q];
    cnt[blockIdx.x] = t;
  }
}

// line_end[k] = position of the k-th break (the '\n' of "\r\n"); pre = exclusive block prefix.
// Each thread owns 32 consecutive bytes so the breaks are numbered in file order.
__global__ void __launch_bounds__(256)
k_obj_line_ends(const unsigned char* __restrict__ s, unsigned long long n, const unsigned* __restrict__ pre,
                unsigned* __restrict__ line_end) {
  __shared__ unsigned w[8];
  const unsigned long long base = (unsigned long long)blockIdx.x * OBJ_CHUNK + (unsigned long long)threadIdx.x * 32;
  unsigned mask = 0;
#pragma unroll 4
  for (int k = 0; k < 32; ++k) {
    const unsigned long long i = base + k;
    if (i < n && obj_break_at(s, n, i)) mask |= 1u << k;
  }
  const unsigned c = __popc(mask);
  unsigned inc = c;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const unsigned o = __shfl_up_sync(0xffffffffu, inc, d);
    if (lane >= d) inc += o;
  }
  if (lane == 31) w[warp] = inc;
  __syncthreads();
  unsigned off = pre[blockIdx.x] + inc - c;
  for (int q = 0; q < warp; ++q) off += w[q];
  while (mask) {
    const int k = __ffs(mask) - 1;
    mask &= mask - 1;
    line_end[off++] = (unsigned)(base + k);
  }
}

// ---- numbers -----------------------------------------------------------------------------
__device__ __forceinline__ int bitlen128(unsigned __int128 m) {
  const unsigned long long hi = (unsigned long long)(m >> 64);
  return hi ? 128 - __clzll((long long)hi) : (m ? 64 - __clzll((long long)(unsigned long long)m) : 0);
}

// m * 2^e (+ a positive amount below one unit of m when sticky) -> nearest double, ties to even.
__device__ double obj_round(unsigned __int128 m, int e, bool sticky, bool neg) {
  const unsigned long long sign = neg ? 0x8000000000000000ull : 0ull;
  if (m == 0) return __longlong_as_double((long long)sign);
  const int nb = bitlen128(m);
  const int te = nb - 1 + e;  // exponent of the leading bit
  if (te > 1023) return __longlong_as_double((long long)(sign | 0x7ff0000000000000ull));
  const bool normal = te >= -1022;
  int drop = normal ? nb - 53 : -1074 - e;
  unsigned long long mant;
  if (drop <= 0) {
    mant = (unsigned long long)(m << (-drop));
  } else {
    bool half, rest;
    unsigned long long kept;
    if (drop > 128) {
      kept = 0;
      half = false;
      rest = true;
    } else {
      kept = drop == 128 ? 0ull : (unsigned long long)(m >> drop);
      half = (m >> (drop - 1)) & 1;
      const unsigned __int128 low = drop - 1 == 0 ? (unsigned __int128)0
                                                  : (m & ((((unsigned __int128)1) << (drop - 1)) - 1));
      rest = low != 0;
    }
    rest = rest || sticky;
    mant = kept + ((half && (rest || (kept & 1))) ? 1ull : 0ull);
  }
  if (normal) {
    int ex = te;
    if (mant == (1ull << 53)) {
      mant >>= 1;
      ++ex;
      if (ex > 1023) return __longlong_as_double((long long)(sign | 0x7ff0000000000000ull));
    }
    return __longlong_as_double((long long)(sign | ((unsigned long long)(ex + 1023) << 52) | (mant & ((1ull << 52) - 1))));
  }
  return __longlong_as_double((long long)(sign | mant));  // subnormal (mant == 2^52 is the least normal)
}

__device__ __forceinline__ unsigned long long pow5_u64(int k) {  // k <= 27
  unsigned long long p = 1;
  for (int i = 0; i < k; ++i) p *= 5;
  return p;
}

// Exact big-integer path (rare: > 19 significant digits or |q| > 27).
constexpr int OBJ_BIG = 96;     // 32-bit limbs (3072 bits)
constexpr int OBJ_MAXD = 768;   // significant digits kept
struct BigU {
  unsigned l[OBJ_BIG];
  int n;  // limbs in use
};
__device__ void big_set_small(BigU& a, unsigned v) {
  a.n = v ? 1 : 0;
  a.l[0] = v;
}
__device__ void big_mul_small_add(BigU& a, unsigned m, unsigned add) {
  unsigned long long carry = add;
  for (int i = 0; i < a.n; ++i) {
    const unsigned long long t = (unsigned long long)a.l[i] * m + carry;
    a.l[i] = (unsigned)t;
    carry = t >> 32;
  }
  if (carry && a.n < OBJ_BIG) a.l[a.n++] = (unsigned)carry;
}
__device__ int big_bitlen(const BigU& a) {
  int n = a.n;
  while (n > 0 && a.l[n - 1] == 0) --n;
  return n ? 32 * (n - 1) + (32 - __clz(a.l[n - 1])) : 0;
}
__device__ void big_shl(BigU& a, int s) {  // a <<= s
  if (a.n == 0 || s == 0) return;
  const int ws = s >> 5, bs = s & 31;
  int nn = a.n + ws + 1;
  if (nn > OBJ_BIG) nn = OBJ_BIG;
  for (int i = nn - 1; i >= 0; --i) {
    const int j = i - ws;
    unsigned hi = (j >= 0 && j < a.n) ? a.l[j] : 0u;
    unsigned lo = (j - 1 >= 0 && j - 1 < a.n) ? a.l[j - 1] : 0u;
    a.l[i] = bs ? (hi << bs) | (lo >> (32 - bs)) : hi;
  }
  a.n = nn;
  while (a.n > 0 && a.l[a.n - 1] == 0) --a.n;
}
__device__ void big_shr1(BigU& a) {
  for (int i = 0; i < a.n; ++i) a.l[i] = (a.l[i] >> 1) | (i + 1 < a.n ? a.l[i + 1] << 31 : 0u);
  while (a.n > 0 && a.l[a.n - 1] == 0) --a.n;
}
__device__ int big_cmp(const BigU& a, const BigU& b) {
  const int n = a.n > b.n ? a.n : b.n;
  for (int i = n - 1; i >= 0; --i) {
    const unsigned x = i < a.n ? a.l[i] : 0u, y = i < b.n ? b.l[i] : 0u;
    if (x != y) return x < y ? -1 : 1;
  }
  return 0;
}
__device__ void big_sub(BigU& a, const BigU& b) {  // a -= b (a >= b)
  long long br = 0;
  for (int i = 0; i < a.n; ++i) {
    long long t = (long long)a.l[i] - (i < b.n ? (long long)b.l[i] : 0ll) - br;
    br = t < 0;
    a.l[i] = (unsigned)(t + (br ? (1ll << 32) : 0ll));
  }
  while (a.n > 0 && a.l[a.n - 1] == 0) --a.n;
}
__device__ bool big_nonzero(const BigU& a) {
  for (int i = 0; i < a.n; ++i)
    if (a.l[i]) return true;
  return false;
}
__device__ void big_mul_pow5(BigU& a, int k) {
  while (k >= 13) {
    big_mul_small_add(a, 1220703125u, 0);  // 5^13
    k -= 13;
  }
  unsigned p = 1;
  while (k-- > 0) p *= 5;
  if (p != 1) big_mul_small_add(a, p, 0);
}
// top 64 bits of a as (m, e, sticky): a = m * 2^e + rest
__device__ void big_top64(const BigU& a, unsigned long long& m, int& e, bool& sticky) {
  const int bl = big_bitlen(a);
  if (bl <= 64) {
    m = 0;
    for (int i = (a.n < 2 ? a.n : 2) - 1; i >= 0; --i) m = (m << 32) | a.l[i];
    e = 0;
    sticky = false;
    return;
  }
  const int sh = bl - 64;
  m = 0;
  for (int b = 0; b < 64; ++b) {  // bits sh .. sh+63
    const int bit = sh + b;
    if ((a.l[bit >> 5] >> (bit & 31)) & 1u) m |= 1ull << b;
  }
  sticky = false;
  for (int bit = 0; bit < sh && !sticky; ++bit) sticky = (a.l[bit >> 5] >> (bit & 31)) & 1u;
  e = sh;
}

// Parse one float token [p, p+len) exactly as Python float(). Returns false on a syntax error.
__device__ bool obj_parse_float(const unsigned char* __restrict__ p, int len, double& out) {
  int i = 0;
  bool neg = false;
  if (i < len && (p[i] == '+' || p[i] == '-')) {
    neg = p[i] == '-';
    ++i;
  }
  // special words (case-insensitive)
  auto word = [&](const char* w, int wl) {
    if (len - i != wl) return false;
    for (int k = 0; k < wl; ++k) {
      unsigned char c = p[i + k];
      if (c >= 'A' && c <= 'Z') c += 32;
      if (c != (unsigned char)w[k]) return false;
    }
    return true;
  };
  if (word("inf", 3) || word("infinity", 8)) {
    out = __longlong_as_double((long long)((neg ? 0x8000000000000000ull : 0ull) | 0x7ff0000000000000ull));
    return true;
  }
  if (word("nan", 3)) {
    out = __longlong_as_double((long long)((neg ? 0x8000000000000000ull : 0ull) | 0x7ff8000000000000ull));
    return true;
  }
  // digits: M = int digits ++ frac digits, value = M * 10^(exp - nfrac)
  unsigned long long w = 0;
  int nsig = 0, ndig = 0;   // significant digits seen (after leading zeros), all digits
  long long nfrac = 0;      // fraction digits
  bool trunc_nz = false;    // nonzero digit beyond OBJ_MAXD
  const int dstart = i;
  auto digitpart = [&](bool frac) -> bool {  // one or more digits, '_' only between digits
    const int s0 = i;
    bool prev_digit = false;
    while (i < len) {
      const unsigned char c = p[i];
      if (c >= '0' && c <= '9') {
        ++ndig;
        if (frac) ++nfrac;
        if (nsig > 0 || c != '0') {
          if (nsig < OBJ_MAXD) {
            if (nsig < 19) w = w * 10 + (c - '0');
          } else if (c != '0') {
            trunc_nz = true;
          }
          ++nsig;
        }
        prev_digit = true;
        ++i;
      } else if (c == '_') {
        if (!prev_digit || i + 1 >= len || p[i + 1] < '0' || p[i + 1] > '9') return false;
        prev_digit = false;
        ++i;
      } else {
        break;
      }
    }
    return i > s0;
  };
  bool have_int = false, have_frac = false;
  if (i < len && p[i] >= '0' && p[i] <= '9') {
    if (!digitpart(false)) return false;
    have_int = true;
  }
  if (i < len && p[i] == '.') {
    ++i;
    if (i < len && p[i] >= '0' && p[i] <= '9') {
      if (!digitpart(true)) return false;
      have_frac = true;
    }
  }
  if (!have_int && !have_frac) return false;
  long long ex = 0;
  if (i < len && (p[i] == 'e' || p[i] == 'E')) {
    ++i;
    bool eneg = false;
    if (i < len && (p[i] == '+' || p[i] == '-')) {
      eneg = p[i] == '-';
      ++i;
    }
    if (!(i < len && p[i] >= '0' && p[i] <= '9')) return false;
    bool prev_digit = false;
    const int e0 = i;
    while (i < len) {
      const unsigned char c = p[i];
      if (c >= '0' && c <= '9') {
        if (ex < 100000000) ex = ex * 10 + (c - '0');
        prev_digit = true;
        ++i;
      } else if (c == '_') {
        if (!prev_digit || i + 1 >= len || p[i + 1] < '0' || p[i + 1] > '9') return false;
        prev_digit = false;
        ++i;
      } else {
        break;
      }
    }
    if (i == e0) return false;
    if (eneg) ex = -ex;
  }
  if (i != len) return false;
  (void)dstart;
  (void)ndig;
  if (nsig == 0) {
    out = __longlong_as_double((long long)(neg ? 0x8000000000000000ull : 0ull));
    return true;
  }
  const int kept = nsig < OBJ_MAXD ? nsig : OBJ_MAXD;
  // value = D * 10^q, D = the first `kept` significant digits
  const long long q = ex - nfrac + (nsig - kept);
  // magnitude bounds: D has `kept` digits, value in [10^(kept-1+q), 10^(kept+q))
  if (kept + q > 310) {
    out = __longlong_as_double((long long)((neg ? 0x8000000000000000ull : 0ull) | 0x7ff0000000000000ull));
    return true;
  }
  if (kept + q < -330) {
    out = __longlong_as_double((long long)(neg ? 0x8000000000000000ull : 0ull));
    return true;
  }
  if (nsig <= 19 && q >= -27 && q <= 27) {
    if (q >= 0) {
      if (w <= (1ull << 53) && q <= 22) {  // both operands exact: one rounding
        const double r = __dmul_rn((double)w, kObjPow10[q]);
        out = neg ? -r : r;
        return true;
      }
      out = obj_round((unsigned __int128)w * pow5_u64((int)q), (int)q, false, neg);
      return true;
    }
    const int k = (int)-q;
    if (w <= (1ull << 53) && k <= 22) {
      const double r = __ddiv_rn((double)w, kObjPow10[k]);
      out = neg ? -r : r;
      return true;
    }
    const unsigned long long b = pow5_u64(k);
    const int s = 127 - (64 - __clzll((long long)w));
    const unsigned __int128 num = ((unsigned __int128)w) << s;
    const unsigned __int128 quo = num / b, rem = num % b;
    out = obj_round(quo, -s - k, rem != 0, neg);
    return true;
  }
  // big-integer path: rebuild D from the token's digits
  BigU A;
  big_set_small(A, 0);
  {
    int taken = 0;
    bool started = false;
    for (int k = 0; k < len && taken < kept; ++k) {
      const unsigned char c = p[k];
      if (c == 'e' || c == 'E') break;
      if (c < '0' || c > '9') continue;
      if (!started && c == '0') continue;
      started = true;
      if (A.n == 0) big_set_small(A, (unsigned)(c - '0'));
      else big_mul_small_add(A, 10u, (unsigned)(c - '0'));
      ++taken;
    }
  }
  if (q >= 0) {
    big_mul_pow5(A, (int)q);
    unsigned long long m;
    int e;
    bool st;
    big_top64(A, m, e, st);
    out = obj_round(m, e + (int)q, st || trunc_nz, neg);
    return true;
  }
  const int k = (int)-q;
  BigU B;
  big_set_small(B, 1);
  big_mul_pow5(B, k);
  const int s = big_bitlen(B) - big_bitlen(A) + 56;
  if (s >= 0) big_shl(A, s);
  else big_shl(B, -s);
  // restoring division: quotient < 2^58
  BigU Bs = B;
  big_shl(Bs, 57);
  unsigned long long Q = 0;
  for (int bit = 57; bit >= 0; --bit) {
    if (big_cmp(A, Bs) >= 0) {
      big_sub(A, Bs);
      Q |= 1ull << bit;
    }
    big_shr1(Bs);
  }
  out = obj_round(Q, -s - k, big_nonzero(A) || trunc_nz, neg);
  return true;
}

// Python int() of an ASCII token (sign, digits, '_' between digits). mag saturates at 2^40.
__device__ bool obj_parse_int(const unsigned char* __restrict__ p, int len, long long& out) {
  int i = 0;
  bool neg = false;
  if (i < len && (p[i] == '+' || p[i] == '-')) {
    neg = p[i] == '-';
    ++i;
  }
  if (i >= len) return false;
  long long v = 0;
  bool prev_digit = false;
  for (; i < len; ++i) {
    const unsigned char c = p[i];
    if (c >= '0' && c <= '9') {
      if (v < (1ll << 40)) v = v * 10 + (c - '0');
      prev_digit = true;
    } else if (c == '_') {
      if (!prev_digit || i + 1 >= len || p[i + 1] < '0' || p[i + 1] > '9') return false;
      prev_digit = false;
    } else {
      return false;
    }
  }
  if (!prev_digit) return false;
  out = neg ? -v : v;
  return true;
}

// ---- per-line passes ---------------------------------------------------------------------
struct ObjLine {
  unsigned long long b, e;  // content bytes [b, e) (comment removed)
};
__device__ __forceinline__ ObjLine obj_line(const unsigned char* __restrict__ s, unsigned long long n,
                                            const unsigned* __restrict__ line_end, unsigned long long L,
                                            unsigned long long li) {
  const unsigned long long b = li == 0 ? 0ull : (unsigned long long)line_end[li - 1] + 1;
  const unsigned long long e = li + 1 == L && (unsigned long long)line_end[li] >= n ? n : line_end[li];
  unsigned long long c = b;
  while (c < e && s[c] != '#') ++c;
  return {b, c};
}
// next token in [pos, e): returns false when none; [tb, te)
__device__ __forceinline__ bool obj_next_token(const unsigned char* __restrict__ s, unsigned long long& pos,
                                               unsigned long long e, unsigned long long& tb, unsigned long long& te) {
  while (pos < e && obj_ws(s[pos])) ++pos;
  if (pos >= e) return false;
  tb = pos;
  while (pos < e && !obj_ws(s[pos])) ++pos;
  te = pos;
  return true;
}
// Python-whitespace characters outside ASCII (UTF-8): U+0085, U+00A0, U+1680, U+2000-200A,
// U+2028, U+2029, U+202F, U+205F, U+3000
__device__ bool obj_has_unicode_ws(const unsigned char* __restrict__ s, unsigned long long b, unsigned long long e) {
  for (unsigned long long i = b; i + 1 < e; ++i) {
    const unsigned char c = s[i], d = s[i + 1];
    if (c == 0xC2 && (d == 0x85 || d == 0xA0)) return true;
    if (i + 2 < e) {
      const unsigned char f = s[i + 2];
      if (c == 0xE1 && d == 0x9A && f == 0x80) return true;
      if (c == 0xE2 && d == 0x80 && (f <= 0x8A || f == 0xA8 || f == 0xA9 || f == 0xAF)) return true;
      if (c == 0xE2 && d == 0x81 && f == 0x9F) return true;
      if (c == 0xE3 && d == 0x80 && f == 0x80) return true;
    }
  }
  return false;
}

// Pass 1: per line (vertex count, triangle count) packed as (v << 32 | t); first error line
// (1-based) into *err via atomicMin.
__global__ void __launch_bounds__(128)
k_obj_classify(const unsigned char* __restrict__ s, unsigned long long n, const unsigned* __restrict__ line_end,
               unsigned long long L, unsigned long long* __restrict__ info, unsigned long long* __restrict__ err) {
  const unsigned long long li = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (li >= L) return;
  const ObjLine ln = obj_line(s, n, line_end, L, li);
  bool ascii = true;
  for (unsigned long long c = ln.b; c < ln.e; ++c) ascii &= s[c] < 0x80;
  unsigned long long pos = ln.b, tb, te;
  unsigned long long r = 0;
  if (obj_next_token(s, pos, ln.e, tb, te)) {
    const bool is_v = te - tb == 1 && s[tb] == 'v', is_f = te - tb == 1 && s[tb] == 'f';
    if (!ascii && (is_v || is_f || obj_has_unicode_ws(s, ln.b, ln.e))) {
      atomicMin(err, li + 1);
    } else if (is_v || is_f) {
      unsigned long long k = 0, a, z;
      while (obj_next_token(s, pos, ln.e, a, z)) ++k;
      if (k < 3) atomicMin(err, li + 1);  // "vertex needs 3 coordinates" / "face needs at least 3 vertices"
      else r = is_v ? (1ull << 32) : (k - 2);
    }
  }
  info[li] = r;
}

// Pass 2: parse and write. vpre/tpre: exclusive prefix of info (vertices << 32 | triangles).
__global__ void __launch_bounds__(128)
k_obj_parse(const unsigned char* __restrict__ s, unsigned long long n, const unsigned* __restrict__ line_end,
            unsigned long long L, const unsigned long long* __restrict__ info, const unsigned long long* __restrict__ pre,
            double* __restrict__ V, int* __restrict__ T, unsigned long long* __restrict__ err) {
  const unsigned long long li = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (li >= L) return;
  const unsigned long long r = info[li];
  if (!r) return;
  const ObjLine ln = obj_line(s, n, line_end, L, li);
  unsigned long long pos = ln.b, tb, te;
  obj_next_token(s, pos, ln.e, tb, te);  // "v" / "f"
  const unsigned long long pv = pre[li];
  const long long nverts = (long long)(pv >> 32);
  if (r >> 32) {  // vertex
    double x[3];
    for (int k = 0; k < 3; ++k) {
      obj_next_token(s, pos, ln.e, tb, te);
      if (!obj_parse_float(s + tb, (int)min(te - tb, 1ull << 30), x[k])) {
        atomicMin(err, li + 1);  // "bad vertex coordinate"
        return;
      }
    }
    double* out = V + 3 * nverts;
    out[0] = x[0];
    out[1] = x[1];
    out[2] = x[2];
    return;
  }
  unsigned long long tri = pv & 0xffffffffull;
  int i0 = 0, prev = 0, k = 0;
  while (obj_next_token(s, pos, ln.e, tb, te)) {
    unsigned long long fe = tb;
    while (fe < te && s[fe] != '/') ++fe;
    long long idx;
    if (!obj_parse_int(s + tb, (int)(fe - tb), idx)) {
      atomicMin(err, li + 1);  // "bad face index"
      return;
    }
    if (idx > 0) idx -= 1;
    else if (idx < 0) idx += nverts;
    else {
      atomicMin(err, li + 1);  // "face index 0 is not valid"
      return;
    }
    if (idx < 0 || idx >= nverts) {
      atomicMin(err, li + 1);  // "face index ... out of range"
      return;
    }
    if (k == 0) i0 = (int)idx;
    else if (k >= 2) {
      int* t = T + 3 * tri++;
      t[0] = i0;
      t[1] = prev;
      t[2] = (int)idx;
    }
    prev = (int)idx;
    ++k;
  }
}

// Exclusive scan of u64 (three-kernel reduce-then-scan, tiles of 2048).
constexpr int OS_TILE = 2048;
__global__ void __launch_bounds__(256)
k_u64_tile_sums(const unsigned long long* __restrict__ in, unsigned long long n, unsigned long long* __restrict__ sums) {
  __shared__ unsigned long long w[8];
  const unsigned long long base = (unsigned long long)blockIdx.x * OS_TILE;
  unsigned long long v = 0;
#pragma unroll
  for (int q = 0; q < OS_TILE / 256; ++q) {
    const unsigned long long i = base + q * 256 + threadIdx.x;
    if (i < n) v += in[i];
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
  if ((threadIdx.x & 31) == 0) w[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t = 0;
    for (int q = 0; q < 8; ++q) t += w[q];
    sums[blockIdx.x] = t;
  }
}
// sums -> exclusive prefix in place, one CTA (sequential over chunks of 1024); total at sums[nt]
__global__ void __launch_bounds__(1024)
k_u64_scan_sums(unsigned long long* __restrict__ sums, unsigned long long nt) {
  __shared__ unsigned long long w[32];
  unsigned long long carry = 0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (unsigned long long base = 0; base < nt; base += 1024) {
    const unsigned long long i = base + threadIdx.x;
    const unsigned long long v = i < nt ? sums[i] : 0ull;
    unsigned long long inc = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const unsigned long long o = __shfl_up_sync(0xffffffffu, inc, d);
      if (lane >= d) inc += o;
    }
    if (lane == 31) w[warp] = inc;
    __syncthreads();
    unsigned long long add = 0, tot = 0;
    for (int q = 0; q < 32; ++q) {
      add += q < warp ? w[q] : 0ull;
      tot += w[q];
    }
    if (i < nt) sums[i] = carry + add + inc - v;
    carry += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) sums[nt] = carry;
}
__global__ void __launch_bounds__(256)
k_u64_tile_apply(const unsigned long long* __restrict__ in, unsigned long long n,
                 const unsigned long long* __restrict__ sums, unsigned long long* __restrict__ out) {
  __shared__ unsigned long long w[8];
  const unsigned long long base = (unsigned long long)blockIdx.x * OS_TILE + (unsigned long long)threadIdx.x * 8;
  unsigned long long v[8], run = 0;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const unsigned long long i = base + q;
    v[q] = i < n ? in[i] : 0ull;
  }
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const unsigned long long c = v[q];
    v[q] = run;
    run += c;
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned long long inc = run;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const unsigned long long o = __shfl_up_sync(0xffffffffu, inc, d);
    if (lane >= d) inc += o;
  }
  if (lane == 31) w[warp] = inc;
  __syncthreads();
  unsigned long long add = sums[blockIdx.x] + inc - run;
  for (int q = 0; q < warp; ++q) add += w[q];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const unsigned long long i = base + q;
    if (i < n) out[i] = add + v[q];
  }
}

}  // namespace pgrid
