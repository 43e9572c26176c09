// pgrid_kernels.cuh -- sm_100a kernels of the parallel uniform-grid build.
//
// Data path:
//   K1 k_boxes_count_scan : triangle AABB -> clamped cell box -> CountCells, fused with a
//                           decoupled-look-back exclusive scan (builders.py:90-101,
//                           gridcore.py:145-167, primitives.py:36-44)
//   K2 k_expand_pairs     : load-balanced <cell, triangle> pair expansion (MakeObjectIds +
//                           InclusiveSum + SegmentedExclusiveSum + MakeCellIds,
//                           builders.py:155-160 / 104-117) + all radix digit histograms
//   K3 k_radix_scatter    : one stable LSD digit pass (tile counts -> row scan -> scatter)
//                           (builders.py:123-125 -> _ckernels.pyx:21-50)
//   K4 k_cell_offsets     : RunLengthEncode -> NonEmptyCells scatter -> ExclusiveSum, fused:
//                           G[c] = #pairs with cell < c (builders.py:126-133)
// All integer work is exact; the only floating point is the f64 sub/div/floor of K1, done
// with explicit round-to-nearest intrinsics so it matches numpy bit for bit.
#pragma once

#include <math_constants.h>
#include <cstdint>

#ifndef PGRID_RANK_BALLOT
#define PGRID_RANK_BALLOT 1
#endif
#include <cuda_runtime.h>

namespace pgrid {

// Checked builds (-DPGRID_CHECKED=1, `make checked`): every computed shared / global index of
// the hot kernels is bounds-checked on the device and a violation traps, so the launch fails
// and the caller sees a CUDA error. The GPU test suite runs against this build as well
// (tools/checked_tests.sh) in place of compute-sanitizer, which this GPU pool does not allow.
#ifndef PGRID_CHECKED
#define PGRID_CHECKED 0
#endif
#define PG_ASSERT(c)                   \
  do {                                 \
    if (PGRID_CHECKED && !(c)) __trap(); \
  } while (0)

// ----------------------------------------------------------------------------------------
// common helpers
// ----------------------------------------------------------------------------------------

// Programmatic dependent launch (the build's kernel chain, pgrid.cu pdl_launch): a kernel
// launched with the programmatic-serialization attribute may become resident while its
// predecessor drains. pdl_wait() returns once the predecessor grid has completed and its
// writes are visible (a no-op for a normal launch), so it comes before any global access, and
// every kernel's wait also orders it after all earlier grids (each waited on its own).
// pdl_trigger() after it would let the successor launch before this grid retires (off, below).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
// The early trigger is compiled out: with every link triggering at kernel entry a cfg3 build
// replayed 6% slower (0.815 vs 0.767 ms; glue-only or bulk-only links were neutral), while the
// untriggered chain (successor launches as the predecessor retires) measured 0.765 ms.
#ifndef PGRID_PDL_TRIGGER
#define PGRID_PDL_TRIGGER 0
#endif
__device__ __forceinline__ void pdl_trigger() {
#if PGRID_PDL_TRIGGER
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}
#define PDL_ENTRY() \
  do {              \
    pdl_wait();     \
    pdl_trigger();  \
  } while (0)

struct DevSpec {
  double lo[3];
  double hi[3];
  double cell[3];
  int dims[3];
  double rcell[3];  // RN(1 / cell): the fast path of floor_quot
};

// Per-pass digit plan for the radix sort.
constexpr int kMaxPasses = 4;
struct PassPlan {
  int npasses;
  int shift[kMaxPasses];
  int bits[kMaxPasses];
};

// A pair count known either on the host (dev == nullptr: val) or only on the device (the
// sync-free build: *dev, bounded by val = the capacity the buffers were sized for). Kernels
// downstream of K1 take their NO this way so a whole build can be enqueued -- and captured
// in a CUDA graph -- without reading NO back first. A device count above the capacity voids
// the build (the host reports it afterwards: capacity / SizeError), so every kernel then
// sees 0 pairs: no kernel ever walks offsets that wrapped past 2^32 (NO > 2^32-1).
struct Count {
  const unsigned long long* dev;
  unsigned val;
  __device__ __forceinline__ unsigned get() const {
    if (!dev) return val;
    const unsigned long long v = *dev;
    return v <= (unsigned long long)val ? (unsigned)v : 0u;
  }
};

__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_relaxed_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_u32(unsigned* p, unsigned v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// numpy float64 -> int64 astype on x86-64 (cvttsd2si): NaN / out-of-range -> INT64_MIN.
// gridcore.py:161-162 floors then casts; CUDA's cvt saturates instead, so emulate x86.
__device__ __forceinline__ long long np_floor_i64(double q) {
  const double f = floor(q);
  return (f >= -9223372036854775808.0 && f < 9223372036854775808.0) ? (long long)f
                                                                     : (long long)(-9223372036854775807LL - 1);
}
// floor(RN(x / c)) -- numpy's `floor((a - lo) / cell_size)` (gridcore.py:161-162) -- exactly,
// mostly without the division: p = RN(x * RN(1/c)) is within 3 ulp of RN(x / c) (two
// roundings of relative size 2^-53 each, plus the quotient's own), so when the window p +-
// 2^-50 |p| holds no integer both have the same floor. Integral or near-integral products,
// huge or non-finite values and degenerate cell sizes take the IEEE division.
__device__ __forceinline__ double floor_quot(double x, double c, double rc) {
  const double p = __dmul_rn(x, rc);
  const double f = floor(p);
  const double ap = fabs(p);
  const double tol = __dmul_rn(ap, 0x1p-50);
  if (ap < 0x1p52 && rc > 0.0 && rc < 1.0e308 && __dsub_rn(p, f) > tol && __dsub_rn(__dadd_rn(f, 1.0), p) > tol)
    return f;
  return floor(__ddiv_rn(x, c));
}

__device__ __forceinline__ unsigned clip_axis(long long v, int dim) {
  return v < 0 ? 0u : (v > (long long)(dim - 1) ? (unsigned)(dim - 1) : (unsigned)v);
}
// clip_axis(np_floor_i64(f), dim) for an already floored f (floor_quot's result), without the
// 64-bit integer detour: NaN and |f| >= 2^63 cast to INT64_MIN on x86 and clip to 0, a negative
// f clips to 0, the rest to min(f, dim - 1) -- all exact in f64 (f is integral). K1 is issue-
// bound next to its HBM stream, so the six per-triangle conversions are kept short.
__device__ __forceinline__ unsigned cell_of(double f, double dmax) {
  return (f >= 0.0 && f < 9223372036854775808.0) ? (unsigned)fmin(f, dmax) : 0u;
}

// Warp-cooperative 32-ary lower_bound: smallest i in [0, n] with load(i) >= x (load(n) = +inf).
// 5 rounds of 32 parallel probes cover 2^25 elements; each round is one L2/HBM latency.
template <typename Load>
__device__ __forceinline__ unsigned long long warp_lower_bound(unsigned long long n, unsigned long long x,
                                                               Load load) {
  const int lane = threadIdx.x & 31;
  unsigned long long lo = 0, hi = n;  // answer in [lo, hi]; load(lo-1) < x; load(hi) >= x or hi == n
  while (lo < hi) {
    const unsigned long long span = hi - lo;
    const unsigned long long step = (span + 31) / 32;
    const unsigned long long p = lo + (unsigned long long)lane * step;
    const bool ge = (p < hi) ? (load(p) >= x) : true;
    const unsigned ball = __ballot_sync(0xffffffffu, ge);
    // f = first lane whose probe is >= x; 32 if every probe is < x (then the answer is past
    // lane 31's probe: all 32 probes can lie inside [lo, hi) when 31*step < span)
    const int f = ball ? __ffs(ball) - 1 : 32;
    if (f == 0) {
      hi = lo;
    } else {
      lo = lo + (unsigned long long)(f - 1) * step + 1;
      if (f < 32) {
        const unsigned long long pf = (lo - 1) + step;
        hi = pf < hi ? pf : hi;
      }
    }
  }
  return lo;
}

// ----------------------------------------------------------------------------------------
// K1: boxes + counts + decoupled-look-back exclusive scan
// ----------------------------------------------------------------------------------------
constexpr int K1_THREADS = 256;
constexpr int K1_ROUNDS = 2;                       // triangles per thread (striped rounds)
constexpr int K1_TILE = K1_THREADS * K1_ROUNDS;    // 512 triangles per CTA
constexpr unsigned long long LB_AGG = 1ull << 62;
constexpr unsigned long long LB_PREFIX = 2ull << 62;
constexpr unsigned long long LB_VALUE = (1ull << 62) - 1;

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned phase) {
  unsigned done = 0;
  while (!done) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
  }
}
// TMA bulk copy global -> shared (no tensor map): 16-byte aligned, size a multiple of 16.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

struct K1Smem {
  double v[K1_TILE * 9];   // the tile's 3*K1_TILE vertices when the mesh is a soup (36 KB)
  int t[K1_TILE * 3];      // the tile's triangle indices (6 KB)
  unsigned long long bar;
  unsigned tile;
};

// Per-triangle record written by K1 and read by K2: {lo_cell, mx, my, pair offset}.
// mx/my are the box extents in x/y; count = mx*my*mz is implied by the offsets.
// Dropped triangles (keep == false, gridcore.py:159) are {0, 1, 1, off} with count 0.
//
// Data movement: one elected thread streams the tile's 6 KB of indices and -- speculatively,
// as if the mesh were an unshared-vertex soup (geometry.py:206-207) -- its 36 KB of vertex
// rows into shared memory with TMA bulk copies on an mbarrier. If every index of the tile
// is 3*i+k the boxes are computed from shared memory; otherwise (indexed meshes) the
// vertices are gathered from global memory. Both paths compute the same IEEE f64 values.
// gridcore.py:155-167 for one triangle: keep flag and clamped cell box (lo, hi inclusive)
__device__ __forceinline__ void tri_box_raw(const double* a, const double* b, const double* c, const DevSpec& s,
                                            unsigned (&lo)[3], unsigned (&hi)[3], bool& keep) {
  keep = true;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const double x0 = a[k], x1 = b[k], x2 = c[k];
    // np.min/np.max propagate NaN, which fails both comparisons (gridcore.py:156-159);
    // fmin/fmax do not, so NaN is folded into keep explicitly.
    const bool nan = isnan(x0) | isnan(x1) | isnan(x2);
    const double mn = fmin(fmin(x0, x1), x2);
    const double mx = fmax(fmax(x0, x1), x2);
    keep &= !nan && (mx >= s.lo[k]) && (mn <= s.hi[k]);
    // one IEEE subtract, one IEEE divide, floor (gridcore.py:161-162)
    const double dmax = (double)(s.dims[k] - 1);
    lo[k] = cell_of(floor_quot(__dsub_rn(mn, s.lo[k]), s.cell[k], s.rcell[k]), dmax);
    hi[k] = cell_of(floor_quot(__dsub_rn(mx, s.lo[k]), s.cell[k], s.rcell[k]), dmax);
  }
}

// Signed pair count prod(hi - lo + 1) of a kept box (builders.py:96): an inverted box (hi < lo
// on some axis: an infinite / > 2^63-cell upper corner casts to INT64_MIN and clips to 0,
// gridcore.py:161-165) counts <= 0, or > 0 when exactly two axes invert.
__device__ __forceinline__ long long signed_count(const unsigned (&lo)[3], const unsigned (&hi)[3]) {
  return ((long long)hi[0] - lo[0] + 1) * ((long long)hi[1] - lo[1] + 1) * ((long long)hi[2] - lo[2] + 1);
}

__device__ __forceinline__ void tri_box(const double* a, const double* b, const double* c, const DevSpec& s,
                                        unsigned dx, unsigned dxy, uint3& box, unsigned& cnt, bool& bad) {
  bool keep;
  unsigned lo[3], hi[3];
  tri_box_raw(a, b, c, s, lo, hi, keep);
  box = make_uint3(0u, 1u, 1u);
  cnt = 0;
  if (!keep) return;
  if (hi[0] < lo[0] || hi[1] < lo[1] || hi[2] < lo[2]) {
    // inverted box: flagged for the host's verdict (count_check). A positive count (two
    // inverted axes) keeps its pairs, {lo_cell 0, mx = count, my = 1} so the expansion stays
    // in [0, count) < ncells; k_inverted_pairs rewrites them with the reference's cells.
    bad = true;
    const long long sc = signed_count(lo, hi);
    if (sc > 0) {
      box = make_uint3(0u, (unsigned)sc, 1u);
      cnt = (unsigned)sc;  // < ncells: |hi - lo + 1| <= dims - 2 on an inverted axis
    }
    return;
  }
  const unsigned ex = hi[0] - lo[0] + 1, ey = hi[1] - lo[1] + 1, ez = hi[2] - lo[2] + 1;
  box = make_uint3(lo[0] + dx * lo[1] + dxy * lo[2], ex, ey);
  cnt = ex * ey * ez;  // <= ncells
}

// Error path of K1 (some kept box is inverted): the reference's verdict depends on the
// number of kept triangles and on the inverted boxes' signed counts (builders.py:90-101 ->
// exclusive_sum rejects a negative count, primitives.py:22-25; mark_boundaries rejects a
// zero count among >= 2 kept objects, primitives.py:66-72). out = {kept, inverted, negative
// counts, zero counts}; positive-count inverted boxes are listed in `list` (*nlist of them).
__global__ void __launch_bounds__(256)
k_inverted_boxes(const double* __restrict__ V, const int* __restrict__ T, long long n, DevSpec s,
                 unsigned long long* __restrict__ out, unsigned* __restrict__ list, unsigned* __restrict__ nlist) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  bool keep = false, inv = false, neg = false, zero = false;
  if (i < n) {
    unsigned lo[3], hi[3];
    tri_box_raw(V + 3 * (long long)T[3 * i], V + 3 * (long long)T[3 * i + 1], V + 3 * (long long)T[3 * i + 2], s, lo,
                hi, keep);
    inv = keep && (hi[0] < lo[0] || hi[1] < lo[1] || hi[2] < lo[2]);
    if (inv) {
      const long long c = signed_count(lo, hi);
      neg = c < 0;
      zero = c == 0;
      if (c > 0 && list) list[atomicAdd(nlist, 1u)] = (unsigned)i;
    }
  }
  const unsigned b[4] = {__ballot_sync(0xffffffffu, keep), __ballot_sync(0xffffffffu, inv),
                         __ballot_sync(0xffffffffu, neg), __ballot_sync(0xffffffffu, zero)};
  if ((threadIdx.x & 31) == 0) {
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (b[q]) atomicAdd(out + q, (unsigned long long)__popc(b[q]));
  }
}

// K1b for the build chain, on many CTAs: CTA c scans tile sums [c*MS_PER, (c+1)*MS_PER) and
// first adds up every tile sum before its range itself (at most ntiles u64 from L2, read in
// one coalesced sweep), so no CTA waits for another; the last CTA writes the total NO.
// (k_scan_tile_sums: the same result on one SM, 9-10 us at cfg3; this one ~3 us.)
constexpr int MS_THREADS = 1024;
constexpr int MS_PER = 1024;  // tiles per CTA
__global__ void __launch_bounds__(MS_THREADS)
k_scan_tile_sums_mc(const unsigned long long* __restrict__ tile_sum, unsigned ntiles, unsigned* __restrict__ tile_pre,
                    unsigned long long* __restrict__ total) {
  PDL_ENTRY();
  __shared__ unsigned long long wsum[MS_THREADS / 32];
  __shared__ unsigned long long pre_sh;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned c0 = blockIdx.x * (unsigned)MS_PER;
  const unsigned i = c0 + tid;
  const unsigned long long v = i < ntiles ? __ldg(&tile_sum[i]) : 0ull;
  unsigned long long part = 0;
#pragma unroll 8
  for (unsigned j = tid; j < c0; j += MS_THREADS) part += __ldg(&tile_sum[j]);
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) part += __shfl_xor_sync(0xffffffffu, part, d);
  if (lane == 0) wsum[warp] = part;
  __syncthreads();
  if (warp == 0) {
    unsigned long long x = wsum[lane];
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) x += __shfl_xor_sync(0xffffffffu, x, d);
    if (lane == 0) pre_sh = x;
  }
  __syncthreads();
  // exclusive scan of this CTA's tile sums
  unsigned long long inc = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const unsigned long long o = __shfl_up_sync(0xffffffffu, inc, d);
    if (lane >= d) inc += o;
  }
  if (lane == 31) wsum[warp] = inc;
  __syncthreads();
  unsigned long long carry = pre_sh, tot = pre_sh;
  for (int w = 0; w < MS_THREADS / 32; ++w) {
    const unsigned long long x = wsum[w];
    carry += w < warp ? x : 0ull;
    tot += x;
  }
  if (i < ntiles) tile_pre[i] = (unsigned)(carry + inc - v);
  if (blockIdx.x == gridDim.x - 1 && tid == 0) *total = tot;
}

// absolute pair offset of triangle o (K1 tiles of K1_TILE triangles)
__device__ __forceinline__ unsigned tri_offset(const uint4* __restrict__ rec, const unsigned* __restrict__ tile_pre,
                                               long long o) {
  return __ldg(&tile_pre[o / K1_TILE]) + __ldg(&rec[o].w);
}

// the index array of an implicit soup (T[i][k] = 3i + k), for the rare paths that read T
__global__ void k_soup_indices(int* __restrict__ T, long long count) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (long long)gridDim.x * blockDim.x)
    T[i] = (int)i;
}

// numpy's `//` on int64 (floor division), as _make_cell_ids uses it (builders.py:111-112)
__device__ __forceinline__ long long floordiv_i64(long long a, long long b) {
  const long long q = a / b;
  return (a % b != 0 && ((a < 0) != (b < 0))) ? q - 1 : q;
}

// Pairs of the listed positive-count inverted boxes, one CTA per box: the reference's cell of
// relative offset rel (_make_cell_ids, builders.py:104-117, signed extents, floor division).
// A cell outside [0, ncells) is the reference's InvariantError (radix_sort_pairs / scatter
// range checks, primitives.py:102-111, 135-136): err |= 1. With `keys` (the pairs in
// generation order, K2's output) the cells are written at the box's pair offset, and a
// coarse histogram of the keys (sharded builds) is corrected for the rewritten keys.
__global__ void __launch_bounds__(256)
k_inverted_pairs(const double* __restrict__ V, const int* __restrict__ T, DevSpec s, const uint4* __restrict__ rec,
                 const unsigned* __restrict__ tile_pre, const unsigned* __restrict__ list,
                 const unsigned* __restrict__ nlist, long long ncells, unsigned* __restrict__ keys,
                 unsigned* __restrict__ coarse, int coarse_shift, unsigned* __restrict__ err) {
  const unsigned nl = *nlist;
  const long long dx = s.dims[0], dy = s.dims[1];
  for (unsigned e = blockIdx.x; e < nl; e += gridDim.x) {
    const long long i = list[e];
    unsigned lo[3], hi[3];
    bool keep;
    tri_box_raw(V + 3 * (long long)T[3 * i], V + 3 * (long long)T[3 * i + 1], V + 3 * (long long)T[3 * i + 2], s, lo,
                hi, keep);
    const long long mx = (long long)hi[0] - lo[0] + 1, my = (long long)hi[1] - lo[1] + 1;
    const long long cnt = signed_count(lo, hi), mxy = mx * my;
    const unsigned off = keys ? tri_offset(rec, tile_pre, i) : 0u;
    for (long long rel = threadIdx.x; rel < cnt; rel += blockDim.x) {
      const long long z = floordiv_i64(rel, mxy);
      const long long y = floordiv_i64(rel - z * mxy, mx);
      const long long x = rel - mx * (y + my * z);
      const long long c = ((long long)lo[0] + x) + dx * (((long long)lo[1] + y) + dy * ((long long)lo[2] + z));
      if (c < 0 || c >= ncells) {
        atomicOr(err, 1u);
        continue;
      }
      if (keys) {
        const unsigned p = off + (unsigned)rel;
        PG_ASSERT(rel < cnt && (unsigned long long)off + (unsigned long long)rel < (1ull << 32));
        if (coarse) {
          atomicSub(&coarse[keys[p] >> coarse_shift], 1u);
          atomicAdd(&coarse[(unsigned)c >> coarse_shift], 1u);
        }
        keys[p] = (unsigned)c;
      }
    }
  }
}

// K1a: boxes + counts of one 512-triangle tile; rec.w = the pair offset relative to the tile
// start, tile_sum[tile] = the tile's pair count (u64). The cross-tile exclusive scan is
// k_scan_tile_sums (reduce-then-scan: a decoupled look-back here serialises at roughly
// window/round-trip tiles per microsecond on B200).
__global__ void __launch_bounds__(K1_THREADS)
k_boxes_count(const double* __restrict__ V, long long nv, const int* __restrict__ T, long long n, DevSpec s,
              int bulk_ok, uint4* __restrict__ rec, unsigned long long* __restrict__ tile_sum,
              unsigned* __restrict__ err, unsigned tile0 = 0) {
  PDL_ENTRY();
  extern __shared__ __align__(128) unsigned char smem_raw[];
  K1Smem& sm = *reinterpret_cast<K1Smem*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned tile = tile0 + blockIdx.x;  // tile0: launches per copied chunk of an implicit soup
  const long long tbase = (long long)tile * K1_TILE;
  const int tcount = (int)min((long long)K1_TILE, n - tbase);
  const bool full = tcount == K1_TILE;
  // speculative soup staging is in range only if the tile's vertex rows exist
  const bool spec_v = bulk_ok && full && 3 * (tbase + K1_TILE) <= nv;
  // T == nullptr: an implicit soup (the host found T[i][k] == 3i + k and did not copy it)
  if (bulk_ok && full) {
    if (tid == 0) {
      mbar_init(&sm.bar, 1);
      const unsigned tb = T ? K1_TILE * 3 * sizeof(int) : 0u, vb = spec_v ? K1_TILE * 9 * sizeof(double) : 0u;
      mbar_expect_tx(&sm.bar, tb + vb);
      if (T) bulk_g2s(sm.t, T + 3 * tbase, tb, &sm.bar);
      if (spec_v) bulk_g2s(sm.v, V + 9 * tbase, vb, &sm.bar);
    }
    if (!T)
      for (int q = tid; q < 3 * tcount; q += K1_THREADS) sm.t[q] = (int)(3 * tbase + q);
    __syncthreads();  // barrier initialised before anyone waits on it
    mbar_wait(&sm.bar, 0);
  } else {
    for (int q = tid; q < 3 * tcount; q += K1_THREADS) sm.t[q] = T ? __ldg(T + 3 * tbase + q) : (int)(3 * tbase + q);
    __syncthreads();
  }
  // soup test over the whole tile (index 3*i+k == 3*(tbase+i)+k) and index validation
  // (geometry.py:41-43: every index in [0, nv), else InvariantError)
  bool mine = true, inrange = true;
  for (int q = tid; q < 3 * tcount; q += K1_THREADS) {
    const int v = sm.t[q];
    mine &= v == (int)(3 * tbase + q);
    inrange &= v >= 0 && (long long)v < nv;
  }
  const bool soup = __syncthreads_and(mine) && spec_v;
  if (!__syncthreads_and(inrange)) {
    if (tid == 0) {
      atomicOr(err, 2u);
      tile_sum[tile] = 0;
    }
    // never gather through an out-of-range index; the tile contributes no pairs, so steps
    // that run on the device count before the host sees the error (PG_DEFER, the graph
    // build) stay in bounds
    for (int i = tid; i < tcount; i += K1_THREADS) rec[tbase + i] = make_uint4(0u, 1u, 1u, 0u);
    return;
  }

  const unsigned dx = (unsigned)s.dims[0], dxy = (unsigned)s.dims[0] * (unsigned)s.dims[1];
  uint3 box[K1_ROUNDS];
  unsigned cnt[K1_ROUNDS];
  bool bad = false;
#pragma unroll
  for (int r = 0; r < K1_ROUNDS; ++r) {
    const int i = r * K1_THREADS + tid;  // striped: coalesced record stores
    box[r] = make_uint3(0u, 1u, 1u);
    cnt[r] = 0;
    if (i < tcount) {
      if (soup) {
        const double* p = sm.v + 9 * i;
        tri_box(p, p + 3, p + 6, s, dx, dxy, box[r], cnt[r], bad);
      } else {
        tri_box(V + 3 * (long long)sm.t[3 * i], V + 3 * (long long)sm.t[3 * i + 1], V + 3 * (long long)sm.t[3 * i + 2],
                s, dx, dxy, box[r], cnt[r], bad);
      }
    }
  }
  if (bad) atomicOr(err, 1u);
  // block-wide exclusive scan in triangle order (round-major, then thread)
  __shared__ unsigned long long rtot[K1_ROUNDS * (K1_THREADS / 32)];
  unsigned long long incl[K1_ROUNDS];
#pragma unroll
  for (int r = 0; r < K1_ROUNDS; ++r) {
    unsigned long long v = cnt[r];
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const unsigned long long o = __shfl_up_sync(0xffffffffu, v, d);
      if (lane >= d) v += o;
    }
    incl[r] = v;
    if (lane == 31) rtot[r * (K1_THREADS / 32) + warp] = v;
  }
  __syncthreads();
  if (warp == 0) {
    constexpr int NE = K1_ROUNDS * (K1_THREADS / 32);
    const unsigned long long e = lane < NE ? rtot[lane] : 0ull;
    unsigned long long ei = e;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const unsigned long long o = __shfl_up_sync(0xffffffffu, ei, d);
      if (lane >= d) ei += o;
    }
    if (lane < NE) rtot[lane] = ei - e;
    if (lane == NE - 1) tile_sum[tile] = ei;
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < K1_ROUNDS; ++r) {
    const int i = r * K1_THREADS + tid;
    if (i < tcount) {
      const unsigned long long off = rtot[r * (K1_THREADS / 32) + warp] + incl[r] - cnt[r];
      rec[tbase + i] = make_uint4(box[r].x, box[r].y, box[r].z, (unsigned)off);
    }
  }
}

// K1b: exclusive scan of the per-tile pair counts (one CTA) -> tile_pre (u32; only used once
// NO <= 2^30 is established) and the total NO (u64, exact).
constexpr int TS_THREADS = 1024;
constexpr int TS_WARPS = TS_THREADS / 32;
constexpr int TS_REG = 20;  // chunks of 32 held in registers per lane (single-pass case)
__global__ void __launch_bounds__(TS_THREADS)
k_scan_tile_sums(const unsigned long long* __restrict__ tile_sum, unsigned ntiles, unsigned* __restrict__ tile_pre,
                 unsigned long long* __restrict__ total) {
  PDL_ENTRY();
  __shared__ unsigned long long wsum[TS_WARPS];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // warp w owns the contiguous segment [w*seg, (w+1)*seg), read in coalesced 32-wide chunks
  const unsigned seg = ((ntiles + TS_WARPS - 1) / TS_WARPS + 31) & ~31u;
  const unsigned s0 = min((unsigned)warp * seg, ntiles), s1 = min(s0 + seg, ntiles);
  if (seg <= 32u * TS_REG) {
    // single pass: every chunk of the segment is loaded at once and kept in registers
    unsigned long long v[TS_REG];
    unsigned long long part = 0;
#pragma unroll
    for (int j = 0; j < TS_REG; ++j) {
      const unsigned i = s0 + 32 * j + lane;
      v[j] = i < s1 ? tile_sum[i] : 0ull;
      part += v[j];
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) part += __shfl_xor_sync(0xffffffffu, part, d);
    if (lane == 0) wsum[warp] = part;
    __syncthreads();
    unsigned long long carry = 0, tot = 0;
    for (int w = 0; w < TS_WARPS; ++w) {
      const unsigned long long x = wsum[w];
      carry += w < warp ? x : 0ull;
      tot += x;
    }
#pragma unroll
    for (int j = 0; j < TS_REG; ++j) {
      const unsigned i = s0 + 32 * j + lane;
      unsigned long long inc = v[j];
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const unsigned long long o = __shfl_up_sync(0xffffffffu, inc, d);
        if (lane >= d) inc += o;
      }
      if (i < s1) tile_pre[i] = (unsigned)(carry + inc - v[j]);
      carry += __shfl_sync(0xffffffffu, inc, 31);
    }
    if (tid == 0) *total = tot;
    return;
  }
  // large inputs: two passes over the segment, loads batched 8 chunks deep
  constexpr int B = 8;
  unsigned long long part = 0;
  for (unsigned c = s0; c < s1; c += 32 * B) {
    unsigned long long v[B];
#pragma unroll
    for (int j = 0; j < B; ++j) {
      const unsigned i = c + 32 * j + lane;
      v[j] = i < s1 ? tile_sum[i] : 0ull;
    }
#pragma unroll
    for (int j = 0; j < B; ++j) part += v[j];
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) part += __shfl_xor_sync(0xffffffffu, part, d);
  if (lane == 0) wsum[warp] = part;
  __syncthreads();
  unsigned long long carry = 0, tot = 0;
  for (int w = 0; w < TS_WARPS; ++w) {
    carry += w < warp ? wsum[w] : 0ull;
    tot += wsum[w];
  }
  for (unsigned c = s0; c < s1; c += 32 * B) {
    unsigned long long v[B];
#pragma unroll
    for (int j = 0; j < B; ++j) {
      const unsigned i = c + 32 * j + lane;
      v[j] = i < s1 ? tile_sum[i] : 0ull;
    }
#pragma unroll
    for (int j = 0; j < B; ++j) {
      const unsigned i = c + 32 * j + lane;
      unsigned long long inc = v[j];
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const unsigned long long o = __shfl_up_sync(0xffffffffu, inc, d);
        if (lane >= d) inc += o;
      }
      if (i < s1) tile_pre[i] = (unsigned)(carry + inc - v[j]);
      carry += __shfl_sync(0xffffffffu, inc, 31);
    }
  }
  if (tid == 0) *total = tot;
}


// ----------------------------------------------------------------------------------------
// K2: load-balanced pair expansion + radix digit histograms
// ----------------------------------------------------------------------------------------
constexpr int K2_THREADS = 256;
constexpr int K2_ITEMS = 8;
constexpr int K2_TILE = K2_THREADS * K2_ITEMS;
constexpr int kMaxDigitBits = 9;
constexpr int kMaxBins = 1 << kMaxDigitBits;  // 512

// Object cache for one expansion tile: box records of the tile's triangles olo, olo+1, ...
// (structure of arrays in shared memory); triangles past OC_CAP are read from global.
#ifndef OC_CAP_OVERRIDE
constexpr int OC_CAP = 2560;
#else
constexpr int OC_CAP = OC_CAP_OVERRIDE;
#endif  // (3*OC_CAP words also host K2's <= 4096-bin coarse histogram)
struct ObjCache {
  unsigned lo_cell[OC_CAP];
  unsigned mx[OC_CAP];
  unsigned my[OC_CAP];
};

// Pair expansion of one tile [p0, p0 + THREADS*ITEMS): thread t produces the cell ids
// (key) and owning triangle ids (own) of its ITEMS consecutive pairs p0 + t*ITEMS + j.
// The owner of every pair is recovered the way Alg. 1 does it (marks at run starts +
// inclusive max-scan), but tile-locally: the tile's first owner comes from
// a 32-ary search over the record offsets, the run starts inside the tile are scattered into
// shared memory (their box records cached alongside), and a block max-scan fills the gaps.
// Inside a thread's consecutive pairs the cell coordinate is stepped incrementally
// (x-fastest); a new run always starts at relative offset 0, so the two divisions of
// _make_cell_ids (builders.py:111-113) only ever run for a thread's first pair.
// Owners and cell ids of a tile's pairs once its run starts are in the slots (expand_tile):
// inclusive max-scan of the slots, then each thread steps its ITEMS consecutive pairs. `box`
// returns an object's {lo_cell, mx, my}.
template <int THREADS, int ITEMS, typename Box>
__device__ __forceinline__ void expand_runs(int* slot, int* warpmax, long long olo, unsigned p0, unsigned pend,
                                            unsigned dx, unsigned dxy, Box box, unsigned (&key)[ITEMS],
                                            int (&own)[ITEMS]) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  auto slot_at = [](unsigned e) { return ((((e >> 2) ^ ((e >> 5) & 7u)) << 2) | (e & 3u)); };
  (void)olo;
  // inclusive max-scan over the slots (blocked: thread t owns slots [ITEMS*t, ITEMS*t + ITEMS))
#pragma unroll
  for (int q = 0; q < ITEMS / 4; ++q) {
    const int4 a = *reinterpret_cast<const int4*>(&slot[slot_at((unsigned)(tid * ITEMS + 4 * q))]);
    own[4 * q] = a.x;
    own[4 * q + 1] = a.y;
    own[4 * q + 2] = a.z;
    own[4 * q + 3] = a.w;
  }
  // alongside the owners, the tile position of the latest run start (a marked slot past
  // position 0, which holds the tile's first owner whatever its start): a thread's first pair
  // then knows its offset in its run without reading the owner's record back
  constexpr int NW = THREADS / 32;
  int prun = -1;
#pragma unroll
  for (int j = 0; j < ITEMS; ++j)
    if (own[j] != -1 && tid * ITEMS + j > 0) prun = tid * ITEMS + j;
  const bool first_starts = tid > 0 && own[0] != -1;
#pragma unroll
  for (int j = 1; j < ITEMS; ++j) own[j] = max(own[j], own[j - 1]);
  int run = own[ITEMS - 1];
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int o = __shfl_up_sync(0xffffffffu, run, d);
    const int po = __shfl_up_sync(0xffffffffu, prun, d);
    if (lane >= d) {
      run = max(run, o);
      prun = max(prun, po);
    }
  }
  if (lane == 31) {
    warpmax[warp] = run;
    warpmax[NW + warp] = prun;
  }
  __syncthreads();
  int carry = __shfl_up_sync(0xffffffffu, run, 1);
  int pcarry = __shfl_up_sync(0xffffffffu, prun, 1);
  if (lane == 0) carry = pcarry = -1;
  for (int w = 0; w < warp; ++w) {
    carry = max(carry, warpmax[w]);
    pcarry = max(pcarry, warpmax[NW + w]);
  }
#pragma unroll
  for (int j = 0; j < ITEMS; ++j) own[j] = max(own[j], carry);
  const int start0 = first_starts ? tid * ITEMS : pcarry;  // tile position of own[0]'s run, or -1

  const unsigned pbase = p0 + (unsigned)tid * ITEMS;
  unsigned cell = 0, x = 0, y = 0, mx = 1, my = 1;
  if (pbase < pend) {  // first pair: may sit anywhere inside its run
    const unsigned rel = start0 >= 0 ? (unsigned)(tid * ITEMS - start0) : pbase - (unsigned)warpmax[2 * NW];
    unsigned lc;
    box(own[0], lc, mx, my);
    if (rel == 0) {
      cell = lc;
    } else {
      const unsigned mxy = mx * my;
      const unsigned z = rel / mxy;
      const unsigned rem = rel - z * mxy;
      y = rem / mx;
      x = rem - y * mx;
      cell = lc + x + dx * y + dxy * z;
    }
  }
  key[0] = cell;
#pragma unroll
  for (int j = 1; j < ITEMS; ++j) {
    if (own[j] != own[j - 1]) {  // a new run starts at its relative offset 0
      box(own[j], cell, mx, my);
      x = 0;
      y = 0;
    } else {
      ++x;
      ++cell;
      if (x == mx) {
        x = 0;
        cell += dx - mx;
        if (++y == my) {
          y = 0;
          cell += dxy - dx * my;
        }
      }
    }
    key[j] = cell;
  }
}


template <int THREADS, int ITEMS>
__device__ __forceinline__ void expand_tile(const uint4* __restrict__ rec, long long n, unsigned p0, unsigned pend,
                                            unsigned dx, unsigned dxy, const unsigned* __restrict__ tile_pre,
                                            const int2* __restrict__ bounds, int* slot, int* warpmax, void* cache,
                                            unsigned (&key)[ITEMS], int (&own)[ITEMS]) {
  constexpr int TILE = THREADS * ITEMS;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // [olo, oend): owner of pair p0, and one past the last triangle whose run starts in the tile
  // (k_pair_tile_bounds precomputed both with 32-ary searches over the offsets)
  const int2 bnd = __ldg(&bounds[p0 / TILE]);
  const long long olo = bnd.x, oend = bnd.y;
  // slots live in 16-byte chunks whose index is XOR-swizzled (slot_at) so the per-thread
  // chunk reads of the max-scan below are bank-conflict free
  auto slot_at = [](unsigned e) { return ((((e >> 2) ^ ((e >> 5) & 7u)) << 2) | (e & 3u)); };
  ObjCache* oc = static_cast<ObjCache*>(cache);
  // the first EXP_PRE records of this thread are requested before the slot initialisation and
  // its barrier, which then hide their DRAM latency (the stall that dominated this phase)
  constexpr int EXP_PRE = 4;
  uint4 pr[EXP_PRE];
  unsigned pt[EXP_PRE];
#pragma unroll
  for (int u = 0; u < EXP_PRE; ++u) {
    const long long o = olo + 1 + tid + (long long)u * THREADS;
    if (o < oend) {
      pr[u] = __ldg(&rec[o]);
      pt[u] = __ldg(&tile_pre[o / K1_TILE]);
    }
  }
#ifndef PGRID_K2_PREF
#define PGRID_K2_PREF 1
#endif
  if (PGRID_K2_PREF) {  // the later records towards L2 now (no registers held), loaded below
    for (long long o = olo + 1 + tid + (long long)EXP_PRE * THREADS; o < oend; o += THREADS)
      asm volatile("prefetch.global.L2 [%0];" ::"l"(rec + o));
  }
  uint4 r0 = make_uint4(0u, 0u, 0u, 0u);
  if (tid == 0) r0 = __ldg(&rec[olo]);
  for (int i = tid; i < TILE; i += THREADS) slot[i] = -1;
  __syncthreads();
  if (tid == 0) {
    slot[0] = (int)olo;  // slot_at(0) == 0
    oc->lo_cell[0] = r0.x;
    oc->mx[0] = r0.y;
    oc->my[0] = r0.z;
    warpmax[2 * (THREADS / 32)] = (int)(__ldg(&tile_pre[olo / K1_TILE]) + r0.w);  // olo's absolute offset
  }
  auto start = [&](long long o, const uint4& r, unsigned tp) {
    PG_ASSERT(tp + r.w >= p0 && tp + r.w - p0 < (unsigned)TILE);
    atomicMax(&slot[slot_at(tp + r.w - p0)], (int)o);  // zero-count triangles share the next start; max wins
    const long long ci = o - olo;
    if (ci < OC_CAP) {
      oc->lo_cell[ci] = r.x;
      oc->mx[ci] = r.y;
      oc->my[ci] = r.z;
    }
  };
#pragma unroll
  for (int u = 0; u < EXP_PRE; ++u) {
    const long long o = olo + 1 + tid + (long long)u * THREADS;
    if (o < oend) start(o, pr[u], pt[u]);
  }
  // the remaining run starts inside the tile (independent loads, no barrier per chunk)
#pragma unroll 4
  for (long long o = olo + 1 + tid + (long long)EXP_PRE * THREADS; o < oend; o += THREADS)
    start(o, __ldg(&rec[o]), __ldg(&tile_pre[o / K1_TILE]));
  __syncthreads();
  expand_runs<THREADS, ITEMS>(slot, warpmax, olo, p0, pend, dx, dxy,
                              [&](int o, unsigned& lc, unsigned& bx, unsigned& by) {
                                const long long ci = (long long)o - olo;
                                if (ci < OC_CAP) {
                                  lc = oc->lo_cell[ci];
                                  bx = oc->mx[ci];
                                  by = oc->my[ci];
                                } else {
                                  const uint4 r = __ldg(&rec[o]);
                                  lc = r.x;
                                  bx = r.y;
                                  by = r.z;
                                }
                              },
                              key, own);
}

// record= stage 0: records with absolute pair offsets
__global__ void k_abs_offsets(const uint4* __restrict__ rec, const unsigned* __restrict__ tile_pre, long long n,
                              uint4* __restrict__ out) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    uint4 r = rec[i];
    r.w += tile_pre[i / K1_TILE];
    out[i] = r;
  }
}

// Tile bounds of the pair expansion, one warp per tile: x = owner of the tile's first pair
// ((#triangles with offset <= p0) - 1), y = one past the last triangle whose run starts
// inside the tile (#triangles with offset < pend). Hoisting these searches out of the
// expansion kernels keeps their CTAs from idling on dependent round trips at launch.
// Two warp-cooperative 32-ary lower_bounds run in lockstep (their loads overlap): smallest
// i in [lo, hi] with load(i) >= x, for (lo0, hi0, x0) and (lo1, hi1, x1).
template <typename Load>
__device__ __forceinline__ void warp_lower_bound2(unsigned long long& lo0, unsigned long long hi0,
                                                  unsigned long long x0, unsigned long long& lo1,
                                                  unsigned long long hi1, unsigned long long x1, Load load) {
  const int lane = threadIdx.x & 31;
  while (lo0 < hi0 || lo1 < hi1) {
    const unsigned long long st0 = (hi0 - lo0 + 31) / 32, st1 = (hi1 - lo1 + 31) / 32;
    const unsigned long long p0 = lo0 + (unsigned long long)lane * st0, p1 = lo1 + (unsigned long long)lane * st1;
    const bool a0 = lo0 < hi0 && p0 < hi0, a1 = lo1 < hi1 && p1 < hi1;
    const unsigned long long v0 = a0 ? load(p0) : 0ull, v1 = a1 ? load(p1) : 0ull;
    const unsigned b0 = __ballot_sync(0xffffffffu, a0 ? v0 >= x0 : true);
    const unsigned b1 = __ballot_sync(0xffffffffu, a1 ? v1 >= x1 : true);
    if (lo0 < hi0) {
      const int f = b0 ? __ffs(b0) - 1 : 32;
      if (f == 0) {
        hi0 = lo0;
      } else {
        lo0 = lo0 + (unsigned long long)(f - 1) * st0 + 1;
        if (f < 32) hi0 = min(hi0, (lo0 - 1) + st0);
      }
    }
    if (lo1 < hi1) {
      const int f = b1 ? __ffs(b1) - 1 : 32;
      if (f == 0) {
        hi1 = lo1;
      } else {
        lo1 = lo1 + (unsigned long long)(f - 1) * st1 + 1;
        if (f < 32) hi1 = min(hi1, (lo1 - 1) + st1);
      }
    }
  }
}

// K2 tile bounds: for pair tile t, a = the object whose pairs contain p0 (last object with
// offset <= p0) and b = the first object starting at or after the tile end. Two levels:
// the K1 tile prefixes (tile_pre, L2-resident) locate the 512-object K1 tile, then the
// objects' offsets inside it; both queries of a tile run in lockstep.
__global__ void __launch_bounds__(256)
k_pair_tile_bounds(const uint4* __restrict__ rec, const unsigned* __restrict__ tile_pre, long long n, Count cno,
                   unsigned tile, int2* __restrict__ bounds, unsigned* __restrict__ zero = nullptr,
                   unsigned nzero = 0) {
  PDL_ENTRY();
  // optional: clear the radix digit totals here (the row scans that fill them run later),
  // so no memset node breaks the launch chain
  if (zero)
    for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < nzero; i += gridDim.x * blockDim.x) zero[i] = 0;
  const unsigned no = cno.get();
  const unsigned ntiles = (no + tile - 1) / tile;
  const unsigned t = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (t >= ntiles) return;
  const unsigned p0 = t * tile;
  const unsigned pend = min(p0 + tile, no);
  const unsigned long long nk1 = (unsigned long long)((n + K1_TILE - 1) / K1_TILE);
  // level 1: J = first K1 tile whose first object's offset >= x; the answer is in
  // ((J-1)*K1_TILE, J*K1_TILE] (clipped to [0, n])
  unsigned long long j0 = 0, j1 = 0;
  warp_lower_bound2(j0, nk1, (unsigned long long)p0 + 1, j1, nk1, (unsigned long long)pend,
                    [&](unsigned long long j) { return (unsigned long long)__ldg(&tile_pre[j]); });
  auto range_lo = [&](unsigned long long J) { return J ? (J - 1) * K1_TILE + 1 : 0ull; };
  auto range_hi = [&](unsigned long long J) { return min(J * (unsigned long long)K1_TILE, (unsigned long long)n); };
  unsigned long long a = range_lo(j0), b = range_lo(j1);
  warp_lower_bound2(a, range_hi(j0), (unsigned long long)p0 + 1, b, range_hi(j1), (unsigned long long)pend,
                    [&](unsigned long long i) { return (unsigned long long)tri_offset(rec, tile_pre, i); });
  if ((threadIdx.x & 31) == 0) bounds[t] = make_int2((int)a - 1, (int)b);
}

// lower_bound(sorted, t * step) for t in [0, nq), one warp per query (K4's key ranges). With
// top_hist (the last radix pass's digit totals), each query is first narrowed to its top
// digit's run [start(d), start(d+1)] -- the run starts are a prefix of top_hist -- so the
// 32-ary search covers ~NO/2^bits keys instead of NO.
__global__ void __launch_bounds__(256)
k_key_tile_bounds(const unsigned* __restrict__ sorted, Count cno, unsigned step, unsigned ncells, unsigned nq,
                  unsigned* __restrict__ out, const unsigned* __restrict__ top_hist = nullptr, int top_shift = 0,
                  int top_bins = 0) {
  PDL_ENTRY();
  __shared__ unsigned start[kMaxBins + 1];
  const unsigned no = cno.get();
  if (top_hist) {
    if (threadIdx.x < 32) {  // exclusive prefix of the (<= 512) digit totals, 16 per lane
      const int lane = threadIdx.x;
      unsigned v[16], run = 0;
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const int d = lane * 16 + q;
        v[q] = run;
        run += d < top_bins ? __ldg(&top_hist[d]) : 0u;
      }
      unsigned inc = run;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const unsigned o = __shfl_up_sync(0xffffffffu, inc, d);
        if (lane >= d) inc += o;
      }
#pragma unroll
      for (int q = 0; q < 16; ++q) start[lane * 16 + q] = inc - run + v[q];
      if (lane == 31) start[kMaxBins] = inc;
    }
    __syncthreads();
  }
  const unsigned t = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (t >= nq) return;
  const unsigned long long c = min((unsigned long long)t * step, (unsigned long long)ncells);
  unsigned long long lo = 0, hi = no;
  if (top_hist) {
    const unsigned d = (unsigned)(c >> top_shift);
    if ((int)d < top_bins) {
      lo = start[d];
      hi = d + 1 < (unsigned)top_bins ? start[d + 1] : no;
    } else {
      lo = hi = no;
    }
  }
  unsigned long long dummy_lo = hi, dummy_hi = hi;
  warp_lower_bound2(lo, hi, c, dummy_lo, dummy_hi, 0ull,
                    [&](unsigned long long i) { return (unsigned long long)__ldg(sorted + i); });
  if ((threadIdx.x & 31) == 0) out[t] = (unsigned)lo;
}

// Pairs in generation (object-major) order -- used when no radix pass follows
// (ncells == 1) and for the record= stage dumps.
__global__ void __launch_bounds__(K2_THREADS)
k_expand_pairs(const uint4* __restrict__ rec, const unsigned* __restrict__ tile_pre, long long n, Count cno,
               unsigned dx, unsigned dxy, const int2* __restrict__ bounds, unsigned* __restrict__ keys,
               unsigned* __restrict__ vals, unsigned val_offset, unsigned* __restrict__ coarse, int coarse_shift,
               int coarse_bins) {
  __shared__ __align__(16) int slot[K2_TILE];
  __shared__ int warpmax[2 * (K2_THREADS / 32) + 1];
  __shared__ ObjCache oc;
  const unsigned no = cno.get();
  const unsigned p0 = blockIdx.x * (unsigned)K2_TILE;
  if (p0 >= no) return;
  const unsigned pend = min(p0 + (unsigned)K2_TILE, no);
  unsigned key[K2_ITEMS];
  int own[K2_ITEMS];
  expand_tile<K2_THREADS, K2_ITEMS>(rec, n, p0, pend, dx, dxy, tile_pre, bounds, slot, warpmax, &oc, key, own);
  const unsigned pbase = p0 + threadIdx.x * K2_ITEMS;
  if (coarse) {  // coarse cell-bucket histogram for slab planning (sharded builds)
    unsigned* hc = reinterpret_cast<unsigned*>(oc.lo_cell);  // object cache is dead now
    __syncthreads();
    for (int b = threadIdx.x; b < coarse_bins; b += K2_THREADS) hc[b] = 0u;
    __syncthreads();
    unsigned cur = 0xffffffffu, cnt = 0;
#pragma unroll
    for (int j = 0; j < K2_ITEMS; ++j)
      if (pbase + j < pend) {
        const unsigned b = key[j] >> coarse_shift;
        if (b != cur) {
          if (cnt) atomicAdd(&hc[cur], cnt);
          cur = b;
          cnt = 0;
        }
        ++cnt;
      }
    if (cnt) atomicAdd(&hc[cur], cnt);
    __syncthreads();
    for (int b = threadIdx.x; b < coarse_bins; b += K2_THREADS)
      if (hc[b]) atomicAdd(&coarse[b], hc[b]);
  }
  if (pbase + K2_ITEMS <= pend) {
    uint4* kd = reinterpret_cast<uint4*>(keys + pbase);
    uint4* vd = reinterpret_cast<uint4*>(vals + pbase);
    kd[0] = make_uint4(key[0], key[1], key[2], key[3]);
    kd[1] = make_uint4(key[4], key[5], key[6], key[7]);
    vd[0] = make_uint4(own[0] + val_offset, own[1] + val_offset, own[2] + val_offset, own[3] + val_offset);
    vd[1] = make_uint4(own[4] + val_offset, own[5] + val_offset, own[6] + val_offset, own[7] + val_offset);
  } else {
#pragma unroll
    for (int j = 0; j < K2_ITEMS; ++j)
      if (pbase + j < pend) {
        keys[pbase + j] = key[j];
        vals[pbase + j] = (unsigned)own[j] + val_offset;
      }
  }
}

// ----------------------------------------------------------------------------------------
// K3: stable LSD radix pass, reduce-then-scan:
//   k_tile_counts       per-tile digit counts          counts[digit][tile]
//   k_scan_tile_counts  exclusive scan of every digit row over the tiles
//   k_radix_scatter     rank the tile stably in shared memory, scatter to
//                       dstart[digit] + offs[digit][tile] + local rank
// (A single-kernel onesweep with decoupled look-back was measured first: its per-digit
//  look-back chains serialised at ~20% of HBM bandwidth on B200.)
// ----------------------------------------------------------------------------------------
#ifndef RS_THREADS_OVERRIDE
constexpr int RS_THREADS = 256;
#else
constexpr int RS_THREADS = RS_THREADS_OVERRIDE;
#endif
constexpr int RS_WARPS = RS_THREADS / 32;
#ifndef RS_ITEMS_OVERRIDE
constexpr int RS_ITEMS = 16;
#else
constexpr int RS_ITEMS = RS_ITEMS_OVERRIDE;
#endif
constexpr int RS_TILE = RS_THREADS * RS_ITEMS;  // 4096 pairs per tile
constexpr int RS_DPT = 2;  // digits per thread in the per-digit phases (threads >= kMaxBins / 2 take none)
static_assert(RS_THREADS * RS_DPT >= kMaxBins, "the per-digit phases need kMaxBins / 2 threads");
#ifndef RS_MIN_CTAS_OVERRIDE
constexpr int RS_MIN_CTAS = 4;
#else
constexpr int RS_MIN_CTAS = RS_MIN_CTAS_OVERRIDE;
#endif  // 64 registers, 45 KB smem: 4 CTAs (32 warps) per SM

struct RsSmem {
  unsigned buf[RS_TILE];     // tile in digit order: keys, then values
  unsigned vstage[RS_TILE];  // values in input order (cp.async staging)
  unsigned short whist[RS_WARPS][kMaxBins];  // per-warp digit counts -> tile offset of (warp, digit)
  unsigned gbase[kMaxBins];                  // global position of buf[0] for each digit
  unsigned hsm[kMaxBins];                    // digit totals (staged)
  unsigned wsum[RS_WARPS];
};

__device__ __forceinline__ void cp_async4(void* smem, const void* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((unsigned)__cvta_generic_to_shared(smem)), "l"(g)
               : "memory");
}
__device__ __forceinline__ void cp_async16(void* smem, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((unsigned)__cvta_generic_to_shared(smem)), "l"(g)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all_but_one() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

// One bit-slice of warp peer detection: keep the lanes whose bit (x & bit) equals ours.
// Written in PTX so ptxas emits LOP3.P (bit -> predicate), VOTE, SEL, LOP3 -- 4 instructions
// per bit and item; the C form compiled to ~7 (the bit extracted twice, once per use).
__device__ __forceinline__ unsigned peers_step(unsigned pm, unsigned x, unsigned bit) {
  unsigned r;
  asm("{\n\t.reg .pred p;\n\t.reg .b32 t, bb, m;\n\t"
      "and.b32 t, %1, %2;\n\tsetp.ne.u32 p, t, 0;\n\t"
      "vote.sync.ballot.b32 bb, p, 0xffffffff;\n\t"
      "selp.b32 m, 0, 0xffffffff, p;\n\t"
      "xor.b32 bb, bb, m;\n\tand.b32 %0, %3, bb;\n\t}"
      : "=r"(r)
      : "r"(x), "r"(bit), "r"(pm));
  return r;
}

// Block-wide exclusive scan of one value per thread (NW warps); also returns the total.
template <int NW>
__device__ __forceinline__ unsigned block_excl_scan(unsigned v, unsigned* wsum, unsigned& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned inc = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const unsigned o = __shfl_up_sync(0xffffffffu, inc, d);
    if (lane >= d) inc += o;
  }
  if (lane == 31) wsum[warp] = inc;
  __syncthreads();
  unsigned add = 0, tot = 0;
#pragma unroll
  for (int w = 0; w < NW; ++w) {
    const unsigned x = wsum[w];
    add += w < warp ? x : 0u;
    tot += x;
  }
  total = tot;
  __syncthreads();  // wsum may be reused by the caller's next scan
  return add + inc - v;
}

// Digit of a key: a bit field, or (slab partitioning) a table lookup of a coarse bucket.
struct DigitFn {
  int shift;
  unsigned mask;
  const unsigned* __restrict__ table;  // non-null: digit = table[key >> shift]
  __device__ __forceinline__ unsigned operator()(unsigned k) const {
    return table ? __ldg(&table[k >> shift]) : (k >> shift) & mask;
  }
};

// Upsweep of a radix pass: per-tile digit counts, TC_TILES tiles per CTA (each digit row of
// the digit-major matrix receives TC_TILES consecutive entries).
#ifndef TC_TILES_OVERRIDE
constexpr int TC_TILES = 2;  // 2 tiles per CTA: 48 registers (4: 78, 1: 32); measured best (r2_ab_upsweep_tiles)
#else
constexpr int TC_TILES = TC_TILES_OVERRIDE;
#endif
__global__ void __launch_bounds__(RS_THREADS)
k_tile_counts(const unsigned* __restrict__ keys, Count cno, DigitFn dig, int nbins, unsigned* __restrict__ counts,
              unsigned ld, unsigned* __restrict__ packed = nullptr) {
  PDL_ENTRY();
  __shared__ unsigned h[TC_TILES][kMaxBins];
  const unsigned no = cno.get();
  const int tid = threadIdx.x;
  const unsigned ntiles = (no + RS_TILE - 1) / RS_TILE;
  const unsigned t0 = blockIdx.x * TC_TILES;
  for (int b = tid; b < TC_TILES * kMaxBins; b += RS_THREADS) (&h[0][0])[b] = 0u;
  __syncthreads();
  // all of the CTA's (full) tiles are loaded before any histogram atomic: TC_TILES x 16 KB in
  // flight per CTA, enough to cover HBM latency at the kernel's occupancy
  constexpr int R = RS_TILE / 4 / RS_THREADS;
  uint4 k[TC_TILES][R];
  auto full = [&](unsigned tile) { return tile < ntiles && (tile + 1) * (unsigned)RS_TILE <= no; };
#pragma unroll
  for (int q = 0; q < TC_TILES; ++q) {
    if (full(t0 + q)) {
      const uint4* src = reinterpret_cast<const uint4*>(keys + (t0 + q) * (unsigned)RS_TILE);
#pragma unroll
      for (int r = 0; r < R; ++r) k[q][r] = __ldcs(src + tid + r * RS_THREADS);
    }
  }
#pragma unroll
  for (int q = 0; q < TC_TILES; ++q) {
    const unsigned tile = t0 + q;
    if (tile >= ntiles) break;
    if (full(tile)) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        atomicAdd(&h[q][dig(k[q][r].x)], 1u);
        atomicAdd(&h[q][dig(k[q][r].y)], 1u);
        atomicAdd(&h[q][dig(k[q][r].z)], 1u);
        atomicAdd(&h[q][dig(k[q][r].w)], 1u);
      }
    } else {
      const unsigned tbase = tile * (unsigned)RS_TILE;
      const unsigned tvalid = min((unsigned)RS_TILE, no - tbase);
      for (unsigned e = tid; e < tvalid; e += RS_THREADS) atomicAdd(&h[q][dig(__ldcs(keys + tbase + e))], 1u);
    }
  }
  __syncthreads();
  if (packed) {  // two digits per word, as K2 writes pass 0 (k_scan_tile_counts_packed unpacks)
    for (int i = tid; i < (nbins / 2) * TC_TILES; i += RS_THREADS) {
      const int b = i / TC_TILES, q = i % TC_TILES;
      if (t0 + q < ntiles) packed[(size_t)b * ld + t0 + q] = h[q][2 * b] | (h[q][2 * b + 1] << 16);
    }
  } else {
    for (int i = tid; i < nbins * TC_TILES; i += RS_THREADS) {
      const int b = i / TC_TILES, q = i % TC_TILES;
      if (t0 + q < ntiles) {
        PG_ASSERT(t0 + q < ld);
        counts[(size_t)b * ld + t0 + q] = h[q][b];
      }
    }
  }
}

constexpr int SC_THREADS = 256;
constexpr int SC_VEC = 5;                  // 16-byte vectors per thread per chunk
constexpr int SC_ITEMS = 4 * SC_VEC;       // 20 tiles per thread, 5120 per chunk (21M pairs)
// One CTA per digit row: counts[row][0..ntiles) -> exclusive prefix over tiles, in place.
// Rows are padded to a multiple of 4 (ld) so each thread moves its entries as 16-byte
// accesses, all issued before the scan (one memory latency per chunk); 512 rows x 256
// threads fit one wave. The row total is the digit's global count (its histogram bin).
__global__ void __launch_bounds__(SC_THREADS)
k_scan_tile_counts(unsigned* __restrict__ counts, Count cno, unsigned ld, unsigned* __restrict__ row_total) {
  PDL_ENTRY();
  __shared__ unsigned wsum[SC_THREADS / 32];
  const unsigned ntiles = (cno.get() + RS_TILE - 1) / RS_TILE;
  const int tid = threadIdx.x;
  unsigned* row = counts + (size_t)blockIdx.x * ld;
  unsigned carry = 0;
  for (unsigned base = 0; base < ntiles; base += SC_THREADS * SC_ITEMS) {
    const unsigned i0 = base + tid * SC_ITEMS;
    uint4 v[SC_VEC];
#pragma unroll
    for (int q = 0; q < SC_VEC; ++q) {
      const unsigned i = i0 + 4 * q;
      v[q] = i < ntiles ? *reinterpret_cast<const uint4*>(row + i) : make_uint4(0u, 0u, 0u, 0u);
    }
    unsigned run = 0;
#pragma unroll
    for (int q = 0; q < SC_VEC; ++q) {
      const unsigned i = i0 + 4 * q;
      // padding columns (>= ntiles) hold garbage
      const unsigned a = i < ntiles ? v[q].x : 0u, b = i + 1 < ntiles ? v[q].y : 0u;
      const unsigned c = i + 2 < ntiles ? v[q].z : 0u, d = i + 3 < ntiles ? v[q].w : 0u;
      v[q] = make_uint4(run, run + a, run + a + b, run + a + b + c);
      run += a + b + c + d;
    }
    unsigned total;
    const unsigned pre = carry + block_excl_scan<SC_THREADS / 32>(run, wsum, total);
#pragma unroll
    for (int q = 0; q < SC_VEC; ++q) {
      const unsigned i = i0 + 4 * q;
      if (i < ntiles)  // the vector never crosses ld (a multiple of 4)
        *reinterpret_cast<uint4*>(row + i) = make_uint4(pre + v[q].x, pre + v[q].y, pre + v[q].z, pre + v[q].w);
    }
    carry += total;
  }
  if (tid == 0) row_total[blockIdx.x] = carry;
}

// k_scan_tile_counts for K2's packed first-pass counts: CTA b scans packed row b (digits 2b in
// the low and 2b+1 in the high half of every word) into rows 2b and 2b+1 of the u32 matrix.
__global__ void __launch_bounds__(SC_THREADS)
k_scan_tile_counts_packed(const unsigned* __restrict__ packed, Count cno, unsigned ld, unsigned* __restrict__ counts,
                          unsigned* __restrict__ row_total) {
  PDL_ENTRY();
  __shared__ unsigned wsum[SC_THREADS / 32];
  const unsigned ntiles = (cno.get() + RS_TILE - 1) / RS_TILE;
  const int tid = threadIdx.x;
  const unsigned* prow = packed + (size_t)blockIdx.x * ld;
  unsigned* row0 = counts + (size_t)(2 * blockIdx.x) * ld;
  unsigned* row1 = row0 + ld;
  unsigned carry0 = 0, carry1 = 0;
  for (unsigned base = 0; base < ntiles; base += SC_THREADS * SC_ITEMS) {
    const unsigned i0 = base + tid * SC_ITEMS;
    uint4 v[SC_VEC];
#pragma unroll
    for (int q = 0; q < SC_VEC; ++q) {
      const unsigned i = i0 + 4 * q;
      v[q] = i < ntiles ? *reinterpret_cast<const uint4*>(prow + i) : make_uint4(0u, 0u, 0u, 0u);
    }
    unsigned run0 = 0, run1 = 0;
    uint4 lo[SC_VEC], hi[SC_VEC];
#pragma unroll
    for (int q = 0; q < SC_VEC; ++q) {
      const unsigned i = i0 + 4 * q;
      // padding columns (>= ntiles) hold garbage
      const unsigned a = i < ntiles ? v[q].x : 0u, b = i + 1 < ntiles ? v[q].y : 0u;
      const unsigned c = i + 2 < ntiles ? v[q].z : 0u, d = i + 3 < ntiles ? v[q].w : 0u;
      const unsigned a0 = a & 0xffffu, b0 = b & 0xffffu, c0 = c & 0xffffu, d0 = d & 0xffffu;
      const unsigned a1 = a >> 16, b1 = b >> 16, c1 = c >> 16, d1 = d >> 16;
      lo[q] = make_uint4(run0, run0 + a0, run0 + a0 + b0, run0 + a0 + b0 + c0);
      hi[q] = make_uint4(run1, run1 + a1, run1 + a1 + b1, run1 + a1 + b1 + c1);
      run0 += a0 + b0 + c0 + d0;
      run1 += a1 + b1 + c1 + d1;
    }
    unsigned tot0, tot1;
    const unsigned pre0 = carry0 + block_excl_scan<SC_THREADS / 32>(run0, wsum, tot0);
    const unsigned pre1 = carry1 + block_excl_scan<SC_THREADS / 32>(run1, wsum, tot1);
#pragma unroll
    for (int q = 0; q < SC_VEC; ++q) {
      const unsigned i = i0 + 4 * q;
      if (i < ntiles) {
        *reinterpret_cast<uint4*>(row0 + i) = make_uint4(pre0 + lo[q].x, pre0 + lo[q].y, pre0 + lo[q].z, pre0 + lo[q].w);
        *reinterpret_cast<uint4*>(row1 + i) = make_uint4(pre1 + hi[q].x, pre1 + hi[q].y, pre1 + hi[q].z, pre1 + hi[q].w);
      }
    }
    carry0 += tot0;
    carry1 += tot1;
  }
  if (tid == 0) {
    row_total[2 * blockIdx.x] = carry0;
    row_total[2 * blockIdx.x + 1] = carry1;
  }
}

// Scatter one tile of a digit pass. Item j of lane l of warp w is tile element
// w*512 + j*32 + l (coalesced loads); ranks follow element order, so the pass is stable.
// Values never occupy registers: cp.async stages them in input order and they are
// permuted shared->shared after the keys have been written. BITS and FULL are compile-time
// so the ranking loop is branch-free and full tiles carry no bounds predicates.
// Fused partition + exchange (sharded build): the destination of slab s is rank s's receive
// buffer -- a peer GPU's memory mapped into this process (symmetric memory / IPC) -- at
// element offset off[s] (this rank's place among the senders to slab s).
constexpr int kMaxP2P = 16;
struct P2PDst {
  unsigned* k[kMaxP2P];
  unsigned* v[kMaxP2P];
  unsigned long long off[kMaxP2P];
};

// Decoupled look-back over <= 16 slab counters per tile (the fused pair dispatch): status[tile]
// [slab] = flag << 62 | count, flag LB_AGG (this tile's count) or LB_PREFIX (inclusive prefix).
// Tiles are claimed in order from a ticket, so every predecessor is resident and publishes.
struct LookBack {
  unsigned long long* status;
};
__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

template <int BITS, bool FULL, bool TABLE = false, bool SRC_SMEM = false, bool P2P = false, bool LB = false>
__device__ __forceinline__ void radix_scatter_tile(RsSmem& sm, const unsigned* __restrict__ keys_in,
                                                   const unsigned* __restrict__ vals_in,
                                                   unsigned* __restrict__ keys_out, unsigned* __restrict__ vals_out,
                                                   unsigned tbase, unsigned tvalid, unsigned tile, unsigned ld,
                                                   int shift, const unsigned* __restrict__ hist,
                                                   const unsigned* __restrict__ offs,
                                                   const unsigned* __restrict__ dtable = nullptr,
                                                   const unsigned* __restrict__ kbase = nullptr,
                                                   const P2PDst* __restrict__ p2p = nullptr,
                                                   const LookBack* __restrict__ lb = nullptr) {
  constexpr int NB = 1 << BITS;
  constexpr unsigned DMASK = (unsigned)NB - 1u;
  static_assert(!P2P || (TABLE && NB <= kMaxP2P), "peer scatter: slab digits only");
  static_assert(!LB || NB <= kMaxP2P, "look-back: slab digits only");
  // digit of a key: bit field, or slab id = dtable[key >> shift] (keys then leave rebased
  // by kbase[slab], i.e. relative to their slab's first cell)
  auto digit = [&](unsigned k) -> unsigned { return TABLE ? __ldg(&dtable[k >> shift]) : (k >> shift) & DMASK; };
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  auto elem = [&](int j) { return (unsigned)warp * (RS_ITEMS * 32) + j * 32 + lane; };
  auto valid = [&](int j) { return FULL || elem(j) < tvalid; };

#ifndef PGRID_KEYS_FIRST
#define PGRID_KEYS_FIRST 1
#endif
#ifndef PGRID_KEYS_REG
#define PGRID_KEYS_REG 1
#endif
  // KREG: the keys stay in registers (digits extracted where used), no re-read for the local
  // scatter: 8-bit pass 102 -> 96 us (r2_ab_keys_reg.txt; values through registers instead of
  // the cp.async staging measured slower at every load point)
  constexpr bool KREG = PGRID_KEYS_REG && PGRID_KEYS_FIRST && !SRC_SMEM && !TABLE;
  // the tile's keys are requested first: the ranking waits on them (the DRAM round trip that
  // heads the pass's stall profile), everything else below overlaps their flight
  const unsigned* ksrc = SRC_SMEM ? keys_in : keys_in + tbase;
  unsigned dg[RS_ITEMS];
  if (PGRID_KEYS_FIRST && !SRC_SMEM) {
#pragma unroll
    for (int j = 0; j < RS_ITEMS; ++j) dg[j] = valid(j) ? __ldg(ksrc + elem(j)) : 0u;
  }
  // the per-digit inputs of this tile (L2 hits: digit totals and this tile's column of the
  // scanned count matrix) are copied into shared memory now, so their latency hides behind
  // the ranking without holding registers
#pragma unroll
  for (int q = 0; q < RS_DPT; ++q) {
    const int d = tid * RS_DPT + q;
    if (d < NB) {
      if (!P2P) cp_async4(&sm.hsm[d], hist + d);
      if (!LB) cp_async4(&sm.gbase[d], offs + (size_t)d * ld + tile);
    }
  }
  cp_async_commit();
  // SRC_SMEM: keys_in points at a shared-memory copy of the tile (element order) and
  // sm.vstage already holds the values
  if (!SRC_SMEM) {
    if (FULL) {
#pragma unroll
      for (int c = tid; c < RS_TILE / 4; c += RS_THREADS) cp_async16(&sm.vstage[4 * c], vals_in + tbase + 4 * c);
    } else {
      for (unsigned e = tid; e < tvalid; e += RS_THREADS) cp_async4(&sm.vstage[e], vals_in + tbase + e);
    }
    cp_async_commit();
  }
  {
    unsigned* row = reinterpret_cast<unsigned*>(&sm.whist[warp][0]);
#pragma unroll
    for (int q = lane; q < NB / 2; q += 32) row[q] = 0u;
  }
  if (KREG) {
  } else if (PGRID_KEYS_FIRST && !SRC_SMEM) {
#pragma unroll
    for (int j = 0; j < RS_ITEMS; ++j) dg[j] = valid(j) ? digit(dg[j]) : 0u;
  } else {
#pragma unroll
    for (int j = 0; j < RS_ITEMS; ++j) dg[j] = valid(j) ? digit(SRC_SMEM ? ksrc[elem(j)] : __ldg(ksrc + elem(j))) : 0u;
  }
  // peers (same-digit lanes) per item: bit-sliced ballots, items interleaved for ILP
  unsigned pm[RS_ITEMS];
#pragma unroll
  for (int j = 0; j < RS_ITEMS; ++j) pm[j] = FULL ? 0xffffffffu : __ballot_sync(0xffffffffu, valid(j));
#pragma unroll
  for (int b = 0; b < BITS; ++b) {
#pragma unroll
    for (int j = 0; j < RS_ITEMS; ++j) pm[j] = peers_step(pm[j], dg[j], KREG ? 1u << (b + shift) : 1u << b);
  }
  auto dig_of = [&](int j) -> unsigned { return KREG ? (dg[j] >> shift) & DMASK : dg[j]; };
  __syncwarp();
  const unsigned lt = lanemask_lt();
  unsigned rank[RS_ITEMS];
#pragma unroll
  for (int j = 0; j < RS_ITEMS; ++j) {
    const unsigned peers = valid(j) ? pm[j] : 0u;
    const int leader = __ffs(peers | (1u << lane)) - 1;  // invalid lanes: themselves
    unsigned old = 0;
    if (lane == leader && peers) {
      old = sm.whist[warp][dig_of(j)];
      sm.whist[warp][dig_of(j)] = (unsigned short)(old + __popc(peers));
    }
    old = __shfl_sync(0xffffffffu, old, leader);
    rank[j] = old + __popc(peers & lt);
    __syncwarp();
  }
  if (SRC_SMEM) cp_async_wait();
  else cp_async_wait_all_but_one();  // the per-digit group (the values' group may stay in flight)
  __syncthreads();
  // per digit (thread t owns digits 2t, 2t+1 -- one 32-bit word of every warp's u16 row):
  // warp offsets and tile counts of both digits in one pass over the rows
  unsigned* rows = reinterpret_cast<unsigned*>(&sm.whist[0][0]);
  unsigned tpk = 0;  // tile counts of both digits, packed (u16 lanes never carry: <= RS_TILE)
  if (tid < NB / 2) {
#pragma unroll
    for (int w = 0; w < RS_WARPS; ++w) tpk += rows[w * (kMaxBins / 2) + tid];
  }
  const unsigned tc[RS_DPT] = {tpk & 0xffffu, tpk >> 16};
  unsigned hs[RS_DPT], toff[RS_DPT];
#pragma unroll
  for (int q = 0; q < RS_DPT; ++q) {
    const int d = tid * RS_DPT + q;
    hs[q] = (!P2P && d < NB) ? sm.hsm[d] : 0u;
    toff[q] = (!LB && d < NB) ? sm.gbase[d] : 0u;
  }
  const unsigned tsum = tc[0] + tc[1], hsum = hs[0] + hs[1];
  if constexpr (LB) {
    // this tile's exclusive prefix per slab over the preceding tiles: decoupled look-back,
    // one warp per slab reading a window of 32 predecessors per round trip
    unsigned long long* row = lb->status + (size_t)tile * kMaxP2P;
    const int lane = tid & 31;
#pragma unroll
    for (int q = 0; q < RS_DPT; ++q) {
      const int d = tid * RS_DPT + q;
      if (d < NB) {
        st_release_u64(row + d, (tile ? LB_AGG : LB_PREFIX) | tc[q]);
        sm.hsm[d] = tc[q];  // (hsm is unused by the peer scatter)
      }
    }
    __syncthreads();
    for (int d = warp; d < NB; d += RS_WARPS) {
      unsigned long long pre = 0;
      if (tile) {
        for (long long j0 = (long long)tile - 1;; j0 -= 32) {
          const long long j = j0 - lane;
          unsigned long long v = 0;
          if (j >= 0) {
            do {
              v = ld_acquire_u64(lb->status + (size_t)j * kMaxP2P + d);
            } while (!(v >> 62));
          }
          const unsigned pm = __ballot_sync(0xffffffffu, j < 0 || (v >> 62) == 2ull);
          const int first = pm ? __ffs(pm) - 1 : 31;  // the closest inclusive prefix ends the walk
          unsigned long long x = (lane <= first && j >= 0) ? (v & LB_VALUE) : 0ull;
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
          pre += x;
          if (pm) break;
        }
        if (lane == 0) st_release_u64(row + d, LB_PREFIX | (pre + sm.hsm[d]));
      }
      if (lane == 0) sm.gbase[d] = (unsigned)pre;
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < RS_DPT; ++q) {
      const int d = tid * RS_DPT + q;
      toff[q] = d < NB ? sm.gbase[d] : 0u;
    }
  }
  unsigned ttot, htot;
  unsigned lpre = block_excl_scan<RS_WARPS>(tsum, sm.wsum, ttot);
  unsigned hpre = block_excl_scan<RS_WARPS>(hsum, sm.wsum, htot);
  if (tid < NB / 2) {
    // every warp's offsets = tile-local digit start + exclusive count over the lower warps
    // (folded in so the items below need one lookup each)
    unsigned run = lpre | ((lpre + tc[0]) << 16);
#pragma unroll
    for (int w = 0; w < RS_WARPS; ++w) {
      const unsigned c = rows[w * (kMaxBins / 2) + tid];
      rows[w * (kMaxBins / 2) + tid] = run;
      run += c;
    }
  }
#pragma unroll
  for (int q = 0; q < RS_DPT; ++q) {
    const int d = tid * RS_DPT + q;
    // P2P: positions inside slab d's receive buffer (32-bit: a receive buffer < 2^32 pairs)
    if (d < NB) sm.gbase[d] = (P2P ? (unsigned)p2p->off[d] : hpre) + toff[q] - lpre;
    lpre += tc[q];
    hpre += hs[q];
  }
  __syncthreads();
  // keys: stable local scatter into digit order (key re-read from L1/L2), run-coalesced write
#pragma unroll
  for (int j = 0; j < RS_ITEMS; ++j) {
    if (valid(j)) {
      rank[j] += sm.whist[warp][dig_of(j)];  // rank -> tile position
      PG_ASSERT(rank[j] < tvalid);
      sm.buf[rank[j]] = KREG ? dg[j] : ksrc[elem(j)];
    }
  }
  __syncthreads();
  unsigned gpos[RS_ITEMS];
  unsigned dpk[P2P ? (RS_ITEMS + 7) / 8 : 1] = {};  // P2P: the items' slabs, 4 bits each
#pragma unroll
  for (int r = 0; r < RS_ITEMS; ++r) {
    const unsigned i = tid + r * RS_THREADS;
    gpos[r] = 0;
    if (FULL || i < tvalid) {
      const unsigned k = sm.buf[i];
      const unsigned d = digit(k);
      gpos[r] = sm.gbase[d] + i;
      PG_ASSERT(P2P || gpos[r] < htot);
      if (P2P) {
        dpk[r / 8] |= d << (4 * (r % 8));
        p2p->k[d][gpos[r]] = k - __ldg(&kbase[d]);
      } else if (keys_out) {
        keys_out[gpos[r]] = TABLE ? k - __ldg(&kbase[d]) : k;
      }
    }
  }
  if (!SRC_SMEM) cp_async_wait();
  __syncthreads();
  // values: shared->shared permutation with the same positions, then write-out
#pragma unroll
  for (int j = 0; j < RS_ITEMS; ++j)
    if (valid(j)) sm.buf[rank[j]] = sm.vstage[elem(j)];
  __syncthreads();
#pragma unroll
  for (int r = 0; r < RS_ITEMS; ++r) {
    const unsigned i = tid + r * RS_THREADS;
    if (FULL || i < tvalid) {
      if (P2P) p2p->v[(dpk[r / 8] >> (4 * (r % 8))) & 15u][gpos[r]] = sm.buf[i];
      else vals_out[gpos[r]] = sm.buf[i];
    }
  }
}


// 9-bit digits: 3 CTAs/SM with 80 registers (no spill) beat 4 with 64 (127 vs 129 us per
// pass at cfg3); narrower digits keep 4 (102 vs 104-106 us), r2_ab_k4_rs_occupancy.txt
#ifndef RS_MIN_CTAS_OVERRIDE
constexpr int rs_min_ctas(int bits) { return bits >= 9 ? 3 : 4; }
#else
constexpr int rs_min_ctas(int) { return RS_MIN_CTAS_OVERRIDE; }
#endif
template <int BITS, bool TABLE>
__global__ void __launch_bounds__(RS_THREADS, rs_min_ctas(BITS))
k_radix_scatter(const unsigned* __restrict__ keys_in, const unsigned* __restrict__ vals_in,
                unsigned* __restrict__ keys_out, unsigned* __restrict__ vals_out, Count cno, int shift,
                const unsigned* __restrict__ hist, const unsigned* __restrict__ offs, unsigned ld,
                const unsigned* __restrict__ dtable, const unsigned* __restrict__ kbase) {
  PDL_ENTRY();
  extern __shared__ __align__(128) unsigned char smem_raw[];
  RsSmem& sm = *reinterpret_cast<RsSmem*>(smem_raw);
  const unsigned no = cno.get();
  const unsigned tile = blockIdx.x;
  const unsigned tbase = tile * (unsigned)RS_TILE;
  if (tbase >= no) return;
  const unsigned tvalid = min((unsigned)RS_TILE, no - tbase);
  if (tvalid == (unsigned)RS_TILE)
    radix_scatter_tile<BITS, true, TABLE>(sm, keys_in, vals_in, keys_out, vals_out, tbase, tvalid, tile, ld, shift,
                                          hist, offs, dtable, kbase);
  else
    radix_scatter_tile<BITS, false, TABLE>(sm, keys_in, vals_in, keys_out, vals_out, tbase, tvalid, tile, ld, shift,
                                           hist, offs, dtable, kbase);
}

// Stable partition by slab whose writes land directly in the slab owners' receive buffers.
template <int BITS>
__global__ void __launch_bounds__(RS_THREADS, RS_MIN_CTAS)
k_partition_send(const unsigned* __restrict__ keys_in, const unsigned* __restrict__ vals_in, Count cno, int shift,
                 const unsigned* __restrict__ offs, unsigned ld, const unsigned* __restrict__ dtable,
                 const unsigned* __restrict__ kbase, const P2PDst dst) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  RsSmem& sm = *reinterpret_cast<RsSmem*>(smem_raw);
  const unsigned no = cno.get();
  const unsigned tile = blockIdx.x;
  const unsigned tbase = tile * (unsigned)RS_TILE;
  if (tbase >= no) return;
  const unsigned tvalid = min((unsigned)RS_TILE, no - tbase);
  if (tvalid == (unsigned)RS_TILE)
    radix_scatter_tile<BITS, true, true, false, true>(sm, keys_in, vals_in, nullptr, nullptr, tbase, tvalid, tile, ld,
                                                      shift, nullptr, offs, dtable, kbase, &dst);
  else
    radix_scatter_tile<BITS, false, true, false, true>(sm, keys_in, vals_in, nullptr, nullptr, tbase, tvalid, tile, ld,
                                                       shift, nullptr, offs, dtable, kbase, &dst);
}

// ----------------------------------------------------------------------------------------
// Sharded build: device-side small collectives over peer memory.
// k_peer_put copies one rank's small array (its coarse histogram, its slab counts) into the
// same slot of every rank's exchange buffer (peer memory mapped into this process); after a
// device barrier every rank holds all ranks' arrays and reduces them itself, so no NCCL call
// and no host round trip sits between the pair expansion and the slab plan.
// ----------------------------------------------------------------------------------------
struct PeerPtrs {
  unsigned* p[kMaxP2P];
};
__global__ void __launch_bounds__(256) k_peer_put(const unsigned* __restrict__ src, unsigned n, PeerPtrs dst,
                                                  int nranks, unsigned long long offset) {
  const unsigned i = blockIdx.x * 256u + threadIdx.x;
  if (i >= n) return;
  const unsigned v = __ldg(src + i);
  for (int r = 0; r < nranks; ++r) dst.p[r][offset + i] = v;
}

// Slab plan on the device, the same arithmetic as distributed.plan_slabs: sum the ranks'
// coarse histograms (hists[r * nb + b]), cum = exclusive scan (nb + 1 entries), cut s =
// first bucket with cum >= ceil(s * total / P) (np.searchsorted, side left), clamped to nb;
// outputs the bucket -> slab table, each slab's first cell (u32, the key rebase) and
// plan = cuts[P+1] | cell_lo[P] | cell_hi[P] | pair_base[P+1] (int64).
constexpr int PLAN_THREADS = 1024;
constexpr int PLAN_MAX_BUCKETS = 4096;
__global__ void __launch_bounds__(PLAN_THREADS)
k_slab_plan(const unsigned* __restrict__ hists, int nranks, int nb, int shift, long long ncells, int P,
            unsigned* __restrict__ table, unsigned* __restrict__ slab_base, long long* __restrict__ plan) {
  __shared__ unsigned long long cum[PLAN_MAX_BUCKETS + 1];
  __shared__ unsigned long long wsum[PLAN_THREADS / 32];
  __shared__ long long cuts[kMaxP2P + 1];
  constexpr int PER = PLAN_MAX_BUCKETS / PLAN_THREADS;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  unsigned long long h[PER], run = 0;
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    const int b = tid * PER + q;
    unsigned long long x = 0;
    if (b < nb)
      for (int r = 0; r < nranks; ++r) x += __ldg(&hists[(size_t)r * nb + b]);
    h[q] = x;
    run += x;
  }
  unsigned long long inc = run;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const unsigned long long o = __shfl_up_sync(0xffffffffu, inc, d);
    if (lane >= d) inc += o;
  }
  if (lane == 31) wsum[warp] = inc;
  __syncthreads();
  unsigned long long pre = inc - run;
  for (int w = 0; w < warp; ++w) pre += wsum[w];
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    const int b = tid * PER + q;
    if (b < nb) cum[b] = pre;
    pre += h[q];
  }
  if (tid == PLAN_THREADS - 1) cum[nb] = pre;  // the last thread's running sum is the total
  __syncthreads();
  const unsigned long long total = cum[nb];
  if (tid <= P) {
    long long c;
    if (tid == 0) {
      c = 0;
    } else if (tid == P) {
      c = nb;
    } else {
      const unsigned long long target = ((unsigned long long)tid * total + (unsigned long long)P - 1) / (unsigned long long)P;
      int lo = 0, hi = nb + 1;  // first i in [0, nb] with cum[i] >= target (nb + 1 if none)
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (cum[mid] >= target) hi = mid;
        else lo = mid + 1;
      }
      c = lo < nb ? lo : nb;
    }
    cuts[tid] = c;
  }
  __syncthreads();
  if (tid == 0) {  // cuts[s] = max(cuts[s-1], ...): searchsorted of rising targets is monotone already
    for (int s2 = 1; s2 <= P; ++s2) cuts[s2] = max(cuts[s2], cuts[s2 - 1]);
  }
  __syncthreads();
  for (int b = tid; b < nb; b += PLAN_THREADS) {
    int sl = 0;
    while (sl + 1 < P && (long long)b >= cuts[sl + 1]) ++sl;
    table[b] = (unsigned)sl;
  }
  if (tid < P) {
    const long long lo = min(cuts[tid] << shift, ncells), hi = min(cuts[tid + 1] << shift, ncells);
    slab_base[tid] = (unsigned)lo;
    plan[P + 1 + tid] = lo;
    plan[2 * P + 1 + tid] = hi;
  }
  if (tid <= P) {
    plan[tid] = cuts[tid];
    plan[3 * P + 1 + tid] = (long long)cum[cuts[tid]];
  }
}

// ----------------------------------------------------------------------------------------
// K2: pair expansion on radix-sort tiles. Each CTA expands RS_TILE pairs, writes them in
// generation (object-major) order with 16-byte stores, and counts the tile's first-pass
// digits (the per-tile counts the first radix pass needs, so that pass skips its own
// upsweep; the row scan turns them into the global histogram too).
// ----------------------------------------------------------------------------------------
struct PeSmem {
  __align__(16) int slot[RS_TILE];  // expansion slots, then the transposed keys
  unsigned h[kMaxBins];
  __align__(16) ObjCache oc;        // object cache, then the transposed values
  int warpmax[2 * RS_WARPS + 1];
};
static_assert(sizeof(ObjCache) >= RS_TILE * 4, "the object cache doubles as the value transpose buffer");

#ifndef K2_MIN_CTAS
#define K2_MIN_CTAS (1024 / RS_THREADS)
#endif
__global__ void __launch_bounds__(RS_THREADS, K2_MIN_CTAS)
k_pairs_emit(const uint4* __restrict__ rec, const unsigned* __restrict__ tile_pre, long long n, Count cno,
             unsigned dx, unsigned dxy, PassPlan plan, const int2* __restrict__ bounds, unsigned* __restrict__ keys, unsigned* __restrict__ vals,
             unsigned* __restrict__ counts0, unsigned ld, unsigned* __restrict__ packed0) {
  PDL_ENTRY();
  extern __shared__ __align__(128) unsigned char smem_raw[];
  PeSmem& sm = *reinterpret_cast<PeSmem*>(smem_raw);
  const int tid = threadIdx.x;
  const unsigned no = cno.get();
  const unsigned p0 = blockIdx.x * (unsigned)RS_TILE;
  if (p0 >= no) return;
  const unsigned pend = min(p0 + (unsigned)RS_TILE, no);
  for (int b = tid; b < kMaxBins; b += RS_THREADS) sm.h[b] = 0u;
  unsigned key[RS_ITEMS];
  int own[RS_ITEMS];
  expand_tile<RS_THREADS, RS_ITEMS>(rec, n, p0, pend, dx, dxy, tile_pre, bounds, sm.slot, sm.warpmax, &sm.oc, key, own);
  const unsigned pbase = p0 + (unsigned)tid * RS_ITEMS;
  const int nvalid = pend > pbase ? (int)min((unsigned)RS_ITEMS, pend - pbase) : 0;
  // transpose through shared memory (the expansion's slots and object cache are dead): a
  // thread's 16 consecutive pairs leave as 16-byte chunks striped over the CTA, so every
  // warp store is 512 contiguous bytes; chunk index c is XOR-swizzled against bank conflicts
  __syncthreads();
  {
    uint4* ks = reinterpret_cast<uint4*>(sm.slot);
    uint4* vs = reinterpret_cast<uint4*>(&sm.oc);
    auto swz = [](unsigned c) { return c ^ ((c >> 3) & 7u); };
#pragma unroll
    for (int q = 0; q < RS_ITEMS / 4; ++q) {
      const unsigned c = (unsigned)tid * (RS_ITEMS / 4) + q;
      ks[swz(c)] = make_uint4(key[4 * q], key[4 * q + 1], key[4 * q + 2], key[4 * q + 3]);
      vs[swz(c)] = make_uint4(own[4 * q], own[4 * q + 1], own[4 * q + 2], own[4 * q + 3]);
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < RS_ITEMS / 4; ++q) {
      const unsigned c = (unsigned)tid + q * RS_THREADS;
      const unsigned e = p0 + 4 * c;
      const uint4 kk = ks[swz(c)], vv = vs[swz(c)];
      if (e + 4 <= pend) {
        reinterpret_cast<uint4*>(keys + e)[0] = kk;
        reinterpret_cast<uint4*>(vals + e)[0] = vv;
      } else {
        const unsigned kx[4] = {kk.x, kk.y, kk.z, kk.w}, vx[4] = {vv.x, vv.y, vv.z, vv.w};
#pragma unroll
        for (int r = 0; r < 4; ++r)
          if (e + r < pend) {
            keys[e + r] = kx[r];
            vals[e + r] = vx[r];
          }
      }
    }
  }
  {  // first-pass digit: consecutive cells rarely share it -- one atomic per pair
    const int sh = plan.shift[0];
    const unsigned mask = (1u << plan.bits[0]) - 1u;
#pragma unroll
    for (int j = 0; j < RS_ITEMS; ++j)
      if (j < nvalid) atomicAdd(&sm.h[(key[j] >> sh) & mask], 1u);
  }
  __syncthreads();
  // straight into the digit-major matrix: one 4-byte entry per digit row (the rows stay in
  // L2 until the row scan reads them, so the scattered writes cost no extra DRAM traffic)
  if (packed0) {  // two digits per word (a tile counts <= 4096 < 2^16): half the scattered stores
    for (int b = tid; b < (1 << plan.bits[0]) / 2; b += RS_THREADS)
      packed0[(size_t)b * ld + blockIdx.x] = sm.h[2 * b] | (sm.h[2 * b + 1] << 16);
  } else {
    for (int b = tid; b < (1 << plan.bits[0]); b += RS_THREADS) counts0[(size_t)b * ld + blockIdx.x] = sm.h[b];
  }
}


#ifndef PGRID_FUSED_DISPATCH
#define PGRID_FUSED_DISPATCH 0  // expansion + slab dispatch in one kernel: measured slower, not shipped
#endif
#if PGRID_FUSED_DISPATCH
// ----------------------------------------------------------------------------------------
// Sharded build, fused dispatch: pair expansion + slab partition + peer stores in ONE kernel.
// Each CTA claims the next 4096-pair tile from a ticket, expands it exactly as K2 does, ranks
// the pairs by slab (table digit, <= 16 slabs) and writes them straight into the slab
// owners' receive buffers (peer memory) at offset[slab] + tile prefix + rank; the tile
// prefixes come from a decoupled look-back over the slab counters (LookBack). So the pairs
// never touch this GPU's memory: no local pair buffer, no partition pass.
// ----------------------------------------------------------------------------------------
struct SendSmem {
  __align__(16) int slot[RS_TILE];  // expansion slots, then the tile's keys in element order
  union {
    struct {
      __align__(16) ObjCache oc;
      int warpmax[2 * RS_WARPS + 1];
    } pe;
    RsSmem rs;  // the slab scatter (its vstage receives the values)
  } u;
  unsigned tile;
};

template <int BITS>
__global__ void __launch_bounds__(RS_THREADS, 3)
k_pairs_send(const uint4* __restrict__ rec, const unsigned* __restrict__ tile_pre, long long n, Count cno,
             unsigned dx, unsigned dxy, const int2* __restrict__ bounds, unsigned val_offset, int shift,
             const unsigned* __restrict__ dtable, const unsigned* __restrict__ kbase, const P2PDst dst,
             LookBack lb, unsigned* __restrict__ ticket) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  SendSmem& sm = *reinterpret_cast<SendSmem*>(smem_raw);
  const int tid = threadIdx.x;
  if (tid == 0) sm.tile = atomicAdd(ticket, 1u);
  __syncthreads();
  const unsigned tile = sm.tile;
  const unsigned no = cno.get();
  const unsigned p0 = tile * (unsigned)RS_TILE;
  if (p0 >= no) return;
  const unsigned pend = min(p0 + (unsigned)RS_TILE, no);
  unsigned key[RS_ITEMS];
  int own[RS_ITEMS];
  expand_tile<RS_THREADS, RS_ITEMS>(rec, n, p0, pend, dx, dxy, tile_pre, bounds, sm.slot, sm.u.pe.warpmax,
                                    &sm.u.pe.oc, key, own);
  __syncthreads();  // the object cache is dead: the scatter's buffers overlay it
  unsigned* skey = reinterpret_cast<unsigned*>(sm.slot);
#pragma unroll
  for (int q = 0; q < RS_ITEMS / 4; ++q) {
    reinterpret_cast<uint4*>(skey)[tid * (RS_ITEMS / 4) + q] =
        make_uint4(key[4 * q], key[4 * q + 1], key[4 * q + 2], key[4 * q + 3]);
    reinterpret_cast<uint4*>(sm.u.rs.vstage)[tid * (RS_ITEMS / 4) + q] =
        make_uint4(own[4 * q] + val_offset, own[4 * q + 1] + val_offset, own[4 * q + 2] + val_offset,
                   own[4 * q + 3] + val_offset);
  }
  __syncthreads();
  const unsigned tvalid = pend - p0;
  if (tvalid == (unsigned)RS_TILE)
    radix_scatter_tile<BITS, true, true, true, true, true>(sm.u.rs, skey, nullptr, nullptr, nullptr, 0, tvalid, tile,
                                                           0, shift, nullptr, nullptr, dtable, kbase, &dst, &lb);
  else
    radix_scatter_tile<BITS, false, true, true, true, true>(sm.u.rs, skey, nullptr, nullptr, nullptr, 0, tvalid, tile,
                                                            0, shift, nullptr, nullptr, dtable, kbase, &dst, &lb);
}

// Coarse histogram of the pair cell ids (cell >> shift) straight from K1's box records,
// before any pair exists (the fused dispatch plans the slabs first): object i's cells are
// my*mz rows of mx consecutive ids lo + y*dx + z*dxy (x fastest, builders.py:104-117); each
// row adds its overlap with every bucket it spans. Counts equal K2's coarse histogram.
// Objects with more than COARSE_BIG rows (walls, floors: up to 65K rows) are queued and
// spread over a whole CTA by k_coarse_big, so no thread walks a wall alone.
constexpr unsigned COARSE_BIG = 256;
__device__ __forceinline__ void coarse_row(unsigned* hsh, unsigned a, unsigned mx, int shift) {
  const unsigned e = a + mx;  // cells [a, e)
  unsigned b = a >> shift;
  const unsigned bl = (e - 1) >> shift;
  if (b == bl) {
    atomicAdd(&hsh[b], mx);
  } else {
    for (; b <= bl; ++b) {
      const unsigned lo = max(a, b << shift), hi = min(e, (b + 1) << shift);
      atomicAdd(&hsh[b], hi - lo);
    }
  }
}
__device__ __forceinline__ unsigned coarse_count(const uint4* __restrict__ rec, const unsigned* __restrict__ tile_pre,
                                                 long long n, unsigned no, long long i, uint4& r) {
  r = __ldg(&rec[i]);
  const unsigned off = __ldg(&tile_pre[i / K1_TILE]) + r.w;
  const unsigned nxt = i + 1 < n ? tri_offset(rec, tile_pre, i + 1) : no;
  return nxt > off ? nxt - off : 0u;
}

__global__ void __launch_bounds__(256)
k_coarse_from_boxes(const uint4* __restrict__ rec, const unsigned* __restrict__ tile_pre, long long n, Count cno,
                    unsigned dx, unsigned dxy, int shift, int nbins, unsigned* __restrict__ coarse,
                    unsigned* __restrict__ big, unsigned big_cap) {
  extern __shared__ unsigned hsh[];
  for (int b = threadIdx.x; b < nbins; b += blockDim.x) hsh[b] = 0u;
  __syncthreads();
  const unsigned no = cno.get();
  // COARSE_U objects per thread per round, their loads issued together (latency-bound loop)
  constexpr int COARSE_U = 4;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i0 = (long long)blockIdx.x * blockDim.x + threadIdx.x; i0 < n; i0 += stride * COARSE_U) {
    uint4 r[COARSE_U];
    unsigned cnt[COARSE_U];
#pragma unroll
    for (int u = 0; u < COARSE_U; ++u) {
      const long long i = i0 + u * stride;
      cnt[u] = i < n ? coarse_count(rec, tile_pre, n, no, i, r[u]) : 0u;
    }
#pragma unroll
    for (int u = 0; u < COARSE_U; ++u) {
      if (!cnt[u]) continue;
      const unsigned mx = r[u].y, my = r[u].z, rows = cnt[u] / mx, mz = rows / my;
      if (rows > COARSE_BIG) {
        const unsigned slot = atomicAdd(&big[0], 1u);
        if (slot < big_cap) {
          big[1 + slot] = (unsigned)(i0 + u * stride);
          continue;
        }
      }
      for (unsigned z = 0; z < mz; ++z)
        for (unsigned y = 0; y < my; ++y) coarse_row(hsh, r[u].x + y * dx + z * dxy, mx, shift);
    }
  }
  __syncthreads();
  for (int b = threadIdx.x; b < nbins; b += blockDim.x)
    if (hsh[b]) atomicAdd(&coarse[b], hsh[b]);
}

// The queued objects, one CTA at a time, rows strided over the CTA's threads.
__global__ void __launch_bounds__(256)
k_coarse_big(const uint4* __restrict__ rec, const unsigned* __restrict__ tile_pre, long long n, Count cno, unsigned dx,
             unsigned dxy, int shift, int nbins, unsigned* __restrict__ coarse, const unsigned* __restrict__ big,
             unsigned big_cap) {
  extern __shared__ unsigned hsh[];
  const unsigned nbig = min(big[0], big_cap);
  if (!nbig) return;
  for (int b = threadIdx.x; b < nbins; b += blockDim.x) hsh[b] = 0u;
  __syncthreads();
  const unsigned no = cno.get();
  // every CTA takes a slice of every queued object's rows
  for (unsigned e = 0; e < nbig; ++e) {
    uint4 r;
    const unsigned cnt = coarse_count(rec, tile_pre, n, no, big[1 + e], r);
    const unsigned mx = r.y, my = r.z, rows = cnt / mx;
    for (unsigned q = blockIdx.x * blockDim.x + threadIdx.x; q < rows; q += gridDim.x * blockDim.x) {
      const unsigned z = q / my, y = q - z * my;
      coarse_row(hsh, r.x + y * dx + z * dxy, mx, shift);
    }
  }
  __syncthreads();
  for (int b = threadIdx.x; b < nbins; b += blockDim.x)
    if (hsh[b]) atomicAdd(&coarse[b], hsh[b]);
}

#endif  // PGRID_FUSED_DISPATCH

// ----------------------------------------------------------------------------------------
// K4: G from the sorted cell ids (RLE -> NonEmptyCells scatter -> ExclusiveSum, fused)
// ----------------------------------------------------------------------------------------
constexpr int G_THREADS = 256;
#ifndef G_ITEMS_OVERRIDE
constexpr int G_ITEMS = 16;
#else
constexpr int G_ITEMS = G_ITEMS_OVERRIDE;
#endif
constexpr int G_TILE = G_THREADS * G_ITEMS;  // cells per CTA

// G[c] = #pairs with cell < c = lower_bound(sorted, c). Each CTA owns cells [c0, c0+G_TILE):
// its key range [i0, i1) comes from k_key_tile_bounds; every first occurrence of a cell marks
// its run start; a block suffix-min fills empty cells with the next run start (or i1).
// The last CTA also writes the sentinel G[ncells] = NO (builders.py:131-133).
#ifndef K4_MIN_CTAS
#define K4_MIN_CTAS 8  // 32 registers, 8 CTAs/SM: 60.4 vs 64.5 us at cfg3 (r2_ab_k4_rs_occupancy.txt)
#endif
__global__ void __launch_bounds__(G_THREADS, K4_MIN_CTAS)
k_cell_offsets(const unsigned* __restrict__ sorted, Count cno, unsigned ncells, const unsigned* __restrict__ kb,
               unsigned* __restrict__ G) {
  PDL_ENTRY();
  const unsigned no = cno.get();
  __shared__ __align__(16) unsigned mark[G_TILE];
  __shared__ unsigned sh_wmin[G_ITEMS / 4 * (G_THREADS / 32)];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned c0 = blockIdx.x * (unsigned)G_TILE;
  const unsigned c1 = min(c0 + (unsigned)G_TILE, ncells);
  const unsigned i0 = __ldg(&kb[blockIdx.x]), i1 = __ldg(&kb[blockIdx.x + 1]);  // k_key_tile_bounds
#pragma unroll
  for (int q = 0; q < G_TILE / 4 / G_THREADS; ++q)
    reinterpret_cast<uint4*>(mark)[tid + q * G_THREADS] = make_uint4(~0u, ~0u, ~0u, ~0u);
  __syncthreads();
  // first occurrences: 4 independent coalesced loads per thread per chunk; the predecessor
  // key comes from the neighbouring lane (lane 0 loads it)
  for (unsigned base = i0; base < i1; base += 4 * G_THREADS) {
    unsigned k[4], pk[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const unsigned i = base + j * G_THREADS + tid;
      k[j] = i < i1 ? __ldg(sorted + i) : 0xffffffffu;
      pk[j] = (lane == 0 && i < i1 && i > 0) ? __ldg(sorted + i - 1) : 0xffffffffu;
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const unsigned i = base + j * G_THREADS + tid;
      const unsigned up = __shfl_up_sync(0xffffffffu, k[j], 1);
      const unsigned prev = lane == 0 ? pk[j] : up;
      if (i < i1 && (i == 0 || prev != k[j])) {
        PG_ASSERT(k[j] >= c0 && k[j] < c1);
        mark[k[j] - c0] = i;
      }
    }
  }
  __syncthreads();
  // block suffix-min over the tile. Cells are handled in G_ITEMS/4 groups: in group g thread t
  // owns cells g*1024 + 4t .. +3 (conflict-free mark loads, coalesced G stores). All groups'
  // warp suffix-mins are computed together and exchanged with ONE barrier.
  constexpr int NG = G_ITEMS / 4;
  uint4 a[NG];
  unsigned suf[NG];
#pragma unroll
  for (int g = 0; g < NG; ++g) {
    a[g] = reinterpret_cast<const uint4*>(mark)[g * G_THREADS + tid];
    suf[g] = min(min(a[g].x, a[g].y), min(a[g].z, a[g].w));
  }
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
#pragma unroll
    for (int g = 0; g < NG; ++g) {
      const unsigned o = __shfl_down_sync(0xffffffffu, suf[g], d);
      if (lane + d < 32) suf[g] = min(suf[g], o);  // inclusive suffix-min over lanes >= lane
    }
  }
  if (lane == 0) {
#pragma unroll
    for (int g = 0; g < NG; ++g) sh_wmin[g * (G_THREADS / 32) + warp] = suf[g];
  }
  __syncthreads();
  unsigned carry = i1;  // min over every cell right of the current group
#pragma unroll
  for (int g = NG - 1; g >= 0; --g) {
    unsigned right = __shfl_down_sync(0xffffffffu, suf[g], 1);
    if (lane == 31) right = 0xffffffffu;
    unsigned gmin = 0xffffffffu;
#pragma unroll
    for (int w = 0; w < G_THREADS / 32; ++w) {
      const unsigned x = sh_wmin[g * (G_THREADS / 32) + w];
      if (w > warp) right = min(right, x);
      gmin = min(gmin, x);
    }
    right = min(right, carry);
    unsigned v3 = min(a[g].w, right);
    unsigned v2 = min(a[g].z, v3);
    unsigned v1 = min(a[g].y, v2);
    unsigned v0 = min(a[g].x, v1);
    const unsigned cb = c0 + (unsigned)(g * G_THREADS + tid) * 4;
    if (cb + 4 <= c1) {
      *reinterpret_cast<uint4*>(G + cb) = make_uint4(v0, v1, v2, v3);
    } else {
      if (cb < c1) G[cb] = v0;
      if (cb + 1 < c1) G[cb + 1] = v1;
      if (cb + 2 < c1) G[cb + 2] = v2;
    }
    carry = min(carry, gmin);
  }
  if (blockIdx.x == gridDim.x - 1 && tid == 0) G[ncells] = no;
}

// ----------------------------------------------------------------------------------------
// K4L: the last sort level fused with G (the MSD-first finish). The radix passes covered only
// the key's top bits [L, key_bits), so the pairs arrive sorted by their bucket key >> L
// (stably: generation order inside a bucket), and a bucket's pairs occupy the same index range
// in O as in the input. Each CTA owns 8 buckets = 2^(L+3) cells [c0, c0 + 2^(L+3)) and their
// pairs [i0, i1) (k_key_tile_bounds: the lower bound is exact at bucket boundaries):
//   1. count its pairs per cell (shared-memory histogram; the first BK_CAP pairs' keys and
//      values are loaded once, into registers, for step 3 too),
//   2. scan the counts: G for its cells (the reference's RLE -> scatter -> ExclusiveSum,
//      builders.py:126-134); the counts become every cell's next O slot, and the buckets'
//      pair ranges and largest cell counts fall out of the same scan,
//   3. in rounds of whole buckets (<= BK_CAP pairs; a larger bucket in slices):
//      - fast path (vals_ascend: the pairs are in generation order, so a cell's values are
//        distinct, ascending triangle ids; cells <= BK_SORT_MAX pairs): every pair takes a slot
//        in its cell with a shared atomic and parks its value there; its rank in the cell is
//        the number of the cell's values below its own; O[cell start + rank] = value;
//      - stable path (any values): the round's keys staged in shared memory, warp w ranks
//        bucket w 32 pairs at a time (bit-sliced ballots over the low L bits, the lowest lane
//        of a cell's peers advances its slot), then the round's values move to O.
//      Either way generation order is kept inside a cell, exactly as the stable LSD pass it
//      replaces (primitives.py:97-113).
// This replaces the last radix pass with its upsweep and row scan, the key write-back, and K4.
// ----------------------------------------------------------------------------------------
#ifndef BK_THREADS_OVERRIDE
constexpr int BK_THREADS = 256;
#else
constexpr int BK_THREADS = BK_THREADS_OVERRIDE;
#endif
constexpr int BK_WARPS = BK_THREADS / 32;  // one bucket per warp
#ifndef BK_CAP_OVERRIDE
constexpr unsigned BK_CAP = 2048;          // pairs per round
#else
constexpr unsigned BK_CAP = BK_CAP_OVERRIDE;
#endif
constexpr unsigned BK_SORT_MAX = 32;       // largest cell ranked by value (else: ballot ranking)
// dynamic shared memory: cnt[2^(L+3)] | pos[BK_CAP] | key[BK_CAP] (u16, relative to c0)
__host__ __device__ constexpr size_t bk_smem_bytes(int L) { return 4u * (1u << (L + 3)) + 4u * BK_CAP + 2u * BK_CAP; }

#ifndef BK_MIN_CTAS
#define BK_MIN_CTAS 5  // 48 registers: 5 CTAs/SM (r2_ab_bucket_*.txt)
#endif
template <int L>
__global__ void __launch_bounds__(BK_THREADS, BK_MIN_CTAS)
k_bucket_sort(const unsigned* __restrict__ keys, const unsigned* __restrict__ vals, Count cno, unsigned ncells,
              const unsigned* __restrict__ kb, unsigned* __restrict__ G, unsigned* __restrict__ O, int vals_ascend) {
  PDL_ENTRY();
  constexpr unsigned NCB = 1u << L, NC = NCB * BK_WARPS;
  constexpr unsigned GC = 4u * BK_THREADS;  // cells per group: thread t owns 4t..4t+3 of each
  constexpr int NG = NC >= GC ? (int)(NC / GC) : 1;
  static_assert(L >= 2 && L <= 10, "bucket width");
  extern __shared__ __align__(16) unsigned bk_dyn[];
  unsigned* cnt = bk_dyn;
  unsigned* pos = bk_dyn + NC;
  unsigned short* key = reinterpret_cast<unsigned short*>(bk_dyn + NC + BK_CAP);

  __shared__ unsigned wsum[NG][BK_WARPS];
  __shared__ unsigned bst[BK_WARPS + 1];
  __shared__ unsigned bmax[BK_WARPS];  // the largest cell count of each bucket
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned no = cno.get();
  const unsigned c0 = blockIdx.x * NC;
  const unsigned i0 = __ldg(&kb[blockIdx.x]), i1 = __ldg(&kb[blockIdx.x + 1]);
  for (unsigned q = tid * 4; q < NC; q += BK_THREADS * 4) *reinterpret_cast<uint4*>(cnt + q) = make_uint4(0, 0, 0, 0);
  if (tid < BK_WARPS) bmax[tid] = 0;
  __syncthreads();
  // 1. histogram. The first BK_CAP pairs (keys and values) are loaded once, up front: they are
  // also the first round's data (step 3), so a CTA with <= BK_CAP pairs reads HBM once
  constexpr int RV = BK_CAP / BK_THREADS;
  unsigned kv[RV], vv[RV];
#pragma unroll
  for (int j = 0; j < RV; ++j) {
    const unsigned i = i0 + j * BK_THREADS + tid;
    kv[j] = i < i1 ? __ldg(keys + i) : 0u;
    vv[j] = i < i1 ? __ldg(vals + i) : 0u;
  }
#pragma unroll
  for (int j = 0; j < RV; ++j) {
    if (i0 + j * BK_THREADS + tid < i1) {
      PG_ASSERT(kv[j] >= c0 && kv[j] - c0 < NC);
      atomicAdd(&cnt[kv[j] - c0], 1u);
    }
  }
  for (unsigned base = i0 + BK_CAP; base < i1; base += 8 * BK_THREADS) {
    unsigned k[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const unsigned i = base + j * BK_THREADS + tid;
      k[j] = i < i1 ? __ldg(keys + i) : 0u;
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (base + j * BK_THREADS + tid < i1) {
        PG_ASSERT(k[j] >= c0 && k[j] - c0 < NC);
        atomicAdd(&cnt[k[j] - c0], 1u);
      }
    }
  }
  __syncthreads();
  // 2. exclusive scan of the counts, offset by i0: every group's warp scan at once (sums
  // first, the counts are re-read for the offsets), one barrier
  unsigned sum[NG], inc[NG];
#pragma unroll
  for (int g = 0; g < NG; ++g) {
    const unsigned q = (unsigned)(g * BK_THREADS + tid) * 4;
    const uint4 a = q < NC ? reinterpret_cast<const uint4*>(cnt)[g * BK_THREADS + tid] : make_uint4(0, 0, 0, 0);
    sum[g] = a.x + a.y + a.z + a.w;
    inc[g] = sum[g];
  }
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
#pragma unroll
    for (int g = 0; g < NG; ++g) {
      const unsigned o = __shfl_up_sync(0xffffffffu, inc[g], d);
      if (lane >= d) inc[g] += o;
    }
  }
  if (lane == 31) {
#pragma unroll
    for (int g = 0; g < NG; ++g) wsum[g][warp] = inc[g];
  }
  __syncthreads();
  unsigned carry = i0;
#pragma unroll
  for (int g = 0; g < NG; ++g) {
    unsigned wpre = 0, gtot = 0;
#pragma unroll
    for (int w = 0; w < BK_WARPS; ++w) {
      const unsigned x = wsum[g][w];
      wpre += w < warp ? x : 0u;
      gtot += x;
    }
    const unsigned q = (unsigned)(g * BK_THREADS + tid) * 4;
    if (q < NC) {
      const uint4 a = reinterpret_cast<const uint4*>(cnt)[g * BK_THREADS + tid];
      const unsigned v0 = carry + wpre + inc[g] - sum[g];
      const uint4 v = make_uint4(v0, v0 + a.x, v0 + a.x + a.y, v0 + a.x + a.y + a.z);
      reinterpret_cast<uint4*>(cnt)[g * BK_THREADS + tid] = v;  // the thread's own cells
      const unsigned c = c0 + q;
      if (c + 4 <= ncells) {
        *reinterpret_cast<uint4*>(G + c) = v;
      } else {
        if (c < ncells) G[c] = v.x;
        if (c + 1 < ncells) G[c + 1] = v.y;
        if (c + 2 < ncells) G[c + 2] = v.z;
      }
      if ((q & (NCB - 1)) == 0) bst[q / NCB] = v0;  // a bucket's first cell (NCB >= 4)
      const unsigned m = max(max(a.x, a.y), max(a.z, a.w));
      if constexpr (NCB >= 128 && NC >= GC) {  // the warp's 128 cells lie in one bucket (all lanes here)
        const unsigned wm = __reduce_max_sync(0xffffffffu, m);
        if (lane == 0 && wm > 1) atomicMax(&bmax[q / NCB], wm);
      } else {
        if (m > 1) atomicMax(&bmax[q / NCB], m);
      }
    }
    carry += gtot;
  }
  if (tid == 0) bst[BK_WARPS] = i1;
  if (blockIdx.x == gridDim.x - 1 && tid == 0) G[ncells] = no;
  __syncthreads();
  // 3. rounds of whole buckets (or slices of one bucket larger than BK_CAP)
  const unsigned lt = lanemask_lt();
  __shared__ unsigned round[4];  // the round's end, first and past-last bucket, fast path
  unsigned rb = i0;               // the round's first pair
  while (rb < i1) {
    if (warp == 0) {  // lane b looks at bucket b: one load each, ballots instead of a serial walk
      const bool in = lane < BK_WARPS;
      const unsigned e1 = in ? bst[lane + 1] : 0xffffffffu;  // bucket lane's end
      const unsigned bm = in ? bmax[lane] : 0u;
      // first bucket not finished (every bucket ending <= rb is done or empty)
      const int ba = __ffs(__ballot_sync(0xffffffffu, in && e1 > rb)) - 1;
      const unsigned eba = __shfl_sync(0xffffffffu, e1, ba);
      int bb = ba + 1;
      unsigned re = min(eba, rb + BK_CAP);
      if (re == eba) {  // whole buckets: extend while they fit in BK_CAP pairs
        const unsigned fit = __ballot_sync(0xffffffffu, in && lane >= ba && e1 - rb <= BK_CAP);
        bb = ba + __ffs(~(fit >> ba)) - 1;  // the run of fitting buckets from ba
        re = __shfl_sync(0xffffffffu, e1, bb - 1);
      }
      // whole buckets whose cells hold <= BK_SORT_MAX pairs each, values ascending in
      // generation order (vals_ascend): slots by shared atomics, ranks by value
      const unsigned m = __reduce_max_sync(0xffffffffu, lane >= ba && lane < bb ? bm : 0u);
      if (lane == 0) {
        round[0] = re;
        round[1] = (unsigned)ba;
        round[2] = (unsigned)bb;
        round[3] = vals_ascend && bst[ba] == rb && re == bst[bb] && m <= BK_SORT_MAX;
      }
    }
    __syncthreads();
    const unsigned re = round[0];
    const int ba = (int)round[1], bb = (int)round[2];
    const bool fast = round[3] != 0;
    const unsigned rn = re - rb;
    if (rb != i0) {  // (the first round's pairs are already in registers)
#pragma unroll
      for (int j = 0; j < RV; ++j) {
        const unsigned e = j * BK_THREADS + tid;
        kv[j] = e < rn ? __ldg(keys + rb + e) : 0u;
        vv[j] = e < rn ? __ldg(vals + rb + e) : 0u;
      }
    }
    if (fast) {
      // a cell's pairs come from distinct triangles in generation (= ascending value) order,
      // so any slot order inside the cell followed by ranking its values is the stable order
#pragma unroll
      for (int j = 0; j < RV; ++j) {
        const unsigned e = j * BK_THREADS + tid;
        if (e < rn) {
          const unsigned slot = atomicAdd(&cnt[kv[j] - c0], 1u) - rb;
          PG_ASSERT(slot < rn);
          pos[slot] = vv[j];
        }
      }
      __syncthreads();
      // each pair's rank inside its cell = the cell's values below its own (a cell holds
      // <= BK_SORT_MAX pairs); the previous cell's slot counter is final: the cell's start
#pragma unroll
      for (int j = 0; j < RV; ++j) {
        const unsigned e = j * BK_THREADS + tid;
        if (e < rn) {
          const unsigned c = kv[j] - c0, v = vv[j];
          const unsigned s0 = c ? cnt[c - 1] : i0, s1 = cnt[c];
          // (cells of 1-4 pairs without a loop: 98% of the multi-pair cells in every config)
          const unsigned nc = s1 - s0;
          unsigned r = 0;
          if (nc > 1) {
            const unsigned* p = pos + (s0 - rb);
            r = (p[0] < v) + (p[1] < v);
            if (nc > 2) {
              r += p[2] < v;
              if (nc > 3) {
                r += p[3] < v;
                for (unsigned x = 4; x < nc; ++x) r += p[x] < v;
              }
            }
          }
          O[s0 + r] = v;
        }
      }
      __syncthreads();
      rb = re;
      continue;
    }
#pragma unroll
    for (int j = 0; j < RV; ++j) {
      const unsigned e = j * BK_THREADS + tid;
      if (e < rn) key[e] = (unsigned short)(kv[j] - c0);
    }
    __syncthreads();
    // warp w ranks bucket ba + w of the round (its pairs in [max(bst, rb), min(bst', re)))
    if (ba + warp < bb) {
      const int bk = ba + warp;
      const unsigned s = max(bst[bk], rb) - rb, t = min(bst[bk + 1], re) - rb;
      for (unsigned base = s; base < t; base += 32) {
        const unsigned e = base + lane;
        const bool ok = e < t;
        const unsigned k = ok ? key[e] : 0u;
        unsigned pm = __ballot_sync(0xffffffffu, ok);
#pragma unroll 5  // (a full unroll at L = 10 crashes ptxas 12.9's register allocator)
        for (int bit = 0; bit < L; ++bit) pm = peers_step(pm, k, 1u << bit);
        const unsigned peers = ok ? pm : 0u;
        const int leader = __ffs(peers | (1u << lane)) - 1;
        unsigned old = 0;
        if (ok && lane == leader) {
          PG_ASSERT((k >> L) == (unsigned)bk);
          old = cnt[k];
          cnt[k] = old + __popc(peers);
        }
        old = __shfl_sync(0xffffffffu, old, leader);
        if (ok) {
          PG_ASSERT(old + __popc(peers & lt) >= bst[bk] && old + __popc(peers & lt) < bst[bk + 1]);
          pos[e] = old + __popc(peers & lt);
        }
        __syncwarp();
      }
    }
    __syncthreads();
    // the round's values into O: coalesced loads, stores inside the round's buckets
#pragma unroll
    for (int j = 0; j < RV; ++j) {
      const unsigned e = j * BK_THREADS + tid;
      if (e < rn) O[pos[e]] = vv[j];
    }
    __syncthreads();
    rb = re;
  }
}

// ----------------------------------------------------------------------------------------
// The paper's comparison builders: "sorted" and "compact" grids
// (builders.py:172-231). Both walk each triangle's whole cell box in one thread, which is
// exactly the per-object load imbalance Alg. 1 removes; they produce the same
// canonical G/O and share K1 with the parallel builder.
// ----------------------------------------------------------------------------------------
__device__ __forceinline__ unsigned tri_offset_or_end(const uint4* __restrict__ rec,
                                                      const unsigned* __restrict__ tile_pre, long long n,
                                                      unsigned no, long long i) {
  return i < n ? tri_offset(rec, tile_pre, i) : no;
}

// pairgen_sorted (_ckernels.pyx:53-70): one thread per triangle writes its cells, x-fastest.
__global__ void __launch_bounds__(256)
k_pairgen_per_object(const uint4* __restrict__ rec, const unsigned* __restrict__ tile_pre, long long n, unsigned no,
                     unsigned dx, unsigned dxy, unsigned* __restrict__ keys, unsigned* __restrict__ vals,
                     unsigned* __restrict__ max_work) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint4 r = __ldg(&rec[i]);
  unsigned pos = tri_offset_or_end(rec, tile_pre, n, no, i);
  const unsigned end = tri_offset_or_end(rec, tile_pre, n, no, i + 1);
  if (end > pos) atomicMax(max_work, end - pos);
  const unsigned mz = (end - pos) / (r.y * r.z);
  for (unsigned z = 0; z < mz; ++z)
    for (unsigned y = 0; y < r.z; ++y) {
      const unsigned row = r.x + dx * y + dxy * z;
      for (unsigned x = 0; x < r.y; ++x) {
        keys[pos] = row + x;
        vals[pos] = (unsigned)i;
        ++pos;
      }
    }
}

// compact_count / compact_fill (_ckernels.pyx:73-109): per-cell counters, then slot claims.
template <bool FILL>
__global__ void __launch_bounds__(256)
k_compact_walk(const uint4* __restrict__ rec, const unsigned* __restrict__ tile_pre, long long n, unsigned no,
               unsigned dx, unsigned dxy, unsigned* __restrict__ cell, unsigned* __restrict__ O,
               unsigned* __restrict__ max_work) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint4 r = __ldg(&rec[i]);
  const unsigned cnt = tri_offset_or_end(rec, tile_pre, n, no, i + 1) - tri_offset_or_end(rec, tile_pre, n, no, i);
  if (!cnt) return;
  if (!FILL && max_work) atomicMax(max_work, cnt);
  const unsigned mz = cnt / (r.y * r.z);
  for (unsigned z = 0; z < mz; ++z)
    for (unsigned y = 0; y < r.z; ++y) {
      const unsigned row = r.x + dx * y + dxy * z;
      unsigned x = 0;
      if (FILL) {  // cell[] = cursors (copy of G); 4 slot claims in flight per step
        for (; x + 4 <= r.y; x += 4) {
          const unsigned s0 = atomicAdd(&cell[row + x], 1u), s1 = atomicAdd(&cell[row + x + 1], 1u);
          const unsigned s2 = atomicAdd(&cell[row + x + 2], 1u), s3 = atomicAdd(&cell[row + x + 3], 1u);
          O[s0] = (unsigned)i;
          O[s1] = (unsigned)i;
          O[s2] = (unsigned)i;
          O[s3] = (unsigned)i;
        }
      }
      for (; x < r.y; ++x) {
        if (FILL)
          O[atomicAdd(&cell[row + x], 1u)] = (unsigned)i;
        else
          atomicAdd(&cell[row + x], 1u);                   // cell[] = counts
      }
    }
}

// Generic exclusive scan of u32[n] -> out[n] (+ out[n] = total when with_total): per-tile sums,
// k_scan_tile_sums over the tiles, then the tile-local scans.
constexpr int XS_THREADS = 256;
constexpr int XS_ITEMS = 16;
constexpr int XS_TILE = XS_THREADS * XS_ITEMS;
__global__ void __launch_bounds__(XS_THREADS)
k_tile_reduce(const unsigned* __restrict__ in, long long n, unsigned long long* __restrict__ tile_sum) {
  __shared__ unsigned long long w[XS_THREADS / 32];
  const long long base = (long long)blockIdx.x * XS_TILE;
  unsigned long long s = 0;
#pragma unroll
  for (int q = 0; q < XS_ITEMS; ++q) {
    const long long i = base + q * XS_THREADS + threadIdx.x;
    s += i < n ? __ldg(in + i) : 0u;
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) s += __shfl_xor_sync(0xffffffffu, s, d);
  if ((threadIdx.x & 31) == 0) w[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t = 0;
    for (int k = 0; k < XS_THREADS / 32; ++k) t += w[k];
    tile_sum[blockIdx.x] = t;
  }
}

__global__ void __launch_bounds__(XS_THREADS)
k_tile_scan_apply(const unsigned* __restrict__ in, long long n, const unsigned* __restrict__ tile_pre,
                  const unsigned long long* __restrict__ total, unsigned* __restrict__ out) {
  __shared__ unsigned wsum[XS_THREADS / 32];
  const long long base = (long long)blockIdx.x * XS_TILE + (long long)threadIdx.x * XS_ITEMS;
  unsigned v[XS_ITEMS], run = 0;
#pragma unroll
  for (int q = 0; q < XS_ITEMS; ++q) {
    const unsigned x = base + q < n ? __ldg(in + base + q) : 0u;
    v[q] = run;
    run += x;
  }
  unsigned tot;
  const unsigned pre = tile_pre[blockIdx.x] + block_excl_scan<XS_THREADS / 32>(run, wsum, tot);
#pragma unroll
  for (int q = 0; q < XS_ITEMS; ++q)
    if (base + q < n) out[base + q] = pre + v[q];
  if (blockIdx.x == 0 && threadIdx.x == 0 && total) out[n] = (unsigned)*total;
}

// Canonicalisation of the compact grid (ids ascending per cell, builders.py:221-225):
// short segments by one thread (insertion sort), longer ones queued for a CTA each.
constexpr int SEG_SMALL = 32;
constexpr int SEG_BLOCK = 4096;
__global__ void __launch_bounds__(256)
k_sort_segments_small(const unsigned* __restrict__ G, unsigned ncells, unsigned* __restrict__ O,
                      unsigned* __restrict__ big, unsigned* __restrict__ nbig) {
  const unsigned c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncells) return;
  const unsigned a = G[c], e = G[c + 1];
  const unsigned len = e - a;
  if (len <= 1) return;
  if (len > SEG_SMALL) {
    big[atomicAdd(nbig, 1u)] = c;
    return;
  }
  for (unsigned k = 1; k < len; ++k) {  // insertion sort (segments are mostly 1-3 ids)
    const unsigned x = O[a + k];
    unsigned m = k;
    while (m > 0 && O[a + m - 1] > x) {
      O[a + m] = O[a + m - 1];
      --m;
    }
    O[a + m] = x;
  }
}

// One CTA per long segment: bitonic sort, all compare-exchanges ascending (the first stage of
// each merge pairs k with its mirror k ^ (size-1)), so virtual +inf padding past the segment
// never moves and compare-exchanges against it can be skipped. Segments of up to SEG_BLOCK
// ids are sorted in shared memory, longer ones (rare) in place in global memory.
template <typename Load, typename Store>
__device__ __forceinline__ void bitonic_ascending(unsigned len, Load ld, Store stv) {
  unsigned p2 = 1;
  while (p2 < len) p2 <<= 1;
  for (unsigned size = 2; size <= p2; size <<= 1)
    for (unsigned stride = size >> 1; stride > 0; stride >>= 1) {
      for (unsigned k = threadIdx.x; k < p2; k += blockDim.x) {
        const unsigned j = stride == (size >> 1) ? (k ^ (size - 1)) : (k ^ stride);
        if (j > k && j < len) {
          const unsigned x = ld(k), y = ld(j);
          if (x > y) {
            stv(k, y);
            stv(j, x);
          }
        }
      }
      __syncthreads();
    }
}

__global__ void __launch_bounds__(1024)
k_sort_segments_big(const unsigned* __restrict__ G, const unsigned* __restrict__ big, const unsigned* __restrict__ nbig,
                    unsigned* __restrict__ O) {
  __shared__ unsigned sh[SEG_BLOCK];
  if (blockIdx.x >= *nbig) return;
  const unsigned c = big[blockIdx.x];
  const unsigned a = G[c], len = G[c + 1] - a;
  if (len <= SEG_BLOCK) {
    for (unsigned k = threadIdx.x; k < len; k += blockDim.x) sh[k] = O[a + k];
    __syncthreads();
    bitonic_ascending(len, [&](unsigned k) { return sh[k]; }, [&](unsigned k, unsigned v) { sh[k] = v; });
    for (unsigned k = threadIdx.x; k < len; k += blockDim.x) O[a + k] = sh[k];
  } else {
    unsigned* seg = O + a;
    bitonic_ascending(len, [&](unsigned k) { return seg[k]; }, [&](unsigned k, unsigned v) { seg[k] = v; });
  }
}


// ----------------------------------------------------------------------------------------
// Grid statistics (stats.py:42-64): the integer inputs of GridStats.
//   stats[0] += #cells with G[c+1] != G[c]     stats[1] += #in-grid objects (count > 0)
//   stats[2] = max cells per in-grid object
// ----------------------------------------------------------------------------------------
__device__ __forceinline__ unsigned long long block_sum_u64(unsigned long long v, unsigned long long* sh) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  unsigned long long t = 0;
  if (threadIdx.x == 0)
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += sh[w];
  return t;
}

__global__ void __launch_bounds__(256)
k_stats_cells(const unsigned* __restrict__ G, long long ncells, unsigned long long* __restrict__ stats) {
  __shared__ unsigned long long sh[8];
  unsigned long long c = 0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < ncells; i += (long long)gridDim.x * blockDim.x)
    c += __ldg(G + i + 1) != __ldg(G + i);
  c = block_sum_u64(c, sh);
  if (threadIdx.x == 0 && c) atomicAdd(stats, c);
}

__global__ void __launch_bounds__(256)
k_stats_objects(const uint4* __restrict__ rec, const unsigned* __restrict__ tile_pre, long long n, unsigned no,
                unsigned long long* __restrict__ stats) {
  __shared__ unsigned long long sh[8];
  unsigned long long kept = 0;
  unsigned mx = 0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const unsigned cnt = tri_offset_or_end(rec, tile_pre, n, no, i + 1) - tri_offset_or_end(rec, tile_pre, n, no, i);
    kept += cnt != 0;
    mx = max(mx, cnt);
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, d));
  if ((threadIdx.x & 31) == 0 && mx) atomicMax(stats + 2, (unsigned long long)mx);
  kept = block_sum_u64(kept, sh);
  if (threadIdx.x == 0 && kept) atomicAdd(stats + 1, kept);
}


// ----------------------------------------------------------------------------------------
// Mesh bounds (geometry.py:55-59 mesh_bounds over ALL vertices, referenced
// or not): per-axis min / max of V (nv x 3 doubles). np.min / np.max propagate NaN, which
// the reference then rejects (Aabb, geometry.py:20-25): a NaN sets flag bit 1 instead.
// Threads stride the flat array by a multiple of 3, so each thread stays on one axis.
// ----------------------------------------------------------------------------------------
constexpr int MB_THREADS = 192;
__global__ void __launch_bounds__(MB_THREADS)
k_mesh_bounds(const double* __restrict__ V, long long nflat, double* __restrict__ part, unsigned* __restrict__ flag) {
  __shared__ double smin[MB_THREADS], smax[MB_THREADS];
  const long long stride = (long long)gridDim.x * MB_THREADS;
  double mn = CUDART_INF, mx = -CUDART_INF;
  bool nan = false;
  for (long long i = (long long)blockIdx.x * MB_THREADS + threadIdx.x; i < nflat; i += stride) {
    const double v = __ldg(V + i);
    nan |= v != v;
    mn = v < mn ? v : mn;
    mx = v > mx ? v : mx;
  }
  if (__any_sync(0xffffffffu, nan) && (threadIdx.x & 31) == 0) atomicOr(flag, 1u);
  smin[threadIdx.x] = mn;
  smax[threadIdx.x] = mx;
  __syncthreads();
  if (threadIdx.x < 3) {  // thread k reduces axis (k + block offset) % 3 entries
    const int axis = (int)(((long long)blockIdx.x * MB_THREADS + threadIdx.x) % 3);
    double a = CUDART_INF, b = -CUDART_INF;
    for (int t = threadIdx.x; t < MB_THREADS; t += 3) {
      a = smin[t] < a ? smin[t] : a;
      b = smax[t] > b ? smax[t] : b;
    }
    part[(size_t)blockIdx.x * 6 + axis] = a;
    part[(size_t)blockIdx.x * 6 + 3 + axis] = b;
  }
}

__global__ void __launch_bounds__(32)
k_mesh_bounds_final(const double* __restrict__ part, int nblocks, double* __restrict__ out) {
  if (threadIdx.x >= 6) return;
  const bool is_min = threadIdx.x < 3;
  double r = is_min ? CUDART_INF : -CUDART_INF;
  for (int b = 0; b < nblocks; ++b) {
    const double v = part[(size_t)b * 6 + threadIdx.x];
    r = is_min ? (v < r ? v : r) : (v > r ? v : r);
  }
  out[threadIdx.x] = r;
}

}  // namespace pgrid
