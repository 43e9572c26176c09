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
#include <cstdint>

#ifndef PGRID_RANK_BALLOT
#define PGRID_RANK_BALLOT 1
#endif
#include <cuda_runtime.h>

namespace pgrid {

// ----------------------------------------------------------------------------------------
// common helpers
// ----------------------------------------------------------------------------------------
struct DevSpec {
  double lo[3];
  double hi[3];
  double cell[3];
  int dims[3];
};

// Per-pass digit plan for the radix sort.
constexpr int kMaxPasses = 4;
struct PassPlan {
  int npasses;
  int shift[kMaxPasses];
  int bits[kMaxPasses];
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
__device__ __forceinline__ unsigned clip_axis(long long v, int dim) {
  return v < 0 ? 0u : (v > (long long)(dim - 1) ? (unsigned)(dim - 1) : (unsigned)v);
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
constexpr int K1_ITEMS = 4;
constexpr int K1_TILE = K1_THREADS * K1_ITEMS;
constexpr unsigned long long LB_AGG = 1ull << 62;
constexpr unsigned long long LB_PREFIX = 2ull << 62;
constexpr unsigned long long LB_VALUE = (1ull << 62) - 1;

// Per-triangle record written by K1 and read by K2: {lo_cell, mx, my, pair offset}.
// mx/my are the box extents in x/y; count = mx*my*mz is implied by the offsets.
// Dropped triangles (keep == false, gridcore.py:159) are {0, 1, 1, off} with count 0.
__global__ void __launch_bounds__(K1_THREADS)
k_boxes_count_scan(const double* __restrict__ V, const int* __restrict__ T, long long n, DevSpec s,
                   uint4* __restrict__ rec, unsigned long long* __restrict__ status,
                   unsigned* __restrict__ tile_ctr, unsigned long long* __restrict__ total,
                   unsigned* __restrict__ err) {
  __shared__ unsigned sh_tile;
  __shared__ unsigned long long sh_warp[K1_THREADS / 32];
  __shared__ unsigned long long sh_excl;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) sh_tile = atomicAdd(tile_ctr, 1u);
  __syncthreads();
  const unsigned tile = sh_tile;
  const unsigned ntiles = (unsigned)((n + K1_TILE - 1) / K1_TILE);
  const long long first = (long long)tile * K1_TILE + (long long)tid * K1_ITEMS;

  uint3 box[K1_ITEMS];
  unsigned cnt[K1_ITEMS];
  const unsigned dx = (unsigned)s.dims[0], dxy = (unsigned)s.dims[0] * (unsigned)s.dims[1];
#pragma unroll
  for (int j = 0; j < K1_ITEMS; ++j) {
    const long long i = first + j;
    box[j] = make_uint3(0u, 1u, 1u);
    cnt[j] = 0;
    if (i < n) {
      const int t0 = __ldg(T + 3 * i), t1 = __ldg(T + 3 * i + 1), t2 = __ldg(T + 3 * i + 2);
      bool keep = true;
      unsigned lo[3], hi[3];
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const double a = __ldg(V + 3 * (long long)t0 + k);
        const double b = __ldg(V + 3 * (long long)t1 + k);
        const double c = __ldg(V + 3 * (long long)t2 + k);
        // np.min/np.max propagate NaN, which fails both comparisons (gridcore.py:156-159);
        // fmin/fmax do not, so NaN is folded into keep explicitly.
        const bool nan = isnan(a) | isnan(b) | isnan(c);
        const double mn = fmin(fmin(a, b), c);
        const double mx = fmax(fmax(a, b), c);
        keep &= !nan && (mx >= s.lo[k]) && (mn <= s.hi[k]);
        const double ql = __ddiv_rn(__dsub_rn(mn, s.lo[k]), s.cell[k]);
        const double qh = __ddiv_rn(__dsub_rn(mx, s.lo[k]), s.cell[k]);
        lo[k] = clip_axis(np_floor_i64(ql), s.dims[k]);
        hi[k] = clip_axis(np_floor_i64(qh), s.dims[k]);
      }
      if (keep && (hi[0] < lo[0] || hi[1] < lo[1] || hi[2] < lo[2])) {
        // +inf / >2^63 upper corners cast to INT64_MIN and clip to 0 below lo: the reference
        // then fails its non-negative / coincident-mark checks (primitives.py:22-25, 71-72).
        atomicOr(err, 1u);
        keep = false;
      }
      if (keep) {
        const unsigned ex = hi[0] - lo[0] + 1, ey = hi[1] - lo[1] + 1, ez = hi[2] - lo[2] + 1;
        box[j] = make_uint3(lo[0] + dx * lo[1] + dxy * lo[2], ex, ey);
        cnt[j] = ex * ey * ez;  // <= ncells <= 2^30
      }
    }
  }
  // block-wide exclusive scan of the counts (blocked arrangement keeps triangle order)
  unsigned long long tsum = 0;
#pragma unroll
  for (int j = 0; j < K1_ITEMS; ++j) tsum += cnt[j];
  unsigned long long incl = tsum;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const unsigned long long o = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += o;
  }
  if (lane == 31) sh_warp[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    unsigned long long w = lane < K1_THREADS / 32 ? sh_warp[lane] : 0ull;
    unsigned long long wi = w;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const unsigned long long o = __shfl_up_sync(0xffffffffu, wi, d);
      if (lane >= d) wi += o;
    }
    const unsigned long long aggregate = __shfl_sync(0xffffffffu, wi, K1_THREADS / 32 - 1);
    if (lane < K1_THREADS / 32) sh_warp[lane] = wi - w;  // exclusive warp prefix
    // decoupled look-back (one warp, 32 predecessors per round)
    unsigned long long excl = 0;
    if (tile == 0) {
      if (lane == 0) st_relaxed_u64(status, LB_PREFIX | aggregate);
    } else {
      if (lane == 0) st_relaxed_u64(status + tile, LB_AGG | aggregate);
      long long pred = (long long)tile - 1 - lane;
      while (true) {
        unsigned long long v = pred >= 0 ? ld_relaxed_u64(status + pred) : LB_PREFIX;
        while (__any_sync(0xffffffffu, (v >> 62) == 0)) {
          if ((v >> 62) == 0) v = ld_relaxed_u64(status + pred);
        }
        const unsigned pmask = __ballot_sync(0xffffffffu, (v >> 62) == 2);
        const int stop = pmask ? __ffs(pmask) - 1 : 31;
        unsigned long long contrib = lane <= stop ? (v & LB_VALUE) : 0ull;
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) contrib += __shfl_xor_sync(0xffffffffu, contrib, d);
        excl += contrib;
        if (pmask) break;
        pred -= 32;
      }
      if (lane == 0) st_relaxed_u64(status + tile, LB_PREFIX | (excl + aggregate));
    }
    if (lane == 0) {
      sh_excl = excl;
      if (tile == ntiles - 1) *total = excl + aggregate;
    }
  }
  __syncthreads();
  unsigned long long off = sh_excl + sh_warp[warp] + (incl - tsum);
#pragma unroll
  for (int j = 0; j < K1_ITEMS; ++j) {
    const long long i = first + j;
    if (i < n) rec[i] = make_uint4(box[j].x, box[j].y, box[j].z, (unsigned)off);
    off += cnt[j];
  }
}

// ----------------------------------------------------------------------------------------
// K2: load-balanced pair expansion + radix digit histograms
// ----------------------------------------------------------------------------------------
constexpr int K2_THREADS = 256;
constexpr int K2_ITEMS = 8;
constexpr int K2_TILE = K2_THREADS * K2_ITEMS;
constexpr int kMaxDigitBits = 9;
constexpr int kMaxBins = 1 << kMaxDigitBits;  // 512

// Each CTA owns pairs [p0, p0 + K2_TILE). The owning triangle of every pair is recovered
// the way Alg. 1 does it (marks at run starts + inclusive max-scan), but
// tile-locally: the tile's first owner comes from a 32-ary search over the record offsets,
// the run starts inside the tile are scattered into shared memory, and a block max-scan
// fills the gaps. Within a thread's 8 consecutive pairs the cell coordinate is stepped
// incrementally (x-fastest), so the two divisions of _make_cell_ids (builders.py:111-113)
// run at most once per thread.
__global__ void __launch_bounds__(K2_THREADS)
k_expand_pairs(const uint4* __restrict__ rec, long long n, unsigned no, unsigned dx, unsigned dxy,
               PassPlan plan, unsigned* __restrict__ keys, unsigned* __restrict__ vals,
               unsigned* __restrict__ hist) {
  __shared__ __align__(16) int slot[K2_TILE];
  __shared__ unsigned sh_hist[kMaxPasses * kMaxBins];
  __shared__ int sh_warpmax[K2_THREADS / 32];
  __shared__ long long sh_olo;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned p0 = blockIdx.x * (unsigned)K2_TILE;
  const unsigned pend = min(p0 + (unsigned)K2_TILE, no);

  for (int i = tid; i < K2_TILE; i += K2_THREADS) slot[i] = -1;
  for (int i = tid; i < plan.npasses * kMaxBins; i += K2_THREADS) sh_hist[i] = 0;
  if (warp == 0) {
    // olo = (#triangles with offset <= p0) - 1: the owner of pair p0.
    const unsigned long long c = warp_lower_bound((unsigned long long)n, (unsigned long long)p0 + 1,
                                                  [&](unsigned long long i) { return (unsigned long long)__ldg(&rec[i].w); });
    if (lane == 0) sh_olo = (long long)c - 1;
  }
  __syncthreads();
  const long long olo = sh_olo;
  if (tid == 0) slot[0] = (int)olo;
  // run starts inside the tile: every triangle after olo whose offset is < pend
  for (long long ob = olo + 1;; ob += K2_THREADS) {
    const long long o = ob + tid;
    bool in = false;
    if (o < n) {
      const unsigned off = __ldg(&rec[o].w);
      if (off < pend) {
        atomicMax(&slot[off - p0], (int)o);  // zero-count triangles share the next start; max wins
        in = true;
      }
    }
    if (!__syncthreads_and(in)) break;
  }
  __syncthreads();
  // inclusive max-scan over the slots (blocked: thread t owns slots [8t, 8t+8))
  int own[K2_ITEMS];
  {
    const int4 a = *reinterpret_cast<const int4*>(&slot[tid * K2_ITEMS]);
    const int4 b = *reinterpret_cast<const int4*>(&slot[tid * K2_ITEMS + 4]);
    own[0] = a.x; own[1] = a.y; own[2] = a.z; own[3] = a.w;
    own[4] = b.x; own[5] = b.y; own[6] = b.z; own[7] = b.w;
  }
#pragma unroll
  for (int j = 1; j < K2_ITEMS; ++j) own[j] = max(own[j], own[j - 1]);
  int run = own[K2_ITEMS - 1];
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int o = __shfl_up_sync(0xffffffffu, run, d);
    if (lane >= d) run = max(run, o);
  }
  if (lane == 31) sh_warpmax[warp] = run;
  __syncthreads();
  int carry = __shfl_up_sync(0xffffffffu, run, 1);
  if (lane == 0) carry = -1;
  for (int w = 0; w < warp; ++w) carry = max(carry, sh_warpmax[w]);
#pragma unroll
  for (int j = 0; j < K2_ITEMS; ++j) own[j] = max(own[j], carry);

  // expansion
  unsigned key[K2_ITEMS];
  const unsigned pbase = p0 + (unsigned)tid * K2_ITEMS;
  int prev = -1;
  unsigned cell = 0, x = 0, y = 0, mx = 1, my = 1;
#pragma unroll
  for (int j = 0; j < K2_ITEMS; ++j) {
    const unsigned p = pbase + j;
    key[j] = 0;
    if (p < pend) {
      const int o = own[j];
      if (o != prev) {
        const uint4 r = __ldg(&rec[o]);
        const unsigned rel = p - r.w;
        mx = r.y;
        my = r.z;
        const unsigned mxy = mx * my;
        const unsigned z = rel / mxy;
        const unsigned rem = rel - z * mxy;
        y = rem / mx;
        x = rem - y * mx;
        cell = r.x + x + dx * y + dxy * z;
        prev = o;
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
  if (pbase + K2_ITEMS <= pend) {
    uint4* kd = reinterpret_cast<uint4*>(keys + pbase);
    uint4* vd = reinterpret_cast<uint4*>(vals + pbase);
    kd[0] = make_uint4(key[0], key[1], key[2], key[3]);
    kd[1] = make_uint4(key[4], key[5], key[6], key[7]);
    vd[0] = make_uint4(own[0], own[1], own[2], own[3]);
    vd[1] = make_uint4(own[4], own[5], own[6], own[7]);
  } else {
#pragma unroll
    for (int j = 0; j < K2_ITEMS; ++j)
      if (pbase + j < pend) {
        keys[pbase + j] = key[j];
        vals[pbase + j] = (unsigned)own[j];
      }
  }
  // digit histograms of every radix pass (consumed by the onesweep passes)
  for (int ps = 0; ps < plan.npasses; ++ps) {
    const unsigned mask = (1u << plan.bits[ps]) - 1u;
#pragma unroll
    for (int j = 0; j < K2_ITEMS; ++j)
      if (pbase + j < pend) atomicAdd(&sh_hist[ps * kMaxBins + ((key[j] >> plan.shift[ps]) & mask)], 1u);
  }
  __syncthreads();
  for (int i = tid; i < plan.npasses * kMaxBins; i += K2_THREADS) {
    const unsigned c = sh_hist[i];
    if (c) atomicAdd(&hist[i], c);
  }
}

// Standalone digit histogram (plugin-seam sort of arbitrary keys).
__global__ void __launch_bounds__(256)
k_digit_hist(const unsigned* __restrict__ keys, long long n, PassPlan plan, unsigned* __restrict__ hist) {
  __shared__ unsigned sh_hist[kMaxPasses * kMaxBins];
  for (int i = threadIdx.x; i < plan.npasses * kMaxBins; i += blockDim.x) sh_hist[i] = 0;
  __syncthreads();
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const unsigned k = keys[i];
    for (int ps = 0; ps < plan.npasses; ++ps)
      atomicAdd(&sh_hist[ps * kMaxBins + ((k >> plan.shift[ps]) & ((1u << plan.bits[ps]) - 1u))], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < plan.npasses * kMaxBins; i += blockDim.x)
    if (sh_hist[i]) atomicAdd(&hist[i], sh_hist[i]);
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
constexpr int RS_THREADS = 256;
constexpr int RS_WARPS = RS_THREADS / 32;
constexpr int RS_ITEMS = 16;
constexpr int RS_TILE = RS_THREADS * RS_ITEMS;  // 4096 pairs per tile
constexpr int RS_DPT = kMaxBins / RS_THREADS;   // digits per thread in the per-digit phases (2)

struct RsSmem {
  unsigned buf[RS_TILE];                     // tile in digit order: keys, then values
  unsigned vstage[RS_TILE];                  // values in input order (cp.async staging)
  unsigned short whist[RS_WARPS][kMaxBins];  // per-warp digit counts -> exclusive warp offsets
  unsigned local_start[kMaxBins];            // tile-local exclusive digit prefix
  unsigned gbase[kMaxBins];                  // global position of buf[0] for each digit
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

__global__ void __launch_bounds__(RS_THREADS)
k_tile_counts(const unsigned* __restrict__ keys, unsigned no, int shift, int bits, unsigned* __restrict__ counts) {
  __shared__ unsigned h[kMaxBins];
  const int tid = threadIdx.x;
  const unsigned ntiles = (no + RS_TILE - 1) / RS_TILE;
  const unsigned tile = blockIdx.x;
  const unsigned tbase = tile * (unsigned)RS_TILE;
  const unsigned tvalid = min((unsigned)RS_TILE, no - tbase);
  const unsigned dmask = (1u << bits) - 1u;
  for (int b = tid; b < kMaxBins; b += RS_THREADS) h[b] = 0u;
  __syncthreads();
  if (tvalid == (unsigned)RS_TILE) {
    const uint4* src = reinterpret_cast<const uint4*>(keys + tbase);
    uint4 k[RS_TILE / 4 / RS_THREADS];
#pragma unroll
    for (int r = 0; r < RS_TILE / 4 / RS_THREADS; ++r) k[r] = __ldcs(src + tid + r * RS_THREADS);
#pragma unroll
    for (int r = 0; r < RS_TILE / 4 / RS_THREADS; ++r) {
      atomicAdd(&h[(k[r].x >> shift) & dmask], 1u);
      atomicAdd(&h[(k[r].y >> shift) & dmask], 1u);
      atomicAdd(&h[(k[r].z >> shift) & dmask], 1u);
      atomicAdd(&h[(k[r].w >> shift) & dmask], 1u);
    }
  } else {
    for (unsigned e = tid; e < tvalid; e += RS_THREADS) atomicAdd(&h[(__ldcs(keys + tbase + e) >> shift) & dmask], 1u);
  }
  __syncthreads();
  for (int b = tid; b < (1 << bits); b += RS_THREADS) counts[(size_t)b * ntiles + tile] = h[b];
}

constexpr int SC_THREADS = 256;
constexpr int SC_ITEMS = 16;
// One CTA per digit row: counts[row][0..ntiles) -> exclusive prefix over tiles, in place.
__global__ void __launch_bounds__(SC_THREADS)
k_scan_tile_counts(unsigned* __restrict__ counts, unsigned ntiles) {
  __shared__ unsigned s[SC_THREADS * SC_ITEMS];
  __shared__ unsigned wsum[SC_THREADS / 32];
  const int tid = threadIdx.x;
  unsigned* row = counts + (size_t)blockIdx.x * ntiles;
  unsigned carry = 0;
  for (unsigned base = 0; base < ntiles; base += SC_THREADS * SC_ITEMS) {
#pragma unroll
    for (int k = 0; k < SC_ITEMS; ++k) {
      const unsigned i = base + tid + k * SC_THREADS;
      s[tid + k * SC_THREADS] = i < ntiles ? row[i] : 0u;
    }
    __syncthreads();
    unsigned v[SC_ITEMS], run = 0;
#pragma unroll
    for (int q = 0; q < SC_ITEMS; ++q) {
      v[q] = run;
      run += s[tid * SC_ITEMS + q];
    }
    unsigned total;
    const unsigned pre = block_excl_scan<SC_THREADS / 32>(run, wsum, total);
#pragma unroll
    for (int q = 0; q < SC_ITEMS; ++q) s[tid * SC_ITEMS + q] = carry + pre + v[q];
    __syncthreads();
#pragma unroll
    for (int k = 0; k < SC_ITEMS; ++k) {
      const unsigned i = base + tid + k * SC_THREADS;
      if (i < ntiles) row[i] = s[tid + k * SC_THREADS];
    }
    carry += total;
    __syncthreads();
  }
}

// Scatter one tile of a digit pass. Item j of lane l of warp w is tile element
// w*512 + j*32 + l (coalesced loads); ranks follow element order, so the pass is stable.
// Values never occupy registers: cp.async stages them in input order and they are
// permuted shared->shared after the keys have been written. BITS and FULL are compile-time
// so the ranking loop is branch-free and full tiles carry no bounds predicates.
template <int BITS, bool FULL>
__device__ __forceinline__ void radix_scatter_tile(RsSmem& sm, const unsigned* __restrict__ keys_in,
                                                   const unsigned* __restrict__ vals_in,
                                                   unsigned* __restrict__ keys_out, unsigned* __restrict__ vals_out,
                                                   unsigned tbase, unsigned tvalid, unsigned tile, unsigned ntiles,
                                                   int shift, const unsigned* __restrict__ hist,
                                                   const unsigned* __restrict__ offs) {
  constexpr int NB = 1 << BITS;
  constexpr unsigned DMASK = (unsigned)NB - 1u;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  auto elem = [&](int j) { return (unsigned)warp * (RS_ITEMS * 32) + j * 32 + lane; };
  auto valid = [&](int j) { return FULL || elem(j) < tvalid; };

  if (FULL) {
#pragma unroll
    for (int c = tid; c < RS_TILE / 4; c += RS_THREADS) cp_async16(&sm.vstage[4 * c], vals_in + tbase + 4 * c);
  } else {
    for (unsigned e = tid; e < tvalid; e += RS_THREADS) cp_async4(&sm.vstage[e], vals_in + tbase + e);
  }
  cp_async_commit();
  {
    unsigned* row = reinterpret_cast<unsigned*>(&sm.whist[warp][0]);
#pragma unroll
    for (int q = lane; q < NB / 2; q += 32) row[q] = 0u;
  }
  unsigned dg[RS_ITEMS];
#pragma unroll
  for (int j = 0; j < RS_ITEMS; ++j) dg[j] = valid(j) ? (__ldg(keys_in + tbase + elem(j)) >> shift) & DMASK : 0u;
  // peers (same-digit lanes) per item: bit-sliced ballots, items interleaved for ILP
  unsigned pm[RS_ITEMS];
#pragma unroll
  for (int j = 0; j < RS_ITEMS; ++j) pm[j] = FULL ? 0xffffffffu : __ballot_sync(0xffffffffu, valid(j));
#pragma unroll
  for (int b = 0; b < BITS; ++b) {
#pragma unroll
    for (int j = 0; j < RS_ITEMS; ++j) {
      const unsigned bb = __ballot_sync(0xffffffffu, (dg[j] >> b) & 1u);
      pm[j] &= ((dg[j] >> b) & 1u) ? bb : ~bb;
    }
  }
  __syncwarp();
  const unsigned lt = lanemask_lt();
  unsigned rank[RS_ITEMS];
#pragma unroll
  for (int j = 0; j < RS_ITEMS; ++j) {
    const unsigned peers = valid(j) ? pm[j] : 0u;
    const int leader = __ffs(peers | (1u << lane)) - 1;  // invalid lanes: themselves
    unsigned old = 0;
    if (lane == leader && peers) {
      old = sm.whist[warp][dg[j]];
      sm.whist[warp][dg[j]] = (unsigned short)(old + __popc(peers));
    }
    old = __shfl_sync(0xffffffffu, old, leader);
    rank[j] = old + __popc(peers & lt);
    __syncwarp();
  }
  __syncthreads();
  // per digit (RS_DPT consecutive digits per thread): warp offsets, tile counts, prefixes
  unsigned tc[RS_DPT], hs[RS_DPT], tsum = 0, hsum = 0;
#pragma unroll
  for (int q = 0; q < RS_DPT; ++q) {
    const int d = tid * RS_DPT + q;
    unsigned run = 0;
    if (d < NB) {
#pragma unroll
      for (int w = 0; w < RS_WARPS; ++w) {
        const unsigned c = sm.whist[w][d];
        sm.whist[w][d] = (unsigned short)run;
        run += c;
      }
    }
    tc[q] = run;
    hs[q] = d < NB ? __ldg(&hist[d]) : 0u;
    tsum += run;
    hsum += hs[q];
  }
  unsigned ttot, htot;
  unsigned lpre = block_excl_scan<RS_WARPS>(tsum, sm.wsum, ttot);
  unsigned hpre = block_excl_scan<RS_WARPS>(hsum, sm.wsum, htot);
#pragma unroll
  for (int q = 0; q < RS_DPT; ++q) {
    const int d = tid * RS_DPT + q;
    if (d < NB) {
      sm.local_start[d] = lpre;
      sm.gbase[d] = hpre + __ldg(&offs[(size_t)d * ntiles + tile]) - lpre;
    }
    lpre += tc[q];
    hpre += hs[q];
  }
  __syncthreads();
  // keys: stable local scatter into digit order (key re-read from L1/L2), run-coalesced write
#pragma unroll
  for (int j = 0; j < RS_ITEMS; ++j) {
    if (valid(j)) {
      rank[j] += sm.local_start[dg[j]] + sm.whist[warp][dg[j]];  // rank -> tile position
      sm.buf[rank[j]] = keys_in[tbase + elem(j)];
    }
  }
  __syncthreads();
  unsigned gpos[RS_ITEMS];
#pragma unroll
  for (int r = 0; r < RS_ITEMS; ++r) {
    const unsigned i = tid + r * RS_THREADS;
    gpos[r] = 0;
    if (FULL || i < tvalid) {
      const unsigned k = sm.buf[i];
      gpos[r] = sm.gbase[(k >> shift) & DMASK] + i;
      if (keys_out) keys_out[gpos[r]] = k;
    }
  }
  cp_async_wait();
  __syncthreads();
  // values: shared->shared permutation with the same positions, then write-out
#pragma unroll
  for (int j = 0; j < RS_ITEMS; ++j)
    if (valid(j)) sm.buf[rank[j]] = sm.vstage[elem(j)];
  __syncthreads();
#pragma unroll
  for (int r = 0; r < RS_ITEMS; ++r) {
    const unsigned i = tid + r * RS_THREADS;
    if (FULL || i < tvalid) vals_out[gpos[r]] = sm.buf[i];
  }
}

template <int BITS>
__global__ void __launch_bounds__(RS_THREADS, 4)
k_radix_scatter(const unsigned* __restrict__ keys_in, const unsigned* __restrict__ vals_in,
                unsigned* __restrict__ keys_out, unsigned* __restrict__ vals_out, unsigned no, int shift,
                const unsigned* __restrict__ hist, const unsigned* __restrict__ offs) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  RsSmem& sm = *reinterpret_cast<RsSmem*>(smem_raw);
  const unsigned ntiles = (no + RS_TILE - 1) / RS_TILE;
  const unsigned tile = blockIdx.x;
  const unsigned tbase = tile * (unsigned)RS_TILE;
  const unsigned tvalid = min((unsigned)RS_TILE, no - tbase);
  if (tvalid == (unsigned)RS_TILE)
    radix_scatter_tile<BITS, true>(sm, keys_in, vals_in, keys_out, vals_out, tbase, tvalid, tile, ntiles, shift,
                                   hist, offs);
  else
    radix_scatter_tile<BITS, false>(sm, keys_in, vals_in, keys_out, vals_out, tbase, tvalid, tile, ntiles, shift,
                                    hist, offs);
}

// ----------------------------------------------------------------------------------------
// K4: G from the sorted cell ids (RLE -> NonEmptyCells scatter -> ExclusiveSum, fused)
// ----------------------------------------------------------------------------------------
constexpr int G_THREADS = 256;
constexpr int G_ITEMS = 16;
constexpr int G_TILE = G_THREADS * G_ITEMS;  // cells per CTA

// G[c] = #pairs with cell < c = lower_bound(sorted, c). Each CTA owns cells [c0, c0+G_TILE):
// two warp searches bound its key range [i0, i1); every first occurrence of a cell marks
// its run start; a block suffix-min fills empty cells with the next run start (or i1).
// The last CTA also writes the sentinel G[ncells] = NO (builders.py:131-133).
__global__ void __launch_bounds__(G_THREADS)
k_cell_offsets(const unsigned* __restrict__ sorted, unsigned no, unsigned ncells, unsigned* __restrict__ G) {
  __shared__ __align__(16) unsigned mark[G_TILE];
  __shared__ unsigned sh_i0, sh_i1;
  __shared__ unsigned sh_wmin[G_THREADS / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned c0 = blockIdx.x * (unsigned)G_TILE;
  const unsigned c1 = min(c0 + (unsigned)G_TILE, ncells);
  auto ld = [&](unsigned long long i) { return (unsigned long long)__ldg(sorted + i); };
  if (warp == 0) {
    const unsigned v = (unsigned)warp_lower_bound(no, c0, ld);
    if (lane == 0) sh_i0 = v;
  } else if (warp == 1) {
    const unsigned v = (unsigned)warp_lower_bound(no, c1, ld);
    if (lane == 0) sh_i1 = v;
  }
  for (int i = tid; i < G_TILE; i += G_THREADS) mark[i] = 0xffffffffu;
  __syncthreads();
  const unsigned i0 = sh_i0, i1 = sh_i1;
  for (unsigned i = i0 + tid; i < i1; i += G_THREADS) {
    const unsigned k = __ldg(sorted + i);
    if (i == 0 || __ldg(sorted + i - 1) != k) mark[k - c0] = i;
  }
  __syncthreads();
  // block suffix-min (thread t owns cells [16t, 16t+16))
  unsigned v[G_ITEMS];
#pragma unroll
  for (int q = 0; q < G_ITEMS / 4; ++q) {
    const uint4 a = *reinterpret_cast<const uint4*>(&mark[tid * G_ITEMS + 4 * q]);
    v[4 * q] = a.x; v[4 * q + 1] = a.y; v[4 * q + 2] = a.z; v[4 * q + 3] = a.w;
  }
  unsigned tmin = i1;
#pragma unroll
  for (int q = 0; q < G_ITEMS; ++q) tmin = min(tmin, v[q]);
  unsigned suf = tmin;  // inclusive suffix-min over lanes >= lane
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const unsigned o = __shfl_down_sync(0xffffffffu, suf, d);
    if (lane + d < 32) suf = min(suf, o);
  }
  if (lane == 0) sh_wmin[warp] = suf;
  __syncthreads();
  unsigned carry = __shfl_down_sync(0xffffffffu, suf, 1);
  if (lane == 31) carry = i1;
  for (int w = warp + 1; w < G_THREADS / 32; ++w) carry = min(carry, sh_wmin[w]);
#pragma unroll
  for (int q = G_ITEMS - 1; q >= 0; --q) {
    carry = min(carry, v[q]);
    v[q] = carry;
  }
  const unsigned cb = c0 + (unsigned)tid * G_ITEMS;
  if (cb + G_ITEMS <= c1) {
    uint4* dst = reinterpret_cast<uint4*>(G + cb);
#pragma unroll
    for (int q = 0; q < G_ITEMS / 4; ++q) dst[q] = make_uint4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
  } else {
#pragma unroll
    for (int q = 0; q < G_ITEMS; ++q)
      if (cb + q < c1) G[cb + q] = v[q];
  }
  if (blockIdx.x == gridDim.x - 1 && tid == 0) G[ncells] = no;
}

}  // namespace pgrid
