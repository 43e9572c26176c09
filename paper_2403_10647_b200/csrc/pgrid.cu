// pgrid.cu -- host orchestration and C ABI of libpgrid.so (see include/pgrid.h).
//
// One pg_builder = one device workspace (grow-only, reused across builds) + events.
// pg_count runs K1 and reads NO back (the only host sync of a build: O's size is dynamic,
// PAPER.md:90); pg_finish runs K2 -> radix passes -> K4 into the caller's G and O.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <atomic>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <thread>

#include <unistd.h>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: ranges for nsys / ncu --nvtx

#include "../../include/pgrid.h"
#include "pgrid_kernels.cuh"
#include "pgrid_dda.cuh"
#include "pgrid_obj.cuh"

using namespace pgrid;

namespace {

thread_local std::string g_err;

// One NVTX range per C-ABI call (the host side of a build in a timeline profile).
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

// Persistent host threads for parallel memcpy (the pageable-input staging path): one copy
// call splits [src, src + n) into equal parts, the caller copies part 0, the workers the
// rest. A single memcpy thread moves ~10 GB/s; the PCIe link takes ~55 GB/s.
class HostCopyPool {
 public:
  static HostCopyPool& get() {
    static HostCopyPool* pool = new HostCopyPool();  // never destroyed: its threads live on
    return *pool;
  }
  void copy(void* dst, const void* src, size_t n) {
    char* d = static_cast<char*>(dst);
    const char* s = static_cast<const char*>(src);
    run(n, [d, s](size_t off, size_t len) { memcpy(d + off, s + off, len); });
  }
  // fn(offset, length) over equal parts of [0, n) (64-byte multiples), in parallel
  void run(size_t n, std::function<void(size_t, size_t)> fn) {
    std::lock_guard<std::mutex> one(call_m_);  // one job at a time (builders on many threads)
    // a forked child inherits this object but not the worker threads: work alone there
    const size_t nw = getpid() == pid_ ? workers_.size() : 0;
    const int parts = (int)std::min<size_t>(nw + 1, std::max<size_t>(1, n >> 20));
    if (parts <= 1) {
      if (n) fn(0, n);
      return;
    }
    const size_t per = (n / parts + 63) & ~size_t(63);
    {
      std::lock_guard<std::mutex> lk(m_);
      fn_ = std::move(fn);
      n_ = n;
      per_ = per;
      parts_ = parts;
      pending_ = parts - 1;
      ++gen_;
    }
    cv_.notify_all();
    fn_(0, std::min(per, n));
    std::unique_lock<std::mutex> lk(m_);
    done_.wait(lk, [&] { return pending_ == 0; });
  }

 private:
  HostCopyPool() : pid_(getpid()) {
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const int nw = (int)std::min(15u, hw > 1 ? hw - 1 : 0u);
    for (int i = 0; i < nw; ++i) workers_.emplace_back([this, i] { loop(i + 1); });
    for (auto& t : workers_) t.detach();  // live for the process
  }
  void loop(int part) {
    uint64_t seen = 0;
    for (;;) {
      size_t off, len;
      std::function<void(size_t, size_t)>* fn;
      {
        std::unique_lock<std::mutex> lk(m_);
        cv_.wait(lk, [&] { return gen_ != seen; });
        seen = gen_;
        if (part >= parts_) continue;
        off = per_ * (size_t)part;
        len = off < n_ ? std::min(per_, n_ - off) : 0;
        fn = &fn_;
      }
      if (len) (*fn)(off, len);
      {
        std::lock_guard<std::mutex> lk(m_);
        if (--pending_ == 0) done_.notify_one();
      }
    }
  }
  const pid_t pid_;
  std::vector<std::thread> workers_;
  std::mutex call_m_, m_;
  std::condition_variable cv_, done_;
  std::function<void(size_t, size_t)> fn_;
  size_t n_ = 0, per_ = 0;
  int parts_ = 0, pending_ = 0;
  uint64_t gen_ = 0;
};

// A triangle soup's index array is T[i][k] = 3i + k, i.e. the flat array is 0, 1, 2, ...
// (gen_scene and unshared-vertex exports; geometry.py:206-207). It carries no information,
// so a host mesh whose T is exactly that is not copied: K1 regenerates the indices. Checked
// exactly, in parallel on the host pool.
bool is_soup_indices(const int32_t* T, int64_t n, int64_t nv) {
  if (n < (1 << 16) || nv < 3 * n) return false;
  std::atomic<bool> ok{true};
  HostCopyPool::get().run((size_t)n * 3 * sizeof(int32_t), [&](size_t off, size_t len) {
    const int32_t* t = T + off / 4;
    const int32_t base = (int32_t)(off / 4);
    const size_t m = len / 4;
    bool good = true;
    for (size_t j = 0; j < m && good; j += 4096) {
      const size_t e = std::min(m, j + 4096);
      int32_t bad = 0;
      for (size_t q = j; q < e; ++q) bad |= t[q] ^ (base + (int32_t)q);
      good = bad == 0 && ok.load(std::memory_order_relaxed);
    }
    if (!good) ok.store(false, std::memory_order_relaxed);
  });
  return ok.load();
}

bool is_pageable(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return true;
  }
  return a.type == cudaMemoryTypeUnregistered;
}

// PGRID_PDL: 0 launches the build's kernel chain without programmatic dependent launch, 1 uses
// it for every link, 2 only for the glue kernels (scans, bounds), 3 only for the bulk passes.
int pdl_mode() {
  static const int m = [] {
    const char* e = getenv("PGRID_PDL");
    return e && *e ? atoi(e) : 1;
  }();
  return m;
}

// First launch error of pdl_launch (cudaLaunchKernelEx's return code) since LAUNCHED last ran.
thread_local cudaError_t g_launch_err = cudaSuccess;

// Launch `k` with the programmatic-serialization attribute: its launch is processed while the
// previous kernel on `st` retires instead of after it (the launch latency between links).
// Only for kernels that open with PDL_ENTRY() (griddepcontrol.wait before any global access);
// after a non-kernel stream operation the launch is an ordinary serialised one.
template <typename... KArgs, typename... Args>
void pdl_launch(bool glue, void (*k)(KArgs...), unsigned grid, unsigned block, size_t smem, cudaStream_t st,
                Args&&... args) {
  const int m = pdl_mode();
  const bool on = m == 1 || (m == 2 && glue) || (m == 3 && !glue);
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cfg.attrs = at;
  cfg.numAttrs = on ? 1 : 0;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
  if (e != cudaSuccess && g_launch_err == cudaSuccess) g_launch_err = e;  // reported by LAUNCHED
}

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CU(call)                                                                          \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess)                                                                \
      return fail(PG_CUDA_ERROR, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), \
                  __FILE__, __LINE__);                                                    \
  } while (0)

constexpr int64_t kMaxIds = 4294967295LL;  // gridcore.py:11
constexpr int64_t kMaxScan = 1LL << 30;    // primitives.py:17

size_t align_up(size_t x, size_t a = 256) { return (x + a - 1) / a * a; }

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  int ensure(size_t need) {
    if (need <= bytes) return PG_OK;
    const size_t want = std::max(need, bytes + bytes / 4);  // grow-only, 25% headroom
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    cudaError_t e = cudaMalloc(&p, want);
    if (e != cudaSuccess) {
      p = nullptr;
      return fail(PG_CUDA_ERROR, "cudaMalloc(%zu) failed: %s", want, cudaGetErrorString(e));
    }
    bytes = want;
    return PG_OK;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  template <typename T>
  T* as(size_t byte_off = 0) const {
    return reinterpret_cast<T*>(static_cast<char*>(p) + byte_off);
  }
};

PassPlan make_plan(int key_bits, int max_digit_bits) {
  PassPlan pl{};
  pl.npasses = key_bits <= 0 ? 0 : (key_bits + max_digit_bits - 1) / max_digit_bits;
  int shift = 0;
  for (int i = 0; i < pl.npasses; ++i) {
    // balanced digits: spread key_bits over the passes (e.g. 26 -> 7,7,6,6)
    const int rem_passes = pl.npasses - i;
    const int b = (key_bits - shift + rem_passes - 1) / rem_passes;
    pl.shift[i] = shift;
    pl.bits[i] = b;
    shift += b;
  }
  return pl;
}

// The MSD-first finish (k_bucket_sort): PGRID_LOCAL=0 turns it off (classic LSD + K4);
// PGRID_LOCAL_ITEMS = the mean pairs per bucket the bucket width is chosen for (256: L = 9 at cfg3).
int local_env(const char* name, int dflt) {
  const char* e = getenv(name);
  return e && *e ? atoi(e) : dflt;
}
bool local_on() {
  static const bool on = local_env("PGRID_LOCAL", 1) != 0;
  return on;
}
int local_items() {
  static const int v = std::max(1, local_env("PGRID_LOCAL_ITEMS", 256));
  return v;
}

// Passes over the key's top bits [lo, key_bits) only (the MSD-first finish sorts [0, lo))
PassPlan make_plan_above(int lo, int key_bits, int max_digit_bits) {
  PassPlan pl = make_plan(key_bits - lo, max_digit_bits);
  for (int i = 0; i < pl.npasses; ++i) pl.shift[i] += lo;
  return pl;
}

// Bucket width L of the MSD-first finish, or -1 for the classic LSD + K4 finish: buckets of
// 2^L cells hold about local_items() pairs on average (L <= 11: a bucket is one warp's serial
// work; at least one radix pass above it).
constexpr int kMinLocalBits = 2, kMaxLocalBits = 10;
int local_bits(int key_bits, int64_t ncells, uint64_t no, uint32_t flags) {
  if (!local_on() || (flags & PG_KEEP_STAGES) || key_bits <= kMinLocalBits || no == 0) return -1;
  int L = kMinLocalBits;
  while (L < kMaxLocalBits && L + 1 < key_bits &&
         ((double)no * (double)(1ull << (L + 1)) <= (double)local_items() * ncells))
    ++L;
  return L;
}

int bit_length(uint64_t v) {
  int b = 0;
  while (v >> b) ++b;
  return b;
}

size_t rs_smem_bytes() { return sizeof(RsSmem); }

template <int BITS, bool TABLE>
void launch_scatter_bits(unsigned ntiles, cudaStream_t st, const unsigned* kin, const unsigned* vin, unsigned* ko,
                         unsigned* vo, Count n, int shift, const unsigned* hist, const unsigned* offs, unsigned ld,
                         const unsigned* dtable, const unsigned* kbase) {
  pdl_launch(false, k_radix_scatter<BITS, TABLE>, ntiles, RS_THREADS, rs_smem_bytes(), st, kin, vin, ko, vo, n, shift,
             hist, offs, ld, dtable, kbase);
}

// K4L over cell tiles of 8 buckets of 2^lbits cells (lbits 2..10)
template <int L>
int launch_bucket_sort_l(unsigned tiles, cudaStream_t st, const unsigned* keys, const unsigned* vals, Count cno,
                         unsigned ncells, const unsigned* kb, unsigned* G, unsigned* O, int vals_ascend) {
  // the shared-memory carveout preference (5 CTAs/SM at 28 KB each) and, for tiles above 48 KB
  // (only in BK_CAP variants), the opt-in: once per device
  static std::atomic<unsigned long long> done{0};
  int dev = 0;
  CU(cudaGetDevice(&dev));
  const unsigned long long bit = 1ull << (dev & 63);
  if (!(done.load() & bit)) {
    if constexpr (bk_smem_bytes(L) > 48 * 1024)
      CU(cudaFuncSetAttribute(k_bucket_sort<L>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bk_smem_bytes(L)));
    CU(cudaFuncSetAttribute(k_bucket_sort<L>, cudaFuncAttributePreferredSharedMemoryCarveout,
                            (int)cudaSharedmemCarveoutMaxShared));
    done.fetch_or(bit);
  }
  pdl_launch(false, k_bucket_sort<L>, tiles, BK_THREADS, bk_smem_bytes(L), st, keys, vals, cno, ncells, kb, G, O,
             vals_ascend);
  return PG_OK;
}
int launch_bucket_sort(int lbits, unsigned tiles, cudaStream_t st, const unsigned* keys, const unsigned* vals,
                       Count cno, unsigned ncells, const unsigned* kb, unsigned* G, unsigned* O, bool vals_ascend) {
  switch (lbits) {
#define PG_BK(l) \
  case l: return launch_bucket_sort_l<l>(tiles, st, keys, vals, cno, ncells, kb, G, O, vals_ascend ? 1 : 0);
    PG_BK(2) PG_BK(3) PG_BK(4) PG_BK(5) PG_BK(6) PG_BK(7) PG_BK(8) PG_BK(9) PG_BK(10)
#undef PG_BK
    default: return fail(PG_INVARIANT_ERROR, "bucket width 2^%d", lbits);
  }
}

// bit-field digits of 1..9 bits, or (dtable != null) slab-table digits of 1..4 bits
void launch_radix_scatter(int bits, unsigned ntiles, cudaStream_t st, const unsigned* kin, const unsigned* vin,
                          unsigned* ko, unsigned* vo, Count n, int shift, const unsigned* hist,
                          const unsigned* offs, unsigned ld, const unsigned* dtable = nullptr,
                          const unsigned* kbase = nullptr) {
  if (dtable) {
    switch (bits) {
#define PG_CASE(B) \
  case B:          \
    launch_scatter_bits<B, true>(ntiles, st, kin, vin, ko, vo, n, shift, hist, offs, ld, dtable, kbase); break;
      PG_CASE(1) PG_CASE(2) PG_CASE(3) PG_CASE(4)
#undef PG_CASE
      default: break;
    }
    return;
  }
  switch (bits) {
#define PG_CASE(B) \
  case B:          \
    launch_scatter_bits<B, false>(ntiles, st, kin, vin, ko, vo, n, shift, hist, offs, ld, nullptr, nullptr); break;
    PG_CASE(1) PG_CASE(2) PG_CASE(3) PG_CASE(4) PG_CASE(5) PG_CASE(6) PG_CASE(7) PG_CASE(8) PG_CASE(9)
#undef PG_CASE
    default: break;
  }
}

template <int BITS>
cudaError_t set_scatter_smem() {
  cudaError_t e = cudaFuncSetAttribute(k_radix_scatter<BITS, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)rs_smem_bytes());

  if (e != cudaSuccess || BITS > 4) return e;
  return cudaFuncSetAttribute(k_radix_scatter<(BITS > 4 ? 1 : BITS), true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)rs_smem_bytes());
}

bool packed0_on() {
  static const bool on = [] {
    const char* e = getenv("PGRID_PACKED0");
    return !e || *e != '0';
  }();
  return on;
}

// PGRID_SYNC_DEBUG=1: synchronise after every launch so a fault names its kernel.
bool sync_debug() {
  static const bool on = [] {
    const char* e = getenv("PGRID_SYNC_DEBUG");
    return e && *e && *e != '0';
  }();
  return on;
}

// PGRID_KTIMES=1: an event after every launch, so pg_kernel_times can report per-kernel
// device times of the last pg_count / pg_finish (profiling aid; off by default).
int g_ktimes = -1;  // -1: from the environment; 0/1: set by pg_kernel_timing
bool ktimes_on() {
  if (g_ktimes < 0) {
    const char* e = getenv("PGRID_KTIMES");
    g_ktimes = (e && *e && *e != '0') ? 1 : 0;
  }
  return g_ktimes == 1;
}
struct KTimer {
  std::vector<std::pair<const char*, cudaEvent_t>> ev;
  size_t used = 0;
  cudaEvent_t next(const char* name) {
    if (used == ev.size()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      ev.push_back({name, e});
    }
    ev[used].first = name;
    return ev[used++].second;
  }
};
thread_local KTimer g_kt;
void ktimer_reset(cudaStream_t st) {
  if (!ktimes_on()) return;
  g_kt.used = 0;
  cudaEventRecord(g_kt.next("start"), st);
}

#define LAUNCHED(name, st)                                                                         \
  do {                                                                                             \
    const cudaError_t le_ = g_launch_err;                                                          \
    g_launch_err = cudaSuccess;                                                                    \
    if (le_ != cudaSuccess)                                                                        \
      return fail(PG_CUDA_ERROR, "launch of %s failed: %s", name, cudaGetErrorString(le_));       \
    CU(cudaGetLastError());                                                                        \
    if (ktimes_on()) cudaEventRecord(g_kt.next(name), st);                                         \
    if (sync_debug()) {                                                                            \
      cudaError_t e2_ = cudaStreamSynchronize(st);                                                 \
      if (e2_ != cudaSuccess)                                                                      \
        return fail(PG_CUDA_ERROR, "kernel %s failed: %s", name, cudaGetErrorString(e2_));         \
    }                                                                                              \
  } while (0)

}  // namespace

struct pg_builder {
  int device = 0;
  cudaEvent_t ev[8] = {};
  unsigned long long* h_scalars = nullptr;  // pinned: [0] NO, [1] error flags
  // inputs staged on device for PG_HOST_INPUT
  DevBuf in_v, in_t;
  // pageable host inputs: a ring of page-locked staging chunks, filled by the host copy pool
  // while the previous chunks' DMA runs (stage_ev[i] = chunk i's copy done)
  static constexpr int kStageBufs = 4;
  static constexpr size_t kStageBytes = 16u << 20;
  unsigned char* stage_h[kStageBufs] = {};
  cudaEvent_t stage_ev[kStageBufs] = {};
  int stage_next = 0;
  // page-locked V of an implicit soup: copied in chunks on a copy stream, K1 launched per
  // chunk as it lands (chunk_ev[i] = chunk i copied)
  static constexpr int kMaxChunks = 32;
  cudaStream_t cst = nullptr;
  cudaEvent_t chunk_ev[kMaxChunks] = {};
  // K1 outputs / scratch
  DevBuf rec, k1_sync;
  // pair buffers and sort scratch
  DevBuf pairs, sort_sync, stage, stage0, gbuf, obuf, cells;
  DevBuf send;  // fused dispatch: tile bounds, look-back status, ticket
  // state of the last pg_count
  bool counted = false;
  bool deferred = false;  // PG_DEFER: NO is on the device only; `no` holds the capacity
  int64_t n = 0;
  uint64_t no = 0;
  int64_t ncells = 0;
  int dims[3] = {1, 1, 1};
  int key_bits = 0;
  bool stages_kept = false;
  size_t stage_sec = 0;  // offset of the kept values inside `stage`
  bool k1_timed = false;  // ev[5]..ev[6] bracket K1 of the last pg_count
  int launches = 0;
  const unsigned* sorted_keys = nullptr;
  const unsigned* tile_pre = nullptr;  // K1 tile prefixes of the last pg_count
  unsigned long long* d_total = nullptr;  // device NO of the last count
  // sync-free build (pg_build_async): private stream, events, and the captured CUDA graph
  cudaStream_t gst = nullptr;
  cudaEvent_t g_in = nullptr, g_out = nullptr;
  cudaGraphExec_t gexec = nullptr;
  std::vector<unsigned char> gkey;
  uint64_t g_cap = 0;
  int glaunches = 0;
  // ray casting (pg_dda_prepare / pg_dda_cast): prepared triangles + staging
  DevBuf tris, dda_err, dda_grid, dda_rays, dda_out;
  int64_t dda_ntri = -1;
  // OBJ ingestion (pg_load_obj / pg_obj_fetch)
  DevBuf obj_bytes, obj_lines, obj_info, obj_pre, obj_scan, obj_v, obj_t;
  int64_t obj_nv = -1, obj_nt = 0;
  // inputs of the last count (for the inverted-box resolution on the error path)
  const double* last_V = nullptr;
  const int32_t* last_T = nullptr;
  DevSpec last_ds{};
  // positive-count inverted boxes of the last count (two inverted axes): their pairs are
  // rewritten with the reference's cells after the expansion (k_inverted_pairs). inv holds
  // [count u32][err u32][pad][list of triangle ids]
  bool inv_fix = false;
  DevBuf inv;
  int64_t stats[6] = {};  // PG_STATS: raw statistics of the last count (pg_count_stats)
  bool phases_ready = false;  // ev[0..4] bracket the phases of the last pg_finish
  // G / O of the last pg_build_async (pg_build_wait's host-counted rebuild)
  uint32_t* g_G = nullptr;
  uint32_t* g_O = nullptr;
  // pg_partition_counts -> pg_partition_send
  int64_t part_n = -1;
  int part_bits = 0;
};

extern "C" {

const char* pg_last_error(void) { return g_err.c_str(); }

int pg_builder_create(int device, pg_builder** out) {
  if (!out) return fail(PG_INVARIANT_ERROR, "null out pointer");
  CU(cudaSetDevice(device));
  pg_builder* b = new pg_builder();
  b->device = device;
  for (auto& e : b->ev) CU(cudaEventCreate(&e));
  CU(cudaMallocHost(&b->h_scalars, 4 * sizeof(unsigned long long)));
  CU(cudaFuncSetAttribute(k_boxes_count, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(K1Smem)));
  CU(cudaFuncSetAttribute(k_pairs_emit, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(PeSmem)));
  CU(set_scatter_smem<1>()); CU(set_scatter_smem<2>()); CU(set_scatter_smem<3>());
  CU(set_scatter_smem<4>()); CU(set_scatter_smem<5>()); CU(set_scatter_smem<6>());
  CU(set_scatter_smem<7>()); CU(set_scatter_smem<8>()); CU(set_scatter_smem<9>());
  for (auto f : {k_partition_send<1>, k_partition_send<2>, k_partition_send<3>, k_partition_send<4>})
    CU(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rs_smem_bytes()));
#if PGRID_FUSED_DISPATCH
  for (auto f : {k_pairs_send<1>, k_pairs_send<2>, k_pairs_send<3>, k_pairs_send<4>})
    CU(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(SendSmem)));
  CU(cudaFuncSetAttribute(k_coarse_from_boxes, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * PLAN_MAX_BUCKETS));
  CU(cudaFuncSetAttribute(k_coarse_big, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * PLAN_MAX_BUCKETS));
#endif
  *out = b;
  return PG_OK;
}

void pg_builder_destroy(pg_builder* b) {
  if (!b) return;
  cudaSetDevice(b->device);
  for (auto& e : b->ev)
    if (e) cudaEventDestroy(e);
  if (b->h_scalars) cudaFreeHost(b->h_scalars);
  for (int i = 0; i < pg_builder::kStageBufs; ++i) {
    if (b->stage_ev[i]) cudaEventSynchronize(b->stage_ev[i]), cudaEventDestroy(b->stage_ev[i]);
    if (b->stage_h[i]) cudaFreeHost(b->stage_h[i]);
  }
  for (auto& e : b->chunk_ev)
    if (e) cudaEventDestroy(e);
  if (b->cst) cudaStreamSynchronize(b->cst), cudaStreamDestroy(b->cst);
  if (b->gexec) cudaGraphExecDestroy(b->gexec);
  if (b->g_in) cudaEventDestroy(b->g_in);
  if (b->g_out) cudaEventDestroy(b->g_out);
  if (b->gst) cudaStreamDestroy(b->gst);
  for (DevBuf* d : {&b->in_v, &b->in_t, &b->rec, &b->k1_sync, &b->pairs, &b->sort_sync, &b->stage, &b->stage0,
                    &b->gbuf, &b->obuf, &b->cells, &b->send})
    d->release();
  delete b;
}

int pg_host_register(void* ptr, uint64_t bytes) {
  if (!ptr || !bytes) return PG_OK;
  CU(cudaHostRegister(ptr, bytes, cudaHostRegisterDefault));
  return PG_OK;
}

int pg_host_alloc(uint64_t bytes, void** out) {
  if (!out) return fail(PG_INVARIANT_ERROR, "null out pointer");
  *out = nullptr;
  if (!bytes) return PG_OK;
  CU(cudaHostAlloc(out, bytes, cudaHostAllocDefault));
  return PG_OK;
}

int pg_host_free(void* ptr) {
  if (ptr) CU(cudaFreeHost(ptr));
  return PG_OK;
}

int pg_host_unregister(void* ptr) {
  if (!ptr) return PG_OK;
  CU(cudaHostUnregister(ptr));
  return PG_OK;
}

int pg_last_launch_count(pg_builder* b) { return b ? b->launches : 0; }

namespace {

// Validation + builder state for a build of (n triangles, spec); fills the device spec.
// Host -> device copy of caller memory. Page-locked sources go straight to the DMA engine.
// Pageable ones (a plain numpy array, the reference caller's case) would make the driver stage
// them at a few GB/s; instead the host copy pool fills a ring of page-locked 16 MB chunks in
// parallel while the previous chunks are in flight, so host copy and PCIe transfer overlap.
int h2d(pg_builder* b, void* dst, const void* src, size_t bytes, cudaStream_t st) {
  if (!bytes) return PG_OK;
  // (small pageable copies: the driver's own staging is fine, and cheaper than the ring's setup)
  if (bytes < pg_builder::kStageBytes || !is_pageable(src)) {
    CU(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st));
    return PG_OK;
  }
  for (int i = 0; i < pg_builder::kStageBufs; ++i) {
    if (!b->stage_h[i]) {
      CU(cudaHostAlloc(reinterpret_cast<void**>(&b->stage_h[i]), pg_builder::kStageBytes, cudaHostAllocDefault));
      CU(cudaEventCreateWithFlags(&b->stage_ev[i], cudaEventDisableTiming));
      CU(cudaEventRecord(b->stage_ev[i], st));
    }
  }
  HostCopyPool& pool = HostCopyPool::get();
  for (size_t off = 0; off < bytes; off += pg_builder::kStageBytes) {
    const size_t len = std::min(pg_builder::kStageBytes, bytes - off);
    const int k = b->stage_next;
    b->stage_next = (k + 1) % pg_builder::kStageBufs;
    CU(cudaEventSynchronize(b->stage_ev[k]));  // that chunk's previous DMA has landed
    pool.copy(b->stage_h[k], static_cast<const char*>(src) + off, len);
    CU(cudaMemcpyAsync(static_cast<char*>(dst) + off, b->stage_h[k], len, cudaMemcpyHostToDevice, st));
    CU(cudaEventRecord(b->stage_ev[k], st));
  }
  return PG_OK;
}

// late_ncells: the host-counted path reports ncells > 2^30 after the count checks, where the
// reference does (its G scan, builders.py:130, runs last); the device-count paths check it here.
int count_setup(pg_builder* b, int64_t nv, int64_t n, const pg_spec* spec, DevSpec& ds, bool late_ncells = false) {
  b->counted = false;
  b->deferred = false;
  b->inv_fix = false;
  b->stages_kept = false;
  b->k1_timed = false;
  b->launches = 0;
  if (n < 0 || nv < 0) return fail(PG_INVARIANT_ERROR, "negative sizes");
  for (int k = 0; k < 3; ++k)
    if (spec->dims[k] < 1) return fail(PG_INVARIANT_ERROR, "dims must be three positive integers");
  int64_t ncells = 1;
  for (int k = 0; k < 3; ++k) {
    ncells *= spec->dims[k];
    if (ncells > kMaxIds) return fail(PG_SIZE_ERROR, "cells exceed 32-bit id space");
  }
  // The reference raises SizeError once the G scan sees more than 2^30 cells
  // (primitives.py:29-31 via builders.py:130); every successful build has ncells <= 2^30.
  if (ncells > kMaxScan && !late_ncells)
    return fail(PG_SIZE_ERROR, "array of %lld elements exceeds the scan size limit", (long long)ncells);
  if (n > kMaxScan) return fail(PG_SIZE_ERROR, "%lld triangles exceed the scan size limit", (long long)n);
  for (int k = 0; k < 3; ++k) {
    ds.lo[k] = spec->lo[k];
    ds.hi[k] = spec->hi[k];
    ds.cell[k] = spec->cell[k];
    ds.rcell[k] = 1.0 / spec->cell[k];
    ds.dims[k] = (int)spec->dims[k];
    b->dims[k] = (int)spec->dims[k];
  }
  b->n = n;
  b->ncells = ncells;
  b->key_bits = bit_length((uint64_t)(ncells - 1));  // builders.py:124
  return PG_OK;
}

// K1 + cross-tile scan on device-resident V/T (n >= 1); NO and the error flags are copied
// to the pinned b->h_scalars asynchronously (read them after the stream is synchronised).
// V chunks of an implicit soup copied on b->cst: chunk i holds triangles [ch[i], ch[i + 1])
// (multiples of K1_TILE) and b->chunk_ev[i] marks its arrival
struct Chunks {
  int count = 0;
  int64_t tri[pg_builder::kMaxChunks + 1];
};

int count_enqueue(pg_builder* b, const double* dV, int64_t nv, const int32_t* dT, int64_t n, const DevSpec& ds,
                  cudaStream_t st, bool readback = true, const Chunks* chunks = nullptr) {
  const unsigned ntiles = (unsigned)((n + K1_TILE - 1) / K1_TILE);
  int rc;
  b->last_V = dV;
  b->last_T = dT;
  b->last_ds = ds;
  if ((rc = b->rec.ensure((size_t)n * sizeof(uint4)))) return rc;
  // K1 area: [tile_sum u64 x ntiles][tile_pre u32 x ntiles][total u64][err u32][pad]
  const size_t ts_bytes = align_up((size_t)ntiles * 8), tp_bytes = align_up((size_t)ntiles * 4);
  if ((rc = b->k1_sync.ensure(ts_bytes + tp_bytes + 256))) return rc;
  unsigned long long* tile_sum = b->k1_sync.as<unsigned long long>();
  unsigned* tile_pre = b->k1_sync.as<unsigned>(ts_bytes);
  // [total u64][err u32][pad u32]: one 16-byte copy lands them in h_scalars[0] and [1]
  unsigned long long* total = b->k1_sync.as<unsigned long long>(ts_bytes + tp_bytes);
  unsigned* err = b->k1_sync.as<unsigned>(ts_bytes + tp_bytes + 8);
  b->tile_pre = tile_pre;
  b->d_total = total;
  CU(cudaMemsetAsync(total, 0, 16, st));
  CU(cudaEventRecord(b->ev[5], st));
  // TMA bulk staging needs 16-byte aligned sources
  const int bulk_ok = ((reinterpret_cast<uintptr_t>(dV) | reinterpret_cast<uintptr_t>(dT)) & 15) == 0;
  if (chunks) {
    // K1 on each chunk as soon as its copy has landed (the copy of the next overlaps it)
    for (int i = 0; i < chunks->count; ++i) {
      const unsigned t0 = (unsigned)(chunks->tri[i] / K1_TILE);
      const unsigned t1 = (unsigned)((chunks->tri[i + 1] + K1_TILE - 1) / K1_TILE);
      CU(cudaStreamWaitEvent(st, b->chunk_ev[i], 0));
      if (t1 > t0)
        k_boxes_count<<<t1 - t0, K1_THREADS, sizeof(K1Smem), st>>>(dV, nv, nullptr, n, ds, bulk_ok, b->rec.as<uint4>(),
                                                                  tile_sum, err, t0);
      LAUNCHED("k_boxes_count", st);
    }
  } else {
    k_boxes_count<<<ntiles, K1_THREADS, sizeof(K1Smem), st>>>(dV, nv, reinterpret_cast<const int*>(dT), n, ds,
                                                              bulk_ok, b->rec.as<uint4>(), tile_sum, err);
    LAUNCHED("k_boxes_count", st);
  }
  // every CTA of the many-CTA scan re-reads the sums before its range (ntiles^2 / 2048 words
  // in all): for up to 256K tiles (134M triangles) that is <= 256 MB of L2 reads; beyond, one CTA
  if (ntiles <= (1u << 18))
    pdl_launch(true, k_scan_tile_sums_mc, (ntiles + MS_PER - 1) / MS_PER, MS_THREADS, 0, st, tile_sum, ntiles,
               tile_pre, total);
  else
    pdl_launch(true, k_scan_tile_sums, 1, TS_THREADS, 0, st, tile_sum, ntiles, tile_pre, total);
  LAUNCHED("k_scan_tile_sums", st);
  CU(cudaEventRecord(b->ev[6], st));
  b->launches = 2;
  b->k1_timed = true;
  if (readback) CU(cudaMemcpyAsync(&b->h_scalars[0], total, 16, cudaMemcpyDeviceToHost, st));
  return PG_OK;
}

// Error path of a count whose K1 flagged an inverted kept box (hi < lo on some axis after
// clipping: an infinite or huge upper corner). Counts the kept triangles and the inverted
// boxes by the sign of their pair count, lists the positive ones (two inverted axes) and, if
// any, checks that every cell the reference computes for them lies in [0, ncells).
struct InvStats {
  unsigned long long kept, inverted, negative, zero, positive;
  bool cells_ok;
};
// K1 ran on an implicit soup (no index array on the device): write it out for the paths
// that gather through T
int materialize_T(pg_builder* b, cudaStream_t st) {
  if (b->last_T) return PG_OK;
  int rc;
  if ((rc = b->in_t.ensure((size_t)b->n * 3 * sizeof(int32_t)))) return rc;
  k_soup_indices<<<1184, 256, 0, st>>>(b->in_t.as<int>(), 3 * b->n);
  CU(cudaGetLastError());
  b->last_T = b->in_t.as<int32_t>();
  return PG_OK;
}

int resolve_inverted(pg_builder* b, InvStats& r) {
  int rc;
  if ((rc = materialize_T(b, nullptr))) return rc;
  const size_t head = 256;
  if ((rc = b->inv.ensure(head + (size_t)std::max<int64_t>(b->n, 1) * 4))) return rc;
  unsigned long long* out = b->inv.as<unsigned long long>(16);
  unsigned* nlist = b->inv.as<unsigned>(0);
  unsigned* err = nlist + 1;
  unsigned* list = b->inv.as<unsigned>(head);
  CU(cudaMemset(b->inv.p, 0, head));
  k_inverted_boxes<<<(unsigned)((b->n + 255) / 256), 256>>>(b->last_V, b->last_T, b->n, b->last_ds, out, list,
                                                            nlist);
  CU(cudaGetLastError());
  unsigned long long h[4];
  CU(cudaMemcpy(h, out, 32, cudaMemcpyDeviceToHost));
  r = {h[0], h[1], h[2], h[3], h[1] - h[2] - h[3], true};
  if (r.positive && !r.negative) {
    k_inverted_pairs<<<(unsigned)std::min<unsigned long long>(r.positive, 4096), 256>>>(
        b->last_V, b->last_T, b->last_ds, nullptr, nullptr, list, nlist, b->ncells, nullptr, nullptr, 0, err);
    CU(cudaGetLastError());
    unsigned he = 0;
    CU(cudaMemcpy(&he, err, 4, cudaMemcpyDeviceToHost));
    r.cells_ok = he == 0;
  }
  return PG_OK;
}

// The reference's cells for the pairs of positive-count inverted boxes, written over K2's
// placeholders in `keys` (generation order); `coarse` (sharded builds) is kept consistent.
int fix_inverted(pg_builder* b, unsigned* keys, cudaStream_t st, unsigned* coarse = nullptr, int coarse_shift = 0) {
  if (!b->inv_fix) return PG_OK;
  unsigned* nlist = b->inv.as<unsigned>(0);
  k_inverted_pairs<<<4096, 256, 0, st>>>(b->last_V, b->last_T, b->last_ds, b->rec.as<uint4>(), b->tile_pre,
                                         b->inv.as<unsigned>(256), nlist, b->ncells, keys, coarse, coarse_shift,
                                         nlist + 1);
  LAUNCHED("k_inverted_pairs", st);
  ++b->launches;
  return PG_OK;
}

// Error checks on the NO / flags that count_enqueue copied back (stream synchronised), in
// the reference's order (builders.py:90-101, 155-160, 125-130): index range (the mesh's own
// check, geometry.py:41-43); a negative pair count (exclusive_sum, primitives.py:22-25);
// NO > 2^32-1 (builders.py:99-100); a zero count among >= 2 kept triangles (mark_boundaries,
// primitives.py:66-72; a lone zero-count triangle gives an empty grid); NO > 2^30
// (inclusive_sum, primitives.py:29-31); cells of two-axis inverted boxes outside [0, ncells)
// (radix_sort_pairs / scatter, primitives.py:102-111, 135-136); ncells > 2^30 (the G scan).
int count_check(pg_builder* b, uint64_t* no_out) {
  uint64_t no = b->h_scalars[0];
  const unsigned errf = (unsigned)(b->h_scalars[1] & 0xffffffffu);
  b->inv_fix = false;
  if (errf & 2u) return fail(PG_INVARIANT_ERROR, "triangle index out of range");
  InvStats r{};
  if (errf & 1u) {
    int rc = resolve_inverted(b, r);
    if (rc) return rc;
    if (r.negative) return fail(PG_INVARIANT_ERROR, "index arrays are non-negative (inverted cell box, negative count)");
  }
  if (no_out) *no_out = no;
  if ((int64_t)no > kMaxIds)
    return fail(PG_SIZE_ERROR, "%llu cell/object pairs exceed 32-bit id space", (unsigned long long)no);
  if (r.zero) {
    if (r.kept >= 2) return fail(PG_INVARIANT_ERROR, "coincident boundary marks (zero-count group?)");
    no = 0;  // the lone kept triangle has no pairs: an empty grid
    if (no_out) *no_out = 0;
  }
  if ((int64_t)no > kMaxScan)
    return fail(PG_SIZE_ERROR, "array of %llu elements exceeds the scan size limit", (unsigned long long)no);
  if (r.positive) {
    if (!r.cells_ok) return fail(PG_INVARIANT_ERROR, "cell of an inverted box outside [0, ncells)");
    b->inv_fix = true;
  }
  if (b->ncells > kMaxScan)
    return fail(PG_SIZE_ERROR, "array of %lld elements exceeds the scan size limit", (long long)b->ncells);
  b->no = no;
  b->counted = true;
  return PG_OK;
}

// PG_STATS: the raw statistics of the count (stream synchronised) instead of a verdict; the
// sharded build sums them over the ranks and decides for the whole mesh.
int count_stats(pg_builder* b, uint64_t* no_out) {
  const uint64_t no = b->h_scalars[0];
  const unsigned errf = (unsigned)(b->h_scalars[1] & 0xffffffffu);
  b->inv_fix = false;
  int64_t* st = b->stats;
  for (int k = 0; k < 6; ++k) st[k] = 0;
  st[0] = (int64_t)no;
  st[1] = (errf & 2u) ? 1 : 0;
  if ((errf & 1u) && !(errf & 2u)) {  // never gather through out-of-range indices
    InvStats r{};
    int rc = resolve_inverted(b, r);
    if (rc) return rc;
    st[2] = (int64_t)r.negative;
    st[3] = (int64_t)r.zero;
    st[4] = (int64_t)r.positive;
    st[5] = (r.positive && !r.negative && !r.cells_ok) ? (int64_t)r.positive : 0;
    b->inv_fix = r.positive && !r.negative && r.cells_ok;
  }
  if (no_out) *no_out = no;
  b->no = no;
  b->counted = true;
  return PG_OK;
}

void drop_graph(pg_builder* b) {
  if (b->gexec) cudaGraphExecDestroy(b->gexec);
  b->gexec = nullptr;
}

}  // namespace

int pg_count(pg_builder* b, const double* V, int64_t nv, const int32_t* T, int64_t n, const pg_spec* spec,
             uint32_t flags, void* stream_, uint64_t* no_out) {
  NvtxRange nvtx_("pg_count");
  if (!b || !spec || !no_out) return fail(PG_INVARIANT_ERROR, "null argument");
  cudaStream_t st = static_cast<cudaStream_t>(stream_);
  CU(cudaSetDevice(b->device));
  drop_graph(b);
  DevSpec ds;
  int rc;
  if ((rc = count_setup(b, nv, n, spec, ds, !(flags & PG_DEFER)))) return rc;
  ktimer_reset(st);
  for (int k = 0; k < 6; ++k) b->stats[k] = 0;
  if (n == 0) {
    if (b->ncells > kMaxScan && !(flags & PG_STATS))
      return fail(PG_SIZE_ERROR, "array of %lld elements exceeds the scan size limit", (long long)b->ncells);
    // an empty mesh (or an empty shard of a sharded build): NO = 0 and no error flags, also
    // on the device for the steps that read them there (pg_peer_put_count, deferred grids)
    if ((rc = b->k1_sync.ensure(256))) return rc;
    b->d_total = b->k1_sync.as<unsigned long long>(0);
    CU(cudaMemsetAsync(b->d_total, 0, 16, st));
    b->h_scalars[0] = 0;
    b->h_scalars[1] = 0;
    b->no = 0;
    *no_out = 0;
    b->counted = true;
    return PG_OK;
  }
  if (!V || !T) return fail(PG_INVARIANT_ERROR, "null mesh arrays");
  const double* dV = V;
  const int32_t* dT = T;
  Chunks chunks;
  if (flags & PG_HOST_INPUT) {
    // V first: a page-locked V streams over PCIe while the host checks T for the implicit soup
    const size_t vbytes = (size_t)nv * 3 * sizeof(double);
    if ((rc = b->in_v.ensure(vbytes))) return rc;
    const bool chunked = vbytes >= (64u << 20) && !is_pageable(V);
    if (chunked) {
      // page-locked V: chunks of ~64 MB (whole K1 tiles of a soup) on the copy stream
      if (!b->cst) {
        CU(cudaStreamCreateWithFlags(&b->cst, cudaStreamNonBlocking));
        for (auto& e : b->chunk_ev) CU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      }
      CU(cudaEventRecord(b->chunk_ev[0], st));  // the copies follow earlier work on st
      CU(cudaStreamWaitEvent(b->cst, b->chunk_ev[0], 0));
      const int64_t per = std::max<int64_t>(K1_TILE, ((int64_t)(64u << 20) / 72 / K1_TILE) * K1_TILE);
      chunks.count = (int)std::min<int64_t>(pg_builder::kMaxChunks, (n + per - 1) / per);
      const int64_t step = ((n + chunks.count - 1) / chunks.count + K1_TILE - 1) / K1_TILE * K1_TILE;
      for (int i = 0; i <= chunks.count; ++i) chunks.tri[i] = std::min<int64_t>(n, (int64_t)i * step);
      for (int i = 0; i < chunks.count; ++i) {
        // rows 3 * tri[i] .. 3 * tri[i + 1]; the last chunk also carries rows past 3n
        const size_t r0 = (size_t)chunks.tri[i] * 3, r1 = i + 1 < chunks.count ? (size_t)chunks.tri[i + 1] * 3 : (size_t)nv;
        if (r1 > r0)
          CU(cudaMemcpyAsync(b->in_v.as<double>() + 3 * r0, V + 3 * r0, (r1 - r0) * 24, cudaMemcpyHostToDevice,
                             b->cst));
        CU(cudaEventRecord(b->chunk_ev[i], b->cst));
      }
    } else if ((rc = h2d(b, b->in_v.p, V, vbytes, st))) {
      return rc;
    }
    dV = b->in_v.as<double>();
    if (is_soup_indices(T, n, nv)) {
      dT = nullptr;  // the implicit soup: 12 bytes per triangle not transferred
    } else {
      if (chunked) {  // an indexed mesh: K1 needs every vertex row
        CU(cudaStreamWaitEvent(st, b->chunk_ev[chunks.count - 1], 0));
        chunks.count = 0;
      }
      if ((rc = b->in_t.ensure((size_t)n * 3 * sizeof(int32_t)))) return rc;
      if ((rc = h2d(b, b->in_t.p, T, (size_t)n * 3 * sizeof(int32_t), st))) return rc;
      dT = b->in_t.as<int32_t>();
    }
  }
  if ((rc = count_enqueue(b, dV, nv, dT, n, ds, st, true, chunks.count ? &chunks : nullptr))) return rc;
  if (flags & PG_DEFER) {
    // no host round trip: the sharded building blocks run on the device count, bounded by
    // the capacity the caller passed in *no_out; pg_count_result checks it afterwards
    const uint64_t cap = *no_out;
    if (cap < 1 || (int64_t)cap > kMaxScan) return fail(PG_INVARIANT_ERROR, "PG_DEFER capacity out of range");
    b->no = cap;
    b->deferred = true;
    b->counted = true;
    return PG_OK;
  }
  CU(cudaStreamSynchronize(st));
  if (flags & PG_STATS) return count_stats(b, no_out);
  return count_check(b, no_out);
}

int pg_count_stats(pg_builder* b, int64_t* out) {
  if (!b || !out) return fail(PG_INVARIANT_ERROR, "null argument");
  if (!b->counted) return fail(PG_STATE_ERROR, "pg_count_stats without a PG_STATS pg_count");
  for (int k = 0; k < 6; ++k) out[k] = b->stats[k];
  return PG_OK;
}

int pg_count_result(pg_builder* b, uint64_t* no_out) {
  if (!b || !no_out) return fail(PG_INVARIANT_ERROR, "null argument");
  if (!b->counted || !b->deferred) return fail(PG_STATE_ERROR, "pg_count_result without a PG_DEFER pg_count");
  CU(cudaSetDevice(b->device));
  const uint64_t cap = b->no;
  const bool inverted = (b->h_scalars[1] & 1u) != 0;
  int rc = count_check(b, no_out);  // reads the scalars copied back by the (synchronised) stream
  b->deferred = true;
  b->counted = rc == PG_OK;
  b->no = cap;
  if (rc) return rc;
  // an accepted inverted box (the reference's empty grid) ran the device steps on the raw
  // count: the results are void, report it like an overflow so the caller rebuilds
  if (inverted) return fail(PG_CAPACITY_ERROR, "deferred build of a mesh with an inverted cell box");
  if (*no_out > cap)
    return fail(PG_CAPACITY_ERROR, "%llu pairs exceed the PG_DEFER capacity %llu", (unsigned long long)*no_out,
                (unsigned long long)cap);
  return PG_OK;
}

namespace {

// LSD passes over (keys0, vals0), ping-ponging with (keys1, vals1); the last pass writes its
// values straight into vals_final (O; null: into the ping-pong buffer, *sorted_vals_out). hist (plan.npasses x 512) must already be filled;
// `counts` holds one [digit][tile] matrix (row stride ld), already filled for pass 0 when
// counts0_ready (K2 emits them).
int run_passes(pg_builder* b, const PassPlan& plan, bool counts0_ready, unsigned* keys0, unsigned* vals0,
               unsigned* keys1, unsigned* vals1, unsigned* vals_final, Count cno, uint64_t cap, unsigned* hist,
               unsigned* counts, cudaStream_t st, const unsigned** sorted_keys_out, unsigned* keys2 = nullptr,
               unsigned* vals2 = nullptr, const unsigned* packed0 = nullptr,
               const unsigned** sorted_vals_out = nullptr) {
  // grids are sized for `cap` pairs; the kernels read the actual count from `cno`
  const unsigned ntiles = (unsigned)((cap + RS_TILE - 1) / RS_TILE);
  const unsigned ld = (ntiles + 3) & ~3u;
  // pass p reads buffer p%2 and writes (p+1)%2; with keys2/vals2 the input (buffer 0) is
  // read-only and passes >= 2 use buffer 2 in its place
  unsigned* kbuf[2] = {keys0, keys1};
  unsigned* vbuf[2] = {vals0, vals1};
  if (sorted_vals_out) *sorted_vals_out = vals0;
  for (int p = 0; p < plan.npasses; ++p) {
    const bool last = p == plan.npasses - 1;
    if (p == 1 && keys2) {
      kbuf[0] = keys2;
      vbuf[0] = vals2;
    }
    unsigned* kin = kbuf[p & 1];
    unsigned* vin = vbuf[p & 1];
    unsigned* ko = kbuf[(p + 1) & 1];
    unsigned* vo = (last && vals_final) ? vals_final : vbuf[(p + 1) & 1];
    // with a packed region (packed0), every pass's tile counts travel two digits per word
    const bool packed = packed0 != nullptr && plan.bits[p] >= 1;
    if (p > 0 || !counts0_ready) {
      const DigitFn dig{plan.shift[p], (1u << plan.bits[p]) - 1u, nullptr};
      pdl_launch(false, k_tile_counts, (ntiles + TC_TILES - 1) / TC_TILES, RS_THREADS, 0, st, kin, cno, dig,
                 1 << plan.bits[p], counts, ld, packed ? const_cast<unsigned*>(packed0) : nullptr);
      LAUNCHED("k_tile_counts", st);
      ++b->launches;
    }
    if (packed) {
      pdl_launch(true, k_scan_tile_counts_packed, 1u << (plan.bits[p] - 1), SC_THREADS, 0, st, packed0, cno, ld,
                 counts, hist + p * kMaxBins);
      LAUNCHED("k_scan_tile_counts", st);
    } else {
      pdl_launch(true, k_scan_tile_counts, 1u << plan.bits[p], SC_THREADS, 0, st, counts, cno, ld,
                 hist + p * kMaxBins);
      LAUNCHED("k_scan_tile_counts", st);
    }
    launch_radix_scatter(plan.bits[p], ntiles, st, kin, vin, ko, vo, cno, plan.shift[p], hist + p * kMaxBins, counts,
                         ld);
    LAUNCHED("k_radix_scatter", st);
    b->launches += 2;
    *sorted_keys_out = ko;
    if (sorted_vals_out) *sorted_vals_out = vo;
  }
  return PG_OK;
}

}  // namespace

int phase_times(pg_builder* b, float* phase_ms);

// Pair expansion -> radix passes -> G for the last counted mesh. `cno` carries the pair
// count (host value, or device pointer for the sync-free build); every buffer and grid is
// sized for `no` = its capacity bound.
int finish_impl(pg_builder* b, uint32_t* G, uint32_t* O, uint32_t flags, cudaStream_t st, float* phase_ms, Count cno,
                uint64_t no) {
  const int64_t ncells = b->ncells;
  // MSD-first finish (lb >= 0): the passes sort by the bucket key >> lb, k_bucket_sort the rest
  const int lb = local_bits(b->key_bits, ncells, no, flags);
  const PassPlan plan = lb >= 0 ? make_plan_above(lb, b->key_bits, kMaxDigitBits) : make_plan(b->key_bits, kMaxDigitBits);
  const unsigned* svals = nullptr;
  int rc;
  unsigned* dG = G;
  unsigned* dO = O;
  if (flags & PG_HOST_OUTPUT) {
    if ((rc = b->gbuf.ensure((size_t)(ncells + 1) * 4))) return rc;
    if ((rc = b->obuf.ensure(std::max<size_t>((size_t)no * 4, 4)))) return rc;
    dG = b->gbuf.as<unsigned>();
    dO = b->obuf.as<unsigned>();
  }
  // pairs: keysA | valsA | keysB | valsB (16 B aligned sections); keysB also holds K2's
  // tile-major first-pass counts before pass 0 runs
  const size_t sec = align_up(std::max<size_t>(std::max<size_t>((size_t)no * 4, 16),
                                               (size_t)((no + RS_TILE - 1) / RS_TILE) * kMaxBins * 4));
  if ((rc = b->pairs.ensure(4 * sec))) return rc;
  unsigned* keysA = b->pairs.as<unsigned>(0);
  unsigned* valsA = b->pairs.as<unsigned>(sec);
  unsigned* keysB = b->pairs.as<unsigned>(2 * sec);
  unsigned* valsB = b->pairs.as<unsigned>(3 * sec);
  // sort scratch: [hist kMaxPasses x 512 (zeroed)][pair-tile bounds][key-tile bounds][tile counts 512 x tiles]
  const unsigned rs_tiles = (unsigned)((no + RS_TILE - 1) / RS_TILE);
  const unsigned k2_tiles = (unsigned)((no + K2_TILE - 1) / K2_TILE);
  const unsigned g_tiles = (unsigned)((ncells + G_TILE - 1) / G_TILE);
  const size_t hist_bytes = align_up(kMaxPasses * kMaxBins * 4);
  const size_t pb_bytes = align_up((size_t)std::max(rs_tiles, k2_tiles) * 8 + 8);
  // cell-tile bounds: K4's tiles, or k_bucket_sort's (8 buckets of 2^lb cells)
  const size_t bk_tiles = lb >= 0 ? (size_t)((ncells + (BK_WARPS << lb) - 1) / (BK_WARPS << lb)) : 0;
  const size_t kb_bytes = align_up((std::max<size_t>(g_tiles, bk_tiles) + 1) * 4);
  if ((rc = b->sort_sync.ensure(hist_bytes + pb_bytes + kb_bytes + (size_t)((rs_tiles + 3) & ~3u) * kMaxBins * 6)))
    return rc;
  unsigned* hist = b->sort_sync.as<unsigned>(0);
  int2* pbounds = b->sort_sync.as<int2>(hist_bytes);
  unsigned* kbounds = b->sort_sync.as<unsigned>(hist_bytes + pb_bytes);
  unsigned* counts = b->sort_sync.as<unsigned>(hist_bytes + pb_bytes + kb_bytes);
  const unsigned ld = (rs_tiles + 3) & ~3u;  // counts row stride

  CU(cudaEventRecord(b->ev[0], st));
  // with radix passes, the pair-tile bounds kernel ahead of K2 clears hist itself
  const bool zero_in_bounds = no > 0 && plan.npasses > 0;
  if (!zero_in_bounds) CU(cudaMemsetAsync(hist, 0, hist_bytes, st));
  const unsigned* sorted = keysA;
  if (no > 0) {
    const unsigned dxu = (unsigned)b->dims[0], dxyu = (unsigned)b->dims[0] * (unsigned)b->dims[1];
    if (plan.npasses == 0 || (flags & PG_KEEP_STAGES)) {
      // pairs in generation order: final when there is no radix pass (vals -> O), and the
      // record= stage dump otherwise
      unsigned* v0 = plan.npasses == 0 ? dO : valsA;
      k_pair_tile_bounds<<<(k2_tiles + 7) / 8, 256, 0, st>>>(b->rec.as<uint4>(), b->tile_pre, b->n, cno, K2_TILE,
                                                            pbounds);
      LAUNCHED("k_pair_tile_bounds", st);
      k_expand_pairs<<<k2_tiles, K2_THREADS, 0, st>>>(b->rec.as<uint4>(), b->tile_pre, b->n, cno, dxu, dxyu, pbounds,
                                                     keysA, v0, 0u, nullptr, 0, 0);
      LAUNCHED("k_expand_pairs", st);
      b->launches += 2;
      if ((rc = fix_inverted(b, keysA, st))) return rc;
      if (flags & PG_KEEP_STAGES) {
        if ((rc = b->stage.ensure(2 * sec))) return rc;
        CU(cudaMemcpyAsync(b->stage.as<unsigned>(0), keysA, no * 4, cudaMemcpyDeviceToDevice, st));
        CU(cudaMemcpyAsync(b->stage.as<unsigned>(sec), v0, no * 4, cudaMemcpyDeviceToDevice, st));
        b->stage_sec = sec;
        b->stages_kept = true;
      }
    }
    if (plan.npasses > 0) {
      // K2 on radix tiles: pairs in generation order + first-pass tile counts
      pdl_launch(true, k_pair_tile_bounds, (rs_tiles + 7) / 8, 256, 0, st, b->rec.as<uint4>(), b->tile_pre, b->n,
                 cno, RS_TILE, pbounds, hist, (unsigned)(hist_bytes / 4));
      LAUNCHED("k_pair_tile_bounds", st);
      // K2 writes its first-pass tile counts straight into the digit-major matrix, two digits
      // per word (the row scan unpacks them): PGRID_PACKED0=0 off
      unsigned* packed0 = (!b->inv_fix && packed0_on() && plan.bits[0] >= 1)
                              ? counts + (size_t)kMaxBins * ld : nullptr;
      pdl_launch(false, k_pairs_emit, rs_tiles, RS_THREADS, sizeof(PeSmem), st, b->rec.as<uint4>(), b->tile_pre, b->n,
                 cno, dxu, dxyu, plan, pbounds, keysA, valsA, counts, ld, packed0);
      LAUNCHED("k_pairs_emit", st);
      b->launches += 2;
      // two-axis inverted boxes: their keys are rewritten, so pass 0 recounts its digits
      if ((rc = fix_inverted(b, keysA, st))) return rc;
      CU(cudaEventRecord(b->ev[1], st));
      if ((rc = run_passes(b, plan, !b->inv_fix, keysA, valsA, keysB, valsB, lb >= 0 ? nullptr : dO, cno, no, hist,
                           counts, st, &sorted, nullptr, nullptr, packed0, &svals)))
        return rc;
    } else {
      CU(cudaEventRecord(b->ev[1], st));
    }
  } else {
    CU(cudaEventRecord(b->ev[1], st));
  }
  CU(cudaEventRecord(b->ev[2], st));
  {
    // searches narrowed with the last pass's digit totals (when a sort ran)
    const int lp = plan.npasses - 1;
    const bool top = lp >= 0 && no > 0 && ncells > 1;
    const unsigned* th = top ? hist + lp * kMaxBins : nullptr;
    const int tsh = top ? plan.shift[lp] : 0, tbins = top ? 1 << plan.bits[lp] : 0;
    if (lb >= 0) {
      const unsigned step = (unsigned)BK_WARPS << lb, tiles = (unsigned)((ncells + step - 1) / step);
      pdl_launch(true, k_key_tile_bounds, (tiles + 1 + 7) / 8, 256, 0, st, sorted, cno, step, (unsigned)ncells,
                 tiles + 1, kbounds, th, tsh, tbins);
      LAUNCHED("k_key_tile_bounds", st);
      // K2's pairs are in generation order: values ascend inside every cell
      if ((rc = launch_bucket_sort(lb, tiles, st, sorted, svals, cno, (unsigned)ncells, kbounds, dG, dO, true)))
        return rc;
      LAUNCHED("k_bucket_sort", st);
      b->launches += 2;
    } else {
      pdl_launch(true, k_key_tile_bounds, (g_tiles + 1 + 7) / 8, 256, 0, st, sorted, cno, G_TILE, (unsigned)ncells,
                 g_tiles + 1, kbounds, th, tsh, tbins);
      LAUNCHED("k_key_tile_bounds", st);
      pdl_launch(false, k_cell_offsets, g_tiles, G_THREADS, 0, st, sorted, cno, (unsigned)ncells, kbounds, dG);
      LAUNCHED("k_cell_offsets", st);
      b->launches += 2;
    }
  }
  b->sorted_keys = sorted;
  CU(cudaEventRecord(b->ev[3], st));
  if (flags & PG_HOST_OUTPUT) {
    CU(cudaMemcpyAsync(G, dG, (size_t)(ncells + 1) * 4, cudaMemcpyDeviceToHost, st));
    if (no) CU(cudaMemcpyAsync(O, dO, no * 4, cudaMemcpyDeviceToHost, st));
  }
  CU(cudaEventRecord(b->ev[4], st));
  b->phases_ready = true;
  if (phase_ms || ((flags & PG_HOST_OUTPUT) && !(flags & PG_ASYNC))) CU(cudaEventSynchronize(b->ev[4]));
  if (phase_ms) return phase_times(b, phase_ms);
  return PG_OK;
}

// The reference's six phases (builders.py:46-54) from the events of the last pg_count +
// pg_finish (their work must have completed).
int phase_times(pg_builder* b, float* phase_ms) {
  float t01 = 0, t12 = 0, t23 = 0, t34 = 0;
  CU(cudaEventElapsedTime(&t01, b->ev[0], b->ev[1]));
  CU(cudaEventElapsedTime(&t12, b->ev[1], b->ev[2]));
  CU(cudaEventElapsedTime(&t23, b->ev[2], b->ev[3]));
  CU(cudaEventElapsedTime(&t34, b->ev[3], b->ev[4]));
  float t_k1 = 0.f;
  if (b->k1_timed) CU(cudaEventElapsedTime(&t_k1, b->ev[5], b->ev[6]));
  phase_ms[0] = t_k1;  // count: K1 device time (callers add their H2D / readback around it)
  phase_ms[1] = 0.f;  // scan: fused into count (K1)
  phase_ms[2] = t01;  // pairgen: tile bounds + K2 (+ first-pass tile counts)
  phase_ms[3] = t12;  // sort: the radix passes
  phase_ms[4] = 0.f;  // rle: fused into finalize (K4)
  phase_ms[5] = t23 + t34;  // finalize: K4 (+ D2H of G/O for host outputs)
  return PG_OK;
}

int pg_finish(pg_builder* b, uint32_t* G, uint32_t* O, uint32_t flags, void* stream_, float* phase_ms) {
  NvtxRange nvtx_("pg_finish");
  if (!b || !b->counted) return fail(PG_STATE_ERROR, "pg_finish without a successful pg_count");
  CU(cudaSetDevice(b->device));
  drop_graph(b);
  if (ktimes_on()) cudaEventRecord(g_kt.next("(host gap)"), static_cast<cudaStream_t>(stream_));
  // after a PG_DEFER count, b->no is the capacity and the kernels read NO from the device
  // (O, host or device, must hold the capacity); pg_count_result validates NO afterwards
  return finish_impl(b, G, O, flags, static_cast<cudaStream_t>(stream_), phase_ms,
                     Count{b->deferred ? b->d_total : nullptr, (unsigned)b->no}, b->no);
}

// Sync-free build on device-resident data: the whole of Alg. 1 is enqueued without reading
// NO back (kernels after K1 take it from device memory; buffers and grids are sized for
// o_capacity). The first call with a given argument set runs eagerly (allocating the
// workspace) and then captures the same enqueue sequence into a CUDA graph; later calls
// with identical arguments replay the graph. Ordering with `stream` is kept with events.
// pg_build_wait() synchronises and reports NO and any error; PG_CAPACITY_ERROR means NO
// exceeded o_capacity (G/O are then invalid: grow O and rebuild).
int pg_build_async(pg_builder* b, const double* V, int64_t nv, const int32_t* T, int64_t n, const pg_spec* spec,
                   uint32_t* G, uint32_t* O, uint64_t o_capacity, void* stream_) {
  NvtxRange nvtx_("pg_build_async");
  if (!b || !spec || !G) return fail(PG_INVARIANT_ERROR, "null argument");
  cudaStream_t st = static_cast<cudaStream_t>(stream_);
  CU(cudaSetDevice(b->device));
  if (!b->gst) {
    CU(cudaStreamCreateWithFlags(&b->gst, cudaStreamNonBlocking));
    CU(cudaEventCreateWithFlags(&b->g_in, cudaEventDisableTiming));
    CU(cudaEventCreateWithFlags(&b->g_out, cudaEventDisableTiming));
  }
  const uint64_t cap = std::max<uint64_t>(std::min<uint64_t>(o_capacity, (uint64_t)kMaxScan), 1);
  // graph key: every argument the enqueue sequence depends on
  std::vector<unsigned char> key(sizeof(pg_spec) + 8 * sizeof(uint64_t));
  {
    const uint64_t k[8] = {(uint64_t)(uintptr_t)V, (uint64_t)nv, (uint64_t)(uintptr_t)T, (uint64_t)n,
                           (uint64_t)(uintptr_t)G, (uint64_t)(uintptr_t)O, cap, 0};
    memcpy(key.data(), spec, sizeof(pg_spec));
    memcpy(key.data() + sizeof(pg_spec), k, sizeof k);
  }
  CU(cudaEventRecord(b->g_in, st));
  CU(cudaStreamWaitEvent(b->gst, b->g_in, 0));
  if (b->gexec && key == b->gkey) {
    CU(cudaGraphLaunch(b->gexec, b->gst));
    b->launches = b->glaunches;
  } else {
    drop_graph(b);
    DevSpec ds;
    int rc;
    if ((rc = count_setup(b, nv, n, spec, ds))) return rc;
    if (n == 0 || !V || !T) return fail(PG_INVARIANT_ERROR, "pg_build_async needs a non-empty device mesh");
    auto enqueue = [&](cudaStream_t s2) -> int {
      int r;
      // NO and the error flags are read back after the build (only the host's post-build
      // check reads them), so K1's scan chains straight into the pair expansion
      if ((r = count_enqueue(b, V, nv, T, n, ds, s2, false))) return r;
      if ((r = finish_impl(b, G, O, 0, s2, nullptr, Count{b->d_total, (unsigned)cap}, cap))) return r;
      CU(cudaMemcpyAsync(&b->h_scalars[0], b->d_total, 16, cudaMemcpyDeviceToHost, s2));
      return PG_OK;
    };
    if ((rc = enqueue(b->gst))) return rc;  // eager run: sizes the workspace
    b->glaunches = b->launches;
    if (!sync_debug()) {
      cudaGraph_t graph = nullptr;
      CU(cudaStreamBeginCapture(b->gst, cudaStreamCaptureModeThreadLocal));
      rc = enqueue(b->gst);
      cudaError_t ec = cudaStreamEndCapture(b->gst, &graph);
      if (rc) return rc;
      if (ec != cudaSuccess) return fail(PG_CUDA_ERROR, "graph capture failed: %s", cudaGetErrorString(ec));
      cudaError_t ei = cudaGraphInstantiate(&b->gexec, graph, 0);
      cudaGraphDestroy(graph);
      if (ei != cudaSuccess) {
        b->gexec = nullptr;
        return fail(PG_CUDA_ERROR, "graph instantiate failed: %s", cudaGetErrorString(ei));
      }
      b->gkey = key;
    }
  }
  b->g_cap = cap;
  b->g_G = G;
  b->g_O = O;
  CU(cudaEventRecord(b->g_out, b->gst));
  CU(cudaStreamWaitEvent(st, b->g_out, 0));
  return PG_OK;
}

int pg_build_wait(pg_builder* b, uint64_t* no_out) {
  NvtxRange nvtx_("pg_build_wait");
  if (!b || !b->gst) return fail(PG_STATE_ERROR, "no asynchronous build in flight");
  CU(cudaSetDevice(b->device));
  CU(cudaStreamSynchronize(b->gst));
  int rc = count_check(b, no_out);
  if (rc) return rc;
  if (b->no > b->g_cap)
    return fail(PG_CAPACITY_ERROR, "NO = %llu exceeds the O capacity %llu", (unsigned long long)b->no,
                (unsigned long long)b->g_cap);
  if (b->inv_fix) {
    // boxes inverted on two axes: the device-count build left placeholders for their pairs;
    // finish again from the host-checked count (K1's records are current), then the graph is
    // re-captured by the next call
    drop_graph(b);
    if ((rc = finish_impl(b, b->g_G, b->g_O, 0, b->gst, nullptr, Count{nullptr, (unsigned)b->no}, b->no))) return rc;
    CU(cudaStreamSynchronize(b->gst));
  }
  return PG_OK;
}

// The paper's comparison builders on the GPU (builders.py:172-231): after pg_count,
// algo 1 = "sorted" (per-object pair generation + the same radix/G tail), algo 2 = "compact"
// (per-cell counters, scan, slot claims, per-cell canonical sort). Same G/O as pg_finish.
int pg_finish_baseline(pg_builder* b, int algo, uint32_t* G, uint32_t* O, uint32_t flags, void* stream_,
                       float* phase_ms, uint64_t* max_task_work) {
  NvtxRange nvtx_("pg_finish_baseline");
  if (!b || !b->counted) return fail(PG_STATE_ERROR, "pg_finish_baseline without a successful pg_count");
  if (b->deferred) return fail(PG_STATE_ERROR, "pg_finish_baseline after a PG_DEFER count");
  if (algo != 1 && algo != 2) return fail(PG_INVARIANT_ERROR, "algo must be 1 (sorted) or 2 (compact)");
  // the reference's per-object walks (_ckernels.pyx:53-109) skip a box inverted on two axes
  // while its count says otherwise: its pairs are uninitialised memory there (np.empty)
  if (b->inv_fix)
    return fail(PG_INVARIANT_ERROR, "cell box inverted on two axes: undefined in the reference's %s builder",
                algo == 1 ? "sorted" : "compact");
  cudaStream_t st = static_cast<cudaStream_t>(stream_);
  CU(cudaSetDevice(b->device));
  drop_graph(b);
  const uint64_t no = b->no;
  const int64_t ncells = b->ncells;
  int rc;
  unsigned* dG = G;
  unsigned* dO = O;
  if (flags & PG_HOST_OUTPUT) {
    if ((rc = b->gbuf.ensure((size_t)(ncells + 1) * 4))) return rc;
    if ((rc = b->obuf.ensure(std::max<size_t>((size_t)no * 4, 4)))) return rc;
    dG = b->gbuf.as<unsigned>();
    dO = b->obuf.as<unsigned>();
  }
  const unsigned dxu = (unsigned)b->dims[0], dxyu = (unsigned)b->dims[0] * (unsigned)b->dims[1];
  const unsigned tgrid = (unsigned)((b->n + 255) / 256);
  CU(cudaEventRecord(b->ev[0], st));
  if (algo == 1) {
    const PassPlan plan = make_plan(b->key_bits, kMaxDigitBits);
    const size_t sec = align_up(std::max<size_t>((size_t)no * 4, 16));
    if ((rc = b->pairs.ensure(4 * sec + 256))) return rc;
    unsigned* kA = b->pairs.as<unsigned>(0);
    unsigned* vA = b->pairs.as<unsigned>(sec);
    unsigned* kB = b->pairs.as<unsigned>(2 * sec);
    unsigned* vB = b->pairs.as<unsigned>(3 * sec);
    unsigned* dmax = b->pairs.as<unsigned>(4 * sec);
    const unsigned rs_tiles = (unsigned)((no + RS_TILE - 1) / RS_TILE);
    const unsigned g_tiles = (unsigned)((ncells + G_TILE - 1) / G_TILE);
    const size_t hist_bytes = align_up(kMaxPasses * kMaxBins * 4), kb_bytes = align_up((size_t)(g_tiles + 1) * 4);
    if ((rc = b->sort_sync.ensure(hist_bytes + kb_bytes + (size_t)((rs_tiles + 3) & ~3u) * kMaxBins * 4))) return rc;
    unsigned* hist = b->sort_sync.as<unsigned>(0);
    unsigned* kbounds = b->sort_sync.as<unsigned>(hist_bytes);
    unsigned* counts = b->sort_sync.as<unsigned>(hist_bytes + kb_bytes);
    CU(cudaMemsetAsync(dmax, 0, 4, st));
    if (b->n) {
      k_pairgen_per_object<<<tgrid, 256, 0, st>>>(b->rec.as<uint4>(), b->tile_pre, b->n, (unsigned)no, dxu, dxyu,
                                                  kA, plan.npasses ? vA : dO, dmax);
      LAUNCHED("k_pairgen_per_object", st);
    }
    CU(cudaEventRecord(b->ev[1], st));
    const unsigned* sorted = kA;
    if (no && plan.npasses) {
      CU(cudaMemsetAsync(hist, 0, hist_bytes, st));
      if ((rc = run_passes(b, plan, false, kA, vA, kB, vB, dO, Count{nullptr, (unsigned)no}, no, hist, counts, st,
                           &sorted)))
        return rc;
    }
    CU(cudaEventRecord(b->ev[2], st));
    k_key_tile_bounds<<<(g_tiles + 1 + 7) / 8, 256, 0, st>>>(sorted, Count{nullptr, (unsigned)no}, G_TILE,
                                                            (unsigned)ncells, g_tiles + 1, kbounds);
    LAUNCHED("k_key_tile_bounds", st);
    k_cell_offsets<<<g_tiles, G_THREADS, 0, st>>>(sorted, Count{nullptr, (unsigned)no}, (unsigned)ncells, kbounds, dG);
    LAUNCHED("k_cell_offsets", st);
    CU(cudaEventRecord(b->ev[3], st));
    unsigned hm = 0;
    CU(cudaMemcpyAsync(&hm, dmax, 4, cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    if (max_task_work) *max_task_work = hm;
  } else {
    // cells: [counts / cursors u32 x ncells][big-segment list u32 x ncells][tile sums][tile prefixes][scalars]
    const unsigned xtiles = (unsigned)((ncells + XS_TILE - 1) / XS_TILE);
    const size_t cbytes = align_up((size_t)ncells * 4);
    const size_t need = 2 * cbytes + align_up((size_t)xtiles * 8) + align_up((size_t)xtiles * 4) + 256;
    if ((rc = b->cells.ensure(need))) return rc;
    unsigned* cnt = b->cells.as<unsigned>(0);
    unsigned* big = b->cells.as<unsigned>(cbytes);
    unsigned long long* tsum = b->cells.as<unsigned long long>(2 * cbytes);
    unsigned* tpre = b->cells.as<unsigned>(2 * cbytes + align_up((size_t)xtiles * 8));
    unsigned* scal = b->cells.as<unsigned>(2 * cbytes + align_up((size_t)xtiles * 8) + align_up((size_t)xtiles * 4));
    unsigned long long* total = reinterpret_cast<unsigned long long*>(scal + 2);
    CU(cudaMemsetAsync(cnt, 0, (size_t)ncells * 4, st));
    CU(cudaMemsetAsync(scal, 0, 16, st));
    if (b->n) {
      k_compact_walk<false><<<tgrid, 256, 0, st>>>(b->rec.as<uint4>(), b->tile_pre, b->n, (unsigned)no, dxu, dxyu,
                                                   cnt, nullptr, scal + 1);
      LAUNCHED("k_compact_walk<count>", st);
    }
    CU(cudaEventRecord(b->ev[1], st));
    k_tile_reduce<<<xtiles, XS_THREADS, 0, st>>>(cnt, ncells, tsum);
    LAUNCHED("k_tile_reduce", st);
    k_scan_tile_sums<<<1, TS_THREADS, 0, st>>>(tsum, xtiles, tpre, total);
    LAUNCHED("k_scan_tile_sums", st);
    k_tile_scan_apply<<<xtiles, XS_THREADS, 0, st>>>(cnt, ncells, tpre, total, dG);
    LAUNCHED("k_tile_scan_apply", st);
    CU(cudaMemcpyAsync(cnt, dG, (size_t)ncells * 4, cudaMemcpyDeviceToDevice, st));  // cursors = G
    CU(cudaEventRecord(b->ev[2], st));
    if (b->n) {
      k_compact_walk<true><<<tgrid, 256, 0, st>>>(b->rec.as<uint4>(), b->tile_pre, b->n, (unsigned)no, dxu, dxyu,
                                                  cnt, dO, nullptr);
      LAUNCHED("k_compact_walk<fill>", st);
    }
    k_sort_segments_small<<<(unsigned)((ncells + 255) / 256), 256, 0, st>>>(dG, (unsigned)ncells, dO, big, scal);
    LAUNCHED("k_sort_segments_small", st);
    unsigned hsc[2] = {0, 0};
    CU(cudaMemcpyAsync(hsc, scal, 8, cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    const unsigned hb = hsc[0];
    if (hb) {
      k_sort_segments_big<<<hb, 1024, 0, st>>>(dG, big, scal, dO);
      LAUNCHED("k_sort_segments_big", st);
    }
    CU(cudaEventRecord(b->ev[3], st));
    if (max_task_work) *max_task_work = hsc[1];  // the largest per-object walk (builders.py:228)
  }
  if (flags & PG_HOST_OUTPUT) {
    CU(cudaMemcpyAsync(G, dG, (size_t)(ncells + 1) * 4, cudaMemcpyDeviceToHost, st));
    if (no) CU(cudaMemcpyAsync(O, dO, no * 4, cudaMemcpyDeviceToHost, st));
  }
  CU(cudaEventRecord(b->ev[4], st));
  CU(cudaEventSynchronize(b->ev[4]));
  if (phase_ms) {
    float t01 = 0, t12 = 0, t23 = 0, t34 = 0, t_k1 = 0;
    CU(cudaEventElapsedTime(&t01, b->ev[0], b->ev[1]));
    CU(cudaEventElapsedTime(&t12, b->ev[1], b->ev[2]));
    CU(cudaEventElapsedTime(&t23, b->ev[2], b->ev[3]));
    CU(cudaEventElapsedTime(&t34, b->ev[3], b->ev[4]));
    if (b->k1_timed) CU(cudaEventElapsedTime(&t_k1, b->ev[5], b->ev[6]));
    phase_ms[0] = t_k1;
    if (algo == 1) {  // count | scan | pairgen | sort | rle | finalize
      phase_ms[1] = 0.f;
      phase_ms[2] = t01;
      phase_ms[3] = t12;
      phase_ms[4] = 0.f;
      phase_ms[5] = t23 + t34;
    } else {          // compact: counting in "count", G scan in "scan", fill in "pairgen", sort in "finalize"
      phase_ms[0] += t01;
      phase_ms[1] = t12;
      phase_ms[2] = t23;
      phase_ms[3] = 0.f;
      phase_ms[4] = 0.f;
      phase_ms[5] = t34;
    }
  }
  return PG_OK;
}

int pg_stage(pg_builder* b, int stage, void* dst, uint32_t flags, void* stream_) {
  NvtxRange nvtx_("pg_stage");
  if (!b || !b->counted) return fail(PG_STATE_ERROR, "no build to read stages from");
  if (b->deferred) return fail(PG_STATE_ERROR, "pg_stage after a PG_DEFER count");
  cudaStream_t st = static_cast<cudaStream_t>(stream_);
  CU(cudaSetDevice(b->device));
  const cudaMemcpyKind kind = (flags & PG_HOST_OUTPUT) ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
  const size_t sec = b->stage_sec;
  switch (stage) {
    case 0:
      if (b->n) {
        int rc;
        if ((rc = b->stage0.ensure((size_t)b->n * 16))) return rc;
        k_abs_offsets<<<(unsigned)std::min<int64_t>((b->n + 255) / 256, 148 * 16), 256, 0, st>>>(
            b->rec.as<uint4>(), b->tile_pre, b->n, b->stage0.as<uint4>());
        LAUNCHED("k_abs_offsets", st);
        CU(cudaMemcpyAsync(dst, b->stage0.p, (size_t)b->n * 16, kind, st));
      }
      break;
    case 1:
    case 2:
      if (!b->stages_kept) return fail(PG_STATE_ERROR, "stages 1-2 need PG_KEEP_STAGES on pg_finish");
      if (b->no) CU(cudaMemcpyAsync(dst, b->stage.as<unsigned>(stage == 1 ? 0 : sec), b->no * 4, kind, st));
      break;
    case 3:
      if (b->no) CU(cudaMemcpyAsync(dst, b->sorted_keys, b->no * 4, kind, st));
      break;
    default:
      return fail(PG_INVARIANT_ERROR, "unknown stage %d", stage);
  }
  CU(cudaStreamSynchronize(st));
  return PG_OK;
}

int pg_radix_sort_pairs(pg_builder* b, const uint32_t* keys, const uint32_t* vals, uint32_t* keys_out,
                        uint32_t* vals_out, int64_t n, int key_bits, uint32_t flags, void* stream_) {
  NvtxRange nvtx_("pg_radix_sort_pairs");
  if (!b) return fail(PG_INVARIANT_ERROR, "null builder");
  if (key_bits < 0 || key_bits > 32) return fail(PG_INVARIANT_ERROR, "key_bits must be in [0, 32]");
  if (n < 0) return fail(PG_INVARIANT_ERROR, "negative length");
  if (n > kMaxScan) return fail(PG_SIZE_ERROR, "sort of %lld pairs exceeds the size limit", (long long)n);
  cudaStream_t st = static_cast<cudaStream_t>(stream_);
  CU(cudaSetDevice(b->device));
  drop_graph(b);
  b->counted = false;
  b->launches = 0;
  if (n == 0) return PG_OK;
  // the reference sorts 8-bit digits [0, 8*ceil(key_bits/8)) (_ckernels.pyx:33)
  const int sort_bits = std::min(32, 8 * ((key_bits + 7) / 8));
  const PassPlan plan = make_plan(sort_bits, 8);
  const size_t sec = align_up((size_t)n * 4);
  int rc;
  if ((rc = b->pairs.ensure(4 * sec))) return rc;
  unsigned* kA = b->pairs.as<unsigned>(0);
  unsigned* vA = b->pairs.as<unsigned>(sec);
  unsigned* kB = b->pairs.as<unsigned>(2 * sec);
  unsigned* vB = b->pairs.as<unsigned>(3 * sec);
  const cudaMemcpyKind in_kind = (flags & PG_HOST_INPUT) ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
  CU(cudaMemcpyAsync(kA, keys, (size_t)n * 4, in_kind, st));
  CU(cudaMemcpyAsync(vA, vals, (size_t)n * 4, in_kind, st));
  const unsigned rs_tiles = (unsigned)((n + RS_TILE - 1) / RS_TILE);
  const size_t hist_bytes = align_up(kMaxPasses * kMaxBins * 4);
  if ((rc = b->sort_sync.ensure(hist_bytes + (size_t)((rs_tiles + 3) & ~3u) * kMaxBins * 4))) return rc;
  unsigned* hist = b->sort_sync.as<unsigned>(0);
  unsigned* counts = b->sort_sync.as<unsigned>(hist_bytes);
  CU(cudaMemsetAsync(hist, 0, hist_bytes, st));
  const unsigned* sorted = kA;
  unsigned* vfinal = vA;
  if (plan.npasses > 0) {
    // host outputs: final values land in the staging section behind the pair buffers
    if ((rc = b->stage.ensure(sec))) return rc;
    unsigned* vdst = (flags & PG_HOST_OUTPUT) ? b->stage.as<unsigned>() : vals_out;
    if ((rc = run_passes(b, plan, false, kA, vA, kB, vB, vdst, Count{nullptr, (unsigned)n}, (uint64_t)n, hist, counts,
                         st, &sorted)))
      return rc;
    vfinal = vdst;
  }
  const cudaMemcpyKind out_kind = (flags & PG_HOST_OUTPUT) ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
  CU(cudaMemcpyAsync(keys_out, sorted, (size_t)n * 4, out_kind, st));
  if (vfinal != vals_out) CU(cudaMemcpyAsync(vals_out, vfinal, (size_t)n * 4, out_kind, st));
  CU(cudaStreamSynchronize(st));
  return PG_OK;
}

// ---------------------------------------------------------------------------------------
// Building blocks of the sharded (multi-GPU) build: pairs of the counted shard, a stable
// partition of pairs into cell slabs, and the sort + G tail over one slab.
// ---------------------------------------------------------------------------------------
int pg_pairs(pg_builder* b, uint32_t* keys, uint32_t* vals, uint32_t val_offset, int coarse_shift, int coarse_bins,
             uint32_t* coarse_hist, void* stream_) {
  NvtxRange nvtx_("pg_pairs");
  if (!b || !b->counted) return fail(PG_STATE_ERROR, "pg_pairs without a successful pg_count");
  if (coarse_hist && (coarse_bins < 1 || coarse_bins > 3 * OC_CAP))
    return fail(PG_INVARIANT_ERROR, "coarse_bins must be in [1, %d]", 3 * OC_CAP);
  cudaStream_t st = static_cast<cudaStream_t>(stream_);
  CU(cudaSetDevice(b->device));
  drop_graph(b);
  const uint64_t no = b->no;  // PG_DEFER: the capacity (grids); the kernels read the device count
  const Count cno{b->deferred ? b->d_total : nullptr, (unsigned)no};
  const unsigned k2_tiles = (unsigned)((no + K2_TILE - 1) / K2_TILE);
  int rc;
  const size_t pb_bytes = align_up((size_t)k2_tiles * 8 + 8);
  if ((rc = b->sort_sync.ensure(pb_bytes))) return rc;
  int2* pbounds = b->sort_sync.as<int2>(0);
  unsigned* dcoarse = coarse_hist;  // device, accumulated (zeroed here), no host round trip
  if (dcoarse) CU(cudaMemsetAsync(dcoarse, 0, (size_t)coarse_bins * 4, st));
  if (no > 0) {
    const unsigned dxu = (unsigned)b->dims[0], dxyu = (unsigned)b->dims[0] * (unsigned)b->dims[1];
    k_pair_tile_bounds<<<(k2_tiles + 7) / 8, 256, 0, st>>>(b->rec.as<uint4>(), b->tile_pre, b->n, cno, K2_TILE,
                                                          pbounds);
    LAUNCHED("k_pair_tile_bounds", st);
    k_expand_pairs<<<k2_tiles, K2_THREADS, 0, st>>>(b->rec.as<uint4>(), b->tile_pre, b->n, cno,
                                                   dxu, dxyu,
                                                   pbounds, keys, vals, val_offset, dcoarse, coarse_shift,
                                                   coarse_bins);
    LAUNCHED("k_expand_pairs", st);
    b->launches += 2;
    if ((rc = fix_inverted(b, keys, st, dcoarse, coarse_shift))) return rc;
  }
  return PG_OK;
}

int pg_partition(pg_builder* b, const uint32_t* keys, const uint32_t* vals, int64_t n, const uint32_t* slab_of_bucket,
                 int bucket_shift, int nslabs, const uint32_t* slab_base, uint32_t* keys_out, uint32_t* vals_out,
                 uint32_t* slab_counts, void* stream_) {
  NvtxRange nvtx_("pg_partition");
  if (!b) return fail(PG_INVARIANT_ERROR, "null builder");
  if (nslabs < 1 || nslabs > 16) return fail(PG_INVARIANT_ERROR, "nslabs must be in [1, 16]");
  if (n < 0 || n > kMaxScan) return fail(PG_SIZE_ERROR, "partition of %lld pairs exceeds the size limit", (long long)n);
  cudaStream_t st = static_cast<cudaStream_t>(stream_);
  CU(cudaSetDevice(b->device));
  drop_graph(b);
  if (n == 0) {
    CU(cudaMemsetAsync(slab_counts, 0, (size_t)nslabs * 4, st));
    return PG_OK;
  }
  const int bits = std::max(1, bit_length((uint64_t)(nslabs - 1)));
  const unsigned ntiles = (unsigned)((n + RS_TILE - 1) / RS_TILE);
  const unsigned ld = (ntiles + 3) & ~3u;
  int rc;
  if ((rc = b->sort_sync.ensure((size_t)ld * kMaxBins * 4))) return rc;
  unsigned* counts = b->sort_sync.as<unsigned>(0);
  // slab_counts (device) receives the row totals = pairs per slab, and serves as the pass's
  // digit histogram; it must hold 2^bits entries
  const DigitFn dig{bucket_shift, 0u, slab_of_bucket};
  const Count cn{nullptr, (unsigned)n};
  k_tile_counts<<<(ntiles + TC_TILES - 1) / TC_TILES, RS_THREADS, 0, st>>>(keys, cn, dig, 1 << bits, counts, ld);
  LAUNCHED("k_tile_counts", st);
  k_scan_tile_counts<<<1u << bits, SC_THREADS, 0, st>>>(counts, cn, ld, slab_counts);
  LAUNCHED("k_scan_tile_counts", st);
  launch_radix_scatter(bits, ntiles, st, keys, vals, keys_out, vals_out, cn, bucket_shift, slab_counts, counts, ld,
                       slab_of_bucket, slab_base);
  LAUNCHED("k_radix_scatter", st);
  b->launches += 3;
  return PG_OK;
}

int pg_sort_cells(pg_builder* b, const uint32_t* keys, const uint32_t* vals, int64_t n, int64_t ncells, uint32_t* G,
                  uint32_t* O, void* stream_) {
  return pg_sort_cells_flags(b, keys, vals, n, ncells, 0, G, O, stream_);
}

int pg_sort_cells_flags(pg_builder* b, const uint32_t* keys, const uint32_t* vals, int64_t n, int64_t ncells,
                        uint32_t flags, uint32_t* G, uint32_t* O, void* stream_) {
  NvtxRange nvtx_("pg_sort_cells");
  if (!b) return fail(PG_INVARIANT_ERROR, "null builder");
  if (ncells < 1 || ncells > kMaxScan) return fail(PG_SIZE_ERROR, "ncells out of range");
  if (n < 0 || n > kMaxScan) return fail(PG_SIZE_ERROR, "sort of %lld pairs exceeds the size limit", (long long)n);
  cudaStream_t st = static_cast<cudaStream_t>(stream_);
  CU(cudaSetDevice(b->device));
  drop_graph(b);
  // the MSD-first finish (K4L) as in finish_impl; arbitrary values take its stable path
  const int key_bits = bit_length((uint64_t)(ncells - 1));
  const int lb = local_bits(key_bits, ncells, (uint64_t)n, 0);
  const PassPlan plan = lb >= 0 ? make_plan_above(lb, key_bits, kMaxDigitBits) : make_plan(key_bits, kMaxDigitBits);
  const size_t sec = align_up(std::max<size_t>((size_t)n * 4, 16));
  int rc;
  if ((rc = b->pairs.ensure(4 * sec))) return rc;
  unsigned* kA = b->pairs.as<unsigned>(0);
  unsigned* vA = b->pairs.as<unsigned>(sec);
  unsigned* kB = b->pairs.as<unsigned>(2 * sec);
  unsigned* vB = b->pairs.as<unsigned>(3 * sec);
  const unsigned rs_tiles = (unsigned)((n + RS_TILE - 1) / RS_TILE);
  const unsigned g_tiles = (unsigned)((ncells + G_TILE - 1) / G_TILE);
  const unsigned step = lb >= 0 ? (unsigned)BK_WARPS << lb : (unsigned)G_TILE;
  const unsigned tiles = (unsigned)((ncells + step - 1) / step);
  const size_t hist_bytes = align_up(kMaxPasses * kMaxBins * 4);
  const size_t kb_bytes = align_up((size_t)(std::max(g_tiles, tiles) + 1) * 4);
  if ((rc = b->sort_sync.ensure(hist_bytes + kb_bytes + (size_t)((rs_tiles + 3) & ~3u) * kMaxBins * 4))) return rc;
  unsigned* hist = b->sort_sync.as<unsigned>(0);
  unsigned* kbounds = b->sort_sync.as<unsigned>(hist_bytes);
  unsigned* counts = b->sort_sync.as<unsigned>(hist_bytes + kb_bytes);
  const Count cn{nullptr, (unsigned)n};
  const unsigned* sorted = keys;
  const unsigned* svals = vals;
  if (n > 0) {
    if (plan.npasses == 0) {
      if (lb < 0) CU(cudaMemcpyAsync(O, vals, (size_t)n * 4, cudaMemcpyDeviceToDevice, st));
    } else {
      CU(cudaMemsetAsync(hist, 0, hist_bytes, st));
      // pass 0 reads the caller's (const) pairs; later passes ping-pong in the workspace
      if ((rc = run_passes(b, plan, false, const_cast<unsigned*>(keys), const_cast<unsigned*>(vals), kB, vB,
                           lb >= 0 ? nullptr : O, cn, (uint64_t)n, hist, counts, st, &sorted, kA, vA, nullptr,
                           &svals)))
        return rc;
    }
  }
  const int lp = plan.npasses - 1;
  const bool top = lp >= 0 && n > 0 && ncells > 1;
  const unsigned* th = top ? hist + lp * kMaxBins : nullptr;
  const int tsh = top ? plan.shift[lp] : 0, tbins = top ? 1 << plan.bits[lp] : 0;
  pdl_launch(true, k_key_tile_bounds, (tiles + 1 + 7) / 8, 256, 0, st, sorted, cn, step, (unsigned)ncells, tiles + 1,
             kbounds, th, tsh, tbins);
  LAUNCHED("k_key_tile_bounds", st);
  if (lb >= 0) {
    if ((rc = launch_bucket_sort(lb, tiles, st, sorted, svals, cn, (unsigned)ncells, kbounds, G, O,
                                 (flags & PG_GEN_ORDER) != 0)))
      return rc;
    LAUNCHED("k_bucket_sort", st);
  } else {
    pdl_launch(false, k_cell_offsets, g_tiles, G_THREADS, 0, st, sorted, cn, (unsigned)ncells, kbounds, G);
    LAUNCHED("k_cell_offsets", st);
  }
  b->launches += 2;
  return PG_OK;
}

int pg_dda_prepare(pg_builder* b, const double* V, int64_t nv, const int32_t* T, int64_t n, uint32_t flags,
                   void* stream_) {
  if (!b) return fail(PG_INVARIANT_ERROR, "null builder");
  if (nv < 0 || n < 0) return fail(PG_INVARIANT_ERROR, "negative mesh size");
  if (n > 0 && (!V || !T)) return fail(PG_INVARIANT_ERROR, "null mesh arrays");
  cudaStream_t st = static_cast<cudaStream_t>(stream_);
  CU(cudaSetDevice(b->device));
  int rc;
  b->dda_ntri = -1;
  if ((rc = b->tris.ensure(std::max<size_t>((size_t)n * sizeof(TriRec), 16)))) return rc;
  if ((rc = b->dda_err.ensure(16))) return rc;
  if (n == 0) {
    b->dda_ntri = 0;
    return PG_OK;
  }
  const double* dV = V;
  const int32_t* dT = T;
  if (flags & PG_HOST_INPUT) {
    if ((rc = b->in_v.ensure(std::max<size_t>((size_t)nv * 24, 16)))) return rc;
    if ((rc = b->in_t.ensure((size_t)n * 12))) return rc;
    if (nv) CU(cudaMemcpyAsync(b->in_v.p, V, (size_t)nv * 24, cudaMemcpyHostToDevice, st));
    CU(cudaMemcpyAsync(b->in_t.p, T, (size_t)n * 12, cudaMemcpyHostToDevice, st));
    dV = b->in_v.as<double>();
    dT = b->in_t.as<int32_t>();
  }
  unsigned* err = b->dda_err.as<unsigned>();
  CU(cudaMemsetAsync(err, 0, 4, st));
  k_dda_prepare<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(dV, nv, dT, n, b->tris.as<TriRec>(), err);
  LAUNCHED("k_dda_prepare", st);
  unsigned herr = 0;
  CU(cudaMemcpyAsync(&herr, err, 4, cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  if (herr & 2u) return fail(PG_INVARIANT_ERROR, "triangle index out of range");
  b->dda_ntri = n;
  return PG_OK;
}

int pg_dda_cast(pg_builder* b, const uint32_t* G, const uint32_t* O, int64_t no, const pg_spec* spec,
                const double* origins, const double* dirs, const double* t_max, int64_t nrays, int64_t* ids,
                double* ts, uint32_t flags, void* stream_) {
  NvtxRange nvtx_("pg_dda_cast");
  if (!b || !spec) return fail(PG_INVARIANT_ERROR, "null argument");
  if (b->dda_ntri < 0) return fail(PG_STATE_ERROR, "pg_dda_cast before a successful pg_dda_prepare");
  if (nrays < 0 || no < 0) return fail(PG_INVARIANT_ERROR, "negative size");
  int64_t ncells = 1;
  for (int k = 0; k < 3; ++k) {
    if (spec->dims[k] < 1) return fail(PG_INVARIANT_ERROR, "dims must be positive");
    ncells *= spec->dims[k];
    if (ncells > kMaxIds) return fail(PG_SIZE_ERROR, "%lld cells exceed 32-bit id space", (long long)ncells);
  }
  if (nrays == 0) return PG_OK;
  if (!G || (no && !O) || !origins || !dirs || !t_max || !ids || !ts)
    return fail(PG_INVARIANT_ERROR, "null array");
  cudaStream_t st = static_cast<cudaStream_t>(stream_);
  CU(cudaSetDevice(b->device));
  int rc;
  const unsigned* dG = G;
  const unsigned* dO = O;
  if (flags & PG_HOST_INPUT) {
    const size_t gb = align_up((size_t)(ncells + 1) * 4);
    if ((rc = b->dda_grid.ensure(gb + std::max<size_t>((size_t)no * 4, 16)))) return rc;
    CU(cudaMemcpyAsync(b->dda_grid.p, G, (size_t)(ncells + 1) * 4, cudaMemcpyHostToDevice, st));
    if (no) CU(cudaMemcpyAsync(b->dda_grid.as<char>(gb), O, (size_t)no * 4, cudaMemcpyHostToDevice, st));
    dG = b->dda_grid.as<unsigned>();
    dO = b->dda_grid.as<unsigned>(gb);
  }
  const double* dor = origins;
  const double* ddi = dirs;
  const double* dtm = t_max;
  if (flags & (PG_HOST_INPUT | PG_HOST_RAYS)) {
    const size_t rb = (size_t)nrays * 24;
    if ((rc = b->dda_rays.ensure(2 * align_up(rb) + (size_t)nrays * 8))) return rc;
    CU(cudaMemcpyAsync(b->dda_rays.p, origins, rb, cudaMemcpyHostToDevice, st));
    CU(cudaMemcpyAsync(b->dda_rays.as<char>(align_up(rb)), dirs, rb, cudaMemcpyHostToDevice, st));
    CU(cudaMemcpyAsync(b->dda_rays.as<char>(2 * align_up(rb)), t_max, (size_t)nrays * 8, cudaMemcpyHostToDevice, st));
    dor = b->dda_rays.as<double>();
    ddi = b->dda_rays.as<double>(align_up(rb));
    dtm = b->dda_rays.as<double>(2 * align_up(rb));
  }
  long long* dids = reinterpret_cast<long long*>(ids);
  double* dts = ts;
  if (flags & PG_HOST_OUTPUT) {
    if ((rc = b->dda_out.ensure(2 * align_up((size_t)nrays * 8)))) return rc;
    dids = b->dda_out.as<long long>();
    dts = b->dda_out.as<double>(align_up((size_t)nrays * 8));
  }
  DdaGrid gs;
  for (int k = 0; k < 3; ++k) {
    gs.lo[k] = spec->lo[k];
    gs.hi[k] = spec->hi[k];
    gs.cs[k] = spec->cell[k];
    gs.nd[k] = spec->dims[k];
  }
  gs.ntri = b->dda_ntri;
  unsigned* err = b->dda_err.as<unsigned>();
  CU(cudaMemsetAsync(err, 0, 4, st));
  k_dda_cast<<<(unsigned)((nrays + 127) / 128), 128, 0, st>>>(dG, dO, b->tris.as<TriRec>(), gs, dor, ddi, dtm, nrays,
                                                               dids, dts, err);
  LAUNCHED("k_dda_cast", st);
  b->launches = 1;
  if (flags & PG_HOST_OUTPUT) {
    CU(cudaMemcpyAsync(ids, dids, (size_t)nrays * 8, cudaMemcpyDeviceToHost, st));
    CU(cudaMemcpyAsync(ts, dts, (size_t)nrays * 8, cudaMemcpyDeviceToHost, st));
  }
  if (flags & PG_CHECK) {
    unsigned herr = 0;
    CU(cudaMemcpyAsync(&herr, err, 4, cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    if (herr & 4u) return fail(PG_INVARIANT_ERROR, "O holds an object id outside the prepared mesh");
  } else if (flags & PG_HOST_OUTPUT) {
    CU(cudaStreamSynchronize(st));
  }
  return PG_OK;
}

int pg_grid_stats(pg_builder* b, const uint32_t* G, uint32_t flags, void* stream_, uint64_t* out) {
  NvtxRange nvtx_("pg_grid_stats");
  if (!b || !out) return fail(PG_INVARIANT_ERROR, "null argument");
  if (!b->counted) return fail(PG_STATE_ERROR, "pg_grid_stats before pg_count");
  if (b->deferred) return fail(PG_STATE_ERROR, "pg_grid_stats after a PG_DEFER count");
  if (!G) return fail(PG_INVARIANT_ERROR, "null G");
  cudaStream_t st = static_cast<cudaStream_t>(stream_);
  CU(cudaSetDevice(b->device));
  int rc;
  const int64_t ncells = b->ncells;
  const unsigned* dG = G;
  if (flags & PG_HOST_INPUT) {
    if ((rc = b->gbuf.ensure((size_t)(ncells + 1) * 4))) return rc;
    CU(cudaMemcpyAsync(b->gbuf.p, G, (size_t)(ncells + 1) * 4, cudaMemcpyHostToDevice, st));
    dG = b->gbuf.as<unsigned>();
  }
  if ((rc = b->dda_err.ensure(64))) return rc;
  unsigned long long* acc = b->dda_err.as<unsigned long long>();
  CU(cudaMemsetAsync(acc, 0, 3 * sizeof(unsigned long long), st));
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, b->device);
  const long long cblocks = std::min<long long>((ncells + 255) / 256, 8LL * sms);
  k_stats_cells<<<(unsigned)std::max<long long>(cblocks, 1), 256, 0, st>>>(dG, ncells, acc);
  LAUNCHED("k_stats_cells", st);
  b->launches = 1;
  if (b->n > 0) {
    const long long oblocks = std::min<long long>((b->n + 255) / 256, 8LL * sms);
    k_stats_objects<<<(unsigned)oblocks, 256, 0, st>>>(b->rec.as<uint4>(), b->tile_pre, b->n, (unsigned)b->no, acc);
    LAUNCHED("k_stats_objects", st);
    ++b->launches;
  }
  CU(cudaMemcpyAsync(b->h_scalars, acc, 3 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  out[0] = b->h_scalars[0];  // nonempty cells
  out[1] = b->h_scalars[1];  // in-grid objects
  out[2] = b->h_scalars[2];  // max cells per in-grid object
  out[3] = b->no;            // NO of the counted mesh
  return PG_OK;
}

int pg_mesh_bounds(pg_builder* b, const double* V, int64_t nv, uint32_t flags, void* stream_, double* lo,
                   double* hi) {
  NvtxRange nvtx_("pg_mesh_bounds");
  if (!b || !lo || !hi) return fail(PG_INVARIANT_ERROR, "null argument");
  if (nv <= 0) return fail(PG_INVARIANT_ERROR, "cannot bound an empty mesh");
  if (!V) return fail(PG_INVARIANT_ERROR, "null vertex array");
  cudaStream_t st = static_cast<cudaStream_t>(stream_);
  CU(cudaSetDevice(b->device));
  int rc;
  const double* dV = V;
  if (flags & PG_HOST_INPUT) {
    if ((rc = b->in_v.ensure((size_t)nv * 24))) return rc;
    CU(cudaMemcpyAsync(b->in_v.p, V, (size_t)nv * 24, cudaMemcpyHostToDevice, st));
    dV = b->in_v.as<double>();
  }
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, b->device);
  const long long nflat = nv * 3;
  const int nblocks = (int)std::max<long long>(1, std::min<long long>(8LL * sms, (nflat + MB_THREADS - 1) / MB_THREADS));
  if ((rc = b->dda_err.ensure(align_up(16) + (size_t)nblocks * 48 + 48))) return rc;
  unsigned* flag = b->dda_err.as<unsigned>();
  double* part = b->dda_err.as<double>(align_up(16));
  double* out = part + (size_t)nblocks * 6;
  CU(cudaMemsetAsync(flag, 0, 4, st));
  k_mesh_bounds<<<nblocks, MB_THREADS, 0, st>>>(dV, nflat, part, flag);
  LAUNCHED("k_mesh_bounds", st);
  k_mesh_bounds_final<<<1, 32, 0, st>>>(part, nblocks, out);
  LAUNCHED("k_mesh_bounds_final", st);
  b->launches = 2;
  double h[6];
  unsigned hf = 0;
  CU(cudaMemcpyAsync(h, out, 48, cudaMemcpyDeviceToHost, st));
  CU(cudaMemcpyAsync(&hf, flag, 4, cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  if (hf & 1u) return fail(PG_INVARIANT_ERROR, "Aabb corners must not be NaN");
  for (int k = 0; k < 3; ++k) {
    lo[k] = h[k];
    hi[k] = h[3 + k];
  }
  return PG_OK;
}

int pg_wait(pg_builder* b) {
  if (!b) return fail(PG_INVARIANT_ERROR, "null builder");
  CU(cudaSetDevice(b->device));
  CU(cudaEventSynchronize(b->ev[4]));
  return PG_OK;
}

int pg_phase_times(pg_builder* b, float* phase_ms) {
  if (!b || !phase_ms) return fail(PG_INVARIANT_ERROR, "null argument");
  if (!b->phases_ready) return fail(PG_STATE_ERROR, "pg_phase_times without a pg_finish");
  CU(cudaSetDevice(b->device));
  CU(cudaEventSynchronize(b->ev[4]));
  return phase_times(b, phase_ms);
}

int pg_kernel_timing(int on) {
  g_ktimes = on ? 1 : 0;
  return PG_OK;
}

int pg_kernel_times(char* buf, int len) {
  if (!buf || len <= 0) return fail(PG_INVARIANT_ERROR, "null buffer");
  std::string out;
  if (g_kt.used > 1) {
    cudaEventSynchronize(g_kt.ev[g_kt.used - 1].second);
    char line[128];
    for (size_t i = 1; i < g_kt.used; ++i) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, g_kt.ev[i - 1].second, g_kt.ev[i].second);
      snprintf(line, sizeof line, "%s %.3f\n", g_kt.ev[i].first, ms * 1e3f);
      out += line;
    }
  }
  snprintf(buf, (size_t)len, "%s", out.c_str());
  return PG_OK;
}

int pg_load_obj(pg_builder* b, const uint8_t* bytes, uint64_t nbytes, uint32_t flags, void* stream_, int64_t* out) {
  NvtxRange nvtx_("pg_load_obj");
  if (!b || !out) return fail(PG_INVARIANT_ERROR, "null argument");
  if (nbytes && !bytes) return fail(PG_INVARIANT_ERROR, "null byte buffer");
  if (nbytes >= (1ull << 32)) return fail(PG_SIZE_ERROR, "OBJ input of %llu bytes exceeds 4 GiB", (unsigned long long)nbytes);
  cudaStream_t st = static_cast<cudaStream_t>(stream_);
  CU(cudaSetDevice(b->device));
  int rc;
  b->obj_nv = -1;
  for (int k = 0; k < 6; ++k) out[k] = 0;
  b->launches = 0;
  if (nbytes == 0) {
    b->obj_nv = 0;
    b->obj_nt = 0;
    return PG_OK;
  }
  const unsigned char* d = bytes;
  if (flags & PG_HOST_INPUT) {
    if ((rc = b->obj_bytes.ensure(nbytes))) return rc;
    CU(cudaMemcpyAsync(b->obj_bytes.p, bytes, nbytes, cudaMemcpyHostToDevice, st));
    d = b->obj_bytes.as<unsigned char>();
  }
  // 1. line breaks: per-chunk counts -> exclusive prefix (+ total) -> break positions
  const unsigned nchunks = (unsigned)((nbytes + OBJ_CHUNK - 1) / OBJ_CHUNK);
  const unsigned xt = (unsigned)((nchunks + XS_TILE - 1) / XS_TILE);
  const size_t cb = align_up((size_t)nchunks * 4), pb = align_up((size_t)(nchunks + 1) * 4);
  const size_t sb = align_up((size_t)xt * 8), tb = align_up((size_t)xt * 4);
  if ((rc = b->obj_scan.ensure(cb + pb + sb + tb + 256))) return rc;
  unsigned* ccount = b->obj_scan.as<unsigned>(0);
  unsigned* cpre = b->obj_scan.as<unsigned>(cb);
  unsigned long long* tsum = b->obj_scan.as<unsigned long long>(cb + pb);
  unsigned* tpre = b->obj_scan.as<unsigned>(cb + pb + sb);
  unsigned long long* scal = b->obj_scan.as<unsigned long long>(cb + pb + sb + tb);  // [0] total, [1] err
  k_obj_count_breaks<<<nchunks, 256, 0, st>>>(d, nbytes, ccount);
  LAUNCHED("k_obj_count_breaks", st);
  k_tile_reduce<<<xt, XS_THREADS, 0, st>>>(ccount, nchunks, tsum);
  LAUNCHED("k_tile_reduce", st);
  k_scan_tile_sums<<<1, TS_THREADS, 0, st>>>(tsum, xt, tpre, scal);
  LAUNCHED("k_scan_tile_sums", st);
  k_tile_scan_apply<<<xt, XS_THREADS, 0, st>>>(ccount, nchunks, tpre, scal, cpre);
  LAUNCHED("k_tile_scan_apply", st);
  unsigned long long nbreaks = 0;
  unsigned char last = 0;
  CU(cudaMemcpyAsync(&nbreaks, scal, 8, cudaMemcpyDeviceToHost, st));
  CU(cudaMemcpyAsync(&last, d + nbytes - 1, 1, cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  const unsigned long long L = nbreaks + ((last == '\n' || last == '\r') ? 0 : 1);
  if ((rc = b->obj_lines.ensure(std::max<size_t>((size_t)L * 4, 16)))) return rc;
  unsigned* line_end = b->obj_lines.as<unsigned>();
  k_obj_line_ends<<<nchunks, 256, 0, st>>>(d, nbytes, cpre, line_end);
  LAUNCHED("k_obj_line_ends", st);
  if (L > nbreaks) {
    const unsigned endpos = (unsigned)nbytes;
    CU(cudaMemcpyAsync(line_end + (L - 1), &endpos, 4, cudaMemcpyHostToDevice, st));
  }
  // 2. classify lines, 3. scan (vertices << 32 | triangles), 4. parse
  const unsigned ot = (unsigned)((L + OS_TILE - 1) / OS_TILE);
  if ((rc = b->obj_info.ensure(align_up((size_t)L * 8) + align_up((size_t)(ot + 1) * 8)))) return rc;
  if ((rc = b->obj_pre.ensure((size_t)(L + 1) * 8))) return rc;
  unsigned long long* info = b->obj_info.as<unsigned long long>();
  unsigned long long* osum = b->obj_info.as<unsigned long long>(align_up((size_t)L * 8));
  unsigned long long* pre = b->obj_pre.as<unsigned long long>();
  unsigned long long* err = scal + 1;
  const unsigned long long none = ~0ull;
  CU(cudaMemcpyAsync(err, &none, 8, cudaMemcpyHostToDevice, st));
  const unsigned lb = (unsigned)((L + 127) / 128);
  k_obj_classify<<<lb, 128, 0, st>>>(d, nbytes, line_end, L, info, err);
  LAUNCHED("k_obj_classify", st);
  k_u64_tile_sums<<<ot, 256, 0, st>>>(info, L, osum);
  LAUNCHED("k_u64_tile_sums", st);
  k_u64_scan_sums<<<1, 1024, 0, st>>>(osum, ot);
  LAUNCHED("k_u64_scan_sums", st);
  k_u64_tile_apply<<<ot, 256, 0, st>>>(info, L, osum, pre);
  LAUNCHED("k_u64_tile_apply", st);
  unsigned long long tot = 0;
  CU(cudaMemcpyAsync(&tot, osum + ot, 8, cudaMemcpyDeviceToHost, st));
  CU(cudaMemcpyAsync(pre + L, osum + ot, 8, cudaMemcpyDeviceToDevice, st));
  CU(cudaStreamSynchronize(st));
  const unsigned long long nv = tot >> 32, nt = tot & 0xffffffffull;
  if (nv >= (1ull << 31)) return fail(PG_SIZE_ERROR, "%llu vertices exceed the int32 index range", nv);
  if ((rc = b->obj_v.ensure(std::max<size_t>((size_t)nv * 24, 16)))) return rc;
  if ((rc = b->obj_t.ensure(std::max<size_t>((size_t)nt * 12, 16)))) return rc;
  k_obj_parse<<<lb, 128, 0, st>>>(d, nbytes, line_end, L, info, pre, b->obj_v.as<double>(), b->obj_t.as<int>(), err);
  LAUNCHED("k_obj_parse", st);
  b->launches = 10;
  unsigned long long herr = 0;
  CU(cudaMemcpyAsync(&herr, err, 8, cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  out[0] = (int64_t)nv;
  out[1] = (int64_t)nt;
  if (herr != ~0ull) {
    // first offending line: its number, the vertices read before it, its byte range
    const unsigned long long li = herr - 1;
    unsigned long long pv = 0;
    unsigned e0 = 0, e1 = 0;
    CU(cudaMemcpy(&pv, pre + li, 8, cudaMemcpyDeviceToHost));
    if (li > 0) CU(cudaMemcpy(&e0, line_end + li - 1, 4, cudaMemcpyDeviceToHost));
    CU(cudaMemcpy(&e1, line_end + li, 4, cudaMemcpyDeviceToHost));
    out[2] = (int64_t)herr;
    out[3] = (int64_t)(pv >> 32);
    out[4] = li > 0 ? (int64_t)e0 + 1 : 0;
    out[5] = (int64_t)e1;
    return fail(PG_PARSE_ERROR, "OBJ parse error at line %llu", herr);
  }
  b->obj_nv = (int64_t)nv;
  b->obj_nt = (int64_t)nt;
  return PG_OK;
}

int pg_obj_fetch(pg_builder* b, double* V, int32_t* T, uint32_t flags, void* stream_) {
  if (!b) return fail(PG_INVARIANT_ERROR, "null builder");
  if (b->obj_nv < 0) return fail(PG_STATE_ERROR, "pg_obj_fetch without a successful pg_load_obj");
  cudaStream_t st = static_cast<cudaStream_t>(stream_);
  CU(cudaSetDevice(b->device));
  const cudaMemcpyKind k = (flags & PG_HOST_OUTPUT) ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
  if (b->obj_nv) CU(cudaMemcpyAsync(V, b->obj_v.p, (size_t)b->obj_nv * 24, k, st));
  if (b->obj_nt) CU(cudaMemcpyAsync(T, b->obj_t.p, (size_t)b->obj_nt * 12, k, st));
  CU(cudaStreamSynchronize(st));
  return PG_OK;
}

int pg_partition_counts(pg_builder* b, const uint32_t* keys, int64_t n, const uint32_t* slab_of_bucket,
                        int bucket_shift, int nslabs, uint32_t* slab_counts, void* stream_) {
  NvtxRange nvtx_("pg_partition_counts");
  if (!b) return fail(PG_INVARIANT_ERROR, "null builder");
  if (nslabs < 1 || nslabs > 16) return fail(PG_INVARIANT_ERROR, "nslabs must be in [1, 16]");
  if (n < 0 || n > kMaxScan) return fail(PG_SIZE_ERROR, "partition of %lld pairs exceeds the size limit", (long long)n);
  cudaStream_t st = static_cast<cudaStream_t>(stream_);
  CU(cudaSetDevice(b->device));
  drop_graph(b);
  b->part_n = -1;
  const int bits = std::max(1, bit_length((uint64_t)(nslabs - 1)));
  if (n == 0) {
    CU(cudaMemsetAsync(slab_counts, 0, (size_t)(1 << bits) * 4, st));
    b->part_n = 0;
    b->part_bits = bits;
    return PG_OK;
  }
  const unsigned ntiles = (unsigned)((n + RS_TILE - 1) / RS_TILE);
  const unsigned ld = (ntiles + 3) & ~3u;
  int rc;
  if ((rc = b->sort_sync.ensure((size_t)ld * kMaxBins * 4))) return rc;
  unsigned* counts = b->sort_sync.as<unsigned>(0);
  const DigitFn dig{bucket_shift, 0u, slab_of_bucket};
  // after a PG_DEFER count these are this builder's pairs: n is their capacity, the device
  // count bounds the kernels
  const Count cn{b->deferred ? b->d_total : nullptr, (unsigned)n};
  k_tile_counts<<<(ntiles + TC_TILES - 1) / TC_TILES, RS_THREADS, 0, st>>>(keys, cn, dig, 1 << bits, counts, ld);
  LAUNCHED("k_tile_counts", st);
  k_scan_tile_counts<<<1u << bits, SC_THREADS, 0, st>>>(counts, cn, ld, slab_counts);
  LAUNCHED("k_scan_tile_counts", st);
  b->launches = 2;
  b->part_n = n;
  b->part_bits = bits;
  return PG_OK;
}

int pg_partition_send(pg_builder* b, const uint32_t* keys, const uint32_t* vals, int64_t n,
                      const uint32_t* slab_of_bucket, int bucket_shift, int nslabs, const uint32_t* slab_base,
                      const uint64_t* dst_keys, const uint64_t* dst_vals, const uint64_t* dst_offset, void* stream_) {
  NvtxRange nvtx_("pg_partition_send");
  if (!b || !dst_keys || !dst_vals || !dst_offset) return fail(PG_INVARIANT_ERROR, "null argument");
  if (b->part_n != n) return fail(PG_STATE_ERROR, "pg_partition_send without pg_partition_counts on these pairs");
  if (nslabs < 1 || nslabs > 16) return fail(PG_INVARIANT_ERROR, "nslabs must be in [1, 16]");
  cudaStream_t st = static_cast<cudaStream_t>(stream_);
  CU(cudaSetDevice(b->device));
  if (n == 0) return PG_OK;
  P2PDst dst{};
  for (int s = 0; s < nslabs; ++s) {
    dst.k[s] = reinterpret_cast<unsigned*>(dst_keys[s]);
    dst.v[s] = reinterpret_cast<unsigned*>(dst_vals[s]);
    dst.off[s] = dst_offset[s];
    if (dst_offset[s] >= (1ull << 32)) return fail(PG_SIZE_ERROR, "receive offset exceeds 32 bits");
  }
  const unsigned ntiles = (unsigned)((n + RS_TILE - 1) / RS_TILE);
  const unsigned ld = (ntiles + 3) & ~3u;
  const unsigned* counts = b->sort_sync.as<unsigned>(0);
  const Count cn{b->deferred ? b->d_total : nullptr, (unsigned)n};
  switch (b->part_bits) {
#define PG_CASE(B)                                                                                          \
  case B:                                                                                                   \
    k_partition_send<B><<<ntiles, RS_THREADS, rs_smem_bytes(), st>>>(keys, vals, cn, bucket_shift, counts, ld, \
                                                                     slab_of_bucket, slab_base, dst);       \
    break;
    PG_CASE(1) PG_CASE(2) PG_CASE(3) PG_CASE(4)
#undef PG_CASE
    default: return fail(PG_INVARIANT_ERROR, "bad slab digit width");
  }
  LAUNCHED("k_partition_send", st);
  b->launches = 1;
  return PG_OK;
}

int pg_features(void) { return PGRID_FUSED_DISPATCH ? PG_FEATURE_FUSED_DISPATCH : 0; }

#if !PGRID_FUSED_DISPATCH
int pg_coarse_hist(pg_builder*, int, int, uint32_t*, void*) {
  return fail(PG_STATE_ERROR, "libpgrid built without PGRID_FUSED_DISPATCH (expansion + dispatch kernel)");
}
int pg_pairs_send(pg_builder*, uint32_t, const uint32_t*, int, int, const uint32_t*, const uint64_t*,
                  const uint64_t*, const uint64_t*, void*) {
  return fail(PG_STATE_ERROR, "libpgrid built without PGRID_FUSED_DISPATCH (expansion + dispatch kernel)");
}
#else
int pg_coarse_hist(pg_builder* b, int coarse_shift, int coarse_bins, uint32_t* coarse_hist, void* stream_) {
  if (!b || !b->counted) return fail(PG_STATE_ERROR, "pg_coarse_hist without a successful pg_count");
  if (!coarse_hist || coarse_bins < 1 || coarse_bins > PLAN_MAX_BUCKETS || coarse_shift < 0 || coarse_shift > 31)
    return fail(PG_INVARIANT_ERROR, "coarse_bins must be in [1, %d]", PLAN_MAX_BUCKETS);
  cudaStream_t st = static_cast<cudaStream_t>(stream_);
  CU(cudaSetDevice(b->device));
  drop_graph(b);
  CU(cudaMemsetAsync(coarse_hist, 0, (size_t)coarse_bins * 4, st));
  if (b->n == 0 || b->no == 0) return PG_OK;
  const Count cno{b->deferred ? b->d_total : nullptr, (unsigned)b->no};
  const unsigned dxu = (unsigned)b->dims[0], dxyu = (unsigned)b->dims[0] * (unsigned)b->dims[1];
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, b->device);
  // queue of objects with many rows (walls): [count][ids...]; a full queue falls back inline
  const unsigned big_cap = 1u << 16;
  int rc;
  if ((rc = b->send.ensure(((size_t)big_cap + 64) * 4))) return rc;
  unsigned* big = b->send.as<unsigned>(0);
  CU(cudaMemsetAsync(big, 0, 4, st));
  const unsigned grid = (unsigned)std::min<long long>((b->n + 255) / 256, 4LL * sms);
  k_coarse_from_boxes<<<grid, 256, (size_t)coarse_bins * 4, st>>>(b->rec.as<uint4>(), b->tile_pre, b->n, cno, dxu,
                                                                  dxyu, coarse_shift, coarse_bins, coarse_hist, big,
                                                                  big_cap);
  LAUNCHED("k_coarse_from_boxes", st);
  k_coarse_big<<<2 * sms, 256, (size_t)coarse_bins * 4, st>>>(b->rec.as<uint4>(), b->tile_pre, b->n, cno, dxu, dxyu,
                                                              coarse_shift, coarse_bins, coarse_hist, big, big_cap);
  LAUNCHED("k_coarse_big", st);
  b->launches = 2;
  return PG_OK;
}

int pg_pairs_send(pg_builder* b, uint32_t val_offset, const uint32_t* slab_of_bucket, int bucket_shift, int nslabs,
                  const uint32_t* slab_base, const uint64_t* dst_keys, const uint64_t* dst_vals,
                  const uint64_t* dst_offset, void* stream_) {
  if (!b || !b->counted) return fail(PG_STATE_ERROR, "pg_pairs_send without a successful pg_count");
  if (!dst_keys || !dst_vals || !dst_offset || !slab_of_bucket || !slab_base)
    return fail(PG_INVARIANT_ERROR, "null argument");
  if (nslabs < 1 || nslabs > kMaxP2P) return fail(PG_INVARIANT_ERROR, "nslabs must be in [1, %d]", kMaxP2P);
  cudaStream_t st = static_cast<cudaStream_t>(stream_);
  CU(cudaSetDevice(b->device));
  drop_graph(b);
  const uint64_t no = b->no;  // PG_DEFER: the capacity (grid); the kernels read the device count
  if (no == 0) return PG_OK;
  P2PDst dst{};
  for (int s2 = 0; s2 < nslabs; ++s2) {
    dst.k[s2] = reinterpret_cast<unsigned*>(dst_keys[s2]);
    dst.v[s2] = reinterpret_cast<unsigned*>(dst_vals[s2]);
    dst.off[s2] = dst_offset[s2];
    if (dst_offset[s2] >= (1ull << 32)) return fail(PG_SIZE_ERROR, "receive offset exceeds 32 bits");
  }
  const Count cno{b->deferred ? b->d_total : nullptr, (unsigned)no};
  const unsigned ntiles = (unsigned)((no + RS_TILE - 1) / RS_TILE);
  const size_t bnd_bytes = align_up((size_t)ntiles * 8 + 8), st_bytes = align_up((size_t)ntiles * kMaxP2P * 8);
  int rc;
  if ((rc = b->send.ensure(bnd_bytes + st_bytes + 256))) return rc;
  int2* bounds = b->send.as<int2>(0);
  unsigned long long* status = b->send.as<unsigned long long>(bnd_bytes);
  unsigned* ticket = b->send.as<unsigned>(bnd_bytes + st_bytes);
  CU(cudaMemsetAsync(status, 0, st_bytes + 256, st));  // look-back flags and the ticket
  const unsigned dxu = (unsigned)b->dims[0], dxyu = (unsigned)b->dims[0] * (unsigned)b->dims[1];
  k_pair_tile_bounds<<<(ntiles + 7) / 8, 256, 0, st>>>(b->rec.as<uint4>(), b->tile_pre, b->n, cno, RS_TILE, bounds);
  LAUNCHED("k_pair_tile_bounds", st);
  const int bits = std::max(1, bit_length((uint64_t)(nslabs - 1)));
  const LookBack lb{status};
  switch (bits) {
#define PG_CASE(B)                                                                                                   \
  case B:                                                                                                            \
    k_pairs_send<B><<<ntiles, RS_THREADS, sizeof(SendSmem), st>>>(b->rec.as<uint4>(), b->tile_pre, b->n, cno, dxu,    \
                                                                  dxyu, bounds, val_offset, bucket_shift,             \
                                                                  slab_of_bucket, slab_base, dst, lb, ticket);        \
    break;
    PG_CASE(1) PG_CASE(2) PG_CASE(3) PG_CASE(4)
#undef PG_CASE
    default: return fail(PG_INVARIANT_ERROR, "bad slab digit width");
  }
  LAUNCHED("k_pairs_send", st);
  b->launches = 2;
  return PG_OK;
}
#endif  // PGRID_FUSED_DISPATCH

int pg_peer_put(const uint32_t* src, int64_t n, const uint64_t* dsts, int nranks, int64_t dst_offset, void* stream_) {
  if (!dsts || (n > 0 && !src)) return fail(PG_INVARIANT_ERROR, "null argument");
  if (nranks < 1 || nranks > kMaxP2P) return fail(PG_INVARIANT_ERROR, "nranks must be in [1, %d]", kMaxP2P);
  if (n < 0 || n > (1ll << 30) || dst_offset < 0) return fail(PG_INVARIANT_ERROR, "bad peer put size");
  if (n == 0) return PG_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream_);
  PeerPtrs p{};
  for (int r = 0; r < nranks; ++r) p.p[r] = reinterpret_cast<unsigned*>(dsts[r]);
  k_peer_put<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(src, (unsigned)n, p, nranks, (unsigned long long)dst_offset);
  CU(cudaGetLastError());
  return PG_OK;
}

int pg_peer_put_count(pg_builder* b, const uint64_t* dsts, int nranks, int64_t dst_offset, void* stream_) {
  if (!b || !b->counted || !b->d_total) return fail(PG_STATE_ERROR, "pg_peer_put_count without a pg_count");
  return pg_peer_put(reinterpret_cast<const uint32_t*>(b->d_total), 3, dsts, nranks, dst_offset, stream_);
}

int pg_slab_plan(const uint32_t* hists, int nranks, int nbuckets, int bucket_shift, int64_t ncells, int nslabs,
                 uint32_t* slab_of_bucket, uint32_t* slab_base, int64_t* plan, void* stream_) {
  if (!hists || !slab_of_bucket || !slab_base || !plan) return fail(PG_INVARIANT_ERROR, "null argument");
  if (nranks < 1 || nranks > kMaxP2P) return fail(PG_INVARIANT_ERROR, "nranks must be in [1, %d]", kMaxP2P);
  if (nslabs < 1 || nslabs > kMaxP2P) return fail(PG_INVARIANT_ERROR, "nslabs must be in [1, %d]", kMaxP2P);
  if (nbuckets < 1 || nbuckets > PLAN_MAX_BUCKETS)
    return fail(PG_INVARIANT_ERROR, "nbuckets must be in [1, %d]", PLAN_MAX_BUCKETS);
  if (bucket_shift < 0 || bucket_shift > 40 || ncells < 1) return fail(PG_INVARIANT_ERROR, "bad slab geometry");
  cudaStream_t st = static_cast<cudaStream_t>(stream_);
  k_slab_plan<<<1, PLAN_THREADS, 0, st>>>(hists, nranks, nbuckets, bucket_shift, (long long)ncells, nslabs,
                                          slab_of_bucket, slab_base, reinterpret_cast<long long*>(plan));
  CU(cudaGetLastError());
  return PG_OK;
}

}  // extern "C"
