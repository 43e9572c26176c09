/*
 * pgrid.h -- C ABI of libpgrid.so, the B200 (sm_100a) parallel uniform-grid builder.
 *
 * This is the drop-in boundary for the reference's hot path
 *   pargrid.builders.build_parallel(mesh, spec, workers=None, record=None)
 *       (/root/reference/pkg/src/pargrid/builders.py:144-169)
 * and for the reference's native plugin seam
 *   kernels.radix_sort_pairs(keys, values, key_bits)
 *       (/root/reference/pkg/src/pargrid/kernels/__init__.py:50-51 -> _ckernels.pyx:21-50).
 * Plain pointers and sizes only; no torch or Python types. Python binds it with ctypes
 * (paper_2403_10647_b200/_native.py); INTEGRATION.md shows the binding a reference
 * maintainer would add.
 *
 * Threading: a pg_builder owns its device workspace and must be used by one thread at a
 * time; distinct builders are independent (the reference is safe for concurrent builds on
 * distinct inputs). Every call is enqueued on the caller's `stream`
 * (a cudaStream_t; NULL = legacy default stream).
 */
#ifndef PGRID_H
#define PGRID_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Return codes. Python maps them onto the reference's exception classes
 * (pargrid/errors.py:4-23): 1 -> SizeError, 2 -> InvariantError, 3 -> GridError. */
#define PG_OK 0
#define PG_SIZE_ERROR 1        /* NO > 2^32-1 (builders.py:99-100); N/NO/ncells > 2^30
                                  (primitives.py:17,29-31); ncells > 2^32-1 (gridcore.py:46) */
#define PG_INVARIANT_ERROR 2   /* precondition violated (primitives.py:22-25, gridcore.py:44-52) */
#define PG_CUDA_ERROR 3        /* CUDA runtime failure */
#define PG_STATE_ERROR 4       /* call sequence violated (finish before count, ...) */
#define PG_PARSE_ERROR 6        /* pg_load_obj: malformed OBJ (-> ObjParseError) */
#define PG_CAPACITY_ERROR 5    /* pg_build_wait / pg_count_result: NO exceeded the capacity given */

/* Flags. */
#define PG_HOST_INPUT 1u       /* V/T (or sort inputs) are host pointers: copied H2D in-call */
#define PG_HOST_OUTPUT 2u      /* G/O (or sort outputs) are host pointers: copied D2H in-call */
#define PG_KEEP_STAGES 4u      /* keep the unsorted pairs for pg_stage (record= support) */
#define PG_HOST_RAYS 8u        /* pg_dda_cast: rays are host pointers (grid stays on device) */
#define PG_CHECK 16u           /* pg_dda_cast: synchronise and report device-side errors */
#define PG_ASYNC 32u           /* pg_finish: return once enqueued (host outputs valid after pg_wait) */
#define PG_DEFER 64u           /* pg_count: no host round trip; *no_out is the pair capacity on entry.
                                  pg_finish (O must hold the capacity), pg_pairs, pg_coarse_hist,
                                  pg_pairs_send and pg_partition_counts/_send (n = that capacity)
                                  then run on the device count; after a stream synchronise
                                  pg_count_result reports NO, or PG_CAPACITY_ERROR when NO exceeded
                                  the capacity or a lone inverted box voided the deferred steps
                                  (rebuild without PG_DEFER). pg_finish_baseline, pg_stage and
                                  pg_grid_stats refuse a deferred count. */
#define PG_STATS 128u          /* pg_count (sharded builds): no local verdict. The count's raw
                                  statistics are kept for pg_count_stats and the caller combines
                                  every rank's into the global verdict (the reference's checks
                                  apply to the whole mesh, not to one shard) */
#define PG_GEN_ORDER 256u      /* pg_sort_cells_flags: the pairs are in generation order, so the
                                  values ascend inside every cell (distinct triangle ids, object-
                                  major emission): the MSD-first finish may rank a cell's pairs
                                  by value instead of by position */

/* Grid specification: the exact host doubles of GridSpec (gridcore.py:36-57). */
typedef struct {
    double lo[3];     /* spec.bounds.lo (padded, gridcore.py:190-194) */
    double hi[3];     /* spec.bounds.hi */
    double cell[3];   /* spec.cell_size = (hi - lo) / dims (gridcore.py:50) */
    int64_t dims[3];  /* spec.dims, x-fastest linearisation (gridcore.py:99-103) */
} pg_spec;

typedef struct pg_builder pg_builder;

/* Phase times in ms, in the reference's PHASES order (builders.py:19):
 * count, scan, pairgen, sort, rle, finalize. Fused phases report 0 for the absorbed step
 * (scan is fused into count; rle into finalize). */
#define PG_NPHASES 6

int  pg_builder_create(int device, pg_builder **out);
void pg_builder_destroy(pg_builder *b);

/* Phase 1 of build_parallel: triangle AABB -> clamped cell box -> CountCells with the tile-
 * local part of the ExclusiveSum, then the cross-tile scan (builders.py:90-101,
 * gridcore.py:145-167). V: f64[nv*3] row-major vertices; T: i32[n*3] triangle vertex
 * indices (geometry.py:33-45), validated on the device (InvariantError when out of range).
 * Returns NO (number of <cell, object> pairs) in *no_out after one device->host readback.
 * SizeError conditions are detected here (NO > 2^32-1, NO > 2^30, ncells > 2^30, n > 2^30). */
int pg_count(pg_builder *b, const double *V, int64_t nv, const int32_t *T, int64_t n,
             const pg_spec *spec, uint32_t flags, void *stream, uint64_t *no_out);

/* Phase 2: pair expansion, stable LSD radix sort on ceil(log2 ncells) key bits, and the
 * RLE -> scatter -> ExclusiveSum tail (builders.py:120-141, 155-160) into caller buffers
 * G[ncells+1] (u32) and O[NO] (u32, original triangle ids ascending within each cell).
 * phase_ms may be NULL. */
int pg_finish(pg_builder *b, uint32_t *G, uint32_t *O, uint32_t flags, void *stream,
              float *phase_ms);

/* The paper's comparison builders (builders.py:172-231), after pg_count: algo 1 = sorted grid
 * (one pair-generation task per object, then the same sort/G tail), algo 2 = compact grid
 * (per-cell counters, scan, slot claims, canonical per-cell sort). Same G/O as pg_finish;
 * max_task_work (may be NULL) receives the largest per-object task (sorted builder). */
int pg_finish_baseline(pg_builder *b, int algo, uint32_t *G, uint32_t *O, uint32_t flags,
                       void *stream, float *phase_ms, uint64_t *max_task_work);

/* Ray casting over a built grid (traverse.py:114-131 ->
 * kernels.dda_cast, kernels/__init__.py:66-67 -> _ckernels.pyx:146-260).
 * pg_dda_prepare stages the mesh once (per-triangle v0/e1/e2 records; PG_HOST_INPUT: V/T are
 * host pointers; index range checked -> PG_INVARIANT_ERROR). pg_dda_cast then walks the
 * grid (G u32[ncells+1], O u32[no]) for nrays rays (origins/dirs f64[nrays][3], t_max
 * f64[nrays]) and writes ids i64 (-1 on a miss) and ts f64 (+inf on a miss), bit-identical
 * to the reference's compiled lane. Flags: PG_HOST_INPUT (grid and rays on the host),
 * PG_HOST_RAYS (rays only), PG_HOST_OUTPUT (ids/ts on the host), PG_CHECK (synchronise and
 * fail on an O entry outside the prepared mesh). */
int pg_dda_prepare(pg_builder *b, const double *V, int64_t nv, const int32_t *T, int64_t n,
                   uint32_t flags, void *stream);
int pg_dda_cast(pg_builder *b, const uint32_t *G, const uint32_t *O, int64_t no, const pg_spec *spec,
                const double *origins, const double *dirs, const double *t_max, int64_t nrays,
                int64_t *ids, double *ts, uint32_t flags, void *stream);

/* Tight mesh bounds on the device (geometry.py:55-59 mesh_bounds, the
 * reduction inside gridcore.spec_for_mesh, gridcore.py:185-198): per-axis min / max over all
 * nv vertices (PG_HOST_INPUT: V is a host pointer). NaN -> PG_INVARIANT_ERROR (Aabb,
 * geometry.py:20-25); nv == 0 -> PG_INVARIANT_ERROR. Padding and dims stay on the host. */
int pg_mesh_bounds(pg_builder *b, const double *V, int64_t nv, uint32_t flags, void *stream,
                   double *lo, double *hi);

/* OBJ ingestion on the device (geometry.py:65-112 load_obj): parse the
 * v/f subset of an OBJ byte buffer (PG_HOST_INPUT: host pointer; < 4 GiB) into vertices
 * (f64 nv x 3) and fan-triangulated faces (i32 nt x 3) kept in the builder. out[0..5] =
 * {nv, nt, first bad line (1-based, 0 if none), vertices before that line, that line's
 * byte range [out[4], out[5])}; a malformed file returns PG_PARSE_ERROR with out[2..5]
 * set so the caller can report the reference's exact message. pg_obj_fetch copies the
 * result out (PG_HOST_OUTPUT: host pointers; else device pointers). */
int pg_load_obj(pg_builder *b, const uint8_t *bytes, uint64_t nbytes, uint32_t flags, void *stream,
                int64_t *out);
int pg_obj_fetch(pg_builder *b, double *V, int32_t *T, uint32_t flags, void *stream);

/* Grid statistics (stats.py:42-64) for the mesh of the last pg_count
 * (the grid's spec) and its grid G (u32[ncells+1]; PG_HOST_INPUT: host pointer):
 * out[0] = non-empty cells, out[1] = in-grid objects, out[2] = max cells per in-grid
 * object, out[3] = NO. The float attributes are derived from these on the host. */
int pg_grid_stats(pg_builder *b, const uint32_t *G, uint32_t flags, void *stream, uint64_t *out);

/* Sync-free build on device-resident V/T/G/O (no host round trip between K1 and the sort):
 * enqueues the whole of Alg. 1 on `stream` with every buffer sized for o_capacity pairs;
 * identical repeated calls replay a captured CUDA graph. pg_build_wait synchronises and
 * returns NO (PG_CAPACITY_ERROR if NO > o_capacity: enlarge O and call again). */
int pg_build_async(pg_builder *b, const double *V, int64_t nv, const int32_t *T, int64_t n,
                   const pg_spec *spec, uint32_t *G, uint32_t *O, uint64_t o_capacity, void *stream);
int pg_build_wait(pg_builder *b, uint64_t *no_out);

/* Record support (builders.py:138-140, 161-163): copy one stage of the last build into dst.
 *   stage 0: per-triangle record u32[n][4] = {lo_cell, mx, my, pair offset} (count==0 <=> dropped)
 *   stage 1: unsorted pair cell ids u32[NO]         stage 2: unsorted pair triangle ids u32[NO]
 *   stage 3: sorted cell ids u32[NO]
 * Stages 1-2 need PG_KEEP_STAGES on the preceding pg_finish. */
int pg_stage(pg_builder *b, int stage, void *dst, uint32_t flags, void *stream);

/* Plugin-seam replacement of kernels.radix_sort_pairs (_ckernels.pyx:21-50): stable LSD
 * sort of (key, value) u32 pairs over the 8*ceil(key_bits/8) low key bits (the digits the
 * reference's 8-bit passes cover). Inputs untouched; outputs are new buffers. */
int pg_radix_sort_pairs(pg_builder *b, const uint32_t *keys, const uint32_t *vals,
                        uint32_t *keys_out, uint32_t *vals_out, int64_t n, int key_bits,
                        uint32_t flags, void *stream);

/* Sharded (multi-GPU) building blocks, device pointers only:
 *   pg_pairs      -- after pg_count on a triangle shard: its <cell, triangle> pairs in
 *                    generation (object-major) order; triangle ids += val_offset (shard base);
 *                    optionally the histogram of cell >> coarse_shift (coarse_bins <= 7680
 *                    u32 bins, device) used to plan the slabs
 *   pg_partition  -- stable partition of pairs into cell slabs: slab = slab_of_bucket[key >>
 *                    bucket_shift] (nslabs <= 16); keys leave rebased by slab_base[slab];
 *                    slab_counts (device, 2^ceil(log2 nslabs) u32) receives the pairs per slab
 * None of the three synchronises the host: sizes stay on the device for the collectives.
 *   pg_sort_cells -- the Alg. 1 tail over arbitrary pairs with keys in [0, ncells): stable
 *                    radix sort + RLE/scatter/scan into G[ncells+1], O[n]
 *                    (builders.py:120-141) */
/* Fused partition + exchange (the "dispatch" all-to-all of the sharded build done by the
 * scatter itself): pg_partition_counts runs the slab upsweep (per-tile slab counts kept in the
 * builder; slab_counts as in pg_partition), then, once the ranks have exchanged their counts,
 * pg_partition_send scatters every pair straight into its slab owner's receive buffer:
 * dst_keys[s] / dst_vals[s] are device pointers (peer memory mapped into this process, e.g.
 * symmetric memory over NVLink) and dst_offset[s] this rank's element offset in slab s's
 * buffer; all three are host arrays of nslabs entries. Same pair order as pg_partition +
 * all-to-all; the caller synchronises the ranks before the receivers read. */
int pg_partition_counts(pg_builder *b, const uint32_t *keys, int64_t n, const uint32_t *slab_of_bucket,
                        int bucket_shift, int nslabs, uint32_t *slab_counts, void *stream);
int pg_partition_send(pg_builder *b, const uint32_t *keys, const uint32_t *vals, int64_t n,
                      const uint32_t *slab_of_bucket, int bucket_shift, int nslabs, const uint32_t *slab_base,
                      const uint64_t *dst_keys, const uint64_t *dst_vals, const uint64_t *dst_offset,
                      void *stream);
int pg_pairs(pg_builder *b, uint32_t *keys, uint32_t *vals, uint32_t val_offset, int coarse_shift,
             int coarse_bins, uint32_t *coarse_hist, void *stream);
int pg_partition(pg_builder *b, const uint32_t *keys, const uint32_t *vals, int64_t n,
                 const uint32_t *slab_of_bucket, int bucket_shift, int nslabs,
                 const uint32_t *slab_base, uint32_t *keys_out, uint32_t *vals_out,
                 uint32_t *slab_counts, void *stream);
int pg_sort_cells(pg_builder *b, const uint32_t *keys, const uint32_t *vals, int64_t n,
                  int64_t ncells, uint32_t *G, uint32_t *O, void *stream);
/* pg_sort_cells with flags: PG_GEN_ORDER (the sharded build's received slab, rank-ordered) */
int pg_sort_cells_flags(pg_builder *b, const uint32_t *keys, const uint32_t *vals, int64_t n,
                        int64_t ncells, uint32_t flags, uint32_t *G, uint32_t *O, void *stream);

/* Device-side small collectives of the sharded build over peer memory (no NCCL call, no host
 * round trip between the pair expansion and the slab plan; replaces the all-reduce of the
 * coarse histogram and the host-side plan_slabs of distributed.py):
 *   pg_peer_put  -- copy n u32 from src (device) to dsts[r] + dst_offset (elements) for the
 *                   nranks <= 16 device pointers in the host array dsts (peer memory mapped into
 *                   this process, e.g. symmetric memory); the caller barriers before readers read
 *   pg_slab_plan -- from the ranks' coarse histograms hists[r * nbuckets + b] (device u32,
 *                   nbuckets <= 4096): slab_of_bucket[nbuckets], slab_base[nslabs] (first cell
 *                   of each slab, u32) and plan[4*nslabs+2] = cuts[nslabs+1] | cell_lo[nslabs] |
 *                   cell_hi[nslabs] | pair_base[nslabs+1] (int64), all device; the same
 *                   arithmetic as distributed.plan_slabs */
int pg_count_result(pg_builder *b, uint64_t *no_out); /* after PG_DEFER + a stream synchronise */
/* After a PG_STATS pg_count: out[6] = {NO of this shard, index out of range (0/1), inverted
 * boxes with a negative count, with a zero count, with a positive count (two inverted axes),
 * positive ones with a cell outside [0, ncells)}. Summed over the ranks these give the
 * reference's verdict in its order (distributed.count_verdict): index range; negative count
 * (primitives.py:22-25); NO > 2^32-1 (builders.py:99-100); a zero count with any other kept
 * triangle (mark_boundaries, primitives.py:66-72); NO > 2^30 (primitives.py:29-31); cells of
 * inverted boxes (primitives.py:102-111, 135-136); ncells > 2^30 (builders.py:130). */
int pg_count_stats(pg_builder *b, int64_t *out);
/* Fused dispatch of the sharded build (pair expansion + slab partition + peer stores in one
 * kernel; replaces pg_pairs + pg_partition_counts + pg_partition_send):
 *   pg_coarse_hist -- after pg_count: the histogram of cell >> coarse_shift (coarse_bins <=
 *                     4096 u32 bins, device) computed from the triangles' cell boxes, before
 *                     any pair exists; equals pg_pairs' coarse histogram
 *   pg_pairs_send  -- expand the counted shard's pairs (triangle ids += val_offset), rank each
 *                    4096-pair tile by slab = slab_of_bucket[cell >> bucket_shift] and store
 *                    every pair into its slab owner's receive buffer (dst_keys/dst_vals[s] +
 *                    dst_offset[s] + this rank's running slab count; keys rebased by
 *                    slab_base[s]). The running counts are a decoupled look-back over the
 *                    tiles. Same pair order as pg_partition_send; the caller barriers the ranks
 *                    before the receivers read. Host arrays of nslabs device pointers/offsets. */
int pg_coarse_hist(pg_builder *b, int coarse_shift, int coarse_bins, uint32_t *coarse_hist, void *stream);
/* Optional parts compiled into this libpgrid (bit mask). The fused dispatch (pg_coarse_hist +
 * pg_pairs_send) measured slower than pg_partition_send and ships only in builds with
 * -DPGRID_FUSED_DISPATCH=1; without it both calls return PG_STATE_ERROR. */
#define PG_FEATURE_FUSED_DISPATCH 1
int pg_features(void);
int pg_pairs_send(pg_builder *b, uint32_t val_offset, const uint32_t *slab_of_bucket, int bucket_shift,
                  int nslabs, const uint32_t *slab_base, const uint64_t *dst_keys, const uint64_t *dst_vals,
                  const uint64_t *dst_offset, void *stream);
int pg_peer_put(const uint32_t *src, int64_t n, const uint64_t *dsts, int nranks, int64_t dst_offset,
                void *stream);
/* pg_peer_put of the builder's device pair count and K1 error flags (NO of its last pg_count,
 * u64 as two u32 words, then the flag word; exact even after a PG_DEFER count), so every rank
 * learns every rank's NO and flags with the count matrix: they agree on capacity overflows
 * and on falling back to the host-checked count when any shard flagged an error */
int pg_peer_put_count(pg_builder *b, const uint64_t *dsts, int nranks, int64_t dst_offset, void *stream);
int pg_slab_plan(const uint32_t *hists, int nranks, int nbuckets, int bucket_shift, int64_t ncells,
                 int nslabs, uint32_t *slab_of_bucket, uint32_t *slab_base, int64_t *plan, void *stream);

/* Wait for the device work (and PG_HOST_OUTPUT copies) of the last pg_finish on b. */
int pg_wait(pg_builder *b);
/* The reference's six phase times (BuildReport.phase_ms, builders.py:46-54: count, scan,
 * pairgen, sort, rle, finalize; device milliseconds) of the last pg_count + pg_finish on b,
 * e.g. after a PG_ASYNC finish and pg_wait (waits for it if needed). */
int pg_phase_times(pg_builder *b, float *phase_ms);

/* Profiling aid: with PGRID_KTIMES=1 in the environment, every launch of the calling thread's
 * last pg_count + pg_finish is bracketed by events; this writes "kernel microseconds" lines
 * (device time between consecutive launch completions) into buf. */
int pg_kernel_times(char *buf, int len);
int pg_kernel_timing(int on); /* switch the per-launch events on / off at run time */

/* Page-lock host memory so PG_HOST_* copies run at full PCIe rate (optional). */
int pg_host_register(void *ptr, uint64_t bytes);
int pg_host_unregister(void *ptr);
/* Page-locked host allocations (the Python side pools them for G/O outputs). */
int pg_host_alloc(uint64_t bytes, void **out);
int pg_host_free(void *ptr);

/* Number of device kernel launches issued by the last pg_count + pg_finish pair. */
int pg_last_launch_count(pg_builder *b);

/* Thread-local message for the last non-zero return code. */
const char *pg_last_error(void);

#ifdef __cplusplus
}
#endif

#endif /* PGRID_H */
