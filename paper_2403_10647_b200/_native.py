"""ctypes binding of libpgrid.so (C ABI declared in include/pgrid.h).

The library is built in-tree (paper_2403_10647_b200/_lib/libpgrid.so) by
`__graft_entry__.build()` / `make -C paper_2403_10647_b200/csrc`. There is no fallback:
if the library or a CUDA device is missing, every build call raises loudly.
"""

import ctypes
import os
import threading

import numpy as np

from .errors import DeviceError, GridError, InvariantError, SizeError

LIB_PATH = os.environ.get("PGRID_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib", "libpgrid.so")

PG_OK = 0
PG_SIZE_ERROR = 1
PG_INVARIANT_ERROR = 2
PG_CUDA_ERROR = 3
PG_STATE_ERROR = 4
PG_CAPACITY_ERROR = 5
PG_PARSE_ERROR = 6

PG_HOST_INPUT = 1
PG_HOST_OUTPUT = 2
PG_KEEP_STAGES = 4
PG_HOST_RAYS = 8
PG_CHECK = 16
PG_ASYNC = 32
PG_DEFER = 64
PG_STATS = 128
PG_GEN_ORDER = 256

NPHASES = 6

# every symbol include/pgrid.h declares (checked by tests/test_boundary.py)
EXPORTS = ("pg_builder_create", "pg_builder_destroy", "pg_count", "pg_finish", "pg_stage",
           "pg_radix_sort_pairs", "pg_pairs", "pg_partition", "pg_sort_cells", "pg_sort_cells_flags", "pg_finish_baseline",
           "pg_dda_prepare", "pg_dda_cast", "pg_grid_stats", "pg_mesh_bounds", "pg_kernel_times", "pg_load_obj", "pg_obj_fetch", "pg_wait", "pg_kernel_timing", "pg_partition_counts", "pg_partition_send", "pg_peer_put", "pg_slab_plan", "pg_count_result",
           "pg_peer_put_count", "pg_coarse_hist", "pg_pairs_send", "pg_count_stats", "pg_features", "pg_phase_times",
           "pg_build_async",
           "pg_build_wait", "pg_host_register",
           "pg_host_unregister", "pg_host_alloc", "pg_host_free", "pg_last_launch_count",
           "pg_last_error")


class PgSpec(ctypes.Structure):
    """pg_spec: the exact host doubles of GridSpec (gridcore.py:36-57)."""
    _fields_ = [("lo", ctypes.c_double * 3), ("hi", ctypes.c_double * 3),
                ("cell", ctypes.c_double * 3), ("dims", ctypes.c_int64 * 3)]

    @classmethod
    def from_spec(cls, spec):
        s = cls()
        lo = np.asarray(spec.bounds.lo, dtype=np.float64)
        hi = np.asarray(spec.bounds.hi, dtype=np.float64)
        cell = np.asarray(spec.cell_size, dtype=np.float64)
        for k in range(3):
            s.lo[k] = float(lo[k])
            s.hi[k] = float(hi[k])
            s.cell[k] = float(cell[k])
            s.dims[k] = int(spec.dims[k])
        return s


_lib = None
_lib_lock = threading.Lock()


def load():
    """Load libpgrid.so (raises GridError if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise GridError(f"native library missing: {LIB_PATH} (run __graft_entry__.build())")
        lib = ctypes.CDLL(LIB_PATH)
        vp, i64, u32, u64 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint32, ctypes.c_uint64
        lib.pg_builder_create.argtypes = [ctypes.c_int, ctypes.POINTER(vp)]
        lib.pg_builder_destroy.argtypes = [vp]
        lib.pg_builder_destroy.restype = None
        lib.pg_count.argtypes = [vp, vp, i64, vp, i64, ctypes.POINTER(PgSpec), u32, vp,
                                 ctypes.POINTER(u64)]
        lib.pg_finish.argtypes = [vp, vp, vp, u32, vp, ctypes.POINTER(ctypes.c_float)]
        lib.pg_stage.argtypes = [vp, ctypes.c_int, vp, u32, vp]
        lib.pg_radix_sort_pairs.argtypes = [vp, vp, vp, vp, vp, i64, ctypes.c_int, u32, vp]
        lib.pg_pairs.argtypes = [vp, vp, vp, u32, ctypes.c_int, ctypes.c_int, vp, vp]
        lib.pg_partition.argtypes = [vp, vp, vp, i64, vp, ctypes.c_int, ctypes.c_int, vp, vp, vp, vp, vp]
        lib.pg_sort_cells.argtypes = [vp, vp, vp, i64, i64, vp, vp, vp]
        lib.pg_sort_cells_flags.argtypes = [vp, vp, vp, i64, i64, u32, vp, vp, vp]
        lib.pg_finish_baseline.argtypes = [vp, ctypes.c_int, vp, vp, u32, vp, ctypes.POINTER(ctypes.c_float),
                                           ctypes.POINTER(u64)]
        lib.pg_dda_prepare.argtypes = [vp, vp, i64, vp, i64, u32, vp]
        lib.pg_dda_cast.argtypes = [vp, vp, vp, i64, ctypes.POINTER(PgSpec), vp, vp, vp, i64, vp, vp, u32, vp]
        lib.pg_kernel_times.argtypes = [ctypes.c_char_p, ctypes.c_int]
        lib.pg_wait.argtypes = [vp]
        lib.pg_partition_counts.argtypes = [vp, vp, i64, vp, ctypes.c_int, ctypes.c_int, vp, vp]
        lib.pg_partition_send.argtypes = [vp, vp, vp, i64, vp, ctypes.c_int, ctypes.c_int, vp,
                                          ctypes.POINTER(u64), ctypes.POINTER(u64), ctypes.POINTER(u64), vp]
        lib.pg_kernel_timing.argtypes = [ctypes.c_int]
        lib.pg_count_result.argtypes = [vp, ctypes.POINTER(u64)]
        lib.pg_count_stats.argtypes = [vp, ctypes.POINTER(i64)]
        lib.pg_coarse_hist.argtypes = [vp, ctypes.c_int, ctypes.c_int, vp, vp]
        lib.pg_pairs_send.argtypes = [vp, u32, vp, ctypes.c_int, ctypes.c_int, vp, ctypes.POINTER(u64),
                                      ctypes.POINTER(u64), ctypes.POINTER(u64), vp]
        lib.pg_peer_put_count.argtypes = [vp, ctypes.POINTER(u64), ctypes.c_int, i64, vp]
        lib.pg_peer_put.argtypes = [vp, i64, ctypes.POINTER(u64), ctypes.c_int, i64, vp]
        lib.pg_slab_plan.argtypes = [vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, i64, ctypes.c_int, vp, vp, vp, vp]
        lib.pg_load_obj.argtypes = [vp, vp, u64, u32, vp, ctypes.POINTER(i64)]
        lib.pg_obj_fetch.argtypes = [vp, vp, vp, u32, vp]
        lib.pg_grid_stats.argtypes = [vp, vp, u32, vp, ctypes.POINTER(u64)]
        lib.pg_mesh_bounds.argtypes = [vp, vp, i64, u32, vp, ctypes.POINTER(ctypes.c_double),
                                       ctypes.POINTER(ctypes.c_double)]
        lib.pg_build_async.argtypes = [vp, vp, i64, vp, i64, ctypes.POINTER(PgSpec), vp, vp, u64, vp]
        lib.pg_build_wait.argtypes = [vp, ctypes.POINTER(u64)]
        lib.pg_host_register.argtypes = [vp, u64]
        lib.pg_host_unregister.argtypes = [vp]
        lib.pg_host_alloc.argtypes = [u64, ctypes.POINTER(vp)]
        lib.pg_host_free.argtypes = [vp]
        lib.pg_last_launch_count.argtypes = [vp]
        lib.pg_last_error.restype = ctypes.c_char_p
        lib.pg_phase_times.argtypes = [vp, ctypes.POINTER(ctypes.c_float)]
        lib.pg_phase_times.restype = ctypes.c_int
        lib.pg_features.argtypes = []
        lib.pg_features.restype = ctypes.c_int
        for name in ("pg_builder_create", "pg_count", "pg_finish", "pg_stage",
                     "pg_radix_sort_pairs", "pg_pairs", "pg_partition", "pg_sort_cells", "pg_sort_cells_flags",
                     "pg_finish_baseline", "pg_count_stats", "pg_dda_prepare", "pg_dda_cast", "pg_grid_stats", "pg_mesh_bounds", "pg_kernel_times", "pg_load_obj", "pg_obj_fetch", "pg_wait", "pg_kernel_timing", "pg_partition_counts", "pg_partition_send", "pg_peer_put", "pg_slab_plan",
           "pg_build_async", "pg_build_wait", "pg_host_register", "pg_host_unregister", "pg_host_alloc", "pg_host_free",
                     "pg_last_launch_count"):
            getattr(lib, name).restype = ctypes.c_int
        _lib = lib
    return _lib


def check(rc):
    """Map a C return code onto the reference's exception classes (errors.py:4-23)."""
    if rc == PG_OK:
        return
    msg = (load().pg_last_error() or b"").decode(errors="replace")
    if rc == PG_SIZE_ERROR:
        raise SizeError(msg)
    if rc == PG_INVARIANT_ERROR:
        raise InvariantError(msg)
    if rc == PG_CUDA_ERROR:
        raise DeviceError(msg)
    raise GridError(f"pgrid error {rc}: {msg}")


def ptr(a):
    """Raw data pointer of a numpy array or a torch tensor (None -> NULL)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data if a.size else None
    if hasattr(a, "data_ptr"):
        return a.data_ptr() if a.numel() else None
    return int(a)


class Builder:
    """One device workspace (libpgrid pg_builder). Use from one thread at a time."""

    def __init__(self, device=0):
        self._lib = load()
        h = ctypes.c_void_p()
        check(self._lib.pg_builder_create(int(device), ctypes.byref(h)))
        self._h = h
        self.device = device

    def close(self):
        if getattr(self, "_h", None):
            self._lib.pg_builder_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def count(self, V, nv, T, n, spec, flags=0, stream=None):
        s = PgSpec.from_spec(spec)
        no = ctypes.c_uint64(0)
        check(self._lib.pg_count(self._h, ptr(V), int(nv), ptr(T), int(n), ctypes.byref(s),
                                 flags, stream, ctypes.byref(no)))
        return int(no.value)

    def count_deferred(self, V, nv, T, n, spec, capacity, flags=0, stream=None):
        """pg_count with PG_DEFER: K1 enqueued, no host round trip; the pair building blocks
        run on the device count bounded by `capacity`. Returns the capacity."""
        s = PgSpec.from_spec(spec)
        no = ctypes.c_uint64(int(capacity))
        check(self._lib.pg_count(self._h, ptr(V), int(nv), ptr(T), int(n), ctypes.byref(s),
                                 flags | PG_DEFER, stream, ctypes.byref(no)))
        return int(capacity)

    def count_stats(self, V, nv, T, n, spec, flags=0, stream=None):
        """pg_count with PG_STATS (sharded builds): no local verdict; returns the shard's raw
        statistics int64[6] = {NO, index out of range, inverted boxes with negative / zero /
        positive counts, positive ones with a cell outside the grid}."""
        s = PgSpec.from_spec(spec)
        no = ctypes.c_uint64(0)
        check(self._lib.pg_count(self._h, ptr(V), int(nv), ptr(T), int(n), ctypes.byref(s),
                                 flags | PG_STATS, stream, ctypes.byref(no)))
        out = (ctypes.c_int64 * 6)()
        check(self._lib.pg_count_stats(self._h, out))
        return np.array(out[:], np.int64)

    def count_result(self):
        """NO of the last PG_DEFER count (the stream must have been synchronised since);
        -NO-1 when the deferred steps are void (NO exceeded the capacity, or an inverted box)."""
        no = ctypes.c_uint64(0)
        rc = self._lib.pg_count_result(self._h, ctypes.byref(no))
        if rc == PG_CAPACITY_ERROR:
            return -int(no.value) - 1      # always negative: rebuild on the host-counted path
        check(rc)
        return int(no.value)

    def peer_put_count(self, dsts, dst_offset, stream=None):
        """Put this builder's device NO (two u32 words) into every dsts[r] + dst_offset."""
        arr = ctypes.c_uint64 * len(dsts)
        check(self._lib.pg_peer_put_count(self._h, arr(*[int(x) for x in dsts]), len(dsts), int(dst_offset),
                                          stream))

    def finish(self, G, O, flags=0, stream=None, timed=True):
        phases = (ctypes.c_float * NPHASES)() if timed else None
        check(self._lib.pg_finish(self._h, ptr(G), ptr(O), flags, stream, phases))
        return list(phases) if timed else None

    def wait(self):
        """Wait for the last finish (PG_ASYNC) including its host-output copies."""
        check(self._lib.pg_wait(self._h))

    def phase_times(self):
        """The six reference phases (device ms) of the last count + finish on this builder."""
        out = (ctypes.c_float * NPHASES)()
        check(self._lib.pg_phase_times(self._h, out))
        return list(out)

    def finish_baseline(self, algo, G, O, flags=0, stream=None):
        """algo 1 = sorted grid, 2 = compact grid (builders.py:172-231); returns (phases, max_task_work)."""
        phases = (ctypes.c_float * NPHASES)()
        mw = ctypes.c_uint64(0)
        check(self._lib.pg_finish_baseline(self._h, int(algo), ptr(G), ptr(O), flags, stream, phases,
                                           ctypes.byref(mw)))
        return list(phases), int(mw.value)

    def dda_prepare(self, V, nv, T, n, flags=0, stream=None):
        check(self._lib.pg_dda_prepare(self._h, ptr(V), int(nv), ptr(T), int(n), flags, stream))

    def dda_cast(self, G, O, no, spec, origins, dirs, t_max, nrays, ids, ts, flags=0, stream=None, pgspec=None):
        s = pgspec or PgSpec.from_spec(spec)
        check(self._lib.pg_dda_cast(self._h, ptr(G), ptr(O), int(no), ctypes.byref(s), ptr(origins), ptr(dirs),
                                    ptr(t_max), int(nrays), ptr(ids), ptr(ts), flags, stream))

    def mesh_bounds(self, V, nv, flags=0, stream=None):
        """Tight per-axis (lo, hi) of all nv vertices, reduced on the device."""
        lo = (ctypes.c_double * 3)()
        hi = (ctypes.c_double * 3)()
        check(self._lib.pg_mesh_bounds(self._h, ptr(V), int(nv), flags, stream, lo, hi))
        return np.array(lo[:], np.float64), np.array(hi[:], np.float64)

    def load_obj(self, data, nbytes, flags=PG_HOST_INPUT, stream=None):
        """Parse an OBJ byte buffer on the device. Returns (rc, out[6]); rc is PG_OK or
        PG_PARSE_ERROR (out[2..5] locate the first bad line); other codes raise."""
        out = (ctypes.c_int64 * 6)()
        rc = self._lib.pg_load_obj(self._h, ptr(data), int(nbytes), flags, stream, out)
        if rc not in (PG_OK, PG_PARSE_ERROR):
            check(rc)
        return rc, [int(x) for x in out]

    def obj_fetch(self, V, T, flags=PG_HOST_OUTPUT, stream=None):
        check(self._lib.pg_obj_fetch(self._h, ptr(V), ptr(T), flags, stream))

    def grid_stats(self, G, flags=0, stream=None):
        """(nonempty cells, in-grid objects, max cells per object, NO) of the last count."""
        out = (ctypes.c_uint64 * 4)()
        check(self._lib.pg_grid_stats(self._h, ptr(G), flags, stream, out))
        return tuple(int(x) for x in out)

    def stage(self, stage, dst, flags=PG_HOST_OUTPUT, stream=None):
        check(self._lib.pg_stage(self._h, int(stage), ptr(dst), flags, stream))

    def radix_sort_pairs(self, keys, vals, keys_out, vals_out, n, key_bits, flags=0, stream=None):
        check(self._lib.pg_radix_sort_pairs(self._h, ptr(keys), ptr(vals), ptr(keys_out),
                                            ptr(vals_out), int(n), int(key_bits), flags, stream))

    def launches(self):
        return int(self._lib.pg_last_launch_count(self._h))

    def build_async(self, V, nv, T, n, spec, G, O, capacity, stream=None, pgspec=None):
        """Sync-free device build (CUDA-graph replay for repeated identical calls)."""
        s = pgspec or PgSpec.from_spec(spec)
        check(self._lib.pg_build_async(self._h, ptr(V), int(nv), ptr(T), int(n), ctypes.byref(s), ptr(G),
                                       ptr(O), int(capacity), stream))

    def build_wait(self):
        """Synchronise the last build_async; returns NO (-NO if it exceeded the capacity)."""
        no = ctypes.c_uint64(0)
        rc = self._lib.pg_build_wait(self._h, ctypes.byref(no))
        if rc == PG_CAPACITY_ERROR:
            return -int(no.value)
        check(rc)
        return int(no.value)

    # sharded-build building blocks (device pointers)
    def pairs(self, keys, vals, val_offset=0, coarse_shift=0, coarse_bins=0, coarse_hist=None, stream=None):
        """Generation-order pairs of the counted shard; with coarse_hist (device u32[coarse_bins])
        also the histogram of cell >> coarse_shift. No host synchronisation."""
        check(self._lib.pg_pairs(self._h, ptr(keys), ptr(vals), int(val_offset), int(coarse_shift),
                                 int(coarse_bins), ptr(coarse_hist), stream))

    def coarse_hist(self, coarse_shift, coarse_bins, coarse_hist, stream=None):
        """Histogram of cell >> coarse_shift of the counted mesh's pairs, from its cell boxes."""
        check(self._lib.pg_coarse_hist(self._h, int(coarse_shift), int(coarse_bins), ptr(coarse_hist), stream))

    def pairs_send(self, val_offset, table, shift, nslabs, base, dst_keys, dst_vals, dst_offset, stream=None):
        """Fused dispatch: expand the pairs and store each into its slab owner's buffer."""
        arr = ctypes.c_uint64 * len(dst_keys)
        check(self._lib.pg_pairs_send(self._h, int(val_offset), ptr(table), int(shift), int(nslabs), ptr(base),
                                      arr(*[int(x) for x in dst_keys]), arr(*[int(x) for x in dst_vals]),
                                      arr(*[int(x) for x in dst_offset]), stream))

    def partition(self, keys, vals, n, slab_of_bucket, bucket_shift, nslabs, slab_base, keys_out,
                  vals_out, slab_counts, stream=None):
        """Stable slab partition; slab_counts (device u32[2^ceil(log2 nslabs)]) receives the
        per-slab pair counts. No host synchronisation."""
        check(self._lib.pg_partition(self._h, ptr(keys), ptr(vals), int(n), ptr(slab_of_bucket),
                                     int(bucket_shift), int(nslabs), ptr(slab_base), ptr(keys_out),
                                     ptr(vals_out), ptr(slab_counts), stream))

    def partition_counts(self, keys, n, table, shift, nslabs, slab_counts, stream=None):
        check(self._lib.pg_partition_counts(self._h, ptr(keys), int(n), ptr(table), int(shift), int(nslabs),
                                            ptr(slab_counts), stream))

    def partition_send(self, keys, vals, n, table, shift, nslabs, base, dst_keys, dst_vals, dst_offset,
                       stream=None):
        arr = ctypes.c_uint64 * len(dst_keys)
        check(self._lib.pg_partition_send(self._h, ptr(keys), ptr(vals), int(n), ptr(table), int(shift),
                                          int(nslabs), ptr(base), arr(*[int(x) for x in dst_keys]),
                                          arr(*[int(x) for x in dst_vals]), arr(*[int(x) for x in dst_offset]),
                                          stream))

    def sort_cells(self, keys, vals, n, ncells, G, O, stream=None, flags=0):
        check(self._lib.pg_sort_cells_flags(self._h, ptr(keys), ptr(vals), int(n), int(ncells), flags, ptr(G),
                                            ptr(O), stream))


_tls = threading.local()


def peer_put(src, n, dsts, dst_offset, stream=None):
    """Copy n u32 from src (device) to every pointer in dsts at element offset dst_offset
    (one launch; peer memory over NVLink). No host synchronisation."""
    arr = ctypes.c_uint64 * len(dsts)
    check(load().pg_peer_put(ptr(src), int(n), arr(*[int(x) for x in dsts]), len(dsts), int(dst_offset), stream))


def slab_plan(hists, nranks, nbuckets, shift, ncells, nslabs, table, slab_base, plan, stream=None):
    """distributed.plan_slabs on the device from the ranks' coarse histograms (device u32
    [nranks * nbuckets]): table u32[nbuckets], slab_base u32[nslabs], plan int64[4*nslabs+2] =
    cuts | cell_lo | cell_hi | pair_base. No host synchronisation."""
    check(load().pg_slab_plan(ptr(hists), int(nranks), int(nbuckets), int(shift), int(ncells), int(nslabs),
                              ptr(table), ptr(slab_base), ptr(plan), stream))


PG_FEATURE_FUSED_DISPATCH = 1


def features():
    """Bit mask of the optional parts compiled into libpgrid (pg_features)."""
    return int(load().pg_features())


def kernel_timing(on):
    """Per-launch device timing (events after every launch) on / off for this process."""
    check(load().pg_kernel_timing(1 if on else 0))


def kernel_times():
    """[(kernel, microseconds)] of this thread's last pg_count + pg_finish (PGRID_KTIMES=1)."""
    buf = ctypes.create_string_buffer(1 << 16)
    check(load().pg_kernel_times(buf, len(buf)))
    out = []
    for line in buf.value.decode().splitlines():
        name, us = line.rsplit(" ", 1)
        out.append((name, float(us)))
    return out


def thread_builder(device=0):
    """Per-thread default builder (concurrent builds on distinct threads stay independent)."""
    b = getattr(_tls, "builder", None)
    if b is None or b.device != device:
        b = Builder(device)
        _tls.builder = b
    return b


def host_register(a):
    check(load().pg_host_register(ptr(a), a.nbytes))


def host_unregister(a):
    check(load().pg_host_unregister(ptr(a)))


class _PinnedBlock:
    """One page-locked allocation; returns itself to the pool when the last array view of it
    is garbage-collected."""

    __slots__ = ("ptr", "nbytes", "pool", "__weakref__")

    def __init__(self, ptr, nbytes, pool):
        self.ptr, self.nbytes, self.pool = ptr, nbytes, pool

    def __del__(self):
        try:
            self.pool._release(self)
        except Exception:
            pass


class PinnedPool:
    """Caching allocator of page-locked host memory for device->host outputs (G and O).

    Outputs in pageable numpy memory copy at ~5 GB/s; page-locked ones at PCIe rate. Blocks
    are recycled once the caller drops every array that views them, so steady-state builds
    allocate nothing. Arrays handed out are ordinary numpy arrays."""

    def __init__(self):
        self._free = {}   # nbytes -> [ptr]
        self._lock = threading.Lock()

    @staticmethod
    def _bucket(nbytes):
        return max(4096, 1 << (int(nbytes) - 1).bit_length())

    def empty(self, count, dtype=np.uint32):
        dtype = np.dtype(dtype)
        nbytes = int(count) * dtype.itemsize
        if nbytes == 0:
            return np.empty(count, dtype)
        size = self._bucket(nbytes)
        with self._lock:
            lst = self._free.get(size)
            ptr = lst.pop() if lst else None
        if ptr is None:
            out = ctypes.c_void_p()
            check(load().pg_host_alloc(size, ctypes.byref(out)))
            ptr = out.value
        block = _PinnedBlock(ptr, size, self)
        buf = (ctypes.c_uint8 * size).from_address(ptr)
        buf._pg_block = block   # keeps the block alive while any view exists
        return np.frombuffer(buf, dtype=dtype, count=int(count))

    def _release(self, block):
        with self._lock:
            self._free.setdefault(block.nbytes, []).append(block.ptr)


pinned_pool = PinnedPool()
