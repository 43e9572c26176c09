"""Drop-in `build_parallel` (pargrid.builders.build_parallel, builders.py:144-169) on B200.

Same signature, same outputs, same errors, same report as the reference:

    grid, report = build_parallel(mesh, spec, workers=None, record=None)

`mesh` is any TriangleMesh-like object (f64 vertices (nv,3), i32 triangles (N,3)) -- the
reference's own or ours; `spec` any GridSpec-like object. The arrays cross the C ABI
(include/pgrid.h) once: host -> device, four kernel stages, device -> host. There is no
CPU compute path; without libpgrid.so or a GPU this raises.
"""

import collections
import time
from dataclasses import dataclass, field

import numpy as np

from . import _native
from .errors import GridError
from .gridcore import CompactGrid

PHASES = ("count", "scan", "pairgen", "sort", "rle", "finalize")   # builders.py:19
PAIRGEN_OPS_PER_PAIR = 8                                           # builders.py:24

# Test hook (builders.py:26-28, 135-137): corrupt O[0] so harnesses can prove detection.
_fault_inject = False


@dataclass
class BuildReport:
    """builders.py:33-43."""
    algo: str
    no: int = 0
    max_task_work: int = 0
    total_work: int = 0
    phase_ms: dict = field(default_factory=lambda: {p: 0.0 for p in PHASES})

    @property
    def total_ms(self):
        return sum(self.phase_ms.values())


def _mesh_arrays(mesh):
    # index range validity (geometry.py:41-43) is checked on the device by K1
    V = np.ascontiguousarray(mesh.vertices, dtype=np.float64).reshape(-1, 3)
    T = np.ascontiguousarray(mesh.triangles, dtype=np.int32).reshape(-1, 3)
    return V, T


def _fill_record(record, b, n, no, G, O):
    """Reproduce the reference's record= arrays (builders.py:138-140, 161-163) from the
    device stages. The reference numbers objects after dropping out-of-grid triangles
    ("compacted" ids); the device keeps original ids, so the stage arrays are re-indexed
    here (presentation only -- G and O come straight from the device)."""
    recs = np.empty((n, 4), np.uint32)
    if n:
        b.stage(0, recs)
    off = recs[:, 3].astype(np.int64)
    counts = np.diff(np.append(off, no)) if n else np.zeros(0, np.int64)
    kept = np.flatnonzero(counts > 0)
    offsets = off[kept]
    gc = np.empty(no, np.uint32)
    go = np.empty(no, np.uint32)
    sc = np.empty(no, np.uint32)
    if no:
        b.stage(1, gc)
        b.stage(2, go)
        b.stage(3, sc)
    obj_ids = np.searchsorted(kept, go.astype(np.int64))
    rel_c = np.arange(no, dtype=np.int64) - offsets[obj_ids] if no else np.zeros(0, np.int64)
    cell_counts = np.diff(G.astype(np.int64))
    uniques = np.flatnonzero(cell_counts)
    record.update(v=counts[kept].astype(np.int64), offsets=offsets, no=int(no),
                  obj_ids=obj_ids.astype(np.int64), rel_c=rel_c, global_c=gc.astype(np.int64),
                  sorted_c=sc.astype(np.int64),
                  sorted_o=np.searchsorted(kept, O.astype(np.int64)).astype(np.int64),
                  rle_uniques=uniques.astype(np.int64), rle_counts=cell_counts[uniques],
                  g=G.astype(np.int64))


def build_parallel(mesh, spec, workers=None, record=None, device=0):
    """Alg. 1 BuildParallelGrid on the GPU; bit-identical to the reference.

    `workers` is accepted for signature parity (builders.py:144) and ignored: the output
    never depends on it (test_builders.py:148-154)."""
    del workers
    V, T = _mesh_arrays(mesh)
    n = len(T)
    b = _native.thread_builder(device)
    ms = {p: 0.0 for p in PHASES}
    t0 = time.perf_counter()
    no = b.count(V, len(V), T, n, spec, flags=_native.PG_HOST_INPUT)
    ms["count"] = (time.perf_counter() - t0) * 1e3
    ncells = int(spec.dims[0]) * int(spec.dims[1]) * int(spec.dims[2])
    # page-locked outputs (recycled once the caller drops them): D2H at PCIe rate
    G = _native.pinned_pool.empty(ncells + 1, np.uint32)
    O = _native.pinned_pool.empty(no, np.uint32)
    flags = _native.PG_HOST_OUTPUT | (_native.PG_KEEP_STAGES if record is not None else 0)
    phases = b.finish(G, O, flags=flags)
    for name, v in zip(PHASES, phases):
        if name != "count":
            ms[name] = float(v)
    if record is not None:
        _fill_record(record, b, n, no, G, O)
    if _fault_inject and no:
        O[0] ^= 1
    report = BuildReport("parallel", no=no,
                         max_task_work=PAIRGEN_OPS_PER_PAIR if no else 0,
                         total_work=PAIRGEN_OPS_PER_PAIR * no, phase_ms=ms)
    return CompactGrid(spec, G, O), report


def _baseline(algo, name, mesh, spec, device):
    V, T = _mesh_arrays(mesh)
    n = len(T)
    b = _native.thread_builder(device)
    ms = {p: 0.0 for p in PHASES}
    t0 = time.perf_counter()
    no = b.count(V, len(V), T, n, spec, flags=_native.PG_HOST_INPUT)
    count_ms = (time.perf_counter() - t0) * 1e3
    ncells = int(spec.dims[0]) * int(spec.dims[1]) * int(spec.dims[2])
    G = _native.pinned_pool.empty(ncells + 1, np.uint32)
    O = _native.pinned_pool.empty(no, np.uint32)
    phases, max_work = b.finish_baseline(algo, G, O, flags=_native.PG_HOST_OUTPUT)
    for p, v in zip(PHASES, phases):
        ms[p] = float(v)
    ms["count"] += count_ms
    return G, O, no, max_work, ms


def build_sorted(mesh, spec, workers=None, record=None, device=0):
    """The paper's sorted-grid baseline on the GPU (builders.py:172-192): one pair-generation
    task per triangle walks its whole cell box (the load imbalance Alg. 1 removes), then the
    same radix sort and G tail. Identical G/O to build_parallel.

    record= fills the same arrays as the reference's build_sorted; its pairs are, by
    construction, the parallel builder's pairs (object-major, x-fastest), so they are taken
    from that path's stage dumps."""
    del workers
    if record is not None:
        rec = {}
        build_parallel(mesh, spec, record=rec, device=device)
        record.update({k: rec[k] for k in ("v", "offsets", "no", "obj_ids", "global_c", "sorted_c", "sorted_o",
                                            "rle_uniques", "rle_counts", "g")})
    G, O, no, max_work, ms = _baseline(1, "sorted", mesh, spec, device)
    if _fault_inject and no:          # shared sorted tail (builders.py:135-137)
        O[0] ^= 1
    report = BuildReport("sorted", no=no, max_task_work=max_work if no else 0, total_work=no, phase_ms=ms)
    return CompactGrid(spec, G, O), report


def build_compact(mesh, spec, workers=None, device=0):
    """The paper's compact-grid baseline on the GPU (builders.py:195-231): per-cell counters,
    exclusive scan into G, slot claims, then a canonical per-cell sort. Identical G/O."""
    del workers
    G, O, no, max_work, ms = _baseline(2, "compact", mesh, spec, device)
    report = BuildReport("compact", no=no, max_task_work=max_work if no else 0, total_work=2 * no, phase_ms=ms)
    return CompactGrid(spec, G, O), report


def device_spec_for_mesh(V, nv, ntriangles, dims=None, density=5.0, device=0, stream=None):
    """gridcore.spec_for_mesh (gridcore.py:185-198) with the bounds reduction on the device:
    V may be a host array or a device tensor of nv x 3 doubles. The min / max are exact, so
    padding and dims (host arithmetic on six doubles) give the reference's spec bit for bit."""
    from .gridcore import spec_from_bounds
    b = _native.thread_builder(device)
    on_host = isinstance(V, np.ndarray)
    lo, hi = b.mesh_bounds(V, nv, flags=_native.PG_HOST_INPUT if on_host else 0, stream=stream)
    return spec_from_bounds(lo, hi, ntriangles, dims=dims, density=density)


def build_from_mesh(mesh, dims=None, density=5.0, device=0):
    """spec_for_mesh + build_parallel with one host->device copy of the mesh: bounds reduced on
    the device (pg_mesh_bounds), spec padded on the host, then Alg. 1 on the resident arrays.
    Returns (grid, report); grid.spec is the reference's spec_for_mesh(mesh, dims, density)."""
    import torch
    V, T = _mesh_arrays(mesh)
    n = len(T)
    dev = torch.device("cuda", device)
    st = torch.cuda.current_stream(dev).cuda_stream
    import warnings
    with warnings.catch_warnings():   # read-only mesh arrays: the tensors are only read
        warnings.simplefilter("ignore", UserWarning)
        Vd = torch.from_numpy(V).to(dev)
        Td = torch.from_numpy(T).to(dev)
    spec = device_spec_for_mesh(Vd, len(V), n, dims=dims, density=density, device=device, stream=st)
    b = _native.thread_builder(device)
    ms = {p: 0.0 for p in PHASES}
    t0 = time.perf_counter()
    no = b.count(Vd, len(V), Td, n, spec, flags=0, stream=st)
    ms["count"] = (time.perf_counter() - t0) * 1e3
    G = _native.pinned_pool.empty(spec.ncells + 1, np.uint32)
    O = _native.pinned_pool.empty(no, np.uint32)
    phases = b.finish(G, O, flags=_native.PG_HOST_OUTPUT, stream=st)
    for name, v in zip(PHASES, phases):
        if name != "count":
            ms[name] = float(v)
    report = BuildReport("parallel", no=no, max_task_work=PAIRGEN_OPS_PER_PAIR if no else 0,
                         total_work=PAIRGEN_OPS_PER_PAIR * no, phase_ms=ms)
    return CompactGrid(spec, G, O), report


class BuildPipeline:
    """Overlapped end-to-end builds of a stream of meshes (host arrays in, host grids out).

    Each slot owns a libpgrid workspace and a CUDA stream. submit() copies the mesh in and
    enqueues Alg. 1 plus the device->host copy of G/O, then returns; result() hands back the
    oldest build once its copies have landed. With two slots the host->device copy of build
    i+1 runs while build i sorts and copies its grid out (separate copy engines), so the
    steady state is bound by the input copy alone. Same grids as build_parallel."""

    def __init__(self, device=0, depth=2):
        import torch
        self.device = device
        self._slots = [(_native.Builder(device), torch.cuda.Stream(device)) for _ in range(depth)]
        self._next = 0
        self._pending = collections.deque()
        self._cap = None    # pair capacity of deferred counts: 1.25 x the largest NO seen

    def submit(self, mesh, spec):
        """Enqueue one build (errors of the build are raised by its result()). After the first,
        the pair count is not read back (PG_DEFER):
        the copy in, Alg. 1 and the copies out are all enqueued without a host round trip, so
        the next submit's input copy follows this one's on the copy engine at once. O is
        copied at the capacity and cut to NO in result(); an overflow rebuilds that mesh."""
        if len(self._pending) == len(self._slots):
            raise RuntimeError("pipeline full: collect a result() first")
        b, st = self._slots[self._next]
        self._next = (self._next + 1) % len(self._slots)
        V, T = _mesh_arrays(mesh)
        t0 = time.perf_counter()
        deferred = self._cap is not None and len(T) > 0
        try:
            if deferred:
                no = b.count_deferred(V, len(V), T, len(T), spec, self._cap, flags=_native.PG_HOST_INPUT,
                                      stream=st.cuda_stream)
            else:
                no = b.count(V, len(V), T, len(T), spec, flags=_native.PG_HOST_INPUT, stream=st.cuda_stream)
        except GridError as e:        # reported by result(), in submission order, like deferred errors
            self._pending.append((e,))
            return
        count_ms = (time.perf_counter() - t0) * 1e3
        ncells = int(spec.dims[0]) * int(spec.dims[1]) * int(spec.dims[2])
        G = _native.pinned_pool.empty(ncells + 1, np.uint32)
        O = _native.pinned_pool.empty(no, np.uint32)
        b.finish(G, O, flags=_native.PG_HOST_OUTPUT | _native.PG_ASYNC, stream=st.cuda_stream, timed=False)
        self._pending.append((b, mesh, spec, G, O, no, count_ms, deferred))

    def _learn(self, no):
        cap = int(no * 1.0625) + 4096      # the O copy-out carries the slack
        self._cap = cap if self._cap is None else max(self._cap, cap)

    @property
    def capacity(self):
        """Pairs copied out per deferred build (O is read back at this size, then cut)."""
        return self._cap

    def result(self):
        entry = self._pending.popleft()
        if len(entry) == 1:
            raise entry[0]
        b, mesh, spec, G, O, no, count_ms, deferred = entry
        b.wait()
        if deferred:
            no = b.count_result()
            if no < 0:            # over the capacity (or a corner the host path resolves): rebuild
                self._learn(-no - 1)
                return build_parallel(mesh, spec, device=self.device)
            O = O[:no]
        self._learn(no)
        # all six phases (builders.py:46-54): the device times of this build's kernels (its
        # events), the host time of the submit (copy enqueue + count) added to "count"
        ms = dict(zip(PHASES, (float(x) for x in b.phase_times())))
        ms["count"] += count_ms
        report = BuildReport("parallel", no=no, max_task_work=PAIRGEN_OPS_PER_PAIR if no else 0,
                             total_work=PAIRGEN_OPS_PER_PAIR * no, phase_ms=ms)
        return CompactGrid(spec, G, O), report

    def __len__(self):
        return len(self._pending)


def build_many(items, device=0, depth=2):
    """Yield (grid, report) for each (mesh, spec) of `items`, builds overlapped (BuildPipeline)."""
    pipe = BuildPipeline(device, depth)
    for mesh, spec in items:
        if len(pipe) == depth:
            yield pipe.result()
        pipe.submit(mesh, spec)
    while len(pipe):
        yield pipe.result()
