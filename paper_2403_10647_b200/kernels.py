"""The "cuda" lane of the reference's kernel-backend registry (plugin seam).

The reference selects hot kernels through `pargrid.kernels` (kernels/__init__.py:10-67):
a backend is a module with BACKEND_NAME and five functions, registered in `_BACKENDS`.
The hot-path one is `radix_sort_pairs(keys u32[n], values u32[n], key_bits) -> (u32[n],
u32[n])` (_ckernels.pyx:21-50): stable LSD, new arrays, inputs untouched. This module
provides it on the GPU (C ABI pg_radix_sort_pairs), and `dda_cast` (_ckernels.pyx:146-260)
on the GPU ray caster (pg_dda_prepare / pg_dda_cast). The remaining three
(pairgen_sorted, compact_count, compact_fill) are the CPU baseline builders' per-object
loops; the GPU baselines run whole (builders.build_sorted / build_compact), so
`compat.install()` delegates those three to the reference's own C lane.
"""

import numpy as np

from . import _native
from .errors import InvariantError

BACKEND_NAME = "cuda"


def radix_sort_pairs(keys, values, key_bits):
    """Stable LSD radix sort of (key, value) u32 pairs on the GPU (_ckernels.pyx:21-50)."""
    k = np.ascontiguousarray(keys, dtype=np.uint32)
    v = np.ascontiguousarray(values, dtype=np.uint32)
    if k.shape != v.shape or k.ndim != 1:
        raise ValueError("keys and values must be 1-D arrays of equal length")
    ko = np.empty_like(k)
    vo = np.empty_like(v)
    b = _native.thread_builder()
    b.radix_sort_pairs(k, v, ko, vo, len(k), int(key_bits),
                       flags=_native.PG_HOST_INPUT | _native.PG_HOST_OUTPUT)
    return ko, vo


class _LaneSpec:
    """Adapter: the lane passes bounds / cell size / dims as loose arrays."""

    def __init__(self, blo, bhi, cs, dims):
        self.bounds = type("B", (), {"lo": np.asarray(blo, np.float64), "hi": np.asarray(bhi, np.float64)})()
        self.cell_size = np.asarray(cs, np.float64)
        self.dims = tuple(int(x) for x in dims)


def dda_cast(G, O, verts, tris, blo, bhi, cs, dims, origins, dirs, t_max):
    """Batch DDA traversal on the GPU; (ids i64 with -1 on a miss, ts f64) exactly as the
    compiled lane returns them (_ckernels.pyx:146-260)."""
    V = np.ascontiguousarray(verts, dtype=np.float64).reshape(-1, 3)
    T = np.ascontiguousarray(tris, dtype=np.int32).reshape(-1, 3)
    o = np.ascontiguousarray(origins, dtype=np.float64).reshape(-1, 3)
    d = np.ascontiguousarray(dirs, dtype=np.float64).reshape(-1, 3)
    t = np.ascontiguousarray(t_max, dtype=np.float64).reshape(-1)
    if not (len(o) == len(d) == len(t)):
        raise InvariantError("origins, dirs and t_max must have one entry per ray")
    n = len(o)
    ids = np.full(n, -1, np.int64)
    ts = np.full(n, np.inf, np.float64)
    if n == 0:
        return ids, ts
    Gc = np.ascontiguousarray(G, dtype=np.uint32)
    Oc = np.ascontiguousarray(O, dtype=np.uint32)
    b = _native.thread_builder()
    b.dda_prepare(V, len(V), T, len(T), flags=_native.PG_HOST_INPUT)
    b.dda_cast(Gc, Oc, len(Oc), _LaneSpec(blo, bhi, cs, dims), o, d, t, n, ids, ts,
               flags=_native.PG_HOST_INPUT | _native.PG_HOST_OUTPUT | _native.PG_CHECK)
    return ids, ts
