"""The "cuda" lane of the reference's kernel-backend registry (plugin seam).

The reference selects hot kernels through `pargrid.kernels` (kernels/__init__.py:10-67):
a backend is a module with BACKEND_NAME and five functions, registered in `_BACKENDS`.
The hot-path one is `radix_sort_pairs(keys u32[n], values u32[n], key_bits) -> (u32[n],
u32[n])` (_ckernels.pyx:21-50): stable LSD, new arrays, inputs untouched. This module
provides it on the GPU (C ABI pg_radix_sort_pairs). The other four entries
(pairgen_sorted, compact_count, compact_fill, dda_cast) belong to the baseline builders and
the ray caster, which are out of scope; `compat.install()` delegates them to
the reference's own C lane when this backend is registered into a live `pargrid`.
"""

import numpy as np

from . import _native

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
