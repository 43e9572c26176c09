"""TEST INFRASTRUCTURE ONLY: ctypes front-end of the C parity oracle (pgrid_oracle.c).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference legs may
import this module, and only as the checker or the timed CPU baseline -- never on the
product path. See pgrid_oracle.c for the reference file:line each routine restates.
"""

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle.so")
_REF_DIR = os.path.join(_HERE, "_ref")

SIZE_ERROR = 1
INVARIANT_ERROR = 2


class OracleSizeError(Exception):
    """The oracle reproduced the reference's SizeError condition."""


class OracleInvariantError(Exception):
    """The oracle reproduced the reference's InvariantError condition (an inverted box)."""


class _Spec(ctypes.Structure):
    _fields_ = [("lo", ctypes.c_double * 3), ("hi", ctypes.c_double * 3),
                ("cell", ctypes.c_double * 3), ("dims", ctypes.c_int64 * 3)]


_lib = None


def build():
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        _lib = ctypes.CDLL(_LIB_PATH)
        p = ctypes.c_void_p
        _lib.orc_count.argtypes = [p, p, ctypes.c_int64, p, p]
        _lib.orc_build_parallel.argtypes = [p, p, ctypes.c_int64, p, p, p, p, p, p, p]
        _lib.orc_radix_sort_pairs.argtypes = [p, p, ctypes.c_int64, ctypes.c_int, p, p]
        _lib.orc_cell_boxes.argtypes = [p, p, ctypes.c_int64, p, p, p, p]
        _lib.orc_dda_cast.argtypes = [p, p, p, p, p, p, p, p, ctypes.c_int64, p, p]
        _lib.orc_brute_cast.argtypes = [p, p, ctypes.c_int64, p, p, p, ctypes.c_int64, p, p]
    return _lib


def _ptr(a):
    return ctypes.c_void_p(a.ctypes.data) if a is not None and a.size else ctypes.c_void_p(0)


def make_spec(lo, hi, cell, dims):
    s = _Spec()
    for k in range(3):
        s.lo[k] = float(lo[k])
        s.hi[k] = float(hi[k])
        s.cell[k] = float(cell[k])
        s.dims[k] = int(dims[k])
    return s


def spec_of(spec):
    """Accepts any GridSpec-like object (bounds.lo/hi, cell_size, dims)."""
    return make_spec(spec.bounds.lo, spec.bounds.hi, spec.cell_size, spec.dims)


def _arrays(vertices, triangles):
    V = np.ascontiguousarray(vertices, dtype=np.float64).reshape(-1, 3)
    T = np.ascontiguousarray(triangles, dtype=np.int32).reshape(-1, 3)
    return V, T


def cell_boxes(vertices, triangles, spec):
    V, T = _arrays(vertices, triangles)
    n = len(T)
    lo = np.zeros((n, 3), np.int32)
    hi = np.zeros((n, 3), np.int32)
    keep = np.zeros(n, np.uint8)
    s = spec_of(spec)
    lib().orc_cell_boxes(_ptr(V), _ptr(T), n, ctypes.byref(s), _ptr(lo), _ptr(hi), _ptr(keep))
    return lo, hi, keep.astype(bool)


def radix_sort_pairs(keys, values, key_bits):
    k = np.ascontiguousarray(keys, dtype=np.uint32)
    v = np.ascontiguousarray(values, dtype=np.uint32)
    ko = np.empty_like(k)
    vo = np.empty_like(v)
    rc = lib().orc_radix_sort_pairs(_ptr(k), _ptr(v), len(k), int(key_bits), _ptr(ko), _ptr(vo))
    if rc:
        raise MemoryError("oracle radix sort failed")
    return ko, vo


def build_parallel(vertices, triangles, spec, stages=False):
    """Returns (G u32[ncells+1], O u32[NO]) or, with stages=True, also a dict of the
    reference's record= arrays that the oracle reproduces."""
    V, T = _arrays(vertices, triangles)
    s = spec_of(spec)
    no = ctypes.c_int64(0)
    rc = lib().orc_count(_ptr(V), _ptr(T), len(T), ctypes.byref(s), ctypes.byref(no))
    if rc == SIZE_ERROR:
        raise OracleSizeError(f"NO={no.value}")
    if rc == INVARIANT_ERROR:
        raise OracleInvariantError("triangle cell box with hi < lo")
    if rc:
        raise MemoryError("oracle count failed")
    NO = no.value
    ncells = int(spec.dims[0]) * int(spec.dims[1]) * int(spec.dims[2])
    # ncells > 2^30 fails the G scan (SizeError) before G is written: no 4 GB buffer for it
    G = np.empty(ncells + 1 if ncells <= (1 << 30) else 1, np.uint32)
    O = np.empty(NO, np.uint32)
    st = [np.empty(NO, np.uint32) for _ in range(4)] if stages else [None] * 4
    rc = lib().orc_build_parallel(_ptr(V), _ptr(T), len(T), ctypes.byref(s), _ptr(G), _ptr(O),
                                  *[_ptr(a) for a in st])
    if rc == SIZE_ERROR:
        raise OracleSizeError(f"ncells={ncells}")
    if rc == INVARIANT_ERROR:
        raise OracleInvariantError("cell of an inverted box outside [0, ncells)")
    if rc:
        raise MemoryError("oracle build failed")
    if not stages:
        return G, O
    return G, O, {"no": NO, "global_c": st[0], "obj_ids": st[1],
                  "sorted_c": st[2], "sorted_o": st[3]}


def _rays(origins, dirs, t_max):
    o = np.ascontiguousarray(origins, dtype=np.float64).reshape(-1, 3)
    d = np.ascontiguousarray(dirs, dtype=np.float64).reshape(-1, 3)
    t = np.ascontiguousarray(t_max, dtype=np.float64).reshape(-1)
    return o, d, t


def dda_cast(G, O, vertices, triangles, spec, origins, dirs, t_max):
    """_ckernels.pyx:146-260 restated in C: (ids i64 with -1 on miss, ts f64)."""
    V, T = _arrays(vertices, triangles)
    G = np.ascontiguousarray(G, dtype=np.uint32)
    O = np.ascontiguousarray(O, dtype=np.uint32)
    o, d, t = _rays(origins, dirs, t_max)
    ids = np.empty(len(o), np.int64)
    ts = np.empty(len(o), np.float64)
    s = spec_of(spec)
    lib().orc_dda_cast(_ptr(G), _ptr(O), _ptr(V), _ptr(T), ctypes.byref(s), _ptr(o), _ptr(d), _ptr(t),
                       len(o), _ptr(ids), _ptr(ts))
    return ids, ts


def brute_cast(vertices, triangles, origins, dirs, t_max):
    """traverse.py:134-170 (all-triangles nearest hit) restated in C."""
    V, T = _arrays(vertices, triangles)
    o, d, t = _rays(origins, dirs, t_max)
    ids = np.empty(len(o), np.int64)
    ts = np.empty(len(o), np.float64)
    lib().orc_brute_cast(_ptr(V), _ptr(T), len(T), _ptr(o), _ptr(d), _ptr(t), len(o), _ptr(ids), _ptr(ts))
    return ids, ts


def reference_module():
    """The unmodified reference package built into oracle/_ref (None if absent)."""
    import sys
    if not os.path.isdir(os.path.join(_REF_DIR, "pargrid")):
        return None
    if _REF_DIR not in sys.path:
        sys.path.insert(0, _REF_DIR)
    try:
        import pargrid  # noqa: F401
        from pargrid import kernels
        if "c" in kernels.available_backends():
            kernels.set_backend("c")
        return pargrid
    except Exception:
        return None
