"""Host-side grid types of the drop-in boundary (mirror of pargrid.gridcore/geometry).

Only what the build path needs lives here: the mesh and spec containers the builder
accepts, the CompactGrid/cell-indexing contract it returns, and the host precondition
`spec_for_mesh` (bounds, padding and dims stay on the host; the
device receives these exact doubles). Every routine cites the reference line it mirrors
so parity can be checked line by line. The builder also accepts the reference's own
TriangleMesh / GridSpec objects (anything with .vertices/.triangles and
.bounds.lo/.bounds.hi/.cell_size/.dims).

Cell linearisation is x-fastest: cell = x + dx*(y + dy*z) (gridcore.py:3).
"""

import numpy as np

from .errors import InvariantError, SizeError

MAX_IDS = (1 << 32) - 1          # gridcore.py:11 -- cells and pairs fit 32-bit ids
MAX_SCAN_LEN = 1 << 30           # primitives.py:17 -- cap of every scanned array
BOUNDS_PAD = 1e-6                # gridcore.py:15


class Aabb:
    """Axis-aligned box (geometry.py:14-30)."""

    __slots__ = ("lo", "hi")

    def __init__(self, lo, hi):
        lo = np.asarray(lo, dtype=np.float64)
        hi = np.asarray(hi, dtype=np.float64)
        if lo.shape != (3,) or hi.shape != (3,):
            raise InvariantError("Aabb corners must be 3-D points")
        if np.isnan(lo).any() or np.isnan(hi).any():
            raise InvariantError("Aabb corners must not be NaN")
        if (lo > hi).any():
            raise InvariantError("Aabb requires lo <= hi")
        self.lo, self.hi = lo, hi

    def __repr__(self):
        return f"Aabb({self.lo.tolist()}, {self.hi.tolist()})"


class TriangleMesh:
    """Read-only f64 vertex / i32 triangle soup (geometry.py:33-52)."""

    __slots__ = ("vertices", "triangles")

    def __init__(self, vertices, triangles):
        v = np.ascontiguousarray(vertices, dtype=np.float64).reshape(-1, 3)
        t = np.ascontiguousarray(triangles, dtype=np.int32).reshape(-1, 3)
        if t.size and (t.min() < 0 or t.max() >= len(v)):
            raise InvariantError("triangle index out of range")
        v.setflags(write=False)
        t.setflags(write=False)
        self.vertices, self.triangles = v, t

    @property
    def ntriangles(self):
        return len(self.triangles)

    def __repr__(self):
        return f"TriangleMesh({len(self.vertices)} vertices, {len(self.triangles)} triangles)"


def cell_count(dims):
    """Product of dims with the 32-bit id check (gridcore.py:89-97)."""
    total = 1
    for d in dims:
        if d < 1:
            raise InvariantError("dims must be positive")
        total *= int(d)
    if total > MAX_IDS:
        raise SizeError(f"{total} cells exceed 32-bit id space")
    return total


class GridSpec:
    """Bounds + integer resolution; cell_size = extent / dims in f64 (gridcore.py:36-57)."""

    __slots__ = ("bounds", "dims", "cell_size")

    def __init__(self, bounds, dims):
        self.dims = tuple(int(d) for d in dims)
        if len(self.dims) != 3 or min(self.dims) < 1:
            raise InvariantError("dims must be three positive integers")
        cell_count(self.dims)
        extent = bounds.hi - bounds.lo
        if (extent <= 0).any():
            raise InvariantError("grid bounds must have positive extent per axis")
        self.bounds = bounds
        self.cell_size = extent / np.array(self.dims, dtype=np.float64)

    @property
    def ncells(self):
        return self.dims[0] * self.dims[1] * self.dims[2]

    def __repr__(self):
        return f"GridSpec(dims={self.dims}, bounds={self.bounds})"


class CompactGrid:
    """G (u32[ncells+1], G[0]=0, G[-1]=NO) + O (u32[NO]), read-only (gridcore.py:60-85)."""

    __slots__ = ("spec", "G", "O")

    def __init__(self, spec, G, O):
        G = np.ascontiguousarray(G, dtype=np.uint32)
        O = np.ascontiguousarray(O, dtype=np.uint32)
        if len(G) != spec.ncells + 1:
            raise InvariantError("G must have ncells + 1 entries")
        if G[0] != 0 or G[-1] != len(O):
            raise InvariantError("G must start at 0 and end at NO")
        G.setflags(write=False)
        O.setflags(write=False)
        self.spec, self.G, self.O = spec, G, O

    @property
    def no(self):
        return len(self.O)

    def __repr__(self):
        return f"CompactGrid({self.spec!r}, NO={self.no})"


def grids_equal(a, b):
    """Bit-level grid equality (gridcore.py:208-211)."""
    return (tuple(a.spec.dims) == tuple(b.spec.dims)
            and np.array_equal(a.G, b.G) and np.array_equal(a.O, b.O))


def mesh_bounds(mesh):
    """Tight bounds over ALL vertices, referenced or not (geometry.py:55-59)."""
    if len(mesh.vertices) == 0:
        raise InvariantError("cannot bound an empty mesh")
    return Aabb(mesh.vertices.min(axis=0), mesh.vertices.max(axis=0))


def compute_dims(bounds, ntriangles, density):
    """~density cells per triangle by volume (gridcore.py:170-182)."""
    if ntriangles < 1:
        raise InvariantError("need at least one triangle")
    extent = (bounds.hi - bounds.lo).astype(np.float64)
    longest = float(extent.max())
    if longest <= 0:
        return (1, 1, 1)
    extent = np.maximum(extent, BOUNDS_PAD * longest)
    per_axis = (density * ntriangles / float(extent.prod())) ** (1.0 / 3.0)
    dims = np.floor(extent * per_axis + 0.5).astype(np.int64)
    return tuple(int(d) for d in np.maximum(1, dims))


def spec_for_mesh(mesh, dims=None, density=5.0):
    """Padded mesh bounds + dims heuristic (gridcore.py:185-198)."""
    tight = mesh_bounds(mesh)
    longest = float((tight.hi - tight.lo).max())
    pad = BOUNDS_PAD * longest if longest > 0 else BOUNDS_PAD
    lo = tight.lo - pad
    hi = np.maximum(tight.hi + pad, lo + 2 * pad)   # degenerate axes get 2*pad of width
    padded = Aabb(lo, hi)
    if dims is None:
        dims = compute_dims(padded, mesh.ntriangles, density)
    return GridSpec(padded, dims)


def spec_from_bounds(lo, hi, ntriangles, dims=None, density=5.0):
    """spec_for_mesh from tight bounds already reduced over shards (min/max are exact, so a
    sharded build sees the same doubles as spec_for_mesh on the whole mesh)."""
    tight = Aabb(lo, hi)
    longest = float((tight.hi - tight.lo).max())
    pad = BOUNDS_PAD * longest if longest > 0 else BOUNDS_PAD
    plo = tight.lo - pad
    phi = np.maximum(tight.hi + pad, plo + 2 * pad)
    padded = Aabb(plo, phi)
    if dims is None:
        dims = compute_dims(padded, ntriangles, density)
    return GridSpec(padded, dims)


def key_bits_for(ncells):
    """Radix key width: (ncells-1).bit_length() (builders.py:124)."""
    return int(ncells - 1).bit_length()
