"""Ray casting over a built grid on the GPU, mirror of pargrid.traverse.

    ids, ts = dda_cast(grid, mesh, origins, directions, t_max)      # traverse.py:114-131
    hit = dda_traverse(grid, mesh, Ray(origin, direction))           # traverse.py:103-111
    caster = RayCaster(grid, mesh); ids, ts = caster.cast(o, d, tm)  # grid + mesh kept resident

Results are bit-identical to the reference's compiled lane (_ckernels.pyx:146-260): ids
int64 with -1 on a miss, ts float64 with +inf on a miss. The kernels are k_dda_prepare /
k_dda_cast (csrc/pgrid_dda.cuh) behind pg_dda_prepare / pg_dda_cast (include/pgrid.h).
There is no CPU path. `brute_force_cast` (traverse.py:134-170) is the reference's validation
oracle; it lives in oracle/ with the other checkers.
"""

import math
from dataclasses import dataclass

import numpy as np

from . import _native
from .errors import InvariantError
from .scenes import uniforms


@dataclass(frozen=True)
class Ray:
    """traverse.py:19-31: unit direction, positive t_max."""
    origin: tuple
    direction: tuple
    t_max: float = math.inf

    def __post_init__(self):
        d = np.asarray(self.direction, dtype=np.float64)
        if abs(float(np.linalg.norm(d)) - 1.0) > 1e-9:
            raise InvariantError("ray direction must be unit length")
        if not self.t_max > 0:
            raise InvariantError("t_max must be positive")


@dataclass(frozen=True)
class Hit:
    """traverse.py:34-37."""
    triangle_id: int
    t: float


def _rays(origins, directions, t_max):
    o = np.ascontiguousarray(origins, dtype=np.float64).reshape(-1, 3)
    d = np.ascontiguousarray(directions, dtype=np.float64).reshape(-1, 3)
    t = np.ascontiguousarray(t_max, dtype=np.float64).reshape(-1)
    if not (len(o) == len(d) == len(t)):
        raise InvariantError("origins, directions and t_max must have one entry per ray")
    return o, d, t


def _mesh(mesh):
    V = np.ascontiguousarray(mesh.vertices, dtype=np.float64).reshape(-1, 3)
    T = np.ascontiguousarray(mesh.triangles, dtype=np.int32).reshape(-1, 3)
    return V, T


def dda_cast(grid, mesh, origins, directions, t_max, device=0):
    """Batch traversal (traverse.py:114-121 -> kernels.dda_cast): (ids i64, ts f64)."""
    o, d, t = _rays(origins, directions, t_max)
    n = len(o)
    ids = np.full(n, -1, np.int64)
    ts = np.full(n, np.inf, np.float64)
    if n == 0:
        return ids, ts
    V, T = _mesh(mesh)
    b = _native.thread_builder(device)
    b.dda_prepare(V, len(V), T, len(T), flags=_native.PG_HOST_INPUT)
    G = np.ascontiguousarray(grid.G, dtype=np.uint32)
    O = np.ascontiguousarray(grid.O, dtype=np.uint32)
    b.dda_cast(G, O, len(O), grid.spec, o, d, t, n, ids, ts,
               flags=_native.PG_HOST_INPUT | _native.PG_HOST_OUTPUT | _native.PG_CHECK)
    return ids, ts


def dda_traverse(grid, mesh, ray, device=0):
    """Nearest hit found by walking the grid; None on a miss (traverse.py:103-111)."""
    ids, ts = dda_cast(grid, mesh, np.asarray([ray.origin], np.float64), np.asarray([ray.direction], np.float64),
                       np.asarray([ray.t_max], np.float64), device=device)
    if ids[0] < 0:
        return None
    return Hit(int(ids[0]), float(ts[0]))


class RayCaster:
    """Grid and prepared mesh resident on the device; rays in, hits out.

    `grid` may be a CompactGrid (copied to the device once) or a (spec, G, O) triple of
    device tensors from a device-resident build. cast() accepts host arrays (copied in and
    results copied out) or device tensors (no copies; results written into `out`)."""

    def __init__(self, grid, mesh, device=0):
        import torch
        self._torch = torch
        self.device = device
        self._b = _native.Builder(device)
        if isinstance(grid, tuple):
            self.spec, self.G, self.O = grid
        else:
            self.spec = grid.spec
            dev = torch.device("cuda", device)
            self.G = torch.from_numpy(np.array(grid.G, np.uint32).view(np.int32)).to(dev)
            self.O = torch.from_numpy(np.array(grid.O, np.uint32).view(np.int32)).to(dev)
        self.no = int(self.O.numel())
        self._pg = _native.PgSpec.from_spec(self.spec)
        V, T = mesh if isinstance(mesh, tuple) else _mesh(mesh)
        on_host = isinstance(V, np.ndarray)
        self._b.dda_prepare(V, len(V), T, len(T), flags=_native.PG_HOST_INPUT if on_host else 0,
                            stream=None if on_host else torch.cuda.current_stream(device).cuda_stream)

    def cast(self, origins, directions, t_max, out=None, stream=None, check=True):
        torch = self._torch
        if isinstance(origins, np.ndarray) or not hasattr(origins, "data_ptr"):
            o, d, t = _rays(origins, directions, t_max)
            n = len(o)
            ids = _native.pinned_pool.empty(n, np.int64)
            ts = _native.pinned_pool.empty(n, np.float64)
            if n:
                self._b.dda_cast(self.G, self.O, self.no, None, o, d, t, n, ids, ts,
                                 flags=_native.PG_HOST_RAYS | _native.PG_HOST_OUTPUT | (_native.PG_CHECK if check else 0),
                                 stream=stream, pgspec=self._pg)
            return ids, ts
        n = int(t_max.numel())
        if out is None:
            out = (torch.empty(n, dtype=torch.int64, device=origins.device),
                   torch.empty(n, dtype=torch.float64, device=origins.device))
        st = stream if stream is not None else torch.cuda.current_stream(origins.device).cuda_stream
        if n:
            self._b.dda_cast(self.G, self.O, self.no, None, origins, directions, t_max, n, out[0], out[1],
                             flags=_native.PG_CHECK if check else 0, stream=st, pgspec=self._pg)
        return out

    def launches(self):
        return self._b.launches()


def make_rays(bounds, n, seed):
    """Seeded rays aimed from outside the bounds at interior targets (cli.py:146-160)."""
    lo = np.asarray(bounds.lo, np.float64)
    hi = np.asarray(bounds.hi, np.float64)
    center = (lo + hi) / 2
    radius = float(np.linalg.norm(hi - lo)) * 1.2 + 1e-3
    u = uniforms(seed, 5 * n, 101).reshape(n, 5)
    phi = 2 * np.pi * u[:, 0]
    cos_th = 2 * u[:, 1] - 1
    sin_th = np.sqrt(np.maximum(0.0, 1 - cos_th ** 2))
    origins = center + radius * np.stack([sin_th * np.cos(phi), sin_th * np.sin(phi), cos_th], axis=1)
    targets = lo + u[:, 2:5] * (hi - lo)
    d = targets - origins
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    t_max = np.full(n, 4.0 * radius)
    return origins, d, t_max


def compare_hits(gids, gts, bids, bts, rel_tol=1e-6):
    """Indices where two casters disagree (cli.py:163-169)."""
    with np.errstate(invalid="ignore"):
        t_mismatch = (gids >= 0) & (bids >= 0) & (np.abs(gts - bts) > rel_tol * np.maximum(1.0, np.abs(bts)))
    return np.flatnonzero((gids != bids) | t_mismatch)
