"""Deterministic synthetic scenes (inputs for tests and bench; not part of the build path).

`gen_scene(kind, n, seed)` for kind in {uniform, skewed, walls} reproduces the
reference's generator bit for bit (geometry.py:124-207): the same counter-based
splitmix64 streams and the same per-scene arithmetic, with the walls loop vectorised.

Two repo-defined kinds implement SURVEY.md §8d for BASELINE.json's configs 2 and 3:
  lognormal -- triangle sizes exp(1.1 z) cell edges, clipped to [0.05, 9]
               (1..~1000 cells per object), z standard normal (Box-Muller, streams 40/41),
               centres stream 42, jitter stream 43;
  arch      -- 64 axis-aligned wall quads (the reference walls formula, stream 30) plus
               n-128 small clutter triangles of size 0.35 cell edges (stream 31).
Sizes derived from transcendental functions are snapped to a dyadic grid so that the
generated doubles do not depend on the host's libm / SIMD dispatch (the GPU box and this
container must produce the same arrays for the golden hashes to apply).
"""

import numpy as np

from .errors import InvariantError
from .gridcore import TriangleMesh

_GAMMA = np.uint64(0x9E3779B97F4A7C15)
_MIX1 = np.uint64(0xBF58476D1CE4E5B9)
_MIX2 = np.uint64(0x94D049BB133111EB)
_SEED_MUL = 0x632BE59BD9B4E019


def _splitmix64_finalize(x):
    """Steele et al. splitmix64 finaliser (geometry.py:124-131)."""
    x = x ^ (x >> np.uint64(30))
    x = x * _MIX1
    x = x ^ (x >> np.uint64(27))
    x = x * _MIX2
    return x ^ (x >> np.uint64(31))


def uniforms(seed, count, stream=0, start=0):
    """`count` doubles in [0,1) from the counter-based stream (geometry.py:134-139);
    `start` skips the first draws, so uniforms(s, b - a, st, a) == uniforms(s, b, st)[a:b]."""
    base = np.uint64((seed * _SEED_MUL + stream) & 0xFFFFFFFFFFFFFFFF)
    with np.errstate(over="ignore"):
        ctr = np.arange(start + 1, start + count + 1, dtype=np.uint64) * _GAMMA + base
        bits = _splitmix64_finalize(ctr)
    return (bits >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def small_triangles(n, seed, stream, size):
    """n jittered triangles of edge ~size in the unit cube (geometry.py:142-145).
    `size` may be a scalar or a per-triangle array."""
    size = np.asarray(size, dtype=np.float64)
    s_c = size[:, None] if size.ndim else size
    s_j = size[:, None, None] if size.ndim else size
    centres = uniforms(seed, 3 * n, stream).reshape(n, 3) * (1.0 - s_c) + s_c / 2
    jitter = (uniforms(seed, 9 * n, stream + 1).reshape(n, 3, 3) - 0.5) * s_j
    return centres[:, None, :] + jitter


def _wall_quads(nquads, seed):
    """Axis-aligned quads split in two triangles (geometry.py:180-200), vectorised."""
    tris = np.empty((2 * nquads, 3, 3))
    if nquads == 0:
        return tris
    u = uniforms(seed, 8 * nquads, 30).reshape(nquads, 8)
    a = (u[:, 0] * 3).astype(np.int64)
    b = (a + 1) % 3
    c = (a + 2) % 3
    lo1 = u[:, 2] * 0.6
    hi1 = lo1 + 0.3 + u[:, 3] * (1.0 - lo1 - 0.3)
    lo2 = u[:, 4] * 0.6
    hi2 = lo2 + 0.3 + u[:, 5] * (1.0 - lo2 - 0.3)
    corners = np.zeros((nquads, 4, 3))
    q = np.arange(nquads)
    corners[q, :, a] = u[:, 1][:, None]
    corners[q, :, b] = np.stack([lo1, hi1, hi1, lo1], axis=1)
    corners[q, :, c] = np.stack([lo2, lo2, hi2, hi2], axis=1)
    tris[0::2] = corners[:, [0, 1, 2]]
    tris[1::2] = corners[:, [0, 2, 3]]
    return tris


def _small_triangles_range(a, b, seed, stream, size):
    """Triangles [a, b) of small_triangles(n, seed, stream, size) (scalar size)."""
    k = b - a
    centres = uniforms(seed, 3 * k, stream, 3 * a).reshape(k, 3) * (1.0 - size) + size / 2
    jitter = (uniforms(seed, 9 * k, stream + 1, 9 * a).reshape(k, 3, 3) - 0.5) * size
    return centres[:, None, :] + jitter


def gen_uniform_chunked(n, seed, chunk=10_000_000):
    """gen_scene("uniform", n, seed) built chunk by chunk (bounded temporaries for 100M+
    triangles); bit-identical to the one-shot generator."""
    size = min(0.05, 0.6 * n ** (-1.0 / 3.0))
    V = np.empty((3 * n, 3), dtype=np.float64)
    for a in range(0, n, chunk):
        b = min(n, a + chunk)
        V[3 * a:3 * b] = _small_triangles_range(a, b, seed, 10, size).reshape(-1, 3)
    return TriangleMesh(V, np.arange(3 * n, dtype=np.int32).reshape(n, 3))


def gen_uniform_shard(n, seed, lo, hi):
    """Triangles [lo, hi) of gen_scene("uniform", n, seed) as an unshared-vertex soup."""
    size = min(0.05, 0.6 * n ** (-1.0 / 3.0))
    return _soup(_small_triangles_range(lo, hi, seed, 10, size))


def gen_shard(kind, n, seed, density, lo, hi):
    """Triangles [lo, hi) of the uniform / arch scene of n triangles (sharded builds: each
    rank generates only its own shard)."""
    if kind == "uniform":
        return gen_uniform_shard(n, seed, lo, hi)
    if kind == "arch":
        return gen_arch_shard(n, seed, density, lo, hi)
    raise InvariantError(f"no shard generator for {kind!r}")


def gen_arch_shard(n, seed, density, lo, hi):
    """Triangles [lo, hi) of gen_scene("arch", n, seed, density) as an unshared-vertex soup
    (for sharded builds: each rank generates only its own shard)."""
    edge = _cell_edge(n, density)
    nquads = min(64, n // 2)
    nwall = 2 * nquads
    parts = []
    if lo < nwall:
        parts.append(_wall_quads(nquads, seed)[lo:min(hi, nwall)])
    a, b = max(lo, nwall) - nwall, hi - nwall
    if b > a:
        parts.append(_small_triangles_range(a, b, seed, 31, 0.35 * edge))
    tris = np.concatenate(parts, axis=0) if parts else np.empty((0, 3, 3))
    return _soup(tris)


def _snap(x, bits):
    return np.rint(np.asarray(x, dtype=np.float64) * 2.0 ** bits) / 2.0 ** bits


def _cell_edge(n, density):
    """Approximate world edge of one cell when a unit cube holds density*n cells."""
    return float(_snap((density * n) ** (-1.0 / 3.0), 40))


def _soup(tris):
    nt = len(tris)
    return TriangleMesh(tris.reshape(nt * 3, 3), np.arange(nt * 3, dtype=np.int32).reshape(nt, 3))


def gen_scene(kind, n, seed, density=5.0):
    """Deterministic scene with n triangles in the unit cube (geometry.py:148-207 for the
    reference kinds; SURVEY.md §8d for lognormal/arch). `density` only shapes the
    repo-defined kinds (their sizes are expressed in cell edges)."""
    if n < 1:
        raise InvariantError("scene needs at least one triangle")
    if kind == "uniform":
        tris = small_triangles(n, seed, 10, min(0.05, 0.6 * n ** (-1.0 / 3.0)))
    elif kind == "skewed":
        k = min(max(1, n // 10000), n)
        tiny = small_triangles(n - k, seed, 20, 0.01) if n > k else np.empty((0, 3, 3))
        big = np.empty((k, 3, 3))
        big[0] = [(0.0, 0.0, 0.0), (1.0, 1.0, 0.0), (1.0, 0.0, 1.0)]
        if k > 1:
            m = k - 1
            h = 0.15 + 0.25 * uniforms(seed, m, 22)
            c = uniforms(seed, 3 * m, 23).reshape(m, 3)
            c = h[:, None] + c * (1.0 - 2.0 * h[:, None])
            big[1:, 0] = c + np.stack([-h, -h, -h], axis=1)
            big[1:, 1] = c + np.stack([h, h, -h], axis=1)
            big[1:, 2] = c + np.stack([h, -h, h], axis=1)
        tris = np.concatenate([big, tiny], axis=0)
    elif kind == "walls":
        nquads = min(max(1, n // 10), n // 2)
        walls = _wall_quads(nquads, seed)
        nclutter = n - 2 * nquads
        clutter = small_triangles(nclutter, seed, 31, 0.02) if nclutter else np.empty((0, 3, 3))
        tris = np.concatenate([walls, clutter], axis=0)
    elif kind == "lognormal":
        edge = _cell_edge(n, density)
        u1 = 1.0 - uniforms(seed, n, 40)            # (0, 1]
        u2 = uniforms(seed, n, 41)
        z = np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u2)
        cells = _snap(np.clip(np.exp(1.1 * z), 0.05, 9.0), 12)
        size = np.minimum(cells * edge, 0.5)
        centres = uniforms(seed, 3 * n, 42).reshape(n, 3) * (1.0 - size[:, None]) + size[:, None] / 2
        jitter = (uniforms(seed, 9 * n, 43).reshape(n, 3, 3) - 0.5) * size[:, None, None]
        tris = centres[:, None, :] + jitter
    elif kind == "arch":
        edge = _cell_edge(n, density)
        nquads = min(64, n // 2)
        walls = _wall_quads(nquads, seed)
        nclutter = n - 2 * nquads
        clutter = (small_triangles(nclutter, seed, 31, 0.35 * edge) if nclutter
                   else np.empty((0, 3, 3)))
        tris = np.concatenate([walls, clutter], axis=0)
    else:
        raise InvariantError(f"unknown scene kind {kind!r}")
    return _soup(tris)


# BASELINE.json configs -> (kind, n, seed, density). Config 3 is the headline workload.
CONFIGS = {
    "cfg1": ("uniform", 100_000, 7, 5.0),
    "cfg2": ("lognormal", 1_000_000, 7, 5.0),
    "cfg3": ("arch", 10_000_000, 7, 4.0),
    "cfg3u": ("uniform", 10_000_000, 7, 5.0),
    # config 4: the 10M uniform scene at grid densities 1 -> 64 (24 -> 30 key bits)
    **{f"cfg4_d{d}": ("uniform", 10_000_000, 7, float(d)) for d in (1, 2, 4, 8, 16, 32, 64)},
    # config 5: 100M triangles (uniform; arch for the sharded north-star run)
    "cfg5": ("uniform", 100_000_000, 7, 5.0),
    "cfg5a": ("arch", 100_000_000, 7, 4.0),
}


def gen_scene_large(kind, n, seed, density=5.0, chunk=10_000_000):
    """gen_scene(kind, n, seed, density) with bounded temporaries for 100M+ triangles
    (uniform / arch): generated chunk by chunk, bit-identical to the one-shot generator."""
    if kind == "uniform":
        return gen_uniform_chunked(n, seed, chunk)
    if kind != "arch":
        return gen_scene(kind, n, seed, density)
    V = np.empty((3 * n, 3), dtype=np.float64)
    for a in range(0, n, chunk):
        b = min(n, a + chunk)
        V[3 * a:3 * b] = gen_arch_shard(n, seed, density, a, b).vertices
    return TriangleMesh(V, np.arange(3 * n, dtype=np.int32).reshape(n, 3))


def config_scene(name):
    """(mesh, spec) for a named BASELINE config."""
    from .gridcore import spec_for_mesh
    kind, n, seed, density = CONFIGS[name]
    mesh = gen_scene_large(kind, n, seed, density) if n > 20_000_000 else gen_scene(kind, n, seed, density)
    return mesh, spec_for_mesh(mesh, density=density)
