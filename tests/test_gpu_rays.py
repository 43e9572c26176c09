"""GPU ray casting against the reference's compiled lane: golden ids/ts
(tests/golden/rays.npz, bit-exact), the C oracle on random rays, and the API's error paths."""

import numpy as np
import pytest

import oracle
from paper_2403_10647_b200 import _native, builders, gen_scene, spec_for_mesh, traverse
from paper_2403_10647_b200.errors import InvariantError
from paper_2403_10647_b200.gridcore import Aabb, CompactGrid, GridSpec, TriangleMesh
from util import RAY_CASES, ray_case, sha

pytestmark = pytest.mark.gpu


def bits_equal(a, b):
    return np.array_equal(np.asarray(a, np.float64).view(np.uint64), np.asarray(b, np.float64).view(np.uint64))


@pytest.mark.parametrize("name", RAY_CASES)
def test_golden_rays(rays, name):
    arrays, meta = rays
    mesh, spec, o, d, t = ray_case(rays, name)
    grid, _ = builders.build_parallel(mesh, spec)
    assert sha(grid.G) == meta[name]["G_sha256"] and sha(grid.O) == meta[name]["O_sha256"]
    ids, ts = traverse.dda_cast(grid, mesh, o, d, t)
    assert np.array_equal(ids, arrays[f"{name}/ids"])
    assert bits_equal(ts, arrays[f"{name}/ts"])


@pytest.mark.parametrize("name", ["validate_3", "inside_walls", "cfg1", "arch1m"])
def test_resident_caster_host_and_device_rays(rays, name):
    import torch
    arrays, _ = rays
    mesh, spec, o, d, t = ray_case(rays, name)
    grid, _ = builders.build_parallel(mesh, spec)
    caster = traverse.RayCaster(grid, mesh)
    ids, ts = caster.cast(o, d, t)
    assert np.array_equal(ids, arrays[f"{name}/ids"]) and bits_equal(ts, arrays[f"{name}/ts"])
    dev = [torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in (o, d, t)]
    gi, gt = caster.cast(*dev)
    torch.cuda.synchronize()
    assert np.array_equal(gi.cpu().numpy(), arrays[f"{name}/ids"]) and bits_equal(gt.cpu().numpy(), arrays[f"{name}/ts"])
    assert caster.launches() == 1


def test_device_resident_build_then_cast():
    """Grid built on the device (pg_count/pg_finish into device tensors) and cast in place."""
    import torch
    mesh = gen_scene("walls", 3000, 5)
    spec = spec_for_mesh(mesh)
    b = _native.Builder(0)
    Vd = torch.from_numpy(mesh.vertices.copy()).cuda()
    Td = torch.from_numpy(mesh.triangles.copy()).cuda()
    st = torch.cuda.current_stream().cuda_stream
    no = b.count(Vd, len(mesh.vertices), Td, len(mesh.triangles), spec, 0, st)
    Gd = torch.empty(spec.ncells + 1, dtype=torch.int32, device="cuda")
    Od = torch.empty(max(no, 1), dtype=torch.int32, device="cuda")
    b.finish(Gd, Od, 0, st, timed=False)
    caster = traverse.RayCaster((spec, Gd, Od[:no]), (Vd, Td))
    o, d, t = traverse.make_rays(spec.bounds, 3000, 8)
    ids, ts = caster.cast(o, d, t)
    G, O = oracle.build_parallel(mesh.vertices, mesh.triangles, spec)
    want = oracle.dda_cast(G, O, mesh.vertices, mesh.triangles, spec, o, d, t)
    assert np.array_equal(ids, want[0]) and bits_equal(ts, want[1])


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_random_rays_vs_oracle(seed):
    rng = np.random.default_rng(seed)
    kind = ("uniform", "skewed", "walls")[seed - 1]
    mesh = gen_scene(kind, 5000 * seed, seed)
    dims = tuple(int(x) for x in rng.integers(1, 60, 3))
    spec = spec_for_mesh(mesh, dims=dims)
    grid, _ = builders.build_parallel(mesh, spec)
    n = 20000
    o = spec.bounds.lo - 0.3 + rng.random((n, 3)) * (spec.bounds.hi - spec.bounds.lo + 0.6)
    d = rng.normal(size=(n, 3))
    d[1::7, 0] = 0.0
    d[::11, 1:] = 0.0
    d[::11, 0] = -1.0
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    t = np.where(rng.random(n) < 0.2, np.inf, rng.random(n) * 2)
    ids, ts = traverse.dda_cast(grid, mesh, o, d, t)
    want = oracle.dda_cast(grid.G, grid.O, mesh.vertices, mesh.triangles, spec, o, d, t)
    assert np.array_equal(ids, want[0]) and bits_equal(ts, want[1])
    assert (ids >= 0).sum() > n // 20


def test_reference_traverse_cases():
    """test_traverse.py:135-152, 166-171 through the GPU caster."""
    mesh = TriangleMesh([[0, 0, 0], [1, 0, 0], [0, 1, 0]], [[0, 1, 2]])
    grid, _ = builders.build_parallel(mesh, spec_for_mesh(mesh, dims=(2, 2, 1)))
    hit = traverse.dda_traverse(grid, mesh, traverse.Ray((0.25, 0.25, -1), (0, 0, 1)))
    assert hit is not None and hit.triangle_id == 0 and hit.t == pytest.approx(1.0)
    assert traverse.dda_traverse(grid, mesh, traverse.Ray((5, 5, -1), (0, 0, 1))) is None
    assert traverse.dda_traverse(grid, mesh, traverse.Ray((0.25, 0.25, -1), (0, 0, 1), t_max=0.5)) is None


def test_degenerate_directions_terminate():
    """A zero direction with an unbounded segment never ends in the reference; here it is cut
    (and misses). NaN directions make every test return t = 0 in the reference (no
    comparison with NaN is true), so they terminate on the first candidate; the GPU matches
    the oracle on all of them, bounded or not."""
    mesh = gen_scene("uniform", 500, 2)
    spec = spec_for_mesh(mesh, dims=(7, 8, 9))
    grid, _ = builders.build_parallel(mesh, spec)
    o = np.array([[0.5, 0.5, 0.5], [0.5, 0.5, 0.5], [0.2, 0.3, 0.4]])
    d = np.array([[0.0, 0.0, 0.0], [np.nan, np.nan, np.nan], [0.0, np.nan, 0.0]])
    for t in (np.array([np.inf, np.inf, np.inf]), np.array([1.0, 1.0, 1.0])):
        ids, ts = traverse.dda_cast(grid, mesh, o, d, t)
        want = oracle.dda_cast(grid.G, grid.O, mesh.vertices, mesh.triangles, spec, o, d, t)
        assert np.array_equal(ids, want[0]) and bits_equal(ts, want[1])
        assert ids[0] == -1 and np.isinf(ts[0])


def test_empty_inputs():
    spec = GridSpec(Aabb([0, 0, 0], [1, 1, 1]), (2, 2, 2))
    empty = TriangleMesh(np.zeros((0, 3)), np.zeros((0, 3), np.int32))
    grid, _ = builders.build_parallel(empty, spec)
    ids, ts = traverse.dda_cast(grid, empty, [[0.5, 0.5, -1]], [[0, 0, 1]], [np.inf])
    assert ids.tolist() == [-1] and np.isinf(ts[0])
    ids, ts = traverse.dda_cast(grid, empty, np.zeros((0, 3)), np.zeros((0, 3)), np.zeros(0))
    assert len(ids) == 0 and len(ts) == 0


def test_errors_are_loud():
    mesh = gen_scene("uniform", 200, 1)
    spec = spec_for_mesh(mesh, dims=(4, 4, 4))
    grid, _ = builders.build_parallel(mesh, spec)
    small = TriangleMesh(mesh.vertices, mesh.triangles[:10])
    with pytest.raises(InvariantError):   # O refers to triangles the mesh does not have
        traverse.dda_cast(grid, small, [[0.5, 0.5, -1]] * 64, [[0, 0, 1]] * 64, [np.inf] * 64)
    b = _native.Builder(0)
    T = np.array([[0, 1, 10**6]], np.int32)
    with pytest.raises(InvariantError):
        b.dda_prepare(mesh.vertices, len(mesh.vertices), T, 1, flags=_native.PG_HOST_INPUT)
    with pytest.raises(InvariantError):
        traverse.dda_cast(grid, mesh, np.zeros((2, 3)), np.zeros((3, 3)), np.zeros(2))
