"""Device-side ingestion: mesh bounds reduced on the GPU give the
reference's spec_for_mesh bit for bit, and build_from_mesh reproduces the golden grids."""

import numpy as np
import pytest

from paper_2403_10647_b200 import builders, gen_scene, spec_for_mesh
from paper_2403_10647_b200.errors import InvariantError
from paper_2403_10647_b200.gridcore import TriangleMesh, mesh_bounds
from util import KAT_NAMES, kat_case, scene_from_recipe, sha

pytestmark = pytest.mark.gpu


def same_spec(a, b):
    return (tuple(a.dims) == tuple(b.dims) and np.array_equal(a.bounds.lo, b.bounds.lo)
            and np.array_equal(a.bounds.hi, b.bounds.hi) and np.array_equal(a.cell_size, b.cell_size))


@pytest.mark.parametrize("name", [k for k in KAT_NAMES if k != "nonfinite"])
def test_kat_meshes(kat, name):
    mesh, _ = kat_case(kat, name)
    for dims, dens in ((None, 5.0), (None, 0.7), ((3, 4, 5), 5.0)):
        want = spec_for_mesh(mesh, dims=dims, density=dens)
        got = builders.device_spec_for_mesh(mesh.vertices, len(mesh.vertices), len(mesh.triangles), dims, dens)
        assert same_spec(got, want)


def test_bounds_exact_and_nan_rejected():
    rng = np.random.default_rng(3)
    for nv in (1, 2, 3, 191, 192, 193, 100_003, 2_000_000):
        V = (rng.random((nv, 3)) - 0.5) * 10.0 ** rng.integers(-3, 8, (nv, 3))
        lo, hi = builders._native.thread_builder().mesh_bounds(V, nv, flags=builders._native.PG_HOST_INPUT)
        ref = mesh_bounds(TriangleMesh(V, np.zeros((0, 3), np.int32)))
        assert np.array_equal(lo, ref.lo) and np.array_equal(hi, ref.hi)
    V[12345, 1] = np.nan
    with pytest.raises(InvariantError):
        builders.device_spec_for_mesh(V, len(V), 1)
    V[12345, 1] = np.inf
    lo, hi = builders._native.thread_builder().mesh_bounds(V, len(V), flags=builders._native.PG_HOST_INPUT)
    assert hi[1] == np.inf
    with pytest.raises(InvariantError):
        builders.device_spec_for_mesh(np.zeros((0, 3)), 0, 1)


@pytest.mark.parametrize("key", ["cfg1", "cfg2", "skewed100k", "walls100k", "sweep1m_d16"])
def test_build_from_mesh_matches_golden(hashes, key):
    h = hashes[key]
    mesh, spec = scene_from_recipe(h["recipe"])
    grid, rep = builders.build_from_mesh(mesh, density=h["recipe"]["density"])
    assert same_spec(grid.spec, spec)
    assert rep.no == h["no"] and sha(grid.G) == h["G_sha256"] and sha(grid.O) == h["O_sha256"]
