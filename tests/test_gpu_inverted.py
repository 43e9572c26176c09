"""Inverted cell boxes on the GPU against the reference's own verdicts (tests/golden/
make_golden_inverted.py): an infinite or huge upper corner clips below the lower one. The
reference raises for negative counts, for zero counts among >= 2 kept triangles and for
cells outside [0, ncells); a box inverted on two axes (positive count) gets the cells of
_make_cell_ids with floor division (builders.py:104-117). Every path must agree: the drop-in
build_parallel (+ record=), the sync-free graph build, the deferred BuildPipeline, the
sharded build (emulated ranks) and the baseline builders (which raise: undefined there)."""

import numpy as np
import pytest
import torch

from paper_2403_10647_b200 import _native, builders
from paper_2403_10647_b200 import distributed as D
from paper_2403_10647_b200.errors import InvariantError, SizeError
from paper_2403_10647_b200.gridcore import TriangleMesh
from util import inverted_cases

pytestmark = pytest.mark.gpu

CASES = inverted_cases()
ERR = {1: SizeError, 2: InvariantError}


def _grid_cases():
    return [c for c in CASES if c[4] == 0 and len(c[6])]


def test_golden_has_two_axis_grids():
    assert len(_grid_cases()) >= 40


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_build_parallel_verdicts(case):
    name, V, T, spec, verdict, G, O = case
    mesh = TriangleMesh(V, T)
    if verdict:
        with pytest.raises(ERR[verdict]):
            builders.build_parallel(mesh, spec)
        return
    grid, rep = builders.build_parallel(mesh, spec)
    assert np.array_equal(grid.G, G) and np.array_equal(grid.O, O) and rep.no == len(O)
    rec = {}
    grid, rep = builders.build_parallel(mesh, spec, record=rec)
    assert np.array_equal(grid.G, G) and np.array_equal(grid.O, O)
    assert rec["no"] == len(O) and np.array_equal(rec["g"], G.astype(np.int64))
    assert np.array_equal(np.sort(rec["global_c"]), rec["sorted_c"])


def test_graph_build_rebuilds_inverted():
    """pg_build_async on a mesh with two-axis inverted boxes: pg_build_wait finishes it on the
    host-checked count, so the returned grid is still the reference's."""
    b = _native.Builder(0)
    for name, V, T, spec, verdict, G, O in _grid_cases()[:12]:
        Vd = torch.from_numpy(V.copy()).cuda()
        Td = torch.from_numpy(T.copy()).cuda()
        Gd = torch.full((spec.ncells + 1,), -1, dtype=torch.int32, device="cuda")
        Od = torch.full((len(O) + 8,), -1, dtype=torch.int32, device="cuda")
        b.build_async(Vd, len(V), Td, len(T), spec, Gd, Od, len(O) + 8)
        assert b.build_wait() == len(O), name
        assert np.array_equal(Gd.cpu().numpy().view(np.uint32), G), name
        assert np.array_equal(Od[:len(O)].cpu().numpy().view(np.uint32), O), name


def test_pipeline_deferred_inverted(hashes):
    from util import scene_from_recipe
    mesh0, spec0 = scene_from_recipe(hashes["cfg1"]["recipe"])
    pipe = builders.BuildPipeline(depth=2)
    pipe.submit(mesh0, spec0)
    pipe.result()                       # learns a capacity: later submits are deferred
    for name, V, T, spec, verdict, G, O in CASES[:60]:
        pipe.submit(TriangleMesh(V, T), spec)
        if verdict:
            with pytest.raises(ERR[verdict]):
                pipe.result()
        else:
            grid, rep = pipe.result()
            assert np.array_equal(grid.G, G) and np.array_equal(grid.O, O), name


@pytest.mark.parametrize("world", [1, 2, 3])
def test_sharded_inverted(world):
    """Sharded build (emulated ranks, NCCL-style copy exchange): the per-shard expansion gets
    the same rewrite, the coarse slab histogram stays consistent."""
    for name, V, T, spec, verdict, G, O in _grid_cases()[:20]:
        Gs, Os = D.run_emulated(D.CudaOps, V, T, spec, world)
        assert np.array_equal(Gs, G) and np.array_equal(Os, O), name


def test_baselines_raise_on_two_axis_inverted():
    name, V, T, spec, verdict, G, O = _grid_cases()[0]
    for fn in (builders.build_sorted, builders.build_compact):
        with pytest.raises(InvariantError):
            fn(TriangleMesh(V, T), spec)


def test_inverted_mixed_into_large_scene():
    """Two-axis inverted boxes inside a 200K-triangle scene (many tiles, 2 radix passes)."""
    import oracle
    from paper_2403_10647_b200 import gen_scene, spec_for_mesh
    mesh = gen_scene("uniform", 200_000, 3)
    spec = spec_for_mesh(mesh)
    V = mesh.vertices.copy()
    rng = np.random.default_rng(5)
    lo, hi = np.asarray(spec.bounds.lo), np.asarray(spec.bounds.hi)
    for t in rng.choice(len(mesh.triangles), 50, replace=False):
        a, bb, c = mesh.triangles[t]
        V[a] = lo + (hi - lo) * rng.uniform(0.05, 0.95, 3)
        V[c] = V[a] + 1e-9
        ax = rng.choice(3, 2, replace=False)                      # two inverted axes: the
        V[bb] = V[a]                                              # cells stay in the grid
        V[bb, ax] = np.inf
    want = oracle.build_parallel(V, mesh.triangles, spec)
    m2 = TriangleMesh(V, mesh.triangles)
    grid, rep = builders.build_parallel(m2, spec)
    assert np.array_equal(grid.G, want[0]) and np.array_equal(grid.O, want[1])
