"""GPU comparison builders: build_sorted / build_compact on the device
must give the reference's G/O bit for bit (builders.py:172-231) and the reference's reports
(test_builders.py:120-136 load-imbalance instrumentation)."""

import numpy as np
import pytest

import oracle
from paper_2403_10647_b200 import builders, gen_scene, spec_for_mesh
from paper_2403_10647_b200.gridcore import Aabb, GridSpec, TriangleMesh
from util import KAT_NAMES, kat_case, scene_from_recipe, sha

pytestmark = pytest.mark.gpu

BASELINES = [builders.build_sorted, builders.build_compact]


@pytest.mark.parametrize("build", BASELINES, ids=lambda f: f.__name__)
@pytest.mark.parametrize("name", KAT_NAMES)
def test_kat(kat, build, name):
    mesh, spec = kat_case(kat, name)
    grid, rep = build(mesh, spec)
    assert np.array_equal(grid.G, kat[f"{name}/G"])
    assert np.array_equal(grid.O, kat[f"{name}/O"])
    assert rep.no == int(kat[f"{name}/no"])


def test_sorted_record_matches_reference_stages(kat):
    mesh, spec = kat_case(kat, "walkthrough")
    rec = {}
    grid, rep = builders.build_sorted(mesh, spec, record=rec)
    for st in ("v", "offsets", "obj_ids", "global_c", "sorted_c", "sorted_o", "rle_uniques", "rle_counts", "g"):
        assert np.array_equal(rec[st], kat[f"walkthrough/{st}"]), st
    assert "rel_c" not in rec and rec["no"] == rep.no == 4


def test_reports_expose_load_imbalance():
    """test_builders.py:120-136: one big triangle among small ones."""
    mesh = gen_scene("skewed", 2000, 3)
    spec = spec_for_mesh(mesh, dims=(16, 16, 16))
    lo, hi, keep = oracle.cell_boxes(mesh.vertices, mesh.triangles, spec)
    counts = np.prod(hi[keep].astype(np.int64) - lo[keep] + 1, axis=1)
    _, rs = builders.build_sorted(mesh, spec)
    _, rc = builders.build_compact(mesh, spec)
    _, rp = builders.build_parallel(mesh, spec)
    assert rs.max_task_work == rc.max_task_work == int(counts.max())
    assert rs.total_work == rs.no == rp.no and rc.total_work == 2 * rc.no
    assert rs.algo == "sorted" and rc.algo == "compact"


@pytest.mark.parametrize("build", BASELINES, ids=lambda f: f.__name__)
def test_empty_and_all_dropped(build):
    spec = GridSpec(Aabb([0, 0, 0], [1, 1, 1]), (2, 2, 2))
    grid, rep = build(TriangleMesh(np.zeros((0, 3)), np.zeros((0, 3), np.int32)), spec)
    assert grid.no == 0 and rep.max_task_work == 0 and grid.G.tolist() == [0] * 9
    far = TriangleMesh(np.array([[5.0, 5, 5], [6, 5, 5], [5, 6, 5]]), np.array([[0, 1, 2]], np.int32))
    grid, rep = build(far, spec)
    assert grid.no == 0 and grid.G.tolist() == [0] * 9


@pytest.mark.parametrize("build", BASELINES, ids=lambda f: f.__name__)
@pytest.mark.parametrize("key", ["cfg1", "skewed100k", "walls100k", "cfg2", "sweep1m_d4", "sweep1m_d64"])
def test_config_hashes(hashes, build, key):
    h = hashes[key]
    mesh, spec = scene_from_recipe(h["recipe"])
    grid, rep = build(mesh, spec)
    assert rep.no == h["no"]
    assert sha(grid.G) == h["G_sha256"] and sha(grid.O) == h["O_sha256"]


@pytest.mark.parametrize("build", BASELINES, ids=lambda f: f.__name__)
def test_crowded_cells_vs_oracle(build):
    """Cells holding >32 and >4096 objects take the compact builder's block and global
    segment-sort paths; a few huge triangles make the sorted builder's walk imbalanced."""
    rng = np.random.default_rng(11)
    n = 9000
    c = rng.random((n, 1, 3)) * 0.02 + 0.49                 # everything near one corner of 8 cells
    tris = c + (rng.random((n, 3, 3)) - 0.5) * 0.004
    big = np.array([[[0, 0, 0], [1, 1, 0], [1, 0, 1]], [[0, 1, 1], [1, 0, 0], [0, 0, 1]]], float)
    tris = np.concatenate([tris, big, rng.random((3000, 3, 3))], axis=0)
    mesh = TriangleMesh(tris.reshape(-1, 3), np.arange(3 * len(tris), dtype=np.int32).reshape(-1, 3))
    for dims in ((2, 2, 2), (17, 5, 33), (64, 64, 64)):
        spec = spec_for_mesh(mesh, dims=dims)
        G, O = oracle.build_parallel(mesh.vertices, mesh.triangles, spec)
        grid, rep = build(mesh, spec)
        assert np.array_equal(grid.G, G) and np.array_equal(grid.O, O), dims


def test_fault_injection_applies_to_sorted_not_compact(kat, monkeypatch):
    mesh, spec = kat_case(kat, "walkthrough")
    monkeypatch.setattr(builders, "_fault_inject", True)
    gs, _ = builders.build_sorted(mesh, spec)
    gc, _ = builders.build_compact(mesh, spec)
    assert gs.O[0] == kat["walkthrough/O"][0] ^ 1
    assert np.array_equal(gc.O, kat["walkthrough/O"])
