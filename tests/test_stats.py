"""Grid statistics: host formulas on CPU (test_stats.py:10-34 rows) and the
GPU reductions against a numpy restatement of stats.py:43-64 over the oracle's cell boxes."""

import numpy as np
import pytest

import oracle
from paper_2403_10647_b200 import stats

FAIRY = (172_170, (141, 37, 141), 3.88, 5.35)
SAN_MIGUEL = (10_480_000, (565, 116, 648), 1.65, 228.03)


def test_estimate_pairs():
    assert stats.estimate_pairs(172_170, 3.88) == 668_020
    assert stats.estimate_pairs(12345, 1.0) == 12345
    assert stats.estimate_pairs(0, 99.0) == 0
    with pytest.raises(ValueError):
        stats.estimate_pairs(-1, 1.0)


@pytest.mark.parametrize("ntris,dims,avg,mb", [FAIRY, SAN_MIGUEL])
def test_memory_model_reproduces_published_mb(ntris, dims, avg, mb):
    ncells = dims[0] * dims[1] * dims[2]
    got = stats.grid_memory_bytes(ncells, stats.estimate_pairs(ntris, avg)) / stats.MB
    assert got == pytest.approx(mb, rel=0.005)
    assert stats.grid_memory_bytes(735_597, 668_020) == 5_614_472


def expected_stats(grid, mesh):
    """stats.py:43-64 restated with numpy over the oracle's boxes (checker only)."""
    lo, hi, keep = oracle.cell_boxes(mesh.vertices, mesh.triangles, grid.spec)
    widths = np.diff(grid.G.astype(np.int64))
    nonempty = int(np.count_nonzero(widths))
    cpi = (hi[keep].astype(np.int64) - lo[keep] + 1).prod(axis=1)
    n_in = int(keep.sum())
    nc = grid.spec.ncells
    return stats.GridStats(len(mesh.triangles), grid.spec.dims, nc, grid.no, 100.0 * (nc - nonempty) / nc,
                           grid.no / nonempty if nonempty else 0.0, int(cpi.max()) if n_in else 0,
                           grid.no / n_in if n_in else 0.0, stats.grid_memory_bytes(nc, grid.no))


@pytest.mark.gpu
@pytest.mark.parametrize("kind,n,dims", [("uniform", 300, (6, 6, 6)), ("skewed", 5000, (30, 20, 10)),
                                         ("walls", 3000, None), ("lognormal", 200_000, None)])
def test_compute_stats_gpu(kind, n, dims):
    from paper_2403_10647_b200 import builders, gen_scene, spec_for_mesh
    mesh = gen_scene(kind, n, 21)
    spec = spec_for_mesh(mesh, dims=dims)
    grid, rep = builders.build_parallel(mesh, spec)
    got = stats.compute_stats(grid, mesh)
    assert got == expected_stats(grid, mesh)
    assert got.no == rep.no and got.memory_bytes == 4 * (spec.ncells + 1) + 4 * rep.no


@pytest.mark.gpu
def test_compute_stats_gpu_empty_and_dropped(kat):
    from paper_2403_10647_b200 import builders
    from paper_2403_10647_b200.gridcore import Aabb, GridSpec, TriangleMesh
    from util import kat_case
    spec = GridSpec(Aabb([0, 0, 0], [1, 1, 1]), (3, 3, 3))
    empty = TriangleMesh(np.zeros((0, 3)), np.zeros((0, 3), np.int32))
    grid, _ = builders.build_parallel(empty, spec)
    st = stats.compute_stats(grid, empty)
    assert st.pct_empty == 100.0 and st.no == 0 and st.memory_bytes == 4 * 28
    assert st.avg_items_per_nonempty_cell == 0.0 and st.max_cells_per_item == 0
    for name in ("dropped", "sparse_kept", "nonfinite"):
        mesh, spec = kat_case(kat, name)
        grid, _ = builders.build_parallel(mesh, spec)
        assert stats.compute_stats(grid, mesh) == expected_stats(grid, mesh)
