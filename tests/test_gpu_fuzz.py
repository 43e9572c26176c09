"""Randomised parity campaign on the GPU: many seeded scenes of every kind and size class,
random grid resolutions and bounds (dropped / clipped triangles, degenerate axes), injected
NaN / inf / huge coordinates and indexed meshes -- the CUDA build against the C oracle, bit
for bit, through build_parallel, the comparison builders and the sync-free graph path."""

import os

import numpy as np
import pytest
import torch

import oracle
from paper_2403_10647_b200 import _native, builders, gen_scene
from paper_2403_10647_b200.gridcore import Aabb, GridSpec, TriangleMesh

pytestmark = pytest.mark.gpu
FUZZ_BLOCKS = int(os.environ.get("PGRID_FUZZ_BLOCKS", "8"))   # 25 random scenes per block


def random_case(rng):
    kind = rng.choice(["uniform", "skewed", "walls", "lognormal", "arch", "indexed"])
    n = int(rng.choice([1, 2, 7, 100, 1000, 4095, 4096, 4097, 20000, 150000]))
    if kind == "indexed":
        nv = max(3, n // 2)
        V = rng.random((nv, 3)) * rng.choice([1.0, 1e-3, 1e4])
        T = rng.integers(0, nv, (n, 3)).astype(np.int32)
    else:
        m = gen_scene(kind, n, int(rng.integers(1, 1 << 30)), float(rng.choice([1.0, 4.0, 20.0])))
        V, T = m.vertices.copy(), m.triangles.copy()
    if rng.random() < 0.3:                       # poison a few coordinates
        idx = rng.integers(0, len(V), max(1, len(V) // 500))
        V[idx, rng.integers(0, 3, len(idx))] = rng.choice([np.nan, np.inf, -np.inf, 1e300, -1e300], len(idx))
    lo, hi = np.nanmin(np.where(np.isfinite(V), V, np.nan), 0), np.nanmax(np.where(np.isfinite(V), V, np.nan), 0)
    lo, hi = np.nan_to_num(lo), np.nan_to_num(hi, nan=1.0)
    if rng.random() < 0.2 and kind != "indexed":  # boxes inverted on two axes (the reference builds them)
        for t in rng.choice(len(T), max(1, len(T) // 1000), replace=False):
            a, b, c = T[t]
            V[b] = V[a]
            V[c] = V[a] + 1e-9
            V[b, rng.choice(3, 2, replace=False)] = rng.choice([np.inf, 1e300])
    span = np.maximum(hi - lo, 1e-6)
    if rng.random() < 0.4:                       # a sub-box: many triangles dropped or clipped
        a = lo + rng.random(3) * 0.5 * span
        b = a + (0.1 + rng.random(3) * 0.9) * span
    else:
        a, b = lo - 0.01 * span, hi + 0.01 * span
    dims = tuple(int(x) for x in rng.choice([1, 2, 3, 17, 64, 129, 300], 3))
    if rng.random() < 0.2:
        dims = (int(rng.integers(1, 5000)), 1, int(rng.integers(1, 50)))
    return TriangleMesh(V, T), GridSpec(Aabb(a, b), dims)


def two_axis_inverted(mesh, spec):
    """Does a kept box invert on exactly two axes (the reference's sorted / compact builders
    leave its pairs uninitialised; the GPU versions raise)?"""
    lo, hi, keep = oracle.cell_boxes(mesh.vertices, mesh.triangles, spec)
    e = hi.astype(np.int64) - lo + 1
    return bool(np.any(keep & (e.prod(axis=1) > 0) & (e < 0).any(axis=1)))


def oracle_or_error(mesh, spec):
    try:
        return oracle.build_parallel(mesh.vertices, mesh.triangles, spec)
    except oracle.OracleSizeError:
        return None
    except oracle.OracleInvariantError:
        return "invariant"


@pytest.mark.parametrize("block", range(FUZZ_BLOCKS))
def test_fuzz_build_parallel(block):
    from paper_2403_10647_b200.errors import InvariantError
    rng = np.random.default_rng(1000 + block)
    for case in range(25):
        mesh, spec = random_case(rng)
        want = oracle_or_error(mesh, spec)
        if want is None:
            continue
        if isinstance(want, str):
            with pytest.raises(InvariantError):
                builders.build_parallel(mesh, spec)
            continue
        grid, rep = builders.build_parallel(mesh, spec)
        assert np.array_equal(grid.G, want[0]) and np.array_equal(grid.O, want[1]), (block, case, spec)
        if case % 5 == 0:
            for build in (builders.build_sorted, builders.build_compact):
                if two_axis_inverted(mesh, spec):
                    with pytest.raises(InvariantError):
                        build(mesh, spec)
                    continue
                g2, _ = build(mesh, spec)
                assert np.array_equal(g2.G, want[0]) and np.array_equal(g2.O, want[1]), (build.__name__, case)


def test_fuzz_graph_path():
    """The sync-free CUDA-graph build (pg_build_async) on a stream of random scenes."""
    rng = np.random.default_rng(77)
    b = _native.Builder(0)
    st = torch.cuda.current_stream().cuda_stream
    for case in range(30):
        mesh, spec = random_case(rng)
        want = oracle_or_error(mesh, spec)
        if want is None or isinstance(want, str) or len(mesh.triangles) == 0:
            continue
        Vd = torch.from_numpy(mesh.vertices.copy()).cuda()
        Td = torch.from_numpy(mesh.triangles.copy()).cuda()
        cap = len(want[1]) + int(rng.integers(0, 1000))
        Gd = torch.empty(spec.ncells + 1, dtype=torch.int32, device="cuda")
        Od = torch.empty(max(cap, 1), dtype=torch.int32, device="cuda")
        for _ in range(2):                       # eager, then graph replay
            b.build_async(Vd, len(mesh.vertices), Td, len(mesh.triangles), spec, Gd, Od, cap, st)
            assert b.build_wait() == len(want[1])
            assert np.array_equal(Gd.cpu().numpy().view(np.uint32), want[0])
            assert np.array_equal(Od[:len(want[1])].cpu().numpy().view(np.uint32), want[1])


@pytest.mark.parametrize("block", range(max(1, FUZZ_BLOCKS // 4)))
def test_fuzz_pipeline_deferred(block):
    """BuildPipeline (deferred counts after the first build, rebuilds on overflow) on a stream
    of random scenes: results in order and equal to the oracle's."""
    from paper_2403_10647_b200.errors import InvariantError
    rng = np.random.default_rng(5000 + block)
    cases = []
    while len(cases) < 20:
        mesh, spec = random_case(rng)
        want = oracle_or_error(mesh, spec)
        if want is not None:
            cases.append((mesh, spec, want))
    pipe = builders.BuildPipeline(depth=2)
    pending = []
    def collect():
        mesh, spec, want = pending.pop(0)
        if isinstance(want, str):
            with pytest.raises(InvariantError):
                pipe.result()
            return
        grid, rep = pipe.result()
        assert np.array_equal(grid.G, want[0]) and np.array_equal(grid.O, want[1]), (block, spec)
    for c in cases:
        if len(pending) == 2:
            collect()
        pipe.submit(c[0], c[1])
        pending.append(c)
    while pending:
        collect()


@pytest.mark.parametrize("block", range(max(1, FUZZ_BLOCKS // 4)))
def test_fuzz_sharded_emulated(block):
    """The sharded orchestration (device plan + peer-store partition, and the fused dispatch)
    on random scenes and rank counts, every virtual rank on this GPU."""
    from paper_2403_10647_b200 import distributed as D
    rng = np.random.default_rng(9000 + block)
    done = 0
    while done < 6:
        mesh, spec = random_case(rng)
        want = oracle_or_error(mesh, spec)
        if want is None or isinstance(want, str) or len(mesh.triangles) < 2:
            continue
        world = int(rng.integers(1, 9))
        from paper_2403_10647_b200 import _native
        fused = ("fused",) if _native.features() & _native.PG_FEATURE_FUSED_DISPATCH else ()
        for mode in ("copy", "p2p") + fused:
            G, O = D.run_emulated(D.CudaOps, mesh.vertices, mesh.triangles, spec, world, exchange=mode)
            assert np.array_equal(G, want[0]) and np.array_equal(O, want[1]), (block, mode, world, spec)
        done += 1
