"""Sharded (multi-GPU) build orchestration: world_size 2 and 3 over gloo on CPU with the
numpy per-rank ops, and slab planning properties. The result must equal the single-device
build (the C oracle / the reference's golden hashes) bit for bit."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2403_10647_b200 import distributed as D
from paper_2403_10647_b200 import gen_scene, spec_for_mesh


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, kind, n, seed, dims, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from np_ops import NumpyOps
        mesh = gen_scene(kind, n, seed)
        spec = spec_for_mesh(mesh, dims=dims)
        lo, hi = D.shard_range(mesh.ntriangles, rank, world)
        res = D.build_sharded(NumpyOps(), D.TorchComm(), mesh.vertices, mesh.triangles[lo:hi], lo, spec)
        if rank == 0:
            np.savez(out_path, G=res[0], O=res[1])
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("kind,n,seed,dims", [("walls", 3000, 5, (40, 30, 20)),
                                              ("skewed", 2500, 9, (33, 17, 21))])
def test_sharded_build_gloo(tmp_path, world, kind, n, seed, dims):
    out = str(tmp_path / "res.npz")
    mp.spawn(_worker, args=(world, _free_port(), kind, n, seed, dims, out), nprocs=world, join=True)
    res = np.load(out)
    mesh = gen_scene(kind, n, seed)
    G, O = oracle.build_parallel(mesh.vertices, mesh.triangles, spec_for_mesh(mesh, dims=dims))
    assert np.array_equal(res["G"], G) and np.array_equal(res["O"], O)


def _gather_worker(rank, world, port, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from np_ops import NumpyOps
        mesh = gen_scene("walls", 3000, 5)
        spec = spec_for_mesh(mesh, dims=(40, 30, 20))
        lo, hi = D.shard_range(mesh.ntriangles, rank, world)
        res = D.build_sharded(NumpyOps(), D.TorchComm(), mesh.vertices, mesh.triangles[lo:hi], lo, spec,
                              gather="device")
        if rank == 0:
            np.savez(out_path, G=res[0].numpy().view(np.uint32), O=res[1].numpy().view(np.uint32))
        else:
            assert res is None
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gather_slabs_to_rank0_gloo(tmp_path, world):
    """gather="device": the slabs go to rank 0 point-to-point (tensors; NCCL on GPUs) and G is
    rebased there -- the gathered-output mode of SURVEY.md §8e."""
    out = str(tmp_path / "g.npz")
    mp.spawn(_gather_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    res = np.load(out)
    mesh = gen_scene("walls", 3000, 5)
    G, O = oracle.build_parallel(mesh.vertices, mesh.triangles, spec_for_mesh(mesh, dims=(40, 30, 20)))
    assert np.array_equal(res["G"], G) and np.array_equal(res["O"], O)


@pytest.mark.parametrize("world", [1, 2, 4, 8, 16])
def test_emulated_ranks_match_oracle(world):
    from np_ops import NumpyOps
    mesh = gen_scene("uniform", 4000, 3)
    spec = spec_for_mesh(mesh, dims=(37, 29, 31))
    G, O = D.run_emulated(NumpyOps, mesh.vertices, mesh.triangles, spec, world)
    Gr, Or = oracle.build_parallel(mesh.vertices, mesh.triangles, spec)
    assert np.array_equal(G, Gr) and np.array_equal(O, Or)


def test_slab_plan_properties():
    rng = np.random.default_rng(0)
    hist = rng.integers(0, 100, 4096)
    hist[100:400] = 0
    for world in (1, 2, 3, 8, 16):
        plan = D.plan_slabs(hist, 40_001_688, world)
        assert plan.cuts[0] == 0 and plan.cuts[-1] == len(hist)
        assert np.all(np.diff(plan.cuts) >= 0)
        assert plan.cell_lo[0] == 0 and plan.cell_hi[-1] == 40_001_688
        assert np.array_equal(plan.cell_lo[1:], plan.cell_hi[:-1])
        assert plan.pair_base[-1] == hist.sum()
        sizes = np.diff(plan.pair_base)
        assert sizes.max() <= hist.sum() / world + hist.max()      # balanced up to a bucket
        assert np.all(plan.table[plan.cuts[1]:plan.cuts[2]] == 1) if world > 1 else True


def test_empty_and_tiny_scenes_emulated():
    from np_ops import NumpyOps
    mesh = gen_scene("uniform", 3, 1)
    spec = spec_for_mesh(mesh, dims=(2, 1, 1))
    G, O = D.run_emulated(NumpyOps, mesh.vertices, mesh.triangles, spec, 4)
    Gr, Or = oracle.build_parallel(mesh.vertices, mesh.triangles, spec)
    assert np.array_equal(G, Gr) and np.array_equal(O, Or)


def test_slab_matrix_and_count_slots():
    """Host helpers of the device-side exchange: the per-rank slab matrix from coarse
    histograms equals summing each rank's buckets by slab, and the control-buffer count slots
    decode to the matrix and the 64-bit NOs."""
    rng = np.random.default_rng(3)
    for world in (1, 2, 5, 16):
        nb = 4096
        hists = rng.integers(0, 1000, size=(world, nb)).astype(np.int64)
        hists[:, rng.integers(0, nb, 50)] = 0
        plan = D.plan_slabs(hists.sum(axis=0), 1 << 26, world)
        m = D.slab_matrix(hists, plan.cuts)
        want = np.array([[h[plan.table == s].sum() for s in range(world)] for h in hists])
        assert np.array_equal(m, want) and np.array_equal(m.sum(axis=1), hists.sum(axis=1))
        slots = np.zeros((world, D.CTL_CNT), np.uint32)
        nos = rng.integers(0, 1 << 40, size=world)
        slots[:, :world] = m.astype(np.uint32)
        slots[:, 16] = nos & 0xFFFFFFFF
        slots[:, 17] = nos >> 32
        errs = rng.integers(0, 4, size=world)
        slots[:, 18] = errs
        mm, nn, ee = D._split_counts(slots.view(np.int32).reshape(-1), world)
        assert np.array_equal(mm, m) and np.array_equal(nn, nos) and np.array_equal(ee, errs)


@pytest.mark.parametrize("n", [1, 3, 7])
def test_emulated_more_ranks_than_triangles(n):
    """Ranks with empty shards (N < P) still take part in the plan and the exchange."""
    from np_ops import NumpyOps
    mesh = gen_scene("uniform", n, 11)
    spec = spec_for_mesh(mesh, dims=(9, 5, 7))
    G, O = D.run_emulated(NumpyOps, mesh.vertices, mesh.triangles, spec, 8)
    Gr, Or = oracle.build_parallel(mesh.vertices, mesh.triangles, spec)
    assert np.array_equal(G, Gr) and np.array_equal(O, Or)


def _err_worker(rank, world, port, case, out_path):
    """One sharded build whose mesh is bad in ONE shard (or only globally); every rank must
    raise the reference's class, at the same point, without hanging."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    got = "none"
    try:
        from np_ops import NumpyOps
        from paper_2403_10647_b200.errors import InvariantError, SizeError
        from paper_2403_10647_b200.gridcore import Aabb, GridSpec
        V, T, spec = _err_case(case, world)
        lo, hi = D.shard_range(len(T), rank, world)
        try:
            D.build_sharded(NumpyOps(), D.TorchComm(), V, T[lo:hi], lo, spec)
        except SizeError:
            got = "SizeError"
        except InvariantError:
            got = "InvariantError"
        # the process group is still usable afterwards (no rank was left in a collective)
        t = torch.ones(1)
        dist.all_reduce(t)
        assert int(t.item()) == world
        with open(f"{out_path}.{rank}", "w") as fh:
            fh.write(got)
    finally:
        dist.destroy_process_group()


def _err_case(case, world):
    from paper_2403_10647_b200.gridcore import Aabb, GridSpec
    good = gen_scene("uniform", 600, 3)
    V = good.vertices.copy()
    T = good.triangles.copy()
    unit = GridSpec(Aabb([0, 0, 0], [1, 1, 1]), (16, 16, 16))
    if case == "index":                    # one bad index in the LAST shard only
        T[-1, 2] = len(V) + 5
        return V, T, unit
    if case == "negative":                 # one-axis inverted box in the first shard
        V[T[0, 0]] = [0.6, 0.1, 0.1]
        V[T[0, 1]] = [np.inf, 0.2, 0.1]
        V[T[0, 2]] = [0.7, 0.1, 0.2]
        return V, T, unit
    if case == "zero":                     # zero-count box alone in its shard, not in the mesh
        zt = np.array([[0.1, 0.1, 0.5], [np.inf, 0.2, 0.5], [0.12, 0.2, 0.5]])   # x: lo 1, hi 0
        far = np.array([[5.0, 5, 5], [6, 5, 5], [5, 6, 5]])
        tris = [zt] + [far] * (2 * world - 1) + [good.vertices[good.triangles[0]]]
        Vz = np.concatenate(tris)
        return Vz, np.arange(len(Vz), dtype=np.int32).reshape(-1, 3), unit
    if case == "global_no":                # every shard < 2^32 pairs, the mesh > 2^32-1
        Vf = np.array([[-1, -1, -1], [3, -1, 2], [-1, 3, 2]], np.float64)
        Tf = np.zeros((17, 3), np.int32)
        Tf[:] = [0, 1, 2]
        return Vf, Tf, GridSpec(Aabb([0, 0, 0], [1, 1, 1]), (1024, 512, 512))
    raise ValueError(case)


@pytest.mark.timeout(300)
@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("case,want", [("index", "InvariantError"), ("negative", "InvariantError"),
                                       ("zero", "InvariantError"), ("global_no", "SizeError")])
def test_sharded_errors_agree_gloo(tmp_path, world, case, want):
    """The reference's verdict for the whole mesh on every rank: a bad shard on one rank, a
    zero-count box that is alone in its shard but not in the mesh, and a pair count that
    overflows 2^32-1 only in total (builders.py:99-100, primitives.py:22-25, 66-72)."""
    out = str(tmp_path / "verdict")
    mp.spawn(_err_worker, args=(world, _free_port(), case, out), nprocs=world, join=True)
    got = [open(f"{out}.{r}").read() for r in range(world)]
    assert got == [want] * world, got
    V, T, spec = _err_case(case, world)
    if case != "index":                    # the single-device oracle agrees
        exc = oracle.OracleSizeError if want == "SizeError" else oracle.OracleInvariantError
        with pytest.raises(exc):
            oracle.build_parallel(V, T, spec)


def test_count_verdict_order():
    from paper_2403_10647_b200.errors import InvariantError, SizeError
    ok = D.count_verdict([100, 0, 0, 0, 0, 0], 1000)
    assert ok == 100
    with pytest.raises(InvariantError):
        D.count_verdict([1 << 33, 0, 1, 0, 0, 0], 1000)      # negative count before SizeError
    with pytest.raises(SizeError):
        D.count_verdict([1 << 33, 0, 0, 1, 0, 0], 1000)      # NO > 2^32-1 before the zero count
    with pytest.raises(InvariantError):
        D.count_verdict([5, 0, 0, 1, 0, 0], 1000)            # zero count next to a kept box
    assert D.count_verdict([0, 0, 0, 1, 0, 0], 1000) == 0    # a lone zero-count box: empty grid
    with pytest.raises(SizeError):
        D.count_verdict([(1 << 30) + 1, 0, 0, 0, 0, 0], 1000)
    with pytest.raises(InvariantError):
        D.count_verdict([9, 0, 0, 0, 1, 1], 1 << 31)         # bad cells before the ncells cap
    with pytest.raises(SizeError):
        D.count_verdict([9, 0, 0, 0, 0, 0], 1 << 31)
