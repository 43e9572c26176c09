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
        mm, nn = D._split_counts(slots.view(np.int32).reshape(-1), world)
        assert np.array_equal(mm, m) and np.array_equal(nn, nos)


@pytest.mark.parametrize("n", [1, 3, 7])
def test_emulated_more_ranks_than_triangles(n):
    """Ranks with empty shards (N < P) still take part in the plan and the exchange."""
    from np_ops import NumpyOps
    mesh = gen_scene("uniform", n, 11)
    spec = spec_for_mesh(mesh, dims=(9, 5, 7))
    G, O = D.run_emulated(NumpyOps, mesh.vertices, mesh.triangles, spec, 8)
    Gr, Or = oracle.build_parallel(mesh.vertices, mesh.triangles, spec)
    assert np.array_equal(G, Gr) and np.array_equal(O, Or)
