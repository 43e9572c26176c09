"""Sharded-build building blocks on the GPU (pg_pairs / pg_partition / pg_sort_cells) and
the whole sharded orchestration with every rank's phases emulated in sequence on one
device (no rank waits on another). Bit-exact against the oracle / golden hashes."""

import numpy as np
import pytest
import torch

import oracle
from paper_2403_10647_b200 import distributed as D
from paper_2403_10647_b200 import gen_scene, spec_for_mesh
from util import scene_from_recipe, sha

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_emulated_sharded_build(world):
    mesh = gen_scene("walls", 30000, 4)
    spec = spec_for_mesh(mesh, dims=(61, 47, 53))
    G, O = D.run_emulated(D.CudaOps, mesh.vertices, mesh.triangles, spec, world)
    Gr, Or = oracle.build_parallel(mesh.vertices, mesh.triangles, spec)
    assert np.array_equal(G, Gr) and np.array_equal(O, Or)


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8, 16])
def test_emulated_fused_exchange(world):
    """Fused partition + send (pg_partition_send into per-rank receive buffers) == oracle."""
    mesh = gen_scene("walls", 30000, 4)
    spec = spec_for_mesh(mesh, dims=(61, 47, 53))
    G, O = D.run_emulated(D.CudaOps, mesh.vertices, mesh.triangles, spec, world, exchange="p2p")
    Gr, Or = oracle.build_parallel(mesh.vertices, mesh.triangles, spec)
    assert np.array_equal(G, Gr) and np.array_equal(O, Or)


def test_emulated_fused_exchange_cfg2_hash(hashes):
    h = hashes["cfg2"]
    mesh, spec = scene_from_recipe(h["recipe"])
    G, O = D.run_emulated(D.CudaOps, mesh.vertices, mesh.triangles, spec, 8, exchange="p2p")
    assert len(O) == h["no"] and sha(G) == h["G_sha256"] and sha(O) == h["O_sha256"]


def test_partition_send_matches_partition():
    """pg_partition_send into one buffer per slab == pg_partition's slab ranges."""
    ops = D.CudaOps()
    rng = np.random.default_rng(9)
    n, ncells, ns = 250_003, 1 << 21, 7
    keys = rng.integers(0, ncells, n).astype(np.uint32)
    vals = np.arange(n, dtype=np.uint32)
    shift = D.coarse_shift(ncells)
    hist = np.bincount(keys >> shift, minlength=((ncells - 1) >> shift) + 1)
    plan = D.plan_slabs(hist, ncells, ns)
    kt = torch.from_numpy(keys.view(np.int32)).cuda()
    vt = torch.from_numpy(vals.view(np.int32)).cuda()
    base = plan.cell_lo.astype(np.uint32)
    ko, vo, counts = ops.partition(kt, vt, plan.table, plan.shift, ns, base)
    want_k, want_v = ops.to_numpy(ko).copy(), ops.to_numpy(vo).copy()
    c = ops.partition_counts(kt, plan.table, plan.shift, ns)
    cnt = ops.to_numpy(c)[:ns].astype(np.int64)
    pad = 1000                              # each slab's pairs land after a 1000-pair offset
    dst = [torch.full((2 * (int(x) + pad),), -1, dtype=torch.int32, device="cuda") for x in cnt]
    ops.partition_send(kt, vt, plan.table, plan.shift, ns, base, [d.data_ptr() for d in dst],
                       [d.data_ptr() + 4 * (int(x) + pad) for d, x in zip(dst, cnt)], [pad] * ns)
    torch.cuda.synchronize()
    pos = np.concatenate([[0], np.cumsum(cnt)])
    for s in range(ns):
        x = int(cnt[s])
        got = dst[s].cpu().numpy().view(np.uint32)
        assert np.array_equal(got[pad:pad + x], want_k[pos[s]:pos[s + 1]])
        assert np.array_equal(got[x + 2 * pad:2 * (x + pad)], want_v[pos[s]:pos[s + 1]])
        assert (got[:pad] == 0xFFFFFFFF).all()


def test_emulated_sharded_cfg2_hash(hashes):
    h = hashes["cfg2"]
    mesh, spec = scene_from_recipe(h["recipe"])
    G, O = D.run_emulated(D.CudaOps, mesh.vertices, mesh.triangles, spec, 4)
    assert len(O) == h["no"] and sha(G) == h["G_sha256"] and sha(O) == h["O_sha256"]


def test_partition_kernel_is_stable_and_rebased():
    ops = D.CudaOps()
    rng = np.random.default_rng(7)
    n, ncells = 300_001, 1 << 20
    keys = rng.integers(0, ncells, n).astype(np.uint32)
    vals = np.arange(n, dtype=np.uint32)
    shift = D.coarse_shift(ncells)
    hist = np.bincount(keys >> shift, minlength=((ncells - 1) >> shift) + 1)
    plan = D.plan_slabs(hist, ncells, 5)
    kt = torch.from_numpy(keys.view(np.int32)).cuda()
    vt = torch.from_numpy(vals.view(np.int32)).cuda()
    ko, vo, counts = ops.partition(kt, vt, plan.table, plan.shift, 5, plan.cell_lo.astype(np.uint32))
    slab = plan.table[keys >> shift].astype(np.int64)
    order = np.argsort(slab, kind="stable")
    assert ops.to_numpy(counts)[:5].tolist() == np.bincount(slab, minlength=5).tolist()
    assert np.array_equal(ops.to_numpy(vo), vals[order])
    assert np.array_equal(ops.to_numpy(ko), (keys[order] - plan.cell_lo[slab[order]]).astype(np.uint32))


@pytest.mark.parametrize("ncells", [1, 2, 1000, 1 << 17, 3_000_001])
def test_sort_cells_matches_oracle(ncells):
    ops = D.CudaOps()
    rng = np.random.default_rng(ncells)
    n = 200_000
    keys = rng.integers(0, ncells, n).astype(np.uint32)
    vals = rng.integers(0, 1 << 30, n).astype(np.uint32)
    G, O = ops.sort_cells(torch.from_numpy(keys.view(np.int32)).cuda(),
                          torch.from_numpy(vals.view(np.int32)).cuda(), n, ncells)
    ks, vs = oracle.radix_sort_pairs(keys, vals, int(ncells - 1).bit_length())
    Gr = np.zeros(ncells + 1, np.uint32)
    Gr[1:] = np.cumsum(np.bincount(ks.astype(np.int64), minlength=ncells))
    assert np.array_equal(ops.to_numpy(O), vs) and np.array_equal(ops.to_numpy(G), Gr)


def test_single_rank_nccl_path(tmp_path):
    import os
    import torch.distributed as dist
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29531")
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        mesh = gen_scene("skewed", 20000, 2)
        spec = spec_for_mesh(mesh, dims=(50, 40, 30))
        comm = D.TorchComm(device=torch.device("cuda", 0))
        G, O = D.build_sharded(D.CudaOps(), comm, mesh.vertices, mesh.triangles, 0, spec)
        Gr, Or = oracle.build_parallel(mesh.vertices, mesh.triangles, spec)
        assert np.array_equal(G, Gr) and np.array_equal(O, Or)
        # the fused exchange through symmetric memory (peer pointers; one rank here)
        ex = D.PeerExchange(comm, torch.device("cuda", 0))
        for _ in range(2):
            G, O = D.build_sharded(D.CudaOps(), comm, mesh.vertices, mesh.triangles, 0, spec, exchange=ex)
            assert np.array_equal(G, Gr) and np.array_equal(O, Or)
    finally:
        dist.destroy_process_group()
