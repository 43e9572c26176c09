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


def _fused_dispatch_built():
    from paper_2403_10647_b200 import _native
    return bool(_native.features() & _native.PG_FEATURE_FUSED_DISPATCH)


needs_fused = pytest.mark.skipif("not _fused_dispatch_built()",
                                 reason="libpgrid built without PGRID_FUSED_DISPATCH (measured slower, not shipped)")


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


@pytest.mark.parametrize("gen_order", [False, True])
@pytest.mark.parametrize("ncells", [1, 2, 1000, 1 << 17, 3_000_001])
def test_sort_cells_matches_oracle(ncells, gen_order):
    """Arbitrary values (stable by position) and generation-ordered ones (PG_GEN_ORDER: values
    ascend inside a cell, the MSD-first finish ranks them by value)."""
    ops = D.CudaOps()
    rng = np.random.default_rng(ncells)
    n = 200_000
    keys = rng.integers(0, ncells, n).astype(np.uint32)
    vals = rng.integers(0, 1 << 30, n).astype(np.uint32)
    if gen_order:   # object-major emission: ids ascend along the pairs, distinct inside a cell
        vals = np.sort(vals)
        keys = keys[np.lexsort((keys, vals))]
        _, first = np.unique(np.stack([keys, vals]), axis=1, return_index=True)
        keep = np.zeros(n, bool)
        keep[first] = True
        keys, vals = keys[keep], vals[keep]
        n = len(keys)
    G, O = ops.sort_cells(torch.from_numpy(keys.view(np.int32)).cuda(),
                          torch.from_numpy(vals.view(np.int32)).cuda(), n, ncells, gen_order=gen_order)
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
        Gd, Od = D.build_sharded(D.CudaOps(), comm, mesh.vertices, mesh.triangles, 0, spec, gather="device",
                                 exchange=ex)
        assert np.array_equal(Gd.cpu().numpy().view(np.uint32), Gr) and np.array_equal(Od.cpu().numpy().view(np.uint32), Or)
        ex.fused = _fused_dispatch_built()   # expansion + dispatch in one kernel (pg_pairs_send)
        ex.no_capacity = None
        for _ in range(2):
            G, O = D.build_sharded(D.CudaOps(), comm, mesh.vertices, mesh.triangles, 0, spec, exchange=ex)
            assert np.array_equal(G, Gr) and np.array_equal(O, Or)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [1, 2, 3, 8, 16])
def test_device_slab_plan_matches_plan_slabs(world):
    """pg_slab_plan (the device plan of the fused exchange) == distributed.plan_slabs, on
    skewed, sparse, empty and tiny histograms."""
    rng = np.random.default_rng(world)
    ops = D.CudaOps()
    for ncells, kind in [(40_001_688, "lognormal"), (40_001_688, "spike"), (5_000_211, "sparse"),
                         (4096, "zero"), (7, "uniform"), (1 << 30, "uniform")]:
        shift = D.coarse_shift(ncells)
        nb = ((ncells - 1) >> shift) + 1
        per_rank = []
        for _ in range(world):
            if kind == "lognormal":
                h = rng.lognormal(3, 2, nb).astype(np.int64)
            elif kind == "spike":
                h = np.zeros(nb, np.int64)
                h[rng.integers(0, nb, 3)] = rng.integers(1, 10**6, 3)
            elif kind == "sparse":
                h = np.where(rng.random(nb) < 0.01, rng.integers(0, 1000, nb), 0)
            elif kind == "zero":
                h = np.zeros(nb, np.int64)
            else:
                h = rng.integers(0, 50, nb)
            per_rank.append(np.minimum(h, 2**31 - 1).astype(np.uint32))
        hists = torch.from_numpy(np.concatenate(per_rank).view(np.int32)).cuda()
        table, base, plan = ops.slab_plan(hists, world, nb, shift, ncells, world)
        ref = D.plan_slabs(np.sum([h.astype(np.int64) for h in per_rank], axis=0), ncells, world)
        a = plan.cpu().numpy()
        P = world
        assert np.array_equal(a[:P + 1], ref.cuts), kind
        assert np.array_equal(a[P + 1:2 * P + 1], ref.cell_lo), kind
        assert np.array_equal(a[2 * P + 1:3 * P + 1], ref.cell_hi), kind
        assert np.array_equal(a[3 * P + 1:], ref.pair_base), kind
        assert np.array_equal(ops.to_numpy(table)[:nb], ref.table), kind
        assert np.array_equal(ops.to_numpy(base)[:P], ref.cell_lo.astype(np.uint32)), kind


def test_peer_put_fills_every_slot():
    from paper_2403_10647_b200 import _native
    world = 5
    bufs = [torch.full((world * 100,), -1, dtype=torch.int32, device="cuda") for _ in range(world)]
    ptrs = [b.data_ptr() for b in bufs]
    srcs = [torch.arange(r * 1000, r * 1000 + 77, dtype=torch.int32, device="cuda") for r in range(world)]
    for r in range(world):
        _native.peer_put(srcs[r], 77, ptrs, r * 100, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    for b in bufs:
        v = b.view(world, 100).cpu().numpy()
        for r in range(world):
            assert np.array_equal(v[r, :77], np.arange(r * 1000, r * 1000 + 77)) and (v[r, 77:] == -1).all()


@pytest.mark.parametrize("world", [1, 3, 8])
def test_emulated_fused_exchange_deferred_count(world):
    """PG_DEFER counts (no NO read back; pair buffers sized by a capacity) == oracle; a
    capacity below some rank's NO is detected by every rank (the exchanged NOs)."""
    mesh = gen_scene("walls", 30000, 4)
    spec = spec_for_mesh(mesh, dims=(61, 47, 53))
    Gr, Or = oracle.build_parallel(mesh.vertices, mesh.triangles, spec)
    G, O = D.run_emulated(D.CudaOps, mesh.vertices, mesh.triangles, spec, world, exchange="p2p",
                          capacity=len(Or))
    assert np.array_equal(G, Gr) and np.array_equal(O, Or)
    assert D.run_emulated(D.CudaOps, mesh.vertices, mesh.triangles, spec, world, exchange="p2p",
                          capacity=len(Or) // world // 2) is None


@needs_fused
@pytest.mark.parametrize("world", [1, 2, 3, 4, 8, 16])
def test_emulated_fused_dispatch(world):
    """pg_coarse_hist + device plan + pg_pairs_send (expansion, slab ranking with a decoupled
    look-back and peer stores in one kernel) == oracle, with and without a deferred count."""
    mesh = gen_scene("walls", 30000, 4)
    spec = spec_for_mesh(mesh, dims=(61, 47, 53))
    Gr, Or = oracle.build_parallel(mesh.vertices, mesh.triangles, spec)
    for cap in (None, len(Or)):
        G, O = D.run_emulated(D.CudaOps, mesh.vertices, mesh.triangles, spec, world, exchange="fused",
                              capacity=cap)
        assert np.array_equal(G, Gr) and np.array_equal(O, Or)
    assert D.run_emulated(D.CudaOps, mesh.vertices, mesh.triangles, spec, world, exchange="fused",
                          capacity=max(1, len(Or) // world // 2)) is None


@needs_fused
def test_emulated_fused_dispatch_cfg2_hash(hashes):
    h = hashes["cfg2"]
    mesh, spec = scene_from_recipe(h["recipe"])
    G, O = D.run_emulated(D.CudaOps, mesh.vertices, mesh.triangles, spec, 8, exchange="fused")
    assert len(O) == h["no"] and sha(G) == h["G_sha256"] and sha(O) == h["O_sha256"]


@needs_fused
@pytest.mark.parametrize("scene,n,dims", [("walls", 20000, None), ("skewed", 20000, (50, 40, 30)),
                                          ("lognormal", 50000, None), ("uniform", 30000, (4096, 2, 3)),
                                          ("walls", 5000, (1, 1, 7)), ("uniform", 30000, (97, 1, 1))])
def test_coarse_hist_from_boxes_matches_pairs(scene, n, dims):
    """The coarse histogram from the cell boxes (before any pair exists) == pg_pairs' one,
    including rows that span many buckets (flat grids)."""
    mesh = gen_scene(scene, n, 3)
    spec = spec_for_mesh(mesh, dims=dims) if dims else spec_for_mesh(mesh)
    ops = D.CudaOps()
    ncells = int(np.prod(spec.dims))
    shift = D.coarse_shift(ncells)
    nb = ((ncells - 1) >> shift) + 1
    no = ops.count(mesh.vertices, mesh.triangles, spec)
    h1 = ops.to_numpy(ops.coarse_hist(shift, nb)).copy()
    _, _, h2 = ops.pairs(no, 0, shift, nb)
    assert np.array_equal(h1, ops.to_numpy(h2)) and int(h1.sum()) == no


@pytest.mark.parametrize("mode", ["copy", "p2p", pytest.param("fused", marks=needs_fused)])
def test_emulated_more_ranks_than_triangles(mode):
    """Empty shards (N < P) on the device paths: the device NO of an empty count is 0."""
    for n in (1, 3, 7):
        mesh = gen_scene("uniform", n, 11)
        spec = spec_for_mesh(mesh, dims=(9, 5, 7))
        G, O = D.run_emulated(D.CudaOps, mesh.vertices, mesh.triangles, spec, 8, exchange=mode)
        Gr, Or = oracle.build_parallel(mesh.vertices, mesh.triangles, spec)
        assert np.array_equal(G, Gr) and np.array_equal(O, Or)
