"""GPU parity: the CUDA path (through the C ABI) against the reference's golden vectors and
the CPU oracle. Bit-exact: this path is integer/index work plus an IEEE f64 floor."""

import numpy as np
import pytest

import oracle
from paper_2403_10647_b200 import _native, builders, gen_scene, grids_equal, spec_for_mesh
from paper_2403_10647_b200.errors import InvariantError, SizeError
from paper_2403_10647_b200.gridcore import Aabb, GridSpec, TriangleMesh
from paper_2403_10647_b200.kernels import radix_sort_pairs
from util import KAT_NAMES, kat_case, scene_from_recipe, sha

pytestmark = pytest.mark.gpu

STAGES = ("v", "offsets", "obj_ids", "rel_c", "global_c", "sorted_c", "sorted_o",
          "rle_uniques", "rle_counts", "g")


@pytest.mark.parametrize("name", KAT_NAMES)
def test_kat_every_stage(kat, name):
    mesh, spec = kat_case(kat, name)
    rec = {}
    grid, rep = builders.build_parallel(mesh, spec, record=rec)
    assert np.array_equal(grid.G, kat[f"{name}/G"])
    assert np.array_equal(grid.O, kat[f"{name}/O"])
    assert rep.no == int(kat[f"{name}/no"]) == rec["no"]
    for st in STAGES:
        assert np.array_equal(rec[st], kat[f"{name}/{st}"]), st


def test_walkthrough_report(kat):
    mesh, spec = kat_case(kat, "walkthrough")
    grid, rep = builders.build_parallel(mesh, spec)
    assert grid.G.tolist() == [0, 1, 3, 3, 4] and grid.O.tolist() == [0, 0, 1, 1]
    assert rep.algo == "parallel" and rep.no == 4
    assert rep.max_task_work == 8 and rep.total_work == 32
    assert set(rep.phase_ms) == set(builders.PHASES) and rep.total_ms > 0


def test_empty_mesh(kat):
    spec = GridSpec(Aabb([0, 0, 0], [1, 1, 1]), (2, 2, 2))
    grid, rep = builders.build_parallel(TriangleMesh(np.zeros((0, 3)), np.zeros((0, 3), np.int32)), spec)
    assert np.array_equal(grid.G, kat["empty/G"]) and grid.no == 0 and rep.no == 0
    assert rep.max_task_work == 0


@pytest.mark.parametrize("kind", ["uniform", "skewed", "walls"])
@pytest.mark.parametrize("seed", [1, 2, 3])
def test_random_scenes(kat, kind, seed):
    mesh = gen_scene(kind, 400 + 100 * seed, seed)
    spec = spec_for_mesh(mesh, dims=(9, 7, 11))
    grid, rep = builders.build_parallel(mesh, spec)
    assert np.array_equal(grid.G, kat[f"rand_{kind}_{seed}/G"])
    assert np.array_equal(grid.O, kat[f"rand_{kind}_{seed}/O"])
    assert grid.G[-1] == grid.no == rep.no
    assert np.all(np.diff(grid.G.astype(np.int64)) >= 0)


def test_acceptance_100_scenes(hashes):
    """The reference's validate recipe (cli.py:171-196, test_acceptance.py:24-32)."""
    for key in [k for k in hashes if k.startswith("accept_")]:
        h = hashes[key]
        mesh, spec = scene_from_recipe(h["recipe"])
        grid, rep = builders.build_parallel(mesh, spec)
        assert rep.no == h["no"], key
        assert sha(grid.G) == h["G_sha256"] and sha(grid.O) == h["O_sha256"], key


@pytest.mark.parametrize("key", ["cfg1", "skewed100k", "walls100k", "cfg2"] +
                         [f"sweep1m_d{d}" for d in (1, 2, 4, 8, 16, 32, 64)])
def test_config_hashes(hashes, key):
    h = hashes[key]
    mesh, spec = scene_from_recipe(h["recipe"])
    assert list(spec.dims) == h["dims"]
    grid, rep = builders.build_parallel(mesh, spec)
    assert rep.no == h["no"]
    assert sha(grid.G) == h["G_sha256"] and sha(grid.O) == h["O_sha256"]


@pytest.mark.slow
@pytest.mark.parametrize("key", ["cfg3", "cfg3u"])
def test_headline_config_hashes(hashes, key):
    h = hashes[key]
    mesh, spec = scene_from_recipe(h["recipe"])
    grid, rep = builders.build_parallel(mesh, spec)
    assert rep.no == h["no"]
    assert sha(grid.G) == h["G_sha256"] and sha(grid.O) == h["O_sha256"]


def test_random_vs_oracle():
    """Scenes without committed goldens: compare with the C oracle directly."""
    rng = np.random.default_rng(3)
    for i in range(20):
        kind = ("uniform", "skewed", "walls", "lognormal", "arch")[i % 5]
        n = int(rng.integers(1, 60000))
        mesh = gen_scene(kind, n, 50 + i)
        dims = tuple(int(d) for d in rng.integers(1, 90, 3)) if i % 2 else None
        spec = spec_for_mesh(mesh, dims=dims) if dims else spec_for_mesh(mesh, density=float(rng.integers(1, 30)))
        grid, rep = builders.build_parallel(mesh, spec)
        G, O = oracle.build_parallel(mesh.vertices, mesh.triangles, spec)
        assert np.array_equal(grid.G, G) and np.array_equal(grid.O, O), (kind, n, spec.dims)


def test_indexed_mesh_and_custom_bounds_vs_oracle():
    """Shared vertices, unreferenced vertices, a spec that drops most triangles."""
    rng = np.random.default_rng(9)
    V = rng.random((5000, 3)) * 1.4 - 0.2
    T = rng.integers(0, 4000, size=(3000, 3)).astype(np.int32)
    T[::5, 1:] = T[::5, :1] + rng.integers(0, 3, size=(600, 2))   # some small triangles
    mesh = TriangleMesh(V, T)
    for dims in ((1, 1, 1), (3, 1, 1), (17, 23, 5), (40, 30, 20)):
        spec = GridSpec(Aabb([0.2, 0.1, 0.3], [0.9, 0.6, 0.7]), dims)
        grid, _ = builders.build_parallel(mesh, spec)
        G, O = oracle.build_parallel(V, T, spec)
        assert np.array_equal(grid.G, G) and np.array_equal(grid.O, O), dims


def test_huge_object_and_tile_spanning():
    """One triangle covering every cell plus small ones: owner search across many tiles."""
    mesh = gen_scene("skewed", 3000, 4)
    spec = spec_for_mesh(mesh, dims=(160, 150, 140))     # 3.36M cells, NO > 3.36M
    grid, rep = builders.build_parallel(mesh, spec)
    G, O = oracle.build_parallel(mesh.vertices, mesh.triangles, spec)
    assert np.array_equal(grid.G, G) and np.array_equal(grid.O, O)


def test_size_errors():
    V = np.array([[-1, -1, -1], [3, -1, 2], [-1, 3, 2]], np.float64)
    T = np.array([[0, 1, 2]], np.int32)
    mesh = TriangleMesh(V, T)
    with pytest.raises(SizeError):   # ncells > 2^30: the reference's G scan cap
        builders.build_parallel(mesh, GridSpec(Aabb([0, 0, 0], [1, 1, 1]), (1025, 1024, 1024)))
    # NO > 2^30 pairs from 2 full-cover triangles on 2^29+ cells
    mesh2 = TriangleMesh(V, np.array([[0, 1, 2], [0, 1, 2], [0, 1, 2]], np.int32))
    with pytest.raises(SizeError):
        builders.build_parallel(mesh2, GridSpec(Aabb([0, 0, 0], [1, 1, 1]), (1024, 1024, 512)))


def test_invariant_error_on_inverted_box():
    """+inf upper corner with lo > 0: the reference fails its non-negative check."""
    V = np.array([[0.6, 0.6, 0.6], [np.inf, 0.7, 0.7], [0.7, 0.6, 0.7]], np.float64)
    mesh = TriangleMesh(V, np.array([[0, 1, 2]], np.int32))
    with pytest.raises(InvariantError):
        builders.build_parallel(mesh, GridSpec(Aabb([0, 0, 0], [1, 1, 1]), (4, 4, 4)))


def test_repeat_builds_identical_and_workers_ignored():
    mesh = gen_scene("walls", 3000, 5)
    spec = spec_for_mesh(mesh, dims=(30, 31, 29))
    first, _ = builders.build_parallel(mesh, spec, workers=1)
    for w in (None, 8, 64):
        again, _ = builders.build_parallel(mesh, spec, workers=w)
        assert grids_equal(first, again)


def test_fault_injection_hook():
    mesh = gen_scene("uniform", 100, 2)
    spec = spec_for_mesh(mesh, dims=(4, 4, 4))
    clean, _ = builders.build_parallel(mesh, spec)
    builders._fault_inject = True
    try:
        faulty, _ = builders.build_parallel(mesh, spec)
    finally:
        builders._fault_inject = False
    assert not grids_equal(clean, faulty)


@pytest.mark.parametrize("bits", [0, 1, 7, 8, 9, 19, 26, 32])
def test_plugin_radix_sort_kat(kat, bits):
    ks, vs = radix_sort_pairs(kat[f"radix{bits}/keys"], kat[f"radix{bits}/vals"], bits)
    assert np.array_equal(ks, kat[f"radix{bits}/sorted_keys"])
    assert np.array_equal(vs, kat[f"radix{bits}/sorted_vals"])


@pytest.mark.parametrize("n,bits", [(1, 5), (4095, 12), (4097, 16), (1_000_003, 30), (2_000_000, 32)])
def test_plugin_radix_sort_vs_oracle(n, bits):
    rng = np.random.default_rng(n)
    keys = rng.integers(0, 1 << bits, n, dtype=np.uint64).astype(np.uint32)
    keys[::5] = keys[7 % n]
    vals = rng.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32)
    ks, vs = radix_sort_pairs(keys, vals, bits)
    ok, ov = oracle.radix_sort_pairs(keys, vals, bits)
    assert np.array_equal(ks, ok) and np.array_equal(vs, ov)


def test_launch_count_is_native():
    """The build runs our kernels: K1 + K2 + passes + K4 launches are reported."""
    mesh = gen_scene("uniform", 20000, 1)
    spec = spec_for_mesh(mesh)
    g, _ = builders.build_parallel(mesh, spec)
    b = _native.thread_builder()
    nbits = int(spec.ncells - 1).bit_length()
    no = len(g.O)
    # the MSD-first finish: buckets of 2^L cells (~256 pairs each, 2 <= L <= 10), passes over
    # the top nbits - L bits, then k_bucket_sort (pgrid.cu local_bits)
    L = 2
    while L < 10 and L + 1 < nbits and no * (1 << (L + 1)) <= 256 * spec.ncells:
        L += 1
    passes = (nbits - L + 8) // 9                     # <= 9-bit digits
    # K1 + tile scan, tile bounds + K2, count/scan/scatter per pass (pass 0 counted by K2),
    # and k_bucket_sort + its bounds
    assert b.launches() == 5 + 3 * passes


def test_index_out_of_range_detected_on_device():
    """geometry.py:41-43 raises InvariantError for bad indices; duck-typed meshes skip that
    constructor, so K1 validates every index on the device."""
    class RawMesh:
        pass
    m = RawMesh()
    m.vertices = np.random.default_rng(1).random((30, 3))
    m.triangles = np.array([[0, 1, 2], [3, 4, 30]], np.int32)
    m.ntriangles = 2
    spec = GridSpec(Aabb([0, 0, 0], [1, 1, 1]), (4, 4, 4))
    with pytest.raises(InvariantError):
        builders.build_parallel(m, spec)
    m.triangles = np.array([[0, 1, -1]], np.int32)
    with pytest.raises(InvariantError):
        builders.build_parallel(m, spec)


def test_pinned_outputs_are_recycled_and_independent():
    mesh = gen_scene("uniform", 5000, 3)
    spec = spec_for_mesh(mesh)
    g1, _ = builders.build_parallel(mesh, spec)
    keep = (g1.G.copy(), g1.O.copy())
    g2, _ = builders.build_parallel(mesh, spec)       # g1 still alive: distinct buffers
    assert np.array_equal(g1.G, keep[0]) and np.array_equal(g1.O, keep[1])
    assert np.array_equal(g2.G, keep[0]) and np.array_equal(g2.O, keep[1])
    assert g1.G.ctypes.data != g2.G.ctypes.data


def test_sync_free_graph_build_matches_and_reports_capacity(hashes):
    """pg_build_async: eager run, then CUDA-graph replays; identical G/O; capacity errors."""
    import torch
    h = hashes["cfg1"]
    mesh, spec = scene_from_recipe(h["recipe"])
    b = _native.Builder(0)
    Vd = torch.from_numpy(mesh.vertices.copy()).cuda()
    Td = torch.from_numpy(mesh.triangles.copy()).cuda()
    Gd = torch.empty(spec.ncells + 1, dtype=torch.int32, device="cuda")
    Od = torch.empty(h["no"] + 100, dtype=torch.int32, device="cuda")
    for _ in range(3):      # eager + capture, then replays
        Gd.fill_(-1)
        b.build_async(Vd, len(mesh.vertices), Td, len(mesh.triangles), spec, Gd, Od, h["no"] + 100)
        assert b.build_wait() == h["no"]
        assert sha(Gd.cpu().numpy().view(np.uint32)) == h["G_sha256"]
        assert sha(Od[:h["no"]].cpu().numpy().view(np.uint32)) == h["O_sha256"]
    small = torch.empty(1000, dtype=torch.int32, device="cuda")
    b.build_async(Vd, len(mesh.vertices), Td, len(mesh.triangles), spec, Gd, small, 1000)
    assert b.build_wait() == -h["no"]          # capacity exceeded is reported, not silent


def test_build_pipeline_matches_build_parallel(kat, hashes):
    """BuildPipeline / build_many: overlapped builds, results in submission order."""
    items = [kat_case(kat, name) for name in KAT_NAMES]
    items += [scene_from_recipe(hashes[k]["recipe"]) for k in ("cfg1", "skewed100k", "walls100k")]
    items = items * 2
    got = list(builders.build_many(items, depth=2))
    assert len(got) == len(items)
    for (mesh, spec), (grid, rep) in zip(items, got):
        want, wrep = builders.build_parallel(mesh, spec)
        assert np.array_equal(grid.G, want.G) and np.array_equal(grid.O, want.O)
        assert rep.no == wrep.no and rep.total_work == wrep.total_work
    pipe = builders.BuildPipeline(depth=2)
    pipe.submit(*items[0])
    pipe.submit(*items[1])
    with pytest.raises(RuntimeError):
        pipe.submit(*items[2])
    assert pipe.result()[1].no == got[0][1].no and pipe.result()[1].no == got[1][1].no


def test_inverted_boxes_match_reference_verdicts():
    """A lone zero-count inverted box builds an empty grid, two inverted axes build the
    reference's cells, the rest raises (the oracle's verdicts, pinned to the reference)."""
    from test_oracle import _inverted_cases
    for V, T, spec in _inverted_cases():
        try:
            want = oracle.build_parallel(V, T, spec)
        except oracle.OracleInvariantError:
            want = None
        if want is None:
            with pytest.raises(InvariantError):
                builders.build_parallel(TriangleMesh(V, T), spec)
        else:
            grid, rep = builders.build_parallel(TriangleMesh(V, T), spec)
            assert np.array_equal(grid.G, want[0]) and np.array_equal(grid.O, want[1]) and rep.no == len(want[1])


def test_build_pipeline_deferred_corners(hashes):
    """Deferred submits (no NO read back): inverted boxes and out-of-range indices give the
    reference's verdicts at result(), and the pipeline keeps working afterwards."""
    import types
    from test_oracle import _inverted_cases
    mesh0, spec0 = scene_from_recipe(hashes["cfg1"]["recipe"])
    want0, _ = builders.build_parallel(mesh0, spec0)
    pipe = builders.BuildPipeline(depth=1)
    pipe.submit(mesh0, spec0)
    pipe.result()                       # learns a capacity: every later submit is deferred
    for V, T, spec in _inverted_cases():
        try:
            want = oracle.build_parallel(V, T, spec)
        except oracle.OracleInvariantError:
            want = None
        pipe.submit(TriangleMesh(V, T), spec)
        if want is None:
            with pytest.raises(InvariantError):
                pipe.result()
        else:
            grid, rep = pipe.result()
            assert np.array_equal(grid.G, want[0]) and np.array_equal(grid.O, want[1]) and rep.no == len(want[1])
    bad = mesh0.triangles.copy()
    bad[5, 1] = len(mesh0.vertices) + 7   # bypasses TriangleMesh's host check
    pipe.submit(types.SimpleNamespace(vertices=mesh0.vertices, triangles=bad), spec0)
    with pytest.raises(InvariantError):
        pipe.result()
    pipe.submit(mesh0, spec0)
    grid, rep = pipe.result()
    assert np.array_equal(grid.G, want0.G) and np.array_equal(grid.O, want0.O)


def test_cell_boundary_coordinates_bit_exact():
    """K1 floors (a - lo) / cell with a reciprocal-product fast path that defers to the IEEE
    division near integers: vertices exactly on, and a few ulps either side of, cell
    boundaries (and the padded bounds themselves) give the oracle's boxes."""
    rng = np.random.default_rng(11)
    dims = (37, 23, 41)
    lo, hi = np.array([-1.3, 0.7, 2.0]), np.array([4.1, 3.3, 9.7])
    spec = GridSpec(Aabb(lo, hi), dims)
    cell = np.asarray(spec.cell_size, dtype=np.float64)
    n = 60000
    k = rng.integers(0, np.array(dims) + 1, size=(3 * n, 3))
    V = np.asarray(spec.bounds.lo) + k * cell                 # exactly on boundaries (as rounded)
    ulps = rng.integers(-4, 5, size=V.shape)
    V = np.where(ulps > 0, np.nextafter(V, np.inf), V)
    V = np.where(ulps < 0, np.nextafter(V, -np.inf), V)
    m = rng.random(V.shape) < 0.3
    V[m] = (np.asarray(spec.bounds.lo) + rng.random(V.shape) * (hi - lo))[m]
    V[0], V[1], V[2] = spec.bounds.lo, spec.bounds.hi, -np.asarray(spec.bounds.lo)
    T = np.arange(3 * n, dtype=np.int32).reshape(n, 3)
    grid, rep = builders.build_parallel(TriangleMesh(V, T), spec)
    G, O = oracle.build_parallel(V, T, spec)
    assert np.array_equal(grid.G, G) and np.array_equal(grid.O, O) and rep.no == len(O)


def test_no_above_2_32_on_device_count_paths():
    """NO > 2^32-1 (17 full-cover triangles on 2^28 cells): the reference's SizeError
    (builders.py:99-100) on the paths that never read NO back before the expansion -- the
    sync-free graph build and the deferred BuildPipeline -- without a device fault (the
    over-capacity device count voids every kernel after K1)."""
    import torch
    V = np.array([[-1, -1, -1], [3, -1, 2], [-1, 3, 2]], np.float64)
    T = np.zeros((17, 3), np.int32)
    T[:] = [0, 1, 2]
    spec = GridSpec(Aabb([0, 0, 0], [1, 1, 1]), (1024, 512, 512))
    b = _native.Builder(0)
    Vd = torch.from_numpy(V).cuda()
    Td = torch.from_numpy(T).cuda()
    Gd = torch.empty(spec.ncells + 1, dtype=torch.int32, device="cuda")
    Od = torch.empty(4096, dtype=torch.int32, device="cuda")
    for _ in range(2):
        b.build_async(Vd, len(V), Td, len(T), spec, Gd, Od, 4096)
        with pytest.raises(SizeError):
            b.build_wait()
    torch.cuda.synchronize()                      # the context survived
    small = gen_scene("uniform", 500, 1)
    sspec = spec_for_mesh(small)
    pipe = builders.BuildPipeline(depth=2)
    pipe.submit(small, sspec)
    want, _ = pipe.result()                       # learns a capacity: the next submit is deferred
    pipe.submit(TriangleMesh(V, T), spec)
    pipe.submit(small, sspec)
    with pytest.raises(SizeError):
        pipe.result()
    again, _ = pipe.result()
    assert grids_equal(want, again)


def test_host_input_soup_and_near_soup():
    """Host meshes whose index array is exactly the soup 0, 1, 2, ... skip its transfer (K1
    regenerates it); a single different index must take the copied path. Pageable and
    page-locked inputs, against the oracle."""
    mesh = gen_scene("lognormal", 300_000, 5)
    spec = spec_for_mesh(mesh)
    V = np.ascontiguousarray(mesh.vertices).copy()
    T = np.ascontiguousarray(mesh.triangles).copy()
    G, O = oracle.build_parallel(V, T, spec)
    grid, _ = builders.build_parallel(TriangleMesh(V, T), spec)          # pageable, implicit soup
    assert np.array_equal(grid.G, G) and np.array_equal(grid.O, O)
    T2 = T.copy()
    T2[123_457, 1], T2[200_001, 2] = T2[200_001, 2], T2[123_457, 1]      # not a soup any more
    G2, O2 = oracle.build_parallel(V, T2, spec)
    grid, _ = builders.build_parallel(TriangleMesh(V, T2), spec)
    assert np.array_equal(grid.G, G2) and np.array_equal(grid.O, O2)
    _native.host_register(V)
    _native.host_register(T)
    try:                                                                  # page-locked inputs
        grid, _ = builders.build_parallel(TriangleMesh(V, T), spec)
        assert np.array_equal(grid.G, G) and np.array_equal(grid.O, O)
    finally:
        _native.host_unregister(V)
        _native.host_unregister(T)


def test_pinned_soup_chunked_copy_with_k1_per_chunk(hashes):
    """A page-locked soup of >= 64 MB of vertices is copied in chunks on a copy stream and K1
    runs on each chunk as it lands (cfg2: 1M triangles, 72 MB); an indexed variant of the same
    mesh takes the whole-V path. Golden hash / oracle."""
    h = hashes["cfg2"]
    mesh, spec = scene_from_recipe(h["recipe"])
    V = np.ascontiguousarray(mesh.vertices).copy()
    T = np.ascontiguousarray(mesh.triangles).copy()
    assert V.nbytes >= 64 << 20
    _native.host_register(V)
    _native.host_register(T)
    try:
        for _ in range(2):
            grid, rep = builders.build_parallel(TriangleMesh(V, T), spec)
            assert sha(grid.G) == h["G_sha256"] and sha(grid.O) == h["O_sha256"] and rep.no == h["no"]
        pipe = builders.BuildPipeline(depth=2)
        for _ in range(3):
            pipe.submit(TriangleMesh(V, T), spec)
            if len(pipe) == 2:
                g, _ = pipe.result()
                assert sha(g.G) == h["G_sha256"] and sha(g.O) == h["O_sha256"]
        while len(pipe):
            g, _ = pipe.result()
            assert sha(g.G) == h["G_sha256"] and sha(g.O) == h["O_sha256"]
        T2 = T.copy()
        T2[0, 0], T2[-1, 2] = T2[-1, 2], T2[0, 0]        # not a soup: K1 waits for every row
        _native.host_register(T2)
        try:
            G2, O2 = oracle.build_parallel(V, T2, spec)
            grid, _ = builders.build_parallel(TriangleMesh(V, T2), spec)
            assert np.array_equal(grid.G, G2) and np.array_equal(grid.O, O2)
        finally:
            _native.host_unregister(T2)
    finally:
        _native.host_unregister(V)
        _native.host_unregister(T)
