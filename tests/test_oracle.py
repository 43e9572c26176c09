"""The CPU oracle (oracle/pgrid_oracle.c) pinned against the reference's golden vectors.

Golden vectors come from running the unmodified reference (tests/golden/make_golden.py);
when oracle/_ref holds a built reference, the oracle is also cross-checked live.
"""

import numpy as np
import pytest

import oracle
from util import KAT_NAMES, kat_case, scene_from_recipe, sha


@pytest.mark.parametrize("name", KAT_NAMES)
def test_oracle_kat_all_stages(kat, name):
    mesh, spec = kat_case(kat, name)
    lo, hi, keep = oracle.cell_boxes(mesh.vertices, mesh.triangles, spec)
    assert np.array_equal(lo, kat[f"{name}/box_lo"])
    assert np.array_equal(hi, kat[f"{name}/box_hi"])
    assert np.array_equal(keep, kat[f"{name}/keep"])
    G, O, st = oracle.build_parallel(mesh.vertices, mesh.triangles, spec, stages=True)
    assert np.array_equal(G, kat[f"{name}/G"])
    assert np.array_equal(O, kat[f"{name}/O"])
    assert st["no"] == int(kat[f"{name}/no"])
    assert np.array_equal(st["global_c"], kat[f"{name}/global_c"])
    assert np.array_equal(st["obj_ids"], kat[f"{name}/obj_ids"])
    assert np.array_equal(st["sorted_c"], kat[f"{name}/sorted_c"])
    assert np.array_equal(st["sorted_o"], kat[f"{name}/sorted_o"])


def test_oracle_empty(kat):
    from paper_2403_10647_b200.gridcore import Aabb, GridSpec
    spec = GridSpec(Aabb([0, 0, 0], [1, 1, 1]), (2, 2, 2))
    G, O = oracle.build_parallel(np.zeros((0, 3)), np.zeros((0, 3), np.int32), spec)
    assert np.array_equal(G, kat["empty/G"]) and len(O) == 0


@pytest.mark.parametrize("bits", [0, 1, 7, 8, 9, 19, 26, 32])
def test_oracle_radix_kat(kat, bits):
    ks, vs = oracle.radix_sort_pairs(kat[f"radix{bits}/keys"], kat[f"radix{bits}/vals"], bits)
    assert np.array_equal(ks, kat[f"radix{bits}/sorted_keys"])
    assert np.array_equal(vs, kat[f"radix{bits}/sorted_vals"])


@pytest.mark.parametrize("kind", ["uniform", "skewed", "walls"])
@pytest.mark.parametrize("seed", [1, 2, 3])
def test_oracle_random_scenes(kat, kind, seed):
    from paper_2403_10647_b200 import gen_scene, spec_for_mesh
    mesh = gen_scene(kind, 400 + 100 * seed, seed)
    spec = spec_for_mesh(mesh, dims=(9, 7, 11))
    G, O = oracle.build_parallel(mesh.vertices, mesh.triangles, spec)
    assert np.array_equal(G, kat[f"rand_{kind}_{seed}/G"])
    assert np.array_equal(O, kat[f"rand_{kind}_{seed}/O"])


def test_oracle_acceptance_100_scenes(hashes):
    keys = [k for k in hashes if k.startswith("accept_")]
    assert len(keys) == 100
    for key in keys:
        h = hashes[key]
        mesh, spec = scene_from_recipe(h["recipe"])
        assert list(spec.dims) == h["dims"]
        G, O = oracle.build_parallel(mesh.vertices, mesh.triangles, spec)
        assert len(O) == h["no"] and sha(G) == h["G_sha256"] and sha(O) == h["O_sha256"], key


@pytest.mark.parametrize("key", ["cfg1", "skewed100k", "cfg2", "sweep1m_d1", "sweep1m_d64"])
def test_oracle_config_hashes(hashes, key):
    h = hashes[key]
    mesh, spec = scene_from_recipe(h["recipe"])
    assert list(spec.dims) == h["dims"]
    G, O = oracle.build_parallel(mesh.vertices, mesh.triangles, spec)
    assert len(O) == h["no"]
    assert sha(G) == h["G_sha256"] and sha(O) == h["O_sha256"]


def test_oracle_vs_live_reference():
    ref = oracle.reference_module()
    if ref is None:
        pytest.skip("oracle/_ref not built")
    rng = np.random.default_rng(11)
    for i in range(12):
        n = int(rng.integers(1, 3000))
        kind = ("uniform", "skewed", "walls")[i % 3]
        mesh = ref.gen_scene(kind, n, 1000 + i)
        dims = tuple(int(d) for d in rng.integers(1, 40, 3))
        spec = ref.spec_for_mesh(mesh, dims=dims)
        g, rep = ref.build_parallel(mesh, spec)
        G, O = oracle.build_parallel(mesh.vertices, mesh.triangles, spec)
        assert np.array_equal(G, g.G) and np.array_equal(O, g.O)


def test_oracle_size_error():
    from paper_2403_10647_b200.gridcore import Aabb, GridSpec
    # one triangle covering 1024^3 cells: NO > 2^30 scan cap -> SizeError in the reference
    spec = GridSpec(Aabb([0, 0, 0], [1, 1, 1]), (1025, 1024, 1024))
    V = np.array([[-1, -1, -1], [3, -1, 2], [-1, 3, 2]], np.float64)
    with pytest.raises(oracle.OracleSizeError):
        oracle.build_parallel(V, np.array([[0, 1, 2]], np.int32), spec)


def _inverted_cases():
    """Triangles whose clipped box inverts (an infinite upper corner): the reference accepts a
    lone zero-count one (empty grid) and builds cells from a box inverted on two axes (a
    positive count) when they land in [0, ncells); every other arrangement raises."""
    from paper_2403_10647_b200.gridcore import Aabb, GridSpec
    inv1 = [[0.6, 0.1, 0.1], [np.inf, 0.2, 0.1], [0.7, 0.1, 0.2]]          # one inverted axis
    inv3 = [[0.6, 0.6, 0.6], [np.inf, np.inf, np.inf], [0.7, 0.7, 0.7]]    # negative count at 4^3
    inv2 = [[0.6, 0.6, 0.1], [np.inf, np.inf, 0.2], [0.7, 0.7, 0.2]]       # two axes: one pair, cell 10
    inv2w = [[0.8, 0.8, 0.3], [np.inf, np.inf, 0.6], [0.85, 0.85, 0.3]]    # 8 pairs at 5^3
    inv2n = [[0.1, 0.8, 0.8], [np.inf, 1e300, np.inf], [0.1, 0.85, 0.85]]  # 3 axes: 1 x -3 x -3 ... at 5^3
    good = [[0.1, 0.1, 0.1], [0.2, 0.2, 0.2], [0.1, 0.2, 0.1]]
    far = [[5.0, 5, 5], [6, 5, 5], [5, 6, 5]]                              # dropped
    cases = []
    for tris, dims in (([inv1], (2, 2, 2)), ([inv1, far], (2, 2, 2)), ([far, inv1, far], (3, 3, 3)),
                       ([good, inv1], (2, 2, 2)), ([inv1, good], (2, 2, 2)), ([inv3], (4, 4, 4)),
                       ([inv1, inv1], (2, 2, 2)), ([inv2], (4, 4, 4)), ([good, inv2, far], (4, 4, 4)),
                       ([inv2, good, inv2], (4, 4, 4)), ([inv2w], (5, 5, 5)), ([good, inv2w], (5, 5, 5)),
                       ([inv2n], (5, 5, 5)), ([inv2, inv1], (4, 4, 4))):
        V = np.array([v for t in tris for v in t], float)
        T = np.arange(len(V), dtype=np.int32).reshape(-1, 3)
        cases.append((V, T, GridSpec(Aabb([0, 0, 0], [1, 1, 1]), dims)))
    return cases


def test_oracle_inverted_boxes_vs_live_reference():
    ref = oracle.reference_module()
    if ref is None:
        pytest.skip("oracle/_ref not built")
    import warnings
    from pargrid.geometry import Aabb as RA, TriangleMesh as RM
    from pargrid.gridcore import GridSpec as RS
    for V, T, spec in _inverted_cases():
        rspec = RS(RA(spec.bounds.lo, spec.bounds.hi), spec.dims)
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            try:
                g, _ = ref.build_parallel(RM(V, T), rspec)
                want = (g.G, g.O)
            except ref.errors.InvariantError:
                want = None
        try:
            got = oracle.build_parallel(V, T, spec)
        except oracle.OracleInvariantError:
            got = None
        assert (want is None) == (got is None), (V, spec.dims)
        if want is not None:
            assert np.array_equal(got[0], want[0]) and np.array_equal(got[1], want[1])


def test_oracle_inverted_golden():
    """Every golden inverted-box verdict (and grid) of the reference, make_golden_inverted.py."""
    from util import inverted_cases
    n_grid = 0
    for name, V, T, spec, verdict, G, O in inverted_cases():
        try:
            got = oracle.build_parallel(V, T, spec)
            code = 0
        except oracle.OracleSizeError:
            code = 1
        except oracle.OracleInvariantError:
            code = 2
        assert code == verdict, name
        if verdict == 0:
            n_grid += 1
            assert np.array_equal(got[0], G) and np.array_equal(got[1], O), name
    assert n_grid >= 40
