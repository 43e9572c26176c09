"""The ray-casting oracle (oracle/pgrid_oracle.c: orc_dda_cast / orc_brute_cast) pinned to the
reference: golden vectors from the reference's compiled lane (tests/golden/rays.npz) and,
where oracle/_ref is built, the live reference. CPU only."""

import numpy as np
import pytest

import oracle
from paper_2403_10647_b200 import traverse
from util import RAY_CASES, ray_case, sha


@pytest.mark.parametrize("name", RAY_CASES)
def test_oracle_dda_matches_reference_golden(rays, name):
    arrays, meta = rays
    mesh, spec, o, d, t = ray_case(rays, name)
    G, O = oracle.build_parallel(mesh.vertices, mesh.triangles, spec)
    assert sha(G) == meta[name]["G_sha256"] and sha(O) == meta[name]["O_sha256"]
    ids, ts = oracle.dda_cast(G, O, mesh.vertices, mesh.triangles, spec, o, d, t)
    assert np.array_equal(ids, arrays[f"{name}/ids"])
    assert np.array_equal(ts.view(np.uint64), arrays[f"{name}/ts"].view(np.uint64))  # bit-exact


@pytest.mark.parametrize("name", [c for c in RAY_CASES if c not in ("cfg2", "arch1m")])
def test_oracle_brute_force_matches_reference(rays, name):
    arrays, _ = rays
    mesh, spec, o, d, t = ray_case(rays, name)
    sl = slice(None, None, 8 if name == "cfg1" else 1)   # keep the CPU suite short
    bids, bts = oracle.brute_cast(mesh.vertices, mesh.triangles, o[sl], d[sl], t[sl])
    assert len(traverse.compare_hits(bids, bts, arrays[f"{name}/brute_ids"][sl], arrays[f"{name}/brute_ts"][sl])) == 0


@pytest.mark.parametrize("name", [c for c in RAY_CASES if c not in ("cfg2", "arch1m")])
def test_dda_agrees_with_brute_force(rays, name):
    """The reference's own end-to-end property (test_traverse.py:173-198, cli.py:199-218)."""
    arrays, _ = rays
    assert len(traverse.compare_hits(arrays[f"{name}/ids"], arrays[f"{name}/ts"],
                                     arrays[f"{name}/brute_ids"], arrays[f"{name}/brute_ts"])) == 0


def test_make_rays_mirror_vs_live_reference():
    ref = oracle.reference_module()
    if ref is None:
        pytest.skip("oracle/_ref not built")
    from pargrid.cli import make_rays
    from paper_2403_10647_b200 import gen_scene, spec_for_mesh
    spec = spec_for_mesh(gen_scene("uniform", 500, 3))
    a = make_rays(spec.bounds, 300, 9)
    b = traverse.make_rays(spec.bounds, 300, 9)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


def test_oracle_dda_vs_live_reference_random():
    ref = oracle.reference_module()
    if ref is None:
        pytest.skip("oracle/_ref not built")
    from pargrid.traverse import dda_cast as ref_dda
    rng = np.random.default_rng(4)
    for kind, n in (("uniform", 3000), ("walls", 400), ("skewed", 5000)):
        m = ref.gen_scene(kind, n, 11)
        dims = tuple(int(x) for x in rng.integers(1, 40, 3))
        spec = ref.spec_for_mesh(m, dims=dims)
        grid, _ = ref.build_parallel(m, spec)
        o = spec.bounds.lo - 0.3 + rng.random((2000, 3)) * (spec.bounds.hi - spec.bounds.lo + 0.6)
        d = rng.normal(size=(2000, 3))
        d[1::7, 0] = 0.0
        d[::11, 1:] = 0.0         # (never both: a zero direction never terminates in the reference)
        d[::11, 0] = 1.0
        d /= np.linalg.norm(d, axis=1, keepdims=True)
        t = np.where(rng.random(2000) < 0.2, np.inf, rng.random(2000) * 2)
        want = ref_dda(grid, m, o, d, t)
        got = oracle.dda_cast(grid.G, grid.O, m.vertices, m.triangles, spec, o, d, t)
        assert np.array_equal(got[0], want[0]) and np.array_equal(got[1].view(np.uint64), want[1].view(np.uint64))


def test_ray_validation():
    from paper_2403_10647_b200.errors import InvariantError
    with pytest.raises(InvariantError):
        traverse.Ray((0, 0, 0), (0, 0, 2))
    with pytest.raises(InvariantError):
        traverse.Ray((0, 0, 0), (0, 0, 1), t_max=0)
