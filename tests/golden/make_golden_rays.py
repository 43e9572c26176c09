"""Golden ray-casting fixtures from the UNMODIFIED reference.

    python tests/golden/make_golden_rays.py      # needs oracle/_ref (make -C oracle ref)

For every case: the rays (stored explicitly: make_rays uses libm sin/cos, whose last bit
may differ across hosts), the reference's compiled-lane dda_cast result (ids, ts) and its
brute_force_cast result. Scenes are regenerated from recipes (gen_scene is bit-identical
across hosts) and gridded with the reference build_parallel; the grid hashes are stored so
a test can confirm it casts against the same grid.
Output: tests/golden/rays.npz (committed).
"""

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle", "_ref"))

import pargrid  # noqa: E402  (the reference)
from pargrid import kernels as ref_kernels  # noqa: E402
from pargrid.cli import make_rays  # noqa: E402
from pargrid.geometry import Aabb as RAabb, TriangleMesh as RMesh  # noqa: E402
from pargrid.gridcore import GridSpec as RSpec  # noqa: E402
from pargrid.traverse import brute_force_cast, dda_cast  # noqa: E402

from paper_2403_10647_b200 import scenes  # noqa: E402


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def special_rays(spec, rng, n):
    """Edge-case rays: axis-aligned (zero direction components), origins on cell planes,
    inside the grid, tangent to the bounds, pointing away, short t_max."""
    lo, hi, cs = spec.bounds.lo, spec.bounds.hi, spec.cell_size
    out_o, out_d, out_t = [], [], []
    for i in range(n):
        kind = i % 6
        if kind == 0:      # axis-aligned from outside through cell centres / planes
            ax = i % 3
            o = lo + (rng.integers(0, spec.dims) + (0.5 if i % 4 else 0.0)) * cs
            d = np.zeros(3)
            sgn = 1.0 if (i // 3) % 2 else -1.0
            o[ax] = lo[ax] - 0.25 if sgn > 0 else hi[ax] + 0.25
            d[ax] = sgn
        elif kind == 1:    # two zero components is covered above; one zero component here
            o = lo + rng.random(3) * (hi - lo)
            d = rng.normal(size=3)
            d[i % 3] = 0.0
        elif kind == 2:    # origin on a cell corner inside the grid
            o = lo + rng.integers(0, spec.dims) * cs
            d = rng.normal(size=3)
        elif kind == 3:    # along a bounds face (tangent)
            o = lo.copy()
            o[i % 3] = lo[i % 3] if i % 2 else hi[i % 3]
            o[(i + 1) % 3] = lo[(i + 1) % 3] - 0.1
            o[(i + 2) % 3] = lo[(i + 2) % 3] + rng.random() * (hi - lo)[(i + 2) % 3]
            d = np.zeros(3)
            d[(i + 1) % 3] = 1.0
        elif kind == 4:    # pointing away from the grid
            o = hi + 0.5 + rng.random(3)
            d = np.abs(rng.normal(size=3)) + 0.1
        else:              # random inside, short segment
            o = lo + rng.random(3) * (hi - lo)
            d = rng.normal(size=3)
        d = d / np.linalg.norm(d)
        t = [0.05, 0.3, 2.0, np.inf][i % 4] if kind == 5 else (np.inf if i % 5 == 0 else 10.0)
        out_o.append(o)
        out_d.append(d)
        out_t.append(t)
    return np.array(out_o), np.array(out_d), np.array(out_t, dtype=np.float64)


def main():
    ref_kernels.set_backend("c")
    arrays = {}
    meta = {}

    def put(name, recipe, mesh, spec, o, d, t, brute=True):
        grid, _ = pargrid.build_parallel(mesh, spec)
        ids, ts = dda_cast(grid, mesh, o, d, t)
        arrays[f"{name}/origins"] = o
        arrays[f"{name}/dirs"] = d
        arrays[f"{name}/t_max"] = t
        arrays[f"{name}/ids"] = ids
        arrays[f"{name}/ts"] = ts
        if brute:
            bids, bts = brute_force_cast(mesh, o, d, t)
            arrays[f"{name}/brute_ids"] = bids
            arrays[f"{name}/brute_ts"] = bts
        meta[name] = {"recipe": recipe, "dims": list(spec.dims), "G_sha256": sha(grid.G),
                      "O_sha256": sha(grid.O), "hits": int((ids >= 0).sum()), "rays": len(o)}
        print(name, spec.dims, len(o), "hits", int((ids >= 0).sum()), flush=True)

    # unit triangle (test_traverse.py:15-16, 135-152)
    mesh = RMesh([[0, 0, 0], [1, 0, 0], [0, 1, 0]], [[0, 1, 2]])
    spec = pargrid.spec_for_mesh(mesh, dims=(2, 2, 1))
    o = np.array([[0.25, 0.25, -1], [5, 5, -1], [0.25, 0.25, -1], [0.5, 0.0, -1], [0.25, 0.25, -1],
                  [0.0, 0.0, 1.0], [0.5, 0.5, -1], [1e-10, 1e-10, 3.0]], float)
    d = np.array([[0, 0, 1], [0, 0, 1], [0, 0, 1], [0, 0, 1], [0, 0, -1], [0, 0, -1], [0, 0, 1], [0, 0, -1]],
                 float)
    t = np.array([np.inf, np.inf, 0.5, np.inf, np.inf, 1.0, np.inf, 5.0])
    put("unit", {"kind": "unit_triangle", "dims": [2, 2, 1]}, mesh, spec, o, d, t)

    # the reference's validate_raycast recipe (cli.py:199-218), seed 20260823, 2000 rays
    seed, nsc = 20260823, 10
    for i in range(nsc):
        kind = ("uniform", "skewed", "walls")[i % 3]
        scene_seed = seed * 2_000_003 + i
        mesh = pargrid.gen_scene(kind, 200 + 37 * i, scene_seed)
        spec = pargrid.spec_for_mesh(mesh, density=5.0)
        o, d, t = make_rays(spec.bounds, 200, scene_seed)
        put(f"validate_{i}", {"kind": kind, "n": 200 + 37 * i, "seed": scene_seed, "density": 5.0},
            mesh, spec, o, d, t)

    # rays from inside (test_traverse.py:187-198) and special rays, three scene kinds
    for kind, n, s in (("walls", 200, 17), ("uniform", 2000, 18), ("skewed", 3000, 19)):
        mesh = pargrid.gen_scene(kind, n, s)
        spec = pargrid.spec_for_mesh(mesh)
        rng = np.random.default_rng(s)
        oi = spec.bounds.lo + rng.random((300, 3)) * (spec.bounds.hi - spec.bounds.lo)
        di = rng.normal(size=(300, 3))
        di /= np.linalg.norm(di, axis=1, keepdims=True)
        ti = np.full(300, 10.0)
        os_, ds, ts_ = special_rays(spec, rng, 300)
        put(f"inside_{kind}", {"kind": kind, "n": n, "seed": s, "density": 5.0}, mesh, spec,
            np.concatenate([oi, os_]), np.concatenate([di, ds]), np.concatenate([ti, ts_]))

    # larger scenes: BASELINE configs 1 and 2 recipes and a 1M arch scene (hits only vs the
    # compiled lane; brute force is O(rays x triangles))
    for name, kind, n, dens, nr in (("cfg1", "uniform", 100_000, 5.0, 4000),
                                    ("cfg2", "lognormal", 1_000_000, 5.0, 4000),
                                    ("arch1m", "arch", 1_000_000, 4.0, 4000)):
        m = scenes.gen_scene(kind, n, 7, dens)
        mesh = RMesh(m.vertices, m.triangles)
        spec = pargrid.spec_for_mesh(mesh, density=dens)
        o, d, t = make_rays(spec.bounds, nr, 31)
        rng = np.random.default_rng(32)
        os_, ds, ts_ = special_rays(spec, rng, 600)
        put(name, {"kind": kind, "n": n, "seed": 7, "density": dens}, mesh, spec,
            np.concatenate([o, os_]), np.concatenate([d, ds]), np.concatenate([t, ts_]), brute=(n <= 100_000))

    np.savez_compressed(os.path.join(HERE, "rays.npz"), **arrays)
    with open(os.path.join(HERE, "rays.json"), "w") as fh:
        json.dump({"reference": "pargrid 0.1.0 from /root/reference/pkg (C lane dda_cast)", "cases": meta},
                  fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
