"""Generate the golden parity fixtures by running the UNMODIFIED reference package.

Run in the build container (where /root/reference exists and `make -C oracle ref` has
installed it into oracle/_ref):

    python tests/golden/make_golden.py            # small fixtures + config hashes
    python tests/golden/make_golden.py --quick    # skip the 10M-triangle configs

Outputs (committed):
  tests/golden/kat.npz      small scenes with full G/O and every record= stage array
  tests/golden/hashes.json  sha256 of G and O (+ NO, dims) for scenes too large to commit
Inputs are regenerated from recipes (paper_2403_10647_b200.scenes, bit-identical to the
reference's gen_scene for its kinds), so the fixtures stay small.
"""

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle", "_ref"))

import pargrid  # noqa: E402  (the reference)
from pargrid import kernels as ref_kernels  # noqa: E402
from pargrid.geometry import Aabb as RAabb, TriangleMesh as RMesh  # noqa: E402
from pargrid.gridcore import GridSpec as RSpec, object_cell_boxes  # noqa: E402

from paper_2403_10647_b200 import scenes  # noqa: E402


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def kat_scenes():
    """Hand-built scenes pinning edge semantics: (name, vertices, triangles, lo, hi, dims)."""
    out = []
    # test_builders.py:13-29 walkthrough
    out.append(("walkthrough",
                [[0.1, 0.1, 0.5], [1.5, 0.3, 0.5], [0.8, 0.9, 0.5],
                 [1.2, 0.5, 0.3], [1.9, 1.8, 0.3], [1.5, 1.2, 0.3]],
                [[0, 1, 2], [3, 4, 5]], [0, 0, 0], [2, 2, 1], (2, 2, 1)))
    # test_builders.py:76-83 full cover
    out.append(("full_cover", [[-1, -1, -1], [3, -1, 2], [-1, 3, 2]], [[0, 1, 2]],
                [0, 0, 0], [1, 1, 1], (2, 2, 2)))
    # test_builders.py:99-107 dropped triangle keeps original ids
    out.append(("dropped", [[5, 5, 5], [6, 5, 5], [5, 6, 5],
                            [0.1, 0.1, 0.1], [0.2, 0.1, 0.1], [0.1, 0.2, 0.1]],
                [[0, 1, 2], [3, 4, 5]], [0, 0, 0], [1, 1, 1], (2, 2, 2)))
    # max-face clamp (test_gridcore.py:94-96) and min-face touching
    out.append(("faces", [[1, 1, 1], [1, 1, 1], [1, 1, 1], [0, 0, 0], [0, 0, 0], [0, 0, 0],
                          [1.0, 0.5, 0.5], [2.0, 0.5, 0.5], [1.5, 0.6, 0.5]],
                [[0, 1, 2], [3, 4, 5], [6, 7, 8]], [0, 0, 0], [1, 1, 1], (4, 3, 5)))
    # non-finite coordinates: NaN drops, +/-inf and huge values hit the int64 cast path
    big = 1e300
    out.append(("nonfinite",
                [[np.nan, 0.2, 0.2], [0.3, 0.3, 0.3], [0.4, 0.2, 0.3],
                 [-np.inf, 0.2, 0.2], [0.3, 0.3, 0.3], [0.4, 0.2, 0.3],
                 [0.2, 0.2, 0.2], [np.inf, 0.3, 0.3], [0.4, 0.2, 0.3],
                 [-big, 0.5, 0.5], [big, 0.6, 0.6], [0.5, 0.7, 0.5],
                 [0.1, 0.1, 0.1], [0.2, np.nan, 0.2], [0.3, 0.3, 0.3],
                 [0.5, 0.5, 0.5], [0.6, 0.5, 0.5], [0.55, 0.6, 0.5]],
                [[0, 1, 2], [3, 4, 5], [6, 7, 8], [9, 10, 11], [12, 13, 14], [15, 16, 17]],
                [0, 0, 0], [1, 1, 1], (3, 4, 5)))
    # shared (indexed, non-soup) vertices, unreferenced vertices, degenerate triangles
    rng = np.random.default_rng(5)
    v = rng.random((40, 3))
    t = rng.integers(0, 30, size=(60, 3))
    t[::7] = t[::7, :1]  # degenerate: all three corners equal
    out.append(("indexed", v.tolist(), t.tolist(), [0, 0, 0], [1, 1, 1], (5, 6, 7)))
    # one-cell grid (key_bits = 0: no radix pass)
    out.append(("one_cell", v.tolist(), t.tolist(), [0, 0, 0], [1, 1, 1], (1, 1, 1)))
    # many zero-count (dropped) objects between kept ones
    vv = []
    tt = []
    for i in range(300):
        base = [0.5, 0.5, 0.5] if i % 37 == 0 else [3.0 + i, 3.0, 3.0]
        vv += [base, [base[0] + 0.01, base[1], base[2]], [base[0], base[1] + 0.01, base[2]]]
        tt.append([3 * i, 3 * i + 1, 3 * i + 2])
    out.append(("sparse_kept", vv, tt, [0, 0, 0], [1, 1, 1], (3, 3, 3)))
    return out


def record_arrays(mesh, spec):
    rec = {}
    grid, report = pargrid.build_parallel(mesh, spec, record=rec)
    lo, hi, keep = object_cell_boxes(mesh, spec)
    out = {"G": grid.G, "O": grid.O, "no": np.int64(report.no),
           "box_lo": lo, "box_hi": hi, "keep": keep}
    for k in ("v", "offsets", "obj_ids", "rel_c", "global_c", "sorted_c", "sorted_o",
              "rle_uniques", "rle_counts", "g"):
        out[k] = np.asarray(rec.get(k, np.zeros(0, np.int64)))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    args = ap.parse_args()
    ref_kernels.set_backend("c")
    arrays = {}
    hashes = {"reference": "pargrid 0.1.0 from /root/reference/pkg (C lane)", "scenes": {}}

    for name, v, t, lo, hi, dims in kat_scenes():
        mesh = RMesh(np.array(v, dtype=np.float64), np.array(t, dtype=np.int32))
        spec = RSpec(RAabb(lo, hi), dims)
        arrays[f"{name}/V"] = mesh.vertices
        arrays[f"{name}/T"] = mesh.triangles
        arrays[f"{name}/lo"] = spec.bounds.lo
        arrays[f"{name}/hi"] = spec.bounds.hi
        arrays[f"{name}/dims"] = np.array(dims, np.int64)
        for k, a in record_arrays(mesh, spec).items():
            arrays[f"{name}/{k}"] = a
    # empty mesh (test_builders.py:66-73)
    empty = RMesh(np.zeros((0, 3)), np.zeros((0, 3), np.int32))
    g, r = pargrid.build_parallel(empty, RSpec(RAabb([0, 0, 0], [1, 1, 1]), (2, 2, 2)))
    arrays["empty/G"] = g.G
    arrays["empty/O"] = g.O

    # radix-sort KATs (test_primitives.py:90-124): stability on duplicate keys
    rng = np.random.default_rng(20260823)
    for bits in (0, 1, 7, 8, 9, 19, 26, 32):
        n = 5000
        keys = (rng.integers(0, 1 << 32, n, dtype=np.uint64) & ((1 << bits) - 1)).astype(np.uint32) \
            if bits else np.zeros(n, np.uint32)
        keys[::3] = keys[0]
        vals = np.arange(n, dtype=np.uint32)[::-1].copy()
        ks, vs = pargrid.primitives.radix_sort_pairs(keys, vals, bits)
        arrays[f"radix{bits}/keys"] = keys
        arrays[f"radix{bits}/vals"] = vals
        arrays[f"radix{bits}/sorted_keys"] = np.asarray(ks, np.uint32)
        arrays[f"radix{bits}/sorted_vals"] = np.asarray(vs, np.uint32)

    # randomised equivalence scenes (test_builders.py:86-96) -- full arrays
    for kind in ("uniform", "skewed", "walls"):
        for seed in (1, 2, 3):
            n = 400 + 100 * seed
            mesh = pargrid.gen_scene(kind, n, seed)
            spec = pargrid.spec_for_mesh(mesh, dims=(9, 7, 11))
            g, _ = pargrid.build_parallel(mesh, spec)
            arrays[f"rand_{kind}_{seed}/G"] = g.G
            arrays[f"rand_{kind}_{seed}/O"] = g.O

    # acceptance recipe (test_acceptance.py:24-32 -> cli.py:171-196): hashes only
    def put(key, recipe, mesh, spec, t0):
        g, rep = pargrid.build_parallel(mesh, spec)
        hashes["scenes"][key] = {"recipe": recipe, "dims": list(spec.dims), "no": int(rep.no),
                                 "G_sha256": sha(g.G), "O_sha256": sha(g.O),
                                 "ref_seconds": round(time.perf_counter() - t0, 3)}
        print(key, spec.dims, rep.no, f"{time.perf_counter() - t0:.2f}s", flush=True)

    # the reference's own validate recipe: u = _uniforms(seed, 2*nscenes, 201)
    nsc, vseed = 100, 20260823
    u = pargrid.geometry._uniforms(vseed, 2 * nsc, 201).reshape(nsc, 2)
    for i in range(nsc):
        kind = ("uniform", "skewed", "walls")[i % 3]
        n = 1 + int(u[i, 0] * (2000 - 1))
        scene_seed = vseed * 1_000_003 + i
        dims = tuple(1 + int(x * (32 - 1)) for x in pargrid.geometry._uniforms(scene_seed, 3, 202))
        mesh = pargrid.gen_scene(kind, n, scene_seed)
        spec = pargrid.spec_for_mesh(mesh, dims=dims)
        put(f"accept_{i}", {"kind": kind, "n": n, "seed": scene_seed, "dims": list(dims)},
            mesh, spec, time.perf_counter())

    configs = [("cfg1", "uniform", 100_000, 7, 5.0), ("cfg2", "lognormal", 1_000_000, 7, 5.0),
               ("skewed100k", "skewed", 100_000, 7, 5.0), ("walls100k", "walls", 100_000, 7, 5.0)]
    for d in (1.0, 2.0, 4.0, 8.0, 16.0, 32.0, 64.0):
        configs.append((f"sweep1m_d{int(d)}", "uniform", 1_000_000, 7, d))
    if not args.quick:
        configs += [("cfg3", "arch", 10_000_000, 7, 4.0), ("cfg3u", "uniform", 10_000_000, 7, 5.0)]
    for key, kind, n, seed, density in configs:
        t0 = time.perf_counter()
        m = scenes.gen_scene(kind, n, seed, density)
        mesh = RMesh(m.vertices, m.triangles)
        spec = pargrid.spec_for_mesh(mesh, density=density)
        put(key, {"kind": kind, "n": n, "seed": seed, "density": density}, mesh, spec, t0)

    np.savez_compressed(os.path.join(HERE, "kat.npz"), **arrays)
    with open(os.path.join(HERE, "hashes.json"), "w") as fh:
        json.dump(hashes, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
