"""Golden hashes for BASELINE.json configs 4 and 5 (10M at grid densities 1..64, 100M).

    python tests/golden/make_golden_big.py [--only cfg4_d1,cfg5] [--ref-cfg5]

Config 4 (10M uniform triangles, density 1 -> 64: 24 -> 30 key bits, up to 640M cells,
the four-pass radix plan) is built by the UNMODIFIED reference (oracle/_ref, C lane) AND by
the C oracle; the two must agree bit for bit, which pins the oracle at this scale. Config 5
(100M triangles: cfg5 uniform density 5, cfg5a arch density 4) is built by the C oracle --
the reference needs ~40 GB of int64 temporaries there; --ref-cfg5 runs it too where RAM
allows. Results are merged into tests/golden/hashes_big.json (sha256 of G and O, NO, dims,
which builder produced them and how long it took).
"""

import argparse
import hashlib
import json
import os
import sys
import time
import warnings

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]

import oracle  # noqa: E402  (the C restatement, pinned below)
from paper_2403_10647_b200 import scenes  # noqa: E402
from paper_2403_10647_b200.gridcore import spec_for_mesh  # noqa: E402

OUT = os.path.join(HERE, "hashes_big.json")


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def ref_build(mesh, density):
    sys.path.insert(0, os.path.join(ROOT, "oracle", "_ref"))
    import pargrid
    from pargrid import kernels as rk
    from pargrid.geometry import TriangleMesh as RMesh
    rk.set_backend("c")
    rmesh = RMesh(mesh.vertices, mesh.triangles)
    spec = pargrid.spec_for_mesh(rmesh, density=density)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        g, rep = pargrid.build_parallel(rmesh, spec)
    return np.asarray(g.G, np.uint32), np.asarray(g.O, np.uint32), tuple(spec.dims)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="")
    ap.add_argument("--ref-cfg5", action="store_true")
    a = ap.parse_args()
    names = [f"cfg4_d{d}" for d in (1, 8, 64)] + ["cfg5", "cfg5a"]
    if a.only:
        names = [n for n in names if n in a.only.split(",")]
    out = json.load(open(OUT)) if os.path.exists(OUT) else {"scenes": {}}
    mesh_key, mesh = None, None
    for name in names:
        kind, n, seed, density = scenes.CONFIGS[name]
        if mesh_key != (kind, n, seed):
            mesh = None
            t0 = time.perf_counter()
            mesh = scenes.gen_scene_large(kind, n, seed, density) if n > 20_000_000 else \
                scenes.gen_scene(kind, n, seed, density)
            mesh_key = (kind, n, seed)
            print(name, "scene", f"{time.perf_counter() - t0:.1f}s", flush=True)
        spec = spec_for_mesh(mesh, density=density)
        t0 = time.perf_counter()
        G, O = oracle.build_parallel(mesh.vertices, mesh.triangles, spec)
        t_orc = time.perf_counter() - t0
        rec = {"recipe": {"kind": kind, "n": n, "seed": seed, "density": density},
               "dims": list(spec.dims), "ncells": int(spec.ncells),
               "key_bits": int(spec.ncells - 1).bit_length(), "no": int(len(O)),
               "G_sha256": sha(G), "O_sha256": sha(O), "oracle_seconds": round(t_orc, 1)}
        del G
        if n <= 20_000_000 or a.ref_cfg5:
            t0 = time.perf_counter()
            Gr, Or, dims = ref_build(mesh, density)
            rec["reference_seconds"] = round(time.perf_counter() - t0, 1)
            assert dims == tuple(spec.dims), (dims, spec.dims)
            assert sha(Gr) == rec["G_sha256"] and sha(Or) == rec["O_sha256"], f"{name}: oracle != reference"
            rec["source"] = "reference (oracle/_ref, C lane) == C oracle"
            del Gr, Or
        else:
            rec["source"] = "C oracle (pinned to the reference on cfg4 and every smaller golden)"
        out["scenes"][name] = rec
        print(name, json.dumps(rec), flush=True)
        with open(OUT, "w") as fh:
            json.dump(out, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
