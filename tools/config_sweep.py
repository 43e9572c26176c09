"""Throughput + parity over BASELINE.json's configs on one GPU (configs 1-4).

    python tools/config_sweep.py [--oracle] [--steps 10]

cfg1/cfg2/cfg3 are checked against the reference's golden hashes; the density sweep
(config 4: 10M uniform triangles, density 1..64) against the C oracle when --oracle is
given (the oracle is test infrastructure; it only checks, it is never timed here)."""
import argparse, hashlib, json, os, sys, time
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
from paper_2403_10647_b200 import _native, scenes
from paper_2403_10647_b200.gridcore import spec_for_mesh

ap = argparse.ArgumentParser()
ap.add_argument("--oracle", action="store_true")
ap.add_argument("--steps", type=int, default=10)
ap.add_argument("--only", default="")
a = ap.parse_args()
hashes = json.load(open(os.path.join(ROOT, "tests", "golden", "hashes.json")))["scenes"]
big = json.load(open(os.path.join(ROOT, "tests", "golden", "hashes_big.json")))["scenes"]
hashes.update({{"cfg5": "cfg5_1gpu", "cfg5a": "cfg5a_1gpu"}.get(k, k): v for k, v in big.items()})
runs = [("cfg1", "uniform", 100_000, 5.0), ("cfg2", "lognormal", 1_000_000, 5.0), ("cfg3", "arch", 10_000_000, 4.0),
        ("cfg3u", "uniform", 10_000_000, 5.0)]
runs += [(f"cfg4_d{d}", "uniform", 10_000_000, float(d)) for d in (1, 2, 4, 8, 16, 32, 64)]
runs += [("cfg5_1gpu", "uniform", 100_000_000, 5.0),   # config 5's scenes on one B200
         ("cfg5a_1gpu", "arch", 100_000_000, 4.0)]
if a.only:
    runs = [r for r in runs if r[0] in a.only.split(",")]
b = _native.Builder(0)
sp = torch.cuda.current_stream().cuda_stream
cache = {}
for name, kind, n, dens in runs:
    key = (kind, n)
    if key not in cache:
        cache.clear()
        m = (scenes.gen_scene_large(kind, n, 7, dens) if n > 20_000_000 else
             scenes.gen_scene(kind, n, 7, dens if kind in ("lognormal", "arch") else 5.0))
        cache[key] = (m, torch.from_numpy(m.vertices.copy()).cuda(), torch.from_numpy(m.triangles.copy()).cuda())
    mesh, Vd, Td = cache[key]
    spec = spec_for_mesh(mesh, density=dens)
    no = b.count(Vd, len(mesh.vertices), Td, n, spec, 0, sp)
    Gd = torch.empty(spec.ncells + 1, dtype=torch.int32, device="cuda")
    Od = torch.empty(max(no, 1), dtype=torch.int32, device="cuda")
    pg = _native.PgSpec.from_spec(spec)
    for _ in range(3):
        b.build_async(Vd, len(mesh.vertices), Td, n, spec, Gd, Od, no, sp, pg)
    assert b.build_wait() == no
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.steps):
        b.build_async(Vd, len(mesh.vertices), Td, n, spec, Gd, Od, no, sp, pg)
    e1.record()
    torch.cuda.synchronize()
    assert b.build_wait() == no
    ms = e0.elapsed_time(e1) / a.steps
    G = Gd.cpu().numpy().view(np.uint32)
    O = Od[:no].cpu().numpy().view(np.uint32)
    parity = "unchecked"
    h = hashes.get(name)
    if h:
        ok = hashlib.sha256(G.tobytes()).hexdigest() == h["G_sha256"] and hashlib.sha256(O.tobytes()).hexdigest() == h["O_sha256"]
        parity = "golden-sha256 " + ("OK" if ok else "MISMATCH")
    elif a.oracle:
        import oracle
        Gr, Or = oracle.build_parallel(mesh.vertices, mesh.triangles, spec)
        parity = "oracle " + ("OK" if np.array_equal(G, Gr) and np.array_equal(O, Or) else "MISMATCH")
    B = 84 * n + 4 * (spec.ncells + 1) + 4 * no
    print(json.dumps({"config": name, "scene": kind, "triangles": n, "density": dens, "dims": list(spec.dims),
                      "ncells": spec.ncells, "key_bits": int(spec.ncells - 1).bit_length(), "no": no,
                      "ms": round(ms, 4), "builds_per_s": round(1e3 / ms, 2), "mpairs_per_s": round(no / ms / 1e3, 1),
                      "hbm_gbs": round(B / ms / 1e6, 1), "parity": parity}), flush=True)
