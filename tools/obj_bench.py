"""OBJ ingestion throughput on one B200.

    python tools/obj_bench.py [--config cfg2] [--steps 5]

Writes the config scene with save_obj (Python repr floats, as the reference's save_obj),
then times load_obj on the device: bytes already in pinned host memory (H2D inside the
timing) and bytes already on the device; parity: vertices/triangles bit-identical to the
scene arrays the file was written from. The reference's Python load_obj is timed on a
prefix of the file (oracle/_ref when present)."""
import argparse, json, os, sys, tempfile, time
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
from paper_2403_10647_b200 import _native, obj, scenes

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg2")
ap.add_argument("--steps", type=int, default=5)
ap.add_argument("--cpu-lines", type=int, default=200_000)
a = ap.parse_args()
kind, n, seed, dens = scenes.CONFIGS[a.config]
mesh = scenes.gen_scene(kind, n, seed, dens)
with tempfile.TemporaryDirectory() as d:
    path = os.path.join(d, "scene.obj")
    obj.save_obj(mesh, path)
    data = open(path, "rb").read()
buf = np.frombuffer(data, np.uint8).copy()
_native.host_register(buf)
b = _native.thread_builder()
m = obj.load_obj_bytes(buf)
ok = np.array_equal(m.vertices.view(np.uint64), mesh.vertices.view(np.uint64)) and np.array_equal(m.triangles, mesh.triangles)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(a.steps):
    rc, out = b.load_obj(buf, len(buf), flags=_native.PG_HOST_INPUT)
host_ms = (time.perf_counter() - t0) * 1e3 / a.steps
dbuf = torch.from_numpy(buf).cuda()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(a.steps):
    rc, out = b.load_obj(dbuf, len(buf), flags=0)
dev_ms = (time.perf_counter() - t0) * 1e3 / a.steps
_native.host_unregister(buf)
# reference loader on a prefix (whole lines)
cut = 0
for _ in range(a.cpu_lines):
    cut = data.index(b"\n", cut) + 1 if b"\n" in data[cut:cut + 4096] else cut
prefix = data[:cut]
import oracle
ref = oracle.reference_module()
cpu = None
if ref is not None:
    from pargrid.geometry import load_obj as ref_load
    with tempfile.TemporaryDirectory() as d:
        p = os.path.join(d, "prefix.obj")
        open(p, "wb").write(prefix)
        t0 = time.perf_counter()
        try:
            ref_load(p)
        except Exception:
            pass
        cpu_s = time.perf_counter() - t0
    cpu = {"kind": "reference (pargrid.geometry.load_obj)", "cores": 1, "bytes": len(prefix),
           "mb_per_s": round(len(prefix) / cpu_s / 1e6, 2)}
print(json.dumps({"config": a.config, "bytes": len(data), "vertices": len(mesh.vertices), "triangles": n,
                  "host_input_ms": round(host_ms, 3), "host_input_gb_per_s": round(len(data) / host_ms / 1e6, 2),
                  "device_input_ms": round(dev_ms, 3), "device_input_gb_per_s": round(len(data) / dev_ms / 1e6, 2),
                  "launches": b.launches(), "parity": "bit-exact" if ok else "MISMATCH", "cpu": cpu}), flush=True)
