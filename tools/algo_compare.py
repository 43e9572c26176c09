"""Alg. 1 vs the paper's comparison builders on one B200.

    python tools/algo_compare.py [--steps 10] [--only cfg1,cfg2]

Device-resident inputs; each step = count (K1) + finish, synchronous path, timed with CUDA
events on the launching stream (the same for all three algorithms). Every algorithm's G/O
is checked against the parallel builder's output (which the golden tests pin)."""
import argparse, json, os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT]
from paper_2403_10647_b200 import _native, scenes
from paper_2403_10647_b200.gridcore import spec_for_mesh

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=10)
ap.add_argument("--only", default="")
a = ap.parse_args()
runs = [("cfg1", "uniform", 100_000, 5.0), ("skewed1m", "skewed", 1_000_000, 5.0),
        ("walls100k", "walls", 100_000, 5.0), ("cfg2", "lognormal", 1_000_000, 5.0),
        ("cfg3", "arch", 10_000_000, 4.0), ("cfg3u", "uniform", 10_000_000, 5.0)]
if a.only:
    runs = [r for r in runs if r[0] in a.only.split(",")]
b = _native.Builder(0)
sp = torch.cuda.current_stream().cuda_stream
for name, kind, n, dens in runs:
    mesh = scenes.gen_scene(kind, n, 7, dens)
    spec = spec_for_mesh(mesh, density=dens)
    Vd = torch.from_numpy(mesh.vertices.copy()).cuda()
    Td = torch.from_numpy(mesh.triangles.copy()).cuda()
    nv = len(mesh.vertices)
    no = b.count(Vd, nv, Td, n, spec, 0, sp)
    Gd = torch.empty(spec.ncells + 1, dtype=torch.int32, device="cuda")
    Od = torch.empty(max(no, 1), dtype=torch.int32, device="cuda")
    row = {"config": name, "scene": kind, "triangles": n, "ncells": spec.ncells, "no": no}
    ref = None
    for algo in ("parallel", "sorted", "compact"):
        def step():
            b.count(Vd, nv, Td, n, spec, 0, sp)
            if algo == "parallel":
                return b.finish(Gd, Od, 0, sp, timed=True), None
            return b.finish_baseline(1 if algo == "sorted" else 2, Gd, Od, 0, sp)
        for _ in range(3):
            ph, mw = step()
        out = (Gd.cpu().numpy().copy(), Od[:no].cpu().numpy().copy())
        if ref is None:
            ref = out
        ok = np.array_equal(out[0], ref[0]) and np.array_equal(out[1], ref[1])
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(a.steps):
            ph, mw = step()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.steps
        row[algo] = {"ms": round(ms, 4), "phases_ms": [round(x, 4) for x in ph], "same_as_parallel": ok}
        if mw is not None:
            row[algo]["max_task_work"] = mw
    row["sorted_over_parallel"] = round(row["sorted"]["ms"] / row["parallel"]["ms"], 2)
    row["compact_over_parallel"] = round(row["compact"]["ms"] / row["parallel"]["ms"], 2)
    print(json.dumps(row), flush=True)
