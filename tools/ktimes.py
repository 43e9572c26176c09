"""Warm per-kernel device times of one config build (PGRID_KTIMES=1 event brackets).

    PGRID_KTIMES=1 python tools/ktimes.py [--config cfg3] [--builds 10]
Reports the per-kernel median over the builds (device time between launch completions)."""
import argparse, collections, os, sys
import numpy as np
import torch
os.environ.setdefault("PGRID_KTIMES", "1")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT]
from paper_2403_10647_b200 import _native, scenes

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg3")
ap.add_argument("--builds", type=int, default=10)
a = ap.parse_args()
mesh, spec = scenes.config_scene(a.config)
b = _native.Builder(0)
Vd = torch.from_numpy(mesh.vertices.copy()).cuda()
Td = torch.from_numpy(mesh.triangles.copy()).cuda()
st = torch.cuda.current_stream().cuda_stream
no = b.count(Vd, len(mesh.vertices), Td, len(mesh.triangles), spec, 0, st)
Gd = torch.empty(spec.ncells + 1, dtype=torch.int32, device="cuda")
Od = torch.empty(max(no, 1), dtype=torch.int32, device="cuda")
runs = []
for i in range(a.builds + 2):
    b.count(Vd, len(mesh.vertices), Td, len(mesh.triangles), spec, 0, st)
    b.finish(Gd, Od, 0, st, timed=False)
    torch.cuda.synchronize()
    if i >= 2:
        runs.append(_native.kernel_times())
per = collections.defaultdict(list)
order = []
for r in runs:
    seen = collections.Counter()
    for name, us in r:
        key = f"{name}#{seen[name]}"
        seen[name] += 1
        if key not in per:
            order.append(key)
        per[key].append(us)
tot = 0.0
for k in order:
    m = float(np.median(per[k]))
    if not k.startswith("(host gap)"):
        tot += m
    print(f"{k:34s} {m:9.2f} us")
print(f"{'total (device)':34s} {tot:9.2f} us   NO={no}")
