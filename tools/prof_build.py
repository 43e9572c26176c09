"""Profiling driver: N builds of a config with device-resident inputs (for ncu)."""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_10647_b200 import _native, scenes  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg3")
ap.add_argument("--builds", type=int, default=2)
a = ap.parse_args()
mesh, spec = scenes.config_scene(a.config)
Vd = torch.from_numpy(mesh.vertices.copy()).cuda()
Td = torch.from_numpy(mesh.triangles.copy()).cuda()
b = _native.Builder(0)
sp = torch.cuda.current_stream().cuda_stream
no = b.count(Vd, len(mesh.vertices), Td, len(mesh.triangles), spec, 0, sp)
Gd = torch.empty(spec.ncells + 1, dtype=torch.int32, device="cuda")
Od = torch.empty(max(no, 1), dtype=torch.int32, device="cuda")
b.finish(Gd, Od, 0, sp, timed=False)
for _ in range(a.builds):
    b.count(Vd, len(mesh.vertices), Td, len(mesh.triangles), spec, 0, sp)
    b.finish(Gd, Od, 0, sp, timed=False)
torch.cuda.synchronize()
print("launches per build", b.launches(), "NO", no)
