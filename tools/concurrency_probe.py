"""Two independent cfg3 builds in flight on two streams (two workspaces, captured graphs):
throughput vs one stream. Device-resident inputs; CUDA events; parity checked."""
import hashlib, json, os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT]
from paper_2403_10647_b200 import _native, scenes

mesh, spec = scenes.config_scene("cfg3")
n, nv = len(mesh.triangles), len(mesh.vertices)
Vd = torch.from_numpy(mesh.vertices.copy()).cuda()
Td = torch.from_numpy(mesh.triangles.copy()).cuda()
pg = _native.PgSpec.from_spec(spec)
b0 = _native.Builder(0)
no = b0.count(Vd, nv, Td, n, spec, 0, torch.cuda.current_stream().cuda_stream)
slots = []
for i in range(2):
    b = _native.Builder(0)
    G = torch.empty(spec.ncells + 1, dtype=torch.int32, device="cuda")
    O = torch.empty(no, dtype=torch.int32, device="cuda")
    s = torch.cuda.Stream()
    slots.append((b, G, O, s))
for b, G, O, s in slots:
    for _ in range(3):
        b.build_async(Vd, nv, Td, n, spec, G, O, no, s.cuda_stream, pg)
    b.build_wait()
torch.cuda.synchronize()
def run(k, nstreams):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for i in range(k):
        b, G, O, s = slots[i % nstreams]
        s.wait_event(e0) if i < nstreams else None
        b.build_async(Vd, nv, Td, n, spec, G, O, no, s.cuda_stream, pg)
    for b, G, O, s in slots[:nstreams]:
        torch.cuda.current_stream().wait_stream(s)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / k
one = run(40, 1)
two = run(40, 2)
hs = {hashlib.sha256(G.cpu().numpy().tobytes()).hexdigest() for b, G, O, s in slots}
print(json.dumps({"one_stream_ms": round(one, 4), "two_streams_ms_per_build": round(two, 4),
                  "gain": round(one / two, 3), "identical_outputs": len(hs) == 1}))
