"""Ray casting over a built grid on one B200.

    python tools/ray_bench.py [--configs cfg2,cfg3] [--rays 4000000] [--steps 5] [--cpu-rays 20000]

Per config: grid built on the device (Alg. 1), mesh prepared once, then
  device  : K casts of R device-resident rays (CUDA events on the launching stream)
  e2e     : RayCaster.cast with host rays (H2D rays + D2H ids/ts inside the timing)
  cpu     : the reference's compiled lane (oracle/_ref, one core) on the first --cpu-rays rays
            (falls back to the C oracle port when oracle/_ref is absent)
Parity: ids/ts of the sample bit-exact against the CPU result."""
import argparse, json, os, sys, time
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
from paper_2403_10647_b200 import _native, scenes, traverse
from paper_2403_10647_b200.gridcore import spec_for_mesh

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="cfg2,cfg3")
ap.add_argument("--rays", type=int, default=4_000_000)
ap.add_argument("--steps", type=int, default=5)
ap.add_argument("--cpu-rays", type=int, default=20000)
a = ap.parse_args()
for name in a.configs.split(","):
    kind, n, seed, dens = scenes.CONFIGS[name]
    mesh = scenes.gen_scene(kind, n, seed, dens)
    spec = spec_for_mesh(mesh, density=dens)
    b = _native.Builder(0)
    Vd = torch.from_numpy(mesh.vertices.copy()).cuda()
    Td = torch.from_numpy(mesh.triangles.copy()).cuda()
    st = torch.cuda.current_stream().cuda_stream
    no = b.count(Vd, len(mesh.vertices), Td, n, spec, 0, st)
    Gd = torch.empty(spec.ncells + 1, dtype=torch.int32, device="cuda")
    Od = torch.empty(max(no, 1), dtype=torch.int32, device="cuda")
    b.finish(Gd, Od, 0, st, timed=False)
    caster = traverse.RayCaster((spec, Gd, Od[:no]), (Vd, Td))
    o, d, t = traverse.make_rays(spec.bounds, a.rays, 77)
    od, dd, td = (torch.from_numpy(x).cuda() for x in (o, d, t))
    out = caster.cast(od, dd, td)
    for _ in range(2):
        caster.cast(od, dd, td, out=out, check=False)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.steps):
        caster.cast(od, dd, td, out=out, check=False)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.steps
    ids = out[0].cpu().numpy()
    ts = out[1].cpu().numpy()
    for x in (o, d, t):
        _native.host_register(x)
    caster.cast(o, d, t)
    t0 = time.perf_counter()
    for _ in range(a.steps):
        hi, ht = caster.cast(o, d, t)
    e2e_ms = (time.perf_counter() - t0) * 1e3 / a.steps
    for x in (o, d, t):
        _native.host_unregister(x)
    assert np.array_equal(hi, ids) and np.array_equal(ht.view(np.uint64), ts.view(np.uint64))
    k = min(a.cpu_rays, a.rays)
    import oracle
    ref = oracle.reference_module()
    G = Gd.cpu().numpy().view(np.uint32)
    O = Od[:no].cpu().numpy().view(np.uint32)
    t0 = time.perf_counter()
    if ref is not None:
        from pargrid.kernels import _ckernels
        cids, cts = _ckernels.dda_cast(G, O, mesh.vertices, mesh.triangles, spec.bounds.lo, spec.bounds.hi,
                                       spec.cell_size, spec.dims, o[:k], d[:k], t[:k])
        kind_cpu = "reference"
    else:
        cids, cts = oracle.dda_cast(G, O, mesh.vertices, mesh.triangles, spec, o[:k], d[:k], t[:k])
        kind_cpu = "port"
    cpu_s = time.perf_counter() - t0
    ok = np.array_equal(cids, ids[:k]) and np.array_equal(cts.view(np.uint64), ts[:k].view(np.uint64))
    print(json.dumps({"config": name, "triangles": n, "dims": list(spec.dims), "no": no, "rays": a.rays,
                      "hits": int((ids >= 0).sum()), "device_ms": round(ms, 3),
                      "mrays_per_s": round(a.rays / ms / 1e3, 1), "e2e_ms": round(e2e_ms, 3),
                      "e2e_mrays_per_s": round(a.rays / e2e_ms / 1e3, 1),
                      "cpu": {"kind": kind_cpu, "cores": 1, "rays": k, "mrays_per_s": round(k / cpu_s / 1e6, 4)},
                      "parity_sample": "bit-exact" if ok else "MISMATCH"}), flush=True)
    del caster, Gd, Od, Vd, Td, od, dd, td, out
    torch.cuda.empty_cache()
