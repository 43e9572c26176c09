"""Small workloads for compute-sanitizer (tools/sanitize.sh): every device path of libpgrid
once, at sizes the sanitizers finish in minutes, each result checked against the C oracle.

    compute-sanitizer --tool memcheck python tools/sanitize_drive.py [--quick]

Paths: host-counted build (K1 -> K2 -> radix passes -> K4, 1-4 radix passes), the record=
stage dumps, the sync-free graph build (pg_build_async), the deferred BuildPipeline, the
plugin radix sort, the comparison builders, and the sharded orchestration emulated for 4
ranks with the NCCL-style copy exchange, the fused peer-store exchange and the fused
expansion + dispatch kernel."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]

import oracle  # noqa: E402  (checker only)
import torch  # noqa: E402
from paper_2403_10647_b200 import _native, builders, gen_scene, spec_for_mesh  # noqa: E402
from paper_2403_10647_b200 import distributed as D  # noqa: E402

quick = "--quick" in sys.argv


def check(tag, G, O, mesh, spec):
    Gr, Or = oracle.build_parallel(mesh.vertices, mesh.triangles, spec)
    assert np.array_equal(G, Gr) and np.array_equal(O, Or), tag
    print("ok", tag, flush=True)


scenes = [("uniform", 3000, 1, None), ("walls", 2000, 2, (41, 37, 29)), ("lognormal", 4000, 3, None),
          ("uniform", 2000, 4, (1024, 1024, 512))]       # 29 key bits: four radix passes
for kind, n, seed, dims in scenes:
    mesh = gen_scene(kind, n, seed)
    spec = spec_for_mesh(mesh, dims=dims)
    g, _ = builders.build_parallel(mesh, spec)
    check(f"build_parallel {kind} {spec.dims}", g.G, g.O, mesh, spec)
    rec = {}
    g, _ = builders.build_parallel(mesh, spec, record=rec)
    check(f"record {kind}", g.G, g.O, mesh, spec)
    if quick:
        break

mesh = gen_scene("walls", 3000, 5)
spec = spec_for_mesh(mesh, dims=(50, 40, 30))
# sync-free graph build: eager run, capture, one replay
Vd = torch.from_numpy(mesh.vertices.copy()).cuda()
Td = torch.from_numpy(mesh.triangles.copy()).cuda()
Gd = torch.empty(spec.ncells + 1, dtype=torch.int32, device="cuda")
Gr, Or = oracle.build_parallel(mesh.vertices, mesh.triangles, spec)
Od = torch.empty(len(Or) + 100, dtype=torch.int32, device="cuda")
b = _native.Builder(0)
for _ in range(2):
    b.build_async(Vd, len(mesh.vertices), Td, len(mesh.triangles), spec, Gd, Od, len(Or) + 100)
    no = b.build_wait()
    G = Gd.cpu().numpy().view(np.uint32)
    O = Od.cpu().numpy().view(np.uint32)[:no]
    check("graph build", G, O, mesh, spec)

# deferred pipeline: first build host-counted, then PG_DEFER
items = [(gen_scene("uniform", 2500, s), None) for s in range(3)]
items = [(m, spec_for_mesh(m)) for m, _ in items]
for (m, sp), (g, _) in zip(items, builders.build_many(items)):
    check("pipeline", g.G, g.O, m, sp)

# plugin radix sort (pg_radix_sort_pairs)
from paper_2403_10647_b200 import kernels  # noqa: E402
rng = np.random.default_rng(1)
for bits in (7, 19, 32):
    k = rng.integers(0, 1 << bits, 9000, dtype=np.uint64).astype(np.uint32)
    v = rng.integers(0, 1 << 32, 9000, dtype=np.uint64).astype(np.uint32)
    ks, vs = kernels.radix_sort_pairs(k, v, bits)
    o = np.argsort(k, kind="stable")
    assert np.array_equal(ks, k[o]) and np.array_equal(vs, v[o])
    print("ok radix", bits, flush=True)

# comparison builders
g, _ = builders.build_sorted(mesh, spec)
check("build_sorted", g.G, g.O, mesh, spec)
g, _ = builders.build_compact(mesh, spec)
check("build_compact", g.G, g.O, mesh, spec)

# sharded orchestration, 4 emulated ranks on this device
for exchange in ("copy", "p2p") + (("fused",) if _native.features() & _native.PG_FEATURE_FUSED_DISPATCH else ()):
    G, O = D.run_emulated(D.CudaOps, mesh.vertices, mesh.triangles, spec, 4, exchange=exchange)
    check(f"sharded x4 {exchange}", G, O, mesh, spec)
torch.cuda.synchronize()
print("sanitize drive done")
