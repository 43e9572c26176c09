"""The MSD-first finish (radix passes over the top key bits, then k_bucket_sort: per-cell counts
-> G, and a stable warp-per-bucket sort of the low bits into O) against the oracle, for every
bucket width the planner can pick (PGRID_LOCAL_ITEMS moves it from 1-cell buckets to 2^11) and
against the classic LSD + K4 finish (PGRID_LOCAL=0). The environment is read once per process,
so each setting runs in a subprocess."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys, numpy as np
sys.path[:0] = [%(root)r, %(root)r + '/oracle']
import oracle
from paper_2403_10647_b200 import builders, gen_scene, spec_for_mesh, _native
import torch
cases = [("uniform", 3000, 1, None), ("walls", 5000, 2, (41, 37, 29)), ("lognormal", 20000, 3, None),
         ("uniform", 2000, 4, (1024, 1024, 512)), ("arch", 30000, 5, None), ("uniform", 4000, 6, (3, 5, 7)),
         ("walls", 2000, 7, (1, 1, 2)), ("uniform", 50000, 8, (300, 1, 1))]
for kind, n, seed, dims in cases:
    mesh = gen_scene(kind, n, seed)
    spec = spec_for_mesh(mesh, dims=dims)
    Gr, Or = oracle.build_parallel(mesh.vertices, mesh.triangles, spec)
    g, _ = builders.build_parallel(mesh, spec)
    assert np.array_equal(g.G, Gr) and np.array_equal(g.O, Or), (kind, n, seed, dims)
    # the sync-free graph build and the deferred pipeline take the same finish
    Vd = torch.from_numpy(mesh.vertices.copy()).cuda(); Td = torch.from_numpy(mesh.triangles.copy()).cuda()
    Gd = torch.empty(spec.ncells + 1, dtype=torch.int32, device="cuda")
    Od = torch.empty(len(Or) + 64, dtype=torch.int32, device="cuda")
    b = _native.Builder(0)
    for _ in range(2):
        b.build_async(Vd, len(mesh.vertices), Td, len(mesh.triangles), spec, Gd, Od, len(Or) + 64)
        no = b.build_wait()
        assert no == len(Or)
        assert np.array_equal(Gd.cpu().numpy().view(np.uint32), Gr)
        assert np.array_equal(Od.cpu().numpy().view(np.uint32)[:no], Or)
    b.close()
items = [(gen_scene("uniform", 2500 + 100 * s, s), None) for s in range(3)]
items = [(m, spec_for_mesh(m)) for m, _ in items]
for (m, sp), (g, _) in zip(items, builders.build_many(items)):
    Gr, Or = oracle.build_parallel(m.vertices, m.triangles, sp)
    assert np.array_equal(g.G, Gr) and np.array_equal(g.O, Or)
print("ok")
"""


@pytest.mark.timeout(900)
@pytest.mark.parametrize("env", [{"PGRID_LOCAL": "0"}, {"PGRID_LOCAL_ITEMS": "1"}, {"PGRID_LOCAL_ITEMS": "16"},
                                 {}, {"PGRID_LOCAL_ITEMS": "4096"}, {"PGRID_LOCAL_ITEMS": "100000000"}],
                         ids=["classic", "items1", "items16", "default", "items4096", "widest"])
def test_bucket_finish_matches_oracle(env):
    e = dict(os.environ, **env)
    r = subprocess.run([sys.executable, "-c", SCRIPT % {"root": ROOT}], env=e, capture_output=True, text=True,
                       timeout=880)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]
