"""BASELINE.json configs 4 and 5 on the GPU against committed golden hashes
(tests/golden/make_golden_big.py: the reference itself for config 4 -- 10M uniform triangles
at grid densities 1, 8, 64, i.e. 24, 27 and 30 key bits with up to 640M cells and the
four-pass radix plan -- and the C oracle, pinned to it, for the 100M-triangle config 5).
Both device entry points: the host-counted pg_count + pg_finish and the sync-free
pg_build_async CUDA-graph build (in-kernel digit-total clearing, top-digit narrowing of K4's
bound searches)."""

import json
import os

import numpy as np
import pytest
import torch

from paper_2403_10647_b200 import _native, scenes
from util import sha

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

HB = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "hashes_big.json")
with open(HB) as fh:
    BIG = json.load(fh)["scenes"]
KEYS = [k for k in ("cfg4_d1", "cfg4_d8", "cfg4_d64", "cfg5") if k in BIG]

_cache = {}


def _mesh(kind, n, seed, density):
    key = (kind, n, seed)
    if key not in _cache:
        _cache.clear()
        torch.cuda.empty_cache()
        m = scenes.gen_scene_large(kind, n, seed, density) if n > 20_000_000 else scenes.gen_scene(kind, n, seed, density)
        _cache[key] = (m, torch.from_numpy(m.vertices).cuda(), torch.from_numpy(m.triangles).cuda())
    return _cache[key]


@pytest.mark.parametrize("key", KEYS)
def test_big_config_hashes(key):
    from paper_2403_10647_b200.gridcore import spec_for_mesh
    h = BIG[key]
    r = h["recipe"]
    mesh, Vd, Td = _mesh(r["kind"], r["n"], r["seed"], r["density"])
    spec = spec_for_mesh(mesh, density=r["density"])
    assert list(spec.dims) == h["dims"] and int(spec.ncells - 1).bit_length() == h["key_bits"]
    b = _native.Builder(0)
    st = torch.cuda.current_stream().cuda_stream
    no = b.count(Vd, len(mesh.vertices), Td, len(mesh.triangles), spec, 0, st)
    assert no == h["no"]
    Gd = torch.empty(spec.ncells + 1, dtype=torch.int32, device="cuda")
    Od = torch.empty(no, dtype=torch.int32, device="cuda")
    b.finish(Gd, Od, 0, st, timed=False)
    torch.cuda.synchronize()
    assert sha(Gd.cpu().numpy().view(np.uint32)) == h["G_sha256"], "G (pg_finish)"
    assert sha(Od.cpu().numpy().view(np.uint32)) == h["O_sha256"], "O (pg_finish)"
    for _ in range(2):          # eager + capture, then a replay
        Gd.fill_(-1)
        Od.fill_(-1)
        b.build_async(Vd, len(mesh.vertices), Td, len(mesh.triangles), spec, Gd, Od, no, st)
        assert b.build_wait() == no
        assert sha(Gd.cpu().numpy().view(np.uint32)) == h["G_sha256"], "G (graph)"
        assert sha(Od.cpu().numpy().view(np.uint32)) == h["O_sha256"], "O (graph)"
    b.close()
    del Gd, Od
