"""CPU checks of the drop-in boundary: the C-ABI library loads and exports exactly what
include/pgrid.h declares; host-side mirrors match the reference (no device compute here)."""

import ctypes
import os
import re

import numpy as np
import pytest

from paper_2403_10647_b200 import _native, gridcore, scenes
from paper_2403_10647_b200.errors import GridError, InvariantError, SizeError

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "pgrid.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|void|const char \*)\s*(pg_\w+)\s*\(", src, re.M)))


def test_header_declares_every_binding():
    assert declared_symbols() == sorted(_native.EXPORTS)


def test_library_loads_and_exports_all_symbols():
    lib = ctypes.CDLL(_native.LIB_PATH)
    for name in declared_symbols():
        assert hasattr(lib, name), name
    # pg_last_error is callable without a device
    lib.pg_last_error.restype = ctypes.c_char_p
    assert lib.pg_last_error() is not None


def test_sass_is_sm100a():
    """The library carries sm_100a SASS (cuobjdump present in the image)."""
    import shutil
    import subprocess
    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(tool):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([tool, "--list-elf", _native.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_error_mapping(monkeypatch):
    class FakeLib:
        def pg_last_error(self):
            return b"boom"
    monkeypatch.setattr(_native, "_lib", FakeLib())
    with pytest.raises(SizeError):
        _native.check(_native.PG_SIZE_ERROR)
    with pytest.raises(InvariantError):
        _native.check(_native.PG_INVARIANT_ERROR)
    with pytest.raises(GridError):
        _native.check(_native.PG_CUDA_ERROR)
    _native.check(_native.PG_OK)


def test_pgspec_carries_exact_doubles():
    mesh = scenes.gen_scene("uniform", 1000, 3)
    spec = gridcore.spec_for_mesh(mesh)
    s = _native.PgSpec.from_spec(spec)
    for k in range(3):
        assert s.lo[k] == spec.bounds.lo[k] and s.hi[k] == spec.bounds.hi[k]
        assert s.cell[k] == spec.cell_size[k] and s.dims[k] == spec.dims[k]


def test_scenes_match_reference_generator():
    import oracle
    ref = oracle.reference_module()
    if ref is None:
        pytest.skip("oracle/_ref not built")
    for kind in ("uniform", "skewed", "walls"):
        for n, seed in ((1, 1), (777, 5), (30001, 7)):
            a = ref.gen_scene(kind, n, seed)
            b = scenes.gen_scene(kind, n, seed)
            assert np.array_equal(a.vertices, b.vertices) and np.array_equal(a.triangles, b.triangles)
            sa, sb = ref.spec_for_mesh(a), gridcore.spec_for_mesh(b)
            assert sa.dims == sb.dims
            assert np.array_equal(sa.cell_size, sb.cell_size)
            assert np.array_equal(sa.bounds.lo, sb.bounds.lo) and np.array_equal(sa.bounds.hi, sb.bounds.hi)


def test_gridcore_contract():
    with pytest.raises(SizeError):
        gridcore.GridSpec(gridcore.Aabb([0, 0, 0], [1, 1, 1]), (1 << 16, 1 << 16, 2))
    with pytest.raises(InvariantError):
        gridcore.GridSpec(gridcore.Aabb([0, 0, 0], [1, 1, 1]), (0, 1, 1))
    spec = gridcore.GridSpec(gridcore.Aabb([0, 0, 0], [1, 1, 1]), (2, 2, 2))
    with pytest.raises(InvariantError):
        gridcore.CompactGrid(spec, np.zeros(8, np.uint32), np.zeros(0, np.uint32))
    g = gridcore.CompactGrid(spec, np.zeros(9, np.uint32), np.zeros(0, np.uint32))
    assert g.no == 0 and not g.G.flags.writeable
    assert gridcore.key_bits_for(1) == 0 and gridcore.key_bits_for(493039) == 19
