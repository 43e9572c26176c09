"""OBJ ingestion. CPU: the host pieces (save_obj mirror, the error wording
for the line the device flags) against the reference's fixtures. GPU: the device loader
against every golden case (tests/golden/make_golden_obj.py), bit for bit."""

import hashlib
import json
import os

import numpy as np
import pytest

from paper_2403_10647_b200 import obj, scenes
from paper_2403_10647_b200.errors import ObjParseError

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def objgold():
    with np.load(os.path.join(GOLDEN, "obj.npz")) as z:
        arrays = {k: z[k] for k in z.files}
    with open(os.path.join(GOLDEN, "obj.json")) as fh:
        return arrays, json.load(fh)


def _lines(data):
    return data.decode("utf-8", errors="replace").replace("\r\n", "\n").replace("\r", "\n").split("\n")


def test_error_wording_matches_reference(objgold):
    arrays, meta = objgold
    for name, m in meta["cases"].items():
        if m["ok"]:
            continue
        data = arrays[f"{name}/bytes"].tobytes()
        lines = _lines(data)
        ln = m["line"]
        nverts = sum(1 for t in lines[:ln - 1] if t.split("#", 1)[0].split()[:1] == ["v"])
        with pytest.raises(ObjParseError) as e:
            obj._raise_line_error(lines[ln - 1].encode(), ln, nverts)
        assert str(e.value) == m["message"] and e.value.line_number == ln, name


def test_save_obj_mirror_bytes(objgold, tmp_path):
    big = objgold[1]["cfg1_save_obj"]
    mesh = scenes.gen_scene("uniform", big["recipe"]["n"], big["recipe"]["seed"])
    p = tmp_path / "cfg1.obj"
    obj.save_obj(mesh, p)
    assert hashlib.sha256(p.read_bytes()).hexdigest() == big["bytes_sha256"]


@pytest.mark.gpu
def test_device_loader_golden_cases(objgold):
    arrays, meta = objgold
    for name, m in meta["cases"].items():
        data = arrays[f"{name}/bytes"].tobytes()
        if m["ok"]:
            mesh = obj.load_obj_bytes(data)
            assert np.array_equal(mesh.vertices.view(np.uint64), arrays[f"{name}/V"].view(np.uint64)), name
            assert np.array_equal(mesh.triangles, arrays[f"{name}/T"]), name
        else:
            with pytest.raises(ObjParseError) as e:
                obj.load_obj_bytes(data)
            assert str(e.value) == m["message"] and e.value.line_number == m["line"], name


@pytest.mark.gpu
def test_device_loader_cfg1_file_and_device_output(objgold, tmp_path):
    import torch
    big = objgold[1]["cfg1_save_obj"]
    mesh = scenes.gen_scene("uniform", big["recipe"]["n"], big["recipe"]["seed"])
    p = tmp_path / "cfg1.obj"
    obj.save_obj(mesh, p)
    got = obj.load_obj(p)
    assert hashlib.sha256(got.vertices.tobytes()).hexdigest() == big["V_sha256"]
    assert hashlib.sha256(got.triangles.tobytes()).hexdigest() == big["T_sha256"]
    V, T = obj.load_obj(p, on_device=True)
    torch.cuda.synchronize()
    assert np.array_equal(V.cpu().numpy(), got.vertices) and np.array_equal(T.cpu().numpy(), got.triangles)


@pytest.mark.gpu
def test_unsupported_non_ascii_statement_is_loud():
    with pytest.raises(ObjParseError) as e:
        obj.load_obj_bytes("v 1 2 3\nv\u00a01 2 3\n".encode())
    assert e.value.line_number == 2 and "non-ASCII" in str(e.value)
