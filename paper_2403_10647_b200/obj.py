"""OBJ ingestion on the GPU, mirror of pargrid.geometry.load_obj.

    mesh = load_obj(path)                 # geometry.py:84-112: TriangleMesh on the host
    V, T = load_obj(path, on_device=True) # torch tensors resident on the GPU (no host copy)

The file's bytes go to the device once; line splitting, tokenising, Python-exact float /
int parsing, negative-index resolution and fan triangulation run in CUDA
(csrc/pgrid_obj.cuh, C ABI pg_load_obj / pg_obj_fetch). On a malformed file the device
reports the first offending line; its message is then produced by restating the
reference's per-line checks on that one line (geometry.py:65-81, 91-109), so the
ObjParseError text and line number are the reference's own. Lines carrying non-ASCII
characters in a v/f statement (or non-ASCII whitespace) are rejected with an
ObjParseError naming the limitation: the device tokeniser implements Python's ASCII
semantics only.
"""

import numpy as np

from . import _native
from .errors import ObjParseError
from .gridcore import TriangleMesh


def _parse_face_index(token, nverts, line_number):
    """geometry.py:65-81 (used only to word the error of the line the device flagged)."""
    first = token.split("/")[0]
    try:
        idx = int(first)
    except ValueError:
        raise ObjParseError(f"bad face index {token!r}", line_number) from None
    if idx > 0:
        idx -= 1
    elif idx < 0:
        idx += nverts
    else:
        raise ObjParseError("face index 0 is not valid", line_number)
    if not 0 <= idx < nverts:
        raise ObjParseError(f"face index {first} out of range", line_number)
    return idx


def _raise_line_error(raw, lineno, nverts):
    """Re-run the reference's checks (geometry.py:91-109) on the flagged line."""
    line = raw.decode("utf-8", errors="replace").split("#", 1)[0].strip()
    parts = line.split()
    if parts and parts[0] == "v":
        if len(parts) < 4:
            raise ObjParseError("vertex needs 3 coordinates", lineno)
        try:
            float(parts[1]), float(parts[2]), float(parts[3])
        except ValueError:
            raise ObjParseError("bad vertex coordinate", lineno) from None
    elif parts and parts[0] == "f":
        if len(parts) < 4:
            raise ObjParseError("face needs at least 3 vertices", lineno)
        for tok in parts[1:]:
            _parse_face_index(tok, nverts, lineno)
    raise ObjParseError("non-ASCII characters in a v/f statement are not supported by the device OBJ loader",
                        lineno)


def load_obj_bytes(data, device=0, on_device=False):
    """Parse OBJ text held in memory (bytes / bytearray / uint8 array)."""
    buf = np.frombuffer(memoryview(data), dtype=np.uint8) if not isinstance(data, np.ndarray) else data
    buf = np.ascontiguousarray(buf, dtype=np.uint8)
    b = _native.thread_builder(device)
    rc, out = b.load_obj(buf, len(buf), flags=_native.PG_HOST_INPUT)
    if rc == _native.PG_PARSE_ERROR:
        lineno, nverts, lb, le = out[2], out[3], out[4], out[5]
        _raise_line_error(bytes(buf[lb:le]), lineno, nverts)
    nv, nt = out[0], out[1]
    if on_device:
        import torch
        dev = torch.device("cuda", device)
        V = torch.empty((nv, 3), dtype=torch.float64, device=dev)
        T = torch.empty((nt, 3), dtype=torch.int32, device=dev)
        b.obj_fetch(V, T, flags=0, stream=torch.cuda.current_stream(dev).cuda_stream)
        return V, T
    V = np.empty((nv, 3), np.float64)
    T = np.empty((nt, 3), np.int32)
    b.obj_fetch(V, T, flags=_native.PG_HOST_OUTPUT)
    return TriangleMesh(V, T)


def load_obj(path, device=0, on_device=False):
    """geometry.py:84-112 on the GPU: TriangleMesh (or device (V, T) with on_device=True)."""
    with open(path, "rb") as fh:
        data = fh.read()
    return load_obj_bytes(data, device=device, on_device=on_device)


def save_obj(mesh, path):
    """geometry.py:115-121 (host text writer, v and f lines)."""
    with open(path, "w", encoding="utf-8") as fh:
        for v in mesh.vertices:
            fh.write(f"v {float(v[0])!r} {float(v[1])!r} {float(v[2])!r}\n")
        for t in mesh.triangles:
            fh.write(f"f {t[0] + 1} {t[1] + 1} {t[2] + 1}\n")
