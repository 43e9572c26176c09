"""Golden OBJ-ingestion fixtures from the UNMODIFIED reference loader.

    python tests/golden/make_golden_obj.py      # needs oracle/_ref (make -C oracle ref)

Writes tests/golden/obj.npz (committed): for every case the OBJ bytes and either the
reference's load_obj result (vertices as raw float64 bits, triangles) or its ObjParseError
(message, line number). Cases: the reference's own test texts, hand-written edge cases
(newline styles, comments, whitespace, slash forms, negative indices, polygons, Python
float/int syntax corners), decimal -> double hard cases (ties, subnormals, overflow, very
long digit strings from exact halfway points), a seeded format-fuzzed file, and error
cases. tests/golden/obj.json holds the sha256 of the reference's result for the save_obj
text of the cfg1 scene (regenerated on the GPU box from the recipe).
"""

import decimal
import hashlib
import json
import os
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle", "_ref"))

import pargrid  # noqa: E402  (the reference)
from pargrid.errors import ObjParseError  # noqa: E402
from pargrid.geometry import load_obj, save_obj  # noqa: E402

from paper_2403_10647_b200 import scenes  # noqa: E402


def ref_load(data):
    with tempfile.NamedTemporaryFile(suffix=".obj", delete=False) as fh:
        fh.write(data)
        path = fh.name
    try:
        m = load_obj(path)
        return ("ok", m.vertices.copy(), m.triangles.copy())
    except ObjParseError as e:
        return ("err", str(e), e.line_number)
    finally:
        os.unlink(path)


def halfway_strings(rng, count):
    """Exact decimal expansions of midpoints between adjacent doubles (and 1-ulp-of-decimal
    neighbours): the inputs where only an exact conversion rounds correctly."""
    decimal.getcontext().prec = 2000
    out = []
    for i in range(count):
        e = int(rng.integers(-1074, 1000)) if i % 3 else int(rng.integers(-30, 30))
        x = float(np.ldexp(1.0 + rng.random(), e)) if e > -1022 else float(np.ldexp(rng.random(), -1022))
        if not np.isfinite(x) or x == 0.0:
            continue
        y = float(np.nextafter(x, np.inf))
        mid = (decimal.Decimal(x) + decimal.Decimal(y)) / 2
        s = format(mid, "f") if abs(e) < 60 else format(mid, "e")
        out.append(s)
        if "e" not in s and "." in s:
            out.append(s + "1")           # just above the tie
        if i % 5 == 0:
            out.append("-" + s)
    return out


def edge_cases():
    c = {}
    # the reference's own tests (test_geometry.py:15-60)
    c["single"] = b"v 0 0 0\nv 1 0 0\nv 0 1 0\nf 1 2 3\n"
    c["quad_fan"] = b"v 0 0 0\nv 1 0 0\nv 1 1 0\nv 0 1 0\nf 1 2 3 4\n"
    c["slash"] = b"v 0 0 0\nv 1 0 0\nv 0 1 0\nf 1/1/1 2/2/2 3/3/3\n"
    c["dslash_neg"] = b"v 0 0 0\nv 1 0 0\nv 0 1 0\nf -3//1 -2//2 -1//3\n"
    c["skip"] = b"# c\nvn 0 0 1\nvt 0 0\no thing\nv 0 0 0\nv 1 0 0\nv 0 1 0\nusemtl m\nf 1 2 3\n"
    c["bad_vertex"] = b"v 0 0\n"
    c["face_oob"] = b"v 0 0 0\nv 1 0 0\nv 0 1 0\nf 1 2 9\n"
    # newline styles, comments, whitespace
    c["crlf"] = b"v 0 0 0\r\nv 1 0 0\r\nv 0 1 0\r\nf 1 2 3\r\n"
    c["cr_only"] = b"v 0 0 0\rv 1 0 0\rv 0 1 0\rf 1 2 3"
    c["mixed_nl"] = b"v 0 0 0\r\nv 1 0 0\rv 0 1 0\n\n\r\rf 1 2 3  # tri\r\n# end"
    c["no_trailing_nl"] = b"v 1 2 3\nv 4 5 6\nv 7 8 9\nf 3 2 1"
    c["ws"] = b"  v\t1\x0b2\x0c3  \n\x1cv 4 5 6\x1d\n v 7\x1e8\x1f9\n\tf  1  2\t3 \n"
    c["comments"] = b"v 1 2 3 # x\n#v 9 9 9\nv 4 5 6#\nv 7 8 9\nf 1 2 3 # f 9 9 9\n"
    c["extra_tokens"] = b"v 1 2 3 4 5\nv 4 5 6 1\nv 7 8 9\nf 1 2 3\n"
    c["polygon"] = b"".join(b"v %d %d 0\n" % (i, i * i) for i in range(9)) + b"f 1 2 3 4 5 6 7 8 9\nf -1 -2 -3 -4\n"
    c["not_v"] = b"vv 1 2 3\nV 1 2 3\nv1 2 3\nv 1 2 3\nv 1 2 3\nv 1 2 3\nF 1 2 3\nf 1 2 3\n"
    c["empty"] = b""
    c["only_comments"] = b"# a\n\n   \n# b\n"
    c["no_faces"] = b"v 1 2 3\nv 4 5 6\n"
    c["utf8_other_lines"] = "o nñame\ng été\nv 1 2 3 # é\nv 4 5 6\nv 7 8 9\nf 1 2 3\n".encode()
    c["bom"] = b"\xef\xbb\xbfv 1 2 3\nv 1 2 3\nv 4 5 6\nv 7 8 9\nf 1 2 3\n"
    # Python float()/int() syntax corners
    floats = ["0", "-0", "+0.0", "1.", ".5", "-.5e-3", "1e5", "1E+05", "1_000.000_1", "1e1_0", "0001.5000",
              "inf", "-INF", "Infinity", "+iNfInItY", "nan", "-NaN", "NAN", "1e400", "-1e400", "1e-400",
              "4.9406564584124654e-324", "2.4703282292062327e-324", "2.4703282292062328e-324",
              "2.2250738585072011e-308", "2.2250738585072012e-308", "1.7976931348623157e308",
              "1.7976931348623158e308", "1.7976931348623159e308", "9007199254740993", "9007199254740995",
              "0.1", "0.30000000000000004", "1e23", "8.98846567431158e307", "123456789012345678901234567890",
              "0.000000000000000000000000000001", "3.14159265358979323846264338327950288419716939937510",
              "1" + "0" * 400, "0." + "0" * 300 + "1", "9" * 800, "1." + "1" * 900 + "e-5"]
    text = "".join(f"v {a} {floats[(i + 1) % len(floats)]} {floats[(i + 2) % len(floats)]}\n"
                   for i, a in enumerate(floats))
    c["float_syntax"] = text.encode() + b"f 1 2 3\n"
    c["int_syntax"] = (b"v 0 0 0\nv 1 0 0\nv 0 1 0\nv 1 1 0\nf +1 0_2 3\nf 0004/7 -1//2 -0_2\n"
                       b"f 1 2 3 4 -4 -3\n")
    # errors
    c["err_float"] = b"v 0 0 0\nv 1 0 0\nv 1 1_ 0\nf 1 2 3\n"
    c["err_float2"] = b"v 1 2 3\nv 1e 2 3\n"
    c["err_float3"] = b"v 1 2 3\nv 1 2 0x10\n"
    c["err_float4"] = b"v 1 2 3\nv 1 2 1__0\n"
    c["err_float5"] = b"v 1 2 3\nv . 2 3\n"
    c["err_float6"] = b"v 1 2 3\nv infinit 2 3\n"
    c["err_face_zero"] = b"v 0 0 0\nv 1 0 0\nv 0 1 0\nf 0 1 2\n"
    c["err_face_neg_oob"] = b"v 0 0 0\nv 1 0 0\nv 0 1 0\nf -4 1 2\n"
    c["err_face_later_vertex"] = b"v 0 0 0\nv 1 0 0\nf 1 2 3\nv 0 1 0\n"
    c["err_face_short"] = b"v 0 0 0\nf 1 1\n"
    c["err_face_bad"] = b"v 0 0 0\nv 1 0 0\nv 0 1 0\nf 1 /2 3\n"
    c["err_face_bad2"] = b"v 0 0 0\nv 1 0 0\nv 0 1 0\nf 1 2 3x\n"
    c["err_face_bad3"] = b"v 0 0 0\nv 1 0 0\nv 0 1 0\nf 1 2 3_\n"
    c["err_face_huge"] = b"v 0 0 0\nv 1 0 0\nv 0 1 0\nf 1 2 99999999999999999999999\n"
    c["err_first_of_two"] = b"v 0 0 0\nv 0 0\nv 1 1 1\nf 1 2 9\n"
    c["err_vertex_after_comment"] = b"# v 1 2 3\nv 1 2 # 3\n"
    return c


def fuzz_file(rng, nv=3000, nf=4000):
    """Seeded format fuzz: random spacing, newline styles, comments, exponents, slashes."""
    lines = []
    seps = [" ", "  ", "\t", " \t "]
    nls = ["\n", "\r\n", "\r"]
    for i in range(nv):
        xs = []
        for _ in range(3):
            k = rng.integers(0, 8)
            x = float(rng.normal() * 10.0 ** rng.integers(-12, 12))
            if k == 0:
                xs.append(repr(x))
            elif k == 1:
                xs.append(f"{x:.{int(rng.integers(0, 25))}e}")
            elif k == 2:
                xs.append(f"{x:.{int(rng.integers(0, 30))}f}")
            elif k == 3:
                xs.append(f"{x:+.20g}")
            elif k == 4:
                xs.append(str(int(rng.integers(-10**6, 10**6))))
            elif k == 5:
                xs.append(f"{x:.17g}".replace("e", "E"))
            elif k == 6:
                d = "".join(str(int(v)) for v in rng.integers(0, 10, int(rng.integers(1, 40))))
                xs.append(f"{d[:3]}.{d[3:]}e{int(rng.integers(-330, 310))}")
            else:
                xs.append(repr(float(np.ldexp(rng.random(), int(rng.integers(-1074, 1020))))))
        sep = seps[int(rng.integers(0, len(seps)))]
        line = "v" + sep + sep.join(xs)
        if rng.random() < 0.1:
            line += " # comment " + str(i)
        lines.append(line)
        if rng.random() < 0.05:
            lines.append(["# note", "", "   ", "vn 0 0 1", "vt 0.5 0.5", "o obj", "s off"][int(rng.integers(0, 7))])
        if i >= 3 and rng.random() < nf / nv:
            k = int(rng.integers(3, 7))
            toks = []
            for _ in range(k):
                idx = int(rng.integers(1, i + 2))
                t = str(idx) if rng.random() < 0.7 else str(idx - (i + 2))
                form = int(rng.integers(0, 4))
                if form == 1:
                    t += "/" + str(int(rng.integers(1, 9)))
                elif form == 2:
                    t += "//" + str(int(rng.integers(1, 9)))
                elif form == 3:
                    t += "/1/2"
                toks.append(t)
            lines.append("f " + " ".join(toks))
    out = ""
    for ln in lines:
        out += ln + nls[int(rng.integers(0, 3))]
    return out.encode()


def main():
    rng = np.random.default_rng(20261018)
    cases = edge_cases()
    hw = halfway_strings(rng, 600)
    text = "".join(f"v {hw[i]} {hw[(i + 7) % len(hw)]} {hw[(i + 13) % len(hw)]}\n" for i in range(len(hw)))
    cases["halfway"] = text.encode()
    cases["fuzz"] = fuzz_file(rng)
    arrays, meta = {}, {}
    for name, data in cases.items():
        arrays[f"{name}/bytes"] = np.frombuffer(data, np.uint8)
        res = ref_load(data)
        if res[0] == "ok":
            arrays[f"{name}/V"] = res[1]
            arrays[f"{name}/T"] = res[2]
            meta[name] = {"ok": True, "nv": len(res[1]), "nt": len(res[2])}
        else:
            meta[name] = {"ok": False, "message": res[1], "line": res[2]}
        print(name, meta[name] if not meta[name]["ok"] else (meta[name]["nv"], meta[name]["nt"]), flush=True)
    np.savez_compressed(os.path.join(HERE, "obj.npz"), **arrays)
    # a scene file regenerated on the box: cfg1 through the reference save_obj
    mesh = scenes.gen_scene("uniform", 100_000, 7)
    with tempfile.NamedTemporaryFile(suffix=".obj", delete=False) as fh:
        path = fh.name
    save_obj(pargrid.geometry.TriangleMesh(mesh.vertices, mesh.triangles), path)
    with open(path, "rb") as fh:
        data = fh.read()
    m = load_obj(path)
    os.unlink(path)
    big = {"recipe": {"kind": "uniform", "n": 100_000, "seed": 7},
           "bytes_sha256": hashlib.sha256(data).hexdigest(),
           "V_sha256": hashlib.sha256(m.vertices.tobytes()).hexdigest(),
           "T_sha256": hashlib.sha256(m.triangles.tobytes()).hexdigest()}
    with open(os.path.join(HERE, "obj.json"), "w") as fh:
        json.dump({"reference": "pargrid 0.1.0 geometry.load_obj", "cases": meta, "cfg1_save_obj": big},
                  fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
