"""Shared helpers for the parity tests (fixtures are regenerated from recipes)."""

import hashlib

import numpy as np

from paper_2403_10647_b200 import scenes
from paper_2403_10647_b200.gridcore import Aabb, GridSpec, TriangleMesh, spec_for_mesh

KAT_NAMES = ("walkthrough", "full_cover", "dropped", "faces", "nonfinite", "indexed",
             "one_cell", "sparse_kept")


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def kat_case(kat, name):
    mesh = TriangleMesh(kat[f"{name}/V"], kat[f"{name}/T"])
    spec = GridSpec(Aabb(kat[f"{name}/lo"], kat[f"{name}/hi"]), tuple(int(d) for d in kat[f"{name}/dims"]))
    return mesh, spec


def scene_from_recipe(recipe):
    """(mesh, spec) for a hashes.json recipe."""
    mesh = scenes.gen_scene(recipe["kind"], recipe["n"], recipe["seed"], recipe.get("density", 5.0))
    if "dims" in recipe:
        return mesh, spec_for_mesh(mesh, dims=tuple(recipe["dims"]))
    return mesh, spec_for_mesh(mesh, density=recipe["density"])


RAY_CASES = ("unit",) + tuple(f"validate_{i}" for i in range(10)) + \
    ("inside_walls", "inside_uniform", "inside_skewed", "cfg1", "cfg2", "arch1m")


def ray_case(rays, name):
    """(mesh, spec, origins, dirs, t_max) of a golden ray case (make_golden_rays.py)."""
    arrays, meta = rays
    recipe = meta[name]["recipe"]
    if recipe["kind"] == "unit_triangle":
        mesh = TriangleMesh([[0, 0, 0], [1, 0, 0], [0, 1, 0]], [[0, 1, 2]])
        spec = spec_for_mesh(mesh, dims=tuple(recipe["dims"]))
    else:
        mesh, spec = scene_from_recipe(recipe)
    return (mesh, spec, arrays[f"{name}/origins"], arrays[f"{name}/dirs"], arrays[f"{name}/t_max"])


def inverted_cases():
    """Golden inverted-box scenes (tests/golden/make_golden_inverted.py, the reference's own
    verdicts): [(name, mesh arrays V, T, spec, verdict 0 grid / 1 SizeError / 2 InvariantError,
    G, O)]."""
    import os
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "inverted.npz")
    out = []
    with np.load(path) as z:
        for name in z["names"]:
            name = str(name)
            spec = GridSpec(Aabb([0, 0, 0], [1, 1, 1]), tuple(int(d) for d in z[f"{name}/dims"]))
            out.append((name, z[f"{name}/V"], z[f"{name}/T"], spec, int(z[f"{name}/verdict"]),
                        z[f"{name}/G"], z[f"{name}/O"]))
    return out
