"""Break down the public-API (numpy in/out) build time on a config."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_10647_b200 import _native, builders, scenes
from paper_2403_10647_b200.gridcore import TriangleMesh
name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
mesh, spec = scenes.config_scene(name)
V = mesh.vertices.copy(); T = mesh.triangles.copy()
_native.host_register(V); _native.host_register(T)
m = TriangleMesh(V, T)
b = _native.thread_builder()
for it in range(4):
    t0 = time.perf_counter()
    no = b.count(V, len(V), T, len(T), spec, flags=_native.PG_HOST_INPUT)
    t1 = time.perf_counter()
    G = np.empty(spec.ncells + 1, np.uint32); O = np.empty(no, np.uint32)
    t2 = time.perf_counter()
    ph = b.finish(G, O, flags=_native.PG_HOST_OUTPUT)
    t3 = time.perf_counter()
    print(f"count(H2D+K1) {1e3*(t1-t0):.2f} ms  alloc {1e3*(t2-t1):.2f}  finish(+D2H) {1e3*(t3-t2):.2f}  phases {[round(x,3) for x in ph]}")
for it in range(3):
    t0 = time.perf_counter(); g, r = builders.build_parallel(m, spec); t1 = time.perf_counter()
    print(f"build_parallel {1e3*(t1-t0):.2f} ms")
