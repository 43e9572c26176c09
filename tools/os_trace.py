"""Per-tile phase breakdown of the last onesweep pass (PGRID_OS_TRACE=1)."""
import ctypes, os, sys
import numpy as np, torch
os.environ["PGRID_OS_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_10647_b200 import _native, scenes
mesh, spec = scenes.config_scene(sys.argv[1] if len(sys.argv) > 1 else "cfg3")
Vd = torch.from_numpy(mesh.vertices.copy()).cuda(); Td = torch.from_numpy(mesh.triangles.copy()).cuda()
b = _native.Builder(0); sp = torch.cuda.current_stream().cuda_stream
no = b.count(Vd, len(mesh.vertices), Td, len(mesh.triangles), spec, 0, sp)
Gd = torch.empty(spec.ncells + 1, dtype=torch.int32, device="cuda"); Od = torch.empty(no, dtype=torch.int32, device="cuda")
for _ in range(3):
    b.count(Vd, len(mesh.vertices), Td, len(mesh.triangles), spec, 0, sp); b.finish(Gd, Od, 0, sp, timed=False)
torch.cuda.synchronize()
lib = _native.load(); lib.pg_debug_trace.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64]
ntiles = (no + 4095) // 4096
buf = np.zeros(ntiles * 8, np.uint64)
_native.check(lib.pg_debug_trace(b._h, buf.ctypes.data, buf.nbytes))
t = buf.reshape(ntiles, 8).astype(np.int64)
t0 = t[:, 0].min()
names = ["load+rank", "count+scan", "lookback", "keys out+vals wait", "vals perm+out"]
d = np.diff(t[:, :6], axis=1)
print("tiles", ntiles, "pass span us", (t[:, 5].max() - t0) / 1e3)
for i, nm in enumerate(names):
    print(f"{nm:22s} mean {d[:, i].mean()/1e3:7.2f} us  p50 {np.median(d[:, i])/1e3:7.2f}  p90 {np.percentile(d[:, i], 90)/1e3:7.2f}  max {d[:, i].max()/1e3:7.2f}")
tot = t[:, 5] - t[:, 0]
print(f"{'tile total':22s} mean {tot.mean()/1e3:7.2f} us")
# gap between tiles of the same CTA
cta = t[:, 7]
gaps = []
for c in np.unique(cta):
    rows = t[cta == c]; rows = rows[np.argsort(rows[:, 0])]
    gaps += list((rows[1:, 0] - rows[:-1, 5]) / 1e3)
print("inter-tile gap per CTA mean us", np.mean(gaps) if gaps else None, "ctas", len(np.unique(cta)))
# start-time spread of consecutive tiles
st = t[:, 0]
print("start(t) - start(t-1) mean us", np.mean(np.diff(st)) / 1e3, " lookback wait vs predecessor publish:")
pub = t[:, 2]  # after count+scan (aggregate published before this stamp)
print("  tile start lag behind predecessor publish (p50 us)", np.median((t[1:, 1] - pub[:-1])) / 1e3)
