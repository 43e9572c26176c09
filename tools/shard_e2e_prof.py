import os, sys, time
import numpy as np, torch, torch.distributed as dist
sys.path.insert(0, os.getcwd())
from paper_2403_10647_b200 import distributed as D, scenes, gridcore, _native
os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29571")
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
n = 10_000_000
shard = scenes.gen_arch_shard(n, 7, 4.0, 0, n)
spec = gridcore.spec_from_bounds(shard.vertices.min(0), shard.vertices.max(0), n, density=4.0)
ops = D.CudaOps(0); comm = D.TorchComm(device=torch.device("cuda", 0))
ex = D.PeerExchange(comm, torch.device("cuda", 0))
Vh, Th = shard.vertices.copy(), shard.triangles.copy()
_native.host_register(Vh); _native.host_register(Th)
orig = {}
def wrap(obj, name):
    f = getattr(obj, name)
    def g(*a, **k):
        torch.cuda.synchronize(); t0 = time.perf_counter(); r = f(*a, **k); torch.cuda.synchronize()
        orig.setdefault(name, []).append((time.perf_counter() - t0) * 1e3); return r
    setattr(obj, name, g)
for nm in ["count", "count_deferred", "pairs", "slab_plan", "partition_counts", "partition_send", "sort_cells", "to_numpy", "count_result"]:
    wrap(ops, nm)
for nm in ["put_hist", "read_counts", "ensure", "barrier", "put_counts"]:
    wrap(ex, nm)
for it in range(4):
    orig.clear()
    t0 = time.perf_counter()
    r = D.build_sharded(ops, comm, Vh, Th, 0, spec, gather=False, exchange=ex)
    g, o = ops.to_numpy(r[3]), ops.to_numpy(r[4])
    print(f"iter {it}: {(time.perf_counter() - t0) * 1e3:.1f} ms", {k: [round(x, 2) for x in v] for k, v in orig.items()})
dist.destroy_process_group()
