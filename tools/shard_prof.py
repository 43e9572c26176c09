"""Phase timing of the sharded build on one GPU (world 1, NCCL): where do the ms go?"""
import os, sys, time
import numpy as np
import torch
import torch.distributed as dist
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_10647_b200 import distributed as D, scenes, gridcore

os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29561")
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
n = 10_000_000
shard = scenes.gen_arch_shard(n, 7, 4.0, 0, n)
spec = gridcore.spec_from_bounds(shard.vertices.min(0), shard.vertices.max(0), n, density=4.0)
Vd = torch.from_numpy(shard.vertices.copy()).cuda(); Td = torch.from_numpy(shard.triangles.copy()).cuda()
ops = D.CudaOps(0); comm = D.TorchComm(device=torch.device("cuda", 0))
P2P = "--p2p" in sys.argv or "--fused" in sys.argv
FUSED = "--fused" in sys.argv
ex = D.PeerExchange(comm, torch.device("cuda", 0)) if P2P else None
T = {}
E = {}
def tick(name, t0):
    ev = torch.cuda.Event(enable_timing=True); ev.record()
    E.setdefault(name, []).append(ev)
    torch.cuda.synchronize(); T[name] = T.get(name, 0) + time.perf_counter() - t0; return time.perf_counter()
for it in range(6):
    if it == 1: T.clear(); E.clear()
    t = time.perf_counter()
    e0 = torch.cuda.Event(enable_timing=True); e0.record(); E.setdefault("_start", []).append(e0)
    st = D.ShardState(ops, Vd, Td, 0, spec, 0, 1)
    if FUSED:
        h = st.phase_count_fused(ex.no_capacity); t = tick("count+coarse", t)
        ex.put_hist(h, 0); ex.put_no(0, ops); ex.barrier(); t = tick("put+barrier", t)
        st.phase_plan_device(ex.hists(st.nb_coarse)); t = tick("plan_dev", t)
        hists, nos, _, pa = ex.read_hists(st.nb_coarse, st.plan_d); t = tick("read", t)
        ex.no_capacity = int(nos.max() * 1.0625) + 4096
        if st.deferred: ops.count_result()
        plan = st.set_plan(pa); m = D.slab_matrix(hists, plan.cuts); ex.ensure(int(m.sum(axis=0).max()))
        dk, dv = ex.destinations(); nr = st.phase_pairs_send(m, dk, dv); t = tick("pairs_send", t)
        ex.barrier(); kr, vr = ex.received(nr); t = tick("barrier", t)
        r = st.phase_sort(kr, vr); t = tick("sort_cells", t)
        continue
    if P2P and ex.no_capacity:   # deferred count (no NO read back), as build_sharded
        st.deferred = True; st.no = ops.count_deferred(Vd, Td, spec, ex.no_capacity)
    else:
        st.deferred = False; st.no = ops.count(Vd, Td, spec)
    t = tick("count", t)
    st.shift = D.coarse_shift(st.ncells); nb = ((st.ncells - 1) >> st.shift) + 1
    st.nb_coarse = nb
    st.keys, st.vals, h = ops.pairs(st.no, 0, st.shift, nb); t = tick("pairs+hist", t)
    if P2P:   # device plan: peer put + barrier + plan kernel; counts the same way; one readback
        ex.put_hist(h, 0); ex.barrier(); t = tick("put_hist", t)
        st.phase_plan_device(ex.hists(nb)); t = tick("plan_dev", t)
        ex.put_counts(st.phase_partition_counts_device(), 0, ops); t = tick("part_counts", t)
        ex.barrier(); m, nos, _, pa = ex.read_counts(st.plan_d); st.set_plan(pa)
        ex.no_capacity = int(nos.max() * 1.25) + 4096
        if st.deferred: ops.count_result()
        ex.ensure(int(m.sum(axis=0).max())); t = tick("read_counts", t)
        dk, dv = ex.destinations(); nr = st.phase_send(m, dk, dv); t = tick("send", t)
        ex.barrier(); kr, vr = ex.received(nr); t = tick("barrier", t)
    else:
        h = comm.allreduce_sum(h); t = tick("allreduce", t)
        plan = D.plan_slabs(h, st.ncells, 1); t = tick("plan", t)
        sc = st.phase_partition(plan); t = tick("partition", t)
        send, recv = comm.alltoall_counts(sc); t = tick("a2a_counts", t)
        kr, vr = comm.alltoall_pairs(st.kout, st.vout, send, recv, ops); t = tick("a2a_pairs", t)
    r = st.phase_sort(kr, vr); t = tick("sort_cells", t)
torch.cuda.synchronize()
names = list(T)
for k in names:
    prev = [E["_start"][i] if names.index(k) == 0 else E[names[names.index(k) - 1]][i] for i in range(5)]
    dev = sum(p.elapsed_time(e) for p, e in zip(prev, E[k])) / 5
    print(f"{k:12s} host {T[k] / 5 * 1e3:8.3f} ms   device {dev:8.3f} ms")
print("total", sum(T.values()) / 5 * 1e3)
dist.destroy_process_group()
