"""Per-rank time budget of the sharded build at world P, measured on ONE B200 by running every
virtual rank's phases in sequence (distributed.ShardState + EmulatedExchange, as
run_emulated does) and timing each phase of each rank with CUDA events.

    python tools/shard_budget.py [--config cfg5] [--world 8] [--reps 3]

Per rank: K1 + K2 + the coarse histogram on its triangle shard, the slab upsweep, the
peer-store partition (here into this GPU's buffers; across GPUs those stores go over
NVLink), and the slab sort + K4 of its cell slab. The NVLink share is reported as bytes
leaving each rank; the line also gives the one-GPU build of the same scene for the speed-up
estimate. Device-resident inputs; no host round trips inside the timed phases.
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT]
from paper_2403_10647_b200 import _native, scenes  # noqa: E402
from paper_2403_10647_b200 import distributed as D  # noqa: E402
from paper_2403_10647_b200.gridcore import spec_for_mesh  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg5")
ap.add_argument("--world", type=int, default=8)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--ktimes", action="store_true", help="per-kernel times of every rank's K2 + histogram (last rep)")
ap.add_argument("--reverse", action="store_true", help="run the emulated ranks in reverse order")
ap.add_argument("--reverse-timed", action="store_true",
                help="allocate in rank order (rep 0) but time the ranks in reverse order")
a = ap.parse_args()
kind, n, seed, density = scenes.CONFIGS[a.config]
mesh = scenes.gen_scene_large(kind, n, seed, density) if n > 20_000_000 else scenes.gen_scene(kind, n, seed, density)
spec = spec_for_mesh(mesh, density=density)
Vd = torch.from_numpy(mesh.vertices).cuda()
Td = torch.from_numpy(mesh.triangles).cuda()
del mesh
P = a.world
ev = lambda: torch.cuda.Event(enable_timing=True)


def timed(fn):
    e0, e1 = ev(), ev()
    e0.record()
    out = fn()
    e1.record()
    torch.cuda.synchronize()
    return out, e0.elapsed_time(e1)


# one-GPU build of the whole scene (graph replay) for the speed-up estimate
b = _native.Builder(0)
st = torch.cuda.current_stream().cuda_stream
no = b.count(Vd, Vd.shape[0], Td, Td.shape[0], spec, 0, st)
Gd = torch.empty(spec.ncells + 1, dtype=torch.int32, device="cuda")
Od = torch.empty(no, dtype=torch.int32, device="cuda")
for _ in range(3):
    b.build_async(Vd, Vd.shape[0], Td, Td.shape[0], spec, Gd, Od, no, st)
b.build_wait()
one = []
for _ in range(a.reps):
    _, ms = timed(lambda: b.build_async(Vd, Vd.shape[0], Td, Td.shape[0], spec, Gd, Od, no, st))
    one.append(ms)
b.close()
del Gd, Od
torch.cuda.empty_cache()

states = []
for r in range(P):
    # every rank holds only its shard, as a local soup (vertex rows 3lo..3hi, indices from 0),
    # as bench.py's ranks generate it (scenes.gen_shard)
    lo, hi = D.shard_range(n, r, P)
    Tr = (Td[lo:hi] - 3 * lo).contiguous()
    states.append(D.ShardState(D.CudaOps(), Vd[3 * lo:3 * hi], Tr, lo, spec, r, P))
ex = D.EmulatedExchange(torch, torch.device("cuda", 0), P)
rows = []
cap = None
for rep in range(a.reps + 1):
    # rep 0: host-checked counts (the verdict; learns the pair capacity); then deferred counts
    # (PG_DEFER: no host round trip inside K1), as the steady-state sharded build runs them
    t = {r: {} for r in range(P)}
    order = list(range(P))[::-1] if (a.reverse or (a.reverse_timed and rep > 0)) else list(range(P))
    stats = [None] * P
    hists = [None] * P
    for r in order:
        s = states[r]
        st_r, t[r]["k1"] = timed(lambda: s.phase_count_only(cap))
        stats[r] = st_r
        if a.ktimes and rep == a.reps:
            _native.kernel_timing(True)
        h, t[r]["k2_hist"] = timed(lambda: s.phase_pairs())
        if a.ktimes and rep == a.reps:
            print("rank", r, [(k, round(us, 1)) for k, us in _native.kernel_times()], file=sys.stderr)
            _native.kernel_timing(False)
        hists[r] = h
    if cap is None:
        D.count_verdict(np.sum(stats, axis=0), states[0].ncells)
        cap = int(max(s.no for s in states) * 1.25) + 4096
    hist = np.sum([s.ops.to_numpy(h).astype(np.int64) for s, h in zip(states, hists)], axis=0)
    plan = D.plan_slabs(hist, states[0].ncells, P)
    counts = []
    for r, s in enumerate(states):
        c, t[r]["slab_upsweep"] = timed(lambda: s.phase_partition_counts(plan))
        counts.append(s.ops.to_numpy(c)[:P].astype(np.int64))
    matrix = np.array(counts)
    ex.ensure(int(matrix.sum(axis=0).max()))
    dk, dv = ex.destinations()
    nrecv = {}
    for r, s in enumerate(states):
        nrecv[r], t[r]["partition_send"] = timed(lambda: s.phase_send(matrix, dk, dv))
    for r, s in enumerate(states):
        _, t[r]["slab_sort_k4"] = timed(lambda: s.phase_sort(*ex.received(r, nrecv[r])))
    if rep:
        rows.append(t)

med = {r: {k: float(np.median([rows[i][r][k] for i in range(a.reps)])) for k in rows[0][r]} for r in range(P)}
send_bytes = [int(8 * (matrix[r].sum() - matrix[r][r])) for r in range(P)]
recv_bytes = [int(8 * (matrix[:, r].sum() - matrix[r][r])) for r in range(P)]
phase1 = [med[r]["k1"] + med[r]["k2_hist"] + med[r]["slab_upsweep"] + med[r]["partition_send"] for r in range(P)]
phase2 = [med[r]["slab_sort_k4"] for r in range(P)]
# NVLink 5: ~900 GB/s per direction per GPU nominal; the peer stores overlap the partition
# kernel's own HBM traffic, so the estimate charges the larger of the two
nvlink_gbs = 750.0
est = [max(phase1[r], med[r]["k1"] + med[r]["k2_hist"] + med[r]["slab_upsweep"] + send_bytes[r] / nvlink_gbs / 1e6)
       for r in range(P)]
step = max(est) + max(phase2) + 0.05          # + device barriers / one host read (measured ~0.05 ms)
print(json.dumps({
    "config": a.config, "scene": kind, "triangles": n, "dims": list(spec.dims), "no": int(no), "world": P,
    "one_gpu_ms": round(float(np.median(one)), 3),
    "per_rank_ms": {r: {k: round(v, 3) for k, v in med[r].items()} for r in range(P)},
    "send_mb_per_rank": [round(x / 1e6, 1) for x in send_bytes],
    "recv_mb_per_rank": [round(x / 1e6, 1) for x in recv_bytes],
    "phase1_max_ms": round(max(phase1), 3), "phase2_max_ms": round(max(phase2), 3),
    "estimated_step_ms": round(step, 3), "nvlink_gbs_assumed": nvlink_gbs,
    "estimated_speedup": round(float(np.median(one)) / step, 2)}))
