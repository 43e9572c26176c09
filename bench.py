"""Benchmark of the B200 parallel grid build (BASELINE.json metric on its headline config).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg3] [--impl reference]

A "step" is one full build_parallel of the config's scene (default cfg3: the 10M-triangle
architectural scene, density 4, 342^3 cells -- BASELINE.json configs[2], the paper's 25 Hz
case). `value` = builds/s with inputs resident in HBM (device pointers through the C ABI);
`e2e` = the same through the public numpy API (pinned host inputs, H2D + build + D2H of G
and O inside the timed region). Rank 0 prints one JSON line.

N > 1 (torchrun): the sharded build of SURVEY.md §8e on an N x 10M-triangle architectural
scene (weak scaling: 10M triangles per GPU): each rank generates and counts its triangle
shard, pairs are routed to cell slabs by one NCCL all-to-all, every rank sorts its slab and
writes its G/O slice (distributed output).
`--impl reference` times the reference's own CPU build (oracle/_ref, C lane, all host
threads) on the same config instead.
"""

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "grid builds/sec (Hz) + M pairs/s on 10M-tri scene; HBM GB/s vs peak"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="cfg3")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--cpu-budget-s", type=float, default=150.0)
    ap.add_argument("--sharded", action="store_true", help="use the sharded path even at N=1 (testing)")
    ap.add_argument("--nccl-exchange", action="store_true", help="sharded: partition pass + NCCL all_to_all")
    ap.add_argument("--fused-dispatch", action="store_true",
                    help="sharded: expansion + dispatch in one kernel (pg_pairs_send; measured slower, off)")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *exc):
        self.out = ""
        if self.proc is not None:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()
        return False

    def summary(self):
        rows = []
        for line in (self.out or "").strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                rows.append(parts)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[3 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": float(rows[0][1]) if rows[0][1].replace(".", "").isdigit() else None,
                "reasons": reasons, "samples": len(rows)}


def traffic_table():
    """Per-launch DRAM bytes of each kernel from the committed ncu capture (or {})."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            return json.load(fh)
    except Exception:
        return {}


def run_reference(args, world, rank):
    """The reference's own CPU implementation on the same config (oracle/_ref, C lane)."""
    if rank != 0:
        return
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle
    from paper_2403_10647_b200 import scenes
    ref = oracle.reference_module()
    mesh, spec = scenes.config_scene(args.config)
    cores = os.cpu_count() or 1
    if ref is not None:
        kind = "reference"
        rmesh = ref.TriangleMesh(mesh.vertices, mesh.triangles)
        rspec = ref.GridSpec(ref.Aabb(spec.bounds.lo, spec.bounds.hi), spec.dims)

        def one():
            g, rep = ref.build_parallel(rmesh, rspec, workers=cores)
            return rep.no
    else:
        kind = "port"
        cores = 1

        def one():
            G, O = oracle.build_parallel(mesh.vertices, mesh.triangles, spec)
            return len(O)
    t0 = time.perf_counter()
    no = one()                       # warm-up build, also sizes the sample
    t_first = time.perf_counter() - t0
    warm = max(0, min(args.warmup, 1) - 1)
    for _ in range(warm):
        one()
    steps = max(1, min(args.steps, int(args.cpu_budget_s // max(t_first, 1e-3))))
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        one()
        times.append(time.perf_counter() - t0)
    sec = statistics.median(times)
    value = 1.0 / sec
    sample = (f"full {args.config} build ({mesh.ntriangles} tris, dims {spec.dims}), "
              f"{steps} timed of {args.steps} requested (CPU time cap {args.cpu_budget_s:.0f}s), "
              f"workers={cores if kind == 'reference' else 1}, {cpu_model()}")
    line = {"metric": METRIC, "impl": "reference", "value": round(value, 6), "unit": "builds/s",
            "n_gpus": world, "steps": steps, "warmup": 1, "ms_per_step": round(sec * 1e3, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64+u32",
            "data": "synthetic", "mpairs_per_s": round(no / sec / 1e6, 4),
            "config": {"workload": args.config, "triangles": mesh.ntriangles, "dims": list(spec.dims),
                       "no": int(no)},
            "cpu_baseline": {"value": round(value, 6), "unit": "builds/s", "cores": cores, "kind": kind,
                             "sample": sample},
            "e2e": {"value": round(value, 6), "unit": "builds/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def cpu_baseline(args, mesh, spec):
    """Rank 0, N=1 only: the reference CPU build timed once on the same scene (~20-30 s)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle
    ref = oracle.reference_module()
    if ref is not None:
        rmesh = ref.TriangleMesh(mesh.vertices, mesh.triangles)
        rspec = ref.GridSpec(ref.Aabb(spec.bounds.lo, spec.bounds.hi), spec.dims)
        t0 = time.perf_counter()
        ref.build_parallel(rmesh, rspec)
        sec = time.perf_counter() - t0
        return {"value": round(1.0 / sec, 6), "unit": "builds/s", "cores": 1, "kind": "reference",
                "sample": f"1 full {args.config} build, reference pargrid C lane, workers=None "
                          f"(single thread), {sec:.2f}s, {cpu_model()}"}
    t0 = time.perf_counter()
    oracle.build_parallel(mesh.vertices, mesh.triangles, spec)
    sec = time.perf_counter() - t0
    return {"value": round(1.0 / sec, 6), "unit": "builds/s", "cores": 1, "kind": "port",
            "sample": f"1 full {args.config} build, C oracle port, single thread, {sec:.2f}s"}


def run_sharded(args, world, rank, local):
    """N > 1: sharded build over NCCL (paper_2403_10647_b200/distributed.py)."""
    import torch
    import torch.distributed as dist

    from paper_2403_10647_b200 import _native
    from paper_2403_10647_b200 import distributed as D
    from paper_2403_10647_b200 import gridcore, scenes

    kind, n1, seed, density = scenes.CONFIGS[args.config]
    if kind != "arch":
        raise SystemExit("sharded bench supports the arch configs")
    n = n1 * world
    lo, hi = D.shard_range(n, rank, world)
    shard = scenes.gen_arch_shard(n, seed, density, lo, hi)
    dev = torch.device("cuda", local)
    bmin = torch.from_numpy(shard.vertices.min(axis=0).copy()).to(dev)
    bmax = torch.from_numpy(shard.vertices.max(axis=0).copy()).to(dev)
    dist.all_reduce(bmin, op=dist.ReduceOp.MIN)
    dist.all_reduce(bmax, op=dist.ReduceOp.MAX)
    spec = gridcore.spec_from_bounds(bmin.cpu().numpy(), bmax.cpu().numpy(), n, density=density)
    Vd = torch.from_numpy(shard.vertices.copy()).to(dev)
    Td = torch.from_numpy(shard.triangles.copy()).to(dev)
    ops = D.CudaOps(local)
    comm = D.TorchComm(device=dev)
    # the pair exchange: fused into the partition kernel (peer stores into the slab owners'
    # symmetric-memory receive buffers) when symmetric memory comes up on every rank, else a
    # partition pass + NCCL all_to_all; every rank must agree, so the choice is all-reduced
    ex, why = None, ""
    if not args.nccl_exchange:
        try:
            ex = D.PeerExchange(comm, dev)
        except Exception as e:          # noqa: BLE001 -- reported in the JSON line
            why = f"{type(e).__name__}: {e}"[:200]
    if ex is not None and args.fused_dispatch:
        ex.fused = True
    ok = torch.tensor([1 if ex is not None else 0], device=dev)
    dist.all_reduce(ok, op=dist.ReduceOp.MIN)
    if int(ok.item()) == 0:
        ex = None
    exchange_desc = (("expansion + slab dispatch in one kernel, peer stores (symmetric memory)" if ex.fused else
                      "fused partition + peer stores (symmetric memory)") if ex is not None
                     else "partition pass + NCCL all_to_all" + (f" ({why})" if why else ""))

    def step():
        return D.build_sharded(ops, comm, Vd, Td, lo, spec, gather=False, exchange=ex)

    res = step()
    launches = ops.b.launches()
    for _ in range(max(args.warmup, 3)):
        res = step()
    no_local = int(res[4].numel())
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        dist.barrier()
        ev0.record()
        for _ in range(args.steps):
            step()
        ev1.record()
        torch.cuda.synchronize()
        dist.barrier()
    ms = torch.tensor([ev0.elapsed_time(ev1) / args.steps], device=dev)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms = float(ms.item())
    no_t = torch.tensor([no_local], device=dev, dtype=torch.int64)
    dist.all_reduce(no_t)
    no = int(no_t.item())

    # per-kernel device times of one step on this rank (events after every launch)
    _native.kernel_timing(True)
    step()
    torch.cuda.synchronize()
    kt = {}
    for name, us in _native.kernel_times():
        if not name.startswith("("):
            kt.setdefault(name, []).append(us * 1e-3)
    _native.kernel_timing(False)
    peak, peak_kind = peaks()
    sc_name = "k_radix_scatter_wc" if "k_radix_scatter_wc" in kt else "k_radix_scatter"
    sc = kt.get(sc_name, [])
    sc_ms = float(np.mean(sc)) if sc else 0.0
    sc_bytes = 16 * no_local
    roofline = {"bound": "hbm", "kernel": sc_name + " (slab sort, rank 0)",
                "achieved": round(sc_bytes / (sc_ms * 1e-3) / 1e9, 1) if sc_ms else None, "peak": peak,
                "unit": "GB/s", "frac": round(sc_bytes / (sc_ms * 1e-3) / 1e9 / peak, 4) if sc_ms else None,
                "traffic": traffic_table().get(sc_name), "alg_bytes_per_launch": sc_bytes,
                "launch_ms": round(sc_ms, 4), "peak_kind": peak_kind}
    kernels = {k: {"ms_per_launch": round(float(np.mean(v)), 4), "launches": len(v)} for k, v in kt.items()}

    # e2e: pinned host shard in, H2D + sharded build + D2H of this rank's G/O slab out
    Vh, Th = shard.vertices.copy(), shard.triangles.copy()
    _native.host_register(Vh)
    _native.host_register(Th)
    e2e = []
    out_nbytes = 0
    # two untimed rounds warm the page-locked output pool (its first allocations are
    # cudaHostAlloc calls of ~100 ms); each round drops its host slab so the blocks recycle
    for i in range(2 + (args.e2e_steps or min(args.steps, 5))):
        dist.barrier()
        t0 = time.perf_counter()
        r = D.build_sharded(ops, comm, Vh, Th, lo, spec, gather=False, exchange=ex)
        g_host, o_host = ops.to_numpy(r[3]), ops.to_numpy(r[4])     # this rank's slab, D2H
        t = torch.tensor([time.perf_counter() - t0], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        if i >= 2:
            e2e.append(float(t.item()))
        out_nbytes = g_host.nbytes + o_host.nbytes
        del r, g_host, o_host
    e2e_sec = statistics.median(e2e)
    # gathered-to-rank-0 output: device-resident shards, the slabs sent to rank 0
    # point-to-point and rebased there, then rank 0 copies the whole G/O to the host
    gat = []
    for i in range(2 + min(args.steps, 5)):
        dist.barrier()
        t0 = time.perf_counter()
        r = D.build_sharded(ops, comm, Vd, Td, lo, spec, gather="device", exchange=ex)
        if rank == 0:
            gh, oh = ops.to_numpy(r[0]), ops.to_numpy(r[1])
            del gh, oh
        torch.cuda.synchronize()
        t = torch.tensor([time.perf_counter() - t0], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        if i >= 2:
            gat.append(float(t.item()))
        del r
    gathered_ms = statistics.median(gat) * 1e3
    out_bytes = torch.tensor([out_nbytes], device=dev, dtype=torch.int64)
    dist.all_reduce(out_bytes)
    line = {
        # whole-job throughput in the metric's unit: 10M-triangle-scene builds per second
        # (N x builds/s of the N x 10M scene), so weak scaling is value(N) / (N value(1))
        "metric": METRIC, "value": round(world * 1e3 / ms, 3), "unit": "builds/s", "n_gpus": world,
        "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": round(ms, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64+u32",
        "data": "synthetic",
        "config": {"workload": f"{args.config} x{world} (sharded)", "scene": kind, "triangles": n,
                   "triangles_per_gpu": n1, "dims": list(spec.dims), "ncells": spec.ncells, "no": no,
                   "parallelism": f"triangle shards x{world} -> cell slabs",
                   "exchange": exchange_desc,
                   "output": "distributed (each rank its G/O slab)",
                   "value_def": f"{world} x builds/s of the {world} x {n1 // 1_000_000}M-triangle scene",
                   "scene_builds_per_s": round(1e3 / ms, 3),
                   "parity": "orchestration verified by tests/test_distributed.py + test_gpu_distributed.py"},
        "mpairs_per_s": round(no / (ms * 1e-3) / 1e6, 2),
        "roofline": roofline,
        "kernels_rank0": kernels,
        "e2e": {"value": round(world / e2e_sec, 3), "unit": "builds/s",
                "h2d_bytes_per_step": int((Vh.nbytes + Th.nbytes) * world),
                "d2h_bytes_per_step": int(out_bytes.item()), "ms_per_step": round(e2e_sec * 1e3, 2)},
        "gathered_output": {"ms_per_step": round(gathered_ms, 3),
                            "what": "device-resident shards -> slabs sent to rank 0 (NCCL p2p), G rebased, "
                                    "full G/O copied to rank 0's host; max over ranks, wall clock"},
        "gpu_launches": launches * args.steps,
        "clocks": clk.summary(),
    }
    if rank == 0:
        print(json.dumps(line), flush=True)


def main():
    args = parse()
    world, rank, local = dist_env()
    if args.impl == "reference":
        if world > 1:
            import torch.distributed as dist
            dist.init_process_group("gloo")
        run_reference(args, world, rank)
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
            dist.destroy_process_group()
        return

    import torch
    torch.cuda.set_device(local)
    if world > 1 or args.sharded:
        import torch.distributed as dist
        if not dist.is_initialized():
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29533")
            dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", local))
        try:
            run_sharded(args, world, rank, local)
        finally:
            dist.barrier()
            dist.destroy_process_group()
        return

    from paper_2403_10647_b200 import _native, builders, scenes

    mesh, spec = scenes.config_scene(args.config)
    V, T = mesh.vertices, mesh.triangles
    n, nv = len(T), len(V)
    ncells = spec.ncells
    dev = torch.device("cuda", local)
    Vd = torch.from_numpy(np.ascontiguousarray(V)).to(dev)
    Td = torch.from_numpy(np.ascontiguousarray(T)).to(dev)
    b = _native.Builder(local)
    stream = torch.cuda.current_stream(dev)
    sp = stream.cuda_stream
    no = b.count(Vd, nv, Td, n, spec, 0, sp)
    Gd = torch.empty(ncells + 1, dtype=torch.int32, device=dev)
    Od = torch.empty(max(no, 1), dtype=torch.int32, device=dev)

    def step(timed=False):
        b.count(Vd, nv, Td, n, spec, 0, sp)
        return b.finish(Gd, Od, 0, sp, timed=timed)

    step()
    # timed steps use the sync-free build: the whole build is one CUDA-graph replay, no host
    # round trip for NO (capacity = this scene's NO; checked after the timed region)
    pgspec = _native.PgSpec.from_spec(spec)

    def step_graph():
        b.build_async(Vd, nv, Td, n, spec, Gd, Od, no, sp, pgspec)

    step_graph()          # eager run + capture
    step_graph()          # first graph replay: the parity check below reads its G/O
    assert b.build_wait() == no
    launches = b.launches()
    # parity of the measured (graph-replayed) configuration against the reference's golden hashes
    parity = "unchecked"
    try:
        import hashlib
        with open(os.path.join(ROOT, "tests", "golden", "hashes.json")) as fh:
            h = json.load(fh)["scenes"].get(args.config)
        if h:
            torch.cuda.synchronize()
            g = Gd.cpu().numpy().view(np.uint32)
            o = Od[:no].cpu().numpy().view(np.uint32)
            ok = (hashlib.sha256(g.tobytes()).hexdigest() == h["G_sha256"]
                  and hashlib.sha256(o.tobytes()).hexdigest() == h["O_sha256"] and no == h["no"])
            parity = "bit-exact vs reference (sha256 G,O)" if ok else "MISMATCH"
    except Exception as exc:  # pragma: no cover
        parity = f"unchecked ({exc})"

    for _ in range(max(args.warmup, 3)):
        step_graph()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        ev0.record(stream)
        for _ in range(args.steps):
            step_graph()
        ev1.record(stream)
        torch.cuda.synchronize()
    if b.build_wait() != no:
        raise SystemExit("sync-free build exceeded its capacity")
        if world > 1:
            torch.distributed.barrier()
    ms = ev0.elapsed_time(ev1) / args.steps
    if world > 1:
        t = torch.tensor([ms], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())

    # per-kernel CUDA-event breakdown over the same steps (phase events inside the C ABI)
    phases = np.zeros(6)
    for _ in range(args.steps):
        phases += np.array(step(timed=True))
    phases /= args.steps
    k1_ms, k2_ms, sort_ms, k4_ms = phases[0], phases[2], phases[3], phases[5]
    key_bits = int(ncells - 1).bit_length()
    npasses = (key_bits + 8) // 9        # 9-bit digits (make_plan in pgrid.cu)
    pass_ms = sort_ms / max(npasses, 1)

    # per-kernel device time: events after every launch (pg_kernel_timing) over a few
    # synchronous builds on the launching stream; mean duration per launch of each kernel
    _native.kernel_timing(True)
    per = {}
    kt_builds = 5
    for _ in range(kt_builds):
        step(timed=False)
        torch.cuda.synchronize()
        for name, us in _native.kernel_times():
            if not name.startswith("("):
                per.setdefault(name, []).append(us * 1e-3)
    _native.kernel_timing(False)
    ktime = {k: {"ms_per_launch": float(np.mean(v)), "launches": len(v) // kt_builds,
                 "ms_per_build": float(np.sum(v)) / kt_builds} for k, v in per.items()}

    # end to end through the public API: pinned host inputs, H2D + build + D2H every step.
    # BuildPipeline overlaps build i's sort and G/O read-back with build i+1's input copy.
    e2e_steps = args.e2e_steps or max(args.steps, 10)   # amortises the 2-deep pipeline's drain
    Vh = np.ascontiguousarray(V).copy()
    Th = np.ascontiguousarray(T).copy()
    _native.host_register(Vh)
    _native.host_register(Th)
    from paper_2403_10647_b200.gridcore import TriangleMesh
    hmesh = TriangleMesh(Vh, Th)
    grid, rep = builders.build_parallel(hmesh, spec, device=local)
    seq_t = []
    for _ in range(min(e2e_steps, 3)):
        t0 = time.perf_counter()
        grid, rep = builders.build_parallel(hmesh, spec, device=local)
        seq_t.append(time.perf_counter() - t0)
    pipe = builders.BuildPipeline(local, depth=2)
    e2e_parity = True

    def pipe_run(steps):
        ok = True
        last = None
        for i in range(steps):
            if len(pipe) == 2:
                last, _ = pipe.result()
                ok &= int(last.G[-1]) == no
            pipe.submit(hmesh, spec)
            last = None           # drop the host grid so its pinned blocks recycle
        while len(pipe):
            last, _ = pipe.result()
            ok &= int(last.G[-1]) == no
        return ok, last

    pipe_run(4)                   # warm: workspaces and the pinned output pool
    t0 = time.perf_counter()
    e2e_parity, g = pipe_run(e2e_steps)
    e2e_sec = (time.perf_counter() - t0) / e2e_steps
    e2e_parity &= hashlib.sha256(g.G.tobytes()).hexdigest() == hashlib.sha256(grid.G.tobytes()).hexdigest()
    e2e_parity &= hashlib.sha256(g.O.tobytes()).hexdigest() == hashlib.sha256(grid.O.tobytes()).hexdigest()
    _native.host_unregister(Vh)
    _native.host_unregister(Th)

    peak, peak_kind = peaks()
    B = 12 * n + 24 * nv + 4 * (ncells + 1) + 4 * no          # SURVEY §8d compulsory bytes
    def kt(name):
        return ktime.get(name, {"ms_per_launch": 0.0, "launches": 0, "ms_per_build": 0.0})
    # algorithmic bytes per launch: K1 reads T and V, writes a 16-byte record per
    # triangle; K2 reads the records and writes the (cell, object) pairs; every radix scatter
    # reads and writes 8 bytes per pair; K4 reads the sorted cells and writes G
    kern = {
        "k_boxes_count": {"alg_bytes": 12 * n + 24 * nv + 16 * n},
        "k_pairs_emit": {"alg_bytes": 16 * n + 8 * no},
        ("k_radix_scatter_wc" if "k_radix_scatter_wc" in ktime else "k_radix_scatter"): {"alg_bytes": 16 * no},
        "k_cell_offsets": {"alg_bytes": 4 * no + 4 * (ncells + 1)},
    }
    for k, v in kern.items():
        t = kt(k)
        v.update(ms=t["ms_per_launch"], launches=t["launches"], ms_per_build=t["ms_per_build"])
        v["gbs"] = v["alg_bytes"] / (v["ms"] * 1e-3) / 1e9 if v["ms"] > 0 else None
        v["frac"] = v["gbs"] / peak if v["gbs"] else None
    glue = {k: round(v["ms_per_build"] * 1e3, 2) for k, v in ktime.items() if k not in kern}
    dom = max(kern, key=lambda k: kern[k]["ms_per_build"])
    traffic = traffic_table().get(dom)
    value = world / (ms * 1e-3)
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "builds/s", "n_gpus": world,
        "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": round(ms, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64+u32",
        "data": "synthetic",
        "config": {"workload": args.config, "scene": scenes.CONFIGS[args.config][0],
                   "triangles": n, "dims": list(spec.dims), "ncells": ncells, "no": no,
                   "key_bits": key_bits, "parallelism": f"replicas{world}" if world > 1 else "single",
                   "l2": "inputs larger than L2 (%.0f MB read per build)" % ((12 * n + 24 * nv) / 1e6),
                   "parity": parity},
        "mpairs_per_s": round(no / (ms * 1e-3) / 1e6 * world, 2),
        "hbm": {"compulsory_bytes": B, "achieved_gbs": round(B / (ms * 1e-3) / 1e9, 1),
                "frac_of_peak": round(B / (ms * 1e-3) / 1e9 / peak, 4), "peak_gbs": peak,
                "peak_kind": peak_kind},
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": round(kern[dom]["gbs"], 1),
                     "peak": peak, "unit": "GB/s", "frac": round(kern[dom]["frac"], 4),
                     "traffic": traffic, "alg_bytes_per_launch": kern[dom]["alg_bytes"],
                     "launch_ms": round(kern[dom]["ms"], 4), "peak_kind": peak_kind},
        "kernels": {k: {kk: (round(vv, 4) if isinstance(vv, float) else vv) for kk, vv in v.items()}
                    for k, v in kern.items()},
        "glue_us_per_build": glue,
        "e2e": {"value": round(1.0 / e2e_sec * world, 3), "unit": "builds/s",
                "h2d_bytes_per_step": int(Vh.nbytes + Th.nbytes),
                "d2h_bytes_per_step": int(grid.G.nbytes + 4 * max(pipe.capacity or 0, len(grid.O))),
                "ms_per_step": round(e2e_sec * 1e3, 2),
                "api": "builders.BuildPipeline (2 slots, no host round trip per build: build i+1's H2D follows build i's at once; O read back at the pipeline's pair capacity)",
                "parity": "bit-exact vs build_parallel" if e2e_parity else "MISMATCH",
                "sequential_build_parallel_ms": round(statistics.median(seq_t) * 1e3, 2)},
        "gpu_launches": launches * args.steps,
        "clocks": clk.summary(),
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args, mesh, spec)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
