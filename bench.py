"""Benchmark of the B200 parallel grid build (BASELINE.json metric on its headline config).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg3] [--impl reference]

A "step" is one full build_parallel of the config's scene (default cfg3: the 10M-triangle
architectural scene, density 4, 342^3 cells -- BASELINE.json configs[2], the paper's 25 Hz
case). `value` = builds/s with inputs resident in HBM (device pointers through the C ABI);
`e2e` = the same through the public numpy API (pinned host inputs, H2D + build + D2H of G
and O inside the timed region; the single drop-in call with pageable numpy inputs is
reported beside it). Rank 0 prints one JSON line.

N > 1: `--gpus N` launches N ranks itself (torchrun, one process per GPU, 127.0.0.1) unless
it already runs under torchrun (WORLD_SIZE set; it must equal N). The sharded build of
SURVEY.md §8e: each rank generates and counts its triangle shard, pairs are routed to cell
slabs (peer stores into symmetric memory, or one NCCL all-to-all), every rank sorts its slab
and writes its G/O slice (distributed output).
  * cfg1..cfg4 (default cfg3): weak scaling, an N x 10M-triangle scene (10M per GPU);
    `value` = N x builds/s of it, i.e. 10M-scene builds/s, the unit of the N=1 line.
  * cfg5 / cfg5a (100M uniform / arch, BASELINE configs[4]): strong scaling, one 100M scene
    split N ways; `value` = builds/s of the whole scene.
`--dry-run` (CPU, gloo): the sharded orchestration with the numpy test ops on a small scene
-- proves the launcher and the N-rank plumbing without a GPU; no measurement.
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
    ap.add_argument("--dry-run", action="store_true",
                    help="CPU only: N gloo ranks run the sharded orchestration (numpy test ops), no timing")
    return ap.parse_args()


def free_port():
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def self_launch(args):
    """--gpus N outside torchrun: re-run this command as N ranks (one process per GPU) under
    torch.distributed.run on 127.0.0.1; returns its exit code. Fails loudly when fewer than N
    devices are visible."""
    if not args.dry_run and args.impl != "reference":
        import torch
        have = torch.cuda.device_count()
        if have < args.gpus:
            raise SystemExit(f"bench.py --gpus {args.gpus}: only {have} CUDA device(s) visible")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), os.path.abspath(__file__)] + sys.argv[1:]
    print(f"[bench] launching {args.gpus} ranks: {' '.join(cmd[1:6])} ...", file=sys.stderr, flush=True)
    return subprocess.call(cmd)


def config_dict(config, kind, n, spec, no):
    """The workload keys every arm reports identically (the driver compares the arms)."""
    return {"workload": config, "scene": kind, "triangles": int(n), "dims": [int(d) for d in spec.dims],
            "ncells": int(spec.ncells), "no": int(no), "key_bits": int(spec.ncells - 1).bit_length()}


def sharded_config(config, world, kind, n, spec, no):
    d = config_dict(config, kind, n, spec, no)
    strong = sharded_mode(config, world)[0]
    d["workload"] = (f"{config} split x{world} (sharded, strong scaling)" if strong else
                     f"{config} x{world} (sharded, weak scaling: {world} x 10M triangles)")
    return d


def sharded_mode(config, world):
    """(strong, triangles of the whole scene, triangles per rank) of a sharded run."""
    from paper_2403_10647_b200 import scenes
    n1 = scenes.CONFIGS[config][1]
    strong = n1 >= 50_000_000            # config 5: one 100M scene split N ways
    n = n1 if strong else n1 * world
    return strong, n, n // world


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
    # config 5 (100M triangles): the reference needs ~40 GB of int64 temporaries and minutes
    # per build; its C restatement (the oracle port, one thread) stands in there
    if ref is not None and mesh.ntriangles <= 20_000_000:
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
            "config": (config_dict(args.config, scenes.CONFIGS[args.config][0], mesh.ntriangles, spec, no)
                       if world == 1 else
                       sharded_config(args.config, world, scenes.CONFIGS[args.config][0], mesh.ntriangles, spec,
                                      no)),
            "run": {"parallelism": f"CPU, {cores} host thread(s)",
                    "note": ("" if world == 1 else
                             "the reference times one scene of the config on rank 0's host; builds/s of it "
                             "is the unit of the GPU arm's value")},
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
    if ref is not None and mesh.ntriangles <= 20_000_000:
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

    kind, _, seed, density = scenes.CONFIGS[args.config]
    if kind not in ("arch", "uniform"):
        raise SystemExit("sharded bench supports the arch and uniform configs")
    strong, n, n1 = sharded_mode(args.config, world)
    lo, hi = D.shard_range(n, rank, world)
    shard = scenes.gen_shard(kind, n, seed, density, lo, hi)
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
        if not _native.features() & _native.PG_FEATURE_FUSED_DISPATCH:
            raise SystemExit("--fused-dispatch needs libpgrid built with -DPGRID_FUSED_DISPATCH=1")
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
    sc_name = "k_radix_scatter"
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
    # whole-job throughput in the metric's unit. Weak scaling (10M per GPU): 10M-triangle-scene
    # builds per second = N x builds/s of the N x 10M scene, so efficiency is value(N) / (N
    # value(1)). Strong scaling (config 5): builds/s of the one 100M scene.
    value = 1e3 / ms if strong else world * 1e3 / ms
    value_def = (f"builds/s of the {n // 1_000_000}M-triangle scene split {world} ways" if strong else
                 f"{world} x builds/s of the {world} x {n1 // 1_000_000}M-triangle scene")
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "builds/s", "n_gpus": world,
        "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": round(ms, 4),
        "higher_is_better": True, "scaling": "strong" if strong else "weak", "vs_baseline": None,
        "dtype": "f64+u32", "data": "synthetic",
        "config": sharded_config(args.config, world, kind, n, spec, no),
        "run": {"triangles_per_gpu": n1, "parallelism": f"triangle shards x{world} -> cell slabs",
                "exchange": exchange_desc, "output": "distributed (each rank its G/O slab)",
                "value_def": value_def, "scene_builds_per_s": round(1e3 / ms, 3),
                "parity": "orchestration verified by tests/test_distributed.py + test_gpu_distributed.py"},
        "mpairs_per_s": round(no / (ms * 1e-3) / 1e6, 2),
        "roofline": roofline,
        "kernels_rank0": kernels,
        "e2e": {"value": round((1.0 if strong else world) / e2e_sec, 3), "unit": "builds/s",
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


def run_dry(args, world, rank):
    """--dry-run: the N-rank plumbing on CPU. Every rank runs the sharded orchestration over
    gloo with the numpy per-rank steps of the tests (tests/np_ops.py, test infrastructure)
    on a small scene; rank 0 checks the gathered grid against the C oracle and prints one
    line. Nothing is timed; `value` is null."""
    import torch.distributed as dist
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", str(free_port()))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sys.path[:0] = [os.path.join(ROOT, "tests"), os.path.join(ROOT, "oracle")]
        import oracle
        from np_ops import NumpyOps
        from paper_2403_10647_b200 import distributed as D
        from paper_2403_10647_b200 import gen_scene, spec_for_mesh
        mesh = gen_scene("walls", 3000, 5)
        spec = spec_for_mesh(mesh, dims=(40, 30, 20))
        lo, hi = D.shard_range(mesh.ntriangles, rank, world)
        comm = D.TorchComm()
        res = D.build_sharded(NumpyOps(), comm, mesh.vertices, mesh.triangles[lo:hi], lo, spec)
        print(f"[bench] rank {comm.rank}/{comm.world} (gloo): shard [{lo}, {hi})", file=sys.stderr, flush=True)
        if rank == 0:
            G, O = oracle.build_parallel(mesh.vertices, mesh.triangles, spec)
            ok = np.array_equal(res[0], G) and np.array_equal(res[1], O)
            line = {"metric": METRIC, "value": None, "unit": "builds/s", "n_gpus": world, "steps": 0,
                    "warmup": 0, "dry_run": True, "higher_is_better": True,
                    "scaling": "strong" if sharded_mode(args.config, world)[0] else "weak",
                    "config": {"workload": "dry run: walls 3000 triangles, dims (40, 30, 20)",
                               "parallelism": f"triangle shards x{world} -> cell slabs (gloo, numpy test ops)"},
                    "parity": "bit-exact vs the C oracle" if ok else "MISMATCH"}
            print(json.dumps(line), flush=True)
            if not ok:
                raise SystemExit(1)
        dist.barrier()
    finally:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        raise SystemExit(self_launch(args))
    world, rank, local = dist_env()
    if "WORLD_SIZE" in os.environ and args.gpus not in (1, world):
        raise SystemExit(f"bench.py --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.dry_run:
        run_dry(args, world, rank)
        return
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
        # one line per rank on stderr: the communicator really spans `world` ranks / GPUs
        print(f"[bench] rank {dist.get_rank()}/{dist.get_world_size()}: NCCL "
              f"{'.'.join(map(str, torch.cuda.nccl.version()))} communicator on cuda:{local} "
              f"({torch.cuda.get_device_name(local)})", file=sys.stderr, flush=True)
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

    # a soup's index array (T[i][k] = 3i + k, checked exactly by the C ABI) is not transferred
    soup = bool(n >= (1 << 16) and nv >= 3 * n and
                np.array_equal(Th.reshape(-1), np.arange(3 * n, dtype=np.int32)))
    h2d_bytes = int(Vh.nbytes + (0 if soup else Th.nbytes))
    # the single call's copy bound: the same bytes moved alone (pinned H2D of V, T; D2H of
    # G, O), serialised as a build must (outputs exist only after the inputs)
    dbuf = torch.empty(Vh.nbytes + Th.nbytes, dtype=torch.uint8, device=dev)
    gh = _native.pinned_pool.empty(ncells + 1, np.uint32)
    oh = _native.pinned_pool.empty(no, np.uint32)
    cb = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        dbuf[:Vh.nbytes].copy_(torch.from_numpy(Vh.view(np.uint8).reshape(-1)), non_blocking=True)
        if not soup:
            dbuf[Vh.nbytes:].copy_(torch.from_numpy(Th.view(np.uint8).reshape(-1)), non_blocking=True)
        torch.from_numpy(gh.view(np.uint8)).copy_(dbuf[:gh.nbytes], non_blocking=True)
        torch.from_numpy(oh.view(np.uint8)).copy_(dbuf[gh.nbytes:gh.nbytes + oh.nbytes], non_blocking=True)
        e1.record(stream)
        torch.cuda.synchronize()
        cb.append(e0.elapsed_time(e1))
    copy_bound_ms = statistics.median(cb)
    del dbuf, gh, oh
    _native.host_unregister(Vh)
    _native.host_unregister(Th)
    # the drop-in call as a reference caller makes it: plain (pageable) numpy arrays, one
    # build_parallel per step, H2D + build + D2H inside (builders.py:144 contract)
    pmesh = TriangleMesh(np.ascontiguousarray(V).copy(), np.ascontiguousarray(T).copy())
    builders.build_parallel(pmesh, spec, device=local)
    page_t = []
    for _ in range(min(e2e_steps, 3)):
        t0 = time.perf_counter()
        gp, _ = builders.build_parallel(pmesh, spec, device=local)
        page_t.append(time.perf_counter() - t0)
    page_ok = np.array_equal(gp.G, grid.G) and np.array_equal(gp.O, grid.O)
    del pmesh, gp

    peak, peak_kind = peaks()
    B = 12 * n + 24 * nv + 4 * (ncells + 1) + 4 * no          # SURVEY §8d compulsory bytes
    def kt(name):
        return ktime.get(name, {"ms_per_launch": 0.0, "launches": 0, "ms_per_build": 0.0})
    # algorithmic bytes per launch: K1 reads T and V, writes a 16-byte record per
    # triangle; K2 reads the records and writes the (cell, object) pairs; every radix scatter
    # reads and writes 8 bytes per pair; K4L (k_bucket_sort, the MSD-first finish) reads the
    # bucket-sorted pairs and writes O and G; K4 (the classic finish, PGRID_LOCAL=0) reads the
    # sorted cells and writes G
    alg = {"k_boxes_count": 12 * n + 24 * nv + 16 * n, "k_pairs_emit": 16 * n + 8 * no,
           "k_radix_scatter": 16 * no, "k_bucket_sort": 12 * no + 4 * (ncells + 1),
           "k_cell_offsets": 4 * no + 4 * (ncells + 1)}
    kern = {k: {"alg_bytes": v} for k, v in alg.items() if k in ktime}
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
        "config": config_dict(args.config, scenes.CONFIGS[args.config][0], n, spec, no),
        "run": {"parallelism": "single GPU",
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
                "h2d_bytes_per_step": h2d_bytes,
                "h2d_note": ("V only: T is the implicit soup 0, 1, 2, ... (checked on the host, regenerated by K1)"
                             if soup else "V and T"),
                "d2h_bytes_per_step": int(grid.G.nbytes + 4 * max(pipe.capacity or 0, len(grid.O))),
                "ms_per_step": round(e2e_sec * 1e3, 2),
                "api": "builders.BuildPipeline (2 slots, no host round trip per build: build i+1's H2D follows build i's at once; O read back at the pipeline's pair capacity)",
                "parity": "bit-exact vs build_parallel" if e2e_parity else "MISMATCH",
                "sequential_build_parallel_ms": round(statistics.median(seq_t) * 1e3, 2),
                "single_call_copy_bound_ms": round(copy_bound_ms, 2),
                "pageable_build_parallel": {
                    "ms_per_step": round(statistics.median(page_t) * 1e3, 2),
                    "builds_per_s": round(1.0 / statistics.median(page_t), 3),
                    "what": "one drop-in build_parallel per step on plain (pageable) numpy arrays",
                    "parity": "bit-exact vs build_parallel" if page_ok else "MISMATCH"}},
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
