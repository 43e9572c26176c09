"""Sharded build across GPUs: triangle shards -> cell slabs -> one all-to-all.

Every rank r of P owns the contiguous triangle shard [r*N/P, (r+1)*N/P) and runs the count
and pair-expansion kernels on it. A coarse cell-id histogram (all-reduce) cuts the cell range
into P slabs of about NO/P pairs. Each rank stably partitions its pairs by slab and one
variable-size all-to-all routes them to the slab owners. all_to_all delivers the chunks in
source-rank order and the shards are ascending triangle ranges, so a rank's received pairs
are in global object-major order: the local stable radix sort by cell then reproduces the
reference's order exactly (`builders.py:123-125`, ascending object ids per cell). Each
slab's G is rebased by the exclusive scan of the slab pair totals; the global G and O are
the slab-ordered concatenations.

The orchestration is written against two small interfaces so the same code runs
  * on GPUs: `CudaOps` (libpgrid kernels on this rank's device) + `TorchComm` (NCCL), and
  * in tests: any ops object with the same methods + `TorchComm` over gloo, or
    `run_emulated` (every rank's phases executed in sequence in one process).
"""

from dataclasses import dataclass

import numpy as np

from . import _native
from .errors import InvariantError, SizeError

COARSE_BITS = 12       # slab cuts at 2^12-bucket granularity of the cell-id range
MAX_SLABS = 16         # pg_partition's digit table limit
CTL_HIST = 1 << COARSE_BITS   # words per rank slot of the exchange control buffer (histograms)
CTL_CNT = 32                  # words per rank slot: slab counts [0, 16), the rank's NO [16, 18), K1 flags [18]
MAX_IDS = (1 << 32) - 1       # gridcore.py:11
MAX_SCAN = 1 << 30            # primitives.py:17


def count_verdict(stats, ncells):
    """The reference's verdict for the WHOLE mesh from the shards' count statistics summed
    over the ranks (pg_count_stats: NO, index out of range, inverted boxes with negative /
    zero / positive counts, positive ones with a cell outside the grid). Raised identically
    on every rank, in the reference's order: the mesh's index check (geometry.py:41-43);
    exclusive_sum's non-negativity (primitives.py:22-25); NO > 2^32-1 (builders.py:99-100);
    mark_boundaries' zero-count group, i.e. a zero count next to any other kept triangle --
    every kept non-inverted box counts >= 1, so that is NO > 0 or a second zero
    (primitives.py:66-72); NO > 2^30 (inclusive_sum, primitives.py:29-31); the radix sort /
    scatter range checks on the inverted boxes' cells (primitives.py:102-111, 135-136); the
    G scan's ncells > 2^30 (builders.py:130). Returns the global NO."""
    no, oob, neg, zero, pos, bad = (int(x) for x in np.asarray(stats, dtype=np.int64)[:6])
    if oob:
        raise InvariantError("triangle index out of range")
    if neg:
        raise InvariantError("index arrays are non-negative (inverted cell box, negative count)")
    if no > MAX_IDS:
        raise SizeError(f"{no} cell/object pairs exceed 32-bit id space")
    if zero and (zero >= 2 or no > 0):
        raise InvariantError("coincident boundary marks (zero-count group?)")
    if no > MAX_SCAN:
        raise SizeError(f"array of {no} elements exceeds the scan size limit")
    if bad:
        raise InvariantError("cell of an inverted box outside [0, ncells)")
    if ncells > MAX_SCAN:
        raise SizeError(f"array of {ncells} elements exceeds the scan size limit")
    return no


@dataclass
class SlabPlan:
    shift: int                 # bucket = cell >> shift
    nbuckets: int
    cuts: np.ndarray           # int64[P+1] bucket boundaries of the slabs
    cell_lo: np.ndarray        # int64[P] first cell of each slab
    cell_hi: np.ndarray        # int64[P] one past the last cell
    pair_base: np.ndarray      # int64[P+1] exclusive scan of the slab pair totals
    table: np.ndarray          # uint32[nbuckets] slab id of every bucket


def coarse_shift(ncells):
    key_bits = int(ncells - 1).bit_length()
    return max(0, key_bits - COARSE_BITS)


def plan_slabs(hist, ncells, nslabs):
    """Balanced slab cuts from the global coarse histogram (identical on every rank)."""
    hist = np.asarray(hist, dtype=np.int64)
    shift = coarse_shift(ncells)
    nb = len(hist)
    total = int(hist.sum())
    cum = np.concatenate([[0], np.cumsum(hist)])          # pairs before bucket b
    cuts = np.zeros(nslabs + 1, dtype=np.int64)
    for s in range(1, nslabs):
        # first bucket whose start has at least s/P of the pairs before it
        cuts[s] = max(cuts[s - 1], int(np.searchsorted(cum, (s * total + nslabs - 1) // nslabs)))
        cuts[s] = min(cuts[s], nb)
    cuts[nslabs] = nb
    cell_lo = np.minimum(cuts[:-1] << shift, ncells)
    cell_hi = np.minimum(cuts[1:] << shift, ncells)
    pair_base = cum[cuts]
    table = np.zeros(nb, dtype=np.uint32)
    for s in range(nslabs):
        table[cuts[s]:cuts[s + 1]] = s
    return SlabPlan(shift, nb, cuts, cell_lo, cell_hi, pair_base, table)


def shard_range(n, rank, world):
    return (n * rank) // world, (n * (rank + 1)) // world


def assemble(slabs, ncells):
    """Global (G, O) from the slab results [(pair_base, G_rel, O)] in slab order."""
    G = np.empty(ncells + 1, dtype=np.uint32)
    parts = []
    pos = 0
    for base, g_rel, o in slabs:
        k = len(g_rel) - 1
        G[pos:pos + k] = np.asarray(g_rel[:-1], dtype=np.int64) + base
        pos += k
        parts.append(np.asarray(o, dtype=np.uint32))
    O = np.concatenate(parts) if parts else np.zeros(0, np.uint32)
    G[ncells] = len(O)
    assert pos == ncells
    return G, O


class ShardState:
    """Per-rank state of one sharded build, advanced phase by phase."""

    def __init__(self, ops, V, T, tri_base, spec, rank, world):
        self.ops, self.rank, self.world = ops, rank, world
        self.spec = spec
        self.ncells = int(spec.dims[0]) * int(spec.dims[1]) * int(spec.dims[2])
        self.V, self.T, self.tri_base = V, T, tri_base

    def phase_count(self, capacity=None, comm=None):
        """K1 + K2 on the shard; returns the local coarse histogram (computed by K2). With a
        pair capacity (ops with PG_DEFER), no host round trip: NO stays on the device and the
        pair buffers hold `capacity` pairs. Otherwise the shards' count statistics are summed
        over `comm` and the whole mesh's verdict is raised on every rank before any pair
        exists (count_verdict)."""
        stats = self.phase_count_only(capacity)
        if stats is not None:
            count_verdict(comm.allreduce_sum(stats) if comm is not None else stats, self.ncells)
        return self.phase_pairs()

    def phase_count_only(self, capacity=None):
        """K1 alone: the shard's count statistics (None when deferred)."""
        self.deferred = bool(capacity) and hasattr(self.ops, "count_deferred")
        if self.deferred:
            self.no = self.ops.count_deferred(self.V, self.T, self.spec, capacity)
            return None
        stats = self.ops.count_stats(self.V, self.T, self.spec)
        self.no = int(stats[0])
        return stats

    def phase_pairs(self):
        """K2 on the counted shard; returns the local coarse histogram."""
        self.shift = coarse_shift(self.ncells)
        nb = ((self.ncells - 1) >> self.shift) + 1
        self.nb_coarse = nb
        self.keys, self.vals, hist = self.ops.pairs(self.no, self.tri_base, self.shift, nb)
        return hist

    def phase_count_fused(self, capacity=None, comm=None):
        """K1 + the coarse histogram from the cell boxes (no pairs yet: the fused dispatch
        expands them straight into the slab owners' buffers after the plan)."""
        self.deferred = bool(capacity)
        if self.deferred:
            self.no = self.ops.count_deferred(self.V, self.T, self.spec, capacity)
        else:
            stats = self.ops.count_stats(self.V, self.T, self.spec)
            total = comm.allreduce_sum(stats) if comm is not None else stats
            count_verdict(total, self.ncells)
            self.global_positive = int(total[4])
            self.no = int(stats[0])
        self.shift = coarse_shift(self.ncells)
        self.nb_coarse = ((self.ncells - 1) >> self.shift) + 1
        return self.ops.coarse_hist(self.shift, self.nb_coarse)

    def phase_pairs_send(self, matrix, dst_keys, dst_vals):
        """Fused dispatch: expand + partition + peer-store every pair (pg_pairs_send)."""
        m = np.asarray(matrix, dtype=np.int64)
        off = [int(m[:self.rank, s].sum()) for s in range(self.world)]
        self.ops.pairs_send(self.tri_base, self.table_d, self.shift, self.world, self.base_d, dst_keys, dst_vals, off)
        return int(m[:, self.rank].sum())

    def phase_plan_device(self, hists):
        """Slab plan on the device from every rank's coarse histogram (exchange buffer);
        partition tables stay on the device. The host learns the plan with the count matrix."""
        self.nb = ((self.ncells - 1) >> self.shift) + 1
        self.table_d, self.base_d, self.plan_d = self.ops.slab_plan(hists, self.world, self.nb, self.shift,
                                                                    self.ncells, self.world)
        return self.plan_d

    def set_plan(self, plan_arr):
        """Host copy of the device plan (cuts | cell_lo | cell_hi | pair_base) -> SlabPlan."""
        P = self.world
        a = np.asarray(plan_arr, dtype=np.int64)
        self.plan = SlabPlan(self.shift, self.nb, a[:P + 1], a[P + 1:2 * P + 1], a[2 * P + 1:3 * P + 1],
                             a[3 * P + 1:4 * P + 2], self.table_d)
        return self.plan

    def phase_partition_counts_device(self):
        """Fused exchange, step 1 with the device plan: slab upsweep; per-slab counts (device)."""
        self.send_counts = self.ops.partition_counts(self.keys, self.table_d, self.shift, self.world)
        return self.send_counts

    def phase_partition(self, plan):
        """Stable partition by slab; returns the per-slab send counts."""
        self.plan = plan
        base = plan.cell_lo.astype(np.uint32)
        self.kout, self.vout, counts = self.ops.partition(self.keys, self.vals, plan.table, plan.shift,
                                                          self.world, base)
        self.send_counts = counts
        return counts

    def phase_partition_counts(self, plan):
        """Fused exchange, step 1: the slab upsweep only; returns the per-slab send counts."""
        self.plan = plan
        self.send_counts = self.ops.partition_counts(self.keys, plan.table, plan.shift, self.world)
        return self.send_counts

    def phase_send(self, matrix, dst_keys, dst_vals):
        """Fused exchange, step 2: scatter every pair into its slab owner's receive buffer.
        matrix[r][s] = pairs rank r sends to slab s; this rank writes after the lower ranks."""
        m = np.asarray(matrix, dtype=np.int64)
        off = [int(m[:self.rank, s].sum()) for s in range(self.world)]
        base = getattr(self, "base_d", None)
        if base is None:
            base = self.plan.cell_lo.astype(np.uint32)
        self.ops.partition_send(self.keys, self.vals, self.plan.table, self.plan.shift, self.world, base,
                                dst_keys, dst_vals, off)
        return int(m[:, self.rank].sum())

    def phase_sort(self, krecv, vrecv):
        """Local stable sort of the received slab + its G (relative), O."""
        lo, hi = int(self.plan.cell_lo[self.rank]), int(self.plan.cell_hi[self.rank])
        n = self.ops.length(krecv)
        if hi == lo:
            return int(self.plan.pair_base[self.rank]), np.zeros(1, np.uint32), np.zeros(0, np.uint32)
        G, O = self.ops.sort_cells(krecv, vrecv, n, hi - lo)
        return int(self.plan.pair_base[self.rank]), G, O


def build_sharded(ops, comm, V, T, tri_base, spec, gather=True, exchange=None):
    """One rank's part of the sharded build (run on every rank of `comm`).

    exchange: a PeerExchange (fused partition + send into the slab owners' receive buffers,
    peer memory over NVLink) or None (partition pass, then NCCL all-to-all).
    Returns (G, O) on rank 0 when gather=True (None elsewhere); with gather=False each rank
    returns its slab as (cell_lo, cell_hi, pair_base, G_rel, O) with G_rel/O left where the
    ops keep them (device memory for CudaOps).

    Errors: the reference's verdicts (SizeError / InvariantError) are decided for the whole
    mesh from every shard's count statistics and raised on every rank at the same point
    (count_verdict), so no rank is left waiting in a collective. Any other failure on a rank
    (a CUDA error, ...) aborts the communicator, so the peers' collectives fail instead of
    hanging."""
    rank, world = comm.rank, comm.world
    if world > MAX_SLABS:
        raise ValueError(f"at most {MAX_SLABS} ranks")
    try:
        return _build_sharded(ops, comm, V, T, tri_base, spec, gather, exchange)
    except (InvariantError, SizeError):
        raise
    except Exception:
        comm.abort()
        raise


def _build_sharded(ops, comm, V, T, tri_base, spec, gather, exchange):
    rank, world = comm.rank, comm.world
    st = ShardState(ops, V, T, tri_base, spec, rank, world)
    fused = exchange is not None and getattr(exchange, "fused", False)
    force_host = False      # some shard flagged an error on a deferred count: decide on host counts
    if fused:
        # fused dispatch: K1, the coarse histogram from the cell boxes, peer-put histograms and
        # NOs, a device barrier, the device plan, ONE host read (histograms, NOs, plan), then a
        # single kernel expands every pair straight into its slab owner's receive buffer
        while True:
            cap = None if force_host else exchange.no_capacity
            hist = st.phase_count_fused(cap, comm)
            if not st.deferred and st.global_positive:
                # boxes inverted on two axes: their pairs are rewritten after a plain
                # expansion (pg_pairs); the fused kernel has no such step
                fused = False
                break
            exchange.put_hist(hist, rank)
            exchange.put_no(rank, ops)
            exchange.barrier()
            st.phase_plan_device(exchange.hists(st.nb_coarse))
            hists, nos, errs, plan_arr = exchange.read_hists(st.nb_coarse, st.plan_d)
            if cap and int(errs.max()):
                force_host = True
                continue
            exchange.no_capacity = int(nos.max() * 1.0625) + 4096
            if not cap or int(nos.max()) <= cap:
                break
    if fused:
        if st.deferred:
            st.no = ops.count_result()
        plan = st.set_plan(plan_arr)
        matrix = slab_matrix(hists, plan.cuts)
        assert st.no == int(nos[rank]) == int(hists[rank].sum()), (st.no, nos[rank], int(hists[rank].sum()))
        exchange.ensure(int(matrix.sum(axis=0).max()))
        dk, dv = exchange.destinations()
        nrecv = st.phase_pairs_send(matrix, dk, dv)
        exchange.barrier()
        krecv, vrecv = exchange.received(nrecv)
    elif exchange is not None:
        # histograms, plan and slab counts stay on the device: each rank puts its array into
        # every rank's exchange buffer (peer stores), a device barrier, then every rank reduces
        # / plans itself; the host reads the count matrix, every rank's NO and the plan once.
        # After the first build the pair count is not read back either (PG_DEFER): the pair
        # buffers are sized by a capacity all ranks agree on (1.25 x the largest NO seen), and
        # an overflow or a K1 error flag -- visible to every rank in the exchanged NOs and
        # flags -- repeats the build with the host-counted path (global verdict first).
        while True:
            cap = None if force_host else exchange.no_capacity
            hist = st.phase_count(cap, comm)
            exchange.put_hist(hist, rank)
            exchange.barrier()
            st.phase_plan_device(exchange.hists(st.nb_coarse))
            exchange.put_counts(st.phase_partition_counts_device(), rank, ops)
            exchange.barrier()
            matrix, nos, errs, plan_arr = exchange.read_counts(st.plan_d)
            if cap and int(errs.max()):
                force_host = True
                continue
            exchange.no_capacity = int(nos.max() * 1.25) + 4096
            if not cap or int(nos.max()) <= cap:
                break
        if st.deferred:
            st.no = ops.count_result()     # validation of the deferred count (errors raise here)
            assert st.no == int(nos[rank]) == int(matrix[rank].sum()), (st.no, nos, matrix)
        plan = st.set_plan(plan_arr)
        exchange.ensure(int(np.asarray(matrix, dtype=np.int64).sum(axis=0).max()))
        dk, dv = exchange.destinations()
        nrecv = st.phase_send(matrix, dk, dv)
        exchange.barrier()
        krecv, vrecv = exchange.received(nrecv)
    else:
        hist = comm.allreduce_sum(st.phase_count(None, comm))
        plan = plan_slabs(hist, st.ncells, world)
        send, recv = comm.alltoall_counts(st.phase_partition(plan))
        krecv, vrecv = comm.alltoall_pairs(st.kout, st.vout, send, recv, ops)
    base, G_rel, O = st.phase_sort(krecv, vrecv)
    if not gather:
        return int(plan.cell_lo[rank]), int(plan.cell_hi[rank]), base, G_rel, O
    if gather == "device":
        # the slabs travel to rank 0's GPU (NCCL point-to-point), G rebased there; rank 0
        # returns device tensors (G int32[ncells+1], O int32[NO] holding u32 bit patterns)
        return comm.gather_slabs_device(plan, st.ncells, G_rel, O)
    slabs = comm.gather_to_root((base, ops.to_numpy(G_rel), ops.to_numpy(O)))
    if rank != 0:
        return None
    return assemble(slabs, st.ncells)


class TorchComm:
    """Collectives over torch.distributed (NCCL on GPUs, gloo on CPU)."""

    def __init__(self, group=None, device=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.device = device

    def _t(self, arr):
        import torch
        t = torch.as_tensor(np.asarray(arr))
        return t.to(self.device) if self.device is not None else t

    def allreduce_sum(self, arr):
        """Sum over ranks; device tensors are reduced where they are (one host copy after)."""
        import torch
        t = arr if isinstance(arr, torch.Tensor) else self._t(arr)
        t = t.to(torch.int64)
        self.dist.all_reduce(t, group=self.group)
        return t.cpu().numpy()

    def alltoall_counts(self, send):
        """Exchange per-slab pair counts; returns (send, recv) as host lists (one host copy)."""
        import torch
        s = (send if isinstance(send, torch.Tensor) else self._t(np.asarray(send, dtype=np.int64)))
        s = s[:self.world].to(torch.int64)
        r = torch.empty_like(s)
        self.dist.all_to_all_single(r, s, group=self.group)
        both = torch.stack([s, r]).cpu().numpy()
        return [int(x) for x in both[0]], [int(x) for x in both[1]]

    def alltoall_pairs(self, keys, vals, send, recv, ops):
        if hasattr(ops, "recv_buffers"):
            kr, vr = ops.recv_buffers(sum(recv))
        else:
            kr, vr = ops.empty_pairs(sum(recv)), ops.empty_pairs(sum(recv))
        self.dist.all_to_all_single(kr, ops.as_tensor(keys), recv, send, group=self.group)
        self.dist.all_to_all_single(vr, ops.as_tensor(vals), recv, send, group=self.group)
        return kr, vr

    def gather_slabs_device(self, plan, ncells, G_rel, O):
        """Every rank's (G_rel, O) slab into one G / O on rank 0 (device tensors, sends in
        rank order); G rebased by the slab's pair base (u32 arithmetic on int32 bits)."""
        import torch
        rank, world = self.rank, self.world
        as_t = lambda a: a if isinstance(a, torch.Tensor) else torch.from_numpy(np.asarray(a, np.uint32).view(np.int32))
        G_rel, O = as_t(G_rel), as_t(O)
        lo, hi = plan.cell_lo.astype(np.int64), plan.cell_hi.astype(np.int64)
        base = plan.pair_base.astype(np.int64)
        if rank != 0:
            if hi[rank] > lo[rank]:
                self.dist.send(G_rel[:hi[rank] - lo[rank]].contiguous(), 0, group=self.group)
                if int(O.numel()):
                    self.dist.send(O.contiguous(), 0, group=self.group)
            return None
        dev = G_rel.device
        no = int(base[world])
        G = torch.empty(ncells + 1, dtype=torch.int32, device=dev)
        Oall = torch.empty(max(no, 1), dtype=torch.int32, device=dev)[:no]
        for r in range(world):
            k, n_r = int(hi[r] - lo[r]), int(base[r + 1] - base[r])
            if k == 0:
                continue
            g = G[lo[r]:hi[r]]
            o = Oall[base[r]:base[r + 1]]
            if r == 0:
                g.copy_(G_rel[:k])
                if n_r:
                    o.copy_(O[:n_r])
            else:
                self.dist.recv(g, r, group=self.group)
                if n_r:
                    self.dist.recv(o, r, group=self.group)
            if base[r]:
                g.add_(int(np.int64(base[r]).astype(np.uint32).view(np.int32)))   # wraps like u32
        G[ncells] = int(np.uint32(no).view(np.int32))
        return G, Oall

    def abort(self):
        """Abort the communicator after a local failure: peers blocked in a collective with
        this rank get an error instead of waiting forever (NCCL ncclCommAbort)."""
        try:
            from torch.distributed import distributed_c10d as c10d
            c10d._abort_process_group(self.group or c10d.GroupMember.WORLD)
        except Exception:
            try:
                self.dist.destroy_process_group(self.group)
            except Exception:
                pass

    def gather_to_root(self, obj):
        out = [None] * self.world if self.rank == 0 else None
        self.dist.gather_object(obj, out, dst=0, group=self.group)
        return out


class PeerExchange:
    """Receive buffers in symmetric memory (torch.distributed._symmetric_memory: every rank maps
    every other rank's buffer), so pg_partition_send writes pairs straight into the slab
    owner's GPU over NVLink -- the dispatch all-to-all fused into the partition kernel.
    Buffers grow collectively (every rank sees the same count matrix, so they agree on the
    capacity)."""

    def __init__(self, comm, device):
        import torch
        import torch.distributed._symmetric_memory as symm
        self.torch, self.symm, self.comm, self.dev = torch, symm, comm, device
        self.cap = 0
        self.buf = self.hdl = None
        self.ensure(1 << 20)
        # control buffer: every rank's coarse histogram (slot r of CTL_HIST words) and slab
        # counts (slot r of 16 words), written by the ranks themselves with peer stores
        w = comm.world
        group = comm.group or comm.dist.group.WORLD
        self.ctl = symm.empty(w * (CTL_HIST + CTL_CNT), dtype=torch.int32, device=device)
        self.ctl_hdl = symm.rendezvous(self.ctl, group)
        self.ctl_ptrs = [int(p) for p in self.ctl_hdl.buffer_ptrs]
        self._read_c = torch.empty(w * CTL_CNT, dtype=torch.int32).pin_memory()
        self._read_p = torch.empty(4 * w + 2, dtype=torch.int64).pin_memory()
        self._read_h = torch.empty(w * CTL_HIST, dtype=torch.int32).pin_memory()
        self.no_capacity = None      # pair capacity of deferred counts (set after the first build)
        # pg_pairs_send (expansion + dispatch in one kernel, look-back slab offsets): correct
        # but measured slower at world 1 (1.23 vs 1.09 ms/build: the coarse histogram from the
        # cell boxes re-reads every record, latency-bound, before the expansion can start); off
        self.fused = False

    def _stream(self):
        return self.torch.cuda.current_stream(self.dev).cuda_stream

    def put_hist(self, hist, rank):
        nb = int(hist.numel())
        _native.peer_put(hist, nb, self.ctl_ptrs, rank * nb, self._stream())

    def hists(self, nb):
        return self.ctl[:self.comm.world * nb]

    def put_counts(self, counts, rank, ops):
        w = self.comm.world
        _native.peer_put(counts, w, self.ctl_ptrs, w * CTL_HIST + rank * CTL_CNT, self._stream())
        ops.b.peer_put_count(self.ctl_ptrs, w * CTL_HIST + rank * CTL_CNT + 16, self._stream())

    def put_no(self, rank, ops):
        w = self.comm.world
        ops.b.peer_put_count(self.ctl_ptrs, w * CTL_HIST + rank * CTL_CNT + 16, self._stream())

    def read_hists(self, nb, plan_d):
        """Every rank's coarse histogram and NO, and the device plan: one host round trip."""
        torch, w = self.torch, self.comm.world
        self._read_h[:w * nb].copy_(self.ctl[:w * nb], non_blocking=True)
        self._read_c.copy_(self.ctl[w * CTL_HIST:w * (CTL_HIST + CTL_CNT)], non_blocking=True)
        self._read_p.copy_(plan_d, non_blocking=True)
        torch.cuda.current_stream(self.dev).synchronize()
        hists = self._read_h[:w * nb].numpy().view(np.uint32).reshape(w, nb).astype(np.int64)
        _, nos, errs = _split_counts(self._read_c.numpy(), w)
        return hists, nos, errs, self._read_p.numpy().copy()

    def read_counts(self, plan_d):
        """The count matrix [rank][slab], every rank's NO and the device plan: one host
        round trip (two small copies into page-locked memory, one synchronise)."""
        torch, w = self.torch, self.comm.world
        self._read_c.copy_(self.ctl[w * CTL_HIST:w * (CTL_HIST + CTL_CNT)], non_blocking=True)
        self._read_p.copy_(plan_d, non_blocking=True)
        torch.cuda.current_stream(self.dev).synchronize()
        return _split_counts(self._read_c.numpy(), w) + (self._read_p.numpy().copy(),)

    def allgather_counts(self, counts):
        """counts: this rank's per-slab send counts (device) -> host matrix [rank][slab]."""
        torch = self.torch
        w = self.comm.world
        c = counts[:w].to(torch.int64) if isinstance(counts, torch.Tensor) else torch.as_tensor(counts[:w])
        out = torch.empty(w * w, dtype=torch.int64, device=c.device)
        self.comm.dist.all_gather_into_tensor(out, c.contiguous(), group=self.comm.group)
        return out.view(w, w).cpu().numpy()

    def ensure(self, n):
        if n <= self.cap:
            return
        cap = (int(n * 1.25) + 1024 + 63) & ~63     # value half 256-byte aligned (vector loads)
        group = self.comm.group or self.comm.dist.group.WORLD
        self.buf = self.symm.empty(2 * cap, dtype=self.torch.int32, device=self.dev)
        self.hdl = self.symm.rendezvous(self.buf, group)
        self.cap = cap
        self.ptrs = [int(p) for p in self.hdl.buffer_ptrs]

    def destinations(self):
        return list(self.ptrs), [p + 4 * self.cap for p in self.ptrs]

    def barrier(self):
        self.hdl.barrier()

    def received(self, n):
        return self.buf[:n], self.buf[self.cap:self.cap + n]


class EmulatedExchange:
    """PeerExchange for run_emulated: every virtual rank's receive buffer lives on this device."""

    def __init__(self, torch, device, world):
        self.torch, self.dev, self.world = torch, device, world
        self.cap = 0
        self.ctl = [torch.zeros(world * (CTL_HIST + CTL_CNT), dtype=torch.int32, device=device)
                    for _ in range(world)]
        self.ctl_ptrs = [int(c.data_ptr()) for c in self.ctl]

    def put_hist(self, hist, rank):
        nb = int(hist.numel())
        _native.peer_put(hist, nb, self.ctl_ptrs, rank * nb, self.torch.cuda.current_stream(self.dev).cuda_stream)

    def hists(self, r, nb):
        return self.ctl[r][:self.world * nb]

    def put_counts(self, counts, rank, ops):
        w = self.world
        sp = self.torch.cuda.current_stream(self.dev).cuda_stream
        _native.peer_put(counts, w, self.ctl_ptrs, w * CTL_HIST + rank * CTL_CNT, sp)
        ops.b.peer_put_count(self.ctl_ptrs, w * CTL_HIST + rank * CTL_CNT + 16, sp)

    def put_no(self, rank, ops):
        w = self.world
        ops.b.peer_put_count(self.ctl_ptrs, w * CTL_HIST + rank * CTL_CNT + 16,
                             self.torch.cuda.current_stream(self.dev).cuda_stream)

    def read_hists(self, r, nb, plan_d):
        w = self.world
        h = self.ctl[r][:w * nb].cpu().numpy().view(np.uint32).reshape(w, nb).astype(np.int64)
        c = self.ctl[r][w * CTL_HIST:w * (CTL_HIST + CTL_CNT)].cpu().numpy()
        _, nos, errs = _split_counts(c, w)
        return h, nos, errs, plan_d.cpu().numpy()

    def read_counts(self, r, plan_d):
        w = self.world
        c = self.ctl[r][w * CTL_HIST:w * (CTL_HIST + CTL_CNT)].cpu().numpy()
        return _split_counts(c, w) + (plan_d.cpu().numpy(),)

    def ensure(self, n):
        if n > self.cap or not hasattr(self, "bufs"):   # (an all-dropped mesh still needs buffers)
            self.cap = (int(max(n, self.cap) * 1.25) + 1024 + 63) & ~63
            self.bufs = [self.torch.empty(2 * self.cap, dtype=self.torch.int32, device=self.dev)
                         for _ in range(self.world)]

    def destinations(self):
        ptrs = [int(b.data_ptr()) for b in self.bufs]
        return ptrs, [p + 4 * self.cap for p in ptrs]

    def received(self, r, n):
        return self.bufs[r][:n], self.bufs[r][self.cap:self.cap + n]


def slab_matrix(hists, cuts):
    """matrix[r][s] = pairs rank r sends to slab s, from the ranks' coarse histograms."""
    cum = np.concatenate([np.zeros((len(hists), 1), np.int64), np.cumsum(hists, axis=1)], axis=1)
    cuts = np.asarray(cuts, np.int64)
    return cum[:, cuts[1:]] - cum[:, cuts[:-1]]


def _split_counts(c, w):
    """Control-buffer count slots (int32 [w][CTL_CNT]) -> (matrix [rank][slab], NO per rank,
    K1 error flags per rank)."""
    c = np.asarray(c).view(np.uint32).reshape(w, CTL_CNT).astype(np.int64)
    return c[:, :w].copy(), c[:, 16] | (c[:, 17] << 32), c[:, 18].copy()


def run_emulated(make_ops, V, T, spec, world, exchange="copy", capacity=None):
    """Every rank's phases executed in sequence in one process (no inter-rank waiting):
    exercises the kernels and the orchestration of the sharded build on a single device.
    exchange="p2p": the fused exchange with the device plan; capacity: deferred counts with
    that pair capacity (returns None when some rank's pairs exceeded it)."""
    n = len(T)
    states = []
    for r in range(world):
        lo, hi = shard_range(n, r, world)
        states.append(ShardState(make_ops(), V, T[lo:hi], lo, spec, r, world))

    def counted(cap=None):
        """K1 on every virtual rank, the whole mesh's verdict, then K2 (as build_sharded)."""
        stats = [s.phase_count_only(cap) for s in states]
        if stats[0] is not None:
            count_verdict(np.sum(stats, axis=0), states[0].ncells)
        return [s.phase_pairs() for s in states]

    if exchange == "copy":
        hists = counted()
        hist = np.sum([s.ops.to_numpy(h).astype(np.int64) for s, h in zip(states, hists)], axis=0)
        plan = plan_slabs(hist, states[0].ncells, world)
    if exchange == "fused":     # expansion + dispatch in one kernel (pg_pairs_send; CudaOps only)
        ex = EmulatedExchange(states[0].ops.torch, states[0].ops.dev, world)
        hists = [s.phase_count_fused(capacity) for s in states]
        for r, s in enumerate(states):
            ex.put_hist(hists[r], r)
            ex.put_no(r, s.ops)
        for r, s in enumerate(states):
            s.phase_plan_device(ex.hists(r, s.nb_coarse))
        for r, s in enumerate(states):
            h, nos, errs, plan_arr = ex.read_hists(r, s.nb_coarse, s.plan_d)
            if capacity and int(nos.max()) > capacity:
                return None
            if s.deferred:
                s.no = s.ops.count_result()
            assert int(nos[r]) == int(h[r].sum()) == s.no
            s.set_plan(plan_arr)
        # the histograms from the cell boxes equal K2's (pg_pairs) coarse histograms
        matrix = slab_matrix(h, states[0].plan.cuts)
        ex.ensure(int(matrix.sum(axis=0).max()))
        dk, dv = ex.destinations()
        nrecv = [s.phase_pairs_send(matrix, dk, dv) for s in states]
        states[0].ops.torch.cuda.synchronize()
        slabs = []
        for r, s in enumerate(states):
            base, G_rel, O = s.phase_sort(*ex.received(r, nrecv[r]))
            slabs.append((base, s.ops.to_numpy(G_rel), s.ops.to_numpy(O)))
        return assemble(slabs, states[0].ncells)
    if exchange == "p2p":       # fused partition + send into the owners' buffers (CudaOps only)
        # as build_sharded with a PeerExchange: histograms, plan and counts through the
        # (emulated) peer buffers, slab plans computed on the device by every rank
        ex = EmulatedExchange(states[0].ops.torch, states[0].ops.dev, world)
        hists = counted(capacity)
        for r, s in enumerate(states):
            ex.put_hist(hists[r], r)
        for r, s in enumerate(states):
            s.phase_plan_device(ex.hists(r, s.nb_coarse))
        for r, s in enumerate(states):
            ex.put_counts(s.phase_partition_counts_device(), r, s.ops)
        plans = []
        for r, s in enumerate(states):
            matrix, nos, errs, plan_arr = ex.read_counts(r, s.plan_d)
            if capacity and int(nos.max()) > capacity:
                assert all(s2.ops.b.count_result() < 0 for s2, n2 in zip(states, nos) if n2 > capacity)
                return None
            if s.deferred:
                s.no = s.ops.count_result()
            assert int(nos[r]) == int(matrix[r].sum()) == s.no
            plans.append(s.set_plan(plan_arr))
        host = plan_slabs(np.sum([s.ops.to_numpy(h).astype(np.int64) for s, h in zip(states, hists)], axis=0),
                          states[0].ncells, world)
        for p in plans:              # the device plan is plan_slabs bit for bit
            for f in ("cuts", "cell_lo", "cell_hi", "pair_base"):
                assert np.array_equal(getattr(p, f), getattr(host, f)), f
            assert np.array_equal(states[0].ops.to_numpy(p.table)[:host.nbuckets], host.table)
        ex.ensure(int(matrix.sum(axis=0).max()))
        dk, dv = ex.destinations()
        nrecv = [s.phase_send(matrix, dk, dv) for s in states]
        states[0].ops.torch.cuda.synchronize()
        slabs = []
        for r, s in enumerate(states):
            base, G_rel, O = s.phase_sort(*ex.received(r, nrecv[r]))
            slabs.append((base, s.ops.to_numpy(G_rel), s.ops.to_numpy(O)))
        return assemble(slabs, states[0].ncells)
    sends = [[int(x) for x in s.ops.to_numpy(s.phase_partition(plan))[:world]] for s in states]
    slabs = []
    for r, s in enumerate(states):
        ops = s.ops
        ks, vs = [], []
        for q, src in enumerate(states):       # source-rank order, like all_to_all
            off = int(np.sum(sends[q][:r]))
            ks.append(ops.slice(src.kout, off, sends[q][r]))
            vs.append(ops.slice(src.vout, off, sends[q][r]))
        krecv, vrecv = ops.concat(ks), ops.concat(vs)
        base, G_rel, O = s.phase_sort(krecv, vrecv)
        slabs.append((base, ops.to_numpy(G_rel), ops.to_numpy(O)))
    return assemble(slabs, states[0].ncells)


class CudaOps:
    """Per-rank device steps on this rank's GPU: libpgrid kernels on torch-allocated memory.

    Buffers are grow-only and reused across builds (named slots), so a steady-state sharded
    build allocates nothing -- cudaMalloc inside the step would serialise the device."""

    def __init__(self, device=0, stream=None):
        import torch

        from . import _native
        self.torch = torch
        self.dev = torch.device("cuda", device)
        self.b = _native.Builder(device)
        self.stream = stream
        self._bufs = {}

    def _sp(self):
        s = self.stream or self.torch.cuda.current_stream(self.dev)
        return s.cuda_stream

    def _buf(self, name, n):
        t = self._bufs.get(name)
        if t is None or t.numel() < n:
            t = self.torch.empty(max(int(n * 1.25), 16), dtype=self.torch.int32, device=self.dev)
            self._bufs[name] = t
        return t[:n]

    def as_tensor(self, x):
        return x

    def empty_pairs(self, n, name=None):
        if name is None:
            return self.torch.empty(n, dtype=self.torch.int32, device=self.dev)
        return self._buf(name, n)

    def recv_buffers(self, n):
        return self._buf("recv_k", n), self._buf("recv_v", n)

    def length(self, x):
        return int(x.numel())

    def slice(self, x, off, n):
        return x[off:off + n]

    def concat(self, xs):
        return self.torch.cat(xs) if xs else self.empty_pairs(0)

    def to_numpy(self, x):
        """Device u32 tensor -> host array in page-locked memory (PCIe-rate copy)."""
        if not hasattr(x, "cpu"):
            return np.asarray(x, np.uint32)
        out = _native.pinned_pool.empty(int(x.numel()), np.uint32)
        if out.size:
            self.torch.from_numpy(out.view(np.int32)).copy_(x.view(self.torch.int32))
        return out

    def count(self, V, T, spec):
        torch = self.torch
        if not isinstance(V, torch.Tensor):
            # host mesh: the C ABI stages it (one H2D at PCIe rate from page-locked arrays)
            V = np.ascontiguousarray(V, dtype=np.float64).reshape(-1, 3)
            T = np.ascontiguousarray(T, dtype=np.int32).reshape(-1, 3)
            self._V, self._T = V, T
            return self.b.count(V, V.shape[0], T, T.shape[0], spec, _native.PG_HOST_INPUT, self._sp())
        self._V, self._T = V, T          # keep alive for the stream
        return self.b.count(V, V.shape[0], T, T.shape[0], spec, 0, self._sp())

    def count_stats(self, V, T, spec):
        """K1 with PG_STATS: the shard's raw count statistics (no local verdict)."""
        flags = 0
        if not isinstance(V, self.torch.Tensor):
            V = np.ascontiguousarray(V, dtype=np.float64).reshape(-1, 3)
            T = np.ascontiguousarray(T, dtype=np.int32).reshape(-1, 3)
            flags = _native.PG_HOST_INPUT
        self._V, self._T = V, T
        return self.b.count_stats(V, V.shape[0], T, T.shape[0], spec, flags, self._sp())

    def count_deferred(self, V, T, spec, capacity):
        """K1 without the NO read back (PG_DEFER)."""
        flags = 0
        if not isinstance(V, self.torch.Tensor):
            V = np.ascontiguousarray(V, dtype=np.float64).reshape(-1, 3)
            T = np.ascontiguousarray(T, dtype=np.int32).reshape(-1, 3)
            flags = _native.PG_HOST_INPUT
        self._V, self._T = V, T
        return self.b.count_deferred(V, V.shape[0], T, T.shape[0], spec, capacity, flags, self._sp())

    def coarse_hist(self, shift, nbuckets):
        hist = self._buf("coarse", nbuckets)
        self.b.coarse_hist(shift, nbuckets, hist, self._sp())
        return hist

    def pairs_send(self, tri_base, table, shift, nslabs, base, dst_keys, dst_vals, dst_offset):
        self._ptab, self._pbase = self._dev_u32(table), self._dev_u32(base)
        self.b.pairs_send(tri_base, self._ptab, shift, nslabs, self._pbase, dst_keys, dst_vals, dst_offset,
                          self._sp())

    def count_result(self):
        no = self.b.count_result()
        if no < 0:
            raise RuntimeError(f"deferred pair count void (NO {-no - 1} over the capacity, or an inverted box)")
        return no

    def pairs(self, no, tri_base, shift, nbuckets):
        k, v = self._buf("pair_k", no), self._buf("pair_v", no)
        hist = self._buf("coarse", nbuckets)
        self.b.pairs(k, v, tri_base, shift, nbuckets, hist, self._sp())
        return k, v, hist.view(self.torch.int32)

    def partition(self, keys, vals, table, shift, nslabs, base):
        torch = self.torch
        n = int(keys.numel())
        dt = torch.from_numpy(np.asarray(table, np.uint32).view(np.int32)).to(self.dev)
        db = torch.from_numpy(np.asarray(base, np.uint32).view(np.int32)).to(self.dev)
        self._tables = (dt, db)
        ko, vo = self._buf("part_k", n), self._buf("part_v", n)
        counts = self._buf("slab_counts", 16)
        self.b.partition(keys, vals, n, dt, shift, nslabs, db, ko, vo, counts, self._sp())
        return ko, vo, counts

    def slab_plan(self, hists, nranks, nbuckets, shift, ncells, nslabs):
        table = self._buf("slab_table", nbuckets)
        base = self._buf("slab_base", nslabs)
        plan = self._bufs.get("slab_plan")
        if plan is None or plan.numel() < 4 * nslabs + 2:
            plan = self.torch.empty(4 * MAX_SLABS + 2, dtype=self.torch.int64, device=self.dev)
            self._bufs["slab_plan"] = plan
        plan = plan[:4 * nslabs + 2]
        _native.slab_plan(hists, nranks, nbuckets, shift, ncells, nslabs, table, base, plan, self._sp())
        return table, base, plan

    def _dev_u32(self, a):
        if isinstance(a, self.torch.Tensor):
            return a
        return self.torch.from_numpy(np.asarray(a, np.uint32).view(np.int32)).to(self.dev)

    def partition_counts(self, keys, table, shift, nslabs):
        n = int(keys.numel())
        self._ptab = self._dev_u32(table)
        counts = self._buf("slab_counts", 16)
        self.b.partition_counts(keys, n, self._ptab, shift, nslabs, counts, self._sp())
        return counts

    def partition_send(self, keys, vals, table, shift, nslabs, base, dst_keys, dst_vals, dst_offset):
        n = int(keys.numel())
        self._pbase = self._dev_u32(base)
        self.b.partition_send(keys, vals, n, self._ptab, shift, nslabs, self._pbase, dst_keys, dst_vals,
                              dst_offset, self._sp())

    def sort_cells(self, keys, vals, n, ncells, gen_order=True):
        G = self._buf("G", ncells + 1)
        O = self._buf("O", n)
        # the received slab is in generation order (stable partition, rank-ordered receive):
        # the MSD-first finish may rank a cell's pairs by triangle id
        self.b.sort_cells(keys, vals, n, ncells, G, O, self._sp(),
                          flags=_native.PG_GEN_ORDER if gen_order else 0)
        return G, O
