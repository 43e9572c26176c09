"""The sharded build's CUDA per-rank ops across REAL processes: two and three ranks (one
process each) share the one GPU of this box, exchanging through gloo with the tensors staged
through host memory (the NCCL-style copy exchange: every collective is host-mediated, so no
rank's kernel ever waits on another rank's). Bit-exact against the oracle; the whole-mesh
verdicts raise the same class on every rank."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2403_10647_b200 import distributed as D
from paper_2403_10647_b200 import gen_scene, spec_for_mesh

pytestmark = pytest.mark.gpu


class StagedComm(D.TorchComm):
    """TorchComm over gloo with device tensors staged through host memory."""

    @staticmethod
    def _host(x, dtype=np.int64):
        if isinstance(x, torch.Tensor):
            x = x.cpu().numpy()
        return torch.as_tensor(np.asarray(x, dtype=dtype))

    def allreduce_sum(self, arr):
        t = self._host(arr)
        self.dist.all_reduce(t)
        return t.numpy()

    def alltoall_counts(self, send):
        s = self._host(send)[:self.world].contiguous()
        r = torch.empty_like(s)
        self.dist.all_to_all_single(r, s)
        return [int(x) for x in s], [int(x) for x in r]

    def alltoall_pairs(self, keys, vals, send, recv, ops):
        out = []
        for x in (keys, vals):
            src = x.cpu() if isinstance(x, torch.Tensor) else torch.as_tensor(np.asarray(x).view(np.int32))
            dst = torch.empty(sum(recv), dtype=torch.int32)
            self.dist.all_to_all_single(dst, src.contiguous(), recv, send)
            out.append(dst.to(ops.dev))
        return out[0], out[1]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, case, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    got = "ok"
    try:
        torch.cuda.set_device(0)
        mesh = gen_scene("walls", 20000, 3)
        V, T = mesh.vertices.copy(), mesh.triangles.copy()
        spec = spec_for_mesh(mesh, dims=(50, 40, 30))
        if case == "negative":                 # a one-axis inverted box in the last shard only
            t = T[-1]
            V[t[0]] = np.asarray(spec.bounds.lo) + 0.6 * (np.asarray(spec.bounds.hi) - spec.bounds.lo)
            V[t[1]] = V[t[0]]
            V[t[1], 0] = np.inf
            V[t[2]] = V[t[0]] + 1e-9
        lo, hi = D.shard_range(len(T), rank, world)
        try:
            res = D.build_sharded(D.CudaOps(0), StagedComm(), V, T[lo:hi], lo, spec)
            if rank == 0:
                np.savez(out_path, G=res[0], O=res[1])
        except D.InvariantError:
            got = "InvariantError"
        with open(f"{out_path}.{rank}", "w") as fh:
            fh.write(got)
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(600)
@pytest.mark.parametrize("world", [2, 3])
def test_cuda_ranks_in_separate_processes(tmp_path, world):
    out = str(tmp_path / "res.npz")
    mp.spawn(_worker, args=(world, _free_port(), "ok", out), nprocs=world, join=True)
    res = np.load(out)
    mesh = gen_scene("walls", 20000, 3)
    G, O = oracle.build_parallel(mesh.vertices, mesh.triangles, spec_for_mesh(mesh, dims=(50, 40, 30)))
    assert np.array_equal(res["G"], G) and np.array_equal(res["O"], O)


@pytest.mark.timeout(600)
def test_cuda_ranks_agree_on_errors(tmp_path):
    out = str(tmp_path / "res.npz")
    mp.spawn(_worker, args=(2, _free_port(), "negative", out), nprocs=2, join=True)
    assert [open(f"{out}.{r}").read() for r in range(2)] == ["InvariantError"] * 2
