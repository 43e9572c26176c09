"""TEST INFRASTRUCTURE: numpy implementation of the per-rank steps of the sharded build
(the interface distributed.CudaOps implements with libpgrid kernels), built on the C
oracle's cell boxes. Lets the multi-rank orchestration run over gloo on CPU."""

import numpy as np
import torch

import oracle


class NumpyOps:
    def as_tensor(self, x):
        return torch.from_numpy(np.ascontiguousarray(np.asarray(x, np.uint32)).view(np.int32))

    def empty_pairs(self, n):
        return torch.empty(n, dtype=torch.int32)

    def length(self, x):
        return len(x)

    def slice(self, x, off, n):
        return x[off:off + n]

    def concat(self, xs):
        return np.concatenate([self.to_numpy(x) for x in xs]) if xs else np.zeros(0, np.uint32)

    def to_numpy(self, x):
        if isinstance(x, torch.Tensor):
            return x.numpy().view(np.uint32)
        return np.asarray(x, np.uint32)

    def count_stats(self, V, T, spec):
        """distributed.ShardState's PG_STATS count: {NO, index out of range, inverted boxes with
        negative / zero / positive counts, positive ones with a cell outside the grid}."""
        V = np.asarray(V)
        T = np.asarray(T)
        if T.size and (T.min() < 0 or T.max() >= len(V)):
            self._cnt = np.zeros(len(T), np.int64)
            return np.array([0, 1, 0, 0, 0, 0], np.int64)
        lo, hi, keep = oracle.cell_boxes(V, T, spec)
        m = hi.astype(np.int64) - lo + 1
        sc = np.where(keep, m[:, 0] * m[:, 1] * m[:, 2], 0)
        inv = keep & (m <= 0).any(axis=1)
        pos = inv & (sc > 0)
        if pos.any():
            raise NotImplementedError("numpy test ops: boxes inverted on two axes (covered on the GPU)")
        self.count(V, T, spec)
        no = int(np.where(inv, 0, sc).sum())
        return np.array([no, 0, int((inv & (sc < 0)).sum()), int((inv & (sc == 0)).sum()), 0, 0], np.int64)

    def count(self, V, T, spec):
        lo, hi, keep = oracle.cell_boxes(V, T, spec)
        self._lo, self._hi, self._keep = lo.astype(np.int64), hi.astype(np.int64), keep
        self._dims = [int(d) for d in spec.dims]
        m = self._hi - self._lo + 1
        self._cnt = np.where(keep & (m > 0).all(axis=1), m[:, 0] * m[:, 1] * m[:, 2], 0)
        return int(self._cnt.sum())

    def pairs(self, no, tri_base, shift, nbuckets):
        keys = np.empty(no, np.uint32)
        vals = np.empty(no, np.uint32)
        dx, dy = self._dims[0], self._dims[1]
        p = 0
        for i in np.flatnonzero(self._cnt):
            lo, hi = self._lo[i], self._hi[i]
            zz, yy, xx = np.meshgrid(np.arange(lo[2], hi[2] + 1), np.arange(lo[1], hi[1] + 1),
                                     np.arange(lo[0], hi[0] + 1), indexing="ij")
            cells = (xx + dx * (yy + dy * zz)).ravel()       # x-fastest (gridcore.py:112-125)
            keys[p:p + len(cells)] = cells
            vals[p:p + len(cells)] = tri_base + i
            p += len(cells)
        hist = np.bincount(keys.astype(np.int64) >> shift, minlength=nbuckets).astype(np.int64)
        return keys, vals, hist

    def partition(self, keys, vals, table, shift, nslabs, base):
        keys = np.asarray(keys, np.uint32)
        slab = np.asarray(table, np.int64)[keys.astype(np.int64) >> shift]
        order = np.argsort(slab, kind="stable")
        ko = (keys[order].astype(np.int64) - np.asarray(base, np.int64)[slab[order]]).astype(np.uint32)
        counts = np.bincount(slab, minlength=nslabs).astype(np.int64)
        return ko, np.asarray(vals, np.uint32)[order], counts

    def sort_cells(self, keys, vals, n, ncells, gen_order=True):
        keys = self.to_numpy(keys)
        vals = self.to_numpy(vals)
        ks, vs = oracle.radix_sort_pairs(keys, vals, int(ncells - 1).bit_length())
        G = np.zeros(ncells + 1, np.uint32)
        G[1:] = np.cumsum(np.bincount(ks.astype(np.int64), minlength=ncells))
        return G, vs
