"""NEXT(4): feature-sharded data parallelism.

PAPER.md line 219 ("a large heterogeneous graph can be partitioned into
several subgraphs") and line 404: when the type-major feature store does not
fit one GPU, rank k of W keeps only the rows [bounds[k], bounds[k+1]) and,
before the layer-0 collect (A2), every batch fetches the rows it needs from
their owners:

  hifuse_shard_plan     ids grouped by owner (stable), per-owner counts
  all_to_all (counts)   how many ids every rank asks of every other
  hifuse_gather_words   ids in owner order -> all_to_all -> owners receive
  hifuse_gather_words   owners gather the requested local rows
  all_to_all (rows)     rows travel back (one NVLink all-to-all with NCCL)
  hifuse_scatter_words  rows back to batch order -> X0 [n, K]

The layer-0 calls then read X0 directly (gather_ids = None).  Every byte of
arithmetic-free data movement runs in the library's kernels; torch supplies
the process group.  The split sizes of the row all-to-all are host values,
so fetch() synchronises once per batch on the counts (it is a data-loading
step, outside the captured compute graph).

`exchange` is injectable: the default uses torch.distributed.all_to_all_single
on device tensors (NCCL); `staging="host"` moves the buffers through host
memory (gloo, e.g. two ranks sharing one GPU in the tests).
"""
from __future__ import annotations

import numpy as np
import torch

from . import hifuse as hf


def shard_bounds(total_rows: int, world: int) -> np.ndarray:
    """Balanced contiguous row ranges: bounds[k] .. bounds[k+1] for rank k."""
    return np.array([total_rows * k // world for k in range(world + 1)], np.int64)


class FeatureShard:
    def __init__(self, local_rows, bounds, rank, world, device, group=None, staging="device"):
        """local_rows: this rank's rows [bounds[rank], bounds[rank+1]) of the
        fp32 feature store, as a device tensor [n_local, K]."""
        self.rows = local_rows
        self.K = int(local_rows.shape[1])
        self.bounds_h = np.asarray(bounds, np.int64)
        self.bounds = torch.from_numpy(self.bounds_h).to(device)
        self.rank, self.world, self.device = rank, world, device
        self.group, self.staging = group, staging
        self.status = torch.zeros(1, dtype=torch.int32, device=device)
        assert local_rows.shape[0] == self.bounds_h[rank + 1] - self.bounds_h[rank]

    def _a2a(self, out, inp, out_splits, in_splits):
        import torch.distributed as dist
        if self.staging == "host":
            o = torch.empty(out.shape, dtype=out.dtype)
            dist.all_to_all_single(o, inp.cpu(), out_splits, in_splits, group=self.group)
            out.copy_(o)
        else:
            dist.all_to_all_single(out, inp, out_splits, in_splits, group=self.group)

    def fetch(self, gid):
        """X0 [len(gid), K] = feature rows gid (global type-major rows) of this
        rank's batch, gathered from their owners."""
        n = int(gid.numel())
        W, K, dev = self.world, self.K, self.device
        counts = torch.zeros(W, dtype=torch.int32, device=dev)
        order = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
        hf.shard_plan(gid, n, self.bounds, W, counts, order, self.status)
        send_ids = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
        hf.gather_words(gid, order, n, 1, 0, send_ids)
        recv_counts = torch.empty_like(counts)
        self._a2a(recv_counts, counts, [1] * W, [1] * W)
        in_splits = counts.cpu().tolist()              # the one host sync of the batch
        out_splits = recv_counts.cpu().tolist()
        m = int(sum(out_splits))
        req = torch.empty(max(m, 1), dtype=torch.int32, device=dev)
        self._a2a(req[:m], send_ids[:n], out_splits, in_splits)
        rows = torch.empty(max(m, 1), K, dtype=torch.float32, device=dev)
        hf.gather_words(self.rows, req, m, K, int(self.bounds_h[self.rank]), rows)
        back = torch.empty(max(n, 1), K, dtype=torch.float32, device=dev)
        self._a2a(back[:n], rows[:m], in_splits, out_splits)
        X0 = torch.empty(max(n, 1), K, dtype=torch.float32, device=dev)
        hf.scatter_words(back, order, n, K, X0)
        return X0[:n]
