"""GPU-sampled training loop with the whole step in CUDA graphs (SURVEY.md
§8(f) NEXT(1); Fig. 2 step (1) and Fig. 6, lines 156 and 339-353:
sampling, graph build and training pipelined).

The sampler writes the PADDED layout (include/hifuse.h
hifuse_sample_blocks_padded): per-type capacities fixed once, so every batch
has the same host shapes and one captured graph serves all batches.  Graph c
(c = i mod 6) runs, for batch i:

  main stream   forward + backward + SGD of batch i   (built by graph i-1)
  side stream   build of batch i+1                   (sampled by graph i-1)
  side stream 2 sampling of batch i+2                (seeds staged by the host)

Buffers: a ring of 3 sampler output sets (batch i uses set i mod 3) and 2 CSR
slots (batch i uses slot i mod 2).  The host checks batch i's counts
(copied to pinned memory after graph i-2) against the capacities before
replaying graph i; a batch past them is re-sampled in the compact layout and
stepped eagerly with its exact shapes, then the pipeline is primed again --
the same result as if it had fitted.  Argument marshalling and scheduling
only: every step runs in libhifuse kernels.
"""
from __future__ import annotations

import numpy as np
import torch

from . import hifuse as hf
from .sampler import GpuSampler, PaddedBatch, SampledBatch


class SampledLoop:
    RING = 3       # sampler output sets (i, i+1, i+2 live at once)
    SLOTS = 2      # CSR slots (batch i computes while i+1 is built)

    def __init__(self, tr, smp: GpuSampler, feat, edge_type, target_type, src_cap, edge_pad,
                 batch_fn):
        """tr: Trainer; smp: GpuSampler with nbuf >= 4 (3 ring sets + 1 compact
        spare); batch_fn(i) -> (seeds pinned int32 [B], labels pinned int32
        [B], 64-bit key) of batch i."""
        if len(smp.bufs) < self.RING + 1:
            raise ValueError("the sampler needs nbuf >= 4")
        self.tr, self.smp, self.feat, self.et = tr, smp, feat, edge_type
        self.target = target_type
        self.src_cap = np.ascontiguousarray(src_cap, np.int64)
        self.edge_pad = np.ascontiguousarray(edge_pad, np.int64)
        self.batch_fn = batch_fn
        dev = tr.device
        B, L, T = smp.B, smp.L, smp.T
        self.L, self.T = L, T
        i32 = lambda: torch.empty(B, dtype=torch.int32, device=dev)
        self.seeds_d = [i32() for _ in range(self.RING + 1)]
        self.labels_d = [i32() for _ in range(self.RING + 1)]
        self.ctl_h = [torch.zeros(2, dtype=torch.int64).pin_memory() for _ in range(self.RING + 1)]
        # pinned staging of each ring set's seeds / labels: the host fills it
        # (numpy) and the graph's own copy nodes move it to the device, so a
        # step costs the host a few array writes and one replay
        self.seeds_h = [torch.zeros(B, dtype=torch.int32).pin_memory()
                        for _ in range(self.RING + 1)]
        self.labels_h = [torch.zeros(B, dtype=torch.int32).pin_memory()
                         for _ in range(self.RING + 1)]
        self.seeds_np = [x.numpy() for x in self.seeds_h]
        self.labels_np = [x.numpy() for x in self.labels_h]
        self.ctl_d = [torch.zeros(2, dtype=torch.int64, device=dev) for _ in range(self.RING + 1)]
        self.cnt_h = [torch.zeros(L * (2 * T + 1), dtype=torch.int32).pin_memory()
                      for _ in range(self.RING + 1)]
        # host views (numpy) of the pinned buffers: the per-step host work is
        # a few array operations, not torch indexing calls
        self.ctl_np = [c.numpy() for c in self.ctl_h]
        self.cnt_np = [c.numpy().reshape(L, 2 * T + 1) for c in self.cnt_h]
        lim = np.full((L, 2 * T + 1), np.iinfo(np.int32).max, np.int64)
        lim[:, :T] = self.src_cap
        lim[:, 2 * T] = self.edge_pad
        self.count_lim = lim             # counts <= lim <=> the padded block fits
        self.ev_ring = [torch.cuda.Event() for _ in range(8)]
        self.pb = {(r, s): PaddedBatch(smp, self.src_cap, self.edge_pad, r, self.labels_d[r],
                                       target_type, slot=s)
                   for r in range(self.RING) for s in range(self.SLOTS)}
        self.side_b = torch.cuda.Stream(device=dev)
        self.side_s = torch.cuda.Stream(device=dev)
        for st in (self.side_b, self.side_s):
            hf.stream_attach(st)
        self._fb_bufs, self._fb_views = {}, {}
        self.graphs = None
        self.done = {}          # batch -> event recorded after its graph / eager step
        self.fallbacks = 0
        self.kernels_per_graph = None

    # ----------------------------------------------------------- pieces
    def _batch(self, i):
        return self.pb[(i % self.RING, i % self.SLOTS)]

    def _fill(self, i, ring=None):
        """Host side of staging batch i: its seeds / labels / {key, stamp}
        into ring set r's pinned buffers."""
        r = i % self.RING if ring is None else ring
        seeds_h, labels_h, key = self.batch_fn(i)
        if seeds_h.numel() != self.smp.B or labels_h.numel() != self.smp.B:
            raise ValueError("a padded batch has exactly B seeds (drop the last partial batch)")
        self.seeds_np[r][:] = seeds_h.numpy()
        self.labels_np[r][:] = labels_h.numpy()
        key = int(key)
        self.ctl_np[r][0] = key - (1 << 64) if key >= (1 << 63) else key
        self.ctl_np[r][1] = self.smp.next_stamp()
        return r

    def _copy_in(self, r):
        """Pinned -> device copies of ring set r's staged inputs (current
        stream; captured into the graphs as copy nodes)."""
        self.seeds_d[r].copy_(self.seeds_h[r], non_blocking=True)
        self.labels_d[r].copy_(self.labels_h[r], non_blocking=True)
        self.ctl_d[r].copy_(self.ctl_h[r], non_blocking=True)

    def _stage(self, i, ring=None):
        """Eager staging of batch i (prime / fallback paths)."""
        self._copy_in(self._fill(i, ring))

    def _sample(self, r):
        self.smp.sample_padded(self.seeds_d[r], self.target, self.src_cap, self.edge_pad,
                               buf=r, d_ctl=self.ctl_d[r])

    def _copy_counts(self, r):
        """Device -> pinned host copy of ring set r's per-layer counts."""
        self.cnt_h[r].copy_(self.smp.counts_all[r], non_blocking=True)

    def _counts(self, r):
        return list(self.cnt_h[r].numpy().reshape(self.L, 2 * self.T + 1))

    def _fits(self, i):
        return bool((self.cnt_np[i % self.RING] <= self.count_lim).all())

    # ----------------------------------------------------------- graphs
    def capture(self):
        """One graph per (ring set, slot) phase; buffers are bound (and
        allocated) by planning every phase eagerly first."""
        tr = self.tr
        for c in range(6):
            tr.plan(self._batch(c), self.feat, self.et, include_build=False)
            tr.build_op(self._batch(c + 1), self.et)
        torch.cuda.synchronize()
        self.graphs = []
        for c in range(6):
            ops = tr.plan(self._batch(c), self.feat, self.et, include_build=False)
            bop = tr.build_op(self._batch(c + 1), self.et)
            g = torch.cuda.CUDAGraph()
            n0 = hf.kernel_launches()
            with torch.cuda.graph(g, stream=tr._hi):
                main = torch.cuda.current_stream()
                self.side_b.wait_stream(main)
                self.side_s.wait_stream(main)
                with torch.cuda.stream(self.side_b):
                    bop()
                with torch.cuda.stream(self.side_s):
                    rs = (c + 2) % self.RING
                    self._copy_in(rs)               # seeds / labels / ctl of batch i+2
                    self._sample(rs)
                    self._copy_counts(rs)           # its counts -> pinned host
                for _, fn in ops:
                    fn()
                hf.sgd(tr.params, tr.grads, tr.lr, 1.0 / max(tr.world, 1))
                main.wait_stream(self.side_b)
                main.wait_stream(self.side_s)
            self.graphs.append(g)
            self.kernels_per_graph = hf.kernel_launches() - n0
        torch.cuda.synchronize()

    # ----------------------------------------------------------- loop
    def _prime(self, i):
        """Eager start (or restart) at batch i: batch i sampled (padded) and
        built, batch i+1 sampled; synchronises."""
        main = torch.cuda.current_stream()
        for j in (i, i + 1):
            self._stage(j)
            self._sample(j % self.RING)
            self._copy_counts(j % self.RING)
        torch.cuda.synchronize()
        if self._fits(i):
            self.tr.build_op(self._batch(i), self.et)()
        ev = torch.cuda.Event()
        ev.record(main)
        self.done[i - 1] = ev
        self.done[i - 2] = ev

    def _fallback(self, i):
        """Batch i did not fit the capacities: compact re-sample into the spare
        set, eager step with its exact shapes (CSR slot 2), prime i+1."""
        torch.cuda.synchronize()
        self.fallbacks += 1
        spare = self.RING
        self._stage(i, ring=spare)
        self.smp.sample(self.seeds_d[spare], self.target, 0, buf=spare, d_ctl=self.ctl_d[spare])
        self._copy_counts(spare)
        torch.cuda.synchronize()
        sb = SampledBatch(self.smp, self._counts(spare), self.labels_d[spare], self.target,
                          slot=2, buf=spare)
        # the eager step gets its own activation / workspace / CSR buffers: a
        # batch past the capacities may need larger ones, and reallocating
        # the buffers the graphs are bound to would leave them dangling
        tr = self.tr
        bound = (tr._bufs, tr._views)
        tr._bufs, tr._views = self._fb_bufs, self._fb_views
        try:
            tr.step(sb, self.feat, self.et)
        finally:
            tr._bufs, tr._views = bound
        # batch i+1 was sampled (padded) by graph i-1 / the previous prime
        torch.cuda.synchronize()
        if self._fits(i + 1):
            self.tr.build_op(self._batch(i + 1), self.et)()
        self._stage(i + 2)
        self._sample((i + 2) % self.RING)
        self._copy_counts((i + 2) % self.RING)
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream())
        self.done[i] = ev
        self.done[i - 1] = ev

    def run(self, start, n, prime=True):
        """Steps batches start .. start+n-1 (asynchronous; returns after the
        last replay is enqueued).  Call capture() first.  prime=False continues
        a previous run that ended at batch start-1 (its replays built batch
        start and sampled start+1)."""
        if self.graphs is None:
            raise RuntimeError("capture() first")
        main = torch.cuda.current_stream()
        if prime:
            self._prime(start)
        for i in range(start, start + n):
            self.done.pop(i - 3, None)
            self.done[i - 2].synchronize()          # counts of batch i are on the host
            if not self._fits(i):
                self._fallback(i)
                continue
            self._fill(i + 2)                       # the graph copies it in
            self.graphs[i % 6].replay()
            ev = self.ev_ring[i % len(self.ev_ring)]   # (waited on two batches later)
            ev.record(main)
            self.done[i] = ev
        return self.tr.loss
