"""GPU neighbour sampler: device-resident graph
in-adjacency + hifuse_sample_blocks (include/hifuse.h).  Argument marshalling
and buffer ownership only; sampling runs in libhifuse kernels.

GpuSampler.sample() is stream-ordered and graph-capturable (capacities are
host-known); SampledBatch turns one sampled set of blocks into the object the
Trainer consumes (DeviceBatch's attributes) after a single read of the
per-layer counts (the only data-dependent sizes)."""
from __future__ import annotations

import numpy as np
import torch

from . import hifuse as hf


class GpuSampler:
    def __init__(self, rel_src, rel_dst, type_counts, in_csc, fanout, batch_size, device,
                 gather=True, nbuf=1):
        """in_csc[r] = (ptr [|V_t(r)|+1], src [E_r] ids within type s(r), eid [E_r]
        global edge ids); fanout per layer, outer first.  nbuf output buffer
        sets (2: sample batch i+1 while batch i computes)."""
        hf.lib()
        self.rel_src = np.ascontiguousarray(rel_src, np.int32)
        self.rel_dst = np.ascontiguousarray(rel_dst, np.int32)
        self.counts_h = np.ascontiguousarray(type_counts, np.int64)
        self.T, self.R = len(self.counts_h), len(self.rel_src)
        self.fanout = np.ascontiguousarray(fanout, np.int32)
        self.L = len(self.fanout)
        self.B = int(batch_size)
        self.device = device
        ptrs, srcs, eids, off = [], [], [], []
        pos = n = 0
        for ptr, src, eid in in_csc:
            off.append(n)
            ptrs.append(np.asarray(ptr, np.int64) + pos)
            srcs.append(np.asarray(src, np.int32))
            eids.append(np.asarray(eid, np.int64))
            pos += len(src)
            n += len(ptr)
        self.in_ptr_off = np.ascontiguousarray(off, np.int64)
        cat = lambda a, dt: torch.from_numpy(np.concatenate(a) if a else np.zeros(1, dt)).to(device)
        self.d_ptr = cat(ptrs, np.int64)
        self.d_src = cat(srcs, np.int32)
        self.d_eid = cat(eids, np.int64)
        self.g = hf.GraphCsc(self.T, self.R, self.rel_src.ctypes.data, self.rel_dst.ctypes.data,
                             self.counts_h.ctypes.data, self.in_ptr_off.ctypes.data,
                             self.d_ptr.data_ptr(), self.d_src.data_ptr(), self.d_eid.data_ptr())
        ec, sc, wsb, stn = hf.sample_caps(self.g, self.fanout, self.B)
        self.edge_cap, self.src_cap = ec, sc
        i32 = lambda n: torch.empty(int(n), dtype=torch.int32, device=device)
        self.bufs = []
        self.counts_all = []        # per buffer set: every layer's counts, contiguous
        nc = 2 * self.T + 1
        for _ in range(nbuf):
            outs = []
            call = i32(self.L * nc)
            self.counts_all.append(call)
            for l in range(self.L):
                outs.append(dict(src=i32(ec[l]), dst=i32(ec[l]),
                                 eid=torch.empty(int(ec[l]), dtype=torch.int64, device=device),
                                 gid=i32(sc[l]), counts=call[l * nc:(l + 1) * nc],
                                 gather=i32(sc[l]) if (gather and l == 0) else None))
            blocks = [hf.Block(o["src"].data_ptr(), o["dst"].data_ptr(), o["eid"].data_ptr(),
                               o["gid"].data_ptr(), o["counts"].data_ptr(),
                               o["gather"].data_ptr() if o["gather"] is not None else None)
                      for o in outs]
            self.bufs.append((outs, blocks))
        self.out, self.blocks = self.bufs[0]
        self.ws = torch.empty((wsb + 3) // 4 + 64, dtype=torch.int32, device=device)
        self.state = torch.zeros(int(stn), dtype=torch.int32, device=device)
        self.status = torch.zeros(1, dtype=torch.int32, device=device)
        self.stamp = 1

    def sample(self, seeds, target_type, key, stream=None, buf=0, d_ctl=None):
        """Samples the blocks of ``seeds`` (device int32, ids within the
        target type) into output buffer set ``buf`` (self.out then points at
        it; overwritten by the next call on the same set).  d_ctl: device
        uint64 [2] {key, stamp} read by the kernels instead (graph replays;
        the caller then advances the stamp with next_stamp())."""
        if seeds.numel() > self.B:
            raise ValueError("more seeds than the sampler's capacity")
        self.out, self.blocks = self.bufs[buf]
        hf.sample_blocks(self.g, self.fanout, seeds, target_type, key, self.stamp, self.blocks,
                         self.state, self.ws, self.status, stream, d_ctl=d_ctl)
        if d_ctl is None:
            self.stamp += self.L
        if self.stamp > (1 << 30):          # stamps exhausted: reset the state
            self.state.zero_()
            self.stamp = 1

    def sample_padded(self, seeds, target_type, src_cap, edge_pad, stream=None, buf=0, d_ctl=None,
                      key=0):
        """As sample(), in the padded layout of hifuse_sample_blocks_padded:
        src_cap int64 [L, T] per-type source capacities, edge_pad int64 [L]
        (see padded_caps).  With d_ctl the key and stamp come from device
        memory (graph replays; the caller advances the stamp)."""
        if seeds.numel() > self.B:
            raise ValueError("more seeds than the sampler's capacity")
        self.out, self.blocks = self.bufs[buf]
        hf.sample_blocks_padded(self.g, self.fanout, seeds, target_type, key, self.stamp, src_cap,
                                edge_pad, self.blocks, self.state, self.ws, self.status, stream,
                                d_ctl=d_ctl)
        if d_ctl is None:
            self.stamp += self.L
        if self.stamp > (1 << 30):
            self.state.zero_()
            self.stamp = 1

    def next_stamp(self):
        """Stamp base for the next d_ctl-driven call (resets the state when the
        stamps run out; stream-ordered with the calls)."""
        st = self.stamp
        self.stamp += self.L
        if self.stamp > (1 << 30):
            self.state.zero_()
            self.stamp = 1
            st, self.stamp = 1, 1 + self.L
        return st

    def counts(self, buf=None):
        """Host copy of every layer's [n_src[T], n_dst[T], N] (synchronises)."""
        outs = self.out if buf is None else self.bufs[buf][0]
        return [o["counts"].cpu().numpy() for o in outs]


class SampledBatch:
    """DeviceBatch-compatible view of the sampler's current output (valid
    until the sampler's next call)."""

    def __init__(self, smp: GpuSampler, counts, labels_dev, target_type, slot=0, buf=None):
        T = smp.T
        outs = smp.out if buf is None else smp.bufs[buf][0]
        self.shapes = []
        self.dev = dict(src=[], dst=[], eid=[])
        for l, c in enumerate(counts):
            n_src, n_dst, N = c[:T], c[T:2 * T], int(c[2 * T])
            self.shapes.append(hf.Shape(smp.rel_src, smp.rel_dst, n_src, n_dst, N))
            o = outs[l]
            self.dev["src"].append(o["src"][:max(N, 1)])
            self.dev["dst"].append(o["dst"][:max(N, 1)])
            self.dev["eid"].append(o["eid"][:max(N, 1)])
        self.dev["gid"] = outs[0]["gather"][:max(int(counts[0][:T].sum()), 1)]
        self.dev["labels"] = labels_dev
        self.B = int(labels_dev.numel())
        self.slot = slot
        self.target_type = target_type
        self.h_row0 = int(self.shapes[-1].type_dst_off[target_type])
        self.device = smp.device


def padded_caps(counts_list, T, target_type, B, margin=0.15, slack=64, align=32):
    """Per-layer, per-type source capacities and padded edge counts of the
    padded sampler layout (include/hifuse.h hifuse_sample_blocks_padded) from
    the per-layer counts of some batches sampled in the compact layout.

    A padded layer's destinations are the previous (inner) layer's padded
    sources, so its sources need cap_src[l+1] + (new sources of layer l); the
    new sources and the edges are the same in both layouts (the sample is a
    function of the batch key).  Each observed maximum grows by ``margin``
    plus ``slack`` (aligned to ``align`` rows); a type never seen stays 0.  A
    batch past the capacities is detected on the host (counts) and re-run in
    the compact layout (SampledLoop)."""
    L = len(counts_list[0])
    new = np.zeros((L, T), np.int64)
    inner = np.zeros(T, np.int64)
    edges = np.zeros(L, np.int64)
    for counts in counts_list:
        for l, c in enumerate(counts):
            c = np.asarray(c, np.int64)
            new[l] = np.maximum(new[l], c[:T] - c[T:2 * T])
            edges[l] = max(edges[l], c[2 * T])
        inner = np.maximum(inner, np.asarray(counts[-1], np.int64)[:T])

    def grow(x):
        x = int(x)
        if x == 0:
            return 0
        return -(-(int(np.ceil(x * (1 + margin))) + slack) // align) * align

    src_cap = np.zeros((L, T), np.int64)
    for l in range(L - 1, -1, -1):
        for t in range(T):
            if l == L - 1:
                src_cap[l, t] = max(grow(inner[t]), B if t == target_type else 0)
            else:
                src_cap[l, t] = src_cap[l + 1, t] + grow(new[l, t])
    edge_pad = np.array([grow(e) for e in edges], np.int64)
    return src_cap, edge_pad


def counts_fit(counts, src_cap, edge_pad):
    """True if a padded block's counts fit its capacities."""
    T = src_cap.shape[1]
    return all(np.all(np.asarray(c[:T]) <= src_cap[l]) and int(c[2 * T]) <= int(edge_pad[l])
               for l, c in enumerate(counts))


class PaddedBatch:
    """DeviceBatch-compatible view of a padded sampler output buffer set: its
    host shapes are the capacities, so every batch sampled into it has the
    same shapes and one captured CUDA graph serves all of them."""

    def __init__(self, smp: GpuSampler, src_cap, edge_pad, buf, labels_dev, target_type, slot=0):
        T, L = smp.T, smp.L
        outs = smp.bufs[buf][0]
        self.shapes = []
        self.dev = dict(src=[], dst=[], eid=[])
        for l in range(L):
            n_src = src_cap[l]
            if l < L - 1:
                n_dst = src_cap[l + 1]
            else:
                n_dst = np.zeros(T, np.int64)
                n_dst[target_type] = labels_dev.numel()
            N = int(edge_pad[l])
            self.shapes.append(hf.Shape(smp.rel_src, smp.rel_dst, n_src, n_dst, N))
            o = outs[l]
            self.dev["src"].append(o["src"][:max(N, 1)])
            self.dev["dst"].append(o["dst"][:max(N, 1)])
            self.dev["eid"].append(o["eid"][:max(N, 1)])
        self.dev["gid"] = outs[0]["gather"][:max(int(src_cap[0].sum()), 1)]
        self.dev["labels"] = labels_dev
        self.B = int(labels_dev.numel())
        self.slot = slot
        self.target_type = target_type
        self.h_row0 = int(self.shapes[-1].type_dst_off[target_type])
        self.device = smp.device
