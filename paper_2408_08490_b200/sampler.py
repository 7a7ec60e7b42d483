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
        for _ in range(nbuf):
            outs = []
            for l in range(self.L):
                outs.append(dict(src=i32(ec[l]), dst=i32(ec[l]),
                                 eid=torch.empty(int(ec[l]), dtype=torch.int64, device=device),
                                 gid=i32(sc[l]), counts=i32(2 * self.T + 1),
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
