"""Data parallelism over independent mini-batches.

Rank k of W processes batches k, k+W, k+2W, ... of the epoch (the sampler's
RNG is keyed by the batch index, so batch contents do not depend on W); the
only exchange per step is one all-reduce (sum) of the flat fp32 gradient
buffer, scaled by 1/W inside the SGD update.  Nothing here touches the CUDA
library, so the host logic runs under the gloo backend on CPU in the tests.
"""
from __future__ import annotations

import numpy as np


def _align4(n):
    return (n + 3) // 4 * 4


class ParamLayout:
    """Offsets of every parameter inside the flat buffer (16-byte aligned)."""

    def __init__(self, T, R, K0, D, H, C, L, model, fusion="sum"):
        self.entries = []
        off = 0

        def add(name, shape):
            nonlocal off
            n = int(np.prod(shape))
            self.entries.append((name, off, shape))
            off += _align4(n)

        for l in range(L):
            K = K0 if l == 0 else D
            add(f"{l}.W_rel", (R, K, D))
            if model == "rgcn":
                add(f"{l}.W_root", (T, K, D))
            add(f"{l}.bias", (T, D))
            if model == "rgat":
                add(f"{l}.att", (R, 2, D))
            if fusion == "han":          # HAN semantic attention (A = D)
                add(f"{l}.sem_W", (D, D))
                add(f"{l}.sem_b", (D,))
                add(f"{l}.sem_q", (D,))
        add("Wc", (D, C))
        add("bc", (C,))
        self.size = off

    def buckets(self, L):
        """Contiguous [lo, hi) ranges of the flat buffer: one per HGNN layer
        (its W_rel, W_root, bias, att, sem_* entries) and one for the classifier
        (Wc, bc), keyed "layer{l}" / "head"."""
        out = {}
        for name, o, shp in self.entries:
            key = f"layer{name.split('.')[0]}" if "." in name else "head"
            n = _align4(int(np.prod(shp)))
            lo, hi = out.get(key, (o, o))
            out[key] = (min(lo, o), max(hi, o + n))
        return out

    def views(self, flat):
        return {name: flat[o:o + int(np.prod(s))].view(*s) for name, o, s in self.entries}

    def flatten(self, grads: dict, like):
        """Packs a {'layers': [...], 'Wc', 'bc'} gradient dict into a flat buffer."""
        out = like.new_zeros(self.size)
        v = self.views(out)
        for name, _, _ in self.entries:
            if "." in name:
                l, k = name.split(".")
                src = grads["layers"][int(l)][k]
            else:
                src = grads[name]
            v[name].copy_(like.new_tensor(np.asarray(src)))
        return out


def rank_batches(rank: int, world: int, count: int):
    """Global batch indices processed by ``rank``: rank, rank + W, ..."""
    return [rank + s * world for s in range(count)]


def allreduce_grads(flat, world: int):
    """Sum of the flat gradient buffer over all ranks (the SGD kernel applies
    the 1/W factor)."""
    if world > 1:
        import torch.distributed as dist
        dist.all_reduce(flat)
    return flat
