"""Seeded mini-batch neighbour sampler (input generator; step (1) of PAPER.md
Fig. 2, "mini-batches are sampled from the original graph on CPU").

It sits OUTSIDE the library boundary and holds no arithmetic of the method.
Contract (reading C12):
  * each (vertex, relation) pair contributes at most ``fanout[hop]`` in-edges,
    drawn uniformly without replacement (all of them when fewer exist);
  * per vertex type the layer's destination vertices are the first
    ``n_dst[t]`` of its source vertices (message-flow block convention); new
    source vertices follow in order of first appearance in the edge list;
  * layers are returned outer first: ``layers[0]`` consumes raw features,
    ``layers[-1]`` produces the seed outputs; layer l's source set is layer
    l-1's destination set;
  * edges of one layer are emitted grouped by destination vertex (type-major,
    then local id), relations interleaved inside a group, which is the order a
    homogeneous sampler over a typed graph produces; Algorithm 2 (PAPER.md
    lines 310-324) must then select them per relation;
  * the RNG of batch b of epoch e is ``default_rng([seed, e, b])`` (S:L156,
    S:L507), so a batch does not depend on which rank samples it.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .configs import SEED, WorkloadConfig
from .graph import HeteroGraph


@dataclass
class LayerBlock:
    n_src: np.ndarray          # int32 [T]
    n_dst: np.ndarray          # int32 [T]
    src_local: np.ndarray      # int32 [N]
    dst_local: np.ndarray      # int32 [N]
    edge_id: np.ndarray        # int64 [N] global edge ids
    src_global: list           # per type int64 [n_src[t]] graph-local ids

    @property
    def num_edges(self) -> int:
        return int(self.src_local.shape[0])


@dataclass
class MiniBatch:
    seeds: np.ndarray          # int64 graph-local ids of the target type
    labels: np.ndarray         # int32 [len(seeds)]
    layers: list               # LayerBlock, outer first
    index: int = 0

    def gather_ids(self, feat_off) -> np.ndarray:
        """Row of the type-major global feature store for every layer-0 source
        vertex, type-major batch order (type offset + local id)."""
        blk = self.layers[0]
        return np.concatenate([np.asarray(feat_off[t] + blk.src_global[t], dtype=np.int64)
                               for t in range(len(blk.src_global))]).astype(np.int32)


def _positions(deg: np.ndarray, f: int, rng) -> tuple:
    """For every row with ``deg[i]`` candidates choose min(deg, f) distinct
    positions uniformly; returns (row index, position) pairs, rows ascending
    and positions ascending inside a row."""
    rows_all, pos_all = [], []
    small = np.nonzero(deg <= f)[0]
    if small.size:
        d = deg[small]
        rows = np.repeat(small, d)
        starts = np.repeat(np.cumsum(d) - d, d)
        rows_all.append(rows)
        pos_all.append(np.arange(rows.size, dtype=np.int64) - starts)
    big = np.nonzero(deg > f)[0]
    if big.size:
        d = deg[big].astype(np.int64)
        # bucket by width (power of two) so random-key argsort stays bounded
        width = np.maximum(1 << np.ceil(np.log2(np.maximum(d, 1))).astype(np.int64), 1)
        for w in np.unique(width):
            sel = np.nonzero(width == w)[0]
            dd = d[sel]
            if w <= 64 * f:
                keys = rng.random((sel.size, int(w)))
                keys[np.arange(int(w))[None, :] >= dd[:, None]] = 2.0
                pick = np.argsort(keys, axis=1)[:, :f]
            else:
                pick = np.floor(rng.random((sel.size, f)) * dd[:, None]).astype(np.int64)
                while True:
                    s = np.sort(pick, axis=1)
                    dup = np.nonzero((s[:, 1:] == s[:, :-1]).any(axis=1))[0]
                    if dup.size == 0:
                        break
                    pick[dup] = np.floor(rng.random((dup.size, f)) * dd[dup, None]).astype(np.int64)
            pick = np.sort(pick, axis=1)
            rows_all.append(np.repeat(big[sel], f))
            pos_all.append(pick.reshape(-1))
    if not rows_all:
        return np.zeros(0, np.int64), np.zeros(0, np.int64)
    rows = np.concatenate(rows_all)
    pos = np.concatenate(pos_all)
    o = np.lexsort((pos, rows))
    return rows[o], pos[o]


def sample_batch(g: HeteroGraph, target_type: int, seeds: np.ndarray, fanout,
                 rng) -> list:
    """Sample ``len(fanout)`` hops around ``seeds``; returns layers outer first."""
    T, R = g.num_types, g.num_rels
    in_lists = g.in_lists()
    frontier = [np.zeros(0, np.int64) for _ in range(T)]
    frontier[target_type] = np.asarray(seeds, dtype=np.int64)
    blocks = []
    for hop, f in enumerate(fanout):
        n_dst = np.array([len(x) for x in frontier], dtype=np.int32)
        dst_off = np.concatenate([[0], np.cumsum(n_dst)]).astype(np.int64)
        keys, rels, eids, dsts = [], [], [], []
        for r in range(R):
            t = int(g.rel_dst[r])
            if n_dst[t] == 0:
                continue
            ptr, order = in_lists[r]
            v = frontier[t]
            deg = ptr[v + 1] - ptr[v]
            rows, pos = _positions(deg, f, rng)
            if rows.size == 0:
                continue
            local = order[ptr[v[rows]] + pos]               # edge index inside relation r
            keys.append(dst_off[t] + rows)
            rels.append(np.full(rows.size, r, np.int32))
            eids.append(g.rel_edge_off[r] + local.astype(np.int64))
            dsts.append(rows.astype(np.int32))
        if keys:
            key = np.concatenate(keys)
            o = np.argsort(key, kind="stable")
            rel = np.concatenate(rels)[o]
            eid = np.concatenate(eids)[o]
            dst_local = np.concatenate(dsts)[o]
        else:
            rel = np.zeros(0, np.int32); eid = np.zeros(0, np.int64)
            dst_local = np.zeros(0, np.int32)
        src_local = np.empty(eid.size, np.int32)
        new_frontier = []
        for s in range(T):
            m = g.rel_src[rel] == s
            idx = np.nonzero(m)[0]
            if idx.size:
                r_of = rel[idx]
                gsrc = np.empty(idx.size, np.int64)
                for r in np.unique(r_of):
                    mm = r_of == r
                    gsrc[mm] = g.src[r][eid[idx[mm]] - g.rel_edge_off[r]]
            else:
                gsrc = np.zeros(0, np.int64)
            base = frontier[s]
            # vertices already in the destination prefix keep their local id
            if base.size:
                sb = np.argsort(base, kind="stable")
                p = np.searchsorted(base[sb], gsrc)
                p = np.minimum(p, base.size - 1)
                hit = base[sb][p] == gsrc
                loc = np.where(hit, sb[p], -1)
            else:
                loc = np.full(gsrc.size, -1, np.int64)
            miss = np.nonzero(loc < 0)[0]
            uniq, first = np.unique(gsrc[miss], return_index=True)
            order_new = np.argsort(first, kind="stable")
            new_ids = uniq[order_new]                      # first-appearance order
            if new_ids.size:
                rank_of_uniq = np.empty(uniq.size, np.int64)
                rank_of_uniq[order_new] = np.arange(uniq.size)
                loc[miss] = base.size + rank_of_uniq[np.searchsorted(uniq, gsrc[miss])]
            src_local[idx] = loc.astype(np.int32)
            new_frontier.append(np.concatenate([base, new_ids]).astype(np.int64))
        n_src = np.array([len(x) for x in new_frontier], dtype=np.int32)
        blocks.append(LayerBlock(n_src=n_src, n_dst=n_dst, src_local=src_local,
                                 dst_local=dst_local, edge_id=eid,
                                 src_global=new_frontier))
        frontier = new_frontier
    return blocks[::-1]


def epoch_seeds(cfg: WorkloadConfig, epoch: int, seed: int = SEED) -> np.ndarray:
    rng = np.random.default_rng([seed, 0x5E, epoch])
    return rng.permutation(cfg.type_counts[cfg.target_type]).astype(np.int64)


def labels_of(cfg: WorkloadConfig, ids: np.ndarray, seed: int = SEED) -> np.ndarray:
    rng = np.random.default_rng([seed, 0x1A])
    lab = rng.integers(0, cfg.num_classes, size=cfg.type_counts[cfg.target_type])
    return lab[ids].astype(np.int32)


def make_batch(cfg: WorkloadConfig, g: HeteroGraph, batch_index: int, epoch: int = 0,
               seed: int = SEED) -> MiniBatch:
    perm = epoch_seeds(cfg, epoch, seed)
    seeds = perm[batch_index * cfg.batch_size:(batch_index + 1) * cfg.batch_size]
    rng = np.random.default_rng([seed, epoch, batch_index])
    layers = sample_batch(g, cfg.target_type, seeds, cfg.fanout, rng)
    return MiniBatch(seeds=seeds, labels=labels_of(cfg, seeds, seed), layers=layers,
                     index=batch_index)


def batch_key(epoch: int, batch: int, seed: int = SEED) -> int:
    """64-bit stream key of batch ``batch`` of epoch ``epoch`` for the GPU
    sampler (splitmix64 chain of (seed, epoch, batch); a
    batch's randomness depends only on its index, not on the rank)."""
    M = (1 << 64) - 1

    def mix(z):
        z = (z + 0x9E3779B97F4A7C15) & M
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
        return z ^ (z >> 31)
    return mix(mix(mix(seed) ^ epoch) ^ batch)
