"""Seeded synthetic heterographs (input generator; no method arithmetic).

Recipe (stated in DESIGN.md §Inputs):
  * endpoint popularity Zipf(a) (a = 0.8 by default) over a per-type random
    permutation of vertex ids, so hubs are not id-correlated (SPEC.md S:L62
    "power-law-skewed distribution controlled by the skew parameter");
  * multi-edges are kept (reading C11);
  * global edge ids are relation-major, so
    ``edge_type[eid]`` is the relation of edge ``eid`` (Alg. 2 line
    316 "IndexSelect(EdgeType, EdgeID[i])");
  * features ~ N(0,1) fp32 in ONE type-major matrix (§4.2 lines
    218-219, "organized by vertex type first"), rows of type t start at
    ``feat_off[t]``.
"""
from __future__ import annotations

import numpy as np

from .configs import SEED, WorkloadConfig


def zipf_endpoints(rng, n: int, size: int, a: float, perm: np.ndarray) -> np.ndarray:
    """Draw ``size`` vertex ids in [0, n) with P(rank k) ~ (k+1)^-a, mapped
    through ``perm`` (continuous inverse-CDF approximation of a finite Zipf)."""
    u = rng.random(size)
    if a == 1.0:
        x = np.exp(u * np.log(n + 1.0))
    else:
        b = 1.0 - a
        x = (u * ((n + 1.0) ** b - 1.0) + 1.0) ** (1.0 / b)
    k = np.minimum(np.floor(x).astype(np.int64) - 1, n - 1)
    k = np.maximum(k, 0)
    return perm[k].astype(np.int32)


class HeteroGraph:
    """Topology of a synthetic heterograph.

    Attributes
      counts[T], rel_src[R], rel_dst[R]   schema
      src[r], dst[r]                      int32 local endpoint ids per relation
      rel_edge_off[R+1]                   global edge id of relation r's first edge
      edge_type[E]                        int32 relation of every global edge id
      in_ptr[r], in_eid[r]                per-relation in-edge lists (sorted by dst,
                                          stable), used only by the sampler
    """

    def __init__(self, counts, rel_src, rel_dst, src, dst):
        self.counts = np.asarray(counts, dtype=np.int64)
        self.rel_src = np.asarray(rel_src, dtype=np.int32)
        self.rel_dst = np.asarray(rel_dst, dtype=np.int32)
        self.src = [np.ascontiguousarray(s, dtype=np.int32) for s in src]
        self.dst = [np.ascontiguousarray(d, dtype=np.int32) for d in dst]
        sizes = np.array([len(s) for s in self.src], dtype=np.int64)
        self.rel_edge_off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
        self.num_edges = int(self.rel_edge_off[-1])
        self.edge_type = np.repeat(np.arange(len(self.src), dtype=np.int32), sizes)
        self._in = None

    @property
    def num_types(self):
        return len(self.counts)

    def in_csc(self):
        """Per relation r: (ptr [|V_t(r)|+1] int64, src [E_r] int32 source ids
        within type s(r), eid [E_r] int64 global edge ids), in-edges grouped by
        destination, stable: the graph format the GPU sampler reads (format
        conversion only)."""
        out = []
        for r, (ptr, order) in enumerate(self.in_lists()):
            out.append((ptr.astype(np.int64), self.src[r][order].astype(np.int32),
                        self.rel_edge_off[r] + order.astype(np.int64)))
        return out

    @property
    def num_rels(self):
        return len(self.src)

    def in_lists(self):
        """Per relation: (in_ptr[n_dst+1], local edge index sorted by dst)."""
        if self._in is None:
            out = []
            for r in range(self.num_rels):
                n = int(self.counts[self.rel_dst[r]])
                d = self.dst[r]
                order = np.argsort(d, kind="stable").astype(np.int32)
                ptr = np.zeros(n + 1, dtype=np.int64)
                np.cumsum(np.bincount(d, minlength=n), out=ptr[1:])
                out.append((ptr, order))
            self._in = out
        return self._in


def generate_graph(cfg: WorkloadConfig, seed: int = SEED) -> HeteroGraph:
    rng = np.random.default_rng([seed, 0x6E])
    perms = [rng.permutation(int(c)) for c in cfg.type_counts]
    src, dst = [], []
    for r, spec in enumerate(cfg.rels):
        if spec.mirror_of >= 0:
            src.append(dst[spec.mirror_of].copy())
            dst.append(src[spec.mirror_of].copy())
            continue
        rr = np.random.default_rng([seed, 0x6E, r])
        ns, nd = cfg.type_counts[spec.src], cfg.type_counts[spec.dst]
        s = zipf_endpoints(rr, ns, spec.edges, cfg.zipf, perms[spec.src])
        d = zipf_endpoints(rr, nd, spec.edges, cfg.zipf, perms[spec.dst])
        if spec.sym:
            s, d = np.concatenate([s, d]), np.concatenate([d, s])
        src.append(s)
        dst.append(d)
    return HeteroGraph(cfg.type_counts, [r.src for r in cfg.rels],
                       [r.dst for r in cfg.rels], src, dst)


def generate_features(counts, dim: int, seed: int = SEED) -> tuple:
    """Type-major feature store: (feat fp32 [sum(counts), dim], feat_off[T+1])."""
    counts = np.asarray(counts, dtype=np.int64)
    off = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    rng = np.random.default_rng([seed, 0xFE, dim])
    feat = rng.standard_normal((int(off[-1]), dim), dtype=np.float32)
    return feat, off


def glorot(rng, shape, fan_in, fan_out) -> np.ndarray:
    """Uniform(+-sqrt(6/(fan_in+fan_out))) fp32."""
    lim = np.sqrt(6.0 / (fan_in + fan_out))
    return rng.uniform(-lim, lim, size=shape).astype(np.float32)
