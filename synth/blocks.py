"""Small seeded random layer blocks for parity tests (input generator only).

A block is one layer of a sampled mini-batch (Alg. 2 inputs
``EdgeIndex[i]``, ``EdgeID[i]``, ``EdgeType``, lines 313-316): batch-local
endpoints per type, global edge ids and the graph-global edge-type table.
"""
from __future__ import annotations

import numpy as np

from .sampler import LayerBlock


def random_schema(rng, T: int, R: int):
    rel_src = rng.integers(0, T, size=R).astype(np.int32)
    rel_dst = rng.integers(0, T, size=R).astype(np.int32)
    return rel_src, rel_dst


def random_block(rng, n_src, n_dst, rel_src, rel_dst, N: int, graph_edges_per_rel: int = 64,
                 hub_frac: float = 0.0, shuffle_edge_type: bool = True):
    """Random block with N edges.  Returns (LayerBlock, edge_type[E_graph]).

    ``hub_frac`` of the edges take source 0 (a long CSC column); destination
    ids are uniform, so rows are ragged and some are empty.
    """
    n_src = np.asarray(n_src, np.int32)
    n_dst = np.minimum(np.asarray(n_dst, np.int32), n_src)
    rel_src = np.asarray(rel_src, np.int32)
    rel_dst = np.asarray(rel_dst, np.int32)
    R = len(rel_src)
    E = R * graph_edges_per_rel
    et = np.repeat(np.arange(R, dtype=np.int32), graph_edges_per_rel)
    if shuffle_edge_type:
        et = et[rng.permutation(E)]
    pools = [np.nonzero(et == r)[0] for r in range(R)]
    live = [r for r in range(R) if n_dst[rel_dst[r]] > 0 and n_src[rel_src[r]] > 0]
    if N > 0 and not live:
        raise ValueError("no relation can carry an edge")
    rel = rng.choice(np.asarray(live, np.int32), size=N) if N else np.zeros(0, np.int32)
    src = np.empty(N, np.int32)
    dst = np.empty(N, np.int32)
    eid = np.empty(N, np.int64)
    for k in range(N):
        r = int(rel[k])
        dst[k] = rng.integers(0, n_dst[rel_dst[r]])
        src[k] = 0 if rng.random() < hub_frac else rng.integers(0, n_src[rel_src[r]])
        eid[k] = pools[r][rng.integers(0, len(pools[r]))]
    blk = LayerBlock(n_src=n_src, n_dst=n_dst, src_local=src, dst_local=dst, edge_id=eid,
                     src_global=[np.arange(n, dtype=np.int64) for n in n_src])
    return blk, et


def block_shape_arrays(blk: LayerBlock, rel_src, rel_dst) -> dict:
    """Host metadata of one layer (the library's ``hifuse_layer_shape``)."""
    return dict(num_types=len(blk.n_src), num_rels=len(rel_src),
                rel_src_type=np.asarray(rel_src, np.int32),
                rel_dst_type=np.asarray(rel_dst, np.int32),
                n_src=np.asarray(blk.n_src, np.int32), n_dst=np.asarray(blk.n_dst, np.int32),
                num_edges=blk.num_edges)
