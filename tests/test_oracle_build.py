"""Pins of the oracle's semantic-graph build (Alg. 2).

The pins are independent of the oracle's own loops: SPEC.md hand examples
(tests/golden), a brute-force partition by numpy's stable lexsort, multiset
invariants, and the CSC recomputed by a library argsort.
"""
import json
import os

import numpy as np
import pytest

import oracle
from synth import random_block, random_schema
from synth.sampler import LayerBlock

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def _blk(src, dst, eid, n_src, n_dst):
    return LayerBlock(n_src=np.asarray(n_src, np.int32), n_dst=np.asarray(n_dst, np.int32),
                      src_local=np.asarray(src, np.int32), dst_local=np.asarray(dst, np.int32),
                      edge_id=np.asarray(eid, np.int64),
                      src_global=[np.arange(n) for n in n_src])


def test_spec_partition_example():
    g = GOLD["partition_0101"]
    rels = g["edge_relations"]
    # 1 type, 2 relations (0->0), 4 edges into dst 0, edge i has relation rels[i]
    blk = _blk([0, 1, 2, 3], [0, 0, 0, 0], [0, 1, 2, 3], [4], [1])
    sh = oracle.Shape([0, 0], [0, 0], [4], [1], 4)
    c = oracle.build(sh, blk, np.asarray(rels, np.int32))
    assert c["status"] == 0
    got = {str(r): c["eperm"][c["row_ptr"][c["rel_row_off"][r]]:c["row_ptr"][c["rel_row_off"][r] + 1]].tolist()
           for r in range(2)}
    assert got == g["expected"]


def test_single_relation_is_stable_sort_by_dst():
    rng = np.random.default_rng(1)
    n = 50
    dst = rng.integers(0, 7, n)
    src = rng.integers(0, 9, n)
    blk = _blk(src, dst, np.arange(n), [9], [7])
    sh = oracle.Shape([0], [0], [9], [7], n)
    c = oracle.build(sh, blk, np.zeros(n, np.int32))
    assert np.array_equal(c["eperm"], np.argsort(dst, kind="stable"))
    assert np.array_equal(c["row_ptr"], np.concatenate([[0], np.cumsum(np.bincount(dst, minlength=7))]))


def brute(blk, et, rel_src, rel_dst):
    """Independent brute force: lexsort by (relation, dst, column)."""
    R = len(rel_src)
    r = et[blk.edge_id]
    order = np.lexsort((np.arange(blk.num_edges), blk.dst_local, r))
    rows_per_rel = [int(blk.n_dst[rel_dst[k]]) for k in range(R)]
    rro = np.concatenate([[0], np.cumsum(rows_per_rel)])
    key = rro[r] + blk.dst_local
    row_ptr = np.concatenate([[0], np.cumsum(np.bincount(key, minlength=rro[-1]))])
    # compact Y rows: sorted unique (relation, src)
    pairs = np.unique(np.stack([r, blk.src_local], 1), axis=0)
    ymap = {(int(a), int(b)): i for i, (a, b) in enumerate(pairs)}
    col = np.array([ymap[(int(r[e]), int(blk.src_local[e]))] for e in order], np.int32)
    csc = np.lexsort((np.arange(len(col)), col))
    return dict(eperm=order, row_ptr=row_ptr, col=col, rel_row_off=rro,
                y_src=pairs[:, 1], U=len(pairs), csc_pos=csc, col_ptr=np.concatenate(
                    [[0], np.cumsum(np.bincount(col, minlength=len(pairs)))]),
                rel_y_off=np.searchsorted(pairs[:, 0], np.arange(R + 1)))


@pytest.mark.parametrize("seed", range(12))
def test_build_matches_bruteforce(seed):
    rng = np.random.default_rng(100 + seed)
    T = int(rng.integers(1, 5))
    R = int(rng.integers(1, 21))
    rs, rd = random_schema(rng, T, R)
    n_src = rng.integers(0, 40, T)
    n_dst = np.minimum(rng.integers(0, 30, T), n_src)
    if not any(n_src[rs[k]] > 0 and n_dst[rd[k]] > 0 for k in range(R)):
        n_src[:] = 5; n_dst[:] = 3
    N = int(rng.integers(0, 500))
    blk, et = random_block(rng, n_src, n_dst, rs, rd, N, hub_frac=0.2 if seed % 2 else 0.0)
    sh = oracle.Shape.of(blk, rs, rd)
    c = oracle.build(sh, blk, et)
    b = brute(blk, et, rs, rd)
    assert c["status"] == 0
    assert c["U"] == b["U"]
    for k in ("eperm", "row_ptr", "col", "rel_row_off", "y_src", "csc_pos", "col_ptr", "rel_y_off"):
        assert np.array_equal(np.asarray(c[k]), np.asarray(b[k])), k
    # csc_row is the merged row of each CSC entry
    row_of = np.repeat(np.arange(sh.rows), np.diff(c["row_ptr"]))
    assert np.array_equal(c["csc_row"], row_of[c["csc_pos"]])
    # csc_col is the Y row of each CSC entry: the CSR column of its position
    nv = int(c["col_ptr"][-1])
    assert np.array_equal(c["csc_col"][:nv], c["col"][c["csc_pos"][:nv]])
    assert (c["csc_col"][nv:] == -1).all()
    # partition invariant: multiset of (src, dst, relation) preserved
    r = et[blk.edge_id]
    got = sorted(zip(blk.src_local[c["eperm"]].tolist(), blk.dst_local[c["eperm"]].tolist(),
                     r[c["eperm"]].tolist()))
    assert got == sorted(zip(blk.src_local.tolist(), blk.dst_local.tolist(), r.tolist()))
    # slot map inverts (relation, src) -> Y row
    so = np.concatenate([[0], np.cumsum([n_src[rs[k]] for k in range(R)])])
    for u in range(c["U"]):
        rr = np.searchsorted(c["rel_y_off"], u, side="right") - 1
        assert c["slot_y"][so[rr] + c["y_src"][u]] == u


def test_invalid_edges_are_flagged_and_dropped():
    blk = _blk([0, 5, 1, 0], [0, 0, 9, 1], [0, 1, 2, 99], [3], [2])
    sh = oracle.Shape([0], [0], [3], [2], 4)
    c = oracle.build(sh, blk, np.zeros(4, np.int32))
    assert c["status"] == (1 | 4 | 8)
    assert c["row_ptr"][-1] == 1 and c["eperm"][0] == 0
    assert (c["eperm"][1:] == -1).all()


@pytest.mark.parametrize("seed", range(4))
def test_null_edges_are_dropped_silently(seed):
    """Edge id -1 (capacity padding, reading C26): the build equals
    the build of the block with those positions removed (eperm re-indexed),
    and no status bit is set.  Pinned against the brute force on the block
    without them."""
    rng = np.random.default_rng(300 + seed)
    T, R = 3, 7
    rs, rd = random_schema(rng, T, R)
    n_src = rng.integers(5, 40, T)
    n_dst = np.minimum(rng.integers(1, 30, T), n_src)
    blk, et = random_block(rng, n_src, n_dst, rs, rd, 400, hub_frac=0.1)
    keep = rng.random(blk.num_edges) > 0.3
    eid = blk.edge_id.copy()
    eid[~keep] = -1
    padded = _blk(blk.src_local, blk.dst_local, eid, n_src, n_dst)
    sh = oracle.Shape.of(padded, rs, rd)
    c = oracle.build(sh, padded, et)
    assert c["status"] == 0
    kept = np.nonzero(keep)[0]
    sub = _blk(blk.src_local[kept], blk.dst_local[kept], blk.edge_id[kept], n_src, n_dst)
    b = brute(sub, et, rs, rd)
    nv = int(c["row_ptr"][-1])
    assert nv == len(kept)
    assert np.array_equal(c["eperm"][:nv], kept[b["eperm"]])
    for k in ("row_ptr", "rel_row_off", "y_src", "rel_y_off", "col_ptr"):
        assert np.array_equal(np.asarray(c[k]), np.asarray(b[k])), k
    assert np.array_equal(c["col"][:nv], b["col"])
    assert (c["eperm"][nv:] == -1).all() and (c["col"][nv:] == -1).all()
