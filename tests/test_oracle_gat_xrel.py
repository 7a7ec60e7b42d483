"""-m "not gpu": pins of the oracle's across-relation RGAT softmax (agg
"gat_xrel", reading C5'): for destination
(t, i) the edge-softmax runs over the union of its in-edges of every relation.
Pinned against special cases and invariants, not against a retyped formula:
  * one relation per destination type: identical to the within-relation GAT;
  * alpha sums to 1 over each destination's union of edges (per head);
  * zero attention: the fused sum over relations is the plain mean over ALL
    neighbours of the destination (dense multiplicity matrices, numpy);
  * the fused output equals a homogeneous GAT on the union graph (one dense
    masked softmax over the stacked relation blocks, numpy);
  * large logits stay finite; backward = finite differences.
"""
import numpy as np
import pytest

import oracle
from synth import random_block, random_schema

from test_oracle_aggregate import case, dense_adj
from test_oracle_backward import gmap, _fd


def fused(sh, csr, Z):
    """sum_r Z[(r,i)] per destination (t, i): the semantic fusion's sum (O4)."""
    tdo = np.concatenate([[0], np.cumsum(sh.n_dst)])
    out = np.zeros((sh.dst_rows, Z.shape[1]))
    for r in range(sh.R):
        t = sh.rel_dst[r]
        a = csr["rel_row_off"][r]
        out[tdo[t]:tdo[t + 1]] += Z[a:a + sh.n_dst[t]]
    return out


def one_rel_per_type_case(seed, D=8, H=2):
    rng = np.random.default_rng(seed)
    T = 3
    rs = np.array([1, 2, 0], np.int32)
    rd = np.array([0, 1, 2], np.int32)          # every dst type has exactly one relation
    n_src = rng.integers(3, 20, T)
    n_dst = np.maximum(np.minimum(rng.integers(1, 12, T), n_src), 1)
    blk, et = random_block(rng, n_src, n_dst, rs, rd, 150)
    sh = oracle.Shape.of(blk, rs, rd)
    csr = oracle.build(sh, blk, et)
    Y = rng.standard_normal((csr["U"], D))
    return rng, sh, blk, et, csr, Y


def test_one_relation_per_type_equals_within_relation():
    rng, sh, blk, et, csr, Y = one_rel_per_type_case(3)
    ss = rng.standard_normal((csr["U"], 2))
    sd = rng.standard_normal((sh.rows, 2))
    a = oracle.aggregate_fwd(sh, blk, et, csr, "gat", 8, 2, Y, ss, sd)
    b = oracle.aggregate_fwd(sh, blk, et, csr, "gat_xrel", 8, 2, Y, ss, sd)
    assert np.array_equal(a["Z"], b["Z"]) and np.array_equal(a["alpha"], b["alpha"])
    G = rng.standard_normal((sh.dst_rows, 8))
    ga = oracle.aggregate_bwd(sh, blk, et, csr, "gat", 8, 2, G, Y, ss, sd)
    gb = oracle.aggregate_bwd(sh, blk, et, csr, "gat_xrel", 8, 2, G, Y, ss, sd)
    for k in ("dY", "ds_src", "ds_dst"):
        assert np.array_equal(ga[k], gb[k]), k


@pytest.mark.parametrize("seed", range(4))
def test_alpha_sums_to_one_per_destination(seed):
    rng, sh, blk, et, csr, ytab, Y, rs, rd = case(200 + seed, T=2, R=6, N=180, D=8, H=2)
    ss = rng.standard_normal((csr["U"], 2)) * (1e4 if seed == 3 else 1.0)
    sd = rng.standard_normal((sh.rows, 2)) * (1e4 if seed == 3 else 1.0)
    out = oracle.aggregate_fwd(sh, blk, et, csr, "gat_xrel", 8, 2, Y, ss, sd)
    assert np.isfinite(out["Z"]).all() and np.isfinite(out["alpha"]).all()
    tdo = np.concatenate([[0], np.cumsum(sh.n_dst)])
    t = rd[et[blk.edge_id]]
    dest = tdo[t] + blk.dst_local
    sums = np.zeros((sh.dst_rows, 2))
    np.add.at(sums, dest, out["alpha"])
    has = np.zeros(sh.dst_rows, bool)
    has[dest] = True
    np.testing.assert_allclose(sums[has], 1.0, atol=1e-12)
    assert not sums[~has].any()


def test_zero_attention_is_mean_over_all_neighbours():
    rng, sh, blk, et, csr, ytab, Y, rs, rd = case(31, T=2, R=5, N=160, D=8, H=4)
    out = oracle.aggregate_fwd(sh, blk, et, csr, "gat_xrel", 8, 4, Y, np.zeros((csr["U"], 4)),
                               np.zeros((sh.rows, 4)))
    F = fused(sh, csr, out["Z"])
    tdo = np.concatenate([[0], np.cumsum(sh.n_dst)])
    for ty in range(sh.T):
        num = np.zeros((int(sh.n_dst[ty]), 8))
        deg = np.zeros(int(sh.n_dst[ty]))
        for r in range(sh.R):
            if rd[r] != ty:
                continue
            A = dense_adj(blk, et, r, rs, rd)
            num += A @ ytab[r]
            deg += A.sum(1)
        ref = np.where(deg[:, None] > 0, num / np.maximum(deg, 1)[:, None], 0.0)
        np.testing.assert_allclose(F[tdo[ty]:tdo[ty + 1]], ref, rtol=1e-13, atol=1e-14)


def test_equals_homogeneous_gat_on_union_graph():
    """Stack the relation blocks of one destination type side by side: one
    dense masked softmax per destination row over all relations' sources
    (numpy), then alpha @ [Y_r1; Y_r2; ...] is the fused output."""
    H, D = 1, 6
    rng, sh, blk, et, csr, ytab, Y, rs, rd = case(41, T=1, R=3, N=120, D=D, H=H)
    ss_tab = [rng.standard_normal(int(blk.n_src[rs[r]])) for r in range(sh.R)]
    ss = np.zeros((csr["U"], 1))
    for r in range(sh.R):
        for u in range(csr["rel_y_off"][r], csr["rel_y_off"][r + 1]):
            ss[u, 0] = ss_tab[r][csr["y_src"][u]]
    sd = rng.standard_normal((sh.rows, 1))
    out = oracle.aggregate_fwd(sh, blk, et, csr, "gat_xrel", D, H, Y, ss, sd)
    A = np.concatenate([dense_adj(blk, et, r, rs, rd) for r in range(sh.R)], axis=1)
    n = int(sh.n_dst[0])
    pre = np.concatenate([ss_tab[r][None, :] + sd[csr["rel_row_off"][r]:csr["rel_row_off"][r] + n]
                          for r in range(sh.R)], axis=1)
    lr = np.where(pre > 0, pre, 0.2 * pre)
    mx = np.where(A > 0, lr, -np.inf).max(1, initial=-np.inf, keepdims=True)
    w = A * np.exp(lr - np.where(np.isfinite(mx), mx, 0.0))
    w = np.where(A.sum(1, keepdims=True) > 0, w / np.maximum(w.sum(1, keepdims=True), 1e-300), 0)
    ref = w @ np.concatenate(ytab, axis=0)
    np.testing.assert_allclose(fused(sh, csr, out["Z"]), ref, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("seed", range(3))
def test_backward_finite_differences(seed):
    H, D = 2, 8
    rng, sh, blk, et, csr, ytab, Y, rs, rd = case(300 + seed, T=2, R=5, D=D, H=H)
    ss = rng.standard_normal((csr["U"], H))
    sd = rng.standard_normal((sh.rows, H))
    G = rng.standard_normal((sh.dst_rows, D))
    Gm = gmap(sh, csr, G)

    def loss():
        return float((oracle.aggregate_fwd(sh, blk, et, csr, "gat_xrel", D, H, Y, ss, sd)["Z"]
                      * Gm).sum())

    b = oracle.aggregate_bwd(sh, blk, et, csr, "gat_xrel", D, H, G, Y, ss, sd)
    for arr, grad in ((Y, b["dY"]), (ss, b["ds_src"]), (sd, b["ds_dst"])):
        for _ in range(8):
            idx = tuple(rng.integers(0, s) for s in arr.shape)
            num = _fd(loss, arr, idx)
            assert abs(num - grad[idx]) <= 1e-4 * max(1.0, abs(num)), (idx, num, grad[idx])
