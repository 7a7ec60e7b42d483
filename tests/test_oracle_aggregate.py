"""Pins of the oracle's merged aggregation (Alg. 1)
and projection / fusion.

Independent references: SPEC.md hand examples (tests/golden), dense
multiplicity-matrix brute force (numpy matmul), torch.sparse.mm for the
single-relation case, closed-form special cases of the edge softmax, and a
dense masked-softmax GAT written with numpy.
"""
import json
import os

import numpy as np
import pytest
import torch

import oracle
from synth import random_block, random_schema
from synth.sampler import LayerBlock

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def _blk(src, dst, eid, n_src, n_dst):
    return LayerBlock(n_src=np.asarray(n_src, np.int32), n_dst=np.asarray(n_dst, np.int32),
                      src_local=np.asarray(src, np.int32), dst_local=np.asarray(dst, np.int32),
                      edge_id=np.asarray(eid, np.int64), src_global=[np.arange(n) for n in n_src])


def case(seed, T=None, R=None, N=None, D=8, H=1):
    rng = np.random.default_rng(seed)
    T = T or int(rng.integers(1, 4))
    R = R or int(rng.integers(1, 9))
    rs, rd = random_schema(rng, T, R)
    n_src = rng.integers(1, 25, T)
    n_dst = np.maximum(np.minimum(rng.integers(0, 15, T), n_src), 1)
    N = int(rng.integers(1, 200)) if N is None else N
    blk, et = random_block(rng, n_src, n_dst, rs, rd, N)
    sh = oracle.Shape.of(blk, rs, rd)
    csr = oracle.build(sh, blk, et)
    # a table Ytab[r][j] for every (relation, source); the oracle's Y holds its
    # compact rows
    ytab = [rng.standard_normal((int(n_src[rs[r]]), D)) for r in range(R)]
    Y = np.zeros((csr["U"], D))
    for r in range(R):
        for u in range(csr["rel_y_off"][r], csr["rel_y_off"][r + 1]):
            Y[u] = ytab[r][csr["y_src"][u]]
    return rng, sh, blk, et, csr, ytab, Y, rs, rd


def dense_adj(blk, et, r, rs, rd):
    A = np.zeros((int(blk.n_dst[rd[r]]), int(blk.n_src[rs[r]])))
    m = et[blk.edge_id] == r
    np.add.at(A, (blk.dst_local[m], blk.src_local[m]), 1.0)
    return A


def test_spec_hand_example():
    g = GOLD["aggregate_hand"]
    blk = _blk(g["edges_src"], g["edges_dst"], [0, 1], [2], [1])
    sh = oracle.Shape([0], [0], [2], [1], 2)
    csr = oracle.build(sh, blk, np.zeros(2, np.int32))
    Y = np.asarray(g["features"])[csr["y_src"]]
    for agg in ("sum", "mean"):
        z = oracle.aggregate_fwd(sh, blk, np.zeros(2, np.int32), csr, agg, 2, 1, Y)["Z"]
        assert np.array_equal(z, np.asarray(g[agg]))


@pytest.mark.parametrize("seed", range(10))
@pytest.mark.parametrize("agg", ["sum", "mean"])
def test_dense_bruteforce(seed, agg):
    rng, sh, blk, et, csr, ytab, Y, rs, rd = case(seed)
    Z = oracle.aggregate_fwd(sh, blk, et, csr, agg, Y.shape[1], 1, Y)["Z"]
    rro = csr["rel_row_off"]
    for r in range(sh.R):
        A = dense_adj(blk, et, r, rs, rd)
        ref = A @ ytab[r]
        if agg == "mean":
            deg = A.sum(1, keepdims=True)
            ref = np.where(deg > 0, ref / np.maximum(deg, 1), 0.0)
        np.testing.assert_allclose(Z[rro[r]:rro[r + 1]], ref, rtol=1e-12, atol=1e-12)


def test_single_relation_equals_torch_sparse_mm():
    rng, sh, blk, et, csr, ytab, Y, rs, rd = case(7, T=1, R=1, N=150)
    A = dense_adj(blk, et, 0, rs, rd)
    deg = A.sum(1)
    W = torch.tensor(A / np.maximum(deg, 1)[:, None]).to_sparse()
    ref = torch.sparse.mm(W, torch.tensor(ytab[0])).numpy()
    Z = oracle.aggregate_fwd(sh, blk, et, csr, "mean", Y.shape[1], 1, Y)["Z"]
    np.testing.assert_allclose(Z, ref, rtol=1e-12, atol=1e-13)


def test_mean_of_constant_is_constant():
    rng, sh, blk, et, csr, ytab, Y, rs, rd = case(3, N=300)
    Yc = np.full_like(Y, 0.375)
    out = oracle.aggregate_fwd(sh, blk, et, csr, "mean", Y.shape[1], 1, Yc)
    nz = out["deg"] > 0
    assert np.array_equal(out["Z"][nz], np.full((nz.sum(), Y.shape[1]), 0.375))
    assert np.array_equal(out["Z"][~nz], np.zeros(((~nz).sum(), Y.shape[1])))


def test_permutation_invariance():
    rng, sh, blk, et, csr, ytab, Y, rs, rd = case(11, N=180)
    Z = oracle.aggregate_fwd(sh, blk, et, csr, "sum", Y.shape[1], 1, Y)["Z"]
    perm = rng.permutation(blk.num_edges)
    blk2 = _blk(blk.src_local[perm], blk.dst_local[perm], blk.edge_id[perm], blk.n_src, blk.n_dst)
    csr2 = oracle.build(sh, blk2, et)
    assert csr2["U"] == csr["U"] and np.array_equal(csr2["y_src"], csr["y_src"])
    Z2 = oracle.aggregate_fwd(sh, blk2, et, csr2, "sum", Y.shape[1], 1, Y)["Z"]
    np.testing.assert_allclose(Z2, Z, rtol=1e-13, atol=1e-13)


# ----------------------------------------------------------------- RGAT ----

def test_gat_singleton_alpha_is_one():
    blk = _blk([3], [0], [0], [5], [2])
    sh = oracle.Shape([0], [0], [5], [2], 1)
    csr = oracle.build(sh, blk, np.zeros(1, np.int32))
    Y = np.array([[1.5, -2.0, 0.25, 4.0]])
    out = oracle.aggregate_fwd(sh, blk, np.zeros(1, np.int32), csr, "gat", 4, 2, Y,
                               np.array([[30.0, -7.0]]), np.array([[1.0, 2.0], [0.0, 0.0]]))
    assert np.array_equal(out["alpha"], np.full((1, 2), GOLD["rgat_singleton"]["alpha"]))
    assert np.array_equal(out["Z"][0], Y[0])


def test_gat_uniform_scores_give_inverse_degree():
    rng, sh, blk, et, csr, ytab, Y, rs, rd = case(5, D=8, H=2)
    ss = np.full((csr["U"], 2), 0.3)
    sd = np.full((sh.rows, 2), -0.1)
    out = oracle.aggregate_fwd(sh, blk, et, csr, "gat", 8, 2, Y, ss, sd)
    r = et[blk.edge_id]
    row = csr["rel_row_off"][r] + blk.dst_local
    np.testing.assert_allclose(out["alpha"], np.repeat((1.0 / out["deg"][row])[:, None], 2, 1),
                               rtol=1e-15)


def test_gat_zero_attention_reduces_to_mean():
    rng, sh, blk, et, csr, ytab, Y, rs, rd = case(9, D=8, H=4)
    Zm = oracle.aggregate_fwd(sh, blk, et, csr, "mean", 8, 1, Y)["Z"]
    out = oracle.aggregate_fwd(sh, blk, et, csr, "gat", 8, 4, Y, np.zeros((csr["U"], 4)),
                               np.zeros((sh.rows, 4)))
    np.testing.assert_allclose(out["Z"], Zm, rtol=1e-14, atol=1e-15)


def test_gat_alpha_sums_to_one_and_large_logits_are_finite():
    rng, sh, blk, et, csr, ytab, Y, rs, rd = case(13, D=8, H=2, N=190)
    ss = rng.standard_normal((csr["U"], 2)) * 1e4
    sd = rng.standard_normal((sh.rows, 2)) * 1e4
    out = oracle.aggregate_fwd(sh, blk, et, csr, "gat", 8, 2, Y, ss, sd)
    assert np.isfinite(out["Z"]).all() and np.isfinite(out["alpha"]).all()
    r = et[blk.edge_id]
    row = csr["rel_row_off"][r] + blk.dst_local
    sums = np.zeros((sh.rows, 2))
    np.add.at(sums, row, out["alpha"])
    nz = out["deg"] > 0
    np.testing.assert_allclose(sums[nz], 1.0, atol=1e-12)


def test_gat_dense_masked_softmax_single_relation():
    """R = T = H = 1: dense GAT, softmax over a masked score matrix (numpy).
    Multi-edges count once per copy (reading C11), so the mask carries them."""
    rng, sh, blk, et, csr, ytab, Y, rs, rd = case(17, T=1, R=1, N=120, D=6, H=1)
    a_src = rng.standard_normal(csr["U"])
    s_tab = np.zeros(int(blk.n_src[0]))
    s_tab[csr["y_src"]] = a_src
    sd = rng.standard_normal(sh.rows)
    out = oracle.aggregate_fwd(sh, blk, et, csr, "gat", 6, 1, Y, a_src[:, None], sd[:, None])
    A = dense_adj(blk, et, 0, rs, rd)
    pre = s_tab[None, :] + sd[:, None]
    lr = np.where(pre > 0, pre, 0.2 * pre)
    w = A * np.exp(lr - np.where(A > 0, lr, -np.inf).max(1, initial=-np.inf, keepdims=True))
    w = np.where(A.sum(1, keepdims=True) > 0, w / np.maximum(w.sum(1, keepdims=True), 1e-300), 0)
    np.testing.assert_allclose(out["Z"], w @ ytab[0], rtol=1e-12, atol=1e-12)


# ------------------------------------------------------- projection, fuse ---

def test_project_matches_numpy_matmul():
    rng, sh, blk, et, csr, ytab, Y, rs, rd = case(21, D=8, H=2)
    K, D, H = 6, 8, 2
    X = rng.standard_normal((sh.src_rows + 3, K))
    gid = rng.permutation(sh.src_rows + 3)[:sh.src_rows].astype(np.int32)
    W = rng.standard_normal((sh.R, K, D))
    Wr = rng.standard_normal((sh.T, K, D))
    att = rng.standard_normal((sh.R, 2, D))
    pr = oracle.project(sh, csr, K, D, H, X, gid, W, Wr, att)
    tso = np.concatenate([[0], np.cumsum(sh.n_src)])
    tdo = np.concatenate([[0], np.cumsum(sh.n_dst)])
    rro = csr["rel_row_off"]
    for r in range(sh.R):
        sl = slice(csr["rel_y_off"][r], csr["rel_y_off"][r + 1])
        xs = X[gid[tso[rs[r]] + csr["y_src"][sl]]]
        np.testing.assert_allclose(pr["Y"][sl], xs @ W[r], rtol=1e-12, atol=1e-12)
        ref_src = (pr["Y"][sl].reshape(-1, H, D // H) * att[r, 0].reshape(H, D // H)).sum(-1)
        np.testing.assert_allclose(pr["s_src"][sl], ref_src, rtol=1e-12, atol=1e-12)
        xd = X[gid[tso[rd[r]] + np.arange(sh.n_dst[rd[r]])]]
        ref_dst = ((xd @ W[r]).reshape(-1, H, D // H) * att[r, 1].reshape(H, D // H)).sum(-1)
        np.testing.assert_allclose(pr["s_dst"][rro[r]:rro[r + 1]], ref_dst, rtol=1e-12, atol=1e-12)
    for t in range(sh.T):
        xd = X[gid[tso[t] + np.arange(sh.n_dst[t])]]
        np.testing.assert_allclose(pr["R0"][tdo[t]:tdo[t + 1]], xd @ Wr[t], rtol=1e-12, atol=1e-12)


def test_identity_layer_is_mean_of_neighbours():
    """identity weights, zero root/bias, one relation, no
    activation -> the layer output is the mean of the neighbour features."""
    rng, sh, blk, et, csr, ytab, Y, rs, rd = case(23, T=1, R=1, N=90, D=5)
    X = rng.standard_normal((sh.src_rows, 5))
    pr = oracle.project(sh, csr, 5, 5, 1, X, None, np.eye(5)[None], np.zeros((1, 5, 5)), None)
    ag = oracle.aggregate_fwd(sh, blk, et, csr, "mean", 5, 1, pr["Y"])
    Hh = oracle.fuse(sh, 5, 0, ag["Z"], pr["R0"], np.zeros((1, 5)))
    A = dense_adj(blk, et, 0, rs, rd)
    deg = A.sum(1, keepdims=True)
    np.testing.assert_allclose(Hh, np.where(deg > 0, A @ X / np.maximum(deg, 1), 0), rtol=1e-12,
                               atol=1e-14)


def test_fuse_zero_in_degree_and_relu_mask():
    """A destination without in-edges gets act(R0 + b)."""
    blk = _blk([0], [0], [0], [3], [2])
    sh = oracle.Shape([0, 0], [0, 0], [3], [2], 1)
    Z = np.array([[1.0, -4.0], [0.0, 0.0], [2.0, 1.0], [0.0, 0.0]])   # rows (r0,i0) (r0,i1) (r1,i0) (r1,i1)
    R0 = np.array([[0.5, 0.5], [-1.0, 3.0]])
    b = np.array([[0.25, 0.25]])
    Hh = oracle.fuse(sh, 2, 1, Z, R0, b)
    assert np.array_equal(Hh, np.array([[3.75, 0.0], [0.0, 3.25]]))
