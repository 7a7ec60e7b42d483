"""Pins of the oracle's aggregate-first RGCN input layer (O6; SURVEY.md §8(f)
NEXT(3)): Alg. 1 over the raw
features followed by the projection of the aggregated rows.

Independent references: the SPEC hand example (tests/golden), a
dense multiplicity-matrix brute force (numpy), and the linearity identity
against the project-first oracle path (O2 then O3 forward, O5 backward),
which is pinned on its own by tests/test_oracle_aggregate.py and
tests/test_oracle_backward.py.
"""
import json
import os

import numpy as np
import pytest

import oracle
from synth import random_block, random_schema
from synth.sampler import LayerBlock

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def case(seed, K=6, D=5):
    rng = np.random.default_rng(seed)
    T = int(rng.integers(1, 4))
    R = int(rng.integers(1, 8))
    rs, rd = random_schema(rng, T, R)
    n_src = rng.integers(1, 25, T)
    n_dst = np.maximum(np.minimum(rng.integers(0, 15, T), n_src), 1)
    blk, et = random_block(rng, n_src, n_dst, rs, rd, int(rng.integers(1, 250)))
    sh = oracle.Shape.of(blk, rs, rd)
    xr = sh.src_rows + 7
    X = rng.standard_normal((xr, K))
    gid = rng.permutation(xr)[:sh.src_rows].astype(np.int32)
    W = rng.standard_normal((R, K, D))
    Wr = rng.standard_normal((T, K, D))
    return rng, sh, blk, et, rs, rd, X, gid, W, Wr


def test_spec_hand_example():
    """Edges (0->0), (1->0), f0 = [1,0], f1 = [3,2]: sum [4,2], mean [2,1]."""
    g = GOLD["aggregate_hand"]
    blk = LayerBlock(n_src=np.array([2], np.int32), n_dst=np.array([1], np.int32),
                     src_local=np.asarray(g["edges_src"], np.int32),
                     dst_local=np.asarray(g["edges_dst"], np.int32),
                     edge_id=np.array([0, 1], np.int64), src_global=[np.arange(2)])
    sh = oracle.Shape([0], [0], [2], [1], 2)
    X = np.asarray(g["features"], np.float64)
    et = np.zeros(2, np.int32)
    assert np.array_equal(oracle.aggregate_features(sh, blk, et, "sum", 2, X, None)[0], g["sum"][0])
    assert np.array_equal(oracle.aggregate_features(sh, blk, et, "mean", 2, X, None)[0], g["mean"][0])
    # identity projection keeps the aggregate
    out = oracle.project_aggregated(sh, 2, 2, np.array(g["mean"], float), X, None,
                                    np.eye(2)[None], None)
    assert np.array_equal(out["Z"][0], g["mean"][0])


@pytest.mark.parametrize("agg", ["sum", "mean"])
@pytest.mark.parametrize("seed", range(6))
def test_aggregate_features_dense_brute_force(seed, agg):
    rng, sh, blk, et, rs, rd, X, gid, W, Wr = case(seed)
    Xa = oracle.aggregate_features(sh, blk, et, agg, X.shape[1], X, gid)
    row = 0
    tso = np.concatenate([[0], np.cumsum(blk.n_src)])
    for r in range(sh.R):
        A = np.zeros((int(blk.n_dst[rd[r]]), int(blk.n_src[rs[r]])))
        m = et[blk.edge_id] == r
        np.add.at(A, (blk.dst_local[m], blk.src_local[m]), 1.0)
        if agg == "mean":
            deg = A.sum(1, keepdims=True)
            A = np.divide(A, deg, out=np.zeros_like(A), where=deg > 0)
        Xs = X[gid[tso[rs[r]]:tso[rs[r] + 1]]]
        np.testing.assert_allclose(Xa[row:row + A.shape[0]], A @ Xs, rtol=1e-12, atol=1e-12)
        row += A.shape[0]


@pytest.mark.parametrize("agg", ["sum", "mean"])
@pytest.mark.parametrize("seed", range(6))
def test_linearity_matches_project_first(seed, agg):
    """(A_r X) W_r = A_r (X W_r): forward Z and R0, and the weight gradients
    of the same loss through both orders."""
    rng, sh, blk, et, rs, rd, X, gid, W, Wr = case(100 + seed)
    K, D = W.shape[1], W.shape[2]
    Xa = oracle.aggregate_features(sh, blk, et, agg, K, X, gid)
    af = oracle.project_aggregated(sh, K, D, Xa, X, gid, W, Wr)
    csr = oracle.build(sh, blk, et)
    pf = oracle.project(sh, csr, K, D, 1, X, gid, W, Wr, None)
    Z = oracle.aggregate_fwd(sh, blk, et, csr, agg, D, 1, pf["Y"])["Z"]
    np.testing.assert_allclose(af["Z"], Z, rtol=1e-10, atol=1e-10)
    np.testing.assert_allclose(af["R0"], pf["R0"], rtol=1e-12, atol=1e-12)
    # backward: G is the gradient of every Z row (r, i) = G_t(r)[i] and of R0
    G = rng.standard_normal((sh.dst_rows, D))
    ab = oracle.project_aggregated_bwd(sh, K, D, Xa, X, gid, G)
    dY = oracle.aggregate_bwd(sh, blk, et, csr, agg, D, 1, G, pf["Y"])["dY"]
    pb = oracle.project_bwd(sh, csr, K, D, 1, X, gid, W, Wr, None, None, dY, G, None, None,
                            need_dX=False)
    np.testing.assert_allclose(ab["dW_rel"], pb["dW_rel"], rtol=1e-10, atol=1e-10)
    np.testing.assert_allclose(ab["dW_root"], pb["dW_root"], rtol=1e-10, atol=1e-10)


def test_weight_gradient_finite_differences():
    """dW of L = <G, fuse(Z, R0)> (no activation) by central differences."""
    rng, sh, blk, et, rs, rd, X, gid, W, Wr = case(7, K=3, D=2)
    K, D = 3, 2
    Xa = oracle.aggregate_features(sh, blk, et, "mean", K, X, gid)
    G = rng.standard_normal((sh.dst_rows, D))
    bias = np.zeros((sh.T, D))

    def loss(Wv, Wrv):
        o = oracle.project_aggregated(sh, K, D, Xa, X, gid, Wv, Wrv)
        return float(np.sum(G * oracle.fuse(sh, D, 0, o["Z"], o["R0"], bias)))

    ab = oracle.project_aggregated_bwd(sh, K, D, Xa, X, gid, G)
    h = 1e-6
    for (arr, grad) in ((W, ab["dW_rel"]), (Wr, ab["dW_root"])):
        for idx in [tuple(rng.integers(0, s) for s in arr.shape) for _ in range(6)]:
            p, m = arr.copy(), arr.copy()
            p[idx] += h
            m[idx] -= h
            num = ((loss(p, Wr) - loss(m, Wr)) if arr is W else (loss(W, p) - loss(W, m))) / (2 * h)
            assert abs(num - grad[idx]) <= 1e-6 * max(1.0, abs(num))
