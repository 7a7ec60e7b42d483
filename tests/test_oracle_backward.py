"""Pins of the oracle's backward functions: SPEC.md hand examples, the adjoint
identity for the linear (sum/mean) aggregation, and central finite
differences of the oracle's own forward (an independent function) for GAT,
fusion, projection and the full 2-layer model."""
import json
import os

import numpy as np
import pytest

import oracle
import oracle.model as om
from synth import random_block, random_schema, make_params, CONFIGS
from synth.sampler import LayerBlock

from test_oracle_aggregate import case, _blk

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def gmap(sh, csr, G):
    """dZ[(r,i)] = G_{t(r)}[i] laid out on the merged rows."""
    tdo = np.concatenate([[0], np.cumsum(sh.n_dst)])
    out = np.zeros((sh.rows, G.shape[1]))
    for r in range(sh.R):
        t = sh.rel_dst[r]
        a = csr["rel_row_off"][r]
        out[a:a + sh.n_dst[t]] = G[tdo[t]:tdo[t + 1]]
    return out


def test_spec_backward_hand():
    g = GOLD["backward_hand"]
    go = np.asarray(g["grad_out"])
    blk = _blk([0], [0], [0], [1], [1])
    sh = oracle.Shape([0], [0], [1], [1], 1)
    csr = oracle.build(sh, blk, np.zeros(1, np.int32))
    dY = oracle.aggregate_bwd(sh, blk, np.zeros(1, np.int32), csr, "sum", 2, 1, go, np.zeros((1, 2)))["dY"]
    assert np.array_equal(dY, np.asarray(g["single_sum_grad_in"]))
    blk = _blk([0, 1], [0, 0], [0, 1], [2], [1])
    sh = oracle.Shape([0], [0], [2], [1], 2)
    csr = oracle.build(sh, blk, np.zeros(2, np.int32))
    dY = oracle.aggregate_bwd(sh, blk, np.zeros(2, np.int32), csr, "mean", 2, 1, go, np.zeros((2, 2)))["dY"]
    assert np.array_equal(dY, np.asarray(g["two_mean_grad_in"]))


@pytest.mark.parametrize("seed", range(6))
@pytest.mark.parametrize("agg", ["sum", "mean"])
def test_adjoint_identity(seed, agg):
    rng, sh, blk, et, csr, ytab, Y, rs, rd = case(40 + seed)
    G = rng.standard_normal((sh.dst_rows, Y.shape[1]))
    Z = oracle.aggregate_fwd(sh, blk, et, csr, agg, Y.shape[1], 1, Y)["Z"]
    dY = oracle.aggregate_bwd(sh, blk, et, csr, agg, Y.shape[1], 1, G, Y)["dY"]
    lhs = float((Z * gmap(sh, csr, G)).sum())
    rhs = float((Y * dY).sum())
    assert abs(lhs - rhs) <= 1e-11 * max(1.0, abs(lhs))


def _fd(f, x, idx, h=1e-6):
    x0 = x[idx]
    x[idx] = x0 + h
    fp = f()
    x[idx] = x0 - h
    fm = f()
    x[idx] = x0
    return (fp - fm) / (2 * h)


@pytest.mark.parametrize("seed", range(4))
def test_gat_backward_finite_differences(seed):
    H, D = 2, 8
    rng, sh, blk, et, csr, ytab, Y, rs, rd = case(60 + seed, D=D, H=H)
    ss = rng.standard_normal((csr["U"], H))
    sd = rng.standard_normal((sh.rows, H))
    G = rng.standard_normal((sh.dst_rows, D))
    Gm = gmap(sh, csr, G)

    def loss():
        return float((oracle.aggregate_fwd(sh, blk, et, csr, "gat", D, H, Y, ss, sd)["Z"] * Gm).sum())

    b = oracle.aggregate_bwd(sh, blk, et, csr, "gat", D, H, G, Y, ss, sd)
    for arr, grad in ((Y, b["dY"]), (ss, b["ds_src"]), (sd, b["ds_dst"])):
        for _ in range(6):
            idx = tuple(rng.integers(0, s) for s in arr.shape)
            num = _fd(loss, arr, idx)
            assert abs(num - grad[idx]) <= 1e-4 * max(1.0, abs(num)), (idx, num, grad[idx])


def test_fuse_backward_finite_differences():
    rng, sh, blk, et, csr, ytab, Y, rs, rd = case(71, D=6)
    Z = rng.standard_normal((sh.rows, 6))
    R0 = rng.standard_normal((sh.dst_rows, 6))
    b = rng.standard_normal((sh.T, 6))
    dH = rng.standard_normal((sh.dst_rows, 6))
    Hh = oracle.fuse(sh, 6, 1, Z, R0, b)
    G, db = oracle.fuse_bwd(sh, 6, 1, dH, Hh)
    loss = lambda: float((oracle.fuse(sh, 6, 1, Z, R0, b) * dH).sum())
    for _ in range(8):
        idx = tuple(rng.integers(0, s) for s in R0.shape)
        assert abs(_fd(loss, R0, idx) - G[idx]) < 1e-6
        idx = tuple(rng.integers(0, s) for s in b.shape)
        assert abs(_fd(loss, b, idx) - db[idx]) < 1e-6
    # dZ of every relation row equals G of its destination type
    Gm = gmap(sh, csr, G)
    for _ in range(8):
        idx = tuple(rng.integers(0, s) for s in Z.shape)
        assert abs(_fd(loss, Z, idx) - Gm[idx]) < 1e-6


@pytest.mark.parametrize("att_on", [False, True])
def test_project_backward_finite_differences(att_on):
    K, D, H = 5, 8, 2
    rng, sh, blk, et, csr, ytab, Y, rs, rd = case(81, D=D, H=H)
    X = rng.standard_normal((sh.src_rows, K))
    W = rng.standard_normal((sh.R, K, D))
    Wr = None if att_on else rng.standard_normal((sh.T, K, D))
    att = rng.standard_normal((sh.R, 2, D)) if att_on else None
    pr = oracle.project(sh, csr, K, D, H, X, None, W, Wr, att)
    dY = rng.standard_normal(pr["Y"].shape)
    G = rng.standard_normal(pr["R0"].shape)
    dss = rng.standard_normal(pr["s_src"].shape) if att_on else np.zeros(pr["s_src"].shape)
    dsd = rng.standard_normal(pr["s_dst"].shape) if att_on else np.zeros(pr["s_dst"].shape)

    def loss():
        p = oracle.project(sh, csr, K, D, H, X, None, W, Wr, att)
        v = (p["Y"] * dY).sum()
        if Wr is not None:
            v += (p["R0"] * G).sum()
        if att_on:
            v += (p["s_src"] * dss).sum() + (p["s_dst"] * dsd).sum()
        return float(v)

    b = oracle.project_bwd(sh, csr, K, D, H, X, None, W, Wr, att, pr["Y"], dY, G, dss, dsd)
    pairs = [(X, b["dX"]), (W, b["dW_rel"])]
    if Wr is not None:
        pairs.append((Wr, b["dW_root"]))
    if att_on:
        pairs.append((att, b["datt"]))
    for arr, grad in pairs:
        for _ in range(8):
            idx = tuple(rng.integers(0, s) for s in arr.shape)
            num = _fd(loss, arr, idx)
            assert abs(num - grad[idx]) <= 1e-5 * max(1.0, abs(num)), (idx, num, grad[idx])


def tiny_batch(model, seed):
    """A 2-layer mini-batch on a tiny random heterograph (chained blocks)."""
    rng = np.random.default_rng(seed)
    T, R = 3, 5
    rs, rd = random_schema(rng, T, R)
    rd[0] = 0
    n2 = np.array([4, 0, 0], np.int32)                 # seeds of type 0
    n1 = np.array([4, 5, 3], np.int32)
    n0 = np.array([9, 8, 6], np.int32)
    b1, et = random_block(rng, n1, n2, rs, rd, 20)
    b0, _ = random_block(rng, n0, n1, rs, rd, 60)
    b0.edge_id = rng.choice(np.arange(len(et)), size=60)  # re-draw ids consistent with et
    # make b0 consistent: pick relation per edge from et, endpoints within range
    r = et[b0.edge_id]
    ok = (n0[rs[r]] > 0) & (n1[rd[r]] > 0)
    b0.edge_id = b0.edge_id[ok]
    r = r[ok]
    b0.src_local = np.array([rng.integers(0, n0[rs[k]]) for k in r], np.int32)
    b0.dst_local = np.array([rng.integers(0, n1[rd[k]]) for k in r], np.int32)
    K, D, C, H = 6, 8, 3, (2 if model == "rgat" else 1)
    X0 = rng.standard_normal((int(n0.sum()) + 2, K))
    gid = rng.permutation(int(n0.sum()) + 2)[:int(n0.sum())].astype(np.int32)
    params = dict(layers=[], Wc=rng.standard_normal((D, C)), bc=rng.standard_normal(C))
    for l in range(2):
        k = K if l == 0 else D
        params["layers"].append(dict(
            W_rel=rng.standard_normal((R, k, D)) * 0.5,
            W_root=rng.standard_normal((T, k, D)) * 0.5 if model == "rgcn" else None,
            bias=rng.standard_normal((T, D)) * 0.1,
            att=rng.standard_normal((R, 2, D)) * 0.5 if model == "rgat" else None))
    labels = rng.integers(0, C, 4)
    return [b0, b1], et, rs, rd, X0, gid, params, labels, H


@pytest.mark.parametrize("model", ["rgcn", "rgat"])
def test_model_finite_differences(model):
    layers, et, rs, rd, X0, gid, params, labels, H = tiny_batch(model, 5)
    agg = "gat" if model == "rgat" else "mean"
    fw = om.forward(layers, et, rs, rd, X0, gid, params, agg, H, labels=labels)
    g = om.backward(fw, layers, et, params, labels, agg, H)
    loss = lambda: om.forward(layers, et, rs, rd, X0, gid, params, agg, H, labels=labels)["loss"]
    rng = np.random.default_rng(0)
    checks = [(params["Wc"], g["Wc"]), (params["bc"], g["bc"])]
    for l in range(2):
        for k in ("W_rel", "W_root", "bias", "att"):
            if params["layers"][l][k] is not None:
                checks.append((params["layers"][l][k], g["layers"][l][k]))
    for arr, grad in checks:
        for _ in range(5):
            idx = tuple(rng.integers(0, s) for s in arr.shape)
            num = _fd(loss, arr, idx)
            assert abs(num - grad[idx]) <= 1e-4 * max(1e-3, abs(num)) + 1e-9, (idx, num, grad[idx])
