"""Pins of the oracle's NEXT(2) functions, against
closed forms, special cases and finite differences -- not against retyped
formulas:

* multiplicative attention (agg "gat_mul", reading C23: per edge and head the
  logit s_src[col] * s_dst[row], then the segment softmax):
  - s_dst = 0 makes every logit 0: alpha = 1/deg and Z equals the oracle's
    MEAN aggregation (a different code path of O3);
  - R = T = H = 1 equals a dense masked-softmax attention in numpy;
  - sum alpha = 1, finite at logits of +-1e4;
  - central finite differences of <Z, G> for Y, s_src, s_dst.
* HAN semantic-attention fusion (O4', reading C22):
  - one relation per destination type: beta = 1, fusion identical to O4;
  - q = 0: beta uniform over the relations of a type (closed form);
  - Ws = 0: w_r = q . tanh(bs) for every relation (closed form);
  - sum beta = 1 per type;
  - finite differences of <G, fused sum> for Z, Ws, bs, q (O5a');
  - the per-merged-row gradient path of O5b (g_rows) equals the type-major
    path when every row of a type carries G_t;
  - full 2-layer RGAT + HAN and RGAT-multiplicative models: finite differences
    of the loss for every parameter (SPEC.md S:L411's model check).
The semantic choices themselves are "parity unpinned by the paper" (the paper
gives no attention or fusion formula)."""
import numpy as np
import pytest

import oracle
import oracle.model as om
from synth import random_block, random_schema

from test_oracle_aggregate import case
from test_oracle_backward import gmap, _fd, tiny_batch


# ---------------------------------------------------------------- gat_mul --
@pytest.mark.parametrize("seed", range(4))
def test_gat_mul_zero_dst_scores_is_mean(seed):
    H, D = 2, 8
    rng, sh, blk, et, csr, ytab, Y, rs, rd = case(600 + seed, D=D, H=H)
    ss = rng.standard_normal((csr["U"], H)) * 3
    sd = np.zeros((sh.rows, H))
    got = oracle.aggregate_fwd(sh, blk, et, csr, "gat_mul", D, H, Y, ss, sd)
    ref = oracle.aggregate_fwd(sh, blk, et, csr, "mean", D, 1, Y)
    np.testing.assert_allclose(got["Z"], ref["Z"], rtol=1e-13, atol=1e-14)


def test_gat_mul_dense_single_relation():
    rng = np.random.default_rng(7)
    rs, rd = np.array([0], np.int32), np.array([0], np.int32)
    n_src, n_dst = np.array([30], np.int32), np.array([12], np.int32)
    blk, et = random_block(rng, n_src, n_dst, rs, rd, 150)
    sh = oracle.Shape.of(blk, rs, rd)
    csr = oracle.build(sh, blk, et)
    D = 4
    X = rng.standard_normal((30, D))                   # source features
    Y = X[csr["y_src"]]
    k = rng.standard_normal(30)                        # key per source
    qv = rng.standard_normal(12)                       # query per destination
    got = oracle.aggregate_fwd(sh, blk, et, csr, "gat_mul", D, 1, Y, k[csr["y_src"]][:, None],
                               qv[:, None])
    A = np.zeros((12, 30))
    np.add.at(A, (blk.dst_local, blk.src_local), 1.0)  # edge multiplicities
    L = np.outer(qv, k)
    want = np.zeros((12, D))
    for i in range(12):
        if A[i].sum() == 0:
            continue
        m = L[i][A[i] > 0].max()
        p = A[i] * np.exp(L[i] - m)
        want[i] = (p / p.sum()) @ X
    np.testing.assert_allclose(got["Z"], want, rtol=1e-12, atol=1e-13)


def test_gat_mul_softmax_sums_to_one_and_is_finite():
    H, D = 2, 8
    rng, sh, blk, et, csr, ytab, Y, rs, rd = case(611, D=D, H=H, N=180)
    ss = rng.choice([-1e2, 1e2], size=(csr["U"], H))
    sd = rng.choice([-1e2, 1e2], size=(sh.rows, H))          # logits +-1e4
    fw = oracle.aggregate_fwd(sh, blk, et, csr, "gat_mul", D, H, Y, ss, sd)
    assert np.isfinite(fw["Z"]).all()
    nv = csr["row_ptr"][-1]
    rows = np.repeat(np.arange(sh.rows), np.diff(csr["row_ptr"]))
    s = np.zeros((sh.rows, H))
    np.add.at(s, rows, fw["alpha"][csr["eperm"][:nv]])
    has = np.diff(csr["row_ptr"]) > 0
    np.testing.assert_allclose(s[has], 1.0, atol=1e-12)


@pytest.mark.parametrize("seed", range(3))
def test_gat_mul_backward_finite_differences(seed):
    H, D = 2, 8
    rng, sh, blk, et, csr, ytab, Y, rs, rd = case(620 + seed, D=D, H=H)
    ss = rng.standard_normal((csr["U"], H))
    sd = rng.standard_normal((sh.rows, H))
    G = rng.standard_normal((sh.dst_rows, D))
    Gm = gmap(sh, csr, G)

    def loss():
        return float((oracle.aggregate_fwd(sh, blk, et, csr, "gat_mul", D, H, Y, ss, sd)["Z"]
                      * Gm).sum())

    b = oracle.aggregate_bwd(sh, blk, et, csr, "gat_mul", D, H, G, Y, ss, sd)
    for arr, grad in ((Y, b["dY"]), (ss, b["ds_src"]), (sd, b["ds_dst"])):
        for _ in range(8):
            idx = tuple(rng.integers(0, s) for s in arr.shape)
            num = _fd(loss, arr, idx)
            assert abs(num - grad[idx]) <= 1e-6 * max(1.0, abs(num)), (idx, num, grad[idx])


# -------------------------------------------------------------------- HAN --
def _han_case(seed, D=8, A=5, T=None, R=None):
    rng, sh, blk, et, csr, ytab, Y, rs, rd = case(seed, D=D, T=T, R=R)
    Z = rng.standard_normal((sh.rows, D))
    Ws = rng.standard_normal((D, A)) * 0.4
    bs = rng.standard_normal(A) * 0.3
    q = rng.standard_normal(A)
    return rng, sh, blk, et, csr, rs, rd, Z, Ws, bs, q


def test_han_one_relation_per_type_is_plain_fusion():
    rng = np.random.default_rng(3)
    T = 3
    rs = np.array([1, 2, 0], np.int32)
    rd = np.array([0, 1, 2], np.int32)                    # each type has one relation in
    n_src = np.array([9, 7, 8], np.int32)
    n_dst = np.array([4, 3, 5], np.int32)
    blk, et = random_block(rng, n_src, n_dst, rs, rd, 60)
    sh = oracle.Shape.of(blk, rs, rd)
    D = 6
    Z = rng.standard_normal((sh.rows, D))
    w, beta = oracle.sem_att(sh, D, Z, rng.standard_normal((D, 4)), rng.standard_normal(4),
                             rng.standard_normal(4))
    assert np.array_equal(beta, np.ones(3))
    R0 = rng.standard_normal((sh.dst_rows, D))
    bias = rng.standard_normal((T, D))
    assert np.array_equal(oracle.fuse(sh, D, 1, Z, R0, bias, beta=beta),
                          oracle.fuse(sh, D, 1, Z, R0, bias))


@pytest.mark.parametrize("seed", range(3))
def test_han_closed_forms(seed):
    rng, sh, blk, et, csr, rs, rd, Z, Ws, bs, q = _han_case(640 + seed)
    D, A = Z.shape[1], len(q)
    # q = 0: every w is 0 -> beta uniform over the relations of the type
    w, beta = oracle.sem_att(sh, D, Z, Ws, bs, np.zeros(A))
    assert np.array_equal(w, np.zeros(sh.R))
    for r in range(sh.R):
        assert abs(beta[r] - 1.0 / np.sum(sh.rel_dst == sh.rel_dst[r])) < 1e-15
    # Ws = 0: w_r = q . tanh(bs) for every relation with destinations
    w, beta = oracle.sem_att(sh, D, Z, np.zeros((D, A)), bs, q)
    for r in range(sh.R):
        want = float(q @ np.tanh(bs)) if sh.n_dst[sh.rel_dst[r]] > 0 else 0.0
        assert abs(w[r] - want) < 1e-14
    # sum beta = 1 per destination type
    w, beta = oracle.sem_att(sh, D, Z, Ws, bs, q)
    for t in np.unique(sh.rel_dst):
        assert abs(beta[sh.rel_dst == t].sum() - 1.0) < 1e-14


@pytest.mark.parametrize("seed", range(3))
def test_han_backward_finite_differences(seed):
    rng, sh, blk, et, csr, rs, rd, Z, Ws, bs, q = _han_case(650 + seed)
    D = Z.shape[1]
    G = rng.standard_normal((sh.dst_rows, D))

    def loss():   # <G, sum_r beta_r Z_r> (the pre-activation fused value without R0, bias)
        _, beta = oracle.sem_att(sh, D, Z, Ws, bs, q)
        return float((oracle.fuse(sh, D, 0, Z, None, np.zeros((sh.T, D)), beta=beta) * G).sum())

    _, beta = oracle.sem_att(sh, D, Z, Ws, bs, q)
    b = oracle.sem_att_bwd(sh, D, Z, Ws, bs, q, beta, G)
    for arr, grad in ((Z, b["dZ"]), (Ws, b["dWs"]), (bs, b["dbs"]), (q, b["dq"])):
        for _ in range(8):
            idx = tuple(rng.integers(0, s) for s in arr.shape)
            num = _fd(loss, arr, idx)
            assert abs(num - grad[idx]) <= 1e-6 * max(1.0, abs(num)), (idx, num, grad[idx])


@pytest.mark.parametrize("agg,H", [("mean", 1), ("gat", 2), ("gat_mul", 2)])
def test_aggregate_bwd_row_gradient_path(agg, H):
    D = 8
    rng, sh, blk, et, csr, ytab, Y, rs, rd = case(660, D=D, H=H)
    ss = rng.standard_normal((csr["U"], H))
    sd = rng.standard_normal((sh.rows, H))
    G = rng.standard_normal((sh.dst_rows, D))
    a = oracle.aggregate_bwd(sh, blk, et, csr, agg, D, H, G, Y, ss, sd)
    b = oracle.aggregate_bwd(sh, blk, et, csr, agg, D, H, gmap(sh, csr, G), Y, ss, sd,
                             g_rows=True)
    for k in a:
        assert np.array_equal(a[k], b[k]), k


@pytest.mark.parametrize("variant", ["han", "mul", "han_mul", "rgcn_han"])
def test_model_finite_differences_next2(variant):
    model = "rgcn" if variant.startswith("rgcn") else "rgat"
    layers, et, rs, rd, X0, gid, params, labels, H = tiny_batch(model, 9)
    agg = "gat_mul" if "mul" in variant else ("gat" if model == "rgat" else "mean")
    rng = np.random.default_rng(1)
    if "han" in variant:
        D = params["layers"][0]["W_rel"].shape[2]
        for lay in params["layers"]:
            lay.update(sem_W=rng.standard_normal((D, 5)) * 0.4, sem_b=rng.standard_normal(5) * 0.3,
                       sem_q=rng.standard_normal(5))
    fw = om.forward(layers, et, rs, rd, X0, gid, params, agg, H, labels=labels)
    g = om.backward(fw, layers, et, params, labels, agg, H)
    loss = lambda: om.forward(layers, et, rs, rd, X0, gid, params, agg, H, labels=labels)["loss"]
    checks = [(params["Wc"], g["Wc"]), (params["bc"], g["bc"])]
    for l in range(2):
        for k in ("W_rel", "W_root", "bias", "att", "sem_W", "sem_b", "sem_q"):
            if params["layers"][l].get(k) is not None:
                checks.append((params["layers"][l][k], g["layers"][l][k]))
    for arr, grad in checks:
        for _ in range(4):
            idx = tuple(rng.integers(0, s) for s in arr.shape)
            num = _fd(loss, arr, idx)
            assert abs(num - grad[idx]) <= 1e-4 * max(1e-3, abs(num)) + 1e-9, (idx, num, grad[idx])
