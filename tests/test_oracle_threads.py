"""The oracle's OpenMP loops (oracle_set_threads) write disjoint outputs and
keep the serial summation order: projection forward and backward are
BIT-IDENTICAL at 1 and 4 threads (RGCN with root weights and gathered rows,
RGAT with attention vectors).  The bench times the oracle at the box's core
count (cpu_baseline), the tests run it at 1 thread."""
import numpy as np
import pytest

import oracle
from synth import random_block, random_schema


def _case(seed, att_on):
    rng = np.random.default_rng(seed)
    T, R, K, D, H = 3, 7, 16, 32, 4
    rs, rd = random_schema(rng, T, R)
    n_src = rng.integers(40, 120, T)
    n_dst = np.minimum(rng.integers(10, 40, T), n_src)
    blk, et = random_block(rng, n_src, n_dst, rs, rd, 900)
    sh = oracle.Shape.of(blk, rs, rd)
    csr = oracle.build(sh, blk, et)
    xr = sh.src_rows + 9
    X = rng.standard_normal((xr, K))
    gid = rng.permutation(xr)[:sh.src_rows].astype(np.int32)
    W = rng.standard_normal((R, K, D))
    Wr = rng.standard_normal((T, K, D))
    att = rng.standard_normal((R, 2, D)) if att_on else None
    return rng, sh, csr, K, D, H, X, gid, W, Wr, att


@pytest.mark.parametrize("att_on", [False, True])
def test_projection_bit_identical_across_threads(att_on):
    rng, sh, csr, K, D, H, X, gid, W, Wr, att = _case(7, att_on)
    U = csr["U"]
    dY = rng.standard_normal((U, D))
    G = rng.standard_normal((sh.dst_rows, D))
    dss = rng.standard_normal((U, H))
    dsd = rng.standard_normal((sh.rows, H))
    out = []
    for n in (1, 4):
        oracle.set_threads(n)
        try:
            p = oracle.project(sh, csr, K, D, H, X, gid, W, Wr, att)
            b = oracle.project_bwd(sh, csr, K, D, H, X, gid, W, Wr, att, p["Y"], dY, G, dss, dsd)
        finally:
            oracle.set_threads(1)
        out.append((p, b))
    (p1, b1), (p4, b4) = out
    for k in p1:
        assert np.array_equal(p1[k], p4[k]), k
    for k in b1:
        if b1[k] is not None:
            assert np.array_equal(b1[k], b4[k]), k


def test_project_bwd_matches_matrix_form():
    """dW_r = X_s(r)[y_src]^T dYt_r (+ the s_dst chain), dW_root,t = X_t^T G_t,
    datt, dX -- written as dense numpy matrix products (independent of the
    oracle's loops), with attention and root weights both on."""
    rng, sh, csr, K, D, H, X, gid, W, Wr, att = _case(11, True)
    U = csr["U"]
    dh = D // H
    dY = rng.standard_normal((U, D))
    G = rng.standard_normal((sh.dst_rows, D))
    dss = rng.standard_normal((U, H))
    dsd = rng.standard_normal((sh.rows, H))
    p = oracle.project(sh, csr, K, D, H, X, gid, W, Wr, att)
    b = oracle.project_bwd(sh, csr, K, D, H, X, gid, W, Wr, att, p["Y"], dY, G, dss, dsd)
    tso = np.concatenate([[0], np.cumsum(sh.n_src)])
    tdo = np.concatenate([[0], np.cumsum(sh.n_dst)])
    dW = np.zeros_like(W)
    datt = np.zeros_like(att)
    dX = np.zeros_like(X)
    row0 = 0
    for r in range(sh.R):
        a, e = csr["rel_y_off"][r], csr["rel_y_off"][r + 1]
        rows = gid[tso[sh.rel_src[r]] + csr["y_src"][a:e]]
        dYt = dY[a:e] + np.repeat(dss[a:e], dh, axis=1) * att[r, 0]
        dW[r] += X[rows].T @ dYt
        datt[r, 0] += (np.repeat(dss[a:e], dh, axis=1) * p["Y"][a:e]).sum(0)
        np.add.at(dX, rows, dYt @ W[r].T)
        t = sh.rel_dst[r]
        nt = sh.n_dst[t]
        drows = gid[tso[t] + np.arange(nt)]
        gd = np.repeat(dsd[row0:row0 + nt], dh, axis=1) * att[r, 1]
        dW[r] += X[drows].T @ gd
        datt[r, 1] += (np.repeat(dsd[row0:row0 + nt], dh, axis=1) * (X[drows] @ W[r])).sum(0)
        np.add.at(dX, drows, gd @ W[r].T)
        row0 += nt
    dWr = np.zeros_like(Wr)
    for t in range(sh.T):
        drows = gid[tso[t] + np.arange(sh.n_dst[t])]
        dWr[t] = X[drows].T @ G[tdo[t]:tdo[t + 1]]
        np.add.at(dX, drows, G[tdo[t]:tdo[t + 1]] @ Wr[t].T)
    np.testing.assert_allclose(b["dW_rel"], dW, rtol=1e-12, atol=1e-11)
    np.testing.assert_allclose(b["dW_root"], dWr, rtol=1e-12, atol=1e-11)
    np.testing.assert_allclose(b["datt"], datt, rtol=1e-12, atol=1e-11)
    np.testing.assert_allclose(b["dX"], dX, rtol=1e-12, atol=1e-11)
