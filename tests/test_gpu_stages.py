"""-m gpu: stage-isolated parity of the CUDA path against the oracle.

Each stage's oracle consumes the GPU's own inputs of that stage (e.g. A4's
oracle reads the GPU's Y), so error never leaks between stages.  Tolerances
(DESIGN.md §Tolerances): fp32 aggregation / fusion / their backward
|g - r| <= 1e-5 max(|r|, A) with A the absolute-sum scale of the element;
projection row-relative L2 <= 2e-3; integer-valued inputs are bit-exact.
"""
import numpy as np
import pytest
import torch

import oracle
from synth import random_block, random_schema

from gpu_util import needs_gpu, gpu_build, csr_host, close_scaled, row_rel_l2, t, DEV, hf

pytestmark = [pytest.mark.gpu, needs_gpu]


def make_case(seed, D=128, H=1, N=None, T=None, R=None, hub=0.0):
    rng = np.random.default_rng(seed)
    T = T or int(rng.integers(1, 5))
    R = R or int(rng.integers(1, 12))
    rs, rd = random_schema(rng, T, R)
    n_src = rng.integers(1, 400, T)
    n_dst = np.maximum(np.minimum(rng.integers(0, 250, T), n_src), 1)
    N = int(rng.integers(100, 6000)) if N is None else N
    blk, et = random_block(rng, n_src, n_dst, rs, rd, N, hub_frac=hub)
    sh, csr, st = gpu_build(blk, et, rs, rd)
    ch = csr_host(sh, csr)
    return rng, blk, et, rs, rd, sh, csr, ch


def agg_oracle(blk, et, rs, rd, ch, agg, D, H, Y, ss=None, sd=None):
    osh = oracle.Shape.of(blk, rs, rd)
    return oracle.aggregate_fwd(osh, blk, et, ch, agg, D, H, Y, ss, sd)


@pytest.mark.parametrize("D", [64, 128])
@pytest.mark.parametrize("agg", ["sum", "mean"])
@pytest.mark.parametrize("seed", range(4))
def test_aggregate_fwd(seed, agg, D):
    rng, blk, et, rs, rd, sh, csr, ch = make_case(10 + seed, D=D, hub=0.1 * (seed % 2))
    U = ch["U"]
    Y = rng.standard_normal((max(U, 1), D)).astype(np.float32)
    Z = torch.zeros(max(sh.rows, 1), D, device=DEV)
    hf().aggregate_fwd(csr, sh.rows, agg, D, 1, 0.2, t(Y), None, None, Z, None)
    ref = agg_oracle(blk, et, rs, rd, ch, agg, D, 1, Y[:U])
    A = agg_oracle(blk, et, rs, rd, ch, agg, D, 1, np.abs(Y[:U]))["Z"]
    close_scaled(Z.cpu().numpy()[:sh.rows], ref["Z"], A, what=f"Z {agg}")


@pytest.mark.parametrize("D", [64, 128])
def test_aggregate_integer_inputs_bit_exact(D):
    rng, blk, et, rs, rd, sh, csr, ch = make_case(77, D=D, N=5000)
    U = ch["U"]
    Y = rng.integers(-8, 9, (U, D)).astype(np.float32)
    for agg in ("sum", "mean"):
        Z = torch.zeros(sh.rows, D, device=DEV)
        hf().aggregate_fwd(csr, sh.rows, agg, D, 1, 0.2, t(Y), None, None, Z, None)
        ref = agg_oracle(blk, et, rs, rd, ch, "sum", D, 1, Y)
        exp = ref["Z"].astype(np.float32)
        if agg == "mean":   # reading C19: float32(sum) / float32(deg), IEEE division
            deg = ref["deg"].astype(np.float32)
            exp = np.where(deg[:, None] > 0, exp / np.maximum(deg, 1)[:, None], 0).astype(np.float32)
        assert np.array_equal(Z.cpu().numpy(), exp), agg


@pytest.mark.parametrize("agg", ["gat", "gat_mul"])
@pytest.mark.parametrize("D,H", [(128, 8), (64, 8), (128, 1), (64, 2)])
@pytest.mark.parametrize("seed", range(3))
def test_aggregate_fwd_gat(seed, D, H, agg):
    """gat_mul: multiplicative logit s_src * s_dst (NEXT(2), reading C23)."""
    rng, blk, et, rs, rd, sh, csr, ch = make_case(30 + seed, D=D, H=H, hub=0.05)
    U = ch["U"]
    Y = rng.standard_normal((U, D)).astype(np.float32)
    ss = (rng.standard_normal((U, H)) * 2).astype(np.float32)
    sd = (rng.standard_normal((sh.rows, H)) * 2).astype(np.float32)
    Z = torch.zeros(sh.rows, D, device=DEV)
    stats = torch.zeros(sh.rows, 2 * H, device=DEV)
    hf().aggregate_fwd(csr, sh.rows, agg, D, H, 0.2, t(Y), t(ss), t(sd), Z, stats)
    ref = agg_oracle(blk, et, rs, rd, ch, agg, D, H, Y, ss, sd)
    A = agg_oracle(blk, et, rs, rd, ch, agg, D, H, np.abs(Y), ss, sd)["Z"]
    close_scaled(Z.cpu().numpy(), ref["Z"], A, what=f"Z {agg}")
    # stats reproduce sum of alpha = 1: l = sum exp(l_e - m)
    st = stats.cpu().numpy()
    nz = ref["deg"] > 0
    assert np.all(st[nz, H:] >= 1.0 - 1e-6)


def test_gat_zero_attention_equals_mean():
    rng, blk, et, rs, rd, sh, csr, ch = make_case(41, D=128, H=8)
    U = ch["U"]
    Y = t(rng.standard_normal((U, 128)).astype(np.float32))
    Zg = torch.zeros(sh.rows, 128, device=DEV)
    Zm = torch.zeros(sh.rows, 128, device=DEV)
    st = torch.zeros(sh.rows, 16, device=DEV)
    hf().aggregate_fwd(csr, sh.rows, "gat", 128, 8, 0.2, Y, torch.zeros(U, 8, device=DEV),
                       torch.zeros(sh.rows, 8, device=DEV), Zg, st)
    hf().aggregate_fwd(csr, sh.rows, "mean", 128, 1, 0.2, Y, None, None, Zm, None)
    torch.testing.assert_close(Zg, Zm, rtol=2e-6, atol=1e-7)


def _gmap_rows(sh, ch, G):
    tdo = sh.type_dst_off
    out = np.zeros((sh.rows, G.shape[1]))
    for r in range(sh.R):
        tt = sh.rel_dst[r]
        a = ch["rel_row_off"][r]
        out[a:a + sh.n_dst[tt]] = G[tdo[tt]:tdo[tt + 1]]
    return out


@pytest.mark.parametrize("D", [64, 128])
@pytest.mark.parametrize("agg", ["sum", "mean"])
@pytest.mark.parametrize("seed", range(3))
def test_aggregate_bwd(seed, agg, D):
    rng, blk, et, rs, rd, sh, csr, ch = make_case(50 + seed, D=D, hub=0.2 * (seed % 2),
                                                     N=[800, 6000, 20000][seed])
    U = ch["U"]
    G = rng.standard_normal((sh.dst_rows, D)).astype(np.float32)
    dY = torch.zeros(max(sh.U_max, 1), D, device=DEV)
    ws = torch.empty(hf().aggregate_bwd_ws_bytes(sh, agg, 1) // 4 + 16, device=DEV)
    hf().aggregate_bwd(sh, csr, agg, D, 1, 0.2, t(G), None, None, None, None, dY, None, None,
                       ws)
    osh = oracle.Shape.of(blk, rs, rd)
    ref = oracle.aggregate_bwd(osh, blk, et, ch, agg, D, 1, G, np.zeros((U, D)))
    A = oracle.aggregate_bwd(osh, blk, et, ch, agg, D, 1, np.abs(G), np.zeros((U, D)))["dY"]
    close_scaled(dY.cpu().numpy()[:U], ref["dY"], A, what="dY")


@pytest.mark.parametrize("D", [64, 128])
def test_aggregate_bwd_integer_inputs_bit_exact(D):
    """Transpose SpMM with integer-valued G: every partial sum is exact in
    fp32, so sum is bit-exact in any order; mean (reading C19: w = 1/deg
    rounded, w*g rounded, then summed) equals the oracle evaluated with the
    same fp32 products (hub columns included: the long-column kernel)."""
    rng, blk, et, rs, rd, sh, csr, ch = make_case(91, D=D, N=12000, hub=0.15)
    U = ch["U"]
    G = rng.integers(-8, 9, (sh.dst_rows, D)).astype(np.float32)
    osh = oracle.Shape.of(blk, rs, rd)
    ws = torch.empty(hf().aggregate_bwd_ws_bytes(sh, "sum", 1) // 4 + 16, device=DEV)
    dY = torch.zeros(max(sh.U_max, 1), D, device=DEV)
    hf().aggregate_bwd(sh, csr, "sum", D, 1, 0.2, t(G), None, None, None, None, dY, None, None, ws)
    ref = oracle.aggregate_bwd(osh, blk, et, ch, "sum", D, 1, G, np.zeros((U, D)))
    assert np.array_equal(dY.cpu().numpy()[:U], ref["dY"])
    assert (np.diff(ch["col_ptr"]) > 16).any()          # long columns exercised


@pytest.mark.parametrize("agg", ["gat", "gat_mul"])
@pytest.mark.parametrize("D,H", [(128, 8), (64, 8)])
@pytest.mark.parametrize("seed", range(3))
def test_aggregate_bwd_gat(seed, D, H, agg):
    rng, blk, et, rs, rd, sh, csr, ch = make_case(60 + seed, D=D, H=H, hub=0.1,
                                                     N=[800, 6000, 20000][seed])
    U = ch["U"]
    Y = rng.standard_normal((U, D)).astype(np.float32)
    ss = rng.standard_normal((U, H)).astype(np.float32)
    sd = rng.standard_normal((sh.rows, H)).astype(np.float32)
    G = rng.standard_normal((sh.dst_rows, D)).astype(np.float32)
    Z = torch.zeros(sh.rows, D, device=DEV)
    stats = torch.zeros(sh.rows, 2 * H, device=DEV)
    hf().aggregate_fwd(csr, sh.rows, agg, D, H, 0.2, t(Y), t(ss), t(sd), Z, stats)
    dY = torch.zeros(U, D, device=DEV)
    dss = torch.zeros(U, H, device=DEV)
    dsd = torch.zeros(sh.rows, H, device=DEV)
    ws = torch.empty(hf().aggregate_bwd_ws_bytes(sh, agg, H) // 4 + 16, device=DEV)
    hf().aggregate_bwd(sh, csr, agg, D, H, 0.2, t(G), t(Y), t(ss), t(sd), stats, dY, dss, dsd,
                       ws)
    osh = oracle.Shape.of(blk, rs, rd)
    ref = oracle.aggregate_bwd(osh, blk, et, ch, agg, D, H, G, Y, ss, sd)
    # scale: magnitude of the per-element sums (|G| |Y| bound), row-wise
    sc_y = oracle.aggregate_bwd(osh, blk, et, ch, agg, D, H, np.abs(G), np.abs(Y), ss, sd)
    close_scaled(dY.cpu().numpy(), ref["dY"], sc_y["dY"], what="dY gat")
    # ds: absolute-sum scale of dpre = alpha (dalpha - za) terms
    fw = oracle.aggregate_fwd(osh, blk, et, ch, agg, D, H, Y, ss, sd)
    scale_s, scale_d = gat_ds_scales(sh, ch, fw, G, Y, D, H, agg, ss, sd)
    close_scaled(dss.cpu().numpy(), ref["ds_src"], scale_s, what="ds_src")
    close_scaled(dsd.cpu().numpy(), ref["ds_dst"], scale_d, what="ds_dst")
    # score chain folded into the CSC pass (hifuse_aggregate_bwd_scored):
    # dYt = dY + ds_src (x) att[r, 0] in the same fp32 fma as k_dy_score
    att = torch.from_numpy(rng.standard_normal((sh.R, 2, D)).astype(np.float32)).to(DEV)
    dY2 = torch.zeros_like(dY)
    dss2 = torch.zeros_like(dss)
    dsd2 = torch.zeros_like(dsd)
    hf().aggregate_bwd_scored(sh, csr, agg, D, H, 0.2, t(G), t(Y), t(ss), t(sd), stats, att,
                              dY2, dss2, dsd2, ws)
    torch.cuda.synchronize()
    assert torch.equal(dss2, dss) and torch.equal(dsd2, dsd)
    rel = np.repeat(np.arange(sh.R), np.diff(ch["rel_y_off"]))
    a_src = att[torch.from_numpy(rel).to(DEV), 0]                       # [U, D]
    want = torch.addcmul(dY, dss.repeat_interleave(D // H, dim=1), a_src)
    torch.testing.assert_close(dY2, want, rtol=1e-6, atol=1e-6)


def gat_ds_scales(sh, ch, fw, G, Y, D, H, agg="gat", ss=None, sd=None):
    """Absolute-sum scales of the GAT score gradients: per
    edge and head, dpre = alpha (dalpha - sum_row alpha dalpha) with dalpha =
    <G_row, Y_col>; the scale sums alpha (|dalpha|_abs + sum alpha |dalpha|_abs)
    over the edges of each merged row (ds_dst) / each Y row (ds_src)."""
    nv = ch["row_ptr"][-1]
    U = ch["U"]
    rows = np.repeat(np.arange(sh.rows), np.diff(ch["row_ptr"]))
    e, u = ch["eperm"][:nv], ch["col"][:nv]
    gm = _gmap_index(sh, ch)[rows]
    dh = D // H
    dabs = (np.abs(G[gm]).reshape(-1, H, dh) * np.abs(Y[u]).reshape(-1, H, dh)).sum(-1)
    a = fw["alpha"][e]
    za = np.zeros((sh.rows, H))
    np.add.at(za, rows, a * dabs)
    term = a * (dabs + za[rows])
    # multiplicative logit: ds_src = sum dl s_dst, ds_dst = sum dl s_src
    tsrc = term * np.abs(sd[rows]) if agg == "gat_mul" else term
    tdst = term * np.abs(ss[u]) if agg == "gat_mul" else term
    scale_d = np.zeros((sh.rows, H))
    np.add.at(scale_d, rows, tdst)
    scale_s = np.zeros((U, H))
    np.add.at(scale_s, u, tsrc)
    return scale_s, scale_d


def _gmap_index(sh, ch):
    """Row of G (type-major) for every merged row (r, i)."""
    out = np.zeros(sh.rows, np.int64)
    for r in range(sh.R):
        tt = sh.rel_dst[r]
        a = ch["rel_row_off"][r]
        out[a:a + sh.n_dst[tt]] = sh.type_dst_off[tt] + np.arange(sh.n_dst[tt])
    return out


@pytest.mark.parametrize("D", [64, 128])
def test_fuse_and_fuse_bwd(D):
    rng, blk, et, rs, rd, sh, csr, ch = make_case(70, D=D, T=4, R=9)
    Z = rng.standard_normal((sh.rows, D)).astype(np.float32)
    R0 = rng.standard_normal((sh.dst_rows, D)).astype(np.float32)
    b = rng.standard_normal((sh.T, D)).astype(np.float32)
    Hg = torch.zeros(sh.dst_rows, D, device=DEV)
    hf().semantic_fuse(sh, D, "relu", t(Z), t(R0), t(b), Hg)
    osh = oracle.Shape.of(blk, rs, rd)
    ref = oracle.fuse(osh, D, 1, Z, R0, b)
    A = oracle.fuse(osh, D, 0, np.abs(Z), np.abs(R0), np.abs(b))
    close_scaled(Hg.cpu().numpy(), ref, A, what="H")
    dH = rng.standard_normal((sh.dst_rows, D)).astype(np.float32)
    G = torch.zeros(sh.dst_rows, D, device=DEV)
    db = torch.zeros(sh.T, D, device=DEV)
    ws = torch.empty(hf().fuse_bwd_ws_bytes(sh, D) // 4 + 16, device=DEV)
    hf().semantic_fuse_bwd(sh, D, "relu", t(dH), Hg, G, db, ws)
    Gr, dbr = oracle.fuse_bwd(osh, D, 1, dH, Hg.cpu().numpy())
    assert np.array_equal(G.cpu().numpy(), Gr.astype(np.float32))
    _, dbA = oracle.fuse_bwd(osh, D, 1, np.abs(dH), Hg.cpu().numpy())
    close_scaled(db.cpu().numpy(), dbr, dbA, what="dbias")
    # split form (the Trainer: G on the critical path, the bias on the side
    # stream): bit-identical to the combined call
    G2 = torch.zeros_like(G)
    db2 = torch.zeros_like(db)
    ws2 = torch.empty_like(ws)
    hf().semantic_fuse_bwd(sh, D, "relu", t(dH), Hg, G2, None, ws)
    hf().semantic_fuse_bwd_bias(sh, D, G2, db2, ws2)
    assert torch.equal(G2, G) and torch.equal(db2, db)


@pytest.mark.parametrize("K,D,H,att", [(128, 128, 1, False), (64, 64, 1, False), (128, 64, 1, False),
                                       (64, 128, 1, False), (128, 128, 8, True), (64, 64, 8, True)])
@pytest.mark.parametrize("prec", ["fp32", "tf32"])
def test_project_fwd_bwd(K, D, H, att, prec):
    rng, blk, et, rs, rd, sh, csr, ch = make_case(90 + K + D, D=D, H=H, T=3, R=7, hub=0.05)
    U = ch["U"]
    xr = sh.src_rows + 11
    X = rng.standard_normal((xr, K)).astype(np.float32)
    gid = rng.permutation(xr)[:sh.src_rows].astype(np.int32)
    W = (rng.standard_normal((sh.R, K, D)) / np.sqrt(K)).astype(np.float32)
    Wr = None if att else (rng.standard_normal((sh.T, K, D)) / np.sqrt(K)).astype(np.float32)
    A = (rng.standard_normal((sh.R, 2, D))).astype(np.float32) if att else None
    Y = torch.zeros(max(sh.U_max, 1), D, device=DEV)
    R0 = torch.zeros(sh.dst_rows, D, device=DEV) if Wr is not None else None
    ss = torch.zeros(max(sh.U_max, 1), H, device=DEV) if att else None
    sd = torch.zeros(sh.rows, H, device=DEV) if att else None
    ws = torch.empty(hf().project_ws_bytes(sh, K, D, H) // 4 + 16, device=DEV)
    tn = lambda a: None if a is None else t(a)
    hf().project(sh, csr, K, D, H, t(X), t(gid, torch.int32), t(W), tn(Wr), tn(A), Y, R0, ss, sd,
                 ws, prec=prec)
    osh = oracle.Shape.of(blk, rs, rd)
    ref = oracle.project(osh, ch, K, D, H, X, gid, W, Wr, A)
    tol = 2e-3 if prec != "fp32" else 1e-5
    row_rel_l2(Y.cpu().numpy()[:U], ref["Y"], tol, "Y")
    if Wr is not None:
        row_rel_l2(R0.cpu().numpy(), ref["R0"], tol, "R0")
    if att:
        row_rel_l2(ss.cpu().numpy()[:U], ref["s_src"], max(tol, 1e-4), "s_src")
        row_rel_l2(sd.cpu().numpy(), ref["s_dst"], 1e-4, "s_dst")
    # backward (X without gather for dX)
    Xl = rng.standard_normal((sh.src_rows, K)).astype(np.float32)
    dYn = rng.standard_normal((max(U, 1), D)).astype(np.float32)
    Gn = rng.standard_normal((sh.dst_rows, D)).astype(np.float32)
    dssn = rng.standard_normal((max(U, 1), H)).astype(np.float32) if att else None
    dsdn = rng.standard_normal((sh.rows, H)).astype(np.float32) if att else None
    Yl = rng.standard_normal((max(U, 1), D)).astype(np.float32)
    dYg = t(dYn)
    dX = torch.zeros(sh.src_rows, K, device=DEV)
    dW = torch.zeros(sh.R, K, D, device=DEV)
    dWr = torch.zeros(sh.T, K, D, device=DEV) if Wr is not None else None
    datt = torch.zeros(sh.R, 2, D, device=DEV) if att else None
    wsb = torch.empty(hf().project_bwd_ws_bytes(sh, K, D, H) // 4 + 16, device=DEV)
    hf().project_bwd(sh, csr, K, D, H, t(Xl), None, t(W), tn(Wr), tn(A), t(Yl), dYg, t(Gn),
                     tn(dssn), tn(dsdn), dX, dW, dWr, datt, wsb, prec=prec)
    ob = oracle.project_bwd(osh, ch, K, D, H, Xl, None, W, Wr, A, Yl[:U], dYn[:U], Gn,
                            None if dssn is None else dssn[:U], dsdn)
    wt = 1e-4 if prec == "fp32" else 3e-3
    row_rel_l2(dW.cpu().numpy().reshape(-1, D), ob["dW_rel"].reshape(-1, D), wt, "dW_rel")
    if Wr is not None:
        row_rel_l2(dWr.cpu().numpy().reshape(-1, D), ob["dW_root"].reshape(-1, D), wt, "dW_root")
    row_rel_l2(dX.cpu().numpy(), ob["dX"], wt, "dX")
    if att:
        row_rel_l2(datt.cpu().numpy().reshape(-1, D), ob["datt"].reshape(-1, D), wt, "datt")
    if not att:
        # split form (input gradient alone, then weights alone with dX = NULL,
        # the Trainer's side-stream schedule): bit-identical to the combined call
        dX2 = torch.zeros_like(dX)
        dW2 = torch.zeros_like(dW)
        dWr2 = torch.zeros_like(dWr) if dWr is not None else None
        wsc = torch.empty_like(wsb)
        hf().project_bwd(sh, csr, K, D, H, t(Xl), None, t(W), tn(Wr), None, t(Yl), t(dYn), t(Gn),
                         None, None, dX2, None, None, None, wsb, prec=prec)
        hf().project_bwd(sh, csr, K, D, H, t(Xl), None, t(W), tn(Wr), None, t(Yl), t(dYn), t(Gn),
                         None, None, None, dW2, dWr2, None, wsc, prec=prec)
        assert torch.equal(dX2, dX) and torch.equal(dW2, dW)
        if dWr is not None:
            assert torch.equal(dWr2, dWr)
    else:
        # RGAT split form (Trainer: input gradient on the critical path, the
        # weight / attention gradients on the side stream), on dYt (dYg now
        # holds it: the combined call above applied the score chain in place):
        # bit-identical to the combined scored call
        outs = []
        for split in (False, True):
            dXs = torch.zeros_like(dX)
            dWs = torch.zeros_like(dW)
            das = torch.zeros_like(datt)
            w1, w2 = torch.empty_like(wsb), torch.empty_like(wsb)
            args = (sh, csr, K, D, H, t(Xl), None, t(W), None, t(A), t(Yl), dYg.clone(), t(Gn),
                    t(dssn), t(dsdn))
            if split:
                hf().project_bwd_scored(*args, dXs, None, None, None, w1, prec=prec)
                hf().project_bwd_scored(*args, None, dWs, None, das, w2, prec=prec)
            else:
                hf().project_bwd_scored(*args, dXs, dWs, None, das, w1, prec=prec)
            outs.append((dXs, dWs, das))
        for a_, b_ in zip(*outs):
            assert torch.equal(a_, b_)
        row_rel_l2(outs[1][0].cpu().numpy(), ob["dX"], wt, "dX split")


@pytest.mark.parametrize("K,D", [(128, 128), (64, 64), (128, 64), (64, 128)])
def test_project_tf32_exact_on_representable_inputs(K, D):
    """X, W in {-2..2}/4 are exact in TF32 and every partial sum is exact in
    fp32, so the tcgen05 result must equal the oracle bit for bit (catches
    descriptor / swizzle / layout bugs, SURVEY.md §8(c) exactness trick)."""
    rng, blk, et, rs, rd, sh, csr, ch = make_case(123 + K + D, D=D, T=3, R=6, N=4000)
    U = ch["U"]
    X = (rng.integers(-2, 3, (sh.src_rows + 5, K)) / 4).astype(np.float32)
    gid = rng.permutation(sh.src_rows + 5)[:sh.src_rows].astype(np.int32)
    W = (rng.integers(-2, 3, (sh.R, K, D)) / 4).astype(np.float32)
    Wr = (rng.integers(-2, 3, (sh.T, K, D)) / 4).astype(np.float32)
    Y = torch.zeros(max(sh.U_max, 1), D, device=DEV)
    R0 = torch.zeros(sh.dst_rows, D, device=DEV)
    ws = torch.empty(hf().project_ws_bytes(sh, K, D, 1) // 4 + 16, device=DEV)
    hf().project(sh, csr, K, D, 1, t(X), t(gid, torch.int32), t(W), t(Wr), None, Y, R0, None,
                 None, ws, prec="tf32")
    osh = oracle.Shape.of(blk, rs, rd)
    ref = oracle.project(osh, ch, K, D, 1, X, gid, W, Wr, None)
    assert np.array_equal(Y.cpu().numpy()[:U], ref["Y"].astype(np.float32))
    assert np.array_equal(R0.cpu().numpy(), ref["R0"].astype(np.float32))
    # backward (wgrad with MN-major operands, dgrad with K-major) on exact inputs
    Xl = (rng.integers(-2, 3, (sh.src_rows, K)) / 4).astype(np.float32)
    dYn = (rng.integers(-2, 3, (max(U, 1), D)) / 4).astype(np.float32)
    Gn = (rng.integers(-2, 3, (sh.dst_rows, D)) / 4).astype(np.float32)
    dX = torch.zeros(sh.src_rows, K, device=DEV)
    dW = torch.zeros(sh.R, K, D, device=DEV)
    dWr = torch.zeros(sh.T, K, D, device=DEV)
    wsb = torch.empty(hf().project_bwd_ws_bytes(sh, K, D, 1) // 4 + 16, device=DEV)
    hf().project_bwd(sh, csr, K, D, 1, t(Xl), None, t(W), t(Wr), None, None, t(dYn), t(Gn), None,
                     None, dX, dW, dWr, None, wsb, prec="tf32")
    ob = oracle.project_bwd(osh, ch, K, D, 1, Xl, None, W, Wr, None, None, dYn[:U], Gn, None, None)
    assert np.array_equal(dW.cpu().numpy(), ob["dW_rel"].astype(np.float32))
    assert np.array_equal(dWr.cpu().numpy(), ob["dW_root"].astype(np.float32))
    assert np.array_equal(dX.cpu().numpy(), ob["dX"].astype(np.float32))


@pytest.mark.parametrize("K,D", [(128, 128), (128, 64), (64, 128), (64, 64)])
@pytest.mark.parametrize("att", [False, True])
def test_project_bf16(K, D, att):
    """HIFUSE_PREC_BF16 (reading C24): Y, R0 and the epilogue's s_src against
    the oracle fed BF16-rounded X and W (every product of two bf16 values is
    exact in fp32, so only the fp32 accumulation differs: 1e-5 row-norm);
    s_dst stays fp32 (unrounded oracle)."""
    H = 2 if att else 1
    rng, blk, et, rs, rd, sh, csr, ch = make_case(300 + K + D, D=D, H=H, T=3, R=7, hub=0.05)
    U = ch["U"]
    xr = sh.src_rows + 7
    X = rng.standard_normal((xr, K)).astype(np.float32)
    gid = rng.permutation(xr)[:sh.src_rows].astype(np.int32)
    W = (rng.standard_normal((sh.R, K, D)) / np.sqrt(K)).astype(np.float32)
    Wr = None if att else (rng.standard_normal((sh.T, K, D)) / np.sqrt(K)).astype(np.float32)
    A = rng.standard_normal((sh.R, 2, D)).astype(np.float32) if att else None
    Y = torch.zeros(max(sh.U_max, 1), D, device=DEV)
    R0 = torch.zeros(sh.dst_rows, D, device=DEV) if Wr is not None else None
    ss = torch.zeros(max(sh.U_max, 1), H, device=DEV) if att else None
    sd = torch.zeros(sh.rows, H, device=DEV) if att else None
    ws = torch.empty(hf().project_ws_bytes(sh, K, D, H) // 4 + 16, device=DEV)
    tn = lambda a: None if a is None else t(a)
    hf().project(sh, csr, K, D, H, t(X), t(gid, torch.int32), t(W), tn(Wr), tn(A), Y, R0, ss, sd,
                 ws, prec="bf16")
    osh = oracle.Shape.of(blk, rs, rd)
    rb = oracle.bf16_round
    ref = oracle.project(osh, ch, K, D, H, rb(X), gid, rb(W), None if Wr is None else rb(Wr), A)
    row_rel_l2(Y.cpu().numpy()[:U], ref["Y"], 1e-5, "Y")
    if Wr is not None:
        row_rel_l2(R0.cpu().numpy(), ref["R0"], 1e-5, "R0")
    if att:
        row_rel_l2(ss.cpu().numpy()[:U], ref["s_src"], 1e-4, "s_src")
        ref32 = oracle.project(osh, ch, K, D, H, X, gid, W, None, A)
        row_rel_l2(sd.cpu().numpy(), ref32["s_dst"], 1e-4, "s_dst")


@pytest.mark.parametrize("K,D", [(128, 128), (64, 64)])
def test_project_bf16_exact_on_representable_inputs(K, D):
    """X, W in {-2..2}/4 are exact in bf16 and every partial sum is exact in
    fp32: the kind::f16 result equals the oracle bit for bit (layout /
    descriptor check of the BF16 operand path)."""
    rng, blk, et, rs, rd, sh, csr, ch = make_case(321 + K + D, D=D, T=3, R=6, N=4000)
    U = ch["U"]
    X = (rng.integers(-2, 3, (sh.src_rows + 5, K)) / 4).astype(np.float32)
    gid = rng.permutation(sh.src_rows + 5)[:sh.src_rows].astype(np.int32)
    W = (rng.integers(-2, 3, (sh.R, K, D)) / 4).astype(np.float32)
    Wr = (rng.integers(-2, 3, (sh.T, K, D)) / 4).astype(np.float32)
    Y = torch.zeros(max(sh.U_max, 1), D, device=DEV)
    R0 = torch.zeros(sh.dst_rows, D, device=DEV)
    ws = torch.empty(hf().project_ws_bytes(sh, K, D, 1) // 4 + 16, device=DEV)
    hf().project(sh, csr, K, D, 1, t(X), t(gid, torch.int32), t(W), t(Wr), None, Y, R0, None,
                 None, ws, prec="bf16")
    osh = oracle.Shape.of(blk, rs, rd)
    ref = oracle.project(osh, ch, K, D, 1, X, gid, W, Wr, None)
    assert np.array_equal(Y.cpu().numpy()[:U], ref["Y"].astype(np.float32))
    assert np.array_equal(R0.cpu().numpy(), ref["R0"].astype(np.float32))


@pytest.mark.parametrize("prec", ["tf32", "bf16"])
@pytest.mark.parametrize("K,D", [(128, 128), (64, 64), (128, 64)])
def test_project_y16_and_bf16_aggregation(K, D, prec):
    """NEXT(3) BF16 storage of Y (reading C25): on {-2..2}/4 inputs the fp32
    accumulator is exact, so Yb must be the RN-even bf16 rounding of the fp64
    oracle's Y bit for bit; on random inputs Yb within TF32 + half a bf16 ulp
    (row-norm 5e-3).  The aggregation over Yb (the BF16 gather kernel with
    col_x = csr.col) against the oracle's aggregation of the same rounded Y at
    1e-5 of the absolute-sum scale (sum and mean)."""
    rng, blk, et, rs, rd, sh, csr, ch = make_case(350 + K + D, D=D, T=3, R=6, N=5000, hub=0.1)
    U = ch["U"]
    osh = oracle.Shape.of(blk, rs, rd)
    ws = torch.empty(hf().project_ws_bytes(sh, K, D, 1) // 4 + 16, device=DEV)
    for exact in (True, False):
        if exact:
            X = (rng.integers(-2, 3, (sh.src_rows, K)) / 4).astype(np.float32)
            W = (rng.integers(-2, 3, (sh.R, K, D)) / 4).astype(np.float32)
            Wr = (rng.integers(-2, 3, (sh.T, K, D)) / 4).astype(np.float32)
        else:
            X = rng.standard_normal((sh.src_rows, K)).astype(np.float32)
            W = (rng.standard_normal((sh.R, K, D)) / np.sqrt(K)).astype(np.float32)
            Wr = (rng.standard_normal((sh.T, K, D)) / np.sqrt(K)).astype(np.float32)
        Yb = torch.zeros(max(sh.U_max, 1), D, device=DEV, dtype=torch.bfloat16)
        R0 = torch.zeros(sh.dst_rows, D, device=DEV)
        hf().project_y16(sh, csr, K, D, t(X), None, t(W), t(Wr), Yb, R0, ws, prec=prec)
        rb = oracle.bf16_round if prec == "bf16" else (lambda a: a)
        ref = oracle.project(osh, ch, K, D, 1, rb(X), None, rb(W), rb(Wr), None)
        got = Yb.float().cpu().numpy()[:U]
        if exact:
            assert np.array_equal(got, oracle.bf16_round(ref["Y"]).astype(np.float32))
        else:
            row_rel_l2(got, ref["Y"], 5e-3, "Yb")
        for agg in ("sum", "mean"):
            Z = torch.zeros(sh.rows, D, device=DEV)
            hf().aggregate_features_cols_bf16(sh, csr, agg, D, Yb, csr["col"], None, Z, None)
            Yr = np.zeros((max(U, 1), D))
            Yr[:U] = got
            zr = oracle.aggregate_fwd(osh, blk, et, ch, agg, D, 1, Yr)["Z"]
            za = oracle.aggregate_fwd(osh, blk, et, ch, agg, D, 1, np.abs(Yr))["Z"]
            close_scaled(Z.cpu().numpy(), zr, za, 1e-5, f"Z {agg}")


@pytest.mark.parametrize("split", [False, True])
@pytest.mark.parametrize("B,C", [(5, 3), (128, 7), (1024, 128), (300, 129), (1024, 349),
                                 (64, 600), (2048, 7)])
def test_linear_xent(B, C, split):
    """Classifier head: loss, dH (seed rows; other rows zero), dWc,
    dbc against the fp64 oracle head; register-row (C <= 512) and generic
    softmax paths; weight gradient in the same call or deferred
    (hifuse_linear_xent_wgrad).  3xTF32 GEMMs: fp32-level error, 1e-5 of the
    scale."""
    import oracle.model as om
    rng = np.random.default_rng(B * 1000 + C)
    D, row0, extra = 128, 17, 9
    Hfull = rng.standard_normal((row0 + B + extra, D)).astype(np.float32)
    Wc = (rng.standard_normal((D, C)) * 0.1).astype(np.float32)
    bc = (rng.standard_normal(C) * 0.1).astype(np.float32)
    lab = rng.integers(0, C, B).astype(np.int32)
    ref = om.xent(Hfull[row0:row0 + B], Wc, bc, lab)
    loss = torch.zeros(1, device=DEV)
    dH = torch.full((Hfull.shape[0], D), 7.0, device=DEV)
    dWc = torch.zeros(D, C, device=DEV)
    dbc = torch.zeros(C, device=DEV)
    ws = torch.empty(hf().xent_ws_bytes(B, D, C) // 4 + 64, device=DEV)
    Hd = t(Hfull)
    if split:      # weight gradient deferred to hifuse_linear_xent_wgrad
        hf().linear_xent(B, D, C, Hd, row0, torch.from_numpy(lab).to(DEV), t(Wc), t(bc), loss,
                         dH, None, None, ws)
        hf().linear_xent_wgrad(B, D, C, Hd, row0, dWc, dbc, ws)
    else:
        hf().linear_xent(B, D, C, Hd, row0, torch.from_numpy(lab).to(DEV), t(Wc), t(bc), loss,
                         dH, dWc, dbc, ws)
    torch.cuda.synchronize()
    assert abs(loss.item() - ref["loss"]) <= 1e-5 * max(1.0, abs(ref["loss"]))
    dHh = dH.cpu().numpy()
    assert not dHh[:row0].any() and not dHh[row0 + B:].any()
    sc = np.abs(ref["dlog"]).sum(axis=1, keepdims=True) * np.abs(Wc).max() + 1e-30
    assert np.all(np.abs(dHh[row0:row0 + B] - ref["dhs"]) <= 1e-5 * sc)
    sw = np.abs(Hfull[row0:row0 + B]).T @ np.abs(ref["dlog"]) + 1e-30
    assert np.all(np.abs(dWc.cpu().numpy() - ref["dWc"]) <= 1e-5 * sw)
    assert np.all(np.abs(dbc.cpu().numpy() - ref["dbc"]) <= 1e-5 * np.abs(ref["dlog"]).sum(0) + 1e-12)



@pytest.mark.parametrize("B,C", [(64, 7), (300, 349), (64, 600)])
def test_linear_xent_bad_labels(B, C):
    """Labels outside [0, C) (negative, == C, >= 32 for the small-C kernel)
    set HIFUSE_ST_BAD_LABEL and drop their rows: the loss is the oracle's sum
    over the valid rows divided by B, their dH rows are zero."""
    import oracle.model as om
    rng = np.random.default_rng(B + C)
    D = 128
    Hs = rng.standard_normal((B, D)).astype(np.float32)
    Wc = (rng.standard_normal((D, C)) * 0.1).astype(np.float32)
    bc = (rng.standard_normal(C) * 0.1).astype(np.float32)
    lab = rng.integers(0, C, B).astype(np.int32)
    bad = np.array([1, 5, B - 1])
    lab[bad] = [-1, C, C + 40]
    good = np.setdiff1d(np.arange(B), bad)
    ref = om.xent(Hs[good], Wc, bc, lab[good])
    loss = torch.zeros(1, device=DEV)
    dH = torch.full((B, D), 7.0, device=DEV)
    ws = torch.empty(hf().xent_ws_bytes(B, D, C) // 4 + 64, device=DEV)
    st = torch.zeros(1, dtype=torch.int32, device=DEV)
    hf().linear_xent(B, D, C, t(Hs), 0, torch.from_numpy(lab).to(DEV), t(Wc), t(bc), loss, dH,
                     None, None, ws, status=st)
    torch.cuda.synchronize()
    assert hf().read_status(st) == 32            # HIFUSE_ST_BAD_LABEL
    want = ref["loss"] * len(good) / B
    assert abs(loss.item() - want) <= 1e-5 * max(1.0, abs(want))
    dHh = dH.cpu().numpy()
    assert not dHh[bad].any()
    assert np.isfinite(dHh).all()

# ------------------------------------- GAT, softmax across relations (NEXT(2))
@pytest.mark.parametrize("D,H", [(128, 8), (64, 8), (128, 1), (64, 2)])
@pytest.mark.parametrize("seed", range(3))
def test_aggregate_fwd_gat_xrel(seed, D, H):
    rng, blk, et, rs, rd, sh, csr, ch = make_case(130 + seed, D=D, H=H, hub=0.05,
                                                     T=[1, 2, 4][seed], R=[3, 7, 11][seed])
    U = ch["U"]
    Y = rng.standard_normal((U, D)).astype(np.float32)
    ss = (rng.standard_normal((U, H)) * 2).astype(np.float32)
    sd = (rng.standard_normal((sh.rows, H)) * 2).astype(np.float32)
    Z = torch.full((sh.rows, D), 9.0, device=DEV)
    stats = torch.zeros(sh.rows, 2 * H, device=DEV)
    n0 = hf().kernel_launches()
    hf().aggregate_fwd_xrel(sh, csr, D, H, 0.2, t(Y), t(ss), t(sd), Z, stats)
    assert hf().kernel_launches() - n0 == 1           # one kernel for all relations
    ref = agg_oracle(blk, et, rs, rd, ch, "gat_xrel", D, H, Y, ss, sd)
    A = agg_oracle(blk, et, rs, rd, ch, "gat_xrel", D, H, np.abs(Y), ss, sd)["Z"]
    close_scaled(Z.cpu().numpy(), ref["Z"], A, what="Z gat_xrel")
    # every row of a destination carries the destination's (max, sum): equal
    # across its rows, and the sum >= 1 wherever the destination has edges
    st = stats.cpu().numpy()
    gm = _gmap_index(sh, ch)
    deg_dst = np.zeros(sh.dst_rows)
    np.add.at(deg_dst, gm, ref["deg"])
    for q in range(sh.R):
        for q2 in range(q + 1, sh.R):
            if sh.rel_dst[q] != sh.rel_dst[q2]:
                continue
            a, b = ch["rel_row_off"][q], ch["rel_row_off"][q2]
            n = sh.n_dst[sh.rel_dst[q]]
            assert np.array_equal(st[a:a + n], st[b:b + n])
    nz = deg_dst[gm] > 0
    assert np.all(st[nz, H:] >= 1.0 - 1e-6)


@pytest.mark.parametrize("D,H", [(128, 8), (64, 8)])
@pytest.mark.parametrize("seed", range(3))
def test_aggregate_bwd_gat_xrel(seed, D, H):
    rng, blk, et, rs, rd, sh, csr, ch = make_case(160 + seed, D=D, H=H, hub=0.1,
                                                     N=[800, 6000, 20000][seed], T=2, R=6)
    U = ch["U"]
    Y = rng.standard_normal((U, D)).astype(np.float32)
    ss = rng.standard_normal((U, H)).astype(np.float32)
    sd = rng.standard_normal((sh.rows, H)).astype(np.float32)
    G = rng.standard_normal((sh.dst_rows, D)).astype(np.float32)
    Z = torch.zeros(sh.rows, D, device=DEV)
    stats = torch.zeros(sh.rows, 2 * H, device=DEV)
    hf().aggregate_fwd_xrel(sh, csr, D, H, 0.2, t(Y), t(ss), t(sd), Z, stats)
    dY = torch.zeros(U, D, device=DEV)
    dss = torch.zeros(U, H, device=DEV)
    dsd = torch.zeros(sh.rows, H, device=DEV)
    ws = torch.empty(hf().aggregate_bwd_ws_bytes(sh, "gat_xrel", H) // 4 + 16, device=DEV)
    hf().aggregate_bwd(sh, csr, "gat_xrel", D, H, 0.2, t(G), t(Y), t(ss), t(sd), stats, dY, dss,
                       dsd, ws)
    osh = oracle.Shape.of(blk, rs, rd)
    ref = oracle.aggregate_bwd(osh, blk, et, ch, "gat_xrel", D, H, G, Y, ss, sd)
    sc_y = oracle.aggregate_bwd(osh, blk, et, ch, "gat_xrel", D, H, np.abs(G), np.abs(Y), ss, sd)
    close_scaled(dY.cpu().numpy(), ref["dY"], sc_y["dY"], what="dY gat_xrel")
    # ds: absolute-sum scale of the dpre = alpha (dalpha - za) terms, za over
    # the destination's union of rows
    fw = oracle.aggregate_fwd(osh, blk, et, ch, "gat_xrel", D, H, Y, ss, sd)
    nv = ch["row_ptr"][-1]
    rows = np.repeat(np.arange(sh.rows), np.diff(ch["row_ptr"]))
    e, u = ch["eperm"][:nv], ch["col"][:nv]
    dest = _gmap_index(sh, ch)[rows]
    dh = D // H
    dabs = (np.abs(G[dest]).reshape(-1, H, dh) * np.abs(Y[u]).reshape(-1, H, dh)).sum(-1)
    a = fw["alpha"][e]
    za = np.zeros((sh.dst_rows, H))
    np.add.at(za, dest, a * dabs)
    term = a * (dabs + za[dest])
    scale_d = np.zeros((sh.rows, H))
    np.add.at(scale_d, rows, term)
    scale_s = np.zeros((U, H))
    np.add.at(scale_s, u, term)
    close_scaled(dss.cpu().numpy(), ref["ds_src"], scale_s, what="ds_src xrel")
    close_scaled(dsd.cpu().numpy(), ref["ds_dst"], scale_d, what="ds_dst xrel")


@pytest.mark.parametrize("agg,H", [("mean", 1), ("sum", 1), ("gat", 8), ("gat_mul", 8)])
def test_aggregate_bwd_rows_matches_type_major(agg, H):
    """hifuse_aggregate_bwd_rows (per-merged-row gradient, HAN fusion) fed
    with G_t[i] on every row (r, i) computes exactly what hifuse_aggregate_bwd
    computes from the type-major G (bit-identical), and matches the oracle's
    g_rows path for a genuinely per-row gradient."""
    from test_oracle_backward import gmap
    D = 128
    rng, blk, et, rs, rd, sh, csr, ch = make_case(95, D=D, H=H, N=9000, hub=0.1)
    U = ch["U"]
    Y = rng.standard_normal((U, D)).astype(np.float32)
    ss = rng.standard_normal((U, H)).astype(np.float32)
    sd = rng.standard_normal((sh.rows, H)).astype(np.float32)
    G = rng.standard_normal((sh.dst_rows, D)).astype(np.float32)
    gat = agg.startswith("gat")
    stats = torch.zeros(sh.rows, 2 * H, device=DEV) if gat else None
    if gat:
        Z = torch.zeros(sh.rows, D, device=DEV)
        hf().aggregate_fwd(csr, sh.rows, agg, D, H, 0.2, t(Y), t(ss), t(sd), Z, stats)
    ws = torch.empty(hf().aggregate_bwd_ws_bytes(sh, agg, H) // 4 + 16, device=DEV)
    outs = []
    for rows_mode in (False, True):
        dY = torch.zeros(max(U, 1), D, device=DEV)
        dss = torch.zeros(max(U, 1), H, device=DEV) if gat else None
        dsd = torch.zeros(sh.rows, H, device=DEV) if gat else None
        args = (t(Y), t(ss) if gat else None, t(sd) if gat else None, stats)
        if rows_mode:
            hf().aggregate_bwd_rows(sh, csr, agg, D, H, 0.2, t(gmap(sh, ch, G).astype(np.float32)),
                                    *args, None, dY, dss, dsd, ws)
        else:
            hf().aggregate_bwd(sh, csr, agg, D, H, 0.2, t(G), *args, dY, dss, dsd, ws)
        outs.append([x for x in (dY, dss, dsd) if x is not None])
    for a, b in zip(*outs):
        assert torch.equal(a, b)
    # a per-row gradient that differs between the relations of a type
    dZ = rng.standard_normal((sh.rows, D)).astype(np.float32)
    dY = torch.zeros(max(U, 1), D, device=DEV)
    dss = torch.zeros(max(U, 1), H, device=DEV) if gat else None
    dsd = torch.zeros(sh.rows, H, device=DEV) if gat else None
    hf().aggregate_bwd_rows(sh, csr, agg, D, H, 0.2, t(dZ), t(Y), t(ss) if gat else None,
                            t(sd) if gat else None, stats, None, dY, dss, dsd, ws)
    osh = oracle.Shape.of(blk, rs, rd)
    ref = oracle.aggregate_bwd(osh, blk, et, ch, agg, D, H, dZ, Y, ss, sd, g_rows=True)
    sc = oracle.aggregate_bwd(osh, blk, et, ch, agg, D, H, np.abs(dZ), np.abs(Y), ss, sd,
                              g_rows=True)
    close_scaled(dY.cpu().numpy()[:U], ref["dY"], sc["dY"], what=f"dY rows {agg}")


@pytest.mark.parametrize("D", [64, 128])
@pytest.mark.parametrize("act", ["relu", "none"])
def test_semantic_fuse_att(D, act):
    """HAN semantic-attention fusion (NEXT(2), reading C22), stage-isolated:
    beta and H against the oracle's O4' + O4 on the GPU's own Z; the backward
    (G, per-row dZ, dbias, dWs, dbs, dq) against O5a + O5a'."""
    rng, blk, et, rs, rd, sh, csr, ch = make_case(97, D=D, N=5000, T=3, R=7)
    osh = oracle.Shape.of(blk, rs, rd)
    Z = rng.standard_normal((sh.rows, D)).astype(np.float32)
    R0 = rng.standard_normal((sh.dst_rows, D)).astype(np.float32)
    bias = (rng.standard_normal((sh.T, D)) * 0.1).astype(np.float32)
    Ws = (rng.standard_normal((D, D)) / np.sqrt(D)).astype(np.float32)
    bs = (rng.standard_normal(D) * 0.1).astype(np.float32)
    q = (rng.standard_normal(D) / np.sqrt(D)).astype(np.float32)
    beta = torch.zeros(sh.R, device=DEV)
    w = torch.zeros(sh.R, device=DEV)
    Hd = torch.zeros(sh.dst_rows, D, device=DEV)
    ws = torch.empty(hf().sem_att_ws_bytes(sh, D, D) // 4 + 64, device=DEV)
    hf().semantic_fuse_att(sh, D, D, act, t(Z), t(R0), t(bias), t(Ws), t(bs), t(q), beta, w, Hd,
                           ws)
    w_ref, beta_ref = oracle.sem_att(osh, D, Z, Ws, bs, q)
    np.testing.assert_allclose(w.cpu().numpy(), w_ref, rtol=1e-5, atol=1e-6)
    np.testing.assert_allclose(beta.cpu().numpy(), beta_ref, rtol=1e-5, atol=1e-7)
    a = 1 if act == "relu" else 0
    H_ref = oracle.fuse(osh, D, a, Z, R0, bias, beta=beta_ref)
    A = oracle.fuse(osh, D, 0, np.abs(Z), np.abs(R0), np.abs(bias), beta=beta_ref)
    close_scaled(Hd.cpu().numpy(), H_ref, A, rtol=2e-5, what="H han")
    # backward
    dH = rng.standard_normal((sh.dst_rows, D)).astype(np.float32)
    G = torch.zeros(sh.dst_rows, D, device=DEV)
    dZ = torch.zeros(sh.rows, D, device=DEV)
    dbias = torch.zeros(sh.T, D, device=DEV)
    dWs = torch.zeros(D, D, device=DEV)
    dbs = torch.zeros(D, device=DEV)
    dq = torch.zeros(D, device=DEV)
    hf().semantic_fuse_att_bwd(sh, D, D, act, t(dH), Hd, t(Z), t(Ws), t(bs), t(q), beta, G, dZ,
                               dbias, dWs, dbs, dq, ws)
    G_ref, db_ref = oracle.fuse_bwd(osh, D, a, dH, Hd.cpu().numpy())
    assert np.array_equal(G.cpu().numpy(), G_ref.astype(np.float32))
    sem = oracle.sem_att_bwd(osh, D, Z, Ws, bs, q, beta.cpu().numpy().astype(np.float64), G_ref)

    def rl2(g, r):
        return np.linalg.norm(np.asarray(g, np.float64) - r) / max(np.linalg.norm(r), 1e-30)
    assert rl2(dZ.cpu().numpy(), sem["dZ"]) < 1e-5
    assert rl2(dbias.cpu().numpy(), db_ref) < 1e-6
    for name, got, ref in (("dWs", dWs, sem["dWs"]), ("dbs", dbs, sem["dbs"]),
                           ("dq", dq, sem["dq"])):
        assert rl2(got.cpu().numpy(), ref) < 5e-5, name


@pytest.mark.parametrize("D", [64, 128])
@pytest.mark.parametrize("agg", ["sum", "mean"])
@pytest.mark.parametrize("seed", range(3))
def test_aggregate_fuse_fwd(seed, agg, D):
    """hifuse_aggregate_fuse_fwd (A4 + A5 in one launch) is bit-identical to
    hifuse_aggregate_fwd + hifuse_semantic_fuse, including destinations of a
    type no relation enters, over repeated calls (the arrival counters reset
    themselves), with and without ReLU; H checked against the oracle too."""
    rng = np.random.default_rng(4000 + seed)
    T, R = 5, 8
    rs, rd = random_schema(rng, T, R)
    rd = np.where(rd == T - 1, 0, rd).astype(np.int32)      # type T-1: no relation enters it
    n_src = rng.integers(30, 300, T)
    n_dst = np.maximum(np.minimum(rng.integers(0, 200, T), n_src), 1)
    blk, et = random_block(rng, n_src, n_dst, rs, rd, 3000, hub_frac=0.1 * (seed % 2))
    sh, csr, st = gpu_build(blk, et, rs, rd)
    ch = csr_host(sh, csr)
    U = ch["U"]
    ws = torch.zeros(hf().aggregate_fuse_ws_bytes(sh) // 4 + 16, dtype=torch.int32, device=DEV)
    for it, act in enumerate(("relu", "none", "relu")):
        Y = t(rng.standard_normal((max(U, 1), D)).astype(np.float32))
        R0 = t(rng.standard_normal((sh.dst_rows, D)).astype(np.float32))
        b = t(rng.standard_normal((sh.T, D)).astype(np.float32))
        Z1 = torch.zeros(max(sh.rows, 1), D, device=DEV)
        H1 = torch.full((sh.dst_rows, D), float("nan"), device=DEV)
        hf().aggregate_fwd(csr, sh.rows, agg, D, 1, 0.2, Y, None, None, Z1, None)
        hf().semantic_fuse(sh, D, act, Z1, R0, b, H1)
        Z2 = torch.zeros_like(Z1)
        H2 = torch.full_like(H1, float("nan"))
        hf().aggregate_fuse_fwd(sh, csr, agg, D, act, Y, R0, b, Z2, H2, ws)
        torch.cuda.synchronize()
        assert torch.equal(Z1[:sh.rows], Z2[:sh.rows]), it
        assert torch.equal(H1, H2), it
        assert int(ws.abs().sum().item()) == 0            # counters left zeroed
    osh = oracle.Shape.of(blk, rs, rd)
    Yn = Y.cpu().numpy()[:U]
    Zr = oracle.aggregate_fwd(osh, blk, et, ch, agg, D, 1, Yn)["Z"]
    Za = oracle.aggregate_fwd(osh, blk, et, ch, agg, D, 1, np.abs(Yn))["Z"]
    Hr = oracle.fuse(osh, D, 1, Zr, R0.cpu().numpy(), b.cpu().numpy())
    Ha = oracle.fuse(osh, D, 0, Za, np.abs(R0.cpu().numpy()), np.abs(b.cpu().numpy()))
    close_scaled(H2.cpu().numpy(), Hr, Ha, what="H fused")
