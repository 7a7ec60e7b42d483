"""-m gpu: the aggregate-first RGCN input layer (SURVEY.md §8(f) NEXT(3),
DESIGN.md §9) against the oracle's O6 functions, stage by stage, and the
whole training step against the (project-first) oracle model -- the two
orders are equal by linearity (pinned in tests/test_oracle_aggfirst.py).
"""
import numpy as np
import pytest
import torch

import oracle
from synth import random_block, random_schema

from gpu_util import needs_gpu, gpu_build, csr_host, close_scaled, row_rel_l2, t, DEV, hf

pytestmark = [pytest.mark.gpu, needs_gpu]


def make_case(seed, T=None, R=None, N=None, hub=0.0, csc=True):
    rng = np.random.default_rng(seed)
    T = T or int(rng.integers(1, 5))
    R = R or int(rng.integers(1, 12))
    rs, rd = random_schema(rng, T, R)
    n_src = rng.integers(1, 400, T)
    n_dst = np.maximum(np.minimum(rng.integers(0, 250, T), n_src), 1)
    N = int(rng.integers(100, 6000)) if N is None else N
    blk, et = random_block(rng, n_src, n_dst, rs, rd, N, hub_frac=hub)
    sh, csr, st = gpu_build(blk, et, rs, rd, csc=csc)
    return rng, blk, et, rs, rd, sh, csr


@pytest.mark.parametrize("seed", range(3))
def test_build_without_transpose_is_bit_exact(seed):
    rng, blk, et, rs, rd, sh, csr = make_case(300 + seed, hub=0.1, csc=False)
    ch = csr_host(sh, csr)
    ref = oracle.build(oracle.Shape.of(blk, rs, rd), blk, et)
    assert ch["U"] == ref["U"]
    for k in ("rel_row_off", "row_ptr", "col", "eperm", "rel_y_off", "y_src", "slot_y"):
        assert np.array_equal(ch[k], np.asarray(ref[k])), k


@pytest.mark.parametrize("seed", range(4))
def test_xrow_build(seed):
    """X-row build (no Y numbering, the aggregate-first input layer's form):
    rows, positions and eperm bit-exact against the oracle, col = the
    source's row in the layer's X (type_src_off of the relation's source
    type + the oracle's y_src of its Y row), null edges included; the
    feature rows and the aggregation from it equal those of the Y build."""
    rng = np.random.default_rng(900 + seed)
    T, R = 4, 9
    rs, rd = random_schema(rng, T, R)
    n_src = rng.integers(20, 300, T)
    n_dst = np.maximum(np.minimum(rng.integers(0, 200, T), n_src), 1)
    blk, et = random_block(rng, n_src, n_dst, rs, rd, 4000, hub_frac=0.1 * (seed % 2))
    if seed >= 2:                                   # null (padding) edges
        from synth.sampler import LayerBlock
        eid = blk.edge_id.copy()
        eid[rng.random(len(eid)) < 0.15] = -1
        blk = LayerBlock(n_src=blk.n_src, n_dst=blk.n_dst, src_local=blk.src_local,
                         dst_local=blk.dst_local, edge_id=eid, src_global=blk.src_global)
    sh, csr, st = gpu_build(blk, et, rs, rd, csc=False, xrow=True)
    assert int(st.item()) == 0
    ref = oracle.build(oracle.Shape.of(blk, rs, rd), blk, et)
    g = lambda k, n: csr[k][:n].cpu().numpy()
    assert np.array_equal(g("rel_row_off", sh.R + 1), np.asarray(ref["rel_row_off"]))
    assert np.array_equal(g("row_ptr", sh.rows + 1), np.asarray(ref["row_ptr"]))
    assert np.array_equal(g("eperm", sh.N), np.asarray(ref["eperm"]))
    nv = int(ref["row_ptr"][-1])
    col_ref = np.asarray(ref["col"])[:nv]
    ryo = np.asarray(ref["rel_y_off"])
    r_of = np.searchsorted(ryo, col_ref, side="right") - 1
    tso = np.concatenate([[0], np.cumsum(n_src)])
    want = tso[np.asarray(rs)[r_of]] + np.asarray(ref["y_src"])[col_ref]
    got = g("col", sh.N)
    assert np.array_equal(got[:nv], want) and (got[nv:] == -1).all()
    # feature rows and the aggregation: identical to the Y-numbered build
    sh2, csr2, _ = gpu_build(blk, et, rs, rd, csc=False)
    gid = rng.permutation(sh.src_rows + 7)[:sh.src_rows].astype(np.int32)
    c1 = torch.empty(max(sh.N, 1), dtype=torch.int32, device=DEV)
    c2 = torch.empty_like(c1)
    hf().feature_cols(sh, csr, t(gid, torch.int32), c1)
    hf().feature_cols(sh2, csr2, t(gid, torch.int32), c2)
    assert torch.equal(c1[:nv], c2[:nv])
    K = 128
    X = t(rng.standard_normal((sh.src_rows + 7, K)).astype(np.float32))
    a1 = torch.zeros(max(sh.rows, 1), K, device=DEV)
    a2 = torch.zeros_like(a1)
    hf().aggregate_features_cols(sh, csr, "mean", K, X, c1, a1)
    hf().aggregate_features_cols(sh2, csr2, "mean", K, X, c2, a2)
    assert torch.equal(a1, a2)
    # x_gather: the build writes the feature-store rows itself (the Trainer's
    # aggregate-first layer: col is read as the feature-row map directly)
    gd = t(gid, torch.int32)
    sh3, csr3, st3 = gpu_build(blk, et, rs, rd, csc=False, xrow=True, x_gather=gd)
    assert int(st3.item()) == 0
    assert torch.equal(csr3["col"][:nv], c1[:nv])
    assert (csr3["col"][nv:sh.N] == -1).all()
    a3 = torch.zeros_like(a1)
    hf().aggregate_features_cols(sh3, csr3, "mean", K, X, csr3["col"], a3)
    assert torch.equal(a3, a1)


@pytest.mark.parametrize("K", [64, 128])
@pytest.mark.parametrize("agg", ["sum", "mean"])
@pytest.mark.parametrize("seed", range(3))
def test_aggregate_features(seed, agg, K):
    rng, blk, et, rs, rd, sh, csr = make_case(310 + seed, hub=0.1 * (seed % 2), csc=False)
    xr = sh.src_rows + 13
    X = rng.standard_normal((xr, K)).astype(np.float32)
    gid = rng.permutation(xr)[:sh.src_rows].astype(np.int32)
    Xa = torch.full((max(sh.rows, 1), K), float("nan"), device=DEV)
    ws = torch.empty(hf().aggregate_features_ws_bytes(sh) // 4 + 16, device=DEV)
    hf().aggregate_features_fwd(sh, csr, agg, K, t(X), t(gid, torch.int32), Xa, ws)
    osh = oracle.Shape.of(blk, rs, rd)
    ref = oracle.aggregate_features(osh, blk, et, agg, K, X, gid)
    A = oracle.aggregate_features(osh, blk, et, agg, K, np.abs(X), gid)
    close_scaled(Xa.cpu().numpy()[:sh.rows], ref, A, what=f"Xagg {agg}")
    # the split form (feature rows formed with the build, then the
    # aggregation) is the same computation: bit-identical
    colx = torch.empty(max(sh.N, 1), dtype=torch.int32, device=DEV)
    Xb = torch.full_like(Xa, float("nan"))
    hf().feature_cols(sh, csr, t(gid, torch.int32), colx)
    hf().aggregate_features_cols(sh, csr, agg, K, t(X), colx, Xb)
    assert torch.equal(Xa[:sh.rows], Xb[:sh.rows])


def test_aggregate_features_integer_inputs_bit_exact():
    rng, blk, et, rs, rd, sh, csr = make_case(333, N=5000, csc=False)
    K = 128
    X = rng.integers(-8, 9, (sh.src_rows, K)).astype(np.float32)
    osh = oracle.Shape.of(blk, rs, rd)
    ws = torch.empty(hf().aggregate_features_ws_bytes(sh) // 4 + 16, device=DEV)
    for agg in ("sum", "mean"):
        Xa = torch.zeros(sh.rows, K, device=DEV)
        hf().aggregate_features_fwd(sh, csr, agg, K, t(X), None, Xa, ws)
        ref = oracle.aggregate_features(osh, blk, et, "sum", K, X, None)
        if agg == "mean":     # reading C19: fp32 sum (exact here) / fp32 degree
            deg = np.zeros(sh.rows)
            row = 0
            for r in range(sh.R):
                m = et[blk.edge_id] == r
                np.add.at(deg, row + blk.dst_local[m], 1)
                row += int(blk.n_dst[rd[r]])
            ref = np.where(deg[:, None] > 0, ref.astype(np.float32) /
                           np.maximum(deg, 1)[:, None].astype(np.float32), 0)
        assert np.array_equal(Xa.cpu().numpy(), ref.astype(np.float32)), agg


@pytest.mark.parametrize("K,D", [(128, 128), (64, 64), (128, 64), (64, 128)])
def test_project_aggregated_exact_on_representable_inputs(K, D):
    """Xagg, X, W, G in {-2..2}/4: TF32-exact operands and exact fp32 sums, so
    the tcgen05 forward and wgrad must equal the oracle bit for bit."""
    rng, blk, et, rs, rd, sh, csr = make_case(350 + K + D, T=3, R=6, N=4000, csc=False)
    q = lambda *s: (rng.integers(-2, 3, s) / 4).astype(np.float32)
    Xa, X, W, Wr = q(sh.rows, K), q(sh.src_rows + 5, K), q(sh.R, K, D), q(sh.T, K, D)
    gid = rng.permutation(sh.src_rows + 5)[:sh.src_rows].astype(np.int32)
    Z = torch.zeros(sh.rows, D, device=DEV)
    R0 = torch.zeros(sh.dst_rows, D, device=DEV)
    hf().project_aggregated(sh, csr, K, D, t(Xa), t(X), t(gid, torch.int32), t(W), t(Wr), Z, R0)
    osh = oracle.Shape.of(blk, rs, rd)
    ref = oracle.project_aggregated(osh, K, D, Xa, X, gid, W, Wr)
    assert np.array_equal(Z.cpu().numpy(), ref["Z"].astype(np.float32))
    assert np.array_equal(R0.cpu().numpy(), ref["R0"].astype(np.float32))
    G = q(sh.dst_rows, D)
    dW = torch.zeros(sh.R, K, D, device=DEV)
    dWr = torch.zeros(sh.T, K, D, device=DEV)
    ws = torch.empty(hf().project_aggregated_bwd_ws_bytes(sh, K, D) // 4 + 16, device=DEV)
    hf().project_aggregated_bwd(sh, csr, K, D, t(Xa), t(X), t(gid, torch.int32), t(G), dW, dWr, ws)
    ob = oracle.project_aggregated_bwd(osh, K, D, Xa, X, gid, G)
    assert np.array_equal(dW.cpu().numpy(), ob["dW_rel"].astype(np.float32))
    assert np.array_equal(dWr.cpu().numpy(), ob["dW_root"].astype(np.float32))


@pytest.mark.parametrize("K,D", [(128, 128), (64, 64)])
def test_project_aggregated_random(K, D):
    rng, blk, et, rs, rd, sh, csr = make_case(370 + K, T=4, R=9, N=6000, hub=0.05, csc=False)
    Xa = rng.standard_normal((sh.rows, K)).astype(np.float32)
    X = rng.standard_normal((sh.src_rows, K)).astype(np.float32)
    W = (rng.standard_normal((sh.R, K, D)) / np.sqrt(K)).astype(np.float32)
    Wr = (rng.standard_normal((sh.T, K, D)) / np.sqrt(K)).astype(np.float32)
    Z = torch.zeros(sh.rows, D, device=DEV)
    R0 = torch.zeros(sh.dst_rows, D, device=DEV)
    hf().project_aggregated(sh, csr, K, D, t(Xa), t(X), None, t(W), t(Wr), Z, R0)
    osh = oracle.Shape.of(blk, rs, rd)
    ref = oracle.project_aggregated(osh, K, D, Xa, X, None, W, Wr)
    row_rel_l2(Z.cpu().numpy(), ref["Z"], 2e-3, "Z")
    row_rel_l2(R0.cpu().numpy(), ref["R0"], 2e-3, "R0")
    G = rng.standard_normal((sh.dst_rows, D)).astype(np.float32)
    dW = torch.zeros(sh.R, K, D, device=DEV)
    dWr = torch.zeros(sh.T, K, D, device=DEV)
    ws = torch.empty(hf().project_aggregated_bwd_ws_bytes(sh, K, D) // 4 + 16, device=DEV)
    hf().project_aggregated_bwd(sh, csr, K, D, t(Xa), t(X), None, t(G), dW, dWr, ws)
    ob = oracle.project_aggregated_bwd(osh, K, D, Xa, X, None, G)
    row_rel_l2(dW.cpu().numpy().reshape(-1, D), ob["dW_rel"].reshape(-1, D), 3e-3, "dW_rel")
    row_rel_l2(dWr.cpu().numpy().reshape(-1, D), ob["dW_root"].reshape(-1, D), 3e-3, "dW_root")


@pytest.mark.parametrize("K,D", [(128, 128), (64, 64), (128, 64)])
@pytest.mark.parametrize("act", ["relu", "none"])
def test_project_fuse_aggregated(K, D, act):
    """NEXT(3) fused fusion GEMM: one tcgen05 GEMM per destination type with
    K = (1 + R_in) K_in equals the oracle's O6 projection + O4 fusion: bit-
    exact on TF32-representable inputs (every partial sum exact in fp32), and
    within the TF32 row tolerance on random inputs; identical (same
    rounding class) to the two-call path's H within the same tolerance."""
    rng, blk, et, rs, rd, sh, csr = make_case(340 + K + D, T=3, R=7, N=6000, csc=False)
    osh = oracle.Shape.of(blk, rs, rd)
    a = 1 if act == "relu" else 0
    for exact in (True, False):
        if exact:
            mk = lambda *shape: (rng.integers(-2, 3, shape) / 4).astype(np.float32)
        else:
            mk = lambda *shape: (rng.standard_normal(shape) / np.sqrt(K)).astype(np.float32)
        Xagg = mk(sh.rows, K)
        X = mk(sh.src_rows + 7, K)
        gid = rng.permutation(sh.src_rows + 7)[:sh.src_rows].astype(np.int32)
        W = mk(sh.R, K, D)
        Wr = mk(sh.T, K, D)
        b = mk(sh.T, D)
        H = torch.full((sh.dst_rows, D), float("nan"), device=DEV)
        hf().project_fuse_aggregated(sh, csr, K, D, act, t(Xagg), t(X), t(gid, torch.int32),
                                     t(W), t(Wr), t(b), H)
        torch.cuda.synchronize()
        pr = oracle.project_aggregated(osh, K, D, Xagg, X, gid, W, Wr)
        ref = oracle.fuse(osh, D, a, pr["Z"], pr["R0"], b)
        got = H.cpu().numpy()
        if exact:
            assert np.array_equal(got, ref.astype(np.float32))
        else:
            row_rel_l2(got, ref, 2e-3, what="H fused")


@pytest.mark.parametrize("K", [64, 128])
@pytest.mark.parametrize("agg", ["sum", "mean"])
def test_aggregate_features_bf16(K, agg):
    """NEXT(3) BF16 feature storage: hifuse_aggregate_features_cols_bf16 equals
    the oracle's O6 aggregation of the BF16-ROUNDED features (1e-5 of the
    absolute-sum scale; bit-exact when the sums are exact), and the fp32
    destination rows it writes equal the rounded features exactly."""
    rng, blk, et, rs, rd, sh, csr = make_case(360 + K, hub=0.1, csc=False)
    xr = sh.src_rows + 11
    X = rng.standard_normal((xr, K)).astype(np.float32)
    Xb = torch.from_numpy(X).to(DEV).to(torch.bfloat16)
    Xr = Xb.float().cpu().numpy()                       # the rounded values
    gid = rng.permutation(xr)[:sh.src_rows].astype(np.int32)
    gid_d = t(gid, torch.int32)
    colx = torch.empty(max(sh.N, 1), dtype=torch.int32, device=DEV)
    hf().feature_cols(sh, csr, gid_d, colx)
    Xa = torch.full((max(sh.rows, 1), K), float("nan"), device=DEV)
    Xdst = torch.full((sh.src_rows, K), float("nan"), device=DEV)
    hf().aggregate_features_cols_bf16(sh, csr, agg, K, Xb, colx, gid_d, Xa, Xdst)
    torch.cuda.synchronize()
    osh = oracle.Shape.of(blk, rs, rd)
    ref = oracle.aggregate_features(osh, blk, et, agg, K, Xr, gid)
    A = oracle.aggregate_features(osh, blk, et, agg, K, np.abs(Xr), gid)
    close_scaled(Xa.cpu().numpy()[:sh.rows], ref, A, what=f"Xagg bf16 {agg}")
    xd = Xdst.cpu().numpy()
    for tt in range(sh.T):
        a = int(sh.type_src_off[tt])
        n = int(sh.n_dst[tt])
        assert np.array_equal(xd[a:a + n], Xr[gid[a:a + n]])
