"""-m gpu: element-wise stage parity at BASELINE.json's FULL sizes.

The stage tests of test_gpu_stages.py stop at N <= 20k edges; here the first
sampled batch of the full ogbn-mag and Freebase configurations goes through
the same kernels in the launch configuration bench.py times (relation-major
edge-type offsets, full-size CSR), element by element against the oracle
with the fp32 tolerance |g - r| <= 1e-5 max(|r|, A):

* ogbn-mag layer 0 (N = 472k, rho = 38k): the aggregate-first input layer
  `aggregate_features` (hifuse_feature_cols + hifuse_aggregate_features_cols,
  the bench's headline kernel) -- every output element;
* ogbn-mag layer 0 project-first: the transpose SpMM `aggregate_bwd` (mean)
  over U = 268k Y rows, which runs k_agg_bwd_p's multi-iteration prefetch
  rotation (U > 148*4 blocks x 8 warps x 4 columns) -- every element;
* ogbn-mag layer 0: build bit-exact (CSR + CSC + compact ids);
* Freebase layer 0 (R = 36): GAT forward (Z, stats) and backward (dY, ds_src,
  ds_dst) -- every element.
"""
import numpy as np
import pytest
import torch

import oracle
from synth import CONFIGS, generate_graph, generate_features, make_batch

from gpu_util import needs_gpu, gpu_build, csr_host, close_scaled, t, DEV, hf, assert_build_equal

pytestmark = [pytest.mark.gpu, needs_gpu]

_cache = {}


def _batch(key):
    if key not in _cache:
        cfg = CONFIGS[key]
        g = generate_graph(cfg)
        feat, foff = generate_features(cfg.type_counts, cfg.feat_dim)
        mb = make_batch(cfg, g, 0)
        rs = np.array([r.src for r in cfg.rels], np.int32)
        rd = np.array([r.dst for r in cfg.rels], np.int32)
        _cache[key] = (cfg, g, feat, foff, mb, rs, rd)
    return _cache[key]


def test_mag_build_layer0_bit_exact():
    cfg, g, feat, foff, mb, rs, rd = _batch("mag")
    blk = mb.layers[0]
    sh, csr, st = gpu_build(blk, g.edge_type, rs, rd, csc=True, ranged=True)
    assert hf().read_status(st) == 0
    ref = oracle.build(oracle.Shape.of(blk, rs, rd), blk, g.edge_type)
    assert_build_equal(csr_host(sh, csr), ref)
    assert sh.N > 400_000


def test_mag_aggregate_features_layer0_elementwise():
    cfg, g, feat, foff, mb, rs, rd = _batch("mag")
    blk = mb.layers[0]
    K = cfg.feat_dim
    sh, csr, st = gpu_build(blk, g.edge_type, rs, rd, csc=False, ranged=True)
    gid = mb.gather_ids(foff).astype(np.int32)
    feat_d = torch.from_numpy(feat).to(DEV)
    gid_d = t(gid, torch.int32)
    colx = torch.empty(max(sh.N, 1), dtype=torch.int32, device=DEV)
    Xa = torch.full((sh.rows, K), float("nan"), device=DEV)
    hf().feature_cols(sh, csr, gid_d, colx)
    hf().aggregate_features_cols(sh, csr, cfg.agg, K, feat_d, colx, Xa)
    torch.cuda.synchronize()
    osh = oracle.Shape.of(blk, rs, rd)
    X0 = feat[gid]                               # the gathered rows (same values)
    ref = oracle.aggregate_features(osh, blk, g.edge_type, cfg.agg, K, X0, None)
    A = oracle.aggregate_features(osh, blk, g.edge_type, cfg.agg, K, np.abs(X0), None)
    close_scaled(Xa.cpu().numpy(), ref, A, what="mag Xagg layer 0")
    assert sh.N > 400_000 and sh.rows > 30_000


def test_mag_aggregate_bwd_layer0_elementwise():
    cfg, g, feat, foff, mb, rs, rd = _batch("mag")
    blk = mb.layers[0]
    D = cfg.hidden
    sh, csr, st = gpu_build(blk, g.edge_type, rs, rd, csc=True, ranged=True)
    ch = csr_host(sh, csr)
    U = ch["U"]
    assert U > 148 * 4 * 8 * 4          # the prefetch rotation of k_agg_bwd_p runs > 1 round
    rng = np.random.default_rng(2408)
    G = rng.standard_normal((sh.dst_rows, D)).astype(np.float32)
    dY = torch.full((max(sh.U_max, 1), D), float("nan"), device=DEV)
    ws = torch.empty(hf().aggregate_bwd_ws_bytes(sh, cfg.agg, 1) // 4 + 16, device=DEV)
    hf().aggregate_bwd(sh, csr, cfg.agg, D, 1, 0.2, t(G), None, None, None, None, dY, None,
                       None, ws)
    torch.cuda.synchronize()
    osh = oracle.Shape.of(blk, rs, rd)
    ref = oracle.aggregate_bwd(osh, blk, g.edge_type, ch, cfg.agg, D, 1, G, np.zeros((U, D)))
    A = oracle.aggregate_bwd(osh, blk, g.edge_type, ch, cfg.agg, D, 1, np.abs(G),
                             np.zeros((U, D)))["dY"]
    close_scaled(dY.cpu().numpy()[:U], ref["dY"], A, what="mag dY layer 0")


def test_freebase_gat_layer0_elementwise():
    cfg, g, feat, foff, mb, rs, rd = _batch("freebase")
    blk = mb.layers[0]
    D, H = cfg.hidden, cfg.heads
    sh, csr, st = gpu_build(blk, g.edge_type, rs, rd, csc=True, ranged=True)
    ch = csr_host(sh, csr)
    U = ch["U"]
    rng = np.random.default_rng(36)
    Y = rng.standard_normal((U, D)).astype(np.float32)
    ss = rng.standard_normal((U, H)).astype(np.float32)
    sd = rng.standard_normal((sh.rows, H)).astype(np.float32)
    G = rng.standard_normal((sh.dst_rows, D)).astype(np.float32)
    Z = torch.zeros(sh.rows, D, device=DEV)
    stats = torch.zeros(sh.rows, 2 * H, device=DEV)
    hf().aggregate_fwd(csr, sh.rows, "gat", D, H, 0.2, t(Y), t(ss), t(sd), Z, stats)
    osh = oracle.Shape.of(blk, rs, rd)
    fw = oracle.aggregate_fwd(osh, blk, g.edge_type, ch, "gat", D, H, Y, ss, sd)
    A = oracle.aggregate_fwd(osh, blk, g.edge_type, ch, "gat", D, H, np.abs(Y), ss, sd)["Z"]
    close_scaled(Z.cpu().numpy(), fw["Z"], A, what="freebase Z layer 0")
    dY = torch.zeros(U, D, device=DEV)
    dss = torch.zeros(U, H, device=DEV)
    dsd = torch.zeros(sh.rows, H, device=DEV)
    ws = torch.empty(hf().aggregate_bwd_ws_bytes(sh, "gat", H) // 4 + 16, device=DEV)
    hf().aggregate_bwd(sh, csr, "gat", D, H, 0.2, t(G), t(Y), t(ss), t(sd), stats, dY, dss, dsd,
                       ws)
    torch.cuda.synchronize()
    ref = oracle.aggregate_bwd(osh, blk, g.edge_type, ch, "gat", D, H, G, Y, ss, sd)
    sc = oracle.aggregate_bwd(osh, blk, g.edge_type, ch, "gat", D, H, np.abs(G), np.abs(Y), ss,
                              sd)
    close_scaled(dY.cpu().numpy(), ref["dY"], sc["dY"], what="freebase dY layer 0")
    from test_gpu_stages import gat_ds_scales
    scale_s, scale_d = gat_ds_scales(sh, ch, fw, G, Y, D, H)
    close_scaled(dss.cpu().numpy(), ref["ds_src"], scale_s, what="freebase ds_src layer 0")
    close_scaled(dsd.cpu().numpy(), ref["ds_dst"], scale_d, what="freebase ds_dst layer 0")
