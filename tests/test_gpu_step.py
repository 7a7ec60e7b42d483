"""-m gpu: a whole training step (build, forward, loss, backward, SGD) through
the C ABI against the oracle model, on the first sampled batch of every
BASELINE.json configuration at full size, plus launch-count independence
from R (the paper's kernel-count claim)."""
import numpy as np
import pytest
import torch

import oracle.model as om
from synth import CONFIGS, generate_graph, generate_features, make_batch, make_params

from gpu_util import needs_gpu, DEV, hf

pytestmark = [pytest.mark.gpu, needs_gpu]

_cache = {}


def setup(key):
    if key not in _cache:
        if key.endswith("_xrel"):        # RGAT with the across-relation softmax (NEXT(2))
            import dataclasses
            cfg = dataclasses.replace(CONFIGS[key[:-5]], agg="gat_xrel", key=key)
        elif key.endswith("_mul"):       # RGAT with multiplicative attention (NEXT(2))
            import dataclasses
            cfg = dataclasses.replace(CONFIGS[key[:-4]], agg="gat_mul", key=key)
        elif key.endswith("_han"):       # HAN semantic-attention fusion (NEXT(2))
            cfg = CONFIGS[key[:-4]]
        else:
            cfg = CONFIGS[key]
        g = generate_graph(cfg)
        feat, foff = generate_features(cfg.type_counts, cfg.feat_dim)
        _cache[key] = (cfg, g, feat, foff)
    return _cache[key]


def rel_l2(a, b):
    a = np.asarray(a, np.float64).ravel()
    b = np.asarray(b, np.float64).ravel()
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30)


@pytest.mark.parametrize("prec,order", [("fp32", "project_first"), ("tf32", "project_first"),
                                        ("tf32", "agg_first"), ("tf32", "agg_first_bf16"),
                                        ("bf16", "project_first"), ("tf32", "project_first_y16")])
@pytest.mark.parametrize("key", ["acm", "dblp", "imdb", "freebase", "mag", "imdb_xrel",
                                 "freebase_xrel", "imdb_mul", "freebase_mul", "imdb_han",
                                 "dblp_han", "freebase_han"])
def test_step_matches_oracle(key, prec, order):
    """agg_first (RGCN input layer aggregates raw features, then projects) is
    checked against the same project-first oracle model: equal by linearity."""
    from paper_2408_08490_b200.step import Trainer, DeviceBatch
    cfg, g, feat, foff = setup(key)
    mb = make_batch(cfg, g, 0)
    rs = np.array([r.src for r in cfg.rels], np.int32)
    rd = np.array([r.dst for r in cfg.rels], np.int32)
    fusion = "han" if key.endswith("_han") else "sum"
    params = make_params(cfg, fusion=fusion)
    bf16 = order == "agg_first_bf16"      # NEXT(3): BF16 feature store, oracle fed rounded values
    if bf16 and (cfg.model != "rgcn" or fusion != "sum"):
        pytest.skip("the BF16 feature store needs the aggregate-first RGCN input layer")
    order = "agg_first" if bf16 else order
    y16 = order == "project_first_y16"   # NEXT(3): BF16 storage of Y (reading C25)
    if y16 and (cfg.model != "rgcn" or fusion != "sum"):
        pytest.skip("BF16 Y storage is an RGCN (sum fusion) path")
    order = "project_first" if y16 else order
    if prec == "bf16" and fusion == "han":
        pytest.skip("HAN's semantic-attention adjoint amplifies the BF16 operand error past "
                    "any useful bound (DESIGN.md §5); HAN is checked in fp32 and tf32")
    tr = Trainer(cfg.num_types, cfg.num_rels, rs, rd, cfg.feat_dim, cfg.hidden, cfg.heads,
                 cfg.num_classes, cfg.num_layers, cfg.model, cfg.agg, DEV, lr=0.0, prec=prec,
                 order=order, fusion=fusion, feat_dtype="bf16" if bf16 else "fp32",
                 y_dtype="bf16" if y16 else "fp32")
    if order == "agg_first" and not tr.agg_first:
        pytest.skip("aggregate-first applies to RGCN only")
    tr.load_params(params)
    db = DeviceBatch(mb, rs, rd, foff, cfg.target_type, DEV)
    feat_d = torch.from_numpy(feat).to(DEV)
    if bf16:
        feat_d = feat_d.to(torch.bfloat16)
        feat = feat_d.float().cpu().numpy()          # the oracle sees the rounded store
    et_d = torch.from_numpy(g.edge_type).to(DEV)
    loss = tr.step(db, feat_d, et_d, update=False)
    torch.cuda.synchronize()
    assert hf().read_status(tr.status) == 0
    # oracle on the gathered layer-0 rows (same values as the global store)
    gid = mb.gather_ids(foff)
    X0 = feat[gid].astype(np.float64)
    fw = om.forward(mb.layers, g.edge_type, rs, rd, X0, np.arange(len(gid), dtype=np.int32),
                    params, cfg.agg, cfg.heads, labels=mb.labels, target_type=cfg.target_type)
    gr = om.backward(fw, mb.layers, g.edge_type, params, mb.labels, cfg.agg, cfg.heads)
    # fp32: CUDA-core projection -> tight; tf32: tcgen05 projection (reading
    # C18: kind::tf32 drops the low 13 mantissa bits, u = 2^-10).  The layer-0
    # weight gradients sit behind ~5 chained TF32 GEMMs (fwd proj 0, proj 1,
    # bwd dgrad 1, wgrad 0 + attention), so DESIGN.md §Tolerances allows
    # 5 u x 4 (conditioning) = 2e-2 there; the GEMM kernels themselves are
    # pinned bit-exact on TF32-representable inputs (test_gpu_stages).
    ltol, tol, htol = (1e-5, 2e-4, 1e-5) if prec == "fp32" else (2e-3, 2e-2, 5e-3)
    if prec == "bf16" or y16:
        # BF16 projection operands against the unrounded fp64 oracle: u = 2^-8
        # per operand rounding (~u on H and the loss, the weight
        # gradients behind two BF16 forward GEMMs and the TF32 backward chain
        # ~10 u)
        ltol, tol, htol = 1e-2, 5e-2, 2e-2
    assert abs(float(loss.item()) - fw["loss"]) <= ltol * max(1.0, abs(fw["loss"]))
    checks = [("Wc", gr["Wc"]), ("bc", gr["bc"])]
    for l in range(cfg.num_layers):
        for k in ("W_rel", "W_root", "bias", "att", "sem_W", "sem_b", "sem_q"):
            if gr["layers"][l].get(k) is not None and f"{l}.{k}" in tr.Gd:
                checks.append((f"{l}.{k}", gr["layers"][l][k]))
    for name, ref in checks:
        err = rel_l2(tr.Gd[name].cpu().numpy(), ref)
        # HAN fusion under TF32: every gradient below the fusion goes
        # through dw_r = beta_r (dbeta_r - sum_r' beta_r' dbeta_r'), a softmax
        # adjoint whose terms nearly cancel (3-5 relations per type), so the
        # TF32 errors of the chain above are amplified by |dbeta| / |dw|
        # (~5x measured on IMDB); the same gradients are checked at 2e-4 in
        # fp32
        t_ = 0.1 if (prec != "fp32" and key.endswith("_han")) else tol
        assert err <= t_, f"{key} grad {name}: rel L2 {err:.3e}"
    # logits-level: the last layer's H on the seeds
    last = tr.last["acts"][-1]["H"][db.h_row0:db.h_row0 + db.B].cpu().numpy()
    err = rel_l2(last, fw["hs"])
    assert err <= htol, f"{key} H: {err:.3e}"


def test_sgd_update_and_determinism():
    from paper_2408_08490_b200.step import Trainer, DeviceBatch
    cfg, g, feat, foff = setup("dblp")
    rs = np.array([r.src for r in cfg.rels], np.int32)
    rd = np.array([r.dst for r in cfg.rels], np.int32)
    feat_d = torch.from_numpy(feat).to(DEV)
    et_d = torch.from_numpy(g.edge_type).to(DEV)
    outs = []
    for _ in range(2):
        tr = Trainer(cfg.num_types, cfg.num_rels, rs, rd, cfg.feat_dim, cfg.hidden, cfg.heads,
                     cfg.num_classes, cfg.num_layers, cfg.model, cfg.agg, DEV, lr=0.05, prec="tf32")
        tr.load_params(make_params(cfg))
        p0 = tr.params.clone()
        losses = []
        for b in range(3):
            db = DeviceBatch(make_batch(cfg, g, b), rs, rd, foff, cfg.target_type, DEV)
            losses.append(float(tr.step(db, feat_d, et_d).item()))
        outs.append((losses, tr.params.clone()))
        assert not torch.equal(p0, tr.params)
    assert outs[0][0] == outs[1][0]
    assert torch.equal(outs[0][1], outs[1][1])


def test_kernel_count_independent_of_relations():
    """Forward kernels per layer do not grow with R (merged path)."""
    from synth import random_block, random_schema
    from gpu_util import gpu_build
    counts = []
    for R in (4, 36, 144):
        rng = np.random.default_rng(R)
        rs, rd = random_schema(rng, 4, R)
        blk, et = random_block(rng, [500] * 4, [100] * 4, rs, rd, 3000)
        sh, csr, _ = gpu_build(blk, et, rs, rd)
        Y = torch.randn(max(sh.U_max, 1), 128, device=DEV)
        Z = torch.zeros(sh.rows, 128, device=DEV)
        H = torch.zeros(sh.dst_rows, 128, device=DEV)
        n0 = hf().kernel_launches()
        hf().aggregate_fwd(csr, sh.rows, "mean", 128, 1, 0.2, Y, None, None, Z, None)
        hf().semantic_fuse(sh, 128, "relu", Z, None, None, H)
        counts.append(hf().kernel_launches() - n0)
    assert counts[0] == counts[1] == counts[2] == 2


def test_graph_replay_matches_eager():
    """The captured whole-step CUDA graph computes exactly what eager launches do."""
    from paper_2408_08490_b200.step import Trainer, DeviceBatch
    cfg, g, feat, foff = setup("imdb")
    rs = np.array([r.src for r in cfg.rels], np.int32)
    rd = np.array([r.dst for r in cfg.rels], np.int32)
    feat_d = torch.from_numpy(feat).to(DEV)
    et_d = torch.from_numpy(g.edge_type).to(DEV)
    dbs = [DeviceBatch(make_batch(cfg, g, b), rs, rd, foff, cfg.target_type, DEV) for b in range(2)]
    res = []
    for mode in ("eager", "graph"):
        tr = Trainer(cfg.num_types, cfg.num_rels, rs, rd, cfg.feat_dim, cfg.hidden, cfg.heads,
                     cfg.num_classes, cfg.num_layers, cfg.model, cfg.agg, DEV, lr=0.05, prec="tf32")
        tr.load_params(make_params(cfg))
        for db in dbs:
            tr.step(db, feat_d, et_d, update=False)
        losses = []
        if mode == "graph":
            graphs = [tr.capture(db, feat_d, et_d)[0] for db in dbs]
        for i in range(4):
            if mode == "eager":
                tr.step(dbs[i % 2], feat_d, et_d)
            else:
                graphs[i % 2].replay()
            losses.append(float(tr.loss.item()))
        res.append((losses, tr.params.clone()))
    assert res[0][0] == res[1][0]
    assert torch.equal(res[0][1], res[1][1])
