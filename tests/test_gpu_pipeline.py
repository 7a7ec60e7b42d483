"""-m gpu: the graphs bench.py times are the graphs that are parity-tested.

bench.py replays `Trainer.capture_pipelined` graphs: batch i's compute on a
high-priority stream while a side stream builds batch i+1's semantic graphs
(Fig. 6 pipeline), sharing the build workspace and the
status word.  These tests build the pool and the graphs exactly as bench.py
does (`bench.build_graphs`) and require loss and parameters to be
BIT-IDENTICAL to eager `Trainer.step` on the same batch sequence, including
the wrap from the last pool batch back to batch 0.  Eager steps are in turn
checked against the oracle model in test_gpu_step.py.
"""
import numpy as np
import pytest
import torch

from synth import CONFIGS, generate_graph, generate_features, make_batch, make_params

from gpu_util import needs_gpu, DEV, hf

pytestmark = [pytest.mark.gpu, needs_gpu]


def _setup(key, P):
    import dataclasses
    cfg = CONFIGS[key[:-5]] if key.endswith("_xrel") else CONFIGS[key]
    if key.endswith("_xrel"):
        cfg = dataclasses.replace(cfg, agg="gat_xrel", key=key)
    g = generate_graph(cfg)
    feat, foff = generate_features(cfg.type_counts, cfg.feat_dim)
    rs = np.array([r.src for r in cfg.rels], np.int32)
    rd = np.array([r.dst for r in cfg.rels], np.int32)
    mbs = [make_batch(cfg, g, b) for b in range(P)]
    return cfg, g, feat, foff, rs, rd, mbs


def _trainer(cfg, rs, rd, order, et_d):
    from paper_2408_08490_b200.step import Trainer
    tr = Trainer(cfg.num_types, cfg.num_rels, rs, rd, cfg.feat_dim, cfg.hidden, cfg.heads,
                 cfg.num_classes, cfg.num_layers, cfg.model, cfg.agg, DEV, lr=0.05, prec="tf32",
                 order=order)
    tr.load_params(make_params(cfg))
    tr.prepare_graph(et_d)
    return tr


@pytest.mark.parametrize("key,order", [("mag", "agg_first"), ("mag", "project_first"),
                                       ("imdb", "project_first"), ("freebase", "project_first"),
                                       ("imdb_xrel", "project_first"), ("dblp", "agg_first")])
def test_pipelined_graphs_match_eager(key, order):
    import bench
    from paper_2408_08490_b200.step import DeviceBatch
    P, steps = 3, 7                      # 7 replays: wraps back to batch 0 twice
    cfg, g, feat, foff, rs, rd, mbs = _setup(key, P)
    feat_d = torch.from_numpy(feat).to(DEV)
    et_d = torch.from_numpy(g.edge_type).to(DEV)

    # eager reference: plain Trainer.step over the same batch sequence
    tr_e = _trainer(cfg, rs, rd, order, et_d)
    pool_e = [DeviceBatch(mb, rs, rd, foff, cfg.target_type, DEV) for mb in mbs]
    for i, db in enumerate(pool_e):
        db.slot = i
    eager_losses = []
    for i in range(steps):
        eager_losses.append(float(tr_e.step(pool_e[i % P], feat_d, et_d).item()))
    assert hf().read_status(tr_e.status) == 0

    # the bench's own construction: sizing pass, serial and pipelined graphs
    tr_p = _trainer(cfg, rs, rd, order, et_d)
    pool_p = [DeviceBatch(mb, rs, rd, foff, cfg.target_type, DEV, pin=True) for mb in mbs]
    side = torch.cuda.Stream()
    gset = bench.build_graphs(tr_p, pool_p, feat_d, et_d, side, world=1, pipeline=True)
    tr_p.load_params(make_params(cfg))      # the sizing pass ran with update=False
    assert torch.equal(tr_p.params, _trainer(cfg, rs, rd, order, et_d).params)
    bench.prime_pipeline(tr_p, gset, pool_p, et_d)
    graph_losses = []
    for i in range(steps):
        gset["graphs"][i % P][0].replay()
        graph_losses.append(float(tr_p.loss.item()))
    torch.cuda.synchronize()
    assert hf().read_status(tr_p.status) == 0
    assert graph_losses == eager_losses, (graph_losses, eager_losses)
    assert torch.equal(tr_p.params, tr_e.params)
    assert torch.equal(tr_p.grads, tr_e.grads)

    # the serial graphs (bench's serial_ms_per_step) compute the same
    tr_s = _trainer(cfg, rs, rd, order, et_d)
    gs = bench.build_graphs(tr_s, pool_p, feat_d, et_d, side, world=1, pipeline=False)
    tr_s.load_params(make_params(cfg))
    serial_losses = []
    for i in range(steps):
        gs["graphs"][i % P][0].replay()
        serial_losses.append(float(tr_s.loss.item()))
    assert serial_losses == eager_losses
    assert torch.equal(tr_s.params, tr_e.params)


def test_e2e_loop_matches_eager():
    """bench.py's e2e arm: pinned host -> device copy of each batch's inputs on a
    copy stream two steps ahead, graph replay, device -> host loss read; same
    losses as eager steps (IMDB)."""
    import bench
    from paper_2408_08490_b200.step import DeviceBatch
    P, steps = 4, 9                      # e2e copies run ahead: needs P >= 4
    cfg, g, feat, foff, rs, rd, mbs = _setup("imdb", P)
    feat_d = torch.from_numpy(feat).to(DEV)
    et_d = torch.from_numpy(g.edge_type).to(DEV)
    tr_e = _trainer(cfg, rs, rd, "project_first", et_d)
    pool_e = [DeviceBatch(mb, rs, rd, foff, cfg.target_type, DEV) for mb in mbs]
    for i, db in enumerate(pool_e):
        db.slot = i
    ref = [float(tr_e.step(pool_e[i % P], feat_d, et_d).item()) for i in range(steps)]

    tr = _trainer(cfg, rs, rd, "project_first", et_d)
    pool = [DeviceBatch(mb, rs, rd, foff, cfg.target_type, DEV, pin=True) for mb in mbs]
    side = torch.cuda.Stream()
    gset = bench.build_graphs(tr, pool, feat_d, et_d, side, world=1, pipeline=True)
    tr.load_params(make_params(cfg))
    # scramble the device copies of the inputs: the e2e loop must re-copy them
    for db in pool:
        for v in db.dev.values():
            for t in (v if isinstance(v, list) else [v]):
                t.fill_(0)
    runner = bench.StepRunner(tr, gset, pool, 1, DEV)
    got = runner.run_e2e_losses(steps, et_d)
    assert got == ref, (got, ref)
    assert torch.equal(tr.params, tr_e.params)
