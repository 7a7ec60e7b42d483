"""-m gpu: the padded GPU-sampler layout (hifuse_sample_blocks_padded) and the
graph-mode GPU-sampled training loop (SampledLoop) that bench.py times under
gpu_sampler.

* padded vs compact layout of the same batch key: the same sampled vertices
  in the same order, the same edges (as vertex pairs + edge ids) in the same
  order, null edges in the padded tail, padding slots -1 / gather row of the
  type's first vertex (integer work: bit-exact);
* an eager step on the padded batch gives the compact batch's loss
  bit-for-bit (forward rows are computed independently of the padding rows)
  and its gradients to 1e-5 (padding rows only regroup the weight-gradient
  sums);
* SampledLoop's graph replays (step i, build i+1, sampling i+2 in one graph)
  give parameters BIT-IDENTICAL to eager steps on the same padded batches;
* a batch past the capacities takes the compact fallback and the run still
  matches eager compact steps to the fp32 tolerance.
"""
import numpy as np
import pytest
import torch

from synth import CONFIGS, generate_graph, generate_features, epoch_seeds, batch_key, make_params
from synth.sampler import labels_of

from gpu_util import needs_gpu, DEV, hf

pytestmark = [pytest.mark.gpu, needs_gpu]

_cache = {}


def setup(key):
    if key not in _cache:
        cfg = CONFIGS[key]
        g = generate_graph(cfg)
        feat, foff = generate_features(cfg.type_counts, cfg.feat_dim)
        _cache[key] = (cfg, g, g.in_csc(), feat)
    return _cache[key]


def _sampler(cfg, g, csc, nbuf=4):
    from paper_2408_08490_b200.sampler import GpuSampler
    return GpuSampler(g.rel_src, g.rel_dst, g.counts, csc, list(cfg.fanout)[::-1],
                      cfg.batch_size, DEV, nbuf=nbuf)


def _seeds(cfg, b):
    """Batch b of epoch 0, full batches only (wrapping: the padded layout
    has exactly B seeds per batch)."""
    perm = epoch_seeds(cfg, 0)
    B = cfg.batch_size
    b %= len(perm) // B
    s = perm[b * B:(b + 1) * B]
    return (torch.from_numpy(s.astype(np.int32)).pin_memory(),
            torch.from_numpy(labels_of(cfg, s)).pin_memory(), batch_key(0, b))


def _caps(cfg, smp, nb=2):
    from paper_2408_08490_b200.sampler import padded_caps
    seen = []
    for b in range(nb):
        s, _, k = _seeds(cfg, b)
        smp.sample(s.to(DEV), cfg.target_type, k, buf=0)
        seen.append(smp.counts(buf=0))
    return padded_caps(seen, cfg.num_types, cfg.target_type, cfg.batch_size)


def _trainer(cfg, prec="tf32", order="project_first"):
    from paper_2408_08490_b200.step import Trainer
    rs = np.array([r.src for r in cfg.rels], np.int32)
    rd = np.array([r.dst for r in cfg.rels], np.int32)
    tr = Trainer(cfg.num_types, cfg.num_rels, rs, rd, cfg.feat_dim, cfg.hidden, cfg.heads,
                 cfg.num_classes, cfg.num_layers, cfg.model, cfg.agg, DEV, lr=0.05, prec=prec,
                 order=order)
    tr.load_params(make_params(cfg))
    return tr


@pytest.mark.parametrize("key", ["imdb", "dblp", "mag"])
def test_padded_layout_matches_compact(key):
    cfg, g, csc, _ = setup(key)
    T = cfg.num_types
    smp = _sampler(cfg, g, csc)
    src_cap, edge_pad = _caps(cfg, smp)
    goff = np.concatenate([[0], np.cumsum(smp.counts_h)])
    for b in (2, 3):                       # batches not used for the capacities
        s, _, k = _seeds(cfg, b)
        sd = s.to(DEV)
        smp.sample(sd, cfg.target_type, k, buf=0)
        smp.sample_padded(sd, cfg.target_type, src_cap, edge_pad, buf=1, key=k)
        torch.cuda.synchronize()
        assert hf().read_status(smp.status) == 0
        cc, cp = smp.counts(buf=0), smp.counts(buf=1)
        for l in range(smp.L):
            oc, op = smp.bufs[0][0][l], smp.bufs[1][0][l]
            nc_src, nc_dst, N = cc[l][:T], cc[l][T:2 * T], int(cc[l][2 * T])
            assert int(cp[l][2 * T]) == N
            assert np.all(cp[l][:T] - cp[l][T:2 * T] == nc_src - nc_dst)   # same new sources
            off_c = np.concatenate([[0], np.cumsum(nc_src)])
            off_p = np.concatenate([[0], np.cumsum(src_cap[l])])
            gc = oc["gid"][:off_c[-1]].cpu().numpy()
            gp = op["gid"][:off_p[-1]].cpu().numpy()
            vc, vp = [], []                     # vertex of every local id, per type
            for t in range(T):
                vc.append(gc[off_c[t]:off_c[t + 1]])
                vp.append(gp[off_p[t]:off_p[t + 1]])
                real = vp[t][vp[t] >= 0]
                assert np.array_equal(real, vc[t]), (l, t)   # same vertices, same order
                # padding: -1 slots, gather row = the type's first feature row
                pad = np.nonzero(vp[t] < 0)[0]
                if l == 0 and len(pad):
                    ga = op["gather"][off_p[t]:off_p[t + 1]].cpu().numpy()
                    assert np.all(ga[pad] == goff[t])
                    assert np.array_equal(ga[vp[t] >= 0], goff[t] + real)
            # edges as (src vertex, dst vertex, eid): identical sequences
            rs = np.array([r.src for r in cfg.rels])
            rd = np.array([r.dst for r in cfg.rels])
            et = g.edge_type
            for name, o, v in (("c", oc, vc), ("p", op, vp)):
                eid = o["eid"][:N].cpu().numpy()
                r = et[eid]
                src = o["src"][:N].cpu().numpy()
                dst = o["dst"][:N].cpu().numpy()
                sv = np.array([v[rs[ri]][x] for ri, x in zip(r, src)])
                dv = np.array([v[rd[ri]][x] for ri, x in zip(r, dst)])
                if name == "c":
                    ref = (sv, dv, eid)
                else:
                    assert np.array_equal(ref[0], sv) and np.array_equal(ref[1], dv)
                    assert np.array_equal(ref[2], eid)
            # null tail
            ep = int(edge_pad[l])
            assert np.all(op["eid"][N:ep].cpu().numpy() == -1)


@pytest.mark.parametrize("key,prec,order", [("imdb", "fp32", "project_first"),
                                            ("imdb", "tf32", "project_first"),
                                            ("dblp", "tf32", "agg_first")])
def test_padded_step_matches_compact(key, prec, order):
    from paper_2408_08490_b200.sampler import SampledBatch, PaddedBatch
    cfg, g, csc, feat = setup(key)
    smp = _sampler(cfg, g, csc)
    src_cap, edge_pad = _caps(cfg, smp)
    feat_d = torch.from_numpy(feat).to(DEV)
    et_d = torch.from_numpy(g.edge_type).to(DEV)
    s, lab, k = _seeds(cfg, 2)
    sd, ld = s.to(DEV), lab.to(DEV)
    smp.sample(sd, cfg.target_type, k, buf=0)
    smp.sample_padded(sd, cfg.target_type, src_cap, edge_pad, buf=1, key=k)
    torch.cuda.synchronize()
    tr_c, tr_p = _trainer(cfg, prec, order), _trainer(cfg, prec, order)
    loss_c = float(tr_c.step(SampledBatch(smp, smp.counts(buf=0), ld, cfg.target_type, buf=0),
                             feat_d, et_d, update=False).item())
    loss_p = float(tr_p.step(PaddedBatch(smp, src_cap, edge_pad, 1, ld, cfg.target_type),
                             feat_d, et_d, update=False).item())
    assert hf().read_status(tr_c.status) == 0 and hf().read_status(tr_p.status) == 0
    assert loss_p == loss_c
    gc, gp = tr_c.grads.double(), tr_p.grads.double()
    assert float((gp - gc).norm() / gc.norm()) <= 1e-5
    assert torch.allclose(gp, gc, rtol=1e-4, atol=1e-6 * float(gc.abs().max()))


def _loop(cfg, g, csc, feat, tr, src_cap, edge_pad):
    from paper_2408_08490_b200.sampled_loop import SampledLoop
    smp = _sampler(cfg, g, csc)
    feat_d = torch.from_numpy(feat).to(DEV)
    et_d = torch.from_numpy(g.edge_type).to(DEV)
    tr.prepare_graph(et_d)
    loop = SampledLoop(tr, smp, feat_d, et_d, cfg.target_type, src_cap, edge_pad,
                       lambda i: _seeds(cfg, i))
    return loop, smp, feat_d, et_d


@pytest.mark.parametrize("key,order", [("imdb", "project_first"), ("dblp", "agg_first"),
                                       ("mag", "agg_first")])
def test_sampled_loop_graphs_match_eager(key, order):
    from paper_2408_08490_b200.sampler import PaddedBatch
    cfg, g, csc, feat = setup(key)
    smp0 = _sampler(cfg, g, csc)
    src_cap, edge_pad = _caps(cfg, smp0)
    n = 7
    # eager reference: padded batches, one eager step each
    tr_e = _trainer(cfg, "tf32", order)
    feat_d = torch.from_numpy(feat).to(DEV)
    et_d = torch.from_numpy(g.edge_type).to(DEV)
    tr_e.prepare_graph(et_d)
    losses_e = []
    for i in range(n):
        s, lab, k = _seeds(cfg, i)
        ld = lab.to(DEV)
        smp0.sample_padded(s.to(DEV), cfg.target_type, src_cap, edge_pad, buf=1, key=k)
        losses_e.append(float(tr_e.step(PaddedBatch(smp0, src_cap, edge_pad, 1, ld,
                                                    cfg.target_type), feat_d, et_d).item()))
    # graph mode: two runs (primed, then continued)
    tr_g = _trainer(cfg, "tf32", order)
    loop, smp, _, _ = _loop(cfg, g, csc, feat, tr_g, src_cap, edge_pad)
    loop.capture()
    losses_g = []
    for i in range(n):
        loop.run(i, 1, prime=(i == 0))
        losses_g.append(float(tr_g.loss.item()))
    torch.cuda.synchronize()
    assert loop.fallbacks == 0
    assert hf().read_status(tr_g.status) == 0 and hf().read_status(smp.status) == 0
    assert losses_g == losses_e
    assert torch.equal(tr_g.params, tr_e.params)


def test_sampled_loop_fallback():
    """Capacities from ONE batch with no margin: later batches overflow, take
    the compact fallback, and the run matches eager compact steps."""
    from paper_2408_08490_b200.sampler import SampledBatch, padded_caps
    cfg, g, csc, feat = setup("imdb")
    smp0 = _sampler(cfg, g, csc)
    s, _, k = _seeds(cfg, 0)
    smp0.sample(s.to(DEV), cfg.target_type, k, buf=0)
    src_cap, edge_pad = padded_caps([smp0.counts(buf=0)], cfg.num_types, cfg.target_type,
                                    cfg.batch_size, margin=0.0, slack=0, align=1)
    n = 6
    tr_e = _trainer(cfg, "fp32")
    feat_d = torch.from_numpy(feat).to(DEV)
    et_d = torch.from_numpy(g.edge_type).to(DEV)
    for i in range(n):
        s, lab, k = _seeds(cfg, i)
        smp0.sample(s.to(DEV), cfg.target_type, k, buf=0)
        tr_e.step(SampledBatch(smp0, smp0.counts(buf=0), lab.to(DEV), cfg.target_type, buf=0),
                  feat_d, et_d)
    tr_g = _trainer(cfg, "fp32")
    loop, smp, _, _ = _loop(cfg, g, csc, feat, tr_g, src_cap, edge_pad)
    loop.capture()
    loop.run(0, n)
    torch.cuda.synchronize()
    assert loop.fallbacks >= 1
    assert hf().read_status(tr_g.status) == 0
    # the overflow bit is the sampler's (expected here); nothing else
    assert hf().read_status(smp.status) & ~64 == 0
    d = (tr_g.params.double() - tr_e.params.double()).norm() / tr_e.params.double().norm()
    assert float(d) <= 1e-6
