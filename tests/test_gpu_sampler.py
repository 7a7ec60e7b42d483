"""-m gpu: the GPU neighbour sampler (hifuse_sample_blocks, NEXT(1)) against
the sampler oracle, bit-exact on every output (integer work), on the five
configurations' graphs; invariants at full batch size on ogbn-mag; a training
step fed by the GPU sampler equals one fed the same blocks from the host."""
import numpy as np
import pytest
import torch

from oracle.sampler import sample_blocks as oracle_sample
from synth import CONFIGS, generate_graph, generate_features, epoch_seeds, batch_key, make_params

from gpu_util import needs_gpu, DEV, hf

pytestmark = [pytest.mark.gpu, needs_gpu]

_cache = {}


def setup(key):
    if key not in _cache:
        cfg = CONFIGS[key]
        g = generate_graph(cfg)
        _cache[key] = (cfg, g, g.in_csc())
    return _cache[key]


def gpu_sample(cfg, g, csc, seeds, fanout, key):
    from paper_2408_08490_b200.sampler import GpuSampler
    smp = GpuSampler(g.rel_src, g.rel_dst, g.counts, csc, fanout, len(seeds), DEV)
    smp.sample(torch.from_numpy(np.asarray(seeds, np.int32)).to(DEV), cfg.target_type, key)
    torch.cuda.synchronize()
    assert hf().read_status(smp.status) == 0
    return smp


def compare(cfg, smp, ref):
    T = cfg.num_types
    goff = np.concatenate([[0], np.cumsum(smp.counts_h)])
    for l, (c, o, r) in enumerate(zip(smp.counts(), smp.out, ref)):
        assert np.array_equal(c[:T], r["n_src"]), (l, c[:T], r["n_src"])
        assert np.array_equal(c[T:2 * T], r["n_dst"]), l
        N = int(c[2 * T])
        assert N == len(r["edge_id"]), l
        assert np.array_equal(o["src"][:N].cpu().numpy(), r["src_local"]), l
        assert np.array_equal(o["dst"][:N].cpu().numpy(), r["dst_local"]), l
        assert np.array_equal(o["eid"][:N].cpu().numpy(), r["edge_id"]), l
        S = int(c[:T].sum())
        gid = np.concatenate(r["src_gid"])
        assert np.array_equal(o["gid"][:S].cpu().numpy(), gid), l
        if o["gather"] is not None:
            tt = np.repeat(np.arange(T), r["n_src"])
            assert np.array_equal(o["gather"][:S].cpu().numpy(), goff[tt] + gid), l


@pytest.mark.parametrize("key,nseeds", [("acm", 128), ("dblp", 256), ("imdb", 256),
                                        ("freebase", 128), ("mag", 24)])
def test_sampler_bit_exact(key, nseeds):
    cfg, g, csc = setup(key)
    seeds = epoch_seeds(cfg, 0)[:nseeds]
    k = batch_key(0, 0)
    smp = gpu_sample(cfg, g, csc, seeds, list(cfg.fanout)[::-1], k)
    ref = oracle_sample(csc, g.rel_src, g.rel_dst, g.counts, seeds, cfg.target_type,
                        list(cfg.fanout)[::-1], k)
    compare(cfg, smp, ref)


def test_sampler_mag_full_batch_invariants():
    """1024 seeds, fanout [25, 20]: no phantom edges, message-flow prefix,
    per-(destination, relation) counts = min(deg, fanout), ascending new ids."""
    cfg, g, csc = setup("mag")
    seeds = epoch_seeds(cfg, 0)[:1024]
    fan = list(cfg.fanout)[::-1]
    smp = gpu_sample(cfg, g, csc, seeds, fan, batch_key(0, 3))
    T = cfg.num_types
    cnt = smp.counts()
    et = g.edge_type
    gsrc = np.concatenate(g.src)
    gdst = np.concatenate(g.dst)
    for l, (c, o) in enumerate(zip(cnt, smp.out)):
        n_src, n_dst, N = c[:T], c[T:2 * T], int(c[2 * T])
        src = o["src"][:N].cpu().numpy()
        dst = o["dst"][:N].cpu().numpy()
        eid = o["eid"][:N].cpu().numpy()
        gid = o["gid"][:int(n_src.sum())].cpu().numpy().astype(np.int64)
        so = np.concatenate([[0], np.cumsum(n_src)])
        r = et[eid]
        assert np.all(gid[so[g.rel_src[r]] + src] == gsrc[eid])
        assert np.all(gid[so[g.rel_dst[r]] + dst] == gdst[eid])
        assert np.all(src < n_src[g.rel_src[r]]) and np.all(dst < n_dst[g.rel_dst[r]])
        for t in range(T):
            seg = gid[so[t]:so[t + 1]]
            assert len(np.unique(seg)) == len(seg)
            assert np.all(np.diff(seg[n_dst[t]:]) > 0)
        # per (destination, relation) edge counts
        key_ = (so[g.rel_dst[r]] + dst).astype(np.int64) * 64 + r
        uk, kc = np.unique(key_, return_counts=True)
        v = gid[uk // 64]
        rr = uk % 64
        for q in range(0, len(uk), max(1, len(uk) // 300)):
            ptr = csc[rr[q]][0]
            deg = int(ptr[v[q] + 1] - ptr[v[q]])
            assert kc[q] == min(deg, fan[l]), q
        if l + 1 < len(cnt):
            c2 = cnt[l + 1]
            assert np.array_equal(n_dst, c2[:T])
    assert np.array_equal(smp.out[-1]["gid"][:1024].cpu().numpy(), seeds)


def test_sampler_deterministic_across_stamps():
    cfg, g, csc = setup("imdb")
    from paper_2408_08490_b200.sampler import GpuSampler
    seeds = torch.from_numpy(epoch_seeds(cfg, 1)[:512].astype(np.int32)).to(DEV)
    smp = GpuSampler(g.rel_src, g.rel_dst, g.counts, csc, list(cfg.fanout)[::-1], 512, DEV)
    outs = []
    for k in (77, 78, 77):
        smp.sample(seeds, cfg.target_type, k)
        torch.cuda.synchronize()
        N = int(smp.counts()[0][-1])
        outs.append(smp.out[0]["eid"][:N].cpu().numpy().copy())
    assert np.array_equal(outs[0], outs[2]) and not np.array_equal(outs[0], outs[1])


def test_step_on_gpu_sampled_batch_equals_host_fed():
    """The Trainer consumes a GPU-sampled batch exactly like the same blocks
    uploaded from the host (bit-identical loss and gradients)."""
    from paper_2408_08490_b200.sampler import SampledBatch
    from paper_2408_08490_b200.step import Trainer, DeviceBatch
    from synth.sampler import LayerBlock, MiniBatch, labels_of
    cfg, g, csc = setup("imdb")
    feat, foff = generate_features(cfg.type_counts, cfg.feat_dim)
    seeds = epoch_seeds(cfg, 0)[:256]
    fan = list(cfg.fanout)[::-1]
    k = batch_key(0, 1)
    smp = gpu_sample(cfg, g, csc, seeds, fan, k)
    labels = labels_of(cfg, seeds)
    lab_d = torch.from_numpy(labels).to(DEV)
    sb = SampledBatch(smp, smp.counts(), lab_d, cfg.target_type)
    ref = oracle_sample(csc, g.rel_src, g.rel_dst, g.counts, seeds, cfg.target_type, fan, k)
    mb = MiniBatch(seeds=seeds, labels=labels,
                   layers=[LayerBlock(n_src=x["n_src"], n_dst=x["n_dst"], src_local=x["src_local"],
                                      dst_local=x["dst_local"], edge_id=x["edge_id"],
                                      src_global=x["src_gid"]) for x in ref])
    rs = g.rel_src
    rd = g.rel_dst
    params = make_params(cfg)
    feat_d = torch.from_numpy(feat).to(DEV)
    et_d = torch.from_numpy(g.edge_type).to(DEV)
    res = []
    for b in (sb, DeviceBatch(mb, rs, rd, foff, cfg.target_type, DEV)):
        tr = Trainer(cfg.num_types, cfg.num_rels, rs, rd, cfg.feat_dim, cfg.hidden, cfg.heads,
                     cfg.num_classes, cfg.num_layers, cfg.model, cfg.agg, DEV, lr=0.0)
        tr.load_params(params)
        loss = tr.step(b, feat_d, et_d, update=False)
        torch.cuda.synchronize()
        assert hf().read_status(tr.status) == 0
        res.append((float(loss.item()), tr.grads.cpu().numpy().copy()))
    assert res[0][0] == res[1][0]
    assert np.array_equal(res[0][1], res[1][1])


def test_sampler_graph_replay_with_device_key():
    """One captured graph, key and stamp in device memory (d_ctl): each replay
    equals the eager call with that key."""
    cfg, g, csc = setup("dblp")
    from paper_2408_08490_b200.sampler import GpuSampler
    fan = list(cfg.fanout)[::-1]
    seeds = torch.from_numpy(epoch_seeds(cfg, 0)[:300].astype(np.int32)).to(DEV)
    smp = GpuSampler(g.rel_src, g.rel_dst, g.counts, csc, fan, 300, DEV)
    ref = GpuSampler(g.rel_src, g.rel_dst, g.counts, csc, fan, 300, DEV)
    ctl = torch.zeros(2, dtype=torch.int64, device=DEV)
    ctl.copy_(torch.tensor([5, smp.next_stamp()]))
    smp.sample(seeds, cfg.target_type, 0, d_ctl=ctl)
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        smp.sample(seeds, cfg.target_type, 0, d_ctl=ctl)
    for key in (batch_key(0, 7), batch_key(2, 1), batch_key(0, 7)):
        k = key - (1 << 64) if key >= (1 << 63) else key
        ctl.copy_(torch.tensor([k, smp.next_stamp()]))
        gr.replay()
        ref.sample(seeds, cfg.target_type, key)
        torch.cuda.synchronize()
        for a, b, ca, cb in zip(smp.out, ref.out, smp.counts(), ref.counts()):
            assert np.array_equal(ca, cb)
            N = int(ca[-1])
            assert np.array_equal(a["eid"][:N].cpu().numpy(), b["eid"][:N].cpu().numpy())
            assert np.array_equal(a["src"][:N].cpu().numpy(), b["src"][:N].cpu().numpy())
