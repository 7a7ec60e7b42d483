"""-m gpu: NEXT(4) feature-sharded data parallelism (shard.py, shard.cu).

Two ranks on the box's GPU (gloo, buffers staged through host memory: NCCL
needs one GPU per rank) each hold HALF of the ogbn-mag-shaped feature store.
Every rank fetches the layer-0 rows of its own mini-batch through the
all-to-all exchange; the result must be BIT-IDENTICAL to the replicated
store's rows (pure data movement), and a training step fed with the fetched
rows must equal the replicated step bit for bit (same kernels, same values).
"""
import os

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from gpu_util import needs_gpu, DEV

pytestmark = [pytest.mark.gpu, needs_gpu]


def _worker(rank, world, port, key, outdir):
    import torch.distributed as dist
    from synth import CONFIGS, generate_graph, generate_features, make_batch, make_params
    from paper_2408_08490_b200.shard import FeatureShard, shard_bounds
    from paper_2408_08490_b200.step import Trainer, DeviceBatch
    from paper_2408_08490_b200 import hifuse as hf
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = CONFIGS[key]
    g = generate_graph(cfg)
    feat, foff = generate_features(cfg.type_counts, cfg.feat_dim)
    bounds = shard_bounds(feat.shape[0], world)
    local = torch.from_numpy(feat[bounds[rank]:bounds[rank + 1]]).to(DEV)
    shard = FeatureShard(local, bounds, rank, world, DEV, staging="host")
    mb = make_batch(cfg, g, rank)
    gid = mb.gather_ids(foff).astype(np.int32)
    X0 = shard.fetch(torch.from_numpy(gid).to(DEV))
    torch.cuda.synchronize()
    assert hf.read_status(shard.status) == 0
    np.save(os.path.join(outdir, f"x{rank}.npy"), X0.cpu().numpy())
    # one step fed by the fetched rows (layer 0 reads X0 directly)
    rs = np.array([r.src for r in cfg.rels], np.int32)
    rd = np.array([r.dst for r in cfg.rels], np.int32)
    tr = Trainer(cfg.num_types, cfg.num_rels, rs, rd, cfg.feat_dim, cfg.hidden, cfg.heads,
                 cfg.num_classes, cfg.num_layers, cfg.model, cfg.agg, DEV, lr=0.0, prec="tf32",
                 order="project_first")
    tr.load_params(make_params(cfg))
    db = DeviceBatch(mb, rs, rd, foff, cfg.target_type, DEV)
    db.dev["gid"] = None                          # X0 rows are the layer-0 sources, in order
    loss = tr.step(db, X0, torch.from_numpy(g.edge_type).to(DEV), update=False)
    torch.cuda.synchronize()
    np.save(os.path.join(outdir, f"l{rank}.npy"), np.array([loss.item()]))
    np.save(os.path.join(outdir, f"gr{rank}.npy"), tr.grads.cpu().numpy())
    dist.destroy_process_group()


def test_feature_shard_fetch_and_step(tmp_path):
    from synth import CONFIGS, generate_graph, generate_features, make_batch, make_params
    from paper_2408_08490_b200.step import Trainer, DeviceBatch
    key, world = "mag", 2
    port = 29500 + (os.getpid() % 2000) + 7
    mp.spawn(_worker, args=(world, port, key, str(tmp_path)), nprocs=world, join=True)
    cfg = CONFIGS[key]
    g = generate_graph(cfg)
    feat, foff = generate_features(cfg.type_counts, cfg.feat_dim)
    rs = np.array([r.src for r in cfg.rels], np.int32)
    rd = np.array([r.dst for r in cfg.rels], np.int32)
    feat_d = torch.from_numpy(feat).to(DEV)
    et_d = torch.from_numpy(g.edge_type).to(DEV)
    for r in range(world):
        mb = make_batch(cfg, g, r)
        gid = mb.gather_ids(foff)
        assert np.array_equal(np.load(tmp_path / f"x{r}.npy"), feat[gid]), f"rank {r} rows"
        tr = Trainer(cfg.num_types, cfg.num_rels, rs, rd, cfg.feat_dim, cfg.hidden, cfg.heads,
                     cfg.num_classes, cfg.num_layers, cfg.model, cfg.agg, DEV, lr=0.0,
                     prec="tf32", order="project_first")
        tr.load_params(make_params(cfg))
        db = DeviceBatch(mb, rs, rd, foff, cfg.target_type, DEV)
        loss = tr.step(db, feat_d, et_d, update=False)
        torch.cuda.synchronize()
        assert np.load(tmp_path / f"l{r}.npy")[0] == loss.item()
        assert np.array_equal(np.load(tmp_path / f"gr{r}.npy"), tr.grads.cpu().numpy())
