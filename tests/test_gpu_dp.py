"""-m gpu: data parallelism with the REAL Trainer.

Two ranks (processes) on the box's GPU, gloo process group over CUDA tensors
(NCCL needs one GPU per rank; the collective is the same all-reduce): each
rank takes its own mini-batch (dp.rank_batches), runs one Trainer.step with
the bucketed per-layer all-reduce (Trainer.set_dp) and the 1/W-scaled SGD.
Both ranks must end with parameters BIT-IDENTICAL to a single process that
computes the two batches' gradients, sums them and applies the same SGD
kernel with scale 1/2 (a sum of two fp32 values is order-independent)."""
import os

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from gpu_util import needs_gpu, DEV

pytestmark = [pytest.mark.gpu, needs_gpu]


def _setup(key):
    from synth import CONFIGS, generate_graph, generate_features, make_params
    cfg = CONFIGS[key]
    g = generate_graph(cfg)
    feat, foff = generate_features(cfg.type_counts, cfg.feat_dim)
    rs = np.array([r.src for r in cfg.rels], np.int32)
    rd = np.array([r.dst for r in cfg.rels], np.int32)
    return cfg, g, feat, foff, rs, rd, make_params(cfg)


def _trainer(cfg, rs, rd, params, prec):
    from paper_2408_08490_b200.step import Trainer
    tr = Trainer(cfg.num_types, cfg.num_rels, rs, rd, cfg.feat_dim, cfg.hidden, cfg.heads,
                 cfg.num_classes, cfg.num_layers, cfg.model, cfg.agg, DEV, lr=0.05, prec=prec)
    tr.load_params(params)
    return tr


def _worker(rank, world, port, key, prec, outdir):
    import torch.distributed as dist
    from synth import make_batch
    from paper_2408_08490_b200.step import DeviceBatch
    from paper_2408_08490_b200.dp import rank_batches
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg, g, feat, foff, rs, rd, params = _setup(key)
    tr = _trainer(cfg, rs, rd, params, prec)
    tr.set_dp(world)
    b = rank_batches(rank, world, 1)[0]
    db = DeviceBatch(make_batch(cfg, g, b), rs, rd, foff, cfg.target_type, DEV)
    tr.step(db, torch.from_numpy(feat).to(DEV), torch.from_numpy(g.edge_type).to(DEV))
    torch.cuda.synchronize()
    np.save(os.path.join(outdir, f"p{rank}.npy"), tr.params.cpu().numpy())
    np.save(os.path.join(outdir, f"g{rank}.npy"), tr.grads.cpu().numpy())
    dist.destroy_process_group()


@pytest.mark.parametrize("key,prec", [("dblp", "fp32"), ("imdb", "tf32")])
def test_dp_trainer_matches_single_process(key, prec, tmp_path):
    from synth import make_batch
    from paper_2408_08490_b200 import hifuse as hf
    from paper_2408_08490_b200.step import DeviceBatch
    world, port = 2, 29500 + (os.getpid() % 2000)
    mp.spawn(_worker, args=(world, port, key, prec, str(tmp_path)), nprocs=world, join=True)
    cfg, g, feat, foff, rs, rd, params = _setup(key)
    feat_d = torch.from_numpy(feat).to(DEV)
    et_d = torch.from_numpy(g.edge_type).to(DEV)
    grads = []
    for b in range(world):                       # rank b's batch: global batch index b
        tr = _trainer(cfg, rs, rd, params, prec)
        db = DeviceBatch(make_batch(cfg, g, b), rs, rd, foff, cfg.target_type, DEV)
        tr.step(db, feat_d, et_d, update=False)
        grads.append(tr.grads.clone())
    torch.cuda.synchronize()
    summed = grads[0] + grads[1]
    tr = _trainer(cfg, rs, rd, params, prec)
    p_ref = tr.params.clone()
    hf.sgd(p_ref, summed, 0.05, 1.0 / world)
    torch.cuda.synchronize()
    for r in range(world):
        g_r = np.load(tmp_path / f"g{r}.npy")
        p_r = np.load(tmp_path / f"p{r}.npy")
        assert np.array_equal(g_r, summed.cpu().numpy()), f"rank {r}: all-reduced gradients"
        assert np.array_equal(p_r, p_ref.cpu().numpy()), f"rank {r}: parameters after SGD"
