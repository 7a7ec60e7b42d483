"""Runs a few training steps of one configuration (for ncu / sanitizer runs)."""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from synth import CONFIGS, generate_graph, generate_features, make_params  # noqa: E402
from synth.sampler import make_batch  # noqa: E402
from paper_2408_08490_b200.step import Trainer, DeviceBatch  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="mag")
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--pool", type=int, default=2)
ap.add_argument("--prec", default="tf32")
ap.add_argument("--order", default="agg_first")
ap.add_argument("--feat-dtype", default="fp32")
a = ap.parse_args()
cfg = CONFIGS[a.config]
g = generate_graph(cfg)
feat, foff = generate_features(cfg.type_counts, cfg.feat_dim)
rs = np.array([r.src for r in cfg.rels], np.int32)
rd = np.array([r.dst for r in cfg.rels], np.int32)
nb = -(-cfg.type_counts[cfg.target_type] // cfg.batch_size)
dev = "cuda:0"
pool = [DeviceBatch(make_batch(cfg, g, b % nb, epoch=b // nb), rs, rd, foff, cfg.target_type, dev)
        for b in range(a.pool)]
tr = Trainer(cfg.num_types, cfg.num_rels, rs, rd, cfg.feat_dim, cfg.hidden, cfg.heads,
             cfg.num_classes, cfg.num_layers, cfg.model, cfg.agg, dev, lr=0.01, prec=a.prec,
             order=a.order, feat_dtype=a.feat_dtype)
tr.load_params(make_params(cfg))
fd = torch.from_numpy(feat).to(dev)
if a.feat_dtype == "bf16":
    fd = fd.to(torch.bfloat16)
et = torch.from_numpy(g.edge_type).to(dev)
tr.prepare_graph(et)
for db in pool:
    tr.step(db, fd, et, update=False)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
for i in range(a.steps):
    tr.step(pool[i % len(pool)], fd, et)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("loss", float(tr.loss.item()))
