"""Host-side cost of one eager training step (Python + ctypes launch path):
cProfile over 50 eager steps of the bench config (GPU-sampled batches need
eager steps because their shapes change per batch)."""
import cProfile
import os
import pstats
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from synth import CONFIGS, generate_graph, generate_features, make_batch, make_params  # noqa: E402
from paper_2408_08490_b200.step import Trainer, DeviceBatch  # noqa: E402

key = sys.argv[1] if len(sys.argv) > 1 else "mag"
cfg = CONFIGS[key]
g = generate_graph(cfg)
feat, foff = generate_features(cfg.type_counts, cfg.feat_dim)
rs = np.array([r.src for r in cfg.rels], np.int32)
rd = np.array([r.dst for r in cfg.rels], np.int32)
dev = "cuda:0"
db = DeviceBatch(make_batch(cfg, g, 0), rs, rd, foff, cfg.target_type, dev)
tr = Trainer(cfg.num_types, cfg.num_rels, rs, rd, cfg.feat_dim, cfg.hidden, cfg.heads,
             cfg.num_classes, cfg.num_layers, cfg.model, cfg.agg, dev, order="agg_first")
tr.load_params(make_params(cfg))
feat_d = torch.from_numpy(feat).to(dev)
et_d = torch.from_numpy(g.edge_type).to(dev)
for _ in range(5):
    tr.step(db, feat_d, et_d)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(50):
    tr.step(db, feat_d, et_d)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"{key}: host enqueue {1e6 * (t1 - t0) / 50:.1f} us/step, wall incl. drain "
      f"{1e6 * (t2 - t0) / 50:.1f} us/step")
pr = cProfile.Profile()
pr.enable()
for _ in range(50):
    tr.step(db, feat_d, et_d)
pr.disable()
torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
