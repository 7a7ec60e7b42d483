"""Times hifuse_project / project_bwd alone on the mag layer-0 shapes (graph
replay, CUDA events).  Usage: python scripts/bench_project.py [config]."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from synth import CONFIGS, generate_graph, generate_features, make_params
from synth.sampler import make_batch
from paper_2408_08490_b200.step import Trainer, DeviceBatch
cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "mag"]
g = generate_graph(cfg); feat, foff = generate_features(cfg.type_counts, cfg.feat_dim)
rs = np.array([r.src for r in cfg.rels], np.int32); rd = np.array([r.dst for r in cfg.rels], np.int32)
dev = "cuda:0"
pool = [DeviceBatch(make_batch(cfg, g, b), rs, rd, foff, cfg.target_type, dev) for b in range(2)]
tr = Trainer(cfg.num_types, cfg.num_rels, rs, rd, cfg.feat_dim, cfg.hidden, cfg.heads,
             cfg.num_classes, cfg.num_layers, cfg.model, cfg.agg, dev, prec="tf32")
tr.load_params(make_params(cfg))
fd = torch.from_numpy(feat).to(dev); et = torch.from_numpy(g.edge_type).to(dev)
for db in pool: tr.step(db, fd, et, update=False)
torch.cuda.synchronize()
res = {}
for name, gr, _ in tr.capture_stages(pool[0], fd, et):
    if not name.startswith("project"): continue
    gr.replay(); torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20): gr.replay()
    b.record(); b.synchronize()
    res[name] = round(a.elapsed_time(b) / 20 * 1e3, 1)
print(os.environ.get("HIFUSE_TCP_VARIANT", "0"), res)
