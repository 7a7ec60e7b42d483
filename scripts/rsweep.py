"""Supplementary R-sweep: Freebase-shaped graphs with the
same total edge count and R relations; per R: merged step time (CUDA graph
replay), kernels per step, and per layer the merged-vs-unmerged arms of
comparison/unmerged.py (kernels per layer, same kernel launched per relation,
torch per-relation ops).  Shows "one aggregation kernel per layer regardless
of relation count" (north_star).

  python scripts/rsweep.py [--rels 10 18 36 72 144] [--model rgat|rgcn] > out.jsonl
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from synth import generate_graph, generate_features, make_batch, make_params  # noqa: E402
from synth.configs import freebase_sweep  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rels", type=int, nargs="+", default=[10, 18, 36, 72, 144])
    ap.add_argument("--model", default="rgat", choices=["rgat", "rgcn"])
    ap.add_argument("--pool", type=int, default=4)
    ap.add_argument("--steps", type=int, default=100)
    args = ap.parse_args()
    import torch
    from paper_2408_08490_b200 import hifuse as hf
    from paper_2408_08490_b200.step import Trainer, DeviceBatch
    from comparison.unmerged import compare_layers
    dev = "cuda:0"
    for R in args.rels:
        cfg = freebase_sweep(R, args.model)
        g = generate_graph(cfg)
        feat, foff = generate_features(cfg.type_counts, cfg.feat_dim)
        params = make_params(cfg)
        rs = np.array([r.src for r in cfg.rels], np.int32)
        rd = np.array([r.dst for r in cfg.rels], np.int32)
        pool = [DeviceBatch(make_batch(cfg, g, b), rs, rd, foff, cfg.target_type, dev)
                for b in range(args.pool)]
        for i, db in enumerate(pool):
            db.slot = i
        feat_d = torch.from_numpy(feat).to(dev)
        et_d = torch.from_numpy(g.edge_type).to(dev)
        tr = Trainer(cfg.num_types, cfg.num_rels, rs, rd, cfg.feat_dim, cfg.hidden, cfg.heads,
                     cfg.num_classes, cfg.num_layers, cfg.model, cfg.agg, dev, lr=0.0,
                     order="agg_first")
        tr.load_params(params)
        tr.prepare_graph(et_d)
        for db in pool:
            tr.step(db, feat_d, et_d, update=False)
        torch.cuda.synchronize()
        graphs = [tr.capture(db, feat_d, et_d, update=True) for db in pool]
        for i in range(10):
            graphs[i % len(pool)][0].replay()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        for i in range(args.steps):
            graphs[i % len(pool)][0].replay()
        b.record()
        b.synchronize()
        ms = a.elapsed_time(b) / args.steps
        stages = tr.capture_stages(pool[0], feat_d, et_d)
        sk = {}
        for name, g_, nk in stages:
            g_.replay()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(5):
                g_.replay()
            e1.record()
            e1.synchronize()
            sk[name] = (e0.elapsed_time(e1) / 5, nk)
        tr.load_params(params)
        cmp = compare_layers(hf, tr, pool[0], cfg, feat_d, et_d, params, sk)
        line = {"config": cfg.key, "relations": R, "model": cfg.model,
                "ms_per_step_serial_graph": ms, "mini_batches_per_s": 1e3 / ms,
                "kernels_per_step": graphs[0][1], "build_kernels": sk["build"][1],
                "build_us": round(sk["build"][0] * 1e3, 2), "layers": cmp["layers"]}
        print(json.dumps(line), flush=True)
        del graphs, stages, tr


if __name__ == "__main__":
    main()
