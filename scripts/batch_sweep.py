"""Supplementary batch sweep: ogbn-mag-shaped workload at
1024 ... 16384 seeds per mini-batch, both layer-0 orders, to show the merged
aggregation's asymptotic HBM fraction once a layer's bytes dwarf launch and
tail costs.  Per batch size: whole-step time (serial CUDA graph replay) and,
per aggregation call, device time and algorithmic GB/s (bench.stage_cost,
SURVEY.md §8(d) byte model) against the measured HBM peak.

  python scripts/batch_sweep.py [--batches 1024 2048 4096 8192 16384] > out.jsonl
"""
import argparse
import dataclasses
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402  (stage_cost, layer_sizes, peaks)
from synth import CONFIGS, generate_graph, generate_features, make_batch, make_params  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batches", type=int, nargs="+", default=[1024, 2048, 4096, 8192, 16384])
    ap.add_argument("--config", default="mag")
    ap.add_argument("--pool", type=int, default=2)
    ap.add_argument("--steps", type=int, default=20)
    args = ap.parse_args()
    import torch
    from paper_2408_08490_b200.step import Trainer, DeviceBatch
    dev = "cuda:0"
    base = CONFIGS[args.config]
    g = generate_graph(base)
    feat, foff = generate_features(base.type_counts, base.feat_dim)
    params = make_params(base)
    rs = np.array([r.src for r in base.rels], np.int32)
    rd = np.array([r.dst for r in base.rels], np.int32)
    feat_d = torch.from_numpy(feat).to(dev)
    et_d = torch.from_numpy(g.edge_type).to(dev)
    pk = bench.peaks()
    for B in args.batches:
        cfg = dataclasses.replace(base, batch_size=B)
        mbs = [make_batch(cfg, g, b) for b in range(args.pool)]
        sizes = [bench.layer_sizes(cfg, g, mb, rs, rd) for mb in mbs]
        pool = [DeviceBatch(mb, rs, rd, foff, cfg.target_type, dev) for mb in mbs]
        for i, db in enumerate(pool):
            db.slot = i
        for order in ("agg_first", "project_first"):
            tr = Trainer(cfg.num_types, cfg.num_rels, rs, rd, cfg.feat_dim, cfg.hidden, cfg.heads,
                         cfg.num_classes, cfg.num_layers, cfg.model, cfg.agg, dev, lr=0.0,
                         order=order)
            tr.load_params(params)
            tr.prepare_graph(et_d)
            for db in pool:
                tr.step(db, feat_d, et_d, update=False)
            torch.cuda.synchronize()
            graphs = [tr.capture(db, feat_d, et_d, update=True) for db in pool]
            for i in range(4):
                graphs[i % len(pool)][0].replay()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record()
            for i in range(args.steps):
                graphs[i % len(pool)][0].replay()
            b.record()
            b.synchronize()
            step_ms = a.elapsed_time(b) / args.steps
            agg = {}
            for pi, db in enumerate(pool):
                for name, g_, _ in tr.capture_stages(db, feat_d, et_d):
                    nm, _, ll = name.partition(".")
                    if nm not in ("aggregate_fwd", "aggregate_features", "aggregate_bwd"):
                        continue
                    g_.replay()
                    e0 = torch.cuda.Event(enable_timing=True)
                    e1 = torch.cuda.Event(enable_timing=True)
                    e0.record()
                    for _ in range(5):
                        g_.replay()
                    e1.record()
                    e1.synchronize()
                    us = e0.elapsed_time(e1) / 5 * 1e3
                    l = int(ll)
                    byt = bench.stage_cost(nm, l, cfg, sizes[pi])[0]
                    agg.setdefault(name, []).append((us, byt))
            rec = {"config": args.config, "batch": B, "order": order, "ms_per_step": step_ms,
                   "mini_batches_per_s": 1e3 / step_ms,
                   "edges": [s["N"] for s in sizes[0]], "hbm_peak_gbs": pk["hbm"]}
            for name, v in sorted(agg.items()):
                us = float(np.mean([x for x, _ in v]))
                byt = float(np.mean([y for _, y in v]))
                rec[name] = {"us": round(us, 2), "MB": round(byt / 1e6, 2),
                             "GB/s": round(byt / us / 1e3, 1),
                             "frac_of_hbm": round(byt / us / 1e3 / pk["hbm"], 3)}
            print(json.dumps(rec), flush=True)
            del graphs, tr
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
