"""-m gpu: the bench's supplementary legs run on the Trainer's own state --
the merged-vs-unmerged comparison after an aggregate-first step (whose input
layer is built in X-row mode) and the default bench line end to end on a
small config."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

from synth import CONFIGS, generate_graph, generate_features, make_batch, make_params

from gpu_util import needs_gpu, DEV

pytestmark = [pytest.mark.gpu, needs_gpu]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("key,order", [("dblp", "agg_first"), ("imdb", "project_first")])
def test_compare_layers_after_step(key, order):
    from paper_2408_08490_b200 import hifuse as hf
    from paper_2408_08490_b200.step import Trainer, DeviceBatch
    from comparison.unmerged import compare_layers
    cfg = CONFIGS[key]
    g = generate_graph(cfg)
    feat, foff = generate_features(cfg.type_counts, cfg.feat_dim)
    rs = np.array([r.src for r in cfg.rels], np.int32)
    rd = np.array([r.dst for r in cfg.rels], np.int32)
    params = make_params(cfg)
    tr = Trainer(cfg.num_types, cfg.num_rels, rs, rd, cfg.feat_dim, cfg.hidden, cfg.heads,
                 cfg.num_classes, cfg.num_layers, cfg.model, cfg.agg, DEV, lr=0.0, prec="tf32",
                 order=order)
    tr.load_params(params)
    et_d = torch.from_numpy(g.edge_type).to(DEV)
    tr.prepare_graph(et_d)
    db = DeviceBatch(make_batch(cfg, g, 0), rs, rd, foff, cfg.target_type, DEV)
    feat_d = torch.from_numpy(feat).to(DEV)
    out = compare_layers(hf, tr, db, cfg, feat_d, et_d, params, {})
    torch.cuda.synchronize()
    assert hf.read_status(tr.status) == 0
    for rec in out["layers"]:
        assert rec["per_relation_equals_merged"], rec
        if "cusparse_max_abs_diff" in rec:
            assert rec["cusparse_max_abs_diff"] < 1e-3


def test_default_bench_line_small():
    """`bench.py --config dblp` with every default leg (comparison, GPU
    sampler, CPU baseline) prints one valid JSON line."""
    r = subprocess.run([sys.executable, "bench.py", "--config", "dblp", "--steps", "20",
                        "--warmup", "3", "--repeats", "1"], cwd=ROOT, capture_output=True,
                       text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["value"] > 0 and line["gpu_launches"] > 0
    assert "error" not in (line.get("merged_vs_unmerged") or {})
    assert "error" not in (line.get("gpu_sampler") or {})
