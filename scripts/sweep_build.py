"""Times the A1 build call for every libhifuse.so variant under scratch/v_*
(scripts/build_variants.sh) in ONE process per config, and checks that every
variant's CSR/CSC outputs equal the first variant's bit for bit.
usage: python scripts/sweep_build.py mag:0 imdb:1 ...   (config:csc_on_layer0)"""
import glob
import os
import shutil
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from synth import CONFIGS, generate_graph, make_batch
from paper_2408_08490_b200 import hifuse as hf

variants = sorted(glob.glob("scratch/v_*/libhifuse.so"))
dev = "cuda:0"
for arg in sys.argv[1:]:
    key, csc0 = arg.split(":")
    cfg = CONFIGS[key]
    g = generate_graph(cfg)
    mbs = [make_batch(cfg, g, b) for b in range(2)]
    rs = np.array([r.src for r in cfg.rels], np.int32)
    rd = np.array([r.dst for r in cfg.rels], np.int32)
    t = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a, dt)).to(dev)
    et = t(g.edge_type, np.int32)
    ref = None
    for vp in variants:
        name = vp.split("/")[-2]
        cp = f"/tmp/lib_{name}.so"
        shutil.copy(vp, cp)
        hf._lib = None
        hf.LIB_PATH = cp
        outs, times = [], []
        for mb in mbs:
            shapes = [hf.Shape(rs, rd, b.n_src, b.n_dst, b.num_edges) for b in mb.layers]
            csrs = [hf.CsrBuffers(s, dev, csc=(l > 0 or csc0 == "1")) for l, s in enumerate(shapes)]
            for c in csrs:
                for v in c.t.values():
                    if v is not None:
                        v.fill_(-7)
            src = [t(b.src_local, np.int32) for b in mb.layers]
            dst = [t(b.dst_local, np.int32) for b in mb.layers]
            eid = [t(b.edge_id, np.int64) for b in mb.layers]
            off = torch.empty(len(rs) + 1, dtype=torch.int64, device=dev)
            st = torch.zeros(1, dtype=torch.int32, device=dev)
            hf.edge_type_offsets(et, len(rs), off, st)
            ws = torch.empty(sum(s.build_ws for s in shapes) // 4 + 64, dtype=torch.int32, device=dev)
            run = lambda: hf.build_semantic_graphs(shapes, csrs, src, dst, eid, et, ws, st, rel_edge_off=off)
            for _ in range(3):
                run()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(20):
                run()
            b.record()
            b.synchronize()
            times.append(a.elapsed_time(b) / 20 * 1e3)
            assert hf.read_status(st) == 0
            outs.append([{k: v.cpu().clone() for k, v in c.t.items() if v is not None} for c in csrs])
        same = "ref"
        if ref is None:
            ref = outs
        else:
            same = all(all(torch.equal(o[k], r[k]) for k in r) for ob, rb in zip(outs, ref)
                       for o, r in zip(ob, rb))
        print(f"{key} csc0={csc0} {name}: build {np.mean(times):.1f} us per call "
              f"(batches {', '.join(f'{x:.1f}' for x in times)}) identical={same}", flush=True)
