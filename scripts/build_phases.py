"""CUDA-event time of the semantic-graph build call (all layers of a
config's first batch; per-kernel times: run it under ncu)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from synth import CONFIGS, generate_graph, make_batch
from paper_2408_08490_b200 import hifuse as hf

key = sys.argv[1] if len(sys.argv) > 1 else "mag"
csc0 = (sys.argv[2] if len(sys.argv) > 2 else "1") == "1"
cfg = CONFIGS[key]
g = generate_graph(cfg)
mb = make_batch(cfg, g, 0)
rs = np.array([r.src for r in cfg.rels], np.int32)
rd = np.array([r.dst for r in cfg.rels], np.int32)
dev = "cuda:0"
shapes = [hf.Shape(rs, rd, b.n_src, b.n_dst, b.num_edges) for b in mb.layers]
csrs = [hf.CsrBuffers(s, dev, csc=(l > 0 or csc0)) for l, s in enumerate(shapes)]
t = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a, dt)).to(dev)
src = [t(b.src_local, np.int32) for b in mb.layers]
dst = [t(b.dst_local, np.int32) for b in mb.layers]
eid = [t(b.edge_id, np.int64) for b in mb.layers]
et = t(g.edge_type, np.int32)
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
print(f"{key}: build {a.elapsed_time(b) / 20 * 1e3:.1f} us per call (eager, 20 calls)")
print("status", hf.read_status(st))
