"""Padded-layout GPU-sampler calls for a few mag batches (ncu target)."""
import os
import sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from synth import CONFIGS, generate_graph, epoch_seeds, batch_key  # noqa: E402
from paper_2408_08490_b200.sampler import GpuSampler, padded_caps  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "mag"]
g = generate_graph(cfg)
smp = GpuSampler(g.rel_src, g.rel_dst, g.counts, g.in_csc(), list(cfg.fanout)[::-1],
                 cfg.batch_size, "cuda:0", nbuf=2)
perm = epoch_seeds(cfg, 0)
B = cfg.batch_size
seen = []
for b in range(4):
    s = torch.from_numpy(perm[b * B:(b + 1) * B].astype(np.int32)).cuda()
    smp.sample(s, cfg.target_type, batch_key(0, b), buf=0)
    seen.append(smp.counts(buf=0))
cap, pad = padded_caps(seen, cfg.num_types, cfg.target_type, B)
for b in range(3):
    s = torch.from_numpy(perm[b * B:(b + 1) * B].astype(np.int32)).cuda()
    smp.sample_padded(s, cfg.target_type, cap, pad, buf=1, key=batch_key(0, b))
torch.cuda.synchronize()
print([c.tolist() for c in smp.counts(buf=1)])
