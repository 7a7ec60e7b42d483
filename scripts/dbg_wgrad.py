import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
import oracle
from gpu_util import gpu_build, csr_host, t, DEV, hf
from synth import random_block, random_schema
rng = np.random.default_rng(5)
rs, rd = np.array([0], np.int32), np.array([0], np.int32)
blk, et = random_block(rng, [300], [100], rs, rd, 200)
sh, csr, st = gpu_build(blk, et, rs, rd)
ch = csr_host(sh, csr)
U = ch["U"]; K = D = 128
print("U", U, "rows", sh.rows)
Xl = (rng.integers(-2, 3, (sh.src_rows, K)) / 4).astype(np.float32)
W = (rng.integers(-2, 3, (1, K, D)) / 4).astype(np.float32)
dYn = (rng.integers(-2, 3, (U, D)) / 4).astype(np.float32)
Gn = np.zeros((sh.dst_rows, D), np.float32)
dW = torch.zeros(1, K, D, device=DEV)
dX = torch.zeros(sh.src_rows, K, device=DEV)
nb = hf().project_bwd_ws_bytes(sh, K, D, 1)
wsb = torch.zeros(nb // 4 + 16, device=DEV)
hf().project_bwd(sh, csr, K, D, 1, t(Xl), None, t(W), None, None, None, t(dYn), t(Gn), None, None,
                 dX, dW, None, None, wsb, prec=sys.argv[1] if len(sys.argv) > 1 else "tf32")
torch.cuda.synchronize()
ob = oracle.project_bwd(oracle.Shape.of(blk, rs, rd), ch, K, D, 1, Xl, None, W, None, None, None, dYn, Gn, None, None)
g = dW.cpu().numpy()[0]; r = ob["dW_rel"][0]
print("gpu", g[:3, :6]); print("ref", r[:3, :6])
ws = wsb.view(torch.int32).cpu().numpy()
print("tables", ws[:4], ws[64:68])
pf = wsb.cpu().numpy()[128:128 + 8]
print("partial head", pf)
print("match", np.array_equal(g, r.astype(np.float32)), np.abs(g - r).max())
eq = np.isclose(g, r)
print("rows ok", eq.all(1).sum(), "cols ok", eq.all(0).sum())
# check transposes / permutations
for name, cand in [("rT", r.T)]:
    print(name, np.allclose(g, cand))
print("dX match", np.array_equal(dX.cpu().numpy(), ob["dX"].astype(np.float32)))
