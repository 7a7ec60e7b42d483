"""Times hifuse_linear_xent alone (CUDA events) for a given B, D, C."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2408_08490_b200 import hifuse as hf

B, D, C = (int(a) for a in (sys.argv[1:4] if len(sys.argv) > 3 else (1024, 128, 349)))
dev = "cuda:0"
H = torch.randn(B + 100, D, device=dev)
lab = torch.randint(0, C, (B,), dtype=torch.int32, device=dev)
Wc = torch.randn(D, C, device=dev) * 0.1
bc = torch.zeros(C, device=dev)
loss = torch.zeros(1, device=dev)
dH = torch.empty_like(H)
dWc = torch.empty_like(Wc)
dbc = torch.empty_like(bc)
ws = torch.empty(hf.xent_ws_bytes(B, D, C) // 4 + 64, device=dev)
f = lambda: hf.linear_xent(B, D, C, H, 50, lab, Wc, bc, loss, dH, dWc, dbc, ws)
for _ in range(3):
    f()
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    f()
g.replay()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(50):
    g.replay()
b.record()
b.synchronize()
print(f"B={B} D={D} C={C}: {a.elapsed_time(b) / 50 * 1e3:.1f} us per call (graph replay, warm)")
# check against torch
Hs = H[50:50 + B]
lg = Hs @ Wc + bc
ref = torch.nn.functional.cross_entropy(lg, lab.long())
p = torch.softmax(lg, 1)
p[torch.arange(B), lab.long()] -= 1
p /= B
print("loss err", abs(loss.item() - ref.item()), "dWc err", (dWc - Hs.T @ p).abs().max().item(),
      "dH err", (dH[50:50 + B] - p @ Wc.T).abs().max().item())
