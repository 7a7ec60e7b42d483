"""Per-node cost of tiny kernels inside a CUDA graph on this GPU (context for
the latency-bound build / head kernels)."""
import torch
x = torch.zeros(1, device="cuda")
y = torch.zeros(1 << 20, device="cuda")
for name, fn, n in (("fill_1elem", lambda: x.fill_(1.0), 200),
                    ("add_1M", lambda: y.add_(1.0), 200)):
    g = torch.cuda.CUDAGraph()
    fn()
    torch.cuda.synchronize()
    with torch.cuda.graph(g):
        for _ in range(n):
            fn()
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        g.replay()
    b.record()
    b.synchronize()
    print(f"{name}: {a.elapsed_time(b) / 10 / n * 1e3:.2f} us per graph node")
