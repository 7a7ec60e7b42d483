"""Per-kernel device times of the LAST step in an ncu --cache-control none
launch list (warm L2, serialised kernels)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = None
out = []
for r in rows:
    if r and r[0] == "ID":
        h = r
        continue
    if h and len(r) == len(h) and r[h.index("Metric Name")] == "gpu__time_duration.sum":
        out.append((r[h.index("Kernel Name")].split("(")[0][:44], float(r[h.index("Metric Value")])))
idx = [i for i, (k, _) in enumerate(out) if "k_classify" in k]
start = idx[-2] if len(idx) >= 2 else 0
tot = 0.0
for k, v in out[start:]:
    tot += v
    print(f"{k:46s} {v / 1e3:8.2f} us")
print(f"total {tot / 1e3:.1f} us")
