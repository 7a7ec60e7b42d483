"""Turns an ncu --set full raw CSV (one step) into profiles/traffic.json:
{kernel base name: [dram read+write bytes per launch, in launch order]}."""
import csv
import json
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[0]
units = rows[1]
ki, rd, wr = h.index("Kernel Name"), h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum")
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
out = {}
for r in rows[2:]:
    name = r[ki].split("(")[0].replace("void ", "").split("<")[0].strip().replace("hf::", "")
    b = float(r[rd].replace(",", "")) * scale[units[rd]] + float(r[wr].replace(",", "")) * scale[units[wr]]
    out.setdefault(name, []).append(b)
cfg = sys.argv[3] if len(sys.argv) > 3 else "mag"
order = sys.argv[4] if len(sys.argv) > 4 else "agg_first"
json.dump({"config": cfg, "order": order, "source": sys.argv[1], "kernels": out},
          open(sys.argv[2], "w"), indent=1)
print({k: [round(x / 1e6, 2) for x in v] for k, v in out.items()})
