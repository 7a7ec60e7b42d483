"""Per-kernel table from an `ncu --set full ... --page raw --csv` export:
duration, DRAM bytes and throughput, L2 hit rate and tensor-pipe activity
(sm__pipe_tensor_cycles_active*, the tcgen05 / mma pipe), one row per launch.

  python scripts/ncu_table.py raw.csv > table.md
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[0]
units = rows[1] if len(rows) > 1 else [""] * len(hdr)


def col(pred):
    for i, h in enumerate(hdr):
        if pred(h):
            return i
    return None


c_name = hdr.index("Kernel Name")
c_t = col(lambda h: h == "gpu__time_duration.sum")
c_rd = col(lambda h: h == "dram__bytes_read.sum")
c_wr = col(lambda h: h == "dram__bytes_write.sum")
c_dp = col(lambda h: h == "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed") or \
    col(lambda h: h == "dram__throughput.avg.pct_of_peak_sustained_elapsed")
c_l2 = col(lambda h: h == "lts__t_sector_hit_rate.pct")
c_tp = col(lambda h: h.startswith("sm__pipe_tensor_cycles_active") and "pct_of_peak_sustained_active" in h) \
    or col(lambda h: h.startswith("sm__pipe_tensor") and "pct" in h)


def num(r, c, scale_unit=None):
    if c is None:
        return None
    v = r[c].replace(",", "")
    try:
        x = float(v)
    except ValueError:
        return None
    u = units[c]
    if scale_unit == "bytes":
        x *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6}.get(u, 1)
    if scale_unit == "us":
        x *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1, "us": 1, "msecond": 1e3}.get(u, 1)
    return x


print(f"| # | kernel | us | DRAM MB | DRAM GB/s | DRAM % peak | L2 hit % | tensor pipe % ({hdr[c_tp] if c_tp is not None else 'n/a'}) |")
print("|---|---|---|---|---|---|---|---|")
for i, r in enumerate(rows[2:]):
    if len(r) != len(hdr):
        continue
    t = num(r, c_t, "us")
    b = (num(r, c_rd, "bytes") or 0) + (num(r, c_wr, "bytes") or 0)
    gbs = b / (t * 1e3) if t else 0
    tp = num(r, c_tp)
    print(f"| {i} | {r[c_name].split('(')[0][:40]} | {t:.2f} | {b / 1e6:.2f} | {gbs:.0f} | "
          f"{num(r, c_dp) or 0:.1f} | {num(r, c_l2) or 0:.1f} | {'' if tp is None else f'{tp:.1f}'} |")
