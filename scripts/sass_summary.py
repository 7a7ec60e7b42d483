"""Per-kernel counts of the Blackwell-specific SASS instructions in
libhifuse.so (cuobjdump -sass): tcgen05 MMA (UTCHMMA / UTCQMMA), TMEM loads
(LDTM), tcgen05 barriers/commits (UTCBAR), TMA loads (UTMALDG), bulk copies,
warp-level mma.sync (HMMA) and the instruction total -- the evidence that the
projection contractions run on the 5th-gen tensor cores.

  python scripts/sass_summary.py paper_2408_08490_b200/libhifuse.so > profiles/r2/sass_summary.md
"""
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2408_08490_b200/libhifuse.so"
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
KEYS = ["UTCHMMA", "UTCQMMA", "UTCBAR", "LDTM", "UTMALDG", "UBLKCP", "HMMA", "LDGSTS"]
rows = []
name, cnt, tot = None, None, 0


def flush():
    if name and (any(cnt.values())):
        rows.append((name, dict(cnt), tot))


for line in out.split("\n"):
    m = re.match(r"\s+Function : (\S+)", line)
    if m:
        flush()
        name, cnt, tot = m.group(1), {k: 0 for k in KEYS}, 0
        continue
    if name and re.match(r"\s+/\*[0-9a-f]{4}\*/", line):
        tot += 1
        op = line.split("*/", 1)[1].strip().split()[0] if "*/" in line else ""
        if op.startswith("@"):
            op = line.split("*/", 1)[1].strip().split()[1]
        for k in KEYS:
            if op.startswith(k):
                cnt[k] += 1
flush()
demangle = subprocess.run(["c++filt"], input="\n".join(r[0] for r in rows), capture_output=True,
                          text=True).stdout.split("\n")
print("| kernel | " + " | ".join(KEYS) + " | SASS instructions |")
print("|---|" + "---|" * (len(KEYS) + 1))
for (n, c, t), d in zip(rows, demangle):
    d = d.replace("hf::", "").replace("(anonymous namespace)::", "")
    d = d.split("(")[0]
    print(f"| `{d}` | " + " | ".join(str(c[k]) for k in KEYS) + f" | {t} |")
