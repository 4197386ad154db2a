"""Aggregate an ncu SASS source page (per-instruction warp-stall samples) by CUDA source line.
  ncu -i rep --page source --csv --print-source sass > src.csv
  cuobjdump -xelf all libbubblespec.so; nvdisasm -g -c verify.sm_100a.cubin > all.sass
  python scripts/ncu_lines.py src.csv all.sass <kernel-mangled-name> [top]
Prints the top source lines by stall samples with the dominant stall reasons."""
import csv
import re
import sys
from collections import defaultdict

src_csv, sass, kern = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
# address -> (file, line) from nvdisasm -g
amap = {}
cur = None
inside = False
for ln in open(sass):
    if ".text." in ln and "//---" in ln:
        inside = kern in ln
        continue
    if not inside:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        if "inlined at" not in ln:
            cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", ln)
    if m and cur:
        amap[int(m.group(1), 16)] = cur
rows = list(csv.reader(open(src_csv)))
hdr = rows[1]
ia = hdr.index("Address")
isrc = hdr.index("Source")
iall = hdr.index("Warp Stall Sampling (All Samples)")
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
agg = defaultdict(float)
reasons = defaultdict(lambda: defaultdict(float))
ops = defaultdict(lambda: defaultdict(float))
tot = 0.0
base = None
for r in rows[2:]:
    try:
        base = int(r[ia], 16)
        break
    except (ValueError, IndexError):
        continue
for r in rows[2:]:
    try:
        addr = int(r[ia], 16) - base
        v = float(r[iall] or 0)
    except (ValueError, IndexError):
        continue
    key = amap.get(addr, ("?", 0))
    agg[key] += v
    tot += v
    op = r[isrc].split()[0] if r[isrc].split() else "?"
    if op.startswith("@"):
        op = r[isrc].split()[1]
    ops[key][op.split(".")[0]] += v
    for i in stall_cols:
        try:
            reasons[key][hdr[i][6:]] += float(r[i] or 0)
        except ValueError:
            pass
print(f"total samples {tot:.0f}")
for key, v in sorted(agg.items(), key=lambda x: -x[1])[:top]:
    o = sorted(ops[key].items(), key=lambda x: -x[1])[:4]
    rs = sorted(reasons[key].items(), key=lambda x: -x[1])[:3]
    print(f"{100 * v / tot:5.1f}%  {key[0]}:{key[1]:<5d} ops: " + ", ".join(f"{a} {100 * b / max(v, 1):.0f}%" for a, b in o)
          + "  | " + ", ".join(f"{a} {100 * b / max(v, 1):.0f}%" for a, b in rs))
