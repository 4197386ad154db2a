"""Summarise scripts/ab_variants.sh output: python scripts/ab_report.py DIR [variants...]"""
import json
import os
import sys

d = sys.argv[1]
vs = sys.argv[2:] or sorted({f[4:-4] for f in os.listdir(d) if f.startswith("lat_")})
for v in vs:
    lat = ""
    if os.path.exists(f"{d}/lat_{v}.txt"):
        lat = " ".join(f"{ln.split()[1].rstrip(':')}:{ln.split()[2]}" for ln in open(f"{d}/lat_{v}.txt") if ln.startswith("n="))
    line = ""
    if os.path.exists(f"{d}/bench_{v}.json"):
        for ln in open(f"{d}/bench_{v}.json"):
            if ln.startswith('{"metric"'):
                j = json.loads(ln)
                r = j["roofline"]
                line = f"value {j['value'] / 1e6:.4f} M frac {r['frac']:.4f} steady {r['steady_frac']:.4f}"
    dec = ""
    if os.path.exists(f"{d}/bench_{v}.err"):
        dec = " ".join(ln.split(":", 1)[1].strip() for ln in open(f"{d}/bench_{v}.err") if ln.startswith("[timed] decode"))
    print(f"{v:10s} {lat}\n           {line}  decode ms {dec}")
