"""Aggregate ncu warp-stall samples per CUDA source line.
usage: ncu -i X.ncu-rep --page source --csv --print-source=cuda,sass > s.csv; python tools/ncu_lines.py s.csv [N]"""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
per, src, cur, tot = collections.Counter(), {}, None, 0.0
hdr = None
for r in rows:
    if len(r) > 4 and r[0] == "Line No":
        hdr = r
        i_s = r.index("Warp Stall Sampling (All Samples)")
        continue
    if hdr is None or len(r) <= 4:
        continue
    if r[0]:
        cur = int(r[0]); src[cur] = r[1]
    try:
        v = float(r[i_s] or 0)
    except ValueError:
        continue
    per[cur] += v; tot += v
for line, v in per.most_common(n):
    print(f"{v / tot * 100:5.1f}%  L{line:<5} {src.get(line, '').strip()[:110]}")
