"""Summarize an ncu launch list (--metrics gpu__time_duration.sum --csv) into
per-kernel counts, total time and share (cold-cache, serialised by ncu: compare
SHARES, not absolutes).  usage: python tools/summarize_launches.py launches.csv > summary.md"""
import collections
import csv
import re
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if r]
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ik, im, iv = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
tot = collections.Counter()
cnt = collections.Counter()
for r in rows[hdr + 1:]:
    if len(r) <= iv or r[im] != "gpu__time_duration.sum":
        continue
    name = re.sub(r"\(.*", "", r[ik]).replace("void ", "").replace("rmg::<unnamed>::", "")
    name = re.sub(r"<.*>", lambda m: m.group(0)[:60], name)
    v = float(r[iv].replace(",", ""))
    tot[name] += v
    cnt[name] += 1
all_ns = sum(tot.values())
print(f"| kernel | launches | total ms | share |\n|---|---|---|---|")
for k, v in tot.most_common():
    print(f"| `{k}` | {cnt[k]} | {v / 1e6:.3f} | {v / all_ns * 100:.1f}% |")
print(f"\n{sum(cnt.values())} launches, {all_ns / 1e6:.2f} ms total (ncu-serialised)")
