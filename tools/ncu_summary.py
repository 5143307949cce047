"""One line per captured kernel from an ncu report: duration, DRAM bytes, L2
(lts) sector traffic, achieved occupancy, top stall.  usage:
python tools/ncu_summary.py report.ncu-rep"""
import csv
import io
import subprocess
import sys

raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]


def col(name):
    return hdr.index(name) if name in hdr else None


keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
        "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct", "dram__throughput.avg.pct_of_peak_sustained_elapsed"]
stall = [h for h in hdr if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio")]
print("| kernel | " + " | ".join(k.split(".")[0].replace("__", ".") for k in keys) + " | top stall |")
print("|" + "---|" * (len(keys) + 2))
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")][:48]
    vals = []
    for k in keys:
        i = col(k)
        vals.append(f"{r[i]} {units[i]}" if i is not None else "-")
    st = max(stall, key=lambda h: float(r[hdr.index(h)] or 0))
    print(f"| `{name}` | " + " | ".join(vals) + f" | {st.split('stalled_')[1].split('_per')[0]} {float(r[hdr.index(st)]):.1f} |")
