"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list:
kernel, launches, mean us, share.   python tools/launch_summary.py list.csv "header line" ..."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, agg = None, collections.defaultdict(list)
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0].replace("void ", "")
        v = float(d["Metric Value"].replace(",", ""))
        agg[name].append(v * {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}[d["Metric Unit"]])
tot = sum(sum(v) for v in agg.values())
lines = ["# " + h for h in sys.argv[2:]] + [f"{'kernel':44s} launches   mean_us  share"]
for name, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    lines.append(f"{name[:44]:44s} {len(v):8d} {sum(v) / len(v):9.1f} {100 * sum(v) / tot:5.1f}%")
print("\n".join(lines))
