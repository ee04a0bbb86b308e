"""Aggregate ncu warp-stall samples per source line / enclosing function.

    ncu -i rep --page source --csv --print-source cuda,sass > mix.csv
    python tools/ncu_lines.py mix.csv [top]
"""
import csv
import re
import sys
from collections import defaultdict

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
cur_file = None
line_samples = defaultdict(int)
line_src = {}
with open(path, newline="") as f:
    for row in csv.reader(f):
        if not row:
            continue
        if row[0] == "File Path":
            cur_file = row[1]
            continue
        if row[0] in ("Function Name", "Line No") or cur_file is None or len(row) < 5:
            continue
        if row[2] != "-":
            continue
        try:
            s = int(row[4])
        except ValueError:
            continue
        key = (cur_file, int(row[0]))
        line_samples[key] += s
        line_src[key] = row[1]
total = sum(line_samples.values())
func_re = re.compile(r"^\s*(template\s*<.*>\s*)?(__device__|__global__|static|inline|__forceinline__).*?\b(\w+)\s*\(")
funcs = {}
for fpath in {k[0] for k in line_samples}:
    try:
        lines = open(fpath).read().split("\n")
    except OSError:
        continue
    cur = "?"
    for i, ln in enumerate(lines, 1):
        m = func_re.match(ln)
        if m and not ln.rstrip().endswith(";"):
            cur = m.group(3)
        funcs[(fpath, i)] = cur
per_func = defaultdict(int)
for k, s in line_samples.items():
    per_func[(k[0].split("/")[-1], funcs.get(k, "?"))] += s
print(f"total samples {total}")
for (fn, fun), s in sorted(per_func.items(), key=lambda x: -x[1])[:25]:
    print(f"{100.0 * s / total:6.2f}%  {fn}:{fun}")
print()
for k, s in sorted(line_samples.items(), key=lambda x: -x[1])[:top]:
    print(f"{100.0 * s / total:6.2f}%  {k[0].split('/')[-1]}:{k[1]}  {line_src[k].strip()[:90]}")
