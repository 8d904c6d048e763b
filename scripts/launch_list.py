"""Print the per-kernel launch times of the last frame from an ncu launch
list (`ncu --metrics gpu__time_duration.sum --csv --log-file F ...`).
usage: python scripts/launch_list.py F [first-kernel-substring]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
first = sys.argv[2] if len(sys.argv) > 2 else "k_preprocess"
hdr, out = None, []
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d["Metric Name"] == "gpu__time_duration.sum":
            out.append((d["Kernel Name"][:64], float(d["Metric Value"])))
idx = [i for i, o in enumerate(out) if first in o[0]]
frame = out[idx[-1]:] if idx else out
for name, ns in frame:
    print(f"{ns / 1000:9.2f} us  {name}")
print(f"{sum(ns for _, ns in frame) / 1000:9.2f} us  total")
