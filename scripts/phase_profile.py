"""Per-phase instruction / stall shares of k_raster_fwd from an ncu source
export (`ncu -i R --page source --csv --print-source cuda,sass > S.csv`).
Phases are delimited by the `// ---- <name>` markers in tsb_forward.cu;
inlined tsb_math.h lines are attributed to the calling phase by the SASS
order (the last tsb_forward.cu phase seen)."""
import csv
import re
import sys
from collections import defaultdict

src = open("paper_2506_13348_b200/csrc/tsb_forward.cu").read().splitlines()
k0 = next(i for i, l in enumerate(src) if "k_raster_fwd(RasterParams p) {" in l)
marks = [(i + 1, m.group(1)) for i, l in enumerate(src)
         if i > k0 and (m := re.search(r"// ---- (\w+)", l))]


def phase_of(ln):
    name = "setup"
    for start, nm in marks:
        if ln >= start:
            name = nm
    return name


rows = list(csv.reader(open(sys.argv[1])))
cur, hdr = None, None
agg = defaultdict(lambda: [0, 0])
last = "setup"
for r in rows:
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[0].isdigit():
        try:
            s, i = int(r[4] or 0), int(r[7] or 0)
        except ValueError:
            continue
        ln = int(r[0])
        if cur == "tsb_forward.cu" and ln > k0:
            last = phase_of(ln)
            ph = last
        elif cur == "tsb_forward.cu":
            ph = "helpers(issue/finish)"
        else:
            ph = f"{last}:inlined"
        agg[ph][0] += s
        agg[ph][1] += i
ts = sum(v[0] for v in agg.values())
ti = sum(v[1] for v in agg.values())
for ph, (s, i) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{ph:28s} inst {100 * i / ti:5.1f}%  stall-samples {100 * s / ts:5.1f}%")
print(f"total inst {ti}")
