"""Hot SASS lines (stall samples, executed instructions) per kernel from
`ncu -i R --page source --csv --print-source sass`. usage: sass_hot.py CSV [kernel-substr] [min%]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
want = sys.argv[2] if len(sys.argv) > 2 else ""
thr = float(sys.argv[3]) if len(sys.argv) > 3 else 1.5
blocks, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = [r[1], None, []]
        blocks.append(cur)
    elif r and r[0] == "Address":
        cur[1] = {k: j for j, k in enumerate(r)}
    elif cur and cur[1] and len(r) >= len(cur[1]):
        cur[2].append(r)
for name, idx, data in blocks:
    if want not in name:
        continue
    st = [float(r[idx["Warp Stall Sampling (All Samples)"]] or 0) for r in data]
    ie = [float(r[idx["Instructions Executed"]] or 0) for r in data]
    tot, ti = sum(st) or 1, sum(ie) or 1
    print(f"== {name}: {len(data)} SASS, {ti:.0f} warp inst, {tot:.0f} samples")
    for i, r in enumerate(data):
        if st[i] / tot * 100 >= thr or ie[i] / ti * 100 >= thr:
            print(f"{i:5d} stall {st[i] / tot * 100:5.1f}% inst {ie[i] / ti * 100:5.1f}%  {r[1].strip()[:90]}")
    break
