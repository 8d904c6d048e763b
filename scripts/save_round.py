"""Copy one profile_round.sh result set (gpurun_out/prof) into profiles/ under
a round prefix, summarise the ncu captures and record the per-launch DRAM
traffic of k_raster_fwd (bench.py reads profiles/traffic.json).

    python scripts/save_round.py r01
"""
import csv
import io
import json
import shutil
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
src = ROOT / "gpurun_out" / "prof"
dst = ROOT / "profiles"
tag = sys.argv[1]
table3 = {}
for f in sorted(src.glob("*.json")):
    txt = f.read_text().strip().splitlines()
    if not txt:
        continue
    if f.stem.startswith("t3_"):
        table3[f.stem] = json.loads(txt[-1])
    else:
        shutil.copy(f, dst / f"{tag}_{f.stem}.json")
if table3:
    (dst / f"{tag}_table3.json").write_text(json.dumps(table3, indent=1) + "\n")
shutil.copy(src / "launches.csv", dst / f"{tag}_launches.csv")
if (src / "train_launches.csv").exists():
    shutil.copy(src / "train_launches.csv", dst / f"{tag}_train_launches.csv")
subprocess.run([sys.executable, str(ROOT / "scripts" / "ncu_summary.py"), str(src / "launches.csv"),
                str(src / "full.ncu-rep"), str(dst / f"{tag}_ncu_summary.md")], check=True,
               stdout=subprocess.DEVNULL)
M = ("dram__bytes_read.sum,dram__bytes_write.sum,l1tex__throughput.avg.pct_of_peak_sustained_active,"
     "dram__cycles_active.avg.pct_of_peak_sustained_elapsed,"
     "l1tex__data_pipe_tex_wavefronts.avg.pct_of_peak_sustained_elapsed")
raw = subprocess.run(["ncu", "-i", str(src / "full.ncu-rep"), "--page", "raw", "--csv", "--metrics", M],
                     capture_output=True, text=True).stdout
rows = list(csv.DictReader(io.StringIO(raw)))
for r in rows[1:]:
    if "k_raster_fwd" in r["Kernel Name"]:
        mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        unit_r, unit_w = rows[0]["dram__bytes_read.sum"], rows[0]["dram__bytes_write.sum"]
        tb = (float(r["dram__bytes_read.sum"]) * mult[unit_r] +
              float(r["dram__bytes_write.sum"]) * mult[unit_w])
        out = {"cfg2/hw/rgba32f": int(tb),
               "ncu": {"kernel": "k_raster_fwd (cfg2, hw, rgba32f)",
                       "l1tex_throughput_pct": float(r["l1tex__throughput.avg.pct_of_peak_sustained_active"]),
                       "tex_data_pipe_pct": float(r["l1tex__data_pipe_tex_wavefronts.avg.pct_of_peak_sustained_elapsed"]),
                       "dram_throughput_pct": float(r["dram__cycles_active.avg.pct_of_peak_sustained_elapsed"])}}
        (dst / "traffic.json").write_text(json.dumps(out) + "\n")
        print("k_raster_fwd", out)
        break
