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
for name in ("launches", "launches_cfg5", "train_launches"):
    if (src / f"{name}.csv").exists():
        shutil.copy(src / f"{name}.csv", dst / f"{tag}_{name}.csv")
summ = [("launches", "full", "ncu_summary"), ("launches_cfg5", "full_cfg5", "ncu_summary_cfg5"),
        ("train_launches", "full_bwd", "ncu_summary_train")]
for lname, rname, oname in summ:
    if (src / f"{lname}.csv").exists() and (src / f"{rname}.ncu-rep").exists():
        subprocess.run([sys.executable, str(ROOT / "scripts" / "ncu_summary.py"),
                        str(src / f"{lname}.csv"), str(src / f"{rname}.ncu-rep"),
                        str(dst / f"{tag}_{oname}.md")], check=True, stdout=subprocess.DEVNULL)
M = ("dram__bytes_read.sum,dram__bytes_write.sum,l1tex__throughput.avg.pct_of_peak_sustained_active,"
     "dram__cycles_active.avg.pct_of_peak_sustained_elapsed,"
     "l1tex__data_pipe_tex_wavefronts.avg.pct_of_peak_sustained_elapsed,gpu__time_duration.sum")
mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9}
traffic = {}
for rname, key in (("full", "cfg2/hw/rgba32f"), ("full_cfg5", "cfg5/hw/rgba32f"),
                   ("full_bwd", "cfg4/k_raster_bwd")):
    rep = src / f"{rname}.ncu-rep"
    if not rep.exists():
        continue
    raw = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv", "--metrics", M],
                         capture_output=True, text=True).stdout
    rows = list(csv.DictReader(io.StringIO(raw)))
    for r in rows[1:]:
        want = "k_raster_bwd" if "bwd" in rname else "k_raster_fwd"
        if want not in r["Kernel Name"]:
            continue
        tb = (float(r["dram__bytes_read.sum"]) * mult[rows[0]["dram__bytes_read.sum"]] +
              float(r["dram__bytes_write.sum"]) * mult[rows[0]["dram__bytes_write.sum"]])
        traffic[key] = int(tb)
        traffic[key.replace("/", "_") + "_ncu"] = {
            "kernel": f"{want} ({key})",
            "duration_us": float(r["gpu__time_duration.sum"]) * {
                "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "ns": 1e-3, "us": 1.0, "ms": 1e3}[rows[0]["gpu__time_duration.sum"]],
            "l1tex_throughput_pct": float(r["l1tex__throughput.avg.pct_of_peak_sustained_active"]),
            "tex_data_pipe_pct": float(r["l1tex__data_pipe_tex_wavefronts.avg.pct_of_peak_sustained_elapsed"]),
            "dram_throughput_pct": float(r["dram__cycles_active.avg.pct_of_peak_sustained_elapsed"])}
        break
if "cfg2/hw/rgba32f" in traffic:
    traffic["ncu"] = traffic["cfg2_hw_rgba32f_ncu"]
(dst / "traffic.json").write_text(json.dumps(traffic, indent=1) + "\n")
print(json.dumps(traffic, indent=1))
