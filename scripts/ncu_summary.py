"""Summarise ncu outputs into profiles/ (run here, no GPU needed).

    python scripts/ncu_summary.py LAUNCHES.csv REPORT.ncu-rep OUT.md

LAUNCHES.csv: `ncu --metrics gpu__time_duration.sum --csv --log-file` output.
REPORT.ncu-rep: a `--set full` capture. Writes per-kernel launch times of the
last frame and the key throughput / stall metrics of each profiled kernel.
"""
import csv
import io
import subprocess
import sys
from collections import OrderedDict

KEYS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_tex.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum",
    "smsp__thread_inst_executed_per_inst_executed.ratio",
    "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size",
]
STALLS = ["long_scoreboard", "wait", "short_scoreboard", "barrier", "branch_resolving",
          "not_selected", "selected", "mio_throttle", "math_pipe_throttle", "lg_throttle",
          "tex_throttle", "no_instruction", "dispatch_stall"]


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    out = []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            out.append((int(d["ID"]), d["Kernel Name"], float(d["Metric Value"])))
    return out


def raw(report):
    txt = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    return [dict(zip(hdr, r)) for r in rows[2:]], dict(zip(hdr, units))


def main(lpath, rpath, out):
    lines = ["# ncu summary", ""]
    ls = launches(lpath)
    # last frame: from the last k_preprocess to the end
    # the last complete frame: a k_preprocess .. k_shade run of our kernels (the
    # bench's own torch diagnostics between frames, at::*, are not frame work)
    ls = [x for x in ls if not x[1].lstrip("void ").startswith("at::")]
    starts = [i for i, (_, n, _) in enumerate(ls) if "k_preprocess" in n]
    frame = ls
    for s in reversed(starts):
        ends = [i for i, (_, n, _) in enumerate(ls[s:]) if "k_shade" in n]
        if ends:
            frame = ls[s:s + ends[0] + 1]
            break
    tot = sum(t for _, _, t in frame)
    lines += ["## Launch list of one cfg2 frame (cold-cache, serialised; compare shares)", "",
              "| kernel | ns | share |", "|---|---:|---:|"]
    agg = OrderedDict()
    for _, n, t in frame:
        key = n.split("(")[0].replace("void ", "")[:60]
        if key in agg and not key.startswith("tsb::"):
            key = key + " #" + str(sum(1 for k in agg if k.startswith(key)) + 1)
        agg[key] = agg.get(key, 0.0) + t
    for k, t in agg.items():
        lines.append(f"| `{k}` | {t:.0f} | {100 * t / tot:.1f}% |")
    lines += [f"| **total** | {tot:.0f} | 100% |", ""]
    recs, units = raw(rpath)
    for r in recs:
        name = r.get("Kernel Name", "?").split("(")[0]
        lines += [f"## `{name}` (ncu --set full, id {r.get('ID')})", "",
                  "| metric | value |", "|---|---:|"]
        for k in KEYS:
            if k in r:
                lines.append(f"| {k} ({units.get(k, '')}) | {r[k]} |")
        st = []
        for s in STALLS:
            k = f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio"
            if k in r:
                try:
                    st.append((float(r[k]), s))
                except ValueError:
                    pass
        st.sort(reverse=True)
        lines.append("| stall cycles / issued inst | " +
                     ", ".join(f"{s} {v:.2f}" for v, s in st[:6]) + " |")
        lines.append("")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main(*sys.argv[1:4])
