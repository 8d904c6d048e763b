"""Summarise gpurun_out/sweep/*.json written by scripts/sweep.sh."""
import glob
import json
import os

for f in sorted(glob.glob('gpurun_out/sweep/*.json')):
    try:
        d = json.load(open(f))
    except Exception as e:  # noqa: BLE001
        print(os.path.basename(f), 'ERR', e)
        continue
    print(f"{os.path.basename(f)[:-5]:24s} {d['value']:9.2f} {d.get('unit', '')[:10]} "
          f"{d.get('breakdown_ms')} E={d.get('entries_per_frame')}")
