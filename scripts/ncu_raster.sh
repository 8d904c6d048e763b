#!/bin/bash
# One ncu --set full capture (source-level) of k_raster_fwd at cfg2 -> gpurun_out/$1.ncu-rep
# usage: bash scripts/ncu_raster.sh NAME [profile_frame.py args]
set -u
name=$1; shift
mkdir -p gpurun_out
timeout 300 python scripts/profile_frame.py --frames 3 "$@" > gpurun_out/$name.plain.log 2>&1 || { echo "plain run failed"; tail gpurun_out/$name.plain.log; exit 1; }
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"${KERNEL:-k_raster_fwd}" -s 1 -c 1 \
  -o gpurun_out/$name python scripts/profile_frame.py --frames 3 "$@" > gpurun_out/$name.ncu.log 2>&1
echo "ncu rc=$?"
