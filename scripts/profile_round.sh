#!/bin/bash
# One GPU call that regenerates the round's measured evidence into gpurun_out/prof/.
# usage: bash scripts/profile_round.sh [quick]
set -u
O=gpurun_out/prof; mkdir -p $O
run() { local name=$1; shift; timeout ${TMO:-300} "$@" > $O/$name.json 2> $O/$name.err; echo "$name rc=$?"; tail -c 300 $O/$name.json; echo; }
run bench python bench.py --steps 100 --warmup 10
run train python bench.py --workload train --steps 20 --warmup 3
if [ "${1:-}" != "quick" ]; then
  TMO=600 run cfg3 python bench.py --config cfg3 --steps 3 --warmup 1 --no-cpu-baseline
  TMO=900 run cfg5 python bench.py --config cfg5 --steps 20 --warmup 3 --no-cpu-baseline
  for T in 4 8 16; do for s in flat verify hw; do
    run t3_${s}_T$T python bench.py --texture-res $T --sampler $s --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 5
  done; done
  run hw16f python bench.py --texel-format rgba16f --steps 100 --warmup 10 --no-cpu-baseline
fi
F5="--splats 2000000 --texture-res 16 --width 1920 --height 1080"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/train_launches.csv \
  python scripts/profile_train.py 3 > $O/ncu_train.log 2>&1; echo "ncu train list rc=$?"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
  python scripts/profile_frame.py --frames 3 > $O/ncu_list.log 2>&1; echo "ncu list rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg5.csv \
  python scripts/profile_frame.py --frames 3 $F5 > $O/ncu_list5.log 2>&1; echo "ncu list cfg5 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_raster_fwd|k_preprocess|k_shade|k_dup_tx|k_onesweep" -s 18 -c 9 \
  -o $O/full python scripts/profile_frame.py --frames 3 > $O/ncu_full.log 2>&1; echo "ncu full rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_raster_fwd" -s 1 -c 1 \
  -o $O/full_cfg5 python scripts/profile_frame.py --frames 3 $F5 > $O/ncu_full5.log 2>&1; echo "ncu full cfg5 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_raster_bwd" -s 1 -c 1 \
  -o $O/full_bwd python scripts/profile_train.py 3 > $O/ncu_bwd.log 2>&1; echo "ncu full bwd rc=$?"
