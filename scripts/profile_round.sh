#!/bin/bash
# One GPU call that regenerates the round's measured evidence into gpurun_out/prof/.
# usage: bash scripts/profile_round.sh [quick]
set -u
O=gpurun_out/prof; mkdir -p $O
run() { local name=$1; shift; timeout ${TMO:-300} "$@" > $O/$name.json 2> $O/$name.err; echo "$name rc=$?"; tail -c 400 $O/$name.json; echo; }
run bench python bench.py --steps 100 --warmup 10
run train python bench.py --workload train --steps 20 --warmup 3 --no-cpu-baseline
if [ "${1:-}" != "quick" ]; then
  run cfg3 python bench.py --config cfg3 --steps 30 --warmup 5 --no-cpu-baseline
  TMO=900 run cfg5 python bench.py --config cfg5 --steps 20 --warmup 3 --no-cpu-baseline
  for T in 4 8 16; do for s in flat verify hw; do
    run t3_${s}_T$T python bench.py --texture-res $T --sampler $s --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 5
  done; done
  run hw16f python bench.py --texel-format rgba16f --steps 100 --warmup 10 --no-cpu-baseline
fi
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/train_launches.csv \
  python scripts/profile_train.py 3 > $O/ncu_train.log 2>&1; echo "ncu train list rc=$?"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 3 > $O/ncu_list.log 2>&1; echo "ncu list rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_raster_fwd|k_preprocess|k_shade" -s 10 -c 3 \
  -o $O/full python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 3 > $O/ncu_full.log 2>&1; echo "ncu full rc=$?"
