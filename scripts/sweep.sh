#!/bin/bash
# usage: sweep.sh NAME "bench args" ...  -> gpurun_out/sweep/NAME.json per run
mkdir -p gpurun_out/sweep
while [ $# -gt 1 ]; do
  name=$1; args=$2; shift 2
  timeout ${TMO:-300} python bench.py $args --no-cpu-baseline --e2e-steps 3 > gpurun_out/sweep/$name.json 2> gpurun_out/sweep/$name.err
  echo "$name rc=$?"
done
