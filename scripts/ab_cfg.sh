# usage: CFG="--config cfg5 --steps 20 --warmup 3" ab_cfg.sh variants...
for v in "$@"; do
  TSB_LIB=paper_2506_13348_b200/libtsb$v.so timeout 600 python bench.py $CFG --no-cpu-baseline > gpurun_out/b.json 2>gpurun_out/b.err || tail -3 gpurun_out/b.err
  python -c "import json;d=json.loads(open('gpurun_out/b.json').read().strip().splitlines()[-1]);print('v$v',d['value'],d['e2e']['value'],d['breakdown_ms'])"
done
