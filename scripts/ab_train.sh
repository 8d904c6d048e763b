for v in "$@"; do
  TSB_LIB=paper_2506_13348_b200/libtsb$v.so timeout 600 python bench.py --workload train --steps 30 --warmup 3 --no-cpu-baseline --no-numpy-reference > gpurun_out/b.json 2>gpurun_out/b.err || tail -3 gpurun_out/b.err
  python -c "import json;d=json.loads(open('gpurun_out/b.json').read().strip().splitlines()[-1]);print('v$v',d['value'],d['ms_per_step'],d['e2e']['value'],d['roofline']['k8_ms'])"
done
