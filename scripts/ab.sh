# usage: ab.sh variants... ; runs bench for each variant twice (interleaved)
for rep in ${REPS:-1 2}; do for v in "$@"; do
  TSB_LIB=paper_2506_13348_b200/libtsb$v.so timeout 120 python bench.py --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/b.json 2>gpurun_out/b.err || tail -3 gpurun_out/b.err
  python -c "import json;d=json.load(open('gpurun_out/b.json'));print('v$v',d['value'],d['breakdown_ms'])"
done; done
