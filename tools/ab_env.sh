#!/bin/bash
# A/B of an environment switch on the bench lines: AB_VAR=AKM_PDL CONFIGS="c1 c2" bash tools/ab_env.sh
set -u
mkdir -p gpurun_out
for c in ${CONFIGS-c1 c2 c3 c4}; do
  for v in ${AB_VALS-1 0}; do
    env ${AB_VAR}=$v timeout 600 python bench.py --config $c --steps ${STEPS:-50} --warmup 5 --no-cpu-baseline > gpurun_out/ab_${c}_$v.json 2> gpurun_out/ab_${c}_$v.err
    python - <<PY || tail -5 gpurun_out/ab_${c}_$v.err
import json
d=json.load(open('gpurun_out/ab_${c}_$v.json'))
print('$c ${AB_VAR}=$v', '%.4f ms'%d['ms_per_step'], 'e2e %.3e'%d['e2e']['value'], {k:round(v,4) for k,v in d['stages_ms_per_step'].items()})
PY
  done
done
