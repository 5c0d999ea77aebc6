#!/bin/bash
# Iteration loop on the GPU box: parity tests, bench lines, optional ncu captures.
#   KEXPR="expr" CONFIGS="c2 c4" NCU_C4=1 NCU_C2=1 bash tools/gpu_iter.sh
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; cat gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -x -q ${KEXPR:+-k "$KEXPR"} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
for c in ${CONFIGS-c1 c2 c3 c4}; do
  timeout 600 python bench.py --config $c --steps ${STEPS:-30} --warmup 5 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  python - <<PY || tail -5 gpurun_out/bench_$c.err
import json
d=json.load(open('gpurun_out/bench_$c.json'))
print('$c', '%.4f ms'%d['ms_per_step'], '%.3e pts/s'%d['value'], {k:round(v,4) for k,v in d['stages_ms_per_step'].items()}, d['roofline']['kernel'], 'frac %.3f'%d['roofline']['frac'], 'bins', d['plan']['bin'])
PY
done
if [ "${NCU_C4:-0}" = 1 ]; then
  NC=${NCU_CFG:-c4}
  timeout 300 python tools/prof_run.py --config $NC --calls 2 > gpurun_out/plain_$NC.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${NCU_K:-k_spread|k_interp}" -s ${NCU_S:-2} -c ${NCU_N:-2} \
      -o gpurun_out/prof_$NC -f python tools/prof_run.py --config $NC --calls 2 > gpurun_out/ncu_$NC.log 2>&1
  tail -2 gpurun_out/ncu_$NC.log
fi
if [ "${NCU_C2:-0}" = 1 ]; then
  timeout 300 python tools/prof_run.py --config c2 --calls 3 > gpurun_out/plain_c2.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_" -s ${NCU2_S:-43} -c ${NCU2_N:-9} \
      -o gpurun_out/prof_c2 -f python tools/prof_run.py --config c2 --calls 3 > gpurun_out/ncu_c2.log 2>&1
  tail -2 gpurun_out/ncu_c2.log
fi
echo done
