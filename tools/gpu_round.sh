#!/bin/bash
# One GPU session: parity tests, bench lines for every config, ncu launch list (c2) and a full
# capture of the dominant kernel (c4).  Output under gpurun_out/.
set -u
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest_gpu exit $?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo "bench c2 exit $?"
CONFIGS="${CONFIGS:-c1 c3 c4 c5}" STEPS=30 bash tools/run_bench.sh > gpurun_out/bench_all.txt 2>&1
if [ "${NCU:-1}" = 1 ]; then
  timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/plain.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv \
      python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
  timeout 300 python tools/prof_run.py --config c4 --calls 2 > gpurun_out/plain_c4.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_spread|k_interp" -s 2 -c 4 \
      -o gpurun_out/prof_c4 python tools/prof_run.py --config c4 --calls 2 > gpurun_out/ncu_full.log 2>&1
fi
echo done
