#!/bin/bash
# Round-2 evidence on the GPU box: bench lines for every workload, the launch list of the default
# bench command (c4), ncu --set full captures of the c4 spreading / interpolation kernels; with
# NCU_SMALL=1 (a second call: gpurun merges back at most 64 MiB) the c3 2-D strip kernels and DFT
# passes and the c2 kernels.
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
if [ "${BENCH:-1}" = 1 ]; then
timeout 900 python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "bench default exit $?"
for c in ${CONFIGS-c1 c2 c3 c3r x4}; do
  timeout 600 python bench.py --config $c --steps 50 --warmup 5 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "bench $c exit $?"
done
for c in ${OBJ_CONFIGS-c5 c5a g5}; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "bench $c exit $?"
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err; echo "reference exit $?"
fi
if [ "${NCU:-1}" = 1 ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv \
      python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1; echo "ncu launches exit $?"
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_spread_v5|k_interp_mma" -s 2 -c 3 \
      -o gpurun_out/prof_c4 -f python tools/prof_run.py --config c4 --calls 2 > gpurun_out/ncu_c4.log 2>&1; echo "ncu full exit $?"
fi
if [ "${NCU_SMALL:-0}" = 1 ]; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_spread|k_interp|k_dft" -s 6 -c 6 \
      -o gpurun_out/prof_c3 -f python tools/prof_run.py --config c3 --calls 2 > gpurun_out/ncu_c3.log 2>&1; echo "ncu c3 exit $?"
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_spread|k_plane|k_pencil|k_interp|k_epilogue" -s 6 -c 6 \
      -o gpurun_out/prof_c2 -f python tools/prof_run.py --config c2 --calls 3 > gpurun_out/ncu_c2.log 2>&1; echo "ncu c2 exit $?"
fi
