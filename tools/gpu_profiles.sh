#!/bin/bash
# Round evidence: bench lines for every config (default bench = c2 with cpu_baseline), the ncu
# launch list of the default bench command, and full ncu captures of the top kernels (c2, c4).
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench exit $?"
for c in c1 c3 c4 c5; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 3 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "bench $c exit $?"
done
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err; echo "ref exit $?"
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo "ncu launch exit $?"
timeout 300 python tools/prof_run.py --config c2 --calls 3 > gpurun_out/plain_c2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_spread|k_plane|k_pencil|k_dft|k_interp|k_epilogue" -s 6 -c 6 \
    -o gpurun_out/prof_c2 -f python tools/prof_run.py --config c2 --calls 3 > gpurun_out/ncu_c2.log 2>&1; echo "ncu c2 exit $?"
timeout 300 python tools/prof_run.py --config c4 --calls 2 > gpurun_out/plain_c4.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_spread|k_interp" -s 2 -c 2 \
    -o gpurun_out/prof_c4 -f python tools/prof_run.py --config c4 --calls 2 > gpurun_out/ncu_c4.log 2>&1; echo "ncu c4 exit $?"
echo done
