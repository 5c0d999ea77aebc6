set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -k objective > gpurun_out/pytest_obj.log 2>&1; echo "exit $?" >> gpurun_out/pytest_obj.log
timeout 600 python bench.py --config c5 --steps 5 --warmup 3 > gpurun_out/bench_c5_obj.json 2> gpurun_out/bench_c5_obj.err
echo done
