# quick GPU iteration: build, GPU parity suite, one bench line (no CPU baseline)
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests -m gpu -x -q --timeout 150 ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -30 gpurun_out/pytest_gpu.log
timeout 240 python bench.py --steps 5 --warmup 3 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench.log 2>&1; echo bench=$?
tail -c 2500 gpurun_out/bench.log
if [ -n "$LAUNCHES" ]; then
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo ncu=$?
  python tools/launch_summary.py gpurun_out/launches.csv | head -25
fi
