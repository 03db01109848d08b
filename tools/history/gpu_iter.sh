# quick iteration: build, selected GPU tests (PYTEST_K), timings of CONFIGS (serial, EVOKE_DEBUG)
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
if [ -n "$PYTEST_K" ]; then
timeout 900 python -m pytest tests -m gpu -x -q -k "$PYTEST_K" > gpurun_out/pytest_iter.log 2>&1; echo pytest=$?
tail -15 gpurun_out/pytest_iter.log
fi
for c in ${CONFIGS:-3}; do
  EVOKE_DEBUG=1 timeout 900 python tools/dev_timing.py $c ${REPS:-2} --serial > gpurun_out/timing_$c.log 2>&1; echo t$c=$?
  grep -v "^\[evoke\] \(pair\|c5\) \(mid\|dense\|light\|heavy\)" gpurun_out/timing_$c.log | tail -22
done
if [ -n "$BENCH" ]; then
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_iter.log 2>&1; echo bench=$?
tail -c 1500 gpurun_out/bench_iter.log
fi
