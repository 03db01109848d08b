# final state of round 2: smoke, the full GPU suite (config-5 laps shown), the bench
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_l.log 2>&1; echo smoke=$?
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_l.log 2>&1; echo bench=$?
tail -c 1500 gpurun_out/bench_l.log | head -c 500
timeout 2000 python -m pytest tests -m gpu -x -q -s --durations=12 > gpurun_out/pytest_gpu_l.log 2>&1; echo pytest=$?
grep "config5\]" gpurun_out/pytest_gpu_l.log | cut -c1-330
tail -16 gpurun_out/pytest_gpu_l.log | cut -c1-200
