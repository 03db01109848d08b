# round-2 status check at the current code: smoke, GPU suite, bench, configs 3/5 serial timing
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1800 python -m pytest tests -m gpu -x -q --durations=25 > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -40 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1; echo bench=$?
tail -c 4000 gpurun_out/bench.log
timeout 300 python tools/dev_timing.py 3 2 --serial > gpurun_out/timing3.log 2>&1; echo t3=$?
tail -20 gpurun_out/timing3.log
timeout 900 python tools/dev_timing.py 5 1 --warm 0 --serial > gpurun_out/timing5.log 2>&1; echo t5=$?
tail -20 gpurun_out/timing5.log
