set -x
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 --durations=15 > gpurun_out/r2_pytest.log 2>&1; echo pytest=$?
tail -40 gpurun_out/r2_pytest.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/r2_bench.log 2>&1; echo bench=$?
tail -c 4000 gpurun_out/r2_bench.log
