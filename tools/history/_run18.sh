timeout 1500 python -m pytest tests -m gpu -q --timeout 900 --durations=8 > gpurun_out/r18_pytest.log 2>&1; echo pytest=$?
tail -14 gpurun_out/r18_pytest.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r18_bench.log 2>&1; echo bench=$?
tail -c 5000 gpurun_out/r18_bench.log
