set -x
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/r1_pytest.log 2>&1; echo pytest=$?
tail -5 gpurun_out/r1_pytest.log
for c in 4 2; do
  timeout 300 python tools/dev_timing.py $c 3 > gpurun_out/r1_t$c.log 2>&1
  EVOKE_DEBUG=1 timeout 300 python tools/dev_timing.py $c 1 --serial > gpurun_out/r1_s$c.log 2>&1
done
