set -x
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 -k "not config5" > gpurun_out/r3_pytest.log 2>&1; echo pytest=$?
tail -15 gpurun_out/r3_pytest.log
for c in 4 2; do
  timeout 300 python tools/dev_timing.py $c 3 > gpurun_out/r3_t$c.log 2>&1
  EVOKE_DEBUG=1 EVOKE_C5_HIST=1 timeout 300 python tools/dev_timing.py $c 1 --serial > gpurun_out/r3_s$c.log 2>&1
done
timeout 300 python tools/dev_timing.py 3 1 --serial > gpurun_out/r3_s3.log 2>&1
