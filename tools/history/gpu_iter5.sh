# developer: c5 tier tests, then config 5 (and 3) serial timing with the unit timers
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_tiers.py -x -q -k "${TESTK:-c5 or giant}" > gpurun_out/pytest_tiers.log 2>&1; echo pytest=$?
tail -5 gpurun_out/pytest_tiers.log
for c in ${CFGS:-5 3}; do
  EVOKE_DEBUG=1 timeout 900 python tools/dev_timing.py $c 1 --warm 0 --serial > gpurun_out/it$c.log 2>&1; echo t$c=$?
  grep "units\|c5 big\|endpoints\|wall\|pair_pass\|hub_local\|cycles5\|cliques" gpurun_out/it$c.log
done
