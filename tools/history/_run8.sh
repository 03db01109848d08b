timeout 900 python -m pytest tests/test_gpu_tiers.py -x -q --timeout 300 > gpurun_out/r8_tiers.log 2>&1; echo tiers=$?
tail -3 gpurun_out/r8_tiers.log
python tools/diff_libs.py 2 tools/_ref/libevoke_ref.so
python tools/diff_libs.py 4 tools/_ref/libevoke_ref.so
for c in 2 4 3; do
  echo "== config $c serial"; EVOKE_DEBUG=1 timeout 300 python tools/dev_timing.py $c 2 --serial 2>&1 | grep -E "wall|pair_pass|cycles5|hub_local|c5 endpoints" | sort | uniq
  echo "== config $c default"; timeout 300 python tools/dev_timing.py $c 3 | grep -E "wall"
done
