timeout 900 python -m pytest tests/test_gpu_tiers.py -x -q --timeout 300 > gpurun_out/r12_tiers.log 2>&1; echo tiers=$?
tail -3 gpurun_out/r12_tiers.log
python tools/diff_libs.py 4 tools/_ref/libevoke_ref.so
python tools/diff_libs.py 3 tools/_ref/libevoke_ref.so
for env in "X=1" "EVOKE_PAIR_NO_HOT=1"; do echo "== config 2 $env"; env $env timeout 300 python tools/dev_timing.py 2 3 --serial 2>&1 | grep -E "wall|pair_pass"; done
echo "== config 4"; timeout 300 python tools/dev_timing.py 4 3 2>&1 | grep -v "h2d\|d2h"
echo "== config 3"; timeout 300 python tools/dev_timing.py 3 1 2>&1 | grep -v "h2d\|d2h"
