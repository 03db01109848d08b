timeout 900 python -m pytest tests/test_gpu_tiers.py -x -q --timeout 300 > gpurun_out/r17_tiers.log 2>&1; echo tiers=$?
tail -2 gpurun_out/r17_tiers.log
python tools/diff_libs.py 4 tools/_ref/libevoke_ref.so 2>&1 | tail -3
python tools/diff_libs.py 2 tools/_ref/libevoke_ref.so 2>&1 | tail -3
for c in 4; do echo "== config $c"; timeout 300 python tools/dev_timing.py $c 2 --serial 2>&1 | grep -v "h2d\|d2h"; done
