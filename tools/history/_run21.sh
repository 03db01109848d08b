timeout 900 python -m pytest tests/test_gpu_tiers.py -x -q --timeout 300 > gpurun_out/r21_t.log 2>&1; echo tests=$?
tail -1 gpurun_out/r21_t.log
python tools/diff_libs.py 4 tools/_ref/libevoke_ref.so 2>&1 | tail -2
python tools/diff_libs.py 2 tools/_ref/libevoke_ref.so 2>&1 | tail -2
for c in 4 2; do echo "== config $c"; timeout 300 python tools/dev_timing.py $c 2 --serial 2>&1 | grep -E "wall|cycles5"; done
