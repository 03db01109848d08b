timeout 900 python -m pytest tests/test_gpu_tiers.py -x -q --timeout 300 > gpurun_out/r20_t.log 2>&1; echo tests=$?
tail -1 gpurun_out/r20_t.log
python tools/diff_libs.py 2 tools/_ref/libevoke_ref.so 2>&1 | tail -2
python tools/diff_libs.py 3 tools/_ref/libevoke_ref.so 2>&1 | tail -2
for env in "X=1" "EVOKE_PAIR_NO_DWORK=1"; do
for c in 2 4 3; do echo "== config $c $env"; env $env EVOKE_DEBUG=1 timeout 300 python tools/dev_timing.py $c 1 --serial 2>&1 | grep -E "wall|pair_pass|pair tiers" | sort | uniq; done; done
echo "== config 2 concurrent"; timeout 300 python tools/dev_timing.py 2 5 2>&1 | grep -E "wall|pair_pass"
