timeout 900 python -m pytest tests/test_gpu_tiers.py tests/test_gpu_parity.py -x -q --timeout 300 -k "not config5 and not config4 and not eight" > gpurun_out/r19_t.log 2>&1; echo tests=$?
tail -2 gpurun_out/r19_t.log
python tools/diff_libs.py 4 tools/_ref/libevoke_ref.so 2>&1 | tail -3
for env in "X=1" "EVOKE_TMP_SKIP=1" "EVOKE_TMP_SKIP=2" "EVOKE_TMP_SKIP=3"; do echo "== config 2 $env"; env $env timeout 300 python tools/dev_timing.py 2 3 --serial 2>&1 | grep -E "wall|pair_pass"; done
echo "== config 4"; timeout 300 python tools/dev_timing.py 4 2 --serial 2>&1 | grep -E "wall|cliques|pair_pass"
