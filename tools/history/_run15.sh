timeout 900 python -m pytest tests/test_gpu_tiers.py -x -q --timeout 300 > gpurun_out/r15_tiers.log 2>&1; echo tiers=$?
tail -2 gpurun_out/r15_tiers.log
python tools/diff_libs.py 4 tools/_ref/libevoke_ref.so
python tools/diff_libs.py 3 tools/_ref/libevoke_ref.so
for c in 4 2 3; do echo "== config $c"; EVOKE_DEBUG=1 timeout 300 python tools/dev_timing.py $c 1 --serial 2>&1 | grep -E "wall|hub_local|hub items|cliques_k4"; done
