set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q -k "pair or c5 or small_random or sparse_medium or config3" > gpurun_out/pytest_iter.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_iter.log
for c in 2 4 3; do timeout 300 python tools/dev_timing.py $c 4 --serial 2>&1 | grep -E "wall|pair_pass|cycles5"; EVOKE_PAIR_HOT=0 timeout 300 python tools/dev_timing.py $c 4 --serial 2>&1 | grep -E "wall|pair_pass"; done
