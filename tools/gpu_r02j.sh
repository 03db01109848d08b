# the parity file in suite order with the config-5 lap times shown (-s): where its minutes go
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 2400 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -s --durations=12 > gpurun_out/pytest_parity_s.log 2>&1; echo pytest=$?
grep "config5\]" gpurun_out/pytest_parity_s.log
tail -18 gpurun_out/pytest_parity_s.log
