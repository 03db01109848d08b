set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q -k "small or sparse or dense or tiled or tier or closed or config1 or degenerate or shard or csr or four or noninduced" > gpurun_out/pytest_q.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_q.log
timeout 600 python tools/dev_timing.py 4 3 --serial > gpurun_out/g4.log 2>&1; echo t4=$?
cat gpurun_out/g4.log
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --extra-config 0"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches4.csv $B > gpurun_out/ncu_launch4.log 2>&1; echo launches=$?
python tools/launch_summary.py gpurun_out/launches4.csv 4 | head -45
