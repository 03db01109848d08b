set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q -k "small or sparse or dense or tiled or tier or closed or config1 or degenerate or shard or csr" > gpurun_out/pytest_q.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_q.log
for i in 1 2; do
timeout 600 python tools/dev_timing.py 4 3 --serial > gpurun_out/f4_$i.log 2>&1; echo t4=$?
grep "wall\|pair_pass\|cycles5\|gather\|combine" gpurun_out/f4_$i.log
EVOKE_LIB_PATH=variants/libevoke_mb1.so timeout 600 python tools/dev_timing.py 4 3 --serial > gpurun_out/f4_mb1_$i.log 2>&1; echo mb1=$?
grep "wall\|pair_pass\|cycles5\|gather" gpurun_out/f4_mb1_$i.log
done
timeout 600 python tools/dev_timing.py 3 2 --serial > gpurun_out/f3.log 2>&1; echo t3=$?
grep "wall\|pair_pass\|hub_local\|cycles5\|cliques\|gather" gpurun_out/f3.log
