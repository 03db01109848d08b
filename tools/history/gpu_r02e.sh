set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q -k "small or sparse or dense or tiled or tier or closed or config1 or degenerate or shard or csr" > gpurun_out/pytest_q.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_q.log
timeout 600 python tools/dev_timing.py 4 3 --serial > gpurun_out/e4.log 2>&1; echo t4=$?
grep "wall\|pair_pass\|cycles5\|gather\|combine" gpurun_out/e4.log
for v in lb8 lb6; do
  EVOKE_LIB_PATH=variants/libevoke_$v.so timeout 600 python tools/dev_timing.py 4 3 --serial > gpurun_out/e4_$v.log 2>&1; echo $v=$?
  grep "wall\|cycles5" gpurun_out/e4_$v.log
done
EVOKE_DEBUG=1 timeout 900 python tools/dev_timing.py 5 1 --warm 0 --serial > gpurun_out/e5.log 2>&1; echo t5=$?
grep "units\|c5 big\|endpoints\|wall\|pair_pass\|hub_local\|cycles5\|cliques\|gather\|steps" gpurun_out/e5.log
