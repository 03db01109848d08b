# developer: quick parity subset, then per-pass timings of configs (A/B of an env knob: AB_ENV)
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q -k "${TESTK:-small or sparse or tiled or tier or shard or csr}" > gpurun_out/pytest_q.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_q.log
for c in ${CFGS:-4 3}; do
  timeout 600 python tools/dev_timing.py $c 3 --serial > gpurun_out/ab_$c.log 2>&1; echo t$c=$?
  grep "wall\|pair_pass\|hub_local\|cycles5\|cliques\|gather\|combine" gpurun_out/ab_$c.log
  if [ -n "$AB_ENV" ]; then
    env $AB_ENV timeout 600 python tools/dev_timing.py $c 3 --serial > gpurun_out/ab_${c}_b.log 2>&1; echo t${c}b=$?
    grep "wall\|pair_pass\|hub_local\|cycles5\|cliques\|gather\|combine" gpurun_out/ab_${c}_b.log
  fi
done
