# developer: bench.py ms_per_step under each env setting in $SETTINGS (space-separated VAR=VAL[,VAR=VAL])
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for st in $SETTINGS; do
  for r in $(seq ${REPS:-2}); do
    echo "== $st $(env $(echo $st | tr ',' ' ') python bench.py --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],3))')"
  done
done
