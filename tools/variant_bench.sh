# developer: bench.py ms_per_step (mean of timed steps, L2 flushed) per library variant
for so in variants/*.so; do
  cp "$so" paper_1911_10616_b200/libevoke.so
  for r in $(seq ${REPS:-2}); do
    echo "== $so $(python bench.py --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],3), round(d["e2e"]["value"]/1e6,2))')"
  done
done
