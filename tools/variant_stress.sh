# developer: determinism stress of each prebuilt library variants/*.so
for so in variants/*.so; do
  cp "$so" paper_1911_10616_b200/libevoke.so
  echo "== $so"
  timeout 300 python tools/stress_determinism.py ${CFG:-2} ${REPS:-16} $EXTRA 2>&1 | tail -1
done
