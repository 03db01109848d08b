# developer A/B: dev_timing of config ${CFG:-2} with each prebuilt library variants/*.so
# (copied over the package library in this scratch copy of the repo)
for so in variants/*.so; do
  cp "$so" paper_1911_10616_b200/libevoke.so
  echo "== $so"
  timeout 300 python tools/dev_timing.py ${CFG:-2} ${K:-7} $EXTRA 2>&1 | grep -E "wall|$SHOW"
done
