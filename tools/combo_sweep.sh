# developer: concurrent wall time per library variant and heavy-grid combination
for so in variants/*.so; do
  cp "$so" paper_1911_10616_b200/libevoke.so
  for c in $COMBOS; do
    a=${c%_*}; b=${c#*_}
    echo "== $so c5 $a pair $b"
    EVOKE_C5_HG=$a EVOKE_PAIR_HG=$b timeout 300 python tools/dev_timing.py 2 ${K:-15} | grep wall
  done
done
