# developer sweep: dev_timing of config ${CFG:-2} under each value of env knob $KNOB
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for v in $VALUES; do
  echo "== $KNOB=$v"
  env $KNOB=$v timeout 300 python tools/dev_timing.py ${CFG:-2} ${K:-7} $EXTRA 2>&1 | grep -E "wall|$SHOW"
done
