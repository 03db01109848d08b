set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for r in 1 2; do
  timeout 300 python tools/dev_timing.py 4 4 --serial 2>&1 | grep -E "wall|cycles5|pair_pass"
  EVOKE_C5_BIN_ORDER=1 timeout 300 python tools/dev_timing.py 4 4 --serial 2>&1 | grep -E "wall|cycles5|pair_pass"
done
