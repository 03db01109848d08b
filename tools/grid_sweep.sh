python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for combo in ${COMBOS:-"148 148"}; do
  set -- $combo
  echo "== c5 $1 pair $2"
  EVOKE_C5_HG=$1 EVOKE_PAIR_HG=$2 python tools/dev_timing.py 2 15 | grep wall
done
