for c in 2 4; do
for env in "X=1" "EVOKE_PAIR_NO_HOT=1" "EVOKE_C5_LIGHT_WORK=4096" "EVOKE_C5_LIGHT_WORK=2048" "EVOKE_C5_LIGHT_WORK=1024" "EVOKE_C5_LIGHT_WORK=2048 EVOKE_C5_MID_WORK=16384"; do
  echo "== config $c $env"
  env $env timeout 300 python tools/dev_timing.py $c 2 --serial | grep -E "wall|pair_pass|cycles5"
done
echo "== config $c concurrent"
timeout 300 python tools/dev_timing.py $c 3 | grep -E "wall"
done
python tools/diff_libs.py 2 tools/_ref/libevoke_ref.so
