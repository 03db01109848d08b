for env in "X=1" "EVOKE_C5_MBPS=16" "EVOKE_C5_MBPS=16 EVOKE_C5_SHCAP=64 EVOKE_C5_LBPS=8" "EVOKE_C5_MBPS=16 EVOKE_C5_SHCAP=128 EVOKE_C5_LBPS=5" "EVOKE_C5_MBPS=16 EVOKE_C5_SHCAP=64 EVOKE_C5_LBPS=6"; do
  echo "== config 4 $env"
  env $env timeout 300 python tools/dev_timing.py 4 2 --serial 2>&1 | grep -E "cycles5" 
done
