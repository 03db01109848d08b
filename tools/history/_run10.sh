for c in 4 2; do
for env in "EVOKE_C5_SMID_REC=0" "EVOKE_C5_SMID_REC=0 EVOKE_C5_SHCAP=128 EVOKE_C5_LBPS=5" "EVOKE_C5_SMID_REC=0 EVOKE_C5_SHCAP=64 EVOKE_C5_LBPS=8" "EVOKE_C5_SMID_REC=0 EVOKE_C5_MBPS=8" "EVOKE_C5_SMID_REC=0 EVOKE_C5_MBPS=12" "EVOKE_C5_SMID_REC=0 EVOKE_C5_LIGHT_WORK=4096"; do
  echo "== config $c $env"
  env $env timeout 300 python tools/dev_timing.py $c 2 --serial 2>&1 | grep -E "cycles5" 
done; done
