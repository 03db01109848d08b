for c in 4 2; do
for env in "EVOKE_C5_SMID_REC=0" "EVOKE_C5_SHCAP=512 EVOKE_C5_SMID_REC=0" "EVOKE_C5_LIGHT_REC=256 EVOKE_C5_SHCAP=512" "EVOKE_C5_LIGHT_REC=256 EVOKE_C5_SHCAP=512 EVOKE_C5_SMID_REC=0" "EVOKE_C5_LIGHT_REC=128"; do
  echo "== config $c $env"
  env $env EVOKE_DEBUG=1 timeout 300 python tools/dev_timing.py $c 2 --serial 2>&1 | grep -E "cycles5|c5 endpoints" | sort | uniq
done; done
