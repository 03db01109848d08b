for env in "X=1" "EVOKE_PAIR_LIGHT_MAX=0" "EVOKE_PAIR_LIGHT_MAX=0 EVOKE_PAIR_MIDS_MAX=0" "EVOKE_PAIR_LIGHT_MAX=128"; do echo "== config 2 $env"; env $env EVOKE_DEBUG=1 timeout 300 python tools/dev_timing.py 2 3 --serial 2>&1 | grep -E "wall|pair_pass|phases|pair tiers" | sort | uniq -c | sort -rn | head -5; done
for env in "X=1" "EVOKE_PAIR_LIGHT_MAX=0"; do echo "== config 4 $env"; env $env timeout 300 python tools/dev_timing.py 4 2 --serial 2>&1 | grep -E "wall|pair_pass"; done
python tools/diff_libs.py 2 tools/_ref/libevoke_ref.so
